"""Key metrics of one ncu report (first kernel): pipes, stalls, dram bytes, instruction mix.

usage: python tools/ncu_summary.py rep.ncu-rep [cell_steps]
"""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread",
        "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
        "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
        "sm__cycles_elapsed.avg.per_second"]


def main(rep, cells=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(out.splitlines()))
    hdr, unit, val = r[0], r[1], r[2]
    d = dict(zip(hdr, val))
    u = dict(zip(hdr, unit))
    for k in KEYS:
        if k in d:
            print(f"{k:70s} {d[k]:>20s} {u[k]}")
    stalls = [(float(v.replace(',', '')), h) for h, v in d.items()
              if h.startswith("smsp__average_warp_latency_issue_stalled_") or
              (h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"))]
    for v, h in sorted(stalls, reverse=True)[:12]:
        print(f"  stall {h:80s} {v:8.3f}")
    if cells:
        cells = float(cells)
        fp = sum(float(d.get(k, "0").replace(',', '')) for k in
                 ("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
                  "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
                  "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"))
        ins = float(d["smsp__inst_executed.sum"].replace(',', ''))
        print(f"per cell-step: fp64 thread-ops {fp / cells:.1f}, warp-instructions {ins / cells:.2f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
