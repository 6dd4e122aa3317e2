"""DRAM traffic per launch of one kernel from an `ncu --set full` report ->
profiles/kp_traffic_<workload>.json (read by bench.py for roofline.traffic / fp64).

usage: python tools/ncu_traffic.py rep.ncu-rep kernel_regex out.json [workload cells_per_launch]

bench.py reads profiles/kp_traffic_<workload>.json: dram_bytes_per_cell scales
the capture (a 4096-member probe, tools/kp_probe.py) to the launch it times.
"""
import csv
import io
import json
import re
import subprocess
import sys


def main(rep, pattern, out, workload="config4", cells=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    tscale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}
    recs = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        if not re.search(pattern, d["Kernel Name"]):
            continue
        def val(k, table):
            return float(d[k].replace(",", "")) * table[units[hdr.index(k)]]
        recs.append({
            "kernel": d["Kernel Name"], "grid": d["Grid Size"], "block": d["Block Size"],
            "dram_read_bytes": val("dram__bytes_read.sum", scale),
            "dram_write_bytes": val("dram__bytes_write.sum", scale),
            "duration_ms": val("gpu__time_duration.sum", tscale),
            # the compute side of the roofline (K_P is fp64-issue bound)
            "fp64_pipe_pct": float(d.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                                         "nan").replace(",", "")),
            "issue_active_pct": float(d.get("smsp__issue_active.avg.pct_of_peak_sustained_active",
                                            "nan").replace(",", "")),
            # fp64 arithmetic (thread-level DADD + DMUL + DFMA per cycle, whole GPU)
            # against the pipe's peak (64 per clock per SM)
            "fp64_ops_per_cycle": sum(float(d.get(
                f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed", "0")
                .replace(",", "")) for op in ("dadd", "dmul", "dfma")),
            "fp64_peak_per_cycle": float(d.get(
                "sm__sass_thread_inst_executed_op_dfma_pred_on.sum.peak_sustained", "nan")
                .replace(",", "")),
        })
    r0 = recs[0]
    res = {"source": rep.split("/")[-1], "workload": workload, "kernel": r0["kernel"], "grid": r0["grid"],
           "block": r0["block"],
           "dram_bytes_per_launch": r0["dram_read_bytes"] + r0["dram_write_bytes"],
           "dram_read_bytes": r0["dram_read_bytes"], "dram_write_bytes": r0["dram_write_bytes"],
           "ncu_duration_ms": r0["duration_ms"], "launches_captured": len(recs),
           "fp64_pipe_active_pct": r0["fp64_pipe_pct"], "issue_active_pct": r0["issue_active_pct"],
           "fp64_arith_frac_of_peak": r0["fp64_ops_per_cycle"] / r0["fp64_peak_per_cycle"]}
    if cells:
        res["cells_per_launch"] = int(cells)
        res["dram_bytes_per_cell"] = res["dram_bytes_per_launch"] / int(cells)
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:6])
