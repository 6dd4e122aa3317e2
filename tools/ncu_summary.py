"""Key metrics of one kernel in an ncu report: time, DRAM bytes, pipes, stalls,
instruction mix and (optionally) the hottest source lines.

usage: python tools/ncu_summary.py rep.ncu-rep [--kernel REGEX] [--cells N] [--source TOP]
"""
import argparse
import collections
import csv
import io
import re
import subprocess

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__cycles_elapsed.avg.per_second"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def metrics(rep, kernel):
    r = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    hdr, unit = r[0], r[1]
    for row in r[2:]:
        d = dict(zip(hdr, row))
        if kernel is None or re.search(kernel, d.get("Kernel Name", "")):
            return d, dict(zip(hdr, unit))
    raise SystemExit(f"no kernel matching {kernel!r}")


def source_lines(rep, kernel, top):
    args = ["--page", "source", "--csv", "--print-source", "cuda,sass"]
    if kernel:
        args = ["-k", f"regex:{kernel}"] + args
    rows = list(csv.reader(io.StringIO(ncu(rep, *args))))
    file, hdr, agg = None, None, []
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            file = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or not r or r[0] == "" or len(r) < len(hdr):
            continue
        try:
            samples = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
            inst = int(r[hdr.index("Instructions Executed")])
        except (ValueError, IndexError):
            continue
        stalls = sorted(((int(r[i]) if r[i].isdigit() else 0, h[6:]) for i, h in enumerate(hdr)
                         if h.startswith("stall_") and "Not Issued" not in h), reverse=True)[:3]
        agg.append((samples, inst, file, r[0], r[1].strip()[:80], stalls))
    ts = sum(a[0] for a in agg) or 1
    ti = sum(a[1] for a in agg) or 1
    out = [f"hottest source lines (of {ts} stall samples, {ti} warp-instructions):"]
    for s, i, f, ln, src, st in sorted(agg, reverse=True)[:top]:
        out.append(f"  {100 * s / ts:5.1f}% smp {100 * i / ti:5.1f}% ins  {f}:{ln:<5} {src:<80} "
                   + " ".join(f"{n}={v}" for v, n in st if v))
    return out


def sass_mix(rep, kernel, top=16):
    args = ["--page", "source", "--csv", "--print-source", "sass"]
    if kernel:
        args = ["-k", f"regex:{kernel}"] + args
    rows = list(csv.reader(io.StringIO(ncu(rep, *args))))
    hdr = next((r for r in rows if r and r[0] == "Address"), None)
    if hdr is None:
        return []
    ie = hdr.index("Instructions Executed")
    c, tot = collections.Counter(), 0
    for r in rows:
        if len(r) < len(hdr) or not r[0].startswith("0x"):
            continue
        op = r[1].strip().split()
        if not op:
            continue
        m = (op[1] if op[0].startswith("@") else op[0]).split(".")[0]
        n = int(r[ie] or 0)
        c[m] += n
        tot += n
    return [f"SASS mix (warp-instructions executed, {tot} total):"] + [
        f"  {m:10s} {100 * n / max(tot, 1):5.1f}%" for m, n in c.most_common(top)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--kernel")
    ap.add_argument("--cells", type=float)
    ap.add_argument("--source", type=int, default=0)
    a = ap.parse_args()
    d, u = metrics(a.rep, a.kernel)
    lines = [f"kernel {d.get('Kernel Name')}  grid {d.get('Grid Size')}  block {d.get('Block Size')}"]
    for k in KEYS:
        if k in d:
            lines.append(f"  {k:68s} {d[k]:>20s} {u[k]}")
    stalls = [(float(v.replace(",", "")), h) for h, v in d.items()
              if h.startswith("smsp__average_warps_issue_stalled_")
              and h.endswith("_per_issue_active.ratio")]
    lines.append("warp stalls per issued instruction:")
    for v, h in sorted(stalls, reverse=True)[:10]:
        lines.append(f"  {h[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]:28s} {v:7.3f}")
    if a.cells:
        ins = float(d["smsp__inst_executed.sum"].replace(",", ""))
        lines.append(f"warp-instructions per cell: {ins / a.cells:.2f}")
    if a.source:
        lines += sass_mix(a.rep, a.kernel)
        lines += source_lines(a.rep, a.kernel, a.source)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
