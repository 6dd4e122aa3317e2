"""Summarise an ncu --page source --print-source cuda,sass CSV: hottest source lines.

usage: ncu -i rep.ncu-rep --page source --csv --print-source cuda,sass > src.csv
       python tools/ncu_source_summary.py src.csv [top]
"""
import csv
import sys


def main(path, top=40):
    rows = list(csv.reader(open(path)))
    file = None
    hdr = None
    agg = []
    stall_cols = []
    for r in rows:
        if len(r) == 2 and r[0] == "File Path":
            file = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
            continue
        if hdr is None or not r or r[0] == "" or len(r) < len(hdr):
            continue
        try:
            samples = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
            inst = int(r[hdr.index("Instructions Executed")])
        except (ValueError, IndexError):
            continue
        stalls = sorted(((int(r[i]) if r[i].isdigit() else 0, hdr[i][6:]) for i in stall_cols), reverse=True)[:3]
        agg.append((samples, inst, file, r[0], r[1][:90], stalls))
    tot_s = sum(a[0] for a in agg) or 1
    tot_i = sum(a[1] for a in agg) or 1
    print(f"total samples {tot_s}  total warp-instructions {tot_i}")
    for s, i, f, ln, src, st in sorted(agg, reverse=True)[:top]:
        print(f"{100*s/tot_s:5.1f}% smp {100*i/tot_i:5.1f}% ins  {f}:{ln:<4} {src:<90} "
              + " ".join(f"{n}={v}" for v, n in st if v))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40)
