"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

usage: python tools/launch_summary.py launches.csv [out.txt]
"""
import collections
import csv
import sys


def main(path, out=None):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0] != "ID"]
    per = collections.OrderedDict()
    for r in rows:
        if r[12] != "gpu__time_duration.sum":
            continue
        name = r[4].split("(")[0].replace("void ", "")
        ns = float(r[14].replace(",", ""))
        scale = {"ns": 1.0, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(r[13], 1.0)
        per.setdefault(name, []).append((ns * scale, r[7], r[8]))
    tot = sum(t for v in per.values() for t, _, _ in v)
    lines = [f"{'kernel':60s} {'n':>5s} {'mean us':>10s} {'total us':>11s} {'share':>7s}  block/grid"]
    for name, v in sorted(per.items(), key=lambda kv: -sum(t for t, _, _ in kv[1])):
        s = sum(t for t, _, _ in v)
        lines.append(f"{name[:60]:60s} {len(v):5d} {s / len(v) / 1e3:10.2f} {s / 1e3:11.1f} "
                     f"{s / tot:7.1%}  {v[0][1]} {v[0][2]}")
    lines.append(f"{'total':60s} {sum(len(v) for v in per.values()):5d} {'':10s} {tot / 1e3:11.1f}")
    text = "\n".join(lines)
    print(text)
    if out:
        open(out, "w").write(text + "\n")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
