"""A BASELINE-shaped ensemble stepped on the streaming path, for ncu captures
of one kernel at a representative state.

    python tools/kp_probe.py --workload config5 --members 4096 --warmup 200 --steps 4
    ncu --set full -k regex:nh_stream_kp --launch-skip 2 -c 1 \
        python tools/kp_probe.py ...

The members are the first --members of the workload (same per-cell work as
the full ensemble); --warmup steps run first so that flagged ranges have
formed, then --steps steps with plain launches (no graph) so ncu sees each
kernel.  Prints the per-kernel event times of the --steps window.
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2505_17025_b200 import Criterion, Ensemble  # noqa: E402
from paper_2505_17025_b200 import _device as D  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="config5", choices=["config4", "config5"])
    ap.add_argument("--members", type=int, default=4096)
    ap.add_argument("--warmup", type=int, default=200)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--mode", default="adaptive")
    a = ap.parse_args()
    cfg, recs, h, hu, hw = bench.build_workload(a.workload, 0, 1, members=range(a.members))
    ens = Ensemble(recs, h, hu, hw)
    crit = Criterion("eta_over_d", 1e-3, False)
    ens.advance(a.warmup, a.mode, crit)
    torch.cuda.synchronize()
    D.stream_graphs(False)
    D.stream_timing(True)
    ens.advance(a.steps, a.mode, crit)
    torch.cuda.synchronize()
    t = D.stream_kernel_times()
    D.stream_timing(False)
    st = ens.check()
    frac = float(st["flagged"].sum()) / (ens.B * ens.N * (a.warmup + a.steps))
    print(json.dumps({"workload": a.workload, "members": a.members, "mask_fraction_run": frac,
                      "kernel_ms_per_launch": {k: v[0] / max(v[1], 1) for k, v in t.items()
                                               if v[1]}}))


if __name__ == "__main__":
    main()
