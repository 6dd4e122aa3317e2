"""A throughput config at its full BASELINE length on one GPU: config 5 is
10000 steps, config 4 20000 (bench.py times 20 steps after a spin-up).

    python tools/full_length.py --workload config5 --mode adaptive [--steps 10000]

The run advances in windows of --window steps (CUDA events around each), so
the line shows how the rate moves as the flagged fraction grows and whether
the sustained run hits the power cap; nvidia-smi clocks are sampled
throughout.  Prints one JSON line.
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
from paper_2505_17025_b200._device import read_status  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="config5", choices=["config4", "config5"])
    ap.add_argument("--mode", default="adaptive", choices=["adaptive", "global"])
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--window", type=int, default=500)
    a = ap.parse_args()
    cfg, recs, h, hu, hw = bench.build_workload(a.workload, 0, 1)
    steps = a.steps or cfg.n_steps
    B, N = h.shape[0], h.shape[1]
    ens = Ensemble(recs, h, hu, hw)
    crit = Criterion("eta_over_d", 1e-3, False)
    ens.advance(4, a.mode, crit)   # warm-up (graphs, workspace); part of the run
    torch.cuda.synchronize()
    done, windows, flagged0 = 4, [], 0
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    total_ms = 0.0
    with bench.ClockSampler(0) as clk:
        while done < steps:
            k = min(a.window, steps - done)
            ev0.record()
            ens.advance(k, a.mode, crit)
            ev1.record()
            ev1.synchronize()
            ms = ev0.elapsed_time(ev1)
            total_ms += ms
            done += k
            fl = int(read_status(ens.status)["flagged"].sum())
            windows.append({"steps_done": done, "ms_per_step": ms / k,
                            "g_cell_steps_per_s": B * N * k / ms / 1e6,
                            "mask_fraction": (fl - flagged0) / (B * N * k)})
            flagged0 = fl
    st = ens.check()
    print(json.dumps({
        "workload": a.workload, "mode": a.mode, "members": B, "cells_per_member": N,
        "steps": done, "timed_steps": done - 4, "seconds": total_ms / 1e3,
        "value": B * N * (done - 4) / (total_ms * 1e-3), "unit": "cell-steps/s",
        "ms_per_step": total_ms / (done - 4),
        "mask_fraction_run": float(st["flagged"].sum()) / (B * N * done),
        "resid_max": float(st["resid_max"].max()), "status_ok": True,
        "clocks": clk.summary(), "windows": windows}))


if __name__ == "__main__":
    main()
