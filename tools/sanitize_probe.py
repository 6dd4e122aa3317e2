"""Small launches of every kernel family, for compute-sanitizer.

    compute-sanitizer --tool racecheck  python tools/sanitize_probe.py
    compute-sanitizer --tool synccheck  python tools/sanitize_probe.py
    compute-sanitizer --tool memcheck   python tools/sanitize_probe.py

The streaming kernels (K_P / K_S / K_X / K_C / K_F, fused global K_P, plain
launches and the CUDA-graph loop), the resident cluster kernel, the
single-function kernels and the m-node kernels each run a few steps on a
mixed ensemble that crosses tile boundaries, has flagged ranges touching both
walls and runs every mode.  The barrier elisions of stream_kp.cuh (no
__syncthreads between the Heun stages, none before the pending-trace reads)
are what racecheck is asked to confirm.
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2505_17025_b200 as P  # noqa: E402
from paper_2505_17025_b200 import _device as D, configs  # noqa: E402
from tests.helpers import oracle_depth, smooth_state  # noqa: E402


def ensemble(cfg, idx):
    H, Q, W = zip(*(cfg.host_state(i, oracle_depth) for i in idx))
    return P.Ensemble.from_host(cfg.records(idx), np.stack(H), np.stack(Q), np.stack(W))


def main():
    steps = int(os.environ.get("PROBE_STEPS", "6"))
    cfg = configs.Config4(n_members=6, n_elements=250, n_steps=steps)
    runs = [("adaptive", P.Criterion("eta_over_d", 1e-3, True)),
            ("adaptive", P.Criterion("w_x", 1e-3, False)),
            ("global", None), ("hydrostatic", None)]
    for graphs in (False, True):
        D.stream_graphs(graphs)
        for mode, crit in runs:
            ens = ensemble(cfg, range(6))
            ens.advance(steps, mode, crit, path="stream")
            torch.cuda.synchronize()
            ens.check()
            print(f"stream graphs={graphs} {mode} {crit.kind if crit else ''}: ok", flush=True)
    D.stream_graphs(True)
    # config 5 geometry (slope slide) on the stream path, and the resident kernel
    c5 = configs.Config5(n_members=2, n_elements=300, n_steps=steps)
    ens = ensemble(c5, range(2))
    ens.advance(steps, "global", None, path="stream")
    torch.cuda.synchronize()
    for mode, crit in runs[:3]:
        ens = ensemble(cfg, range(2))
        ens.advance(steps, mode, crit, path="resident")
        torch.cuda.synchronize()
        ens.check()
        print(f"resident {mode}: ok", flush=True)
    # single-function kernels
    grid = P.GridSpec(0.0, 100.0, 150)
    st = smooth_state(grid)
    bathy, bcs = P.FlatBottom(10.0), P.BoundaryPair(P.WALL, P.ABSORBING)
    P.rhs_operator(st, bathy, bcs)
    P.criterion_values(st, bathy, "eta_x")
    co = P.assemble_coefficients(st, bathy, 0.05)
    P.ldg_solve(co, (3, 140), outer_hu=(0.1, 0.2))
    P.apply_correction(st, bathy, 0.05, ((2, 40), (60, 61), (100, 149)), bcs)
    print("single-function kernels: ok", flush=True)
    # m-node kernels (p = 2)
    g2 = P.GridSpec(0.0, 100.0, 60, 2)
    s2 = smooth_state(g2)
    r = P.adaptive_step(s2, 0.02, bathy, bcs, mode="adaptive",
                        crit=P.Criterion("eta_over_d", 1e-3, True))
    print(f"p=2 adaptive_step: mask fraction {r.mask.fraction:.3f}", flush=True)
    print("SANITIZE_PROBE_DONE")


if __name__ == "__main__":
    main()
