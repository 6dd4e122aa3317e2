"""Full-length golden runs of sampled throughput-config members by the REAL
reference (configs 4 and 5: 20000 / 10000 steps), for the GPU parity gate at
the final time (tests/test_gpu_golden.py::test_sampled_members_full_length).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_members.py

One process per (member, mode); BLAS pinned to one thread.  Writes
tests/golden/members_full.npz: per case the final h and hu, the per-step
flagged counts and the reference loop time.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))

CASES = [("config4", 0, "adaptive"), ("config4", 1, "adaptive"), ("config4", 2047, "adaptive"),
         ("config4", 4094, "adaptive"), ("config5", 0, "adaptive"), ("config5", 65535, "adaptive"),
         ("config5", 0, "global"), ("config5", 65535, "global")]


def run(case):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    sys.path.insert(0, ROOT)
    sys.path.insert(0, "/root/reference/pkg/src")
    import numpy as np
    import nhswe as R
    from oracle import nhswe_oracle as O
    from paper_2505_17025_b200 import configs
    from tests.golden.make_golden import Wrapped
    from tests.helpers import oracle_depth
    name, i, mode = case
    cfg = configs.get(name)
    m = cfg.member(i)
    h, hu, hw = cfg.host_state(i, oracle_depth)
    grid = R.GridSpec(m.grid.x_left, m.grid.x_right, m.grid.n_elements)
    b = m.bathymetry
    kind = type(b).__name__
    if kind == "FlatBottom":
        bathy = R.FlatBottom(b.h0)
    elif kind == "SmoothBoxPlate":
        bathy = Wrapped(O.SmoothBox(b.h0, b.zeta0, b.b, b.alpha, b.w))
    else:
        bathy = Wrapped(O.SlopeSlide(b.d_top, b.tan_theta, b.d_max, b.A, b.sigma, b.x0, b.u_t,
                                     b.t0, b.d_stop))
    bcs = R.BoundaryPair(R.BoundaryCondition(m.bcs.left.kind), R.BoundaryCondition(m.bcs.right.kind))
    spec = R.ScenarioSpec(f"{name}_{i}", grid, m.dt, cfg.n_steps * m.dt, bathy, bcs)
    assert spec.n_steps == cfg.n_steps
    init = R.FlowState(R.NodalField(grid, h), R.NodalField(grid, hu), R.NodalField(grid, hw), 0.0)
    crit = R.Criterion("eta_over_d") if mode == "adaptive" else None
    t0 = time.time()
    res = R.simulate(spec, init, mode, crit, record_masks=True)
    fs = res.final_state
    cnt = np.array([sum(e1 - e0 + 1 for e0, e1 in r) for _, _, r in res.mask_history], np.int16)
    key = f"{name}/{i}/{mode}"
    print(key, f"{time.time() - t0:.0f}s", flush=True)
    return key, {"h": fs.h.values, "hu": fs.hu.values, "counts": cnt,
                 "loop_time": np.array(res.loop_time), "time": np.array(fs.time)}


if __name__ == "__main__":
    import numpy as np
    with mp.get_context("spawn").Pool(int(os.environ.get("PROCS", "4"))) as pool:
        out = pool.map(run, CASES, chunksize=1)
    data = {}
    for key, d in out:
        for k, v in d.items():
            data[f"{key}/{k}"] = v
    np.savez_compressed(os.path.join(HERE, "members_full.npz"), **data)
    print("wrote members_full.npz")
