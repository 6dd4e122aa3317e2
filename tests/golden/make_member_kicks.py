"""How far the REAL reference's own final state of a config-4 member moves
under a one-ulp perturbation of its initial state, and reference checkpoints
for windowed parity of the most sensitive members.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_member_kicks.py

Config 4 runs 20000 steps.  For the box-uplift members an ulp-level change is
amplified to 1e-10 .. 1e-8 (relative) by the final time -- in the reference
itself: this script runs every sampled member (members_full.npz) twice with
the reference's adaptive_step, once from the initial state and once with h
raised by one ulp at a single node, and stores the relative L-inf distance of
the two final states ("kick": eta, hu).  The unkicked run must reproduce the
stored golden final state bit for bit.  tests/test_gpu_members.py uses the
distance as the member's resolution: the GPU (whose elliptic solve rounds
differently from LAPACK at every step) must stay within max(1e-9, 10 x kick).

For the CHECKPOINT members the unkicked run also stores its state every 5000
steps, so the GPU can be restarted from the reference's own states and held
to the plain 1e-9 bar with exact masks over every window.
Writes tests/golden/members_kick.npz.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

CHECKPOINT = (21, 227)
EVERY = 5000


def run(args):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    sys.path.insert(0, ROOT)
    sys.path.insert(0, "/root/reference/pkg/src")
    i, kick = args
    import nhswe as R
    from paper_2505_17025_b200 import configs
    from tests.harness.ref_bridge import reference_member
    cfg = configs.Config4()
    _, grid, bathy, bcs, dt, st = reference_member(cfg, i)
    if kick:
        h = st.h.values.copy()
        k = grid.n_elements // 3
        h[k, 0] = np.nextafter(h[k, 0], 2.0 * h[k, 0])
        st = R.FlowState(R.NodalField(grid, h), st.hu, st.hw, st.time)
    crit = R.Criterion("eta_over_d")
    cks = {}
    for s in range(cfg.n_steps):
        st = R.adaptive_step(st, dt, bathy, bcs, mode="adaptive", crit=crit, cfl_warn=False).state
        if not kick and i in CHECKPOINT and (s + 1) % EVERY == 0 and s + 1 < cfg.n_steps:
            cks[s + 1] = (np.stack([st.h.values, st.hu.values, st.hw.values]), st.time)
    print(i, kick, flush=True)
    return i, kick, st.h.values, st.hu.values, st.time, cks


def main():
    from paper_2505_17025_b200 import configs
    from tests.helpers import oracle_depth
    G = np.load(os.path.join(HERE, "members_full.npz"))
    idx = [int(v) for v in G["config4/members"]]
    jobs = [(i, k) for i in idx for k in (0, 1)]
    with mp.get_context("spawn").Pool(int(os.environ.get("PROCS", "7"))) as pool:
        res = pool.map(run, jobs, chunksize=1)
    by = {(i, k): r for (i, k, *r) in res}
    cfg = configs.Config4()
    data = {"members": np.array(idx), "checkpoint_members": np.array(CHECKPOINT),
            "every": np.array(EVERY)}
    for i in idx:
        h0, q0, t0, cks = by[(i, 0)]
        h1, q1, _, _ = by[(i, 1)]
        assert np.array_equal(h0, G[f"config4/{i}/adaptive/h"]), i   # the stored golden run
        assert np.array_equal(q0, G[f"config4/{i}/adaptive/hu"]), i
        m = cfg.member(i)
        d = oracle_depth(m.bathymetry, m.grid.sample_nodes, t0)
        e0, e1 = h0 - d, h1 - d
        data[f"{i}/kick"] = np.array([np.abs(e0 - e1).max() / np.abs(e0).max(),
                                      np.abs(q0 - q1).max() / np.abs(q0).max()])
        for s, (st, t) in cks.items():
            data[f"{i}/ck/s{s}"] = st
            data[f"{i}/ck/t{s}"] = np.array(t)
    np.savez_compressed(os.path.join(HERE, "members_kick.npz"), **data)
    for i in idx:
        print(i, data[f"{i}/kick"])
    print("wrote members_kick.npz")


if __name__ == "__main__":
    main()
