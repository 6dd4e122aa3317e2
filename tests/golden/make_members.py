"""Full-length golden runs of sampled throughput-config members by the REAL
reference (configs 4 and 5: 20000 / 10000 steps), for the GPU parity gate at
the final time with per-step masks (tests/test_gpu_members.py).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_members.py

Members are sampled by `sample_members` below: every parameter-range corner
of the drawn population (argmin / argmax of each drawn parameter, per bottom
kind), both ends of the table, and seeded fill to >= 32 members per config.
A member's parameters depend on (seed, index) only (configs.member_rng), so
the same member runs inside the full 4096 / 65536-member ensembles on the GPU.

One process per (member, mode); BLAS pinned to one thread.  Writes
tests/golden/members_full.npz: the sampled index lists, and per case the final
h and hu, the per-step flagged counts, the per-step mask CRC (crc32 of
np.packbits(flags), as make_golden.digest) and the reference loop time.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import sys
import time
import zlib

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

N_SAMPLE = 32


def sample_members(name: str) -> list[int]:
    """Corners of the drawn parameter ranges + both table ends + seeded fill."""
    from paper_2505_17025_b200 import configs
    cfg = configs.get(name)
    B = cfg.n_members
    pick = [0, 1, B - 2, B - 1]
    if name == "config4":
        d = {k: np.array([configs._config4_draw(cfg.seed, i)[k] for i in range(B)])
             for k in ("h0", "a_rel", "zeta_rel", "b_rel", "alpha")}
        ev, od = np.arange(0, B, 2), np.arange(1, B, 2)
        for k in ("h0", "a_rel"):               # solitary members (even)
            pick += [int(ev[np.argmin(d[k][ev])]), int(ev[np.argmax(d[k][ev])])]
        for k in ("zeta_rel", "b_rel", "alpha"):   # box uplifts (odd)
            pick += [int(od[np.argmin(d[k][od])]), int(od[np.argmax(d[k][od])])]
        # the most impulsive uplift (alpha * zeta0) and the steepest solitary wave
        pick += [int(od[np.argmax((d["alpha"] * d["zeta_rel"])[od])]),
                 int(ev[np.argmax((d["a_rel"] / d["h0"])[ev])])]
    else:
        tab = cfg.table()
        tan_t, A, sigma, x0, u_t = tab.T
        ratio = A / np.minimum(0.1 + x0 * tan_t, 1.0)
        for v in (tan_t, ratio, sigma, u_t):
            pick += [int(np.argmin(v)), int(np.argmax(v))]
    pick = list(dict.fromkeys(pick))
    rng = np.random.default_rng(7)
    while len(pick) < N_SAMPLE:
        i = int(rng.integers(B))
        if i not in pick:
            pick.append(i)
    return sorted(pick)


def run(case):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    sys.path.insert(0, ROOT)
    sys.path.insert(0, "/root/reference/pkg/src")
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
    res = R.simulate(spec, init, mode, crit, record_masks=(mode == "adaptive"))
    fs = res.final_state
    cnt, crc = [], []
    for _, _, ranges in res.mask_history:
        f = np.zeros(grid.n_elements, bool)
        for e0, e1 in ranges:
            f[e0:e1 + 1] = True
        cnt.append(int(f.sum()))
        crc.append(zlib.crc32(np.packbits(f).tobytes()))
    key = f"{name}/{i}/{mode}"
    print(key, f"{time.time() - t0:.0f}s", flush=True)
    return key, {"h": fs.h.values, "hu": fs.hu.values, "counts": np.array(cnt, np.int16),
                 "crc": np.array(crc, np.uint32),
                 "loop_time": np.array(res.loop_time), "time": np.array(fs.time)}


if __name__ == "__main__":
    samples = {c: sample_members(c) for c in ("config4", "config5")}
    cases = [("config4", i, "adaptive") for i in samples["config4"]]
    cases += [("config5", i, mode) for i in samples["config5"] for mode in ("adaptive", "global")]
    print({c: v for c, v in samples.items()}, len(cases), "cases", flush=True)
    # longest first
    cases.sort(key=lambda c: (c[0] != "config5", c[2] != "global"))
    with mp.get_context("spawn").Pool(int(os.environ.get("PROCS", "6"))) as pool:
        out = pool.map(run, cases, chunksize=1)
    data = {f"{c}/members": np.array(v) for c, v in samples.items()}
    for key, d in out:
        for k, v in d.items():
            data[f"{key}/{k}"] = v
    np.savez_compressed(os.path.join(HERE, "members_full.npz"), **data)
    print("wrote members_full.npz")
