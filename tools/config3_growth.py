"""Config 3 sensitivity: from the reference checkpoint at step S, advance the
GPU (resident path), the oracle (the reference's arithmetic bit for bit) and
the oracle with one h value perturbed by 1 ulp, side by side, and print how
far apart the three trajectories drift (relative L-inf of eta and hu).

    python tools/config3_growth.py [S] [n_steps] [chunk]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2505_17025_b200 as P  # noqa: E402
from oracle import nhswe_oracle as O  # noqa: E402
from paper_2505_17025_b200 import configs  # noqa: E402
from tests.helpers import oracle_depth, oracle_member, rel  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 30000
n = int(sys.argv[2]) if len(sys.argv) > 2 else 6000
chunk = int(sys.argv[3]) if len(sys.argv) > 3 else 250
G = np.load("tests/golden/config3_full.npz")
cfg = configs.config3()
m = cfg.member(0)
mem = oracle_member(m.grid, m.bathymetry, m.bcs, m.dt)
r = G[f"ck/s{S}"]
t = float(G[f"ck/t{S}"])
ens = P.Ensemble.from_host(cfg.records(), r[0][None], r[1][None], r[2][None], time=np.array([t]))
o = [r[0].copy(), r[1].copy(), r[2].copy()]
p = [r[0].copy(), r[1].copy(), r[2].copy()]
p[0][4000, 0] = np.nextafter(p[0][4000, 0], np.inf)
ref_cnt = G["adaptive/flag_count"]
to = tp = t
for k in range(0, n, chunk):
    ens.advance(chunk, "adaptive", P.Criterion("eta_over_d"), path="resident")
    fo = fp = 0
    for _ in range(chunk):
        s = O.step(mem, *o, to, "adaptive", cfl_warn=False)
        o = [s.h, s.hu, s.hw]
        to = to + mem.dt
        s2 = O.step(mem, *p, tp, "adaptive", cfl_warn=False)
        p = [s2.h, s2.hu, s2.hw]
        tp = tp + mem.dt
    fo, fp = int(s.flags.sum()), int(s2.flags.sum())
    d = oracle_depth(m.bathymetry, m.grid.sample_nodes, to)
    g = [x[0].cpu().numpy() for x in (ens.h, ens.hu)]
    step = S + k + chunk
    print(f"step {step}: gpu-oracle eta {rel(g[0] - d, o[0] - d):.2e} hu {rel(g[1], o[1]):.2e} | "
          f"perturbed-oracle eta {rel(p[0] - d, o[0] - d):.2e} hu {rel(p[1], o[1]):.2e} | "
          f"flags ref {int(ref_cnt[step - 1])} oracle {fo} perturbed {fp}", flush=True)
