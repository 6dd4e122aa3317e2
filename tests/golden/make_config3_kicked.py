"""Config 3 sensitivity envelope (CPU; the oracle is the reference's
arithmetic bit for bit, tests/test_oracle_golden.py): restart from the
REFERENCE's own step-S checkpoint (config3_full.npz) with h perturbed -- one
value by one ulp, or every value by a relative kick REL -- and run to the
final step, recording the per-step flagged count.  With REL = 1e-10 at
S = 20000 (the size of the GPU's drift there) this is the reference's own
trajectory under a GPU-sized perturbation; tests/test_gpu_golden.py compares
the GPU's full-run statistics with it.  Writes config3_kicked.npz next to
this script (rel > 0 only).

    python tests/golden/make_config3_kicked.py [S] [element] [rel]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from oracle import nhswe_oracle as O  # noqa: E402
from paper_2505_17025_b200 import configs  # noqa: E402
from tests.helpers import oracle_member  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 20000
E = int(sys.argv[2]) if len(sys.argv) > 2 else 1500
REL = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0   # 0: one ulp; else a relative kick of all h
HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "config3_full.npz"))
cfg = configs.config3()
m = cfg.member(0)
mem = oracle_member(m.grid, m.bathymetry, m.bcs, m.dt)
r = G[f"ck/s{S}"]
t = float(G[f"ck/t{S}"])
h, hu, hw = r[0].copy(), r[1].copy(), r[2].copy()
if REL:
    rng = np.random.default_rng(1)
    h = h * (1.0 + REL * rng.standard_normal(h.shape))
else:
    h[E, 0] = np.nextafter(h[E, 0], np.inf)
n = int(G["n_steps"])
ref_counts = G["adaptive/flag_count"].astype(np.int64)
counts = list(ref_counts[:S])
t0 = time.time()
for k in range(S, n):
    o = O.step(mem, h, hu, hw, t, "adaptive", cfl_warn=False)
    h, hu, hw = o.h, o.hu, o.hw
    t = t + mem.dt
    counts.append(int(o.flags.sum()))
    if (k + 1) % 10000 == 0:
        c = np.array(counts)
        print(f"step {k + 1}: running mask fraction perturbed {c.mean() / m.grid.n_elements:.4f} "
              f"reference {ref_counts[:k + 1].mean() / m.grid.n_elements:.4f} "
              f"({time.time() - t0:.0f}s)", flush=True)
c = np.array(counts)
print(f"final: mask fraction mean perturbed {c.mean() / m.grid.n_elements:.4f}, reference "
      f"{float(G['adaptive/mask_fraction']):.4f}")
if REL:
    np.savez_compressed(os.path.join(HERE, "config3_kicked.npz"), start=np.array(S),
                        rel=np.array(REL), counts=c.astype(np.int16),
                        mask_fraction=np.array(c.mean() / m.grid.n_elements))
