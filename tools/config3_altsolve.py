"""Config 3 with an equally valid elliptic solver (CPU oracle): the oracle is
the reference's arithmetic bit for bit except that LAPACK dgbsv factorises
the band system with rows and columns in reverse order (same matrix, same
partial pivoting, different rounding, ~1e-16 relative per solve).  Started
from the reference's own checkpoint at step S, it shows how far a solver that
is as accurate as dgbsv but not bitwise identical to it drifts from the
reference over the rest of the run (per-window mask fractions, as
tools/config3_counts.py prints for the GPU).

    python tools/config3_altsolve.py [S]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import nhswe_oracle as O  # noqa: E402
from paper_2505_17025_b200 import configs  # noqa: E402
from tests.helpers import oracle_member  # noqa: E402

_dgbsv = O._lapack.dgbsv


def dgbsv_reversed(kl, ku, ab, b, overwrite_ab=False, overwrite_b=False):
    """Solve the band system with unknowns and equations in reverse order."""
    assert kl == ku
    r = np.zeros_like(ab)
    top = kl + ku
    r[kl:kl + top + 1] = ab[kl + top:kl - 1:-1, ::-1] if kl > 0 else ab[top::-1, ::-1]
    lu, piv, x, info = _dgbsv(kl, ku, r, np.ascontiguousarray(b[::-1]))
    return lu, piv, x[::-1].copy(), info


O._lapack.dgbsv = dgbsv_reversed

S = int(sys.argv[1]) if len(sys.argv) > 1 else 15000
G = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden", "config3_full.npz"))
cfg = configs.config3()
m = cfg.member(0)
mem = oracle_member(m.grid, m.bathymetry, m.bcs, m.dt)
r = G[f"ck/s{S}"]
t = float(G[f"ck/t{S}"])
h, hu, hw = r[0].copy(), r[1].copy(), r[2].copy()
n = int(G["n_steps"])
ref = G["adaptive/flag_count"].astype(np.int64)
cnt = list(ref[:S])
t0 = time.time()
first = None
for k in range(S, n):
    o = O.step(mem, h, hu, hw, t, "adaptive", cfl_warn=False)
    h, hu, hw = o.h, o.hu, o.hw
    t = t + mem.dt
    cnt.append(int(o.flags.sum()))
    if first is None and cnt[-1] != ref[k]:
        first = k
        print(f"first step where counts differ: {k}", flush=True)
    if (k + 1) % 10000 == 0:
        print(f"step {k + 1} ({time.time() - t0:.0f}s)", flush=True)
cnt = np.array(cnt)
for a, b in [(0, 15000), (15000, 30000), (30000, 60000), (60000, 90000), (90000, n)]:
    print(f"steps {a:6d}-{b:6d}: alt-solver mean frac {cnt[a:b].mean() / 8000:.4f}  "
          f"reference {ref[a:b].mean() / 8000:.4f}")
print(f"full-run mask fraction: alt-solver {cnt.mean() / 8000:.4f} reference "
      f"{float(G['adaptive/mask_fraction']):.4f}")
