"""Config 3 full run on the GPU: per-step flagged counts + final state, saved
for comparison with the reference run (tests/golden/config3_full.npz).

usage: python tools/config3_counts.py out.npz
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2505_17025_b200 as P
from paper_2505_17025_b200 import configs

G = np.load("tests/golden/config3_full.npz")
cfg = configs.config3()
m = cfg.member(0)
n = int(G["n_steps"])
spec = P.ScenarioSpec(cfg.name, m.grid, m.dt, n * m.dt, m.bathymetry, m.bcs)
init = P.FlowState(P.NodalField(m.grid, G["h0"]), P.NodalField(m.grid, G["hu0"]),
                   P.NodalField(m.grid, G["hw0"]), 0.0)
res = P.simulate(spec, init, "adaptive", P.Criterion("eta_over_d"), record_masks=True)
cnt = np.array([sum(e1 - e0 + 1 for e0, e1 in r) for _, _, r in res.mask_history])
ref = G["adaptive/flag_count"]
fin = res.final_state
np.savez_compressed(sys.argv[1], counts=cnt, h=fin.h.values, hu=fin.hu.values, hw=fin.hw.values)
for a, b in [(0, 15000), (15000, 30000), (30000, 60000), (60000, 90000), (90000, n)]:
    print(f"steps {a:6d}-{b:6d}: GPU mean frac {cnt[a:b].mean() / 8000:.4f}  "
          f"reference {ref[a:b].mean() / 8000:.4f}")
print("first step where counts differ:", int(np.flatnonzero(cnt != ref)[0]) if (cnt != ref).any() else None)
