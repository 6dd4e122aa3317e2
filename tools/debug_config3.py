"""Config 3 on the GPU vs the reference checkpoints (tests/golden/config3_full.npz ck/*)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2505_17025_b200 as P
from paper_2505_17025_b200 import configs
from oracle import nhswe_oracle as O
from tests.helpers import oracle_member, oracle_depth
G = np.load('tests/golden/config3_full.npz')
C = {k[3:]: G[k] for k in G.files if k.startswith('ck/')}
cfg = configs.config3(); m = cfg.member(0)
ens = P.Ensemble.from_host(cfg.records(), G['h0'][None], G['hu0'][None], G['hw0'][None])
done = 0
rel = lambda a, b: np.abs(a - b).max() / np.abs(b).max()
for c in sorted(int(k[1:]) for k in C if k.startswith('s')):
    ens.advance(c - done, "adaptive", P.Criterion("eta_over_d"), path=sys.argv[1] if len(sys.argv) > 1 else "auto")
    done = c
    ens.check()
    g = [x[0].cpu().numpy() for x in (ens.h, ens.hu, ens.hw)]
    r = C[f's{c}']
    d = oracle_depth(m.bathymetry, m.grid.sample_nodes, float(C[f't{c}']))
    print(c, "time diff", float(ens.time.item()) - float(C[f't{c}']),
          "eta", rel(g[0] - d, r[0] - d), "hu", rel(g[1], r[1]), "hw", rel(g[2], r[2]), flush=True)
# one-step replay at the last checkpoint: GPU step vs oracle step from the same state
c = done
r = C[f's{c}']; t = float(C[f't{c}'])
mem = oracle_member(m.grid, m.bathymetry, m.bcs, m.dt)
o = O.step(mem, r[0], r[1], r[2], t, "adaptive", cfl_warn=False)
st = P.FlowState(P.NodalField(m.grid, r[0]), P.NodalField(m.grid, r[1]), P.NodalField(m.grid, r[2]), t)
q = P.adaptive_step(st, m.dt, m.bathymetry, m.bcs, mode="adaptive", crit=P.Criterion("eta_over_d"))
print("replay: flags equal", np.array_equal(q.mask.flags, o.flags), "h", rel(q.state.h.values, o.h),
      "hu", rel(q.state.hu.values, o.hu), "hw", rel(q.state.hw.values, o.hw))
