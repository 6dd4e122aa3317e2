"""Small stream-path smoke: B members x N elements, compare with the resident path."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2505_17025_b200 as P
from paper_2505_17025_b200 import configs
from tests.helpers import oracle_depth
B = int(sys.argv[1]); N = int(sys.argv[2]); steps = int(sys.argv[3])
cfg = configs.Config4(n_members=B, n_elements=N)
recs = cfg.records()
st = [cfg.host_state(i, oracle_depth) for i in range(B)]
H, Q, W = (np.stack([s[k] for s in st]) for k in range(3))
out = {}
for path in ("resident", "stream"):
    e = P.Ensemble.from_host(recs, H, Q, W)
    torch.cuda.synchronize(); t0 = time.time()
    e.advance(steps, "adaptive", P.Criterion("eta_over_d"), path=path)
    torch.cuda.synchronize(); dt = time.time() - t0
    s = e.check()
    out[path] = [x.cpu().numpy() for x in (e.h, e.hu, e.hw)]
    print(path, "%.3fs" % dt, "flagged", s["flagged"][:4], flush=True)
for k in range(3):
    a, b = out["resident"][k], out["stream"][k]
    print("field", k, "max abs diff", np.abs(a - b).max(), "scale", np.abs(a).max())
