"""Run a slice of config 4 on the GPU, report failing members and compare one to the oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2505_17025_b200 as P
from paper_2505_17025_b200 import configs, _lib
from paper_2505_17025_b200._device import decode_error, read_status
from oracle import nhswe_oracle as O
from tests.helpers import oracle_member, oracle_depth

n_mem = int(sys.argv[1]) if len(sys.argv) > 1 else 256
n_steps = int(sys.argv[2]) if len(sys.argv) > 2 else 400
cfg = configs.Config4()
idx = list(range(n_mem))
recs = cfg.records(idx)
st = [cfg.host_state(i, oracle_depth) for i in idx]
H, Q, W = (np.stack([s[k] for s in st]) for k in range(3))
ens = P.Ensemble.from_host(recs, H, Q, W)
crit = P.Criterion("eta_over_d")
ens.advance(n_steps, "adaptive", crit)
s = read_status(ens.status)
bad = np.flatnonzero(s["error_key"] != _lib.STATUS_OK_KEY)
print("bad members", bad[:20], "count", bad.size)
for i in bad[:5]:
    print(i, decode_error(s["error_key"][i]), type(cfg.member(i).bathymetry).__name__)
if bad.size:
    i = int(bad[0])
    step, code, el = decode_error(s["error_key"][i])
    m = cfg.member(i)
    mem = oracle_member(m.grid, m.bathymetry, m.bcs, m.dt)
    e1 = P.Ensemble.from_host(recs[i:i + 1], H[i:i + 1], Q[i:i + 1], W[i:i + 1])
    h, hu, hw = H[i], Q[i], W[i]
    t = 0.0
    for k in range(step + 1):
        e1.advance(1, "adaptive", crit)
        o = O.step(mem, h, hu, hw, t, "adaptive", cfl_warn=False)
        t += m.dt
        gh, gq, gw = (x[0].cpu().numpy() for x in (e1.h, e1.hu, e1.hw))
        d = [np.abs(gh - o.h).max(), np.abs(gq - o.hu).max(), np.abs(gw - o.hw).max()]
        ss = read_status(e1.status)
        if k % 10 == 0 or max(d) > 1e-9 or ss["error_key"][0] != _lib.STATUS_OK_KEY:
            print(k, "diff", d, "flags", int(o.flags.sum()), decode_error(ss["error_key"][0]))
        if max(d) > 1e-6:
            bad_e = np.flatnonzero(np.abs(gq - o.hu).max(axis=1) > 1e-9)
            print("diverged at elements", bad_e[:20], "oracle ranges", O.runs(o.flags)[:10])
            break
        h, hu, hw = o.h, o.hu, o.hw
