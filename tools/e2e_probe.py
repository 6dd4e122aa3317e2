"""Where the end-to-end call's time goes (config 4): host->device copy of the
state, Ensemble construction, the first advance (workspace, graph capture),
the step loop, device->host copy -- with a second ensemble alive, as in
bench.py's e2e leg."""
import sys
import time

import torch

sys.path.insert(0, '.')
import bench  # noqa: E402
from paper_2505_17025_b200 import Criterion, Ensemble  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
cfg, recs, h, hu, hw = bench.build_workload("config4", 0, 1)
crit = Criterion("eta_over_d")
ens = Ensemble(recs, h, hu, hw)
ens.advance(3, "adaptive", crit)
torch.cuda.synchronize()
hh = [x.cpu().pin_memory() for x in (h, hu, hw)]
ho = [torch.empty_like(x).pin_memory() for x in hh]
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dh = [x.to("cuda", non_blocking=True) for x in hh]
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    ens2 = Ensemble(recs, *dh)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    ens2.advance(1, "adaptive", crit)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    ens2.advance(steps, "adaptive", crit)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    for dst, src in zip(ho, (ens2.h, ens2.hu, ens2.hw)):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    t5 = time.perf_counter()
    print(f"h2d {1e3*(t1-t0):.1f} ms, ensemble {1e3*(t2-t1):.1f}, first advance(1) "
          f"{1e3*(t3-t2):.1f}, advance({steps}) {1e3*(t4-t3):.1f} "
          f"({(t4-t3)/steps*1e3:.3f}/step), d2h {1e3*(t5-t4):.1f}", flush=True)
    del dh, ens2
