"""Config 4 on both step implementations: the streaming tiles (HBM round trip
per step) and the SMEM-resident cluster kernel (state on chip for the whole
launch), adaptive and global.  Prints cell-steps/s per (path, mode).

    python tools/path_compare.py [steps]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2505_17025_b200 import Criterion, Ensemble  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 200
cfg, recs, h, hu, hw = bench.build_workload("config4", 0, 1)
B, N = h.shape[0], h.shape[1]
for mode in ("adaptive", "global"):
    for path in ("stream", "resident"):
        ens = Ensemble(recs, h.clone(), hu.clone(), hw.clone())
        crit = Criterion("eta_over_d", 1e-3, False)
        ens.advance(3, mode, crit, path=path)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ens.advance(steps, mode, crit, path=path)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        ens.check()
        print(f"{mode:8s} {path:8s}: {B * N * steps / (ms * 1e-3) / 1e9:7.3f} G cell-steps/s "
              f"({ms / steps:.3f} ms/step)", flush=True)
        del ens
