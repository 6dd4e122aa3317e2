"""Per-phase cycle breakdown of the fused step (build with -DNH_PROFILE_PHASES=1, select via NH_LIB)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_2505_17025_b200 import Criterion, Ensemble, _lib
from paper_2505_17025_b200._device import read_status

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
mode = sys.argv[2] if len(sys.argv) > 2 else "adaptive"
cfg, recs, h, hu, hw = bench.build_workload("config4", 0, 1)
lib = _lib.load()
plan = _lib.plan(cfg.n_elements, len(recs))
grid = len(recs) * plan["cluster"]
buf = torch.zeros((grid, 15), dtype=torch.int64, device="cuda")
lib.nh_set_profile_buffer.argtypes = [ctypes.c_void_p]
lib.nh_set_profile_buffer(buf.data_ptr())
ens = Ensemble(recs, h, hu, hw)
crit = Criterion("eta_over_d")
ens.advance(3, mode, crit)
torch.cuda.synchronize()
buf.zero_()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); ens.advance(steps, mode, crit); e1.record(); e1.synchronize()
ms = e0.elapsed_time(e1)
p = buf.cpu().numpy().astype(np.float64) / steps
names = ["stage1", "stage2", "criterion+sync", "condense", "tree(A/B/C)", "unwind+recon", "B3 wait",
         "hw update+sync", "halo push", "B1 wait", " tree: A-up+sync", " tree: B-up", " tree: B2 wait",
         " tree: C+B-down+sync"]
p = p[:, :14]
tot = p[:, :10].sum(axis=1).mean()
print(f"plan {plan}  {ms/steps:.3f} ms/step  {len(recs)*cfg.n_elements*steps/ms/1e6:.2f} G cell-steps/s")
print(f"cycles per CTA-step (mean over CTAs): {tot:.0f}")
for i, n in enumerate(names):
    print(f"  {n:18s} {p[:, i].mean():9.0f}  {100*p[:, i].mean()/tot:5.1f}%   max {p[:, i].max():9.0f}")
