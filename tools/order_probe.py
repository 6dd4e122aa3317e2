"""Probe: what does K_P's member-order indirection (order[b], one dependent
load per tile before its state loads) cost?  Config 4's members stored
already grouped by bottom kind, run with and without the order permutation
(NH_STREAM_ORDER is read once per process, so each variant is its own run).
usage (GPU): NH_STREAM_ORDER=0|1 python tools/order_probe.py [K]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(K=1000):
    import numpy as np
    import torch
    import bench
    from paper_2505_17025_b200 import Criterion, Ensemble, configs
    from paper_2505_17025_b200 import _device as D
    cfg = configs.Config4(n_members=4096)
    recs0 = cfg.records(list(range(4096)))
    idx = list(np.argsort(recs0["bottom_kind"], kind="stable"))   # grouped by kind
    recs = cfg.records(idx)
    h, hu, hw = bench.init_device(cfg, recs, idx)
    B, N = h.shape[0], h.shape[1]
    crit = Criterion("eta_over_d", 1e-3, False)
    ens = Ensemble(recs, h, hu, hw)
    ens.advance(3, "adaptive", crit)
    torch.cuda.synchronize()
    D.stream_timing(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ens.advance(K, "adaptive", crit, path="stream")
    e1.record()
    torch.cuda.synchronize()
    kt = D.stream_kernel_times()
    D.stream_timing(False)
    kp_ms, kp_n = kt["nh_stream_kp"]
    print(json.dumps({"order": os.environ.get("NH_STREAM_ORDER", "1"), "members_grouped_by_kind": True,
                      "event_timed_ms_per_step": e0.elapsed_time(e1) / K,
                      "kp_ms": kp_ms / max(kp_n, 1),
                      "cell_steps_per_s": B * N * K / (e0.elapsed_time(e1) * 1e-3)}))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 1000)
