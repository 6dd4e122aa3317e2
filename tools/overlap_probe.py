"""Probe: does running the ensemble as two member groups on two CUDA streams
overlap one group's latency-bound kernels (K_S, K_X, K_C) with the other's
K_P?  Plain launches (NH_STREAM_GRAPH=0) in every variant, so the graph cache
plays no part.  usage (GPU): NH_STREAM_GRAPH=0 python tools/overlap_probe.py [K]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(K=400):
    import torch
    import bench
    from paper_2505_17025_b200 import Criterion, Ensemble
    cfg, recs, h, hu, hw = bench.build_workload("config4", 0, 1)
    B, N = h.shape[0], h.shape[1]
    crit = Criterion("eta_over_d", 1e-3, False)
    h0, hu0, hw0 = h.clone(), hu.clone(), hw.clone()
    out = {}

    def reset():
        h.copy_(h0); hu.copy_(hu0); hw.copy_(hw0)

    def timed(fn):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / K

    # one group
    reset()
    ens = Ensemble(recs, h, hu, hw)
    ens.advance(3, "adaptive", crit)
    out["one_group_ms_per_step"] = timed(lambda: ens.advance(K, "adaptive", crit, path="stream"))
    del ens
    for prio in ((0, 0), (-1, 0)):
        for G in (2, 4):
            reset()
            sz = B // G
            groups = [Ensemble(recs[g * sz:(g + 1) * sz], h[g * sz:(g + 1) * sz],
                               hu[g * sz:(g + 1) * sz], hw[g * sz:(g + 1) * sz]) for g in range(G)]
            streams = [torch.cuda.Stream(priority=prio[0] if g == 0 else prio[1]) for g in range(G)]
            for e in groups:
                e.advance(3, "adaptive", crit)

            def run():
                cur = torch.cuda.current_stream()
                for e, s in zip(groups, streams):
                    s.wait_stream(cur)
                    with torch.cuda.stream(s):
                        e.advance(K, "adaptive", crit, path="stream")
                for s in streams:
                    cur.wait_stream(s)
            out[f"{G}_groups_prio{prio}_ms_per_step"] = timed(run)
            del groups
    out["cell_steps_per_s_one_group"] = B * N / (out["one_group_ms_per_step"] * 1e-3)
    print(json.dumps(out))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 400)
