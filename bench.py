#!/usr/bin/env python
"""Benchmark: cell-steps/s of the fused adaptive NH-SWE step on B200.

Workload (N=1): BASELINE config 4 -- 4096 members x 4096 P1 elements, fp64,
adaptive mask (|eta/d| > 1e-3), mixed solitary / box-uplift members.  A
"step" is one time step of every member.  W untimed warm-up steps, then K
timed steps of the streaming path (four kernels per step: K_P predictor +
criterion, K_S condensation, K_X tile chain, K_C reconstruction; the 805 MB
state is far larger than the 126 MB L2, so every step streams it from HBM).

Roofline: the dominant kernel is K_P.  Its algorithmic traffic is the state
read + write, 96 B per cell; its average launch time is
measured live with CUDA events recorded between the launches inside the
timed region (nh_stream_timing), and `traffic` is the DRAM bytes per K_P
launch from the committed `ncu --set full` capture (profiles/kp_traffic.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload config4|config5] [--mode adaptive|global]

Multi-GPU (torchrun, one process per GPU): members are sharded over ranks
with no collective on the step path (weak scaling: every rank steps its own
4096-member shard); time = max over ranks of the device-timed region.

--impl reference times the CPU oracle port (oracle/nhswe_oracle.py, the
restatement of the reference's numpy/LAPACK step, bit-exact with it) on all
host cores: one member per process, each advancing K steps.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_CELL_STEP = 96          # read + write of 6 fp64 state values
METRIC = "cell-steps/sec (ensemble x cells x steps) incl. NH correction"


def _kp_traffic():
    """DRAM bytes (read + write) per K_P launch from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "kp_traffic.json")) as f:
            d = json.load(f)
        return float(d["dram_bytes_per_launch"]), d
    except Exception:
        return None, None


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p.get("sm_max_mhz", 1965.0)), "measured"
    except Exception:
        return 6650.0, 1965.0, "fallback"


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        load = [s for s in sm if mx and s > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ workloads

def build_workload(name: str, rank: int, world: int):
    """Member table + device initial state for this rank's shard."""
    import numpy as np
    import torch
    from paper_2505_17025_b200 import configs
    from paper_2505_17025_b200._device import dev
    if name == "config4":
        per = 4096
        cfg = configs.Config4(n_members=per * world)
        idx = range(rank * per, (rank + 1) * per)
    else:
        cfg = configs.Config5()
        per = cfg.n_members // world
        idx = range(rank * per, (rank + 1) * per)
    recs = cfg.records(list(idx))
    h, hu, hw = init_device(cfg, recs, list(idx))
    return cfg, recs, h, hu, hw


def init_device(cfg, recs, idx):
    """Initial state built on the GPU: solitary formulas with torch, still water
    from the bottom-model kernel."""
    import numpy as np
    import torch
    from paper_2505_17025_b200 import _lib
    from paper_2505_17025_b200._device import dev, ptr, require_cuda, stream_ptr, upload_members
    from paper_2505_17025_b200.configs import solitary_state
    lib = require_cuda()
    B, N = len(idx), cfg.n_elements
    h = torch.empty((B, N, 2), dtype=torch.float64, device="cuda")
    hu = torch.zeros_like(h)
    hw = torch.zeros_like(h)
    kinds = recs["bottom_kind"]
    e = torch.arange(N, dtype=torch.float64, device="cuda")
    still = np.flatnonzero(kinds != _lib.BOTTOM_FLAT)
    sol = np.flatnonzero(kinds == _lib.BOTTOM_FLAT)
    if sol.size:
        ms = [cfg.member(idx[i]) for i in sol]
        dx = torch.as_tensor([m.grid.dx for m in ms], device="cuda", dtype=torch.float64)[:, None, None]
        h0 = torch.as_tensor([m.bathymetry.h0 for m in ms], device="cuda", dtype=torch.float64)[:, None, None]
        a = torch.as_tensor([m.init_params["a"] for m in ms], device="cuda", dtype=torch.float64)[:, None, None]
        x0 = torch.as_tensor([m.init_params["x0"] for m in ms], device="cuda", dtype=torch.float64)[:, None, None]
        edges = dx[:, :, 0:1] * e[None, :, None]
        nodes = torch.cat([edges, edges + dx[:, :, 0:1]], -1)
        hs, qs, ws = solitary_state(torch, nodes, h0, a, x0, dx[..., 0])
        si = torch.as_tensor(sol, device="cuda")
        h[si], hu[si], hw[si] = hs, qs, ws
    for c0 in range(0, still.size, 2048):   # bounded temporaries (config 5: 65536 x 16384)
        sel = still[c0:c0 + 2048]
        sub = recs[sel]
        m = upload_members(sub)
        xl = torch.as_tensor(sub["x_left"], device="cuda", dtype=torch.float64)[:, None]
        dxs = torch.as_tensor(sub["dx"], device="cuda", dtype=torch.float64)[:, None]
        eps = torch.as_tensor(sub["eps"], device="cuda", dtype=torch.float64)[:, None]
        edges = xl + dxs * e[None, :]
        x = torch.stack([edges + eps, (edges + dxs) - eps], -1).reshape(len(sel), 2 * N)
        t = torch.zeros(len(sel), dtype=torch.float64, device="cuda")
        out = torch.empty((6, len(sel), 2 * N), dtype=torch.float64, device="cuda")
        # per-member points: the kernel reads x[b*P + i]
        rc = lib.nh_bottom_sample(ptr(m), len(sel), ptr(x), 2 * N, ptr(t), ptr(out), stream_ptr())
        assert rc == 0
        si = torch.as_tensor(sel, device="cuda")
        h[si] = out[0].reshape(len(sel), N, 2)
        del out, x, edges
    torch.cuda.synchronize()
    return h, hu, hw


# ------------------------------------------------------------------ CPU baseline

def _cpu_worker(args):
    wl, i, n_steps, mode = args
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from threadpoolctl import threadpool_limits
    import numpy as np
    from oracle import nhswe_oracle as O
    from paper_2505_17025_b200 import configs
    from tests.helpers import oracle_depth, oracle_member
    with threadpool_limits(1):
        cfg = configs.Config4(n_members=max(4096, i + 1)) if wl == "config4" else configs.Config5()
        m = cfg.member(i)
        h, hu, hw = cfg.host_state(i, oracle_depth)
        mem = oracle_member(m.grid, m.bathymetry, m.bcs, m.dt)
        O.step(mem, h, hu, hw, 0.0, mode)        # warm caches / lru templates
        t0 = time.perf_counter()
        r = O.run(mem, h, hu, hw, n_steps, mode=mode)
        dt = time.perf_counter() - t0
    return cfg.n_elements * n_steps, dt, r.fraction_mean


def cpu_baseline(workload: str, mode: str, n_steps: int, procs: int | None = None):
    """Oracle port on the host cores: one member per process, n_steps each."""
    import multiprocessing as mp
    procs = procs or min(os.cpu_count() or 1, 32)
    jobs = [(workload, 2 * k + (k % 2), n_steps, mode) for k in range(procs)]
    ctx = mp.get_context("spawn")
    t0 = time.perf_counter()
    with ctx.Pool(procs) as pool:
        res = pool.map(_cpu_worker, jobs)
    wall = time.perf_counter() - t0
    cells = sum(r[0] for r in res)
    slowest = max(r[1] for r in res)
    return {"value": cells / slowest, "unit": "cell-steps/s", "cores": procs, "kind": "port",
            "sample": f"{procs} members of {workload} (one per process, BLAS 1 thread), "
                      f"{n_steps} {mode} steps each; rate = cells x steps / slowest process",
            "wall_s": wall, "slowest_s": slowest, "mask_fraction": statistics.mean(r[2] for r in res)}


# ------------------------------------------------------------------ arms

def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def run_reference(args):
    rank, world, _ = dist_env()
    if world > 1 and rank != 0:
        return
    n_steps = args.steps
    base = cpu_baseline(args.workload, args.mode, n_steps)
    from paper_2505_17025_b200 import configs
    cfg = configs.Config4() if args.workload == "config4" else configs.Config5()
    line = {"impl": "reference", "metric": METRIC, "value": base["value"], "unit": "cell-steps/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            # one whole-workload step (all members) at the sampled rate
            "ms_per_step": 1e3 * cfg.n_members * cfg.n_elements / base["value"],
            "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.workload, "mode": args.mode,
                       "members": cfg.n_members, "cells_per_member": cfg.n_elements,
                       "sample": base["sample"]},
            "cpu_baseline": {k: base[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": base["value"], "unit": "cell-steps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_b200(args):
    import numpy as np
    import torch
    import torch.distributed as tdist
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        tdist.init_process_group("nccl")
    from paper_2505_17025_b200 import Criterion, Ensemble, _lib
    from paper_2505_17025_b200 import _device as D
    from paper_2505_17025_b200._device import read_status
    cfg, recs, h, hu, hw = build_workload(args.workload, rank, world)
    B, N = h.shape[0], h.shape[1]
    crit = Criterion("eta_over_d", 1e-3, False)
    ens = Ensemble(recs, h, hu, hw)
    # warm-up steps (untimed)
    ens.advance(args.warmup, args.mode, crit)
    torch.cuda.synchronize()
    ens.reset_status()
    # the state after the warm-up, in pinned host memory: the e2e leg below
    # runs the same K steps as timed region 1 from the host (same window of
    # the workload, so the two numbers differ only by the API and transfers)
    host0 = None
    if args.e2e and B * N * 48 <= 16e9:
        host0 = [x.cpu().pin_memory() for x in (ens.h, ens.hu, ens.hw, ens.time)]
    path = ens.choose_path(args.mode, crit)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        tdist.barrier()
    torch.cuda.synchronize()
    # timed region 1 (the headline value): the time loop as the library runs
    # it by default, a captured CUDA graph of step pairs, no per-kernel events
    D.stream_timing(False)
    n_launch0 = D.launch_count()
    with ClockSampler(local) as clk:
        ev0.record()
        ens.advance(args.steps, args.mode, crit, path=path)
        ev1.record()
        ev1.synchronize()
    ms = ev0.elapsed_time(ev1)
    torch.cuda.synchronize()
    launches = D.launch_count() - n_launch0
    # timed region 2 (roofline and kernel shares): the next K steps as plain
    # launches with a CUDA event between consecutive kernels on the launching
    # stream (nh_stream_timing)
    ktimes, ms_ev = {}, None
    ksteps = args.kernel_steps if args.kernel_steps > 0 else args.steps
    if path == "stream":
        D.stream_timing(True)
        ev0.record()
        ens.advance(ksteps, args.mode, crit, path=path)
        ev1.record()
        ev1.synchronize()
        ms_ev = ev0.elapsed_time(ev1)
        ktimes = D.stream_kernel_times()
        D.stream_timing(False)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
        ms = float(t.item())
    st = read_status(ens.status)
    ok = bool((st["error_key"] == _lib.STATUS_OK_KEY).all())
    from paper_2505_17025_b200._device import decode_error
    bad = np.flatnonzero(st["error_key"] != _lib.STATUS_OK_KEY)
    errors = {"count": int(bad.size),
              "first": [[int(i), *decode_error(st["error_key"][i])] for i in bad[:4]]}
    steps_run = args.steps + (ksteps if ms_ev is not None else 0)   # both timed regions
    frac = float(st["flagged"].sum()) / (B * N * max(steps_run, 1))
    cells = B * N * args.steps * world
    value = cells / (ms * 1e-3)
    peak, _, peak_kind = _peaks()
    if path == "stream":
        kp_ms, kp_n = ktimes["nh_stream_kp"]
        kp_avg = kp_ms / max(kp_n, 1)
        kname = "nh_stream_kp"
    else:   # resident path: one launch covers every step
        kp_avg, kp_n, kname = ms / max(args.steps, 1), args.steps, "nh_step_kernel (per step)"
    # cells per K_P launch: the whole ensemble, or one member block when it is
    # run in blocks (config 5 at full size)
    kp_bytes = BYTES_PER_CELL_STEP * B * N * (ksteps if path == "stream" else args.steps) / max(kp_n, 1)
    achieved = kp_bytes / (kp_avg * 1e-3) / 1e9
    traffic, traffic_src = _kp_traffic()
    if traffic_src and traffic_src.get("workload", "config4") != args.workload:
        traffic, traffic_src = None, None     # the committed capture is of another shape
    shares = {k: {"ms_total": v[0], "launches": v[1], "share": v[0] / ms_ev}
              for k, v in ktimes.items() if v[1]}

    # end to end through the public API: pinned host state -> device, K steps
    # (Ensemble.advance -> nh_stream_advance), device -> pinned host, timed on
    # the wall clock around synchronizes (the larger of wall and event time).
    e2e = None
    if args.e2e and B * N * 48 > 16e9:
        e2e = {"skipped": "state larger than 16 GB; e2e host round trip measured on config4"}
    elif args.e2e:
        hh = host0
        ho = [torch.empty_like(x).pin_memory() for x in hh[:3]]
        torch.cuda.synchronize()
        if world > 1:
            tdist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0 = time.perf_counter()
        e0.record()
        dh = [x.to("cuda", non_blocking=True) for x in hh]   # h, hu, hw, time
        ens2 = Ensemble(recs, *dh)
        ens2.advance(args.steps, args.mode, crit)
        for dst, src in zip(ho, (ens2.h, ens2.hu, ens2.hw)):
            dst.copy_(src, non_blocking=True)
        e1.record()
        e1.synchronize()
        ems = max(e0.elapsed_time(e1), (time.perf_counter() - w0) * 1e3)
        if world > 1:
            t = torch.tensor([ems], device="cuda")
            tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
            ems = float(t.item())
        nbytes_in = sum(x.numel() * 8 for x in hh)
        nbytes = sum(x.numel() * 8 for x in ho)
        e2e = {"value": cells / (ems * 1e-3), "unit": "cell-steps/s",
               "h2d_bytes_per_step": nbytes_in / args.steps,
               "d2h_bytes_per_step": nbytes / args.steps,
               "call": "Ensemble(host state + times -> HBM).advance(K) -> host state, one call "
                       "per K steps, from the post-warm-up state (the K steps of region 1)"}
        del dh, ens2, ho, host0

    cpu = None
    if rank == 0 and world == 1 and args.cpu_steps > 0:
        cpu = cpu_baseline(args.workload, args.mode, args.cpu_steps)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "cell-steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": args.workload, "mode": args.mode, "members": B * world,
                       "cells_per_member": N, "members_per_gpu": B,
                       "criterion": "eta_over_d k_nh=1e-3", "mask_fraction": frac,
                       "path": path,
                       "l2": f"inputs > L2: state {B * N * 48 / 1e6:.0f} MB/GPU vs 126 MB L2, "
                             "streamed every step",
                       "member_chunk": ens.stream_chunk() if path == "stream" else B,
                       "status_ok": ok, "errors": errors},
            "gpu_launches": launches,
            "time_loop": "CUDA graph of step pairs (nh_stream_advance), timed region 1",
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak,
                         "traffic": traffic if path == "stream" else None,
                         "kernel": kname, "kernel_ms_avg": kp_avg, "kernel_launches": kp_n,
                         "algorithmic_bytes_per_launch": kp_bytes,
                         "peak_kind": peak_kind,
                         "traffic_source": traffic_src.get("source") if traffic_src else None,
                         # the binding resource of K_P in the same ncu capture
                         "ncu_fp64_pipe_active_pct": (traffic_src or {}).get("fp64_pipe_active_pct"),
                         "ncu_issue_active_pct": (traffic_src or {}).get("issue_active_pct"),
                         "event_timed_ms_per_step": (ms_ev / ksteps) if ms_ev else None,
                         "note": "algorithmic 96 B/cell (state read + write) x B*N cells per "
                                 "launch / event-timed launch (timed region 2: the K steps after "
                                 "the headline region, plain launches with CUDA events between "
                                 "kernels); K_P is fp64-issue bound, not HBM bound (profiles/)"},
            "kernel_shares": shares,
            "clocks": clk.summary(),
        }
        if e2e:
            line["e2e"] = e2e
        if cpu:
            line["cpu_baseline"] = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
        print(json.dumps(line), flush=True)
    if world > 1:
        tdist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="config4", choices=["config4", "config5"])
    ap.add_argument("--mode", default="adaptive", choices=["adaptive", "global"])
    ap.add_argument("--cpu-steps", type=int, default=1000)
    ap.add_argument("--no-e2e", dest="e2e", action="store_false")
    ap.add_argument("--kernel-steps", type=int, default=0,
                    help="steps of timed region 2 (per-kernel events); default: --steps")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
