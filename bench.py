#!/usr/bin/env python
"""Benchmark: cell-steps/s of the adaptive NH-SWE step on B200.

Workload (N=1): BASELINE config 5 -- 65536 landslide members x 16384 P1
elements, fp64, adaptive mask (|eta/d| > 1e-3), the largest configuration
BASELINE runs on one GPU.  A "step" is one time step of every member.  The
ensemble starts from rest, so `--spinup` untimed steps first carry it into
its flagged regime, then W untimed warm-up steps, then K timed
steps of the streaming path (K_P predictor + criterion, K_S condensation,
K_X tile chain, K_C reconstruction; the 51.5 GB state is far larger than the
126 MB L2, so every step streams it from HBM).

Legs of one run (all on the same ensemble, one after the other):
  value     K steps, the CUDA-graph time loop as the library runs it
  roofline  the next K steps with CUDA events between the kernels: K_P's
            average launch time -> algorithmic GB/s (96 B per cell)
  global    --global-steps steps in global mode on the same state (the
            reference's paired adaptive/global timing, cli.py:259-267)
  e2e       K steps through driver.advance_host from pinned HOST memory:
            copy-in, compute and copy-out pipelined over member blocks
  cpu       the reference's own step (nhswe from baseline/_ref) on the host
            cores, one sampled member per process (rank 0, N=1 only)

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload config5|config4] [--mode adaptive|global]

Multi-GPU (torchrun, one process per GPU): config 5 is sharded evenly over
the ranks with parallel.shard (a member's parameters depend on its index
only, so the shards together are exactly the N=1 ensemble; "scaling":
"strong"), no collective on the step path; time = max over ranks of the
device-timed region; an untimed gather_summaries collects per-member results.

--impl reference times the reference's own adaptive_step (the unmodified
package installed into baseline/_ref) on the host cores, one member per
process over a bounded sample of the same workload window.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BYTES_PER_CELL_STEP = 96          # read + write of 6 fp64 state values
METRIC = "cell-steps/sec (ensemble x cells x steps) incl. NH correction"
SPINUP = {"config5": 1000, "config4": 0}


def _profile_json(name):
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            return json.load(f)
    except Exception:
        return None


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return 7672.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)   # first sample before the region starts
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
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
        for l in self.lines:
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

def get_config(name: str, **kw):
    from paper_2505_17025_b200 import configs
    return configs.Config5(**kw) if name == "config5" else configs.Config4(**kw)


def workload_members(name: str, rank: int, world: int, members=None, **kw):
    """(config, member indices, nh_member records) of this rank's shard:
    parallel.shard of the workload's members, or the given indices.  A
    member's record depends on its index only, so the shards of any world
    size concatenate to the N=1 table (tests/test_parallel.py)."""
    from paper_2505_17025_b200.parallel import shard
    cfg = get_config(name, **kw)
    idx = list(members) if members is not None else list(shard(cfg.n_members, world, rank))
    return cfg, idx, cfg.records(idx)


def build_workload(name: str, rank: int, world: int, members=None):
    """Member table + device initial state of this rank's shard."""
    cfg, idx, recs = workload_members(name, rank, world, members)
    h, hu, hw = init_device(cfg, recs, idx)
    return cfg, recs, h, hu, hw


def init_device(cfg, recs, idx):
    """Initial state built on the GPU: solitary formulas with torch, still water
    from the bottom-model kernel."""
    import numpy as np
    import torch
    from paper_2505_17025_b200 import _lib
    from paper_2505_17025_b200._device import ptr, require_cuda, stream_ptr, upload_members
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


# ------------------------------------------------------------------ CPU legs

def _cpu_worker(args):
    """One member through the reference's own adaptive_step: `spin` untimed
    steps (the same workload window as the GPU legs), then `n_steps` timed."""
    wl, i, spin, n_steps, mode = args
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from threadpoolctl import threadpool_limits
    with threadpool_limits(1):
        cfg = get_config(wl)
        try:
            if os.environ.get("NH_CPU_ARM") == "port":   # tests: force the fallback leg
                raise ImportError("oracle port requested")
            from tests.harness.ref_bridge import reference_member
            R, grid, bathy, bcs, dt, st = reference_member(cfg, i)
            crit = R.Criterion("eta_over_d") if mode == "adaptive" else None
            kind = "reference"

            def step(s):
                return R.adaptive_step(s, dt, bathy, bcs, mode=mode, crit=crit,
                                       cfl_warn=False).state
        except Exception:
            # the reference is not installed: the oracle port (bit-exact restatement)
            from oracle import nhswe_oracle as O
            from tests.helpers import oracle_depth, oracle_member
            m = cfg.member(i)
            mem = oracle_member(m.grid, m.bathymetry, m.bcs, m.dt)
            h, hu, hw = cfg.host_state(i, oracle_depth)
            st = (h, hu, hw, 0.0)
            kind = "port"

            def step(s):
                r = O.step(mem, s[0], s[1], s[2], s[3], mode)
                return (r.h, r.hu, r.hw, s[3] + m.dt)
        for _ in range(spin):
            st = step(st)
        t0 = time.perf_counter()
        for _ in range(n_steps):
            st = step(st)
        dt_s = time.perf_counter() - t0
    return cfg.n_elements * n_steps, dt_s, kind


def cpu_sample(workload: str, mode: str, spin: int, n_steps: int, procs: int | None = None):
    """The reference's step on the host cores: one member per process."""
    import multiprocessing as mp
    procs = procs or min(os.cpu_count() or 1, 32)
    cfg = get_config(workload)
    stride = max(1, cfg.n_members // procs)
    jobs = [(workload, k * stride + (k % 2), spin, n_steps, mode) for k in range(procs)]
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(procs) as pool:
        res = pool.map(_cpu_worker, jobs)
    wall = time.perf_counter() - t0
    cells = sum(r[0] for r in res)
    slowest = max(r[1] for r in res)
    kind = res[0][2]
    who = ("the reference's own adaptive_step (nhswe, baseline/_ref)" if kind == "reference"
           else "the oracle port (reference not installed)")
    return {"value": cells / slowest, "unit": "cell-steps/s", "cores": procs, "kind": kind,
            "sample": f"{procs} members of {workload} (one per process, BLAS 1 thread) through "
                      f"{who}: {spin} untimed spin-up steps, then {n_steps} timed {mode} steps "
                      f"each; rate = cells x steps / slowest process",
            "ms_per_member_step": 1e3 * slowest / n_steps, "wall_s": wall, "slowest_s": slowest}


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def run_reference(args):
    rank, world, _ = dist_env()
    if world > 1 and rank != 0:
        return
    spin = args.spinup + args.warmup
    base = cpu_sample(args.workload, args.mode, spin, args.steps)
    cfg = get_config(args.workload)
    line = {"impl": "reference", "metric": METRIC, "value": base["value"], "unit": "cell-steps/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            # the timed sample's own step time (every process advances its
            # member by one step in parallel)
            "ms_per_step": base["ms_per_member_step"],
            "ms_per_step_full_workload_extrapolated":
                1e3 * cfg.n_members * cfg.n_elements / base["value"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": args.workload, "mode": args.mode,
                       "members": cfg.n_members, "cells_per_member": cfg.n_elements,
                       "spinup_steps": args.spinup, "sample": base["sample"]},
            "cpu_baseline": {k: base[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": base["value"], "unit": "cell-steps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm

def run_b200(args):
    import numpy as np
    import torch
    import torch.distributed as tdist
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_2505_17025_b200 import Criterion, Ensemble, _lib, parallel
    from paper_2505_17025_b200 import _device as D
    from paper_2505_17025_b200._device import decode_error, read_status
    from paper_2505_17025_b200.driver import advance_host
    cfg, recs, h, hu, hw = build_workload(args.workload, rank, world)
    B, N = h.shape[0], h.shape[1]
    crit = Criterion("eta_over_d", 1e-3, False)
    ens = Ensemble(recs, h, hu, hw)
    if args.spinup:
        ens.advance(args.spinup, args.mode, crit)
    ens.advance(args.warmup, args.mode, crit)      # warm-up steps (untimed)
    torch.cuda.synchronize()
    ens.reset_status()
    path = ens.choose_path(args.mode, crit)
    # the state after the warm-up, in pinned host memory, for the e2e leg
    # (the same window of the workload as timed region 1)
    host0, e2e_note = None, None
    if args.e2e:
        import psutil
        need = B * N * 48 + B * 8
        if psutil.virtual_memory().available > 1.25 * need:
            host0 = [torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
                     for x in (ens.h, ens.hu, ens.hw, ens.time)]
            for dst, src in zip(host0, (ens.h, ens.hu, ens.hw, ens.time)):
                dst.copy_(src)
        else:
            e2e_note = f"host RAM below 1.25 x {need / 1e9:.1f} GB of state"
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
    if world > 1:
        tdist.barrier()
    torch.cuda.synchronize()
    ms = parallel.max_over_ranks(ev0.elapsed_time(ev1), device="cuda")
    launches = D.launch_count() - n_launch0
    st1 = read_status(ens.status)
    frac = float(st1["flagged"].sum()) / (B * N * args.steps)
    # timed region 2 (roofline and kernel shares): the next K steps as plain
    # launches with a CUDA event between consecutive kernels on the launching
    # stream (nh_stream_timing)
    ktimes, ms_ev = {}, None
    ksteps = args.kernel_steps if args.kernel_steps > 0 else args.steps
    D.stream_timing(True)
    ev0.record()
    ens.advance(ksteps, args.mode, crit, path=path)
    ev1.record()
    ev1.synchronize()
    ms_ev = ev0.elapsed_time(ev1)
    ktimes = D.stream_kernel_times()
    D.stream_timing(False)
    # global mode on the same ensemble (paired timing, reference cli.py:259-267)
    glob = None
    if args.global_steps > 0 and args.mode == "adaptive":
        torch.cuda.synchronize()
        ev0.record()
        ens.advance(args.global_steps, "global", None, path=path)
        ev1.record()
        ev1.synchronize()
        gms = parallel.max_over_ranks(ev0.elapsed_time(ev1), device="cuda") / args.global_steps
        glob = {"ms_per_step": gms, "value": B * N * world / (gms * 1e-3),
                "steps": args.global_steps,
                "global_over_adaptive_step_time": gms / (ms / args.steps)}
    st = read_status(ens.status)
    ok = bool((st["error_key"] == _lib.STATUS_OK_KEY).all())
    bad = np.flatnonzero(st["error_key"] != _lib.STATUS_OK_KEY)
    errors = {"count": int(bad.size),
              "first": [[int(i), *decode_error(st["error_key"][i])] for i in bad[:4]]}
    cells = B * N * args.steps * world
    value = cells / (ms * 1e-3)
    peak, peak_kind = _peaks()
    kp_ms, kp_n = ktimes["nh_stream_kp"]
    kp_avg = kp_ms / max(kp_n, 1)
    # cells per K_P launch: the whole shard, or one member block when the
    # shard runs in blocks through one workspace
    kp_bytes = BYTES_PER_CELL_STEP * B * N * ksteps / max(kp_n, 1)
    achieved = kp_bytes / (kp_avg * 1e-3) / 1e9
    traffic_src = _profile_json(f"kp_traffic_{args.workload}.json")
    traffic = None
    if traffic_src:   # DRAM bytes per launch of the committed capture, per cell of this launch
        traffic = traffic_src["dram_bytes_per_cell"] * kp_bytes / BYTES_PER_CELL_STEP
    shares = {k: {"ms_total": v[0], "launches": v[1], "share": v[0] / ms_ev}
              for k, v in ktimes.items() if v[1]}

    # end to end through the public API: the post-warm-up state in pinned
    # HOST memory -> driver.advance_host (member blocks: copy-in, K steps,
    # copy-out, pipelined on three streams over three device buffers) -> host; wall clock around
    # synchronizes, max over ranks
    e2e = {"skipped": e2e_note} if e2e_note else None
    if host0 is not None:
        ens.release_workspace()   # advance_host streams through its own buffers
        torch.cuda.synchronize()
        if world > 1:
            tdist.barrier()
        w0 = time.perf_counter()
        advance_host(recs, *host0, args.steps, args.mode, crit, block=args.e2e_block)
        ems = parallel.max_over_ranks((time.perf_counter() - w0) * 1e3, device="cuda")
        nbytes = sum(x.numel() * 8 for x in host0)
        e2e = {"value": cells / (ems * 1e-3), "unit": "cell-steps/s",
               "h2d_bytes_per_step": nbytes / args.steps,
               "d2h_bytes_per_step": nbytes / args.steps,
               "ms": ems, "block_members": args.e2e_block,
               "call": "driver.advance_host(pinned host h, hu, hw, time; K steps): member blocks "
                       "copied in, stepped and copied out, pipelined on 3 CUDA streams and 3 device buffers (both copy directions overlap the compute); from the "
                       "post-warm-up state (the K steps of region 1)"}
        del host0

    # per-member summaries on rank 0 (untimed; the only other collective)
    summ = parallel.gather_summaries({"time": ens.time.cpu().numpy(),
                                      "flagged": st["flagged"].astype(np.int64),
                                      "ok": (st["error_key"] == _lib.STATUS_OK_KEY)})
    cpu = None
    if rank == 0 and world == 1 and args.cpu_steps > 0:
        cpu = cpu_sample(args.workload, args.mode, args.spinup + args.warmup, args.cpu_steps)
    if rank == 0:
        fp64 = _profile_json("fp64_peak.json") or {}
        line = {
            "metric": METRIC, "value": value, "unit": "cell-steps/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": args.workload, "mode": args.mode,
                       "members": int(len(summ["time"])), "cells_per_member": N,
                       "members_per_gpu": B, "parallelism": f"member shards x{world}",
                       "criterion": "eta_over_d k_nh=1e-3", "spinup_steps": args.spinup,
                       "mask_fraction": frac, "path": path,
                       "l2": f"inputs > L2: state {B * N * 48 / 1e9:.1f} GB/GPU vs 126 MB L2, "
                             "streamed every step",
                       "member_chunk": ens.stream_chunk() if path == "stream" else B,
                       "status_ok": ok and bool(summ["ok"].all()), "errors": errors},
            "gpu_launches": launches,
            "time_loop": "CUDA graph of step pairs (nh_stream_advance), timed region 1",
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "nh_stream_kp", "kernel_ms_avg": kp_avg,
                         "kernel_launches": kp_n,
                         "algorithmic_bytes_per_launch": kp_bytes, "peak_kind": peak_kind,
                         "traffic_source": (traffic_src or {}).get("source"),
                         "fp64": {"kp_fp64_pipe_active_pct":
                                      (traffic_src or {}).get("fp64_pipe_active_pct"),
                                  "kp_issue_active_pct": (traffic_src or {}).get("issue_active_pct"),
                                  "kp_fp64_arith_frac_of_peak":
                                      (traffic_src or {}).get("fp64_arith_frac_of_peak"),
                                  "measured_dfma_peak_tflops": fp64.get("tflops"),
                                  "source": "ncu --set full of K_P (profiles/) and "
                                            "profiles/fp64_peak.json"},
                         "event_timed_ms_per_step": ms_ev / ksteps,
                         "note": "algorithmic 96 B/cell (state read + write) x cells per launch / "
                                 "event-timed launch (timed region 2: the K steps after the "
                                 "headline region, plain launches with CUDA events between "
                                 "kernels)"},
            "kernel_shares": shares,
            "clocks": clk.summary(),
        }
        if glob:
            line["global"] = glob
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
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="config5", choices=["config5", "config4"])
    ap.add_argument("--mode", default="adaptive", choices=["adaptive", "global"])
    ap.add_argument("--spinup", type=int, default=None,
                    help="untimed steps before the warm-up (default: 1000 for config5, which "
                         "starts from rest, 0 for config4)")
    ap.add_argument("--global-steps", type=int, default=10)
    ap.add_argument("--cpu-steps", type=int, default=200)
    ap.add_argument("--no-e2e", dest="e2e", action="store_false")
    ap.add_argument("--e2e-block", type=int, default=2048)
    ap.add_argument("--kernel-steps", type=int, default=0,
                    help="steps of timed region 2 (per-kernel events); default: --steps")
    args = ap.parse_args()
    if args.spinup is None:
        args.spinup = SPINUP[args.workload]
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
