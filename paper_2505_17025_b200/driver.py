"""Time loop entry points (reference driver.py:50-103) and the batched API.

``simulate`` keeps the reference signature.  The whole fixed-dt loop is one
launch sequence of the streaming step kernels (a CUDA graph of step pairs,
DESIGN.md §4.1), with gauges and flag bits recorded on the device, so there
is no per-step host synchronisation.  ``loop_time`` is device time (CUDA
events) of the stepping launches, the analogue of the reference's loop-only
perf_counter.

``Ensemble`` / ``simulate_ensemble`` are the batched extension (SURVEY.md
§8(b)): B independent channels of equal N with per-member grids, dt, bottoms
and boundary kinds, stepped together; members shard across GPUs with no
communication on the step path (``paper_2505_17025_b200.parallel``).
"""

from __future__ import annotations

import math
import warnings
from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _lib
from .adaptivity import Criterion, NonHydroMask, contiguous_ranges
from .bathymetry import RHO_WATER
from .corrector import FluxCoefficients
from .grid import FlowState, NodalField
from .scenarios import ScenarioSpec

_MODES = {"hydrostatic": _lib.MODE_HYDROSTATIC, "global": _lib.MODE_GLOBAL,
          "adaptive": _lib.MODE_ADAPTIVE}
# Longest member of the streaming path: K_X chains a member's tiles with one
# warp, 8 tiles of 120 elements per lane (NH_STREAM_MAXCPL).  Longer members
# (the reference has no limit) run the m-node kernels, whose chain is one
# thread per member: correct at any length, at coverage speed.
STREAM_MAX_ELEMENTS = 32 * 8 * 120


@dataclass
class RunResult:
    spec: ScenarioSpec
    mode: str
    criterion: Criterion | None
    final_state: FlowState
    final_p: NodalField | None
    final_mask: NonHydroMask | None
    gauge_times: np.ndarray
    gauge_eta: np.ndarray
    mask_history: list
    mask_fraction_mean: float
    loop_time: float

    def config_echo(self) -> dict:
        grid = self.spec.grid
        c = self.criterion
        return {"scenario": self.spec.name, "mode": self.mode,
                "criterion": c.kind if c else None, "k_nh": c.k_nh if c else None,
                "enlarge": c.enlarge if c else None, "dt": self.spec.dt,
                "t_end": self.spec.t_end, "n_elements": grid.n_elements,
                "poly_order": grid.poly_order, "x_left": grid.x_left,
                "x_right": grid.x_right, "gauges": list(self.spec.gauges)}


class Ensemble:
    """Device-resident state of B channels with N elements each.

    members: nh_member records (numpy MEMBER_DTYPE, length B); h, hu, hw:
    CUDA float64 tensors (B, N, 2); time: CUDA float64 (B,).
    """

    def __init__(self, records: np.ndarray, h, hu, hw, time=None, pm_records=None):
        T = D.torch()
        D.require_cuda()
        self.records = np.ascontiguousarray(records)
        self.members = D.upload_members(self.records)
        self.B, self.N = int(h.shape[0]), int(h.shape[1])
        self.M = int(h.shape[2])   # nodes per element (poly_order + 1)
        # m-node operators (D.pm_record per member): required for M != 2, and
        # selects the generic m-node kernels for M == 2 with path="generic"
        self.pm = None if pm_records is None else D.upload_members(
            np.ascontiguousarray(pm_records))
        if self.M != 2 and self.pm is None:
            raise ValueError("orders p > 1 need the members' pm_records (D.pm_record)")
        self.h, self.hu, self.hw = h, hu, hw
        self.time = time if time is not None else T.zeros(self.B, dtype=T.float64, device="cuda")
        self.status = D.new_status(self.B)

    @classmethod
    def from_host(cls, records, h, hu, hw, time=None, pm_records=None):
        t = D.dev(np.zeros(len(records)) if time is None else np.asarray(time, dtype=np.float64))
        return cls(records, D.dev(h), D.dev(hu), D.dev(hw), t, pm_records)

    def reset_status(self):
        self.status = D.new_status(self.B)

    def choose_path(self, mode: str, criterion: Criterion | None) -> str:
        """The streaming tiles with the CUDA-graph time loop: measured faster
        than the SMEM-resident cluster kernel at every size here, from one
        200-element member (17 vs 22 us/step) to config 3 (23 vs 47 us/step)
        and config 4 (0.83 vs 4.4 ms/step), tools/scenario_paths.py,
        tools/path_compare.py.  Every mode and criterion runs on it (the w /
        w_x first-step fallback of adaptivity.py:153 is K_F); the resident
        kernel stays available as path="resident".  Orders p > 1, and members
        longer than STREAM_MAX_ELEMENTS, run the m-node kernels ("generic")."""
        if self.M != 2 or self.N > STREAM_MAX_ELEMENTS:
            return "generic"
        return "stream"

    def stream_chunk(self, budget: int | None = None) -> int:
        """Members per streaming launch sequence: the whole ensemble when its
        workspace fits next to the state, else the largest block that does
        (config 5 at full size: 51.5 GB of state, 4 MB of workspace per member)."""
        if getattr(self, "_chunk", None) is None:
            lib = D.require_cuda()
            per = int(lib.nh_stream_workspace_bytes(1, self.N))
            if budget is None:
                free, _ = D.torch().cuda.mem_get_info()
                budget = int(free * 0.85)
            self._chunk = int(max(1, min(self.B, budget // per)))
        return self._chunk

    def release_workspace(self):
        """Drop the streaming workspace (re-allocated by the next advance)."""
        self._ws = None
        self._chunk = None
        D.torch().cuda.empty_cache()

    def advance(self, n_steps: int, mode: str = "adaptive", criterion: Criterion | None = None,
                flux: FluxCoefficients = FluxCoefficients(), g: float = 9.81,
                rho: float = RHO_WATER, flag_bits=None, p_out=None, path: str = "auto",
                gauges=None):
        """Enqueue n_steps time steps on the current stream (asynchronous).

        gauges = (int32 device tensor of flat node indices e*2 + j [G],
        float64 device tensor [n_steps][B][G]) records h at those nodes after
        every step on the device (reference driver.py:58-69)."""
        if mode not in _MODES:
            raise ValueError(f"unknown mode {mode!r}")
        if mode == "adaptive" and criterion is None:
            raise ValueError("adaptive mode requires a criterion")
        with D.nvtx_range(f"nhswe.advance[{mode}] B={self.B} N={self.N} steps={n_steps}"):
            self._advance(n_steps, mode, criterion, flux, g, rho, flag_bits, p_out, path, gauges)

    def _advance(self, n_steps, mode, criterion, flux, g, rho, flag_bits, p_out, path, gauges):
        c = criterion if criterion is not None else Criterion("eta_over_d")
        sch = D.scheme(_MODES[mode], c.kind, c.k_nh, c.enlarge, flux, g, rho)
        if path == "auto":
            path = self.choose_path(mode, criterion)
        if path == "stream" and self.N > STREAM_MAX_ELEMENTS:
            path = "generic"   # longer members than K_X chains: the m-node kernels (no cap)
        if path == "generic" and self.pm is None and self.M == 2:
            self.pm = D.upload_members(D.pm_from_members(self.records))
        if mode != "hydrostatic" and (flux.c12 != -0.5 or flux.c22 != 0.0):
            # an LDG flux outside the alternating family: the m-node kernels'
            # band solve per range (P1 members: operators from their records)
            path = "generic"
            if self.pm is None and self.M == 2:
                self.pm = D.upload_members(D.pm_from_members(self.records))
        if self.M != 2 or path == "generic":   # m-node kernels (orders p > 1)
            if self.pm is None:
                raise ValueError("path='generic' needs pm_records")
            D.pm_advance(self.members, self.pm, self.h, self.hu, self.hw, self.time, n_steps,
                         sch, self.status, flag_bits, p_out, gauges)
            return
        if path == "stream":
            chunk = self.stream_chunk()
            if getattr(self, "_ws", None) is None:
                self._ws = D.stream_workspace(chunk, self.N)
            if chunk >= self.B:
                D.stream_advance(self.members, self.h, self.hu, self.hw, self.time, n_steps, sch,
                                 self.status, self._ws, flag_bits, p_out, gauges)
                return
            # members are independent: run the ensemble as consecutive member
            # blocks through one workspace (member-major state -> contiguous views)
            if flag_bits is not None or gauges is not None:
                raise ValueError("per-step flag bits and gauges need the whole ensemble in one "
                                 "workspace")
            mb, sb = self.members, self.status
            rec, st = _lib.MEMBER_DTYPE.itemsize, _lib.STATUS_DTYPE.itemsize
            for c0 in range(0, self.B, chunk):
                c1 = min(self.B, c0 + chunk)
                D.stream_advance(mb[c0 * rec:c1 * rec], self.h[c0:c1], self.hu[c0:c1],
                                 self.hw[c0:c1], self.time[c0:c1], n_steps, sch,
                                 sb[c0 * st:c1 * st], self._ws,
                                 None, None if p_out is None else p_out[c0:c1])
        else:
            D.advance(self.members, self.h, self.hu, self.hw, self.time, n_steps, sch,
                      self.status, flag_bits, p_out, gauges=gauges)

    def check(self, t0=None):
        """Raise the reference exception for the first failed member, if any."""
        st = D.read_status(self.status)
        bad = np.flatnonzero(st["error_key"] != _lib.STATUS_OK_KEY)
        if bad.size:
            i = int(bad[0])
            t0v = 0.0 if t0 is None else np.asarray(t0).ravel()[i]
            D.raise_for_status(st, t0v, self.records["dt"][i], member=i)
        return st


def block_schedule(n_members: int, block: int) -> list[int]:
    """Member-block sizes of advance_host's pipeline: short blocks at both
    ends (block/4, block/2, block, ..., block/2, block/4), so the first
    compute starts after a quarter block's copy-in and only a quarter block's
    copy-out trails the last compute.  Sums to n_members; no block exceeds
    `block` (the workspace is sized for it)."""
    block = max(1, min(n_members, block))
    ramp = [r for r in (block // 4, block // 2) if r >= 64]
    head, tail = (ramp, ramp[::-1]) if n_members >= 2 * sum(ramp) + block else ([], [])
    left = n_members - sum(head) - sum(tail)
    return (list(head) + [block] * (left // block) + ([left % block] if left % block else [])
            + list(tail))


def advance_host(records: np.ndarray, h, hu, hw, time, n_steps: int, mode: str = "adaptive",
                 criterion: Criterion | None = None, block: int | None = None,
                 flux: FluxCoefficients = FluxCoefficients(), g: float = 9.81,
                 rho: float = RHO_WATER) -> np.ndarray:
    """Advance an ensemble that lives in HOST memory by n_steps, in place.

    h, hu, hw: CPU float64 tensors (B, N, 2) -- pinned memory gives
    asynchronous copies; time: CPU float64 (B,).  The members are streamed
    through the GPU in blocks of `block` members, pipelined on three CUDA
    streams: the copy-in of block i+1 and the copy-out of block i-1 both
    overlap the K steps of block i (three device buffers, so the two copy
    directions run at the same time; one streaming workspace).
    This is the end-to-end call for ensembles kept on the host (the bench's
    e2e leg); members are independent, so the result equals
    Ensemble(...).advance(n_steps) bit for bit.  Returns the nh_status
    records of all members.
    """
    if mode not in _MODES:
        raise ValueError(f"unknown mode {mode!r}")
    if mode == "adaptive" and criterion is None:
        raise ValueError("adaptive mode requires a criterion")
    T = D.torch()
    D.require_cuda()
    B, N = int(h.shape[0]), int(h.shape[1])
    if tuple(h.shape[1:]) != (N, 2) or hu.shape != h.shape or hw.shape != h.shape:
        raise ValueError("h, hu, hw must be (B, N, 2) P1 states of equal shape")
    c = criterion if criterion is not None else Criterion("eta_over_d")
    sch = D.scheme(_MODES[mode], c.kind, c.k_nh, c.enlarge, flux, g, rho)
    block = max(1, min(B, block or 2048))
    NBUF = 3   # block i computes while block i+1 copies in and block i-1 copies out
    members = D.upload_members(np.ascontiguousarray(records))
    status = D.new_status(B)
    rec, stb = _lib.MEMBER_DTYPE.itemsize, _lib.STATUS_DTYPE.itemsize
    ws = D.stream_workspace(block, N)
    bufs = [[T.empty((block, N, 2), dtype=T.float64, device="cuda") for _ in range(3)] +
            [T.empty(block, dtype=T.float64, device="cuda")] for _ in range(NBUF)]
    host = (h, hu, hw, time)
    s_in, s_cmp, s_out = T.cuda.Stream(), T.cuda.current_stream(), T.cuda.Stream()
    s_in.wait_stream(s_cmp)
    freed = [None] * NBUF      # event: the buffer's previous copy-out finished
    starts = np.concatenate([[0], np.cumsum(block_schedule(B, block))]).astype(int)
    for i, (c0, c1) in enumerate(zip(starts[:-1], starts[1:])):
        c0, c1 = int(c0), int(c1)
        n, k = c1 - c0, i % NBUF
        buf = bufs[k]
        with T.cuda.stream(s_in):
            if freed[k] is not None:
                s_in.wait_event(freed[k])
            for dst, src in zip(buf, host):
                dst[:n].copy_(src[c0:c1], non_blocking=True)
            loaded = T.cuda.Event()
            loaded.record(s_in)
        s_cmp.wait_event(loaded)
        with T.cuda.stream(s_cmp), D.nvtx_range(f"nhswe.advance_host block {c0}:{c1}"):
            D.stream_advance(members[c0 * rec:c1 * rec], buf[0][:n], buf[1][:n], buf[2][:n],
                             buf[3][:n], n_steps, sch, status[c0 * stb:c1 * stb], ws)
            done = T.cuda.Event()
            done.record(s_cmp)
        s_out.wait_event(done)
        with T.cuda.stream(s_out):
            for dst, src in zip(host, buf):
                dst[c0:c1].copy_(src[:n], non_blocking=True)
            freed[k] = T.cuda.Event()
            freed[k].record(s_out)
    s_cmp.wait_stream(s_out)
    s_cmp.synchronize()
    for b in bufs:   # keep the buffers alive until the copies finished
        del b
    return D.read_status(status)


def simulate(spec: ScenarioSpec, initial: FlowState, mode: str,
             criterion: Criterion | None = None,
             flux: FluxCoefficients = FluxCoefficients(), rho: float = RHO_WATER,
             record_masks: bool = True) -> RunResult:
    """Run the fixed-dt loop to completion (reference driver.py:50-103)."""
    if mode not in _MODES:
        raise ValueError(f"unknown mode {mode!r}")
    if mode == "adaptive" and criterion is None:
        raise ValueError("adaptive mode requires a criterion")
    T = D.torch()
    grid = spec.grid
    n = grid.n_elements
    n_steps = spec.n_steps
    pm = grid.poly_order != 1
    rec = D.member_record(grid, spec.bathymetry, spec.bcs, spec.dt, any_order=pm)
    ens = Ensemble.from_host(rec, initial.h.values[None], initial.hu.values[None],
                             initial.hw.values[None], [initial.time],
                             D.pm_record(grid) if pm else None)
    m_nodes = grid.poly_order + 1
    nw = (n + 31) // 32
    record = record_masks and mode == "adaptive"
    gauge_idx = [grid.nearest_node(x) for x in spec.gauges]
    per_step = len(gauge_idx) > 0
    bits = None
    if mode != "hydrostatic":
        bits = T.zeros((max(n_steps, 1), 1, nw), dtype=T.int32, device="cuda")
    p = T.zeros_like(ens.h) if mode != "hydrostatic" else None
    gauge_h = np.empty((n_steps + 1, len(gauge_idx)))
    times = np.empty(n_steps + 1)
    times[0] = initial.time
    if per_step:
        gauge_h[0] = [initial.h.values[e, j] for e, j in gauge_idx]
    ev0, ev1 = T.cuda.Event(enable_timing=True), T.cuda.Event(enable_timing=True)
    loop_ms = 0.0
    if n_steps > 0:
        # one launch sequence for the whole loop; gauges are recorded on the
        # device after every step (no per-step synchronisation)
        gauges = None
        if per_step:
            nodes = T.as_tensor([m_nodes * e + j for e, j in gauge_idx], dtype=T.int32,
                                device="cuda")
            gauges = (nodes, T.empty((n_steps, 1, len(gauge_idx)), dtype=T.float64,
                                     device="cuda"))
        ev0.record()
        ens.advance(n_steps, mode, criterion, flux, spec.g, rho, bits, p, gauges=gauges)
        ev1.record()
        ev1.synchronize()
        loop_ms = ev0.elapsed_time(ev1)
        if per_step:
            gauge_h[1:] = gauges[1][:, 0, :].cpu().numpy()
    st = ens.check([initial.time])
    t = initial.time
    for s in range(n_steps):
        t = t + spec.dt
        times[s + 1] = t
    final = FlowState._wrap(NodalField._wrap(grid, ens.h[0].cpu().numpy()),
                            NodalField._wrap(grid, ens.hu[0].cpu().numpy()),
                            NodalField._wrap(grid, ens.hw[0].cpu().numpy()), float(ens.time.item()))
    if st["cfl_max"][0] > 1.0:
        warnings.warn(f"advisory CFL number {st['cfl_max'][0]:.3f} exceeded 1 during the run",
                      RuntimeWarning, stacklevel=2)
    mask_history, final_mask, final_p = [], None, None
    if mode == "hydrostatic":
        final_mask = NonHydroMask.from_flags(np.zeros(n, dtype=bool)) if n_steps else None
    elif n_steps:
        allbits = bits.cpu().numpy().view(np.uint32)[:, 0]
        last = D.bits_to_flags(allbits[-1], n)
        final_mask = NonHydroMask.from_flags(last)
        final_p = NodalField._wrap(grid, p[0].cpu().numpy()) if last.any() else None
        if record:
            flags = D.bits_to_flags(allbits, n)
            mask_history = [(s, times[s + 1], contiguous_ranges(flags[s])) for s in range(n_steps)]
    gauge_eta = np.empty((n_steps + 1, len(gauge_idx)))
    if per_step:
        gx = np.array([grid.sample_nodes[e, j] for e, j in gauge_idx])
        for r in range(n_steps + 1):
            gauge_eta[r] = gauge_h[r] - spec.bathymetry.depth(gx, times[r])
    frac = float(st["flagged"][0]) / (n_steps * n) if (n_steps and mode != "hydrostatic") else 0.0
    return RunResult(spec, mode, criterion, final, final_p, final_mask, times, gauge_eta,
                     mask_history, frac, loop_ms * 1e-3)
