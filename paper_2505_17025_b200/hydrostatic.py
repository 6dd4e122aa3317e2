"""Hydrostatic predictor entry points (reference hydrostatic.py:20-223).

``heun_step`` and ``rhs_operator`` keep the reference signatures and run the
B200 kernels: ``heun_step`` is one fused predictor step (``nh_advance`` in
hydrostatic mode), ``rhs_operator`` the standalone tendency kernel.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _lib
from .bathymetry import GRAVITY, BathymetryModel
from .grid import FlowState, NodalField


class PositivityError(RuntimeError):
    """Water column became non-positive somewhere (hydrostatic.py:20-26)."""

    def __init__(self, element: int, time: float):
        super().__init__(f"non-positive water depth in element {element} at t={time:.6g}")
        self.element = element
        self.time = time


@dataclass(frozen=True)
class BoundaryCondition:
    """Wall or zero-gradient ghost rule (hydrostatic.py:29-42)."""

    kind: str

    def __post_init__(self):
        if self.kind not in ("wall", "absorbing"):
            raise ValueError(f"unknown boundary kind {self.kind!r}")

    def ghost(self, h: float, hu: float, hw: float) -> tuple[float, float, float]:
        return (h, -hu, hw) if self.kind == "wall" else (h, hu, hw)


@dataclass(frozen=True)
class BoundaryPair:
    left: BoundaryCondition
    right: BoundaryCondition


WALL = BoundaryCondition("wall")
ABSORBING = BoundaryCondition("absorbing")


def _upload_state(state: FlowState):
    v = [D.dev(f.values[None]) for f in (state.h, state.hu, state.hw)]
    return v[0], v[1], v[2]


def _wrap_state(grid, h, hu, hw, time) -> FlowState:
    return FlowState._wrap(NodalField._wrap(grid, h), NodalField._wrap(grid, hu),
                           NodalField._wrap(grid, hw), time)


def rhs_operator(state: FlowState, bathy: BathymetryModel, bcs: BoundaryPair,
                 g: float = GRAVITY) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Semi-discrete tendency at the state's time (hydrostatic.py:88-184)."""
    lib = D.require_cuda()
    grid = state.grid
    pm = grid.poly_order != 1
    m = D.upload_members(D.member_record(grid, bathy, bcs, None, any_order=pm))
    h, hu, hw = _upload_state(state)
    t = D.dev(np.array([state.time]))
    out = [D.torch().empty_like(h) for _ in range(3)]
    st = D.new_status(1)
    if pm:
        _lib.check(lib.nh_pm_rhs(D.ptr(m), D.ptr(D.upload_members(D.pm_record(grid))),
                                 grid.poly_order + 1, 1, grid.n_elements, D.ptr(h), D.ptr(hu),
                                 D.ptr(hw), D.ptr(t), g, D.ptr(out[0]), D.ptr(out[1]),
                                 D.ptr(out[2]), D.ptr(st), D.stream_ptr()), "nh_pm_rhs")
    else:
        _lib.check(lib.nh_rhs(D.ptr(m), 1, grid.n_elements, D.ptr(h), D.ptr(hu), D.ptr(hw),
                              D.ptr(t), g, D.ptr(out[0]), D.ptr(out[1]), D.ptr(out[2]),
                              D.ptr(st), D.stream_ptr()), "nh_rhs")
    status = D.read_status(st)
    err = D.decode_error(status["error_key"][0])
    if err is not None:
        raise PositivityError(err[2], state.time)
    return tuple(o[0].cpu().numpy() for o in out)


def max_wavespeed(state: FlowState, g: float = GRAVITY) -> float:
    """max |u| + sqrt(g h) (hydrostatic.py:187-189), reduced on the device."""
    lib = D.require_cuda()
    T = D.torch()
    h = D.dev(state.h.values)
    hu = D.dev(state.hu.values)
    out = T.zeros(1, dtype=T.float64, device="cuda")
    _lib.check(lib.nh_max_wavespeed(D.ptr(h), D.ptr(hu), 1, int(h.numel()), float(g), D.ptr(out),
                                    D.stream_ptr()), "nh_max_wavespeed")
    return float(out.item())


RESIDENT_MAX_ELEMENTS = 16 * (3 * 384 - 8)


def _advance_one(state: FlowState, dt: float, bathy, bcs, mode: int, g: float, rho: float,
                 kind="eta_over_d", k_nh=1e-3, enlarge=False, flux=None, want_flags=False,
                 want_p=False, given=None):
    """One fused step of a single member; returns host arrays + flags/p/status."""
    grid = state.grid
    T = D.torch()
    # orders p > 1, and P1 with an LDG flux outside the alternating family,
    # run the m-node kernels (csrc/pm_kernels.cu)
    general = (mode != _lib.MODE_HYDROSTATIC and flux is not None
               and (flux.c12 != -0.5 or flux.c22 != 0.0))
    # ... and so do grids beyond the resident cluster kernel's capacity
    # (16 CTAs x (3 x 384 - 8) elements; the reference has no size limit)
    pm = grid.poly_order != 1 or general or grid.n_elements > RESIDENT_MAX_ELEMENTS
    m = D.upload_members(D.member_record(grid, bathy, bcs, dt, any_order=grid.poly_order != 1))
    h, hu, hw = _upload_state(state)
    t = D.dev(np.array([state.time]))
    st = D.new_status(1)
    nw = (grid.n_elements + 31) // 32
    fb = T.zeros((1, 1, nw), dtype=T.int32, device="cuda") if want_flags else None
    p = T.zeros_like(h) if want_p else None
    gv = D.dev(np.asarray(given, np.uint32).view(np.int32), dtype=np.int32) if given is not None else None
    sch = D.scheme(mode, kind, k_nh, enlarge, flux, g, rho)
    if pm:
        D.pm_advance(m, D.upload_members(D.pm_record(grid)), h, hu, hw, t, 1, sch, st, fb, p,
                     given=gv)
    else:
        D.advance(m, h, hu, hw, t, 1, sch, st, fb, p, gv)
    status = D.read_status(st)
    out = dict(h=h[0].cpu().numpy(), hu=hu[0].cpu().numpy(), hw=hw[0].cpu().numpy(),
               time=float(t.item()), status=status)
    if want_flags:
        out["flags"] = D.bits_to_flags(fb[0, 0].cpu().numpy().view(np.uint32),
                                       grid.n_elements)
    if want_p:
        out["p"] = p[0].cpu().numpy()
    return out


def heun_step(state: FlowState, dt: float, bathy: BathymetryModel, bcs: BoundaryPair,
              g: float = GRAVITY, cfl_warn: bool = True) -> FlowState:
    """One predictor step, forward Euler then trapezoid (hydrostatic.py:192-209)."""
    if dt <= 0:
        raise ValueError("dt must be positive")
    D.require_cuda()
    o = _advance_one(state, dt, bathy, bcs, _lib.MODE_HYDROSTATIC, g, 1000.0)
    D.raise_for_status(o["status"], state.time, dt)
    if cfl_warn and o["status"]["cfl_max"][0] > 1.0:
        warnings.warn(f"advisory CFL number {o['status']['cfl_max'][0]:.3f} exceeds 1 at "
                      f"t={state.time:.6g}", RuntimeWarning, stacklevel=2)
    return _wrap_state(state.grid, o["h"], o["hu"], o["hw"], o["time"])
