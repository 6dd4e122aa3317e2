"""Non-hydrostatic pressure correction entry points (reference corrector.py).

Every function keeps the reference signature and runs on the GPU:

* ``phi_term`` / ``assemble_coefficients`` -> ``nh_coefficients``
* ``ldg_solve`` / ``solve_on_ranges``      -> ``nh_ldg_solve`` (condensed
  element elimination + cluster tree; replaces LAPACK ``dgbsv``)
* ``correct_momentum``                     -> ``nh_correct_momentum``
* ``apply_correction``                     -> the fused step kernel in
  "correct given flags" mode (coefficients, solve and momentum update in one
  launch, corrector.py:485-498).

The condensed chain solve serves the reference's alternating flux family
(c12 = -1/2, c22 = 0, any c11), its default and the one every config uses.
Any other ``FluxCoefficients`` runs the general path of the m-node kernels
(``nh_pm_ldg_solve`` / ``nh_pm_advance``): each range's band system assembled
as the reference assembles it and solved by band elimination with partial
pivoting, what ``dgbsv`` does (a coverage path, one thread per member).  Every
solve carries the reference's residual gate (corrector.py:355-366): the relative
residual of the batched system is evaluated on the device and above
``residual_tol`` raises ``EllipticSolveError``.  Adjacent ranges are separate
systems, as in the reference's block-diagonal batch.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _lib
from .bathymetry import GRAVITY, RHO_WATER, BathymetryModel, BottomSample
from .grid import FlowState, GridSpec, NodalField
from .hydrostatic import BoundaryPair, _advance_one, _upload_state


class EllipticSolveError(RuntimeError):
    """The elliptic system could not be solved reliably (corrector.py:32-33)."""


@dataclass(frozen=True)
class FluxCoefficients:
    """Interface flux constants (corrector.py:40-47)."""

    c11: float = 0.5
    c12: float = -0.5
    c22: float = 0.0


@dataclass(frozen=True)
class EllipticCoefficients:
    """Nodal coefficients on the element window [offset, offset+len) (corrector.py:50-74)."""

    grid: GridSpec
    s11: np.ndarray
    s12: np.ndarray
    s21: np.ndarray
    s22: np.ndarray
    f1: np.ndarray
    f2: np.ndarray
    phi: np.ndarray
    bottom: BottomSample
    dt: float
    rho: float
    offset: int = 0

    def __post_init__(self):
        if np.any(self.s11 + self.s21 != 0.0):
            raise AssertionError("structural condition s11 + s21 = 0 violated")
        if np.any(self.s12 <= 0.0):
            raise AssertionError("structural condition s12 > 0 violated")


@dataclass(frozen=True)
class PressureSolution:
    """Solved pressure and corrected momentum; p = 0 off the ranges."""

    p_nh: NodalField
    hu_corrected: NodalField
    ranges: tuple


def _coef_planes(predictor: FlowState, bathy, dt, g, rho):
    """Device [7][1][N][2] planes s11, s12, s22, f1, f2, phi, d_x."""
    lib = D.require_cuda()
    grid = predictor.grid
    nodes = grid.poly_order + 1
    m = D.upload_members(D.member_record(grid, bathy, None, dt, any_order=nodes != 2))
    h, hu, hw = _upload_state(predictor)
    t = D.dev(np.array([predictor.time]))
    coef = D.torch().empty((7, 1, grid.n_elements, nodes), dtype=D.torch().float64,
                           device="cuda")
    if nodes != 2:   # orders p > 1: the m-node kernels
        _lib.check(lib.nh_pm_coefficients(D.ptr(m), D.ptr(D.upload_members(D.pm_record(grid))),
                                          nodes, 1, grid.n_elements, D.ptr(h), D.ptr(hu),
                                          D.ptr(hw), D.ptr(t), g, rho, D.ptr(coef),
                                          D.stream_ptr()), "nh_pm_coefficients")
    else:
        _lib.check(lib.nh_coefficients(D.ptr(m), 1, grid.n_elements, D.ptr(h), D.ptr(hu),
                                       D.ptr(hw), D.ptr(t), g, rho, D.ptr(coef),
                                       D.stream_ptr()), "nh_coefficients")
    return coef.cpu().numpy()[:, 0]


def phi_term(predictor: FlowState, bathy: BathymetryModel, g: float = GRAVITY,
             rho: float = RHO_WATER, bottom: BottomSample | None = None,
             window: slice = slice(None)):
    """Moving-bottom forcing (corrector.py:100-132): NodalField or window array."""
    phi = _coef_planes(predictor, bathy, 1.0, g, rho)[5]
    if window == slice(None):
        return NodalField(predictor.grid, phi)
    return phi[window]


def assemble_coefficients(predictor: FlowState, bathy: BathymetryModel, dt: float,
                          g: float = GRAVITY, rho: float = RHO_WATER,
                          window: slice = slice(None)) -> EllipticCoefficients:
    """s- and f-fields of the elliptic system (corrector.py:135-170)."""
    grid = predictor.grid
    c = _coef_planes(predictor, bathy, dt, g, rho)
    full = bathy.sample(grid.sample_nodes, predictor.time)
    if window != slice(None):
        full = BottomSample(*(getattr(full, k)[window] for k in
                              ("d", "d_x", "d_t", "d_tt", "d_xt", "d_xx")))
    s11, s12, s22, f1, f2, phi = (c[i][window].copy() for i in range(6))
    off = window.start if window.start is not None else 0
    return EllipticCoefficients(grid, s11, s12, -s11, s22, f1, f2, phi, full, dt, rho, off)


def is_alternating(flux: FluxCoefficients | None) -> bool:
    """The flux family of the condensed chain solve (c12 = -1/2, c22 = 0)."""
    return flux is None or (flux.c12 == -0.5 and flux.c22 == 0.0)


def _has_adjacent(ranges) -> bool:
    return any(r[0] <= q[1] + 1 for q, r in zip(ranges, ranges[1:]))


def _solve_device(coeffs: EllipticCoefficients, ranges, outer_right: np.ndarray,
                  flux: FluxCoefficients, residual_tol: float = 1e-10,
                  outer_left: np.ndarray | None = None):
    """Run nh_ldg_solve; returns full-grid (p, hu) host arrays (hu only valid on ranges).

    outer_left [n]: hu left of each element -- only a flux outside the
    alternating family gives it a weight (0.5 + c12, corrector.py:346)."""
    lib = D.require_cuda()
    general = not is_alternating(flux)
    if general and outer_left is None:
        raise ValueError("a general LDG flux needs the left outer traces")
    grid = coeffs.grid
    n = grid.n_elements
    off = coeffs.offset
    for e0, e1 in ranges:
        if e0 > e1 or e0 < 0 or e1 >= n:
            raise ValueError(f"invalid element range {(e0, e1)}")
        if e0 - off < 0 or e1 - off >= len(coeffs.s11):
            raise ValueError(f"range {(e0, e1)} outside the coefficient window")
    nodes = grid.poly_order + 1
    pm = nodes != 2 or general   # the m-node kernels (also P1 with a general flux)
    if pm and _has_adjacent(ranges):
        # the m-node solves have no range-start input: solve every other range
        # per call, so no two ranges of a call touch
        p, hu = _solve_device(coeffs, ranges[0::2], outer_right, flux, residual_tol, outer_left)
        p2, hu2 = _solve_device(coeffs, ranges[1::2], outer_right, flux, residual_tol, outer_left)
        for e0, e1 in ranges[1::2]:
            p[e0:e1 + 1], hu[e0:e1 + 1] = p2[e0:e1 + 1], hu2[e0:e1 + 1]
        return p, hu
    planes = np.zeros((7, 1, n, nodes))
    sl = slice(off, off + len(coeffs.s11))
    fields = (coeffs.s11, coeffs.s12, coeffs.s22, coeffs.f1, coeffs.f2)
    if pm:   # the m-node solve stores phi / d_x with its element blocks
        fields += (coeffs.phi, coeffs.bottom.d_x)
    for i, arr in enumerate(fields):
        planes[i, 0, sl] = arr
    flags = np.zeros(n, dtype=bool)
    starts = np.zeros(n, dtype=bool)
    for e0, e1 in ranges:
        flags[e0:e1 + 1] = True
        starts[e0] = True
    m = D.upload_members(D.member_record(grid, _FlatPack(), None, coeffs.dt,
                                         any_order=nodes != 2))
    cp = D.dev(planes)
    fb = D.dev(D.flags_to_bits(flags[None]).view(np.int32), dtype=np.int32)
    sb = D.dev(D.flags_to_bits(starts[None]).view(np.int32), dtype=np.int32)
    orr = D.dev(outer_right[None])
    orl = D.dev(np.asarray(outer_left, dtype=np.float64)[None]) if general else None
    T = D.torch()
    p = T.zeros((1, n, nodes), dtype=T.float64, device="cuda")
    hu = T.zeros((1, n, nodes), dtype=T.float64, device="cuda")
    st = D.new_status(1)
    if pm:
        ws = D.pm_workspace(nodes, 1, n)
        _lib.check(lib.nh_pm_ldg_solve(D.ptr(m), D.ptr(D.upload_members(D.pm_record(grid))),
                                       nodes, 1, n, D.ptr(cp), D.ptr(fb), D.ptr(orl), D.ptr(orr),
                                       coeffs.rho, flux.c11, flux.c12, flux.c22,
                                       float(residual_tol), D.ptr(p), D.ptr(hu), D.ptr(st),
                                       D.ptr(ws), ws.numel(), D.stream_ptr()),
                   "nh_pm_ldg_solve")
    else:
        _lib.check(lib.nh_ldg_solve(D.ptr(m), 1, n, D.ptr(cp), D.ptr(fb), D.ptr(sb), D.ptr(orr),
                                    coeffs.rho, flux.c11, flux.c12, flux.c22,
                                    float(residual_tol), D.ptr(p), D.ptr(hu), D.ptr(st),
                                    D.stream_ptr()), "nh_ldg_solve")
    status = D.read_status(st)
    D.raise_for_status(status, 0.0, 0.0)
    return p[0].cpu().numpy(), hu[0].cpu().numpy()


class _FlatPack:
    """Placeholder bottom for kernels that do not read the bathymetry."""

    def pack(self):
        return _lib.BOTTOM_FLAT, [1.0]


def ldg_solve(coeffs: EllipticCoefficients, elements: tuple[int, int],
              outer_hu: tuple[float, float] = (0.0, 0.0),
              flux: FluxCoefficients = FluxCoefficients(),
              residual_tol: float = 1e-10) -> tuple[np.ndarray, np.ndarray]:
    """Solve on one element range (corrector.py:373-385); returns (p, hu) of the range."""
    e0, e1 = (int(v) for v in elements)
    n = coeffs.grid.n_elements
    outer = np.full(n, float(outer_hu[1]))
    p, hu = _solve_device(coeffs, ((e0, e1),), outer, flux, residual_tol,
                          np.full(n, float(outer_hu[0])))
    return p[e0:e1 + 1].copy(), hu[e0:e1 + 1].copy()


def _outer_right(predictor: FlowState, bcs: BoundaryPair) -> np.ndarray:
    """Outer hu trace right of each element (corrector.py:388-403)."""
    hu = predictor.hu.values
    out = np.empty(hu.shape[0])
    out[:-1] = hu[1:, 0]
    out[-1] = bcs.right.ghost(predictor.h.values[-1, -1], hu[-1, -1],
                              predictor.hw.values[-1, -1])[1]
    return out


def _outer_left(predictor: FlowState, bcs: BoundaryPair) -> np.ndarray:
    """Outer hu trace left of each element (corrector.py:388-403)."""
    hu = predictor.hu.values
    out = np.empty(hu.shape[0])
    out[1:] = hu[:-1, -1]
    out[0] = bcs.left.ghost(predictor.h.values[0, 0], hu[0, 0], predictor.hw.values[0, 0])[1]
    return out


def solve_on_ranges(predictor: FlowState, coeffs: EllipticCoefficients, ranges,
                    bcs: BoundaryPair,
                    flux: FluxCoefficients = FluxCoefficients()) -> PressureSolution:
    """Independent per-range solves (corrector.py:406-424)."""
    grid = predictor.grid
    ranges = tuple(sorted(tuple(int(v) for v in r) for r in ranges))
    p, hu = _solve_device(coeffs, ranges, _outer_right(predictor, bcs), flux,
                          outer_left=None if is_alternating(flux) else _outer_left(predictor, bcs))
    p_full = np.zeros_like(predictor.h.values)
    hu_full = predictor.hu.values.copy()
    for e0, e1 in ranges:
        p_full[e0:e1 + 1] = p[e0:e1 + 1]
        hu_full[e0:e1 + 1] = hu[e0:e1 + 1]
    return PressureSolution(NodalField._wrap(grid, p_full), NodalField._wrap(grid, hu_full),
                            ranges)


def correct_momentum(predictor: FlowState, sol: PressureSolution,
                     coeffs: EllipticCoefficients) -> FlowState:
    """hw update from the bottom pressure; mass untouched (corrector.py:441-482)."""
    lib = D.require_cuda()
    grid = predictor.grid
    n = grid.n_elements
    lo = max(sol.ranges[0][0] - 1, 0)
    hi = min(sol.ranges[-1][1] + 1, n - 1)
    off = coeffs.offset
    if lo - off < 0 or hi + 1 - off > len(coeffs.phi):
        raise ValueError("coefficient window does not cover the solved ranges")
    nodes = grid.poly_order + 1
    planes = np.zeros((7, 1, n, nodes))
    sl = slice(off, off + len(coeffs.phi))
    planes[5, 0, sl] = coeffs.phi
    planes[6, 0, sl] = coeffs.bottom.d_x
    flags = np.zeros(n, dtype=bool)
    for e0, e1 in sol.ranges:
        flags[e0:e1 + 1] = True
    m = D.upload_members(D.member_record(grid, _FlatPack(), None, coeffs.dt,
                                         any_order=nodes != 2))
    h = D.dev(predictor.h.values[None])
    p = D.dev(sol.p_nh.values[None])
    hw = D.dev(predictor.hw.values[None])
    out = D.torch().empty_like(hw)
    cp = D.dev(planes)
    fb = D.dev(D.flags_to_bits(flags[None]).view(np.int32), dtype=np.int32)
    if nodes != 2:
        _lib.check(lib.nh_pm_correct_momentum(D.ptr(m),
                                              D.ptr(D.upload_members(D.pm_record(grid))), nodes,
                                              1, n, D.ptr(h), D.ptr(p), D.ptr(cp), D.ptr(fb),
                                              coeffs.rho, D.ptr(hw), D.ptr(out),
                                              D.stream_ptr()), "nh_pm_correct_momentum")
    else:
        _lib.check(lib.nh_correct_momentum(D.ptr(m), 1, n, D.ptr(h), D.ptr(p), D.ptr(cp),
                                           D.ptr(fb), coeffs.rho, D.ptr(hw), D.ptr(out),
                                           D.stream_ptr()), "nh_correct_momentum")
    return FlowState._wrap(predictor.h, sol.hu_corrected,
                           NodalField._wrap(grid, out[0].cpu().numpy()), predictor.time)


def apply_correction(predictor: FlowState, bathy: BathymetryModel, dt: float, ranges,
                     bcs: BoundaryPair, flux: FluxCoefficients = FluxCoefficients(),
                     g: float = GRAVITY, rho: float = RHO_WATER,
                     ) -> tuple[FlowState, PressureSolution]:
    """Full correction on the flagged ranges, one fused launch (corrector.py:485-498)."""
    D.require_cuda()
    grid = predictor.grid
    n = grid.n_elements
    ranges = tuple(sorted(tuple(int(v) for v in r) for r in ranges))
    if not ranges:
        raise ValueError("apply_correction needs at least one range")
    if _has_adjacent(ranges) or not is_alternating(flux):
        # adjacent ranges are separate systems: the reference's own pipeline
        # (corrector.py:485-498) of the three device kernels, whose solve
        # splits the flagged run at the given range starts
        lo, hi = max(ranges[0][0] - 1, 0), min(ranges[-1][1] + 1, n - 1)
        coeffs = assemble_coefficients(predictor, bathy, dt, g, rho, window=slice(lo, hi + 1))
        sol = solve_on_ranges(predictor, coeffs, ranges, bcs, flux)
        return correct_momentum(predictor, sol, coeffs), sol
    flags = np.zeros(n, dtype=bool)
    for e0, e1 in ranges:
        if e0 > e1 or e0 < 0 or e1 >= n:
            raise ValueError(f"invalid element range {(e0, e1)}")
        flags[e0:e1 + 1] = True
    o = _advance_one(predictor, dt, bathy, bcs, _lib.MODE_CORRECT_GIVEN, g, rho, flux=flux,
                     want_p=True, given=D.flags_to_bits(flags[None]))
    D.raise_for_status(o["status"], predictor.time, dt)
    hu = NodalField._wrap(grid, o["hu"])
    state = FlowState._wrap(predictor.h, hu, NodalField._wrap(grid, o["hw"]), predictor.time)
    return state, PressureSolution(NodalField._wrap(grid, o["p"]), hu, ranges)
