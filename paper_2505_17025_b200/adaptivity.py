"""Adaptive mask and the full time step (reference adaptivity.py:1-163).

``adaptive_step`` is one launch of the fused step kernel (predictor,
criterion, flagged-range LDG solve and momentum correction, all on chip).
The mask it returns is read back from the kernel's per-step flag bits.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _lib
from .bathymetry import GRAVITY, RHO_WATER, BathymetryModel
from .corrector import FluxCoefficients
from .grid import FlowState, NodalField
from .hydrostatic import BoundaryPair, _advance_one, _upload_state, _wrap_state

CRITERION_KINDS = ("eta_over_d", "eta_x", "u", "u_x", "w", "w_x")
DEFAULT_THRESHOLD = 0.001


@dataclass(frozen=True)
class Criterion:
    """Indicator kind, threshold and +-1 enlargement (adaptivity.py:26-43)."""

    kind: str
    k_nh: float = DEFAULT_THRESHOLD
    enlarge: bool = False

    def __post_init__(self):
        if self.kind not in CRITERION_KINDS:
            raise ValueError(f"unknown criterion kind {self.kind!r}")
        if self.k_nh <= 0:
            raise ValueError("threshold k_nh must be positive")


def contiguous_ranges(flags: np.ndarray) -> tuple[tuple[int, int], ...]:
    """Maximal runs of True as inclusive (first, last) pairs (adaptivity.py:67-72)."""
    f = np.asarray(flags, dtype=bool)
    if f.size == 0:
        return ()
    edge = np.diff(np.concatenate(([0], f.astype(np.int8), [0])))
    return tuple((int(a), int(b)) for a, b in
                 zip(np.flatnonzero(edge == 1), np.flatnonzero(edge == -1) - 1))


@dataclass(frozen=True)
class NonHydroMask:
    """Per-element flags and their ranges (adaptivity.py:46-64)."""

    flags: np.ndarray
    ranges: tuple

    @classmethod
    def from_flags(cls, flags: np.ndarray) -> "NonHydroMask":
        flags = np.asarray(flags, dtype=bool)
        return cls(flags, contiguous_ranges(flags))

    @property
    def empty(self) -> bool:
        return not bool(self.flags.any())

    @property
    def fraction(self) -> float:
        return float(np.mean(self.flags)) if self.flags.size else 0.0


def enlarge_flags(flags: np.ndarray) -> np.ndarray:
    """+-1 dilation clipped to the domain (adaptivity.py:99-104)."""
    grown = np.array(flags, dtype=bool, copy=True)
    grown[:-1] |= flags[1:]
    grown[1:] |= flags[:-1]
    return grown


def _criterion_device(predictor: FlowState, bathy: BathymetryModel, kind: str):
    lib = D.require_cuda()
    grid = predictor.grid
    pm = grid.poly_order != 1
    m = D.upload_members(D.member_record(grid, bathy, None, None, any_order=pm))
    h, hu, hw = _upload_state(predictor)
    t = D.dev(np.array([predictor.time]))
    out = D.torch().empty_like(h)
    if pm:
        _lib.check(lib.nh_pm_criterion(D.ptr(m), D.ptr(D.upload_members(D.pm_record(grid))),
                                       grid.poly_order + 1, 1, grid.n_elements, D.ptr(h),
                                       D.ptr(hu), D.ptr(hw), D.ptr(t), _lib.CRIT[kind],
                                       D.ptr(out), D.stream_ptr()), "nh_pm_criterion")
    else:
        _lib.check(lib.nh_criterion(D.ptr(m), 1, grid.n_elements, D.ptr(h), D.ptr(hu),
                                    D.ptr(hw), D.ptr(t), _lib.CRIT[kind], D.ptr(out),
                                    D.stream_ptr()), "nh_criterion")
    return out[0]


def criterion_values(predictor: FlowState, bathy: BathymetryModel, kind: str) -> np.ndarray:
    """Nodal indicator values (adaptivity.py:75-96)."""
    if kind not in CRITERION_KINDS:
        raise ValueError(f"unknown criterion kind {kind!r}")
    return _criterion_device(predictor, bathy, kind).cpu().numpy()


def evaluate_criterion(predictor: FlowState, bathy: BathymetryModel,
                       crit: Criterion) -> NonHydroMask:
    """Flag = max nodal indicator > k_nh, optional enlargement (adaptivity.py:107-113)."""
    T = D.torch()
    lib = D.require_cuda()
    v = _criterion_device(predictor, bathy, crit.kind).contiguous()
    n, m = int(v.shape[0]), int(v.shape[1])
    flags = T.empty(n, dtype=T.uint8, device="cuda")
    _lib.check(lib.nh_mask(D.ptr(v), 1, n, m, float(crit.k_nh), 1 if crit.enlarge else 0,
                           D.ptr(flags), D.stream_ptr()), "nh_mask")
    return NonHydroMask.from_flags(flags.cpu().numpy().astype(bool))


def full_mask(n_elements: int) -> NonHydroMask:
    return NonHydroMask.from_flags(np.ones(n_elements, dtype=bool))


@dataclass(frozen=True)
class StepResult:
    state: FlowState
    mask: NonHydroMask
    p_nh: NodalField | None


_MODES = {"hydrostatic": _lib.MODE_HYDROSTATIC, "global": _lib.MODE_GLOBAL,
          "adaptive": _lib.MODE_ADAPTIVE}


def adaptive_step(state: FlowState, dt: float, bathy: BathymetryModel, bcs: BoundaryPair,
                  mode: str = "adaptive", crit: Criterion | None = None,
                  flux: FluxCoefficients = FluxCoefficients(),
                  g: float = GRAVITY, rho: float = RHO_WATER,
                  cfl_warn: bool = True) -> StepResult:
    """One full time step in a single fused launch (adaptivity.py:127-163)."""
    if mode not in _MODES:
        raise ValueError(f"unknown mode {mode!r}")
    if mode == "adaptive" and crit is None:
        raise ValueError("adaptive mode requires a criterion")
    if dt <= 0:
        raise ValueError("dt must be positive")
    D.require_cuda()
    n = state.grid.n_elements
    c = crit if crit is not None else Criterion("eta_over_d")
    o = _advance_one(state, dt, bathy, bcs, _MODES[mode], g, rho, c.kind, c.k_nh, c.enlarge,
                     flux, want_flags=(mode != "hydrostatic"), want_p=(mode != "hydrostatic"))
    D.raise_for_status(o["status"], state.time, dt)
    if cfl_warn and o["status"]["cfl_max"][0] > 1.0:
        warnings.warn(f"advisory CFL number {o['status']['cfl_max'][0]:.3f} exceeds 1 at "
                      f"t={state.time:.6g}", RuntimeWarning, stacklevel=2)
    new = _wrap_state(state.grid, o["h"], o["hu"], o["hw"], o["time"])
    if mode == "hydrostatic":
        return StepResult(new, NonHydroMask.from_flags(np.zeros(n, dtype=bool)), None)
    mask = NonHydroMask.from_flags(o["flags"])
    if mask.empty:
        return StepResult(new, mask, None)
    return StepResult(new, mask, NodalField._wrap(state.grid, o["p"]))
