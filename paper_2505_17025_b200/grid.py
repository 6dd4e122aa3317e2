"""Grid and field types of the reference API (reference grid.py:62-195).

``GridSpec`` computes the element operators with the same numerical recipe as
the reference (Gauss-Lobatto nodes, barycentric Lagrange basis, Gauss-Legendre
quadrature, ``numpy.linalg.inv`` of the mass matrix), so the constants handed
to the kernels carry the reference's exact bits (they are 1-4 ulp off the
closed forms).  This is one-time host setup, like the
reference's constructor; all per-step arithmetic runs on the GPU.

``NodalField`` / ``FlowState`` hold host numpy arrays exactly like the
reference, so code written against ``nhswe`` keeps working; the batched,
device-resident path is ``paper_2505_17025_b200.ensemble``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from numpy.polynomial import legendre as _leg


def gauss_lobatto_nodes(degree: int) -> np.ndarray:
    """Gauss-Lobatto-Legendre nodes on [-1, 1] (reference grid.py:20-28)."""
    if degree < 1:
        raise ValueError(f"polynomial degree must be >= 1, got {degree}")
    if degree == 1:
        return np.array([-1.0, 1.0])
    c = np.zeros(degree + 1)
    c[degree] = 1.0
    inner = np.sort(np.real(_leg.legroots(_leg.legder(c))))
    return np.concatenate(([-1.0], inner, [1.0]))


def _bary_weights(xs: np.ndarray) -> np.ndarray:
    gap = xs[:, None] - xs[None, :]
    np.fill_diagonal(gap, 1.0)
    return 1.0 / np.prod(gap, axis=1)


def _lagrange_at(xs: np.ndarray, pts: np.ndarray) -> np.ndarray:
    """Row i = Lagrange basis on xs evaluated at pts[i] (second barycentric form)."""
    pts = np.atleast_1d(np.asarray(pts, dtype=float))
    w = _bary_weights(xs)
    gap = pts[:, None] - xs[None, :]
    hit = np.isclose(gap, 0.0, atol=1e-14)
    q = w[None, :] / np.where(hit, 1.0, gap)
    out = q / np.sum(q, axis=1)[:, None]
    rows = hit.any(axis=1)
    out[rows] = hit[rows].astype(float)
    return out


def _diff_matrix(xs: np.ndarray) -> np.ndarray:
    w = _bary_weights(xs)
    gap = xs[:, None] - xs[None, :]
    np.fill_diagonal(gap, 1.0)
    d = (w[None, :] / w[:, None]) / gap
    np.fill_diagonal(d, 0.0)
    np.fill_diagonal(d, -np.sum(d, axis=1))
    return d


@dataclass(frozen=True)
class GridSpec:
    """Uniform DG grid on [x_left, x_right]; mirrors reference grid.py:62-123."""

    x_left: float
    x_right: float
    n_elements: int
    poly_order: int = 1

    def __post_init__(self):
        if not self.x_right > self.x_left:
            raise ValueError("x_right must exceed x_left")
        if self.n_elements < 2:
            raise ValueError("n_elements must be >= 2")
        if self.poly_order < 1:
            raise ValueError("poly_order must be >= 1")
        p = self.poly_order
        dx = (self.x_right - self.x_left) / self.n_elements
        ref = gauss_lobatto_nodes(p)
        left = self.x_left + dx * np.arange(self.n_elements)
        nodes = left[:, None] + 0.5 * dx * (ref[None, :] + 1.0)
        eps = 1e-9 * dx
        sample = nodes.copy()
        sample[:, 0] += eps
        sample[:, -1] -= eps
        qx, qw = np.polynomial.legendre.leggauss(p + 1)
        phi = _lagrange_at(ref, qx)
        dref = _diff_matrix(ref)
        dphi = phi @ dref
        mass = 0.5 * dx * (phi.T @ (qw[:, None] * phi))
        stiff = dphi.T @ (qw[:, None] * phi)
        minv = np.linalg.inv(mass)
        for name, val in (("dx", dx), ("ref_nodes", ref), ("nodes", nodes),
                          ("sample_nodes", sample), ("mass", mass), ("mass_inv", minv),
                          ("stiffness", stiff), ("deriv_ref", dref),
                          ("weak_div", minv @ stiff), ("lift_left", minv[:, 0].copy()),
                          ("lift_right", minv[:, -1].copy())):
            object.__setattr__(self, name, val)

    @property
    def n_nodes(self) -> int:
        return self.n_elements * (self.poly_order + 1)

    def element_of(self, x: float) -> int:
        i = int((x - self.x_left) / self.dx)
        return min(max(i, 0), self.n_elements - 1)

    def nearest_node(self, x: float) -> tuple[int, int]:
        flat = np.argmin(np.abs(self.nodes - x))
        return np.unravel_index(flat, self.nodes.shape)


@dataclass(frozen=True)
class NodalField:
    """Per-element nodal values on a grid (reference grid.py:126-162)."""

    grid: GridSpec
    values: np.ndarray

    def __post_init__(self):
        v = np.asarray(self.values, dtype=float)
        shape = (self.grid.n_elements, self.grid.poly_order + 1)
        if v.shape != shape:
            raise ValueError(f"values shape {v.shape}, expected {shape}")
        if not np.isfinite(v.sum()):
            bad = np.argwhere(~np.isfinite(v))[0]
            x = self.grid.nodes[bad[0], bad[1]]
            raise ValueError(f"non-finite nodal value at x={x} (element {bad[0]})")
        object.__setattr__(self, "values", v)

    def at_nodes(self) -> np.ndarray:
        return self.values

    @classmethod
    def _wrap(cls, grid: GridSpec, values: np.ndarray) -> "NodalField":
        f = object.__new__(cls)
        object.__setattr__(f, "grid", grid)
        object.__setattr__(f, "values", values)
        return f


@dataclass(frozen=True)
class FlowState:
    """(h, hu, hw) on one grid at one time (reference grid.py:165-195)."""

    h: NodalField
    hu: NodalField
    hw: NodalField
    time: float

    def __post_init__(self):
        if not (self.h.grid is self.hu.grid is self.hw.grid):
            raise ValueError("flow components must share one grid")
        if self.h.values.min() <= 0.0:
            el = int(np.argwhere(np.any(self.h.values <= 0.0, axis=1))[0][0])
            raise ValueError(f"non-positive water column in element {el} at t={self.time}")

    @property
    def grid(self) -> GridSpec:
        return self.h.grid

    @classmethod
    def _wrap(cls, h: NodalField, hu: NodalField, hw: NodalField, time: float) -> "FlowState":
        s = object.__new__(cls)
        for k, v in (("h", h), ("hu", hu), ("hw", hw), ("time", time)):
            object.__setattr__(s, k, v)
        return s


def derivative_values(grid: GridSpec, values: np.ndarray) -> np.ndarray:
    """Element-local derivative (reference grid.py:214-215).

    Host helper for building initial data; the step kernels evaluate the same
    operator on the device.
    """
    return (values @ grid.deriv_ref.T) * (2.0 / grid.dx)
