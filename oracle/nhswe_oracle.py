"""CPU oracle for the adaptive non-hydrostatic SWE time step.

TEST INFRASTRUCTURE ONLY.  Nothing in the product package imports this
module; only ``tests/``, ``__graft_entry__.smoke()`` and the CPU-baseline
leg of ``bench.py`` may use it, and only as the checker / the timed CPU
reference arm, never as the thing measured or shipped.

This is an independent numpy restatement of the reference package
``nhswe`` (arXiv 2505.17025, mounted read-only at /root/reference) for the
time-step hot path.  It keeps the reference's floating-point operation
order wherever that decides the result bits (numpy ``@`` for the 2x2
element operators, LAPACK ``dgbsv`` for the banded LDG solve), so on the
same host it reproduces the reference bit for bit; ``tests/golden`` holds
vectors produced by the real reference (``tests/golden/make_golden.py``)
that pin it.  Every function cites the reference lines it restates
(paths relative to /root/reference/pkg/src/nhswe/).

Only the P1 (two Gauss-Lobatto nodes per element) discretisation is
restated: every configuration on the hot path is P1.
"""

from __future__ import annotations

import math
import warnings
from dataclasses import dataclass, field

import numpy as np
from scipy.linalg import lapack as _lapack

GRAVITY = 9.81          # bathymetry.py:15
RHO_WATER = 1000.0      # bathymetry.py:16


class OraclePositivityError(RuntimeError):
    """hydrostatic.py:20-26 -- non-positive depth (element, time)."""

    def __init__(self, element: int, time: float):
        super().__init__(f"non-positive water depth in element {element} at t={time:.6g}")
        self.element = element
        self.time = time


class OracleSolveError(RuntimeError):
    """corrector.py:32-33 -- unreliable elliptic solve."""


# --------------------------------------------------------------------------
# P1 element operators  (grid.py:20-114)
# --------------------------------------------------------------------------

def _p1_reference_operators():
    """Reference-element matrices for the linear nodal basis on [-1, 1].

    Same construction as grid.py:71-114: barycentric Lagrange basis on the
    Gauss-Lobatto nodes, two-point Gauss-Legendre quadrature.
    """
    xi = np.array([-1.0, 1.0])                              # grid.py:24-25
    # barycentric weights 1/prod(xi_i - xi_j)  (grid.py:31-34)
    gap = xi[:, None] - xi[None, :]
    np.fill_diagonal(gap, 1.0)
    bw = 1.0 / np.prod(gap, axis=1)
    q, qw = np.polynomial.legendre.leggauss(2)
    # basis at quadrature points (grid.py:37-48); no quadrature point is a node
    rat = bw[None, :] / (q[:, None] - xi[None, :])
    phi = rat / np.sum(rat, axis=1)[:, None]
    # nodal differentiation matrix (grid.py:51-59)
    dmat = (bw[None, :] / bw[:, None]) / gap
    np.fill_diagonal(dmat, 0.0)
    np.fill_diagonal(dmat, -np.sum(dmat, axis=1))
    dphi = phi @ dmat
    mass_ref = phi.T @ (qw[:, None] * phi)
    stiff_ref = dphi.T @ (qw[:, None] * phi)
    return dmat, mass_ref, stiff_ref


@dataclass
class Grid:
    """Uniform P1 grid on [x_left, x_right] (grid.py:62-114)."""

    x_left: float
    x_right: float
    n: int

    def __post_init__(self):
        if not self.x_right > self.x_left or self.n < 2:
            raise ValueError("bad grid")
        self.dx = (self.x_right - self.x_left) / self.n
        dmat, mass_ref, stiff_ref = _p1_reference_operators()
        left = self.x_left + self.dx * np.arange(self.n)
        self.nodes = left[:, None] + 0.5 * self.dx * (np.array([-1.0, 1.0])[None, :] + 1.0)
        eps = 1e-9 * self.dx                                  # grid.py:87-90
        self.sample_nodes = self.nodes.copy()
        self.sample_nodes[:, 0] += eps
        self.sample_nodes[:, 1] -= eps
        self.mass = 0.5 * self.dx * mass_ref
        self.mass_inv = np.linalg.inv(self.mass)
        self.stiffness = stiff_ref
        self.deriv_ref = dmat
        self.weak_div = self.mass_inv @ stiff_ref
        self.lift_left = self.mass_inv[:, 0].copy()
        self.lift_right = self.mass_inv[:, -1].copy()


def elem_derivative(grid: Grid, v: np.ndarray) -> np.ndarray:
    """Element-local derivative, grid.py:214-215."""
    return (v @ grid.deriv_ref.T) * (2.0 / grid.dx)


# --------------------------------------------------------------------------
# Bottom models  (bathymetry.py:66-184, plus harness models for configs 2-5)
# --------------------------------------------------------------------------

class Bottom:
    """d(x, t) and its five derivative channels (bathymetry.py:18, 43-63)."""

    def channels(self, x, t):
        raise NotImplementedError


@dataclass
class Flat(Bottom):
    """bathymetry.py:66-79."""
    h0: float

    def channels(self, x, t):
        z = np.zeros_like(x)
        return np.full_like(x, self.h0), z, z, z, z, z


@dataclass
class Plate(Bottom):
    """Impulsive flat plate |x| < b, bathymetry.py:82-116 (alpha = 1.11 / t_c)."""
    h0: float
    zeta0: float
    b: float
    t_c: float

    def channels(self, x, t):
        a = 1.11 / self.t_c
        inside = np.abs(x) < self.b
        e = np.exp(-a * max(t, 0.0))
        d = np.full_like(x, self.h0)
        d[inside] -= self.zeta0 * (1.0 - e)
        z = np.zeros_like(x)
        return (d, z, np.where(inside, -self.zeta0 * a * e, 0.0),
                np.where(inside, self.zeta0 * a * a * e, 0.0), z, z)


@dataclass
class Motion:
    """Accelerate / coast / brake / stop kinematics, bathymetry.py:119-144."""
    a0: float
    u_t: float
    t1: float
    t2: float
    t3: float

    def at(self, t):
        a0, ut, t1, t2, t3 = self.a0, self.u_t, self.t1, self.t2, self.t3
        s1 = 0.5 * a0 * t1 * t1
        if t <= t1:
            return 0.5 * a0 * t * t, a0 * t, a0
        if t <= t2:
            return s1 + ut * (t - t1), ut, 0.0
        if t <= t3:
            return s1 + ut * (t - t1) - 0.5 * a0 * (t - t2) ** 2, ut - a0 * (t - t2), -a0
        return s1 + ut * (t3 - t1) - 0.5 * a0 * (t3 - t2) ** 2, 0.0, 0.0


@dataclass
class QuarticSlide(Bottom):
    """Quartic bump h0 - Hs(1 - xi^4) moving along a flat bed, bathymetry.py:147-184."""
    h0: float
    Hs: float
    Ls: float
    motion: Motion
    x_start: float = 0.0

    def channels(self, x, t):
        s, sp, spp = self.motion.at(t)
        xi = 2.0 * (x - (self.x_start + s)) / self.Ls
        inside = np.abs(xi) < 1.0
        xi = np.where(inside, xi, 0.0)
        c = 2.0 / self.Ls
        d = np.full_like(x, self.h0)
        d[inside] -= self.Hs * (1.0 - xi[inside] ** 4)
        Hs = self.Hs
        return (d,
                np.where(inside, Hs * 4.0 * xi ** 3 * c, 0.0),
                np.where(inside, Hs * 4.0 * xi ** 3 * (-c * sp), 0.0),
                np.where(inside, Hs * (12.0 * xi ** 2 * (c * sp) ** 2 - 4.0 * xi ** 3 * c * spp), 0.0),
                np.where(inside, Hs * 12.0 * xi ** 2 * c * (-c * sp), 0.0),
                np.where(inside, Hs * 12.0 * xi ** 2 * c * c, 0.0))


# Deterministic elementary functions of the harness models.  The two harness
# bottoms (configs 2-5) are this project's own closed forms (SURVEY.md
# Appendix C), so they are DEFINED through exp / log1p evaluated with IEEE
# +, -, * and / only (Cody-Waite reduction, Horner polynomials, no fused
# multiply-add), which numpy on any host and the CUDA kernels (bathy.cuh
# nh_det_exp / nh_det_log1p, same constants, same order) round identically.
# libm / numpy-SIMD / CUDA exp differ from each other in the last bit, and a
# per-step last-bit difference in d(x, t) random-walks through the predictor.
LN2_HI = float.fromhex("0x1.62e42fee00000p-1")     # k * LN2_HI exact for |k| < 2^11
LN2_LO = float.fromhex("0x1.a39ef35793c76p-33")
INV_LN2 = float.fromhex("0x1.71547652b82fep+0")
LN2 = math.log(2.0)
_EXP_TAYLOR = [1.0 / math.factorial(n) for n in range(13, -1, -1)]   # 1/13!, ..., 1/0!
_ATANH_ODD = [1.0 / (2 * k + 1) for k in range(17, -1, -1)]          # 1/35, ..., 1/1
BOX_YCUT = 23.0      # smoothed box: S(x) = 0 beyond |y| = 23 (E < 1e-20)
SLIDE_RCUT = 10.0    # Gaussian mound: G = 0 beyond |r| = 10 (< 2e-22 A)


def det_exp(x):
    """exp(x) from IEEE +,-,* only: x = k ln2 + r, |r| <= ln2/2, degree-13
    Taylor polynomial of exp(r) by Horner, times 2^k."""
    x = np.asarray(x, dtype=np.float64)
    k = np.rint(x * INV_LN2)
    r = (x - k * LN2_HI) - k * LN2_LO
    p = np.full_like(r, _EXP_TAYLOR[0])
    for c in _EXP_TAYLOR[1:]:
        p = p * r + c
    out = np.ldexp(p, k.astype(np.int64))
    return out if out.ndim else float(out)


def det_log1p(e):
    """log1p(e) for 0 <= e <= 1 as 2 atanh(z), z = e / (2 + e) <= 1/3: odd
    series to z^35 by Horner in z^2."""
    e = np.asarray(e, dtype=np.float64)
    z = e / (2.0 + e)
    w = z * z
    s = np.full_like(z, _ATANH_ODD[0])
    for c in _ATANH_ODD[1:]:
        s = s * w + c
    out = 2.0 * (z * s)
    return out if out.ndim else float(out)


@dataclass
class SmoothBox(Bottom):
    """Harness model (configs 2, 4): box uplift with a tanh edge.

    d = h0 - zeta(t) S(x), zeta = zeta0 (1 - exp(-alpha t)),
    S = (1 - tanh((|x| - b)/w)) / 2, written through E = exp(-2|y|),
    y = (|x| - b)/w, so that no channel suffers cancellation:
    S = E/(1+E) (y >= 0) or 1/(1+E) (y < 0); S' = -2E/(1+E)^2 sign(x)/w;
    S'' = 4E(1-E)/(1+E)^3 sign(y)/w^2; S = S' = S'' = 0 for y >= 23.
    exp is det_exp.  Shared with the CUDA device model (csrc/bathy.cuh) --
    SURVEY.md Appendix C.3.
    """
    h0: float
    zeta0: float
    b: float
    alpha: float
    w: float

    def channels(self, x, t):
        tt = max(t, 0.0)
        e = det_exp(-self.alpha * tt)
        zeta = self.zeta0 * (1.0 - e)
        zt = self.zeta0 * self.alpha * e
        ztt = -self.zeta0 * self.alpha * self.alpha * e
        ax = np.abs(x)
        y = (ax - self.b) / self.w
        on = y < BOX_YCUT
        E = np.where(on, det_exp(-2.0 * np.abs(np.where(on, y, 0.0))), 0.0)
        inv1 = 1.0 / (1.0 + E)
        S = np.where(y >= 0.0, E * inv1, inv1)
        sg = np.where(x >= 0.0, 1.0, -1.0)
        sech2 = 4.0 * E * inv1 * inv1
        Sx = -0.5 * sech2 * sg / self.w
        th = np.where(y >= 0.0, 1.0, -1.0) * (1.0 - E) * inv1
        Sxx = sech2 * th / (self.w * self.w)
        return (self.h0 - zeta * S, -zeta * Sx, -zt * S, -ztt * S, -zt * Sx, -zeta * Sxx)


@dataclass
class SlopeSlide(Bottom):
    """Harness model (configs 3, 5): Gaussian mound sliding down a plane slope.

    d0(x) = min(d_top + x tan(theta), d_max);  G = A exp(-r^2 / 2), r = (x - xc) (1/sigma)
    (0 beyond |x - xc| = 10 sigma);  d = d0 - G.  xc(t) = x0 + u_t t0 ln cosh(t/t0)
    until d0(xc) = d_stop, then frozen (velocity u_t tanh(t/t0), acceleration
    (u_t/t0) sech^2(t/t0)); ln cosh s = s + log1p(E) - ln 2 and
    tanh s = (1 - E)/(1 + E) with E = exp(-2s); exp / log1p are det_exp /
    det_log1p.  d_t = G_x xc', d_tt = -G_xx xc'^2 + G_x xc'', d_xt = G_xx xc',
    d_xx = -G_xx (the slope kink's d0'' is taken as 0).  SURVEY.md Appendix C.4.
    """
    d_top: float
    tan_theta: float
    d_max: float
    A: float
    sigma: float
    x0: float
    u_t: float
    t0: float
    d_stop: float

    @property
    def x_stop(self):
        return (self.d_stop - self.d_top) / self.tan_theta

    @property
    def t_stop(self):
        arg = (self.x_stop - self.x0) / (self.u_t * self.t0)
        if arg <= 0.0:
            return 0.0
        # ln cosh(s) = arg  ->  s = acosh(exp(arg)), written overflow-safe
        return self.t0 * (arg + math.log1p(math.sqrt(-math.expm1(-2.0 * arg))))

    def kinematics(self, t):
        tt = max(t, 0.0)
        ts = self.t_stop
        if tt >= ts:
            return self.x_stop if ts > 0.0 else self.x0, 0.0, 0.0
        s = tt / self.t0
        E = det_exp(-2.0 * s)
        lc = s + det_log1p(E) - LN2                # ln cosh(s)
        th = (1.0 - E) / (1.0 + E)                 # tanh(s)
        return (self.x0 + self.u_t * self.t0 * lc, self.u_t * th,
                (self.u_t / self.t0) * (1.0 - th * th))

    def channels(self, x, t):
        xc, v, acc = self.kinematics(t)
        ramp = self.d_top + x * self.tan_theta
        on_slope = ramp < self.d_max
        d0 = np.where(on_slope, ramp, self.d_max)
        d0x = np.where(on_slope, self.tan_theta, 0.0)
        inv_s = 1.0 / self.sigma                   # the model uses the reciprocal
        r = (x - xc) * inv_s
        on = np.abs(r) < SLIDE_RCUT
        G = np.where(on, self.A * det_exp(-0.5 * r * r), 0.0)
        Gx = -G * r * inv_s
        Gxx = G * (r * r - 1.0) * (inv_s * inv_s)
        return (d0 - G, d0x - Gx, Gx * v, -Gxx * v * v + Gx * acc, Gxx * v, -Gxx)


# --------------------------------------------------------------------------
# Hydrostatic predictor  (hydrostatic.py:88-223)
# --------------------------------------------------------------------------

def _ghost(kind: str, h, hu, hw):
    """hydrostatic.py:39-42."""
    return (h, -hu, hw) if kind == "wall" else (h, hu, hw)


def tendency(grid: Grid, bottom: Bottom, bcs, g, h, hu, hw, t):
    """Semi-discrete tendency of (h, hu, hw) at time t, hydrostatic.py:88-184."""
    if h.min() <= 0.0:
        raise OraclePositivityError(int(np.argwhere(np.any(h <= 0.0, axis=1))[0][0]), t)
    u = hu / h
    f2 = hu * u
    f2 += (0.5 * g) * h * h
    f3 = u * hw
    ch = bottom.channels(grid.sample_nodes, t)
    d, d_x = ch[0], ch[1]

    # interface traces: left side = element e-1 node 1, right = element e node 0
    gl = _ghost(bcs[0], h[0, 0], hu[0, 0], hw[0, 0])
    gr = _ghost(bcs[1], h[-1, 1], hu[-1, 1], hw[-1, 1])
    hL = np.concatenate(([gl[0]], h[:, 1]))
    huL = np.concatenate(([gl[1]], hu[:, 1]))
    hwL = np.concatenate(([gl[2]], hw[:, 1]))
    hR = np.concatenate((h[:, 0], [gr[0]]))
    huR = np.concatenate((hu[:, 0], [gr[1]]))
    hwR = np.concatenate((hw[:, 0], [gr[2]]))
    uL = huL / hL
    uR = huR / hR
    dL = np.concatenate(([d[0, 0]], d[:, 1]))
    dR = np.concatenate((d[:, 0], [d[-1, 1]]))

    jump = not np.array_equal(dL, dR)                      # hydrostatic.py:131
    if jump:                                               # hydrostatic reconstruction
        dm = np.minimum(dL, dR)
        hLs = np.maximum(hL - (dL - dm), 0.0)
        hRs = np.maximum(hR - (dR - dm), 0.0)
        cL = (0.5 * g) * (hL * hL - hLs * hLs)
        cR = (0.5 * g) * (hR * hR - hRs * hRs)
    else:
        hLs, hRs = hL, hR
    lam = 0.5 * np.maximum(np.abs(uL) + np.sqrt(g * hLs), np.abs(uR) + np.sqrt(g * hRs))
    qL = hLs * uL
    qR = hRs * uR
    F1 = 0.5 * (qL + qR) - lam * (hRs - hLs)
    F2 = 0.5 * (qL * uL + qR * uR + (0.5 * g) * (hLs * hLs + hRs * hRs))
    F2 -= lam * (qR - qL)
    wL = (hLs / hL) * hwL
    wR = (hRs / hR) * hwR
    F3 = 0.5 * (wL * uL + wR * uR) - lam * (wR - wL)

    Wt = grid.weak_div.T
    lr = grid.lift_right[None, :]
    ll = grid.lift_left[None, :]
    out1 = hu @ Wt
    out1 -= F1[1:, None] * lr
    out1 += F1[:-1, None] * ll
    out2 = f2 @ Wt
    if jump:
        out2 -= (F2[1:] + cL[1:])[:, None] * lr
        out2 += (F2[:-1] + cR[:-1])[:, None] * ll
    else:
        out2 -= F2[1:, None] * lr
        out2 += F2[:-1, None] * ll
    if d_x.any():
        out2 += (g * h) * d_x
    out3 = f3 @ Wt
    out3 -= F3[1:, None] * lr
    out3 += F3[:-1, None] * ll
    return out1, out2, out3


def heun(grid, bottom, bcs, g, h, hu, hw, t, dt, cfl_warn=True):
    """hydrostatic.py:192-223: forward-Euler stage, then trapezoidal average."""
    if dt <= 0:
        raise ValueError("dt must be positive")
    if cfl_warn:
        cfl = float(np.max(np.abs(hu / h) + np.sqrt(g * h))) * dt / grid.dx
        if cfl > 1.0:
            warnings.warn(f"advisory CFL number {cfl:.3f} exceeds 1 at t={t:.6g}",
                          RuntimeWarning, stacklevel=2)
    t1 = t + dt
    k1 = tendency(grid, bottom, bcs, g, h, hu, hw, t)
    hs = h + dt * k1[0]
    if not hs.min() > 0.0:
        raise OraclePositivityError(-1, t1)
    k2 = tendency(grid, bottom, bcs, g, hs, hu + dt * k1[1], hw + dt * k1[2], t1)
    mh, mq, mw = (0.5 * (a + b) for a, b in zip(k1, k2))
    hn = h + dt * mh
    if not hn.min() > 0.0:
        raise OraclePositivityError(-1, t1)
    return hn, hu + dt * mq, hw + dt * mw


# --------------------------------------------------------------------------
# Criterion mask  (adaptivity.py:67-113)
# --------------------------------------------------------------------------

KINDS = ("eta_over_d", "eta_x", "u", "u_x", "w", "w_x")


def indicator(grid, bottom, kind, h, hu, hw, t):
    """adaptivity.py:75-96."""
    if kind in ("eta_over_d", "eta_x"):
        d = bottom.channels(grid.sample_nodes, t)[0]
        if kind == "eta_over_d":
            return np.abs((h - d) / d)
        return np.abs(elem_derivative(grid, h - d))
    u = hu / h
    if kind == "u":
        return np.abs(u)
    if kind == "u_x":
        return np.abs(elem_derivative(grid, u))
    w = hw / h
    if kind == "w":
        return np.abs(w)
    if kind == "w_x":
        return np.abs(elem_derivative(grid, w))
    raise ValueError(kind)


def flags_from(values, k_nh, enlarge):
    """adaptivity.py:99-113: max over nodes > threshold, optional +-1 dilation."""
    f = values.max(axis=1) > k_nh
    if enlarge:
        g = f.copy()
        g[:-1] |= f[1:]
        g[1:] |= f[:-1]
        f = g
    return f


def runs(flags):
    """Maximal runs of True as inclusive (first, last), adaptivity.py:67-72."""
    f = np.asarray(flags, dtype=bool)
    if f.size == 0:
        return ()
    edge = np.diff(np.concatenate(([0], f.view(np.int8), [0])))
    starts = np.flatnonzero(edge == 1)
    stops = np.flatnonzero(edge == -1) - 1
    return tuple((int(a), int(b)) for a, b in zip(starts, stops))


# --------------------------------------------------------------------------
# LDG pressure correction  (corrector.py:100-498)
# --------------------------------------------------------------------------

@dataclass
class Coeffs:
    """Nodal elliptic coefficients on an element window (corrector.py:50-74)."""
    s11: np.ndarray
    s12: np.ndarray
    s22: np.ndarray
    f1: np.ndarray
    f2: np.ndarray
    phi: np.ndarray
    d_x: np.ndarray
    offset: int
    dt: float
    rho: float


def coefficients(grid, bottom, h, hu, hw, t, dt, g, rho, lo, hi):
    """phi_term + assemble_coefficients on elements lo..hi (corrector.py:100-170)."""
    sl = slice(lo, hi + 1)
    ch = [c[sl] for c in bottom.channels(grid.sample_nodes, t)]
    d, d_x, d_t, d_tt, d_xt, d_xx = ch
    hh, qq, ww = h[sl], hu[sl], hw[sl]
    # phi: accumulate -d_tt, then the drag, then the slope term (corrector.py:116-129)
    acc = -d_tt if d_tt.any() else None
    if d_xt.any() or d_xx.any():
        u = qq / hh
        drag = -2.0 * u * d_xt - u * u * d_xx
        acc = drag if acc is None else acc + drag
    slope_bed = d_x.any()
    if slope_bed:
        sl_term = (g * d_x) * elem_derivative(grid, hh - d)
        acc = sl_term if acc is None else acc + sl_term
        phi = (rho * hh / (4.0 + d_x * d_x)) * acc
    elif acc is None:
        phi = np.zeros_like(hh)
    else:
        phi = (0.25 * rho) * hh * acc
    h_x = elem_derivative(grid, hh)
    ih = 1.0 / hh
    s22 = (3.0 * dt / rho) * ih
    if slope_bed:
        quad = 4.0 + d_x * d_x
        s11 = (h_x - 1.5 * d_x) * ih
        s12 = (0.25 * rho / dt) * quad * ih
        f1 = (0.25 * quad * ih) * (phi * d_x + (rho / dt) * qq)
        f2 = (-2.0 * ww - (0.5 * d_x) * qq) * ih
        f2 -= (0.5 * dt / rho) * quad * phi * ih
    else:
        s11 = h_x * ih
        s12 = (rho / dt) * ih
        f1 = (rho / dt) * qq * ih
        f2 = -2.0 * ww * ih
        if phi.any():
            f2 -= (2.0 * dt / rho) * phi * ih
    if d_t.any():
        f2 -= 2.0 * d_t
    if np.any(s11 + (-s11) != 0.0) or np.any(s12 <= 0.0):
        raise AssertionError("structural condition violated")
    return Coeffs(s11, s12, s22, f1, f2, phi, d_x, lo, dt, rho)


def _band_system(grid, co: Coeffs, ranges, outer, c11, c12, c22):
    """Banded (kl = ku = 3) LDG matrix + rhs for stacked ranges.

    Restates corrector.py:173-281 (sparsity) and :329-349 (values): unknowns
    interleaved (p/rho, hu) per node; every matrix entry is its volume value
    plus at most one face / range-end constant, summed in that order.
    """
    M, K = grid.mass, grid.stiffness
    rho = co.rho
    n = sum(e1 - e0 + 1 for e0, e1 in ranges)
    size = 4 * n
    ab = np.zeros((10, size))                    # LAPACK gbsv layout, 2*kl+ku+1 rows

    def put(r, c, v):
        ab[6 + r - c, c] += v

    b = np.zeros(size)
    # forcing products over the stacked ranges in ONE matmul, as the reference
    # does (corrector.py:343-344): numpy's (n, 2) @ (2, 2) kernel rounds a
    # 1-row operand differently from a many-row one, so per-range products
    # would differ by an ulp on single-element ranges
    stack = np.concatenate([np.arange(e0 - co.offset, e1 + 1 - co.offset) for e0, e1 in ranges])
    f1M = ((co.f1[stack] / rho) @ M.T)
    f2M = (co.f2[stack] @ M.T)
    base = 0
    for (e0, e1), (oL, oR) in zip(ranges, outer):
        idx = slice(e0 - co.offset, e1 + 1 - co.offset)
        s11, s12, s22 = co.s11[idx], co.s12[idx], co.s22[idx]
        m = e1 - e0 + 1
        P = base + 2 * (2 * np.arange(m)[:, None] + np.arange(2)[None, :])   # (m, 2)
        Q = P + 1
        for i in range(2):
            for j in range(2):
                put(P[:, i], P[:, j], -K[i, j] + M[i, j] * s11[:, j])
                put(P[:, i], Q[:, j], M[i, j] * (s12[:, j] / rho))
                put(Q[:, i], Q[:, j], -K[i, j] + M[i, j] * (-s11[:, j]))
                put(Q[:, i], P[:, j], M[i, j] * (rho * s22[:, j]))
        if m > 1:
            pL, pR, qL, qR = P[:-1, 1], P[1:, 0], Q[:-1, 1], Q[1:, 0]
            for (rh, rl, terms) in ((pL, pR, ((pL, 0.5 - c12), (pR, 0.5 + c12), (qL, c22), (qR, -c22))),
                                    (qL, qR, ((qL, 0.5 + c12), (qR, 0.5 - c12), (pL, c11), (pR, -c11)))):
                for col, cf in terms:
                    if cf != 0.0:
                        put(rh, col, cf)
                        put(rl, col, -cf)
        put(Q[0, 0], Q[0, 0], -(0.5 - c12))
        put(Q[0, 0], P[0, 0], c11)
        put(Q[-1, 1], Q[-1, 1], 0.5 + c12)
        put(Q[-1, 1], P[-1, 1], c11)
        b[P.ravel()] = f1M[base // 4:base // 4 + m].ravel()
        b[Q.ravel()] = f2M[base // 4:base // 4 + m].ravel()
        b[Q[0, 0]] += (0.5 + c12) * oL
        b[Q[-1, 1]] -= (0.5 - c12) * oR
        base += 4 * m
    return ab, b


def band_solve(grid, co: Coeffs, ranges, outer, c11=0.5, c12=-0.5, c22=0.0, tol=1e-10):
    """corrector.py:292-370: one dgbsv over all ranges, residual gate, p = rho * x_p."""
    for e0, e1 in ranges:
        if e0 > e1 or e0 < 0 or e1 >= grid.n:
            raise ValueError(f"invalid element range {(e0, e1)}")
    ab, b = _band_system(grid, co, ranges, outer, c11, c12, c22)
    mat = ab[3:].copy()
    bnorm = float(np.linalg.norm(b))
    _, _, x, info = _lapack.dgbsv(3, 3, ab, b, overwrite_ab=True, overwrite_b=False)
    if info != 0:
        raise OracleSolveError(f"singular elliptic system on {ranges} (lapack info {info})")
    if not np.isfinite(x.sum()):
        raise OracleSolveError(f"non-finite elliptic solution on {ranges}")
    Ax = mat[3] * x
    for k in range(1, 4):
        Ax[:-k] += mat[3 - k, k:] * x[k:]
        Ax[k:] += mat[3 + k, :-k] * x[:-k]
    scale = max(bnorm, float(np.abs(mat).max() * np.linalg.norm(x)), 1e-300)
    rel = float(np.linalg.norm(Ax - b)) / scale
    if rel > tol:
        raise OracleSolveError(f"elliptic solve residual {rel:.3e} exceeds {tol:.1e} on {ranges}")
    return co.rho * x[0::2].reshape(-1, 2), x[1::2].reshape(-1, 2)


def outer_traces(bcs, h, hu, hw, e0, e1):
    """corrector.py:388-403: uncorrected hu just outside a range (ghost at the ends)."""
    n = h.shape[0]
    left = hu[e0 - 1, 1] if e0 > 0 else _ghost(bcs[0], h[0, 0], hu[0, 0], hw[0, 0])[1]
    right = hu[e1 + 1, 0] if e1 < n - 1 else _ghost(bcs[1], h[-1, 1], hu[-1, 1], hw[-1, 1])[1]
    return left, right


def central_derivative(grid, v):
    """corrector.py:427-438: element derivative + central-average lifting."""
    out = elem_derivative(grid, v)
    avg = 0.5 * (v[:-1, 1] + v[1:, 0])
    out[:-1] += np.outer(avg - v[:-1, 1], grid.lift_right)
    out[1:] -= np.outer(avg - v[1:, 0], grid.lift_left)
    return out


def correction(grid, bottom, bcs, g, rho, h, hu, hw, t, dt, ranges, c11=0.5, c12=-0.5, c22=0.0):
    """apply_correction (corrector.py:485-498) = coefficients -> solve -> momenta."""
    ranges = tuple(sorted(tuple(int(v) for v in r) for r in ranges))
    n = grid.n
    lo = max(ranges[0][0] - 1, 0)
    hi = min(ranges[-1][1] + 1, n - 1)
    co = coefficients(grid, bottom, h, hu, hw, t, dt, g, rho, lo, hi)
    outer = [outer_traces(bcs, h, hu, hw, e0, e1) for e0, e1 in ranges]
    p_r, q_r = band_solve(grid, co, ranges, outer, c11, c12, c22)
    p = np.zeros_like(h)
    hu_new = hu.copy()
    k = 0
    for e0, e1 in ranges:
        m = e1 - e0 + 1
        p[e0:e1 + 1] = p_r[k:k + m]
        hu_new[e0:e1 + 1] = q_r[k:k + m]
        k += m
    # vertical momentum from the bottom pressure (corrector.py:441-482)
    win = slice(lo, hi + 1)
    pw = p[win]
    dxw = co.d_x
    if dxw.any():
        quad = 4.0 + dxw * dxw
        bp = 6.0 / quad * pw + dxw / quad * central_derivative(grid, h[win] * pw)
    else:
        bp = 1.5 * pw
    if co.phi.any():
        bp += co.phi
    hw_new = hw.copy()
    for e0, e1 in ranges:
        hw_new[e0:e1 + 1] += (dt / rho) * bp[e0 - lo:e1 + 1 - lo]
    return hu_new, hw_new, p


# --------------------------------------------------------------------------
# One step and the time loop  (adaptivity.py:127-163, driver.py:50-103)
# --------------------------------------------------------------------------

@dataclass
class Member:
    """Everything one channel needs: grid, bottom, boundary kinds, dt."""
    grid: Grid
    bottom: Bottom
    bcs: tuple
    dt: float
    g: float = GRAVITY


@dataclass
class StepOut:
    h: np.ndarray
    hu: np.ndarray
    hw: np.ndarray
    flags: np.ndarray
    p: np.ndarray | None


def step(mem: Member, h, hu, hw, t, mode="adaptive", kind="eta_over_d", k_nh=1e-3,
         enlarge=False, rho=RHO_WATER, c11=0.5, c12=-0.5, c22=0.0, cfl_warn=True):
    """adaptivity.py:127-163."""
    if mode not in ("hydrostatic", "global", "adaptive"):
        raise ValueError(f"unknown mode {mode!r}")
    grid, bot, g, dt = mem.grid, mem.bottom, mem.g, mem.dt
    n = grid.n
    ph, pq, pw = heun(grid, bot, mem.bcs, g, h, hu, hw, t, dt, cfl_warn)
    t1 = t + dt
    if mode == "hydrostatic":
        return StepOut(ph, pq, pw, np.zeros(n, bool), None)
    if mode == "global" or (kind in ("w", "w_x") and not np.any(hw)):
        flags = np.ones(n, bool)
    else:
        flags = flags_from(indicator(grid, bot, kind, ph, pq, pw, t1), k_nh, enlarge)
    if not flags.any():
        return StepOut(ph, pq, pw, flags, None)
    q2, w2, p = correction(grid, bot, mem.bcs, g, rho, ph, pq, pw, t1, dt, runs(flags),
                           c11, c12, c22)
    return StepOut(ph, q2, w2, flags, p)


@dataclass
class RunOut:
    h: np.ndarray
    hu: np.ndarray
    hw: np.ndarray
    t: float
    p: np.ndarray | None
    flags: np.ndarray | None
    mask_history: list = field(default_factory=list)
    fraction_mean: float = 0.0
    loop_time: float = 0.0


def run(mem: Member, h, hu, hw, n_steps, t0=0.0, mode="adaptive", kind="eta_over_d",
        k_nh=1e-3, enlarge=False, rho=RHO_WATER, record=False, flag_bits=False):
    """driver.py:50-103: fixed-dt loop; only the step calls are timed.

    Time accumulates as t + dt per step (hydrostatic.py:206-209).  With
    ``record`` the per-step flags are kept (bit-packed when ``flag_bits``).
    """
    import time as _time
    t = t0
    hist = []
    fr = 0.0
    p = flags = None
    spent = 0.0
    for _ in range(n_steps):
        c0 = _time.perf_counter()
        o = step(mem, h, hu, hw, t, mode, kind, k_nh, enlarge, rho)
        spent += _time.perf_counter() - c0
        h, hu, hw, p, flags = o.h, o.hu, o.hw, o.p, o.flags
        t = t + mem.dt
        fr += float(np.mean(flags))
        if record:
            hist.append(np.packbits(flags) if flag_bits else flags.copy())
    return RunOut(h, hu, hw, t, p, flags, hist, fr / n_steps if n_steps else 0.0, spent)
