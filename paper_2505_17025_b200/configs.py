"""The five BASELINE.json configurations as seeded member tables + initial states.

Input generation only (the analogue of the reference's scenarios.py, which
SURVEY.md §2 marks out of the hot path).  A configuration is a table of
members -- geometry, fixed dt, boundary kinds, bottom model -- plus the
recipe for the initial (h, hu, hw):

  * solitary members: eta = a sech^2(k (x - x0)), k = sqrt(3a / (4 h0^3)),
    hu = h c eta / (h0 + eta), c = sqrt(g (h0 + a)) at grid.nodes, and hw from
    the divergence constraint (reference scenarios.py:72-78);
  * still-water members: h = d(sample_nodes, t=0), hu = hw = 0
    (reference scenarios.py:65-69).

dt = 0.5 dx / (3 lambda_max(t = 0)) per member (SURVEY.md F4 / Appendix
C.1), n_steps = round(t_end / dt) for configs 1-3 (scenarios.py:47-49).
The formulas are written against an array module so the same code fills
numpy arrays (parity runs, then uploaded) and CUDA tensors (the 51.5 GB
config-5 ensemble is generated directly in HBM).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from functools import lru_cache

import numpy as np

from . import _lib
from .bathymetry import GRAVITY, FlatBottom, SlopeGaussianSlide, SmoothBoxPlate
from .grid import GridSpec
from .hydrostatic import ABSORBING, WALL, BoundaryPair

SEED_CONFIG4 = 20250523
SEED_CONFIG5 = 20250524


def dt_from_cfl(dx, lam_max, cfl=0.5, p=1):
    """dt = cfl dx / ((2p+1) lambda_max)."""
    return cfl * dx / ((2 * p + 1) * lam_max)


def element_derivative(xp, v, dx):
    """grid.py:214-215 for P1: (-v0/2 + v1/2) (2/dx), same value on both nodes."""
    d = (v[..., 1] * 0.5 + v[..., 0] * -0.5) * (2.0 / dx)
    return xp.stack([d, d], -1)


def solitary_state(xp, nodes, h0, a, x0, dx, g=GRAVITY):
    """(h, hu, hw) of the BASELINE config-1 solitary wave on a flat bed.

    nodes [..., N, 2]; h0, a, x0, dx broadcast over the leading axes.
    """
    k = xp.sqrt(3.0 * a / (4.0 * h0 ** 3))
    c = xp.sqrt(g * (h0 + a))
    eta = a / xp.cosh(k * (nodes - x0)) ** 2
    h = h0 + eta
    hu = h * (c * eta / (h0 + eta))
    hu_x = element_derivative(xp, hu, dx)
    h_x = element_derivative(xp, h, dx)
    # hw = (-h hu_x - hu (2d - h)_x - 2 h d_t) / 2 with d = h0, d_t = 0
    hw = 0.5 * (-h * hu_x - hu * (-h_x))
    return h, hu, hw


@dataclass
class MemberSpec:
    """One channel, in the reference's vocabulary."""
    grid: GridSpec
    bathymetry: object
    bcs: BoundaryPair
    dt: float
    init: str                       # "solitary" | "still"
    init_params: dict = field(default_factory=dict)


@dataclass
class Config:
    name: str
    n_members: int
    n_elements: int
    n_steps: int
    modes: tuple
    t_end: float | None = None

    def member(self, i: int) -> MemberSpec:
        raise NotImplementedError

    def records(self, idx=None) -> np.ndarray:
        """nh_member table for members idx (default: all)."""
        from ._device import member_record
        idx = range(self.n_members) if idx is None else idx
        return np.concatenate([member_record(m.grid, m.bathymetry, m.bcs, m.dt)
                               for m in (self.member(i) for i in idx)])

    def host_state(self, i: int, depth_fn):
        """Initial (h, hu, hw) of member i as numpy (N, 2) arrays.

        depth_fn(model, x, t) supplies still-water depths (the parity tests
        pass the CPU oracle's bottom, the GPU path passes bathymetry.sample).
        """
        m = self.member(i)
        g = m.grid
        if m.init == "solitary":
            p = m.init_params
            return solitary_state(np, g.nodes, m.bathymetry.h0, p["a"], p["x0"], g.dx)
        d = np.asarray(depth_fn(m.bathymetry, g.sample_nodes, 0.0), dtype=np.float64)
        return d.copy(), np.zeros_like(d), np.zeros_like(d)


# ---------------------------------------------------------------- configs 1-3

class _Single(Config):
    def __init__(self, name, spec: MemberSpec, t_end, modes):
        n_steps = int(round(t_end / spec.dt))
        super().__init__(name, 1, spec.grid.n_elements, n_steps, modes, t_end)
        self._spec = spec

    def member(self, i):
        if i != 0:
            raise IndexError(i)
        return self._spec


def config1() -> Config:
    """Solitary wave a=0.1, h0=1, N=2000 on [0,200], x0=40, outflow both ends, t=30 s."""
    h0, a, x0 = 1.0, 0.1, 40.0
    grid = GridSpec(0.0, 200.0, 2000)
    h, hu, _ = solitary_state(np, grid.nodes, h0, a, x0, grid.dx)
    lam = float(np.max(np.abs(hu / h) + np.sqrt(GRAVITY * h)))
    spec = MemberSpec(grid, FlatBottom(h0), BoundaryPair(ABSORBING, ABSORBING),
                      dt_from_cfl(grid.dx, lam), "solitary", {"a": a, "x0": x0})
    return _Single("config1_solitary", spec, 30.0, ("global", "adaptive"))


def config2() -> Config:
    """Smoothed box uplift next to a wall: h0=0.05, N=4000 on [0,10], t=8 s."""
    h0 = 0.05
    grid = GridSpec(0.0, 10.0, 4000)
    spec = MemberSpec(grid, SmoothBoxPlate(h0, 0.005, 0.3, 20.0, 0.01),
                      BoundaryPair(WALL, ABSORBING), dt_from_cfl(grid.dx, math.sqrt(GRAVITY * h0)),
                      "still")
    return _Single("config2_box_uplift", spec, 8.0, ("adaptive",))


def config3() -> Config:
    """Gaussian mound sliding down a 15 deg slope, N=8000 on [0,20], t=15 s."""
    grid = GridSpec(0.0, 20.0, 8000)
    bathy = SlopeGaussianSlide(0.1, math.tan(math.radians(15.0)), 1.0, 0.05, 0.2, 1.0, 1.0,
                               0.5, 0.8)
    spec = MemberSpec(grid, bathy, BoundaryPair(WALL, ABSORBING),
                      dt_from_cfl(grid.dx, math.sqrt(GRAVITY * 1.0)), "still")
    return _Single("config3_slope_slide", spec, 15.0, ("adaptive",))


# ---------------------------------------------------------------- config 4

def member_rng(seed: int, i: int) -> np.random.Generator:
    """Member i's own generator: its parameters depend on (seed, i) only, not
    on the ensemble size, so a member is the same channel in a 4096-member run,
    a 1-member parity run and any rank's shard of a sharded run."""
    return np.random.default_rng([seed, i])


@lru_cache(maxsize=8192)
def _config4_draw(seed: int, i: int):
    rng = member_rng(seed, i)
    return {k: float(rng.uniform(lo, hi)) for k, (lo, hi) in
            (("h0", (0.5, 2.0)), ("a_rel", (0.05, 0.3)), ("zeta_rel", (0.01, 0.1)),
             ("b_rel", (0.1, 1.0)), ("alpha", (5.0, 50.0)))}


class Config4(Config):
    """Mixed ensemble: even members solitary waves, odd members box uplifts.

    Solitary members: h0 ~ U(0.5, 2) m, a/h0 ~ U(0.05, 0.3), x0 = 0.2 L,
    outflow both ends.  Box members: h0 = 0.01 m (lab scale; BASELINE leaves
    their depth unstated), zeta0/h0 ~ U(0.01, 0.1), b ~ U(0.1, 1) h0,
    alpha ~ U(5, 50) 1/s, edge w = 0.2 h0, wall / outflow.  Every member's
    domain is [0, 200 h0].  At field depth (h0 ~ 1 m) an uplift with
    alpha = 30-50 1/s is ~15x more impulsive (alpha sqrt(h0/g)) than the
    reference's own Hammack plate and the reference model itself loses
    positivity within ~0.15 s; at h0 = 0.01 m alpha sqrt(h0/g) spans
    0.16-1.6 around Hammack's 0.61 and every corner of the box parameter
    range runs the full 20000 steps.
    """

    BOX_H0 = 0.01

    def __init__(self, n_members=4096, n_elements=4096, n_steps=20000, seed=SEED_CONFIG4):
        super().__init__("config4_mixed_ensemble", n_members, n_elements, n_steps, ("adaptive",))
        self.seed = seed

    def member(self, i):
        if not 0 <= i < self.n_members:
            raise IndexError(i)
        r = _config4_draw(self.seed, i)
        h0 = r["h0"]
        L = 200.0 * h0
        grid = GridSpec(0.0, L, self.n_elements)
        if i % 2 == 0:
            a = h0 * r["a_rel"]
            x0 = 0.2 * L
            h, hu, _ = solitary_state(np, grid.nodes, h0, a, x0, grid.dx)
            lam = float(np.max(np.abs(hu / h) + np.sqrt(GRAVITY * h)))
            return MemberSpec(grid, FlatBottom(h0), BoundaryPair(ABSORBING, ABSORBING),
                              dt_from_cfl(grid.dx, lam), "solitary", {"a": a, "x0": x0})
        h0 = self.BOX_H0
        L = 200.0 * h0
        grid = GridSpec(0.0, L, self.n_elements)
        bathy = SmoothBoxPlate(h0, h0 * r["zeta_rel"], h0 * r["b_rel"], r["alpha"], 0.2 * h0)
        return MemberSpec(grid, bathy, BoundaryPair(WALL, ABSORBING),
                          dt_from_cfl(grid.dx, math.sqrt(GRAVITY * h0)), "still")


# ---------------------------------------------------------------- config 5

def _slide_ok(tan_t, A, sigma, x0, xs):
    """Vectorised admissibility: wet depth >= 0.04 m for every mound position
    between x0 and the stop point, and a path of >= 0.5 m."""
    x_stop = 0.7 / tan_t
    ok = x_stop >= x0 + 0.5
    worst = np.full(tan_t.shape, np.inf)
    for f in np.linspace(0.0, 1.0, 9):
        xc = x0 + f * np.maximum(x_stop - x0, 0.0)
        r = (xs[None, :] - xc[:, None]) / sigma[:, None]
        d = np.minimum(0.1 + xs[None, :] * tan_t[:, None], 1.0) - A[:, None] * np.exp(-0.5 * r * r)
        worst = np.minimum(worst, d.min(axis=1))
    return ok & (worst >= 0.04)


def _config5_rows(seed: int, idx) -> np.ndarray:
    """(tan_theta, A, sigma, x0, u_t) of members idx, each rejection-sampled
    from its own generator (member_rng): candidates are drawn in rounds and
    checked vectorised; a rejected member draws its next candidate from the
    same generator."""
    idx = np.asarray(idx, dtype=np.int64)
    xs = np.linspace(0.0, 20.0, 321)
    gens = [member_rng(seed, int(i)) for i in idx]
    out = np.zeros((idx.size, 5))
    todo = np.arange(idx.size)
    for _ in range(200):
        if todo.size == 0:
            break
        d = np.array([[gens[k].uniform(5.0, 20.0), gens[k].uniform(0.05, 0.5),
                       gens[k].uniform(0.1, 1.0), gens[k].uniform(0.2, 2.0)] for k in todo])
        tan_t = np.tan(np.radians(d[:, 0]))
        ratio, sigma, u_t = d[:, 1], d[:, 2], d[:, 3]
        x0 = 1.0 + 2.0 * sigma
        A = ratio * np.minimum(0.1 + x0 * tan_t, 1.0)
        ok = _slide_ok(tan_t, A, sigma, x0, xs)
        out[todo[ok]] = np.stack([tan_t, A, sigma, x0, u_t], 1)[ok]
        todo = todo[~ok]
    if todo.size:
        raise RuntimeError("config-5 rejection sampling did not converge")
    return out


@lru_cache(maxsize=2)
def _config5_table(n_members: int, seed: int):
    """Rows of members 0..n_members-1 (row i depends on (seed, i) only)."""
    out = np.zeros((n_members, 5))
    for c0 in range(0, n_members, 8192):
        out[c0:c0 + 8192] = _config5_rows(seed, range(c0, min(c0 + 8192, n_members)))
    return out


class Config5(Config):
    """Landslide ensemble: config-3 geometry with seeded slope / mound / speed.

    slope ~ U(5, 20) deg, mound height / local depth at x_c(0) ~ U(0.05, 0.5),
    sigma ~ U(0.1, 1) m, terminal speed ~ U(0.2, 2) m/s, t0 = 0.5 s, stop at
    depth 0.8 m; x_c(0) = 1 + 2 sigma.  Draws are rejected (and redrawn from
    the same generator) when the wet depth would fall below 0.04 m or the
    mound would travel less than 0.5 m.
    """

    def __init__(self, n_members=65536, n_elements=16384, n_steps=10000, seed=SEED_CONFIG5):
        super().__init__("config5_landslide_ensemble", n_members, n_elements, n_steps,
                         ("global", "adaptive"))
        self.seed = seed
        self.grid = GridSpec(0.0, 20.0, n_elements)
        self.dt = dt_from_cfl(self.grid.dx, math.sqrt(GRAVITY * 1.0))

    def table(self):
        return _config5_table(self.n_members, self.seed)

    def member(self, i):
        tan_t, A, sigma, x0, u_t = (float(v) for v in self.table()[i])
        bathy = SlopeGaussianSlide(0.1, tan_t, 1.0, A, sigma, x0, u_t, 0.5, 0.8)
        return MemberSpec(self.grid, bathy, BoundaryPair(WALL, ABSORBING), self.dt, "still")

    def records(self, idx=None):
        from ._device import member_record
        idx = range(self.n_members) if idx is None else idx
        base = member_record(self.grid, FlatBottom(1.0), BoundaryPair(WALL, ABSORBING), self.dt)
        rec = np.repeat(base, len(idx))
        rec["bottom_kind"] = _lib.BOTTOM_SLOPE_SLIDE
        # the bottom model's own pack(): x_stop / t_stop bit-identical to the
        # model the oracle evaluates
        for k, i in enumerate(idx):
            _, params = self.member(int(i)).bathymetry.pack()
            rec["bottom"][k, :len(params)] = params
        return rec


def get(name: str, **kw) -> Config:
    return {"config1": config1, "config2": config2, "config3": config3,
            "config4": Config4, "config5": Config5}[name](**kw)
