"""Shared test helpers: package <-> oracle object conversion and comparisons."""

import numpy as np

import paper_2505_17025_b200 as P
from oracle import nhswe_oracle as O


def oracle_bottom(b):
    if isinstance(b, P.FlatBottom):
        return O.Flat(b.h0)
    if isinstance(b, P.HammackPlate):
        return O.Plate(b.h0, b.zeta0, b.b, b.t_c)
    if isinstance(b, P.WhittakerSlide):
        m = b.motion
        return O.QuarticSlide(b.h0, b.Hs, b.Ls, O.Motion(m.a0, m.u_t, m.t1, m.t2, m.t3), b.x_start)
    if isinstance(b, P.SmoothBoxPlate):
        return O.SmoothBox(b.h0, b.zeta0, b.b, b.alpha, b.w)
    if isinstance(b, P.SlopeGaussianSlide):
        return O.SlopeSlide(b.d_top, b.tan_theta, b.d_max, b.A, b.sigma, b.x0, b.u_t, b.t0,
                            b.d_stop)
    raise TypeError(type(b))


def oracle_member(grid, bathy, bcs, dt):
    return O.Member(O.Grid(grid.x_left, grid.x_right, grid.n_elements), oracle_bottom(bathy),
                    (bcs.left.kind, bcs.right.kind), dt)


def oracle_depth(model, x, t):
    return oracle_bottom(model).channels(np.asarray(x, dtype=float), t)[0]


def rel(a, b):
    a = np.asarray(a)
    b = np.asarray(b)
    scale = max(np.abs(b).max(), 1e-300)
    return float(np.abs(a - b).max() / scale)


def mask_mismatch_outside_margin(gpu_flags, oracle_vals, k_nh, enlarge=False, margin=1e-12):
    """Elements whose GPU flag differs from the oracle's although the oracle's
    criterion is not within `margin` (relative) of the threshold."""
    v = oracle_vals.max(axis=1)
    f = v > k_nh
    if enlarge:
        g = f.copy(); g[:-1] |= f[1:]; g[1:] |= f[:-1]; f = g
    near = np.abs(v - k_nh) <= margin * k_nh
    if enlarge:
        nn = near.copy(); nn[:-1] |= near[1:]; nn[1:] |= near[:-1]; near = nn
    return np.flatnonzero((np.asarray(gpu_flags) != f) & ~near)


def smooth_state(grid, d0=10.0, amp=0.5, u0=0.2):
    x = grid.nodes
    h = d0 + amp * np.exp(-((x - x.mean()) / 5.0) ** 2)
    hu = u0 * h * np.sin(0.3 * x)
    hw = 0.05 * h * np.cos(0.2 * x)
    return P.FlowState(P.NodalField(grid, h), P.NodalField(grid, hu), P.NodalField(grid, hw), 0.0)


def scenario_cases():
    """(name, grid, bathy, bcs, dt, (h, hu, hw)) small cases covering every bottom model."""
    cases = []
    g = P.GridSpec(0.0, 100.0, 120)
    s = smooth_state(g)
    cases.append(("flat_walls", g, P.FlatBottom(10.0), P.BoundaryPair(P.WALL, P.WALL), 0.02,
                  (s.h.values, s.hu.values, s.hw.values)))
    cases.append(("flat_absorbing", g, P.FlatBottom(10.0),
                  P.BoundaryPair(P.ABSORBING, P.ABSORBING), 0.02,
                  (s.h.values, s.hu.values, s.hw.values)))
    g = P.GridSpec(0.0, 5.0, 200)
    b = P.HammackPlate(0.05, 0.005, 0.6, 0.13)
    d = oracle_depth(b, g.sample_nodes, 0.0)
    cases.append(("plate", g, b, P.BoundaryPair(P.WALL, P.ABSORBING), 0.004,
                  (d, np.zeros_like(d), np.zeros_like(d))))
    g = P.GridSpec(0.0, 15.0, 200)
    b = P.WhittakerSlide(0.175, 0.026, 0.5, P.SlideMotion(1.5, 0.327, 0.218, 2.218, 2.436), 5.0)
    d = oracle_depth(b, g.sample_nodes, 0.0)
    cases.append(("quartic_slide", g, b, P.BoundaryPair(P.ABSORBING, P.ABSORBING), 0.005,
                  (d, np.zeros_like(d), np.zeros_like(d))))
    g = P.GridSpec(0.0, 10.0, 400)
    b = P.SmoothBoxPlate(0.05, 0.005, 0.3, 20.0, 0.01)
    d = oracle_depth(b, g.sample_nodes, 0.0)
    cases.append(("smooth_box", g, b, P.BoundaryPair(P.WALL, P.ABSORBING), 0.0059,
                  (d, np.zeros_like(d), np.zeros_like(d))))
    g = P.GridSpec(0.0, 20.0, 800)
    b = P.SlopeGaussianSlide(0.1, np.tan(np.radians(15.0)), 1.0, 0.05, 0.2, 1.0, 1.0, 0.5, 0.8)
    d = oracle_depth(b, g.sample_nodes, 0.0)
    cases.append(("slope_slide", g, b, P.BoundaryPair(P.WALL, P.ABSORBING), 0.0013,
                  (d, np.zeros_like(d), np.zeros_like(d))))
    return cases


def state_of(grid, arrs, t=0.0):
    h, hu, hw = arrs
    return P.FlowState(P.NodalField(grid, h), P.NodalField(grid, hu), P.NodalField(grid, hw), t)
