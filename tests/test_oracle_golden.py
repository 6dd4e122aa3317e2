"""The CPU oracle reproduces the real reference's outputs (tests/golden/short.npz,
produced by tests/golden/make_golden.py from /root/reference) -- bit for bit on
the host that made them; 1e-13 relative elsewhere (numpy/BLAS rounding)."""

import os

import numpy as np
import pytest

from oracle import nhswe_oracle as O
from tests.oracle_cases import NAMES, load_short, member_from, state_from

D = load_short()
TOL = 1e-13
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def close(a, b, tol=TOL):
    a, b = np.asarray(a), np.asarray(b)
    if np.array_equal(a, b):
        return True
    return np.abs(a - b).max() <= tol * max(np.abs(b).max(), 1e-300)


@pytest.mark.parametrize("name", NAMES)
def test_grid_constants(name):
    m = member_from(D, name)
    for k in ("mass", "mass_inv", "stiffness", "deriv_ref", "weak_div", "lift_left",
              "lift_right", "sample_nodes"):
        assert np.array_equal(getattr(m.grid, k), D[name + "/grid_" + k]), k


@pytest.mark.parametrize("name", NAMES)
def test_rhs_and_heun(name):
    m = member_from(D, name)
    h, hu, hw = state_from(D, name)
    t = O.tendency(m.grid, m.bottom, m.bcs, 9.81, h, hu, hw, 0.0)
    for a, b in zip(t, D[name + "/rhs"]):
        assert close(a, b)
    p = O.heun(m.grid, m.bottom, m.bcs, 9.81, h, hu, hw, 0.0, m.dt, cfl_warn=False)
    for a, b in zip(p, D[name + "/heun"]):
        assert close(a, b)


@pytest.mark.parametrize("name", NAMES)
def test_criteria_coefficients_correction(name):
    m = member_from(D, name)
    h, hu, hw = state_from(D, name)
    ph, pq, pw = O.heun(m.grid, m.bottom, m.bcs, 9.81, h, hu, hw, 0.0, m.dt, cfl_warn=False)
    t1 = 0.0 + m.dt
    for kind in O.KINDS:
        assert close(O.indicator(m.grid, m.bottom, kind, ph, pq, pw, t1), D[name + "/crit_" + kind])
    co = O.coefficients(m.grid, m.bottom, ph, pq, pw, t1, m.dt, 9.81, 1000.0, 0, m.grid.n - 1)
    for a, b in zip((co.s11, co.s12, co.s22, co.f1, co.f2, co.phi), D[name + "/coef"]):
        assert close(a, b)
    ranges = tuple(tuple(int(v) for v in r) for r in D[name + "/corr_ranges"])
    q2, w2, p = O.correction(m.grid, m.bottom, m.bcs, 9.81, 1000.0, ph, pq, pw, t1, m.dt, ranges)
    ref = D[name + "/corr"]
    assert close(q2, ref[0], 1e-12) and close(w2, ref[1], 1e-12) and close(p, ref[2], 1e-12)


@pytest.mark.parametrize("mode", ["hydrostatic", "global", "adaptive", "adaptive_enl",
                                  "adaptive_wx"])
@pytest.mark.parametrize("name", NAMES)
def test_trajectories(name, mode):
    m = member_from(D, name)
    h, hu, hw = state_from(D, name)
    kind = "w_x" if mode == "adaptive_wx" else "eta_over_d"
    t = 0.0
    flags = []
    for _ in range(12):
        o = O.step(m, h, hu, hw, t, mode.split("_")[0], kind, 1e-3, mode == "adaptive_enl",
                   cfl_warn=False)
        h, hu, hw = o.h, o.hu, o.hw
        t += m.dt
        flags.append(o.flags)
    assert np.array_equal(np.array(flags), D[name + "/traj_" + mode + "_flags"])
    for a, b in zip((h, hu, hw), D[name + "/traj_" + mode]):
        assert close(a, b, 1e-12)


def test_manufactured_solve():
    s11, s12, s22, f1, f2 = D["manufactured/coef"]
    g = O.Grid(0.0, 1.0, 48)
    co = O.Coeffs(s11, s12, s22, f1, f2, np.zeros_like(s11), np.zeros_like(s11), 0, 0.1, 1.0)
    p, hu = O.band_solve(g, co, ((3, 40),), [tuple(D["manufactured/outer"])])
    ref = D["manufactured/solution"]
    assert close(p, ref[0], 1e-12) and close(hu, ref[1], 1e-12)


def test_runs_helper():
    assert O.runs(np.array([], bool)) == ()
    assert O.runs(np.array([1, 1, 0, 1], bool)) == ((0, 1), (3, 3))
    assert O.runs(np.ones(4, bool)) == ((0, 3),)


def test_config3_kicked_envelope_file():
    """config3_kicked.npz (make_config3_kicked.py): the reference's arithmetic
    restarted from its own step-20000 checkpoint with h kicked by 1e-10; its
    counts equal the reference's up to the restart and it is a complete run."""
    G = np.load(os.path.join(GOLDEN, "config3_full.npz"))
    K = np.load(os.path.join(GOLDEN, "config3_kicked.npz"))
    s = int(K["start"])
    c = K["counts"].astype(np.int64)
    assert c.size == int(G["n_steps"])
    assert np.array_equal(c[:s], G["adaptive/flag_count"][:s])
    assert abs(c.mean() / 8000 - float(K["mask_fraction"])) < 1e-12
