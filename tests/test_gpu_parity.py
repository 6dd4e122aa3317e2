"""GPU parity: every public hot-path function against the CPU oracle.

The oracle (oracle/nhswe_oracle.py) is pinned bit-for-bit to the reference
by tests/test_oracle_golden.py; here the CUDA path must agree with it
within the north star's tolerances:
  * states: relative L-inf <= 1e-12 after one step, <= 1e-9 after many;
  * masks: identical except for cells whose oracle criterion lies within
    1e-12 (relative) of k_nh.
"""

import numpy as np
import pytest

import paper_2505_17025_b200 as P
from oracle import nhswe_oracle as O
from tests.helpers import (mask_mismatch_outside_margin, oracle_member, rel, scenario_cases,
                           smooth_state, state_of)

pytestmark = pytest.mark.gpu
CASES = scenario_cases()
IDS = [c[0] for c in CASES]


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_rhs_operator(case):
    _, grid, bathy, bcs, dt, arrs = case
    st = state_of(grid, arrs, t=0.37)
    mem = oracle_member(grid, bathy, bcs, dt)
    ref = O.tendency(mem.grid, mem.bottom, mem.bcs, 9.81, *arrs, 0.37)
    got = P.rhs_operator(st, bathy, bcs)
    # still-water tendencies are pure roundoff of g h^2 / dx sized terms
    natural = 9.81 * np.abs(arrs[0]).max() ** 2 / grid.dx
    for a, b in zip(got, ref):
        scale = max(np.abs(b).max(), 1e-3 * natural)
        assert np.abs(a - b).max() <= 1e-11 * scale


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_heun_steps(case):
    _, grid, bathy, bcs, dt, arrs = case
    mem = oracle_member(grid, bathy, bcs, dt)
    st = state_of(grid, arrs)
    h, hu, hw = arrs
    t = 0.0
    for i in range(30):
        st = P.heun_step(st, dt, bathy, bcs, cfl_warn=False)
        h, hu, hw = O.heun(mem.grid, mem.bottom, mem.bcs, 9.81, h, hu, hw, t, dt, cfl_warn=False)
        t = t + dt
        assert st.time == t
    assert rel(st.h.values, h) <= 1e-12
    assert rel(st.hu.values, hu) <= 1e-10 or np.abs(st.hu.values - hu).max() <= 1e-14
    assert np.abs(st.hw.values - hw).max() <= 1e-10 * max(np.abs(hw).max(), 1e-4)


@pytest.mark.parametrize("mode,kind,enlarge", [("global", "eta_over_d", False),
                                               ("adaptive", "eta_over_d", False),
                                               ("adaptive", "eta_over_d", True),
                                               ("adaptive", "u_x", False),
                                               ("adaptive", "w_x", True),
                                               ("adaptive", "eta_x", False)])
@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_adaptive_steps(case, mode, kind, enlarge):
    _, grid, bathy, bcs, dt, arrs = case
    mem = oracle_member(grid, bathy, bcs, dt)
    crit = P.Criterion(kind, 1e-3, enlarge)
    st = state_of(grid, arrs)
    h, hu, hw = arrs
    t = 0.0
    for i in range(25):
        r = P.adaptive_step(st, dt, bathy, bcs, mode=mode, crit=crit, cfl_warn=False)
        ph, pq, pw = O.heun(mem.grid, mem.bottom, mem.bcs, 9.81, h, hu, hw, t, dt, cfl_warn=False)
        o = O.step(mem, h, hu, hw, t, mode, kind, 1e-3, enlarge, cfl_warn=False)
        t = t + dt
        if mode == "adaptive" and not (kind in ("w", "w_x") and not np.any(hw)):
            vals = O.indicator(mem.grid, mem.bottom, kind, ph, pq, pw, t)
            bad = mask_mismatch_outside_margin(r.mask.flags, vals, 1e-3, enlarge)
            assert bad.size == 0, f"step {i}: mask differs at {bad[:10]}"
        else:
            assert np.array_equal(r.mask.flags, o.flags)
        if np.array_equal(r.mask.flags, o.flags):
            # continue from the oracle state so the comparison stays one-step
            assert rel(r.state.h.values, o.h) <= 1e-12
            assert rel(r.state.hu.values, o.hu) <= 1e-9 or np.abs(r.state.hu.values - o.hu).max() < 1e-13
            assert np.abs(r.state.hw.values - o.hw).max() <= 1e-9 * max(np.abs(o.hw).max(), 1e-6)
            if o.p is not None:
                assert r.p_nh is not None
                assert np.abs(r.p_nh.values - o.p).max() <= 1e-9 * max(np.abs(o.p).max(), 1e-6)
        h, hu, hw = o.h, o.hu, o.hw
        st = state_of(grid, (h, hu, hw), t)


def test_ldg_solve_manufactured():
    n = 64
    grid = P.GridSpec(0.0, 1.0, n)
    x = grid.nodes
    s11 = 0.4 * np.sin(2 * np.pi * x)
    s12 = 2 + np.cos(x)
    s22 = 1 + 0.5 * np.sin(3 * x)
    p_ex = np.sin(np.pi * x)
    hu_ex = np.cos(2 * x) + 2
    f1 = np.pi * np.cos(np.pi * x) + s11 * p_ex + s12 * hu_ex
    f2 = -2 * np.sin(2 * x) - s11 * hu_ex + s22 * p_ex
    bottom = P.BottomSample(*(np.zeros_like(x),) * 6)
    co = P.EllipticCoefficients(grid, s11, s12, -s11, s22, f1, f2, np.zeros_like(x), bottom,
                                0.1, 1.0)
    og = O.Grid(0.0, 1.0, n)
    oc = O.Coeffs(s11, s12, s22, f1, f2, np.zeros_like(x), np.zeros_like(x), 0, 0.1, 1.0)
    for (e0, e1) in [(0, 63), (3, 40), (10, 10), (62, 63)]:
        outer = (hu_ex[0, 0], hu_ex[-1, -1])
        p, hu = P.ldg_solve(co, (e0, e1), outer_hu=outer)
        pr, hr = O.band_solve(og, oc, ((e0, e1),), [outer])
        assert rel(p, pr) <= 1e-12
        assert rel(hu, hr) <= 1e-12


def test_solve_on_ranges_and_apply_correction():
    grid = P.GridSpec(0.0, 100.0, 60)
    st = smooth_state(grid)
    bcs = P.BoundaryPair(P.WALL, P.WALL)
    bathy = P.FlatBottom(10.0)
    ranges = ((3, 12), (20, 21), (30, 55), (59, 59))
    co = P.assemble_coefficients(st, bathy, 0.1)
    sol = P.solve_on_ranges(st, co, ranges, bcs)
    mem = oracle_member(grid, bathy, bcs, 0.1)
    hu2, hw2, p = O.correction(mem.grid, mem.bottom, mem.bcs, 9.81, 1000.0, st.h.values,
                               st.hu.values, st.hw.values, 0.0, 0.1, ranges)
    assert rel(sol.p_nh.values, p) <= 1e-11
    assert rel(sol.hu_corrected.values, hu2) <= 1e-12
    corrected, sol2 = P.apply_correction(st, bathy, 0.1, ranges, bcs)
    assert corrected.h is st.h
    assert rel(corrected.hu.values, hu2) <= 1e-12
    assert np.abs(corrected.hw.values - hw2).max() <= 1e-10 * np.abs(hw2).max()
    assert rel(sol2.p_nh.values, p) <= 1e-11
    cm = P.correct_momentum(st, sol, co)
    assert np.abs(cm.hw.values - hw2).max() <= 1e-10 * np.abs(hw2).max()
    assert np.array_equal(corrected.hu.values[:3], st.hu.values[:3])


@pytest.mark.parametrize("case", CASES, ids=IDS)
def test_coefficients_and_criterion(case):
    _, grid, bathy, bcs, dt, arrs = case
    st = state_of(grid, arrs, t=0.21)
    mem = oracle_member(grid, bathy, bcs, dt)
    co = P.assemble_coefficients(st, bathy, dt)
    oc = O.coefficients(mem.grid, mem.bottom, *arrs, 0.21, dt, 9.81, 1000.0, 0, grid.n_elements - 1)
    for a, b in ((co.s11, oc.s11), (co.s12, oc.s12), (co.s22, oc.s22), (co.f1, oc.f1),
                 (co.f2, oc.f2), (co.phi, oc.phi)):
        assert np.abs(a - b).max() <= 1e-12 * max(np.abs(b).max(), 1e-300)
    for kind in O.KINDS:
        v = P.criterion_values(st, bathy, kind)
        w = O.indicator(mem.grid, mem.bottom, kind, *arrs, 0.21)
        assert np.abs(v - w).max() <= 1e-12 * max(np.abs(w).max(), 1e-300)


def test_bottom_sample_all_models():
    x = np.linspace(-0.5, 20.0, 3001)
    for case in CASES:
        bathy = case[2]
        ob = oracle_member(case[1], bathy, case[3], case[4]).bottom
        for t in (0.0, 0.05, 0.7, 3.0):
            got = bathy.sample(x, t)
            ref = ob.channels(x, t)
            for k, r in zip(("d", "d_x", "d_t", "d_tt", "d_xt", "d_xx"), ref):
                a = getattr(got, k)
                assert np.abs(a - r).max() <= 1e-12 * max(np.abs(r).max(), 1e-300), (case[0], k, t)


def test_positivity_error():
    grid = P.GridSpec(0.0, 10.0, 10)
    h = np.ones((10, 2))
    h[4] = 1e-9
    hu = np.zeros((10, 2))
    hu[4] = 5.0
    s = P.FlowState(P.NodalField(grid, h), P.NodalField(grid, hu),
                    P.NodalField(grid, np.zeros((10, 2))), 0.0)
    with pytest.raises(P.PositivityError):
        for _ in range(50):
            s = P.heun_step(s, 0.5, P.FlatBottom(1.0), P.BoundaryPair(P.WALL, P.WALL),
                            cfl_warn=False)


def test_cfl_warning():
    grid = P.GridSpec(0.0, 10.0, 10)
    d = np.ones((10, 2))
    s = P.FlowState(P.NodalField(grid, d), P.NodalField(grid, 0 * d), P.NodalField(grid, 0 * d), 0.0)
    with pytest.warns(RuntimeWarning, match="CFL"):
        P.heun_step(s, 10.0, P.FlatBottom(1.0), P.BoundaryPair(P.WALL, P.WALL))


def test_empty_mask_is_hydrostatic_bitwise():
    grid = P.GridSpec(0.0, 10.0, 20)
    d = np.ones((20, 2))
    s = P.FlowState(P.NodalField(grid, d), P.NodalField(grid, 0 * d), P.NodalField(grid, 0 * d), 0.0)
    bcs = P.BoundaryPair(P.WALL, P.WALL)
    r = P.adaptive_step(s, 0.01, P.FlatBottom(1.0), bcs, mode="adaptive",
                        crit=P.Criterion("eta_over_d"))
    ref = P.heun_step(s, 0.01, P.FlatBottom(1.0), bcs)
    assert r.mask.empty and r.p_nh is None
    assert np.array_equal(r.state.h.values, ref.h.values)
    assert np.array_equal(r.state.hu.values, ref.hu.values)


def test_wx_first_step_falls_back_to_global():
    grid = P.GridSpec(0.0, 10.0, 20)
    d = np.ones((20, 2))
    s = P.FlowState(P.NodalField(grid, d), P.NodalField(grid, 0 * d), P.NodalField(grid, 0 * d), 0.0)
    r = P.adaptive_step(s, 0.01, P.FlatBottom(1.0), P.BoundaryPair(P.WALL, P.WALL),
                        mode="adaptive", crit=P.Criterion("w_x"))
    assert r.mask.fraction == 1.0


def test_full_mask_adaptive_equals_global():
    from paper_2505_17025_b200 import configs
    cfg = configs.config1()
    m = cfg.member(0)
    h, hu, hw = cfg.host_state(0, None)
    st = state_of(m.grid, (h + 1e-8, hu, hw))
    crit = P.Criterion("eta_over_d", k_nh=1e-12)
    sa, sg = st, st
    for _ in range(5):
        ra = P.adaptive_step(sa, m.dt, m.bathymetry, m.bcs, mode="adaptive", crit=crit)
        rg = P.adaptive_step(sg, m.dt, m.bathymetry, m.bcs, mode="global")
        sa, sg = ra.state, rg.state
        assert ra.mask.fraction == 1.0
    assert np.abs(sa.hu.values - sg.hu.values).max() < 1e-12
    assert np.abs(sa.hw.values - sg.hw.values).max() < 1e-12


def test_inline_ieee_division_and_sqrt_match_cuda():
    """The strict predictor's inline division / sqrt (nh_common.cuh) are the
    IEEE round-to-nearest results, bit-identical to __ddiv_rn / __dsqrt_rn."""
    import torch
    from paper_2505_17025_b200 import _device as D
    lib = D.require_cuda()
    bad = torch.zeros(3, dtype=torch.int64, device="cuda")
    n = 1 << 30
    assert lib.nh_selftest_arith(n, 20251020, bad.data_ptr(), D.stream_ptr()) == 0
    torch.cuda.synchronize()
    assert bad.tolist() == [0, 0, 0]


@pytest.mark.parametrize("enlarge", [False, True])
@pytest.mark.parametrize("kind", ["eta_over_d", "u_x", "w"])
def test_evaluate_criterion_and_max_wavespeed(kind, enlarge):
    """evaluate_criterion (adaptivity.py:107-113: nh_criterion + nh_mask on
    the device) equals the oracle's thresholded, enlarged indicator and the
    mask adaptive_step applies; max_wavespeed (hydrostatic.py:187-189,
    nh_max_wavespeed) equals the numpy expression bit for bit."""
    import paper_2505_17025_b200 as P
    from tests.test_gpu_golden import pkg_case
    from tests.helpers import oracle_member
    for name in ("flat_walls", "plate", "slope_slide"):
        g, b, bcs, dt, st = pkg_case(name)
        for _ in range(3):   # a developed state (nonzero hw for the w criterion)
            st = P.adaptive_step(st, dt, b, bcs, mode="global", cfl_warn=False).state
        pred = P.heun_step(st, dt, b, bcs, cfl_warn=False)
        k = 0.5 * float(np.abs(P.criterion_values(pred, b, kind)).max()) or 1e-3
        crit = P.Criterion(kind, k, enlarge)
        mask = P.evaluate_criterion(pred, b, crit)
        mem = oracle_member(g, b, bcs, dt)
        v = O.indicator(mem.grid, mem.bottom, kind, pred.h.values, pred.hu.values,
                        pred.hw.values, pred.time)
        want = v.max(axis=1) > k
        if enlarge:
            want = P.enlarge_flags(want)
        assert 0 < want.sum() < want.size
        assert np.array_equal(mask.flags, want), (name, kind)
        assert mask.ranges == P.contiguous_ranges(want)
        step = P.adaptive_step(st, dt, b, bcs, mode="adaptive", crit=crit, cfl_warn=False)
        assert np.array_equal(step.mask.flags, mask.flags)
        h, hu = pred.h.values, pred.hu.values
        assert P.max_wavespeed(pred) == float(np.max(np.abs(hu / h) + np.sqrt(9.81 * h)))
