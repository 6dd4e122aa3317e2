"""LDG fluxes outside the alternating family (FluxCoefficients,
corrector.py:40-47, :205-231) on the GPU against the REAL reference's
outputs (tests/golden/flux.npz, tests/golden/make_flux_golden.py).

The alternating family (c12 = -1/2, c22 = 0) runs the condensed chain of the
throughput kernels; any other flux runs the m-node kernels' band solve per
range (pm_general_solve: the reference's band system, eliminated with partial
pivoting as dgbsv does), at P1 and at higher orders, through every
reference-named entry point that takes a flux."""

import os

import numpy as np
import pytest

import paper_2505_17025_b200 as P
from tests.harness import paper_cases
from tests.oracle_cases import GOLDEN
from tests.test_gpu_golden import pkg_case, rel

pytestmark = pytest.mark.gpu
F = np.load(os.path.join(GOLDEN, "flux.npz"))
FLUXES = {str(n): tuple(float(x) for x in v) for n, v in zip(F["fluxes"], F["flux_values"])}
CASES = [str(c) for c in F["cases"]]


def _close(a, b, tol, floor=1e-9):
    return np.abs(np.asarray(a) - b).max() <= tol * max(np.abs(b).max(), floor)


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("flux", list(FLUXES))
def test_solves_and_correction(flux, case):
    fx = P.FluxCoefficients(*FLUXES[flux])
    g, b, bcs, dt, st = pkg_case(case)
    key = f"{flux}/{case}/"
    pred = P.heun_step(st, dt, b, bcs, cfl_warn=False)
    co = P.assemble_coefficients(pred, b, dt)
    n = g.n_elements
    p, hu = P.ldg_solve(co, (3, n // 2), (0.2, -0.3), fx)
    assert _close(p, F[key + "ldg_p"], 1e-10) and _close(hu, F[key + "ldg_hu"], 1e-10)
    ranges = tuple(tuple(int(v) for v in r) for r in F[key + "ranges"])
    sol = P.solve_on_ranges(pred, co, ranges, bcs, fx)
    ref = F[key + "sor"]
    assert _close(sol.p_nh.values, ref[0], 1e-10) and _close(sol.hu_corrected.values, ref[1], 1e-10)
    corr, sol2 = P.apply_correction(pred, b, dt, ranges, bcs, fx)
    ref = F[key + "corr"]
    print(flux, case, rel(corr.hu.values, ref[0]), rel(sol2.p_nh.values, ref[2]))
    assert _close(corr.hu.values, ref[0], 1e-10)
    assert _close(corr.hw.values, ref[1], 1e-9)
    assert _close(sol2.p_nh.values, ref[2], 1e-9)


@pytest.mark.parametrize("mode", ["global", "adaptive"])
@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("flux", list(FLUXES))
def test_trajectories(flux, case, mode):
    fx = P.FluxCoefficients(*FLUXES[flux])
    g, b, bcs, dt, st = pkg_case(case)
    crit = P.Criterion("eta_over_d", 1e-3, True) if mode == "adaptive" else None
    counts, pn = [], None
    for _ in range(12):
        r = P.adaptive_step(st, dt, b, bcs, mode=mode, crit=crit, flux=fx, cfl_warn=False)
        st = r.state
        counts.append(int(r.mask.flags.sum()))
        pn = r.p_nh
    key = f"{flux}/{case}/{mode}"
    assert counts == list(F[key + "_counts"])
    ref = F[key]
    assert rel(st.h.values, ref[0]) < 1e-12
    assert _close(st.hu.values, ref[1], 1e-10, 1e-6) and _close(st.hw.values, ref[2], 1e-9, 1e-6)
    if key + "_p" in F.files and pn is not None:
        assert _close(pn.values, F[key + "_p"], 1e-9)


@pytest.mark.parametrize("flux", list(FLUXES))
def test_ensemble_loop_equals_single_steps(flux):
    """Ensemble.advance with a general flux (one launch sequence, the m-node
    kernels on P1 members) equals the reference's 12 single steps."""
    fx = P.FluxCoefficients(*FLUXES[flux])
    from paper_2505_17025_b200 import _device as D
    for case in CASES[:3]:
        g, b, bcs, dt, st = pkg_case(case)
        rec = D.member_record(g, b, bcs, dt)
        ens = P.Ensemble.from_host(rec, st.h.values[None], st.hu.values[None], st.hw.values[None])
        ens.advance(12, "global", None, fx)
        ens.check()
        ref = F[f"{flux}/{case}/global"]
        assert rel(ens.h[0].cpu().numpy(), ref[0]) < 1e-12
        assert _close(ens.hu[0].cpu().numpy(), ref[1], 1e-10, 1e-6)
        assert _close(ens.hw[0].cpu().numpy(), ref[2], 1e-9, 1e-6)


@pytest.mark.parametrize("flux", list(FLUXES))
def test_simulate_solitary(flux):
    fx = P.FluxCoefficients(*FLUXES[flux])
    spec, init = paper_cases.build_scenario("solitary")
    spec = P.ScenarioSpec(spec.name, spec.grid, spec.dt, 60 * spec.dt, spec.bathymetry, spec.bcs,
                          spec.gauges, spec.g)
    res = P.simulate(spec, init, "adaptive", P.Criterion("eta_over_d"), flux=fx)
    ref = F[f"{flux}/simulate"]
    fs = res.final_state
    assert rel(fs.h.values, ref[0]) < 1e-11
    assert _close(fs.hu.values, ref[1], 1e-10) and _close(fs.hw.values, ref[2], 1e-9)
    assert abs(res.mask_fraction_mean - float(F[f"{flux}/simulate_frac"])) < 1e-12
    ge = F[f"{flux}/simulate_gauges"]
    assert res.gauge_eta.shape == ge.shape
    if ge.size:
        assert _close(res.gauge_eta, ge, 1e-10)


@pytest.mark.parametrize("flux", list(FLUXES))
def test_order_two(flux):
    fx = P.FluxCoefficients(*FLUXES[flux])
    g = P.GridSpec(0.0, 100.0, 40, poly_order=2)
    b = P.FlatBottom(10.0)
    bcs = P.BoundaryPair(P.WALL, P.ABSORBING)
    s0, pr = F[f"{flux}/p2/state0"], F[f"{flux}/p2/pred"]
    pred = P.FlowState(P.NodalField(g, pr[0]), P.NodalField(g, pr[1]), P.NodalField(g, pr[2]), 0.05)
    corr, sol = P.apply_correction(pred, b, 0.05, ((1, 12), (13, 20), (30, 39)), bcs, fx)
    ref = F[f"{flux}/p2/corr"]
    assert _close(corr.hu.values, ref[0], 1e-10) and _close(corr.hw.values, ref[1], 1e-9)
    assert _close(sol.p_nh.values, ref[2], 1e-9)
    st = P.FlowState(P.NodalField(g, s0[0]), P.NodalField(g, s0[1]), P.NodalField(g, s0[2]), 0.0)
    for _ in range(10):
        st = P.adaptive_step(st, 0.05, b, bcs, mode="global", flux=fx, cfl_warn=False).state
    ref = F[f"{flux}/p2/global"]
    assert rel(st.h.values, ref[0]) < 1e-12
    assert _close(st.hu.values, ref[1], 1e-10) and _close(st.hw.values, ref[2], 1e-9)
