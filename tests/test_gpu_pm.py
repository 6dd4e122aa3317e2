"""Polynomial orders p = 2, 3 on the GPU (m-node kernels,
csrc/pm_kernels.cu) against the reference's own outputs
(tests/golden/pm.npz, tests/golden/make_pm_golden.py): rhs_operator and
criterion_values on the initial state, and short adaptive_step trajectories
in every mode (final state within 1e-9 relative, per-step flagged counts
equal).  At p = 1 the same kernels (path="generic") are checked against the
P1 streaming kernels on a config-4 style mixed ensemble."""

import json
import os

import numpy as np
import pytest

import paper_2505_17025_b200 as P
from tests.harness import paper_cases
from paper_2505_17025_b200 import _device as D, configs
from tests.helpers import oracle_depth, rel

pytestmark = pytest.mark.gpu

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "pm.npz"))
CASES = json.loads(str(GOLD["cases"]))
BCS = {"wall": P.WALL, "absorbing": P.ABSORBING}


def setup(name):
    s = json.loads(str(GOLD[f"{name}_spec"]))
    grid = P.GridSpec(s["xl"], s["xr"], s["n"], s["p"])
    bathy = (P.FlatBottom(s["h0"]) if s["bottom"] == "flat"
             else P.HammackPlate(s["h0"], s["zeta0"], s["b"], s["t_c"]))
    bcs = P.BoundaryPair(BCS[s["bcs"][0]], BCS[s["bcs"][1]])
    st = P.FlowState(P.NodalField(grid, GOLD[f"{name}_h0"]), P.NodalField(grid, GOLD[f"{name}_hu0"]),
                     P.NodalField(grid, GOLD[f"{name}_hw0"]), 0.0)
    crit = P.Criterion(s["kind"], s["k_nh"], s["enlarge"]) if s["mode"] == "adaptive" else None
    return s, grid, bathy, bcs, st, crit


@pytest.mark.parametrize("name", CASES)
def test_rhs_and_criterion_match_reference(name):
    s, grid, bathy, bcs, st, _ = setup(name)
    t = P.rhs_operator(st, bathy, bcs)
    ref = GOLD[f"{name}_rhs"]
    for f in range(3):
        scale = max(np.abs(ref[f]).max(), 1e-300)
        assert np.abs(t[f] - ref[f]).max() <= 1e-12 * scale, (name, f)
    for k, kind in enumerate(P.CRITERION_KINDS):
        v = P.criterion_values(st, bathy, kind)
        r = GOLD[f"{name}_crit"][k]
        assert np.abs(v - r).max() <= 1e-12 * max(np.abs(r).max(), 1e-300), (name, kind)
        # evaluate_criterion (nh_pm_criterion + nh_mask over m nodes): the
        # reference's thresholded, enlarged mask of its own values, at a
        # threshold away from every value
        vals = np.sort(np.abs(r).max(axis=1))
        if vals[-1] > 0.0:
            k_nh = 0.5 * (vals[len(vals) // 2] + vals[len(vals) // 2 + 1])
            if np.min(np.abs(np.abs(r).max(axis=1) - k_nh)) > 1e-9 * vals[-1]:
                for enl in (False, True):
                    want = r.max(axis=1) > k_nh
                    if enl:
                        want = P.enlarge_flags(want)
                    got = P.evaluate_criterion(st, bathy, P.Criterion(kind, k_nh, enl))
                    assert np.array_equal(got.flags, want), (name, kind, enl)


@pytest.mark.parametrize("name", CASES)
def test_trajectory_matches_reference(name):
    """One launch sequence for the whole run (Ensemble, m-node kernels), per-step
    flag bits recorded on the device."""
    s, grid, bathy, bcs, st, crit = setup(name)
    n = s["steps"]
    rec = D.member_record(grid, bathy, bcs, s["dt"], any_order=True)
    ens = P.Ensemble.from_host(rec, st.h.values[None], st.hu.values[None], st.hw.values[None],
                               [0.0], D.pm_record(grid))
    assert ens.choose_path(s["mode"], crit) == "generic"
    T = D.torch()
    nw = (grid.n_elements + 31) // 32
    bits = T.zeros((n, 1, nw), dtype=T.int32, device="cuda")
    p = T.zeros_like(ens.h)
    ens.advance(n, s["mode"], crit, flag_bits=bits, p_out=p)
    ens.check()
    flags = D.bits_to_flags(bits.cpu().numpy().view(np.uint32)[:, 0], grid.n_elements)
    assert flags.sum(axis=1).tolist() == GOLD[f"{name}_counts"].tolist(), name
    d = bathy.depth(grid.sample_nodes, float(GOLD[f"{name}_t"]))
    h, hu, hw = (x[0].cpu().numpy() for x in (ens.h, ens.hu, ens.hw))
    e_eta = rel(h - d, GOLD[f"{name}_h"] - d)
    e_hu = rel(hu, GOLD[f"{name}_hu"])
    e_hw = rel(hw, GOLD[f"{name}_hw"])
    print(f"{name}: p={s['p']} {n} steps, eta {e_eta:.1e} hu {e_hu:.1e} hw {e_hw:.1e}")
    assert e_eta <= 1e-9 and e_hu <= 1e-9 and e_hw <= 1e-9, name
    assert float(ens.time.item()) == float(GOLD[f"{name}_t"])
    if s["mode"] != "hydrostatic":
        assert rel(p[0].cpu().numpy(), GOLD[f"{name}_p"]) <= 1e-8, name


def test_adaptive_step_api_p2():
    """The reference-signature adaptive_step / heun_step route p > 1 to the
    m-node kernels: one step equals the first step of the reference run."""
    name = "p2_flat_adaptive"
    s, grid, bathy, bcs, st, crit = setup(name)
    r = P.adaptive_step(st, s["dt"], bathy, bcs, mode="adaptive", crit=crit)
    assert int(r.mask.flags.sum()) == int(GOLD[f"{name}_counts"][0])
    assert r.p_nh is not None and r.p_nh.values.shape == (grid.n_elements, 3)
    h = P.heun_step(st, s["dt"], bathy, bcs)
    assert h.h.values.shape == (grid.n_elements, 3) and h.time == s["dt"]


@pytest.mark.parametrize("mode,kind,enlarge", [("adaptive", "eta_over_d", False),
                                               ("adaptive", "u_x", True),
                                               ("global", "eta_over_d", False)])
def test_generic_kernels_at_p1_match_stream_path(mode, kind, enlarge):
    """m = 2 through the m-node kernels equals the P1 streaming kernels
    (mixed solitary / box-uplift ensemble, per-member dx and dt)."""
    cfg = configs.Config4(n_members=6, n_elements=512, n_steps=80)
    recs = cfg.records()
    pm = np.concatenate([D.pm_record(cfg.member(i).grid) for i in range(cfg.n_members)])
    states = [cfg.host_state(i, oracle_depth) for i in range(cfg.n_members)]
    H, Q, W = (np.stack([x[k] for x in states]) for k in range(3))
    crit = P.Criterion(kind, 1e-3, enlarge) if mode == "adaptive" else None
    out = {}
    for path in ("stream", "generic"):
        ens = P.Ensemble.from_host(recs, H, Q, W, None, pm)
        ens.advance(cfg.n_steps, mode, crit, path=path)
        st = ens.check()
        out[path] = ([x.cpu().numpy() for x in (ens.h, ens.hu, ens.hw)], st["flagged"].copy())
    (gh, gq, gw), gf = out["generic"]
    (sh, sq, sw), sf = out["stream"]
    assert np.array_equal(gf, sf)
    for i in range(cfg.n_members):
        h0 = cfg.member(i).bathymetry.h0
        assert rel(gh[i] - h0, sh[i] - h0) <= 1e-9, i
        assert rel(gq[i], sq[i]) <= 1e-9, i
        assert np.abs(gw[i] - sw[i]).max() <= 1e-9 * max(np.abs(sw[i]).max(), 1e-12), i


@pytest.mark.parametrize("name", json.loads(str(GOLD["sims"])))
def test_simulate_paper_scenarios_high_order(name):
    """simulate() of the paper scenarios at p = 2, 3 (gauges recorded on the
    device at flat node index e*m + j) against the reference's simulate()."""
    from dataclasses import replace
    c = json.loads(str(GOLD[f"{name}_cfg"]))
    spec, init = paper_cases.build_scenario(c["scenario"], **c["over"])
    spec = replace(spec, gauges=tuple(c["gauges"]))
    crit = P.Criterion(c["kind"], 1e-3, c["enlarge"]) if c["mode"] == "adaptive" else None
    r = P.simulate(spec, init, c["mode"], crit)
    d = spec.bathymetry.depth(spec.grid.sample_nodes, r.final_state.time)
    e_eta = rel(r.final_state.h.values - d, GOLD[f"{name}_h"] - d)
    e_hu = rel(r.final_state.hu.values, GOLD[f"{name}_hu"])
    e_g = rel(r.gauge_eta, GOLD[f"{name}_gauge_eta"])
    print(f"{name}: {spec.n_steps} steps, eta {e_eta:.1e} hu {e_hu:.1e} gauges {e_g:.1e}, "
          f"mask fraction {r.mask_fraction_mean:.4f} (reference {float(GOLD[f'{name}_frac']):.4f})")
    assert e_eta <= 1e-9 and e_hu <= 1e-9 and e_g <= 1e-9
    assert np.array_equal(r.gauge_times, GOLD[f"{name}_gauge_t"])
    assert abs(r.mask_fraction_mean - float(GOLD[f"{name}_frac"])) <= 1e-12


@pytest.mark.parametrize("name", ["p2_flat_adaptive", "p3_plate_global"])
def test_apply_correction_given_ranges_high_order(name):
    """apply_correction (corrector.py:485-498) on given ranges at p = 2, 3, the
    final state of the reference run as the predictor."""
    s, grid, bathy, bcs, _, _ = setup(name)
    t = float(GOLD[f"{name}_t"])
    pred = P.FlowState(P.NodalField(grid, GOLD[f"{name}_h"]), P.NodalField(grid, GOLD[f"{name}_hu"]),
                       P.NodalField(grid, GOLD[f"{name}_hw"]), t)
    ranges = [tuple(r) for r in GOLD[f"{name}_corr_ranges"].tolist()]
    st, sol = P.apply_correction(pred, bathy, s["dt"], ranges, bcs)
    assert st.h is pred.h and st.time == t
    assert rel(st.hu.values, GOLD[f"{name}_corr_hu"]) <= 1e-10
    assert rel(st.hw.values, GOLD[f"{name}_corr_hw"]) <= 1e-10
    assert rel(sol.p_nh.values, GOLD[f"{name}_corr_p"]) <= 1e-10


@pytest.mark.parametrize("name", ["p2_flat_adaptive", "p3_plate_global"])
def test_coefficient_level_functions_high_order(name):
    """assemble_coefficients (full grid and a window), ldg_solve on one range
    with an outer trace, solve_on_ranges and correct_momentum at p = 2, 3
    against the reference's (corrector.py:100-482)."""
    s, grid, bathy, bcs, _, _ = setup(name)
    pred = P.FlowState(P.NodalField(grid, GOLD[f"{name}_h"]), P.NodalField(grid, GOLD[f"{name}_hu"]),
                       P.NodalField(grid, GOLD[f"{name}_hw"]), float(GOLD[f"{name}_t"]))
    ranges = [tuple(r) for r in GOLD[f"{name}_corr_ranges"].tolist()]
    co = P.assemble_coefficients(pred, bathy, s["dt"])
    for k, f in enumerate(("s11", "s12", "s22", "f1", "f2", "phi")):
        ref = GOLD[f"{name}_coef"][k]
        assert np.abs(getattr(co, f) - ref).max() <= 1e-12 * max(np.abs(ref).max(), 1e-300), f
    lo, hi = ranges[0][0], ranges[-1][1]
    cw = P.assemble_coefficients(pred, bathy, s["dt"], window=slice(lo, hi + 1))
    assert cw.offset == lo and cw.s11.shape == GOLD[f"{name}_coefw"][0].shape
    p, hu = P.ldg_solve(co, ranges[0], outer_hu=(0.0, 0.37))
    assert rel(p, GOLD[f"{name}_ldg_p"]) <= 1e-10 and rel(hu, GOLD[f"{name}_ldg_hu"]) <= 1e-10
    sol = P.solve_on_ranges(pred, co, ranges, bcs)
    assert rel(sol.p_nh.values, GOLD[f"{name}_sor_p"]) <= 1e-10
    assert rel(sol.hu_corrected.values, GOLD[f"{name}_sor_hu"]) <= 1e-10
    cm = P.correct_momentum(pred, sol, co)
    assert cm.h is pred.h
    assert rel(cm.hw.values, GOLD[f"{name}_cm_hw"]) <= 1e-10
