"""Error semantics of the solve and touching ranges, against the REAL
reference's behaviour on the same inputs (tests/golden/errors.npz, made by
`make_golden.py --errors`):

* the residual gate (corrector.py:355-366): the reference passes at the
  default 1e-10 and raises EllipticSolveError at residual_tol = 1e-18; the
  device evaluates the same relative residual and does the same;
* a non-finite right-hand side raises EllipticSolveError in both;
* the structural asserts (corrector.py:70-74) raise AssertionError;
* touching ranges are separate systems (each with P* = 0 at its ends, the
  reference's block-diagonal batch): apply_correction / solve_on_ranges on
  ((2, n/4), (n/4+1, n/2), ...) match the reference;
* a flux outside the alternating family is solved, as in the reference, by
  the band solve of the m-node kernels, with the same residual gate.
"""

import os

import numpy as np
import pytest

import paper_2505_17025_b200 as P
from paper_2505_17025_b200 import _device as D
from tests.oracle_cases import GOLDEN
from tests.test_gpu_golden import pkg_case, rel

pytestmark = pytest.mark.gpu
E = np.load(os.path.join(GOLDEN, "errors.npz"))


def _coeffs(**kw):
    n = 48
    g = P.GridSpec(0.0, 1.0, n)
    s11, s12, s22, f1, f2 = (E["err/coef"][i].copy() for i in range(5))
    base = dict(s11=s11, s12=s12, s21=-s11, s22=s22, f1=f1, f2=f2)
    base.update(kw)
    z = np.zeros_like(s11)
    return P.EllipticCoefficients(g, base["s11"], base["s12"], base["s21"], base["s22"],
                                  base["f1"], base["f2"], z, P.BottomSample(*(z,) * 6), 0.1, 1.0)


def _outcome(fn):
    try:
        fn()
        return "ok"
    except Exception as exc:   # noqa: BLE001
        return type(exc).__name__


def test_residual_gate_matches_reference():
    co = _coeffs()
    assert _outcome(lambda: P.ldg_solve(co, (3, 40), (0.2, 0.3))) == str(E["err/tol_default"])
    assert _outcome(lambda: P.ldg_solve(co, (3, 40), (0.2, 0.3), residual_tol=1e-18)) == \
        str(E["err/tol_1e-18"]) == "EllipticSolveError"


def test_residual_is_recorded_and_small():
    """The device's relative residual of a solve (status.resid_max) is at
    rounding level, far under the reference's 1e-10 gate."""
    T = D.torch()
    cfgrid = P.GridSpec(0.0, 100.0, 300)
    from tests.helpers import smooth_state
    st = smooth_state(cfgrid)
    ens = P.Ensemble.from_host(D.member_record(cfgrid, P.FlatBottom(10.0),
                                               P.BoundaryPair(P.WALL, P.ABSORBING), 0.005),
                               st.h.values[None], st.hu.values[None], st.hw.values[None])
    ens.advance(5, "global", None)
    T.cuda.synchronize()
    s = ens.check()
    print("stream path resid_max", s["resid_max"][0])
    assert 0.0 < s["resid_max"][0] < 1e-13
    ens = P.Ensemble.from_host(D.member_record(cfgrid, P.FlatBottom(10.0),
                                               P.BoundaryPair(P.WALL, P.ABSORBING), 0.005),
                               st.h.values[None], st.hu.values[None], st.hw.values[None])
    ens.advance(5, "global", None, path="resident")
    s = ens.check()
    print("resident path resid_max", s["resid_max"][0])
    assert 0.0 < s["resid_max"][0] < 1e-13


def test_residual_gate_raises_in_a_step():
    """adaptive_step / Ensemble.advance honour the scheme's residual_tol: a
    tolerance under rounding level trips the gate on the first solve."""
    grid = P.GridSpec(0.0, 100.0, 300)
    from tests.helpers import smooth_state
    st = smooth_state(grid)
    rec = D.member_record(grid, P.FlatBottom(10.0), P.BoundaryPair(P.WALL, P.ABSORBING), 0.005)
    for path in ("stream", "resident"):
        ens = P.Ensemble.from_host(rec, st.h.values[None], st.hu.values[None],
                                   st.hw.values[None])
        sch = D.scheme(P.driver._MODES["global"], residual_tol=1e-30)
        if path == "stream":
            ws = D.stream_workspace(1, grid.n_elements)
            D.stream_advance(ens.members, ens.h, ens.hu, ens.hw, ens.time, 3, sch, ens.status, ws)
        else:
            D.advance(ens.members, ens.h, ens.hu, ens.hw, ens.time, 3, sch, ens.status)
        with pytest.raises(P.EllipticSolveError, match="residual"):
            ens.check()
        step, code, _ = D.decode_error(D.read_status(ens.status)["error_key"][0])
        assert step == 0 and code == 6


def test_nonfinite_solve_matches_reference():
    f1 = E["err/coef"][3].copy()
    f1[10, 1] = np.inf
    assert _outcome(lambda: P.ldg_solve(_coeffs(f1=f1), (3, 40))) == str(E["err/nonfinite"])


def test_structural_asserts_match_reference():
    s12 = E["err/coef"][1].copy()
    s12[7, 0] = -1.0
    assert _outcome(lambda: _coeffs(s12=s12)) == str(E["err/s12_negative"]) == "AssertionError"
    s11 = E["err/coef"][0]
    assert _outcome(lambda: _coeffs(s21=-s11 + 1e-3)) == str(E["err/s21_mismatch"])
    # the device re-checks s12 > 0 at every flagged node (a record that
    # slipped past the host check): NH_ERR_STRUCTURE -> AssertionError
    co = _coeffs()
    object.__setattr__(co, "s12", s12)
    with pytest.raises(AssertionError, match="s12"):
        P.ldg_solve(co, (3, 40))


def test_general_flux_is_solved_and_gated():
    """A flux outside the alternating family: the reference solves it, and so
    does the band solve of the m-node kernels (values: tests/test_gpu_flux.py),
    with the same residual gate."""
    assert str(E["err/flux_c12_0"]) == "ok"
    central = P.FluxCoefficients(0.5, 0.0, 0.0)
    assert _outcome(lambda: P.ldg_solve(_coeffs(), (3, 40), (0.2, 0.3), central)) == "ok"
    with pytest.raises(P.EllipticSolveError, match="residual"):
        P.ldg_solve(_coeffs(), (3, 40), (0.2, 0.3), central, residual_tol=1e-18)


@pytest.mark.parametrize("name", ["flat_walls", "flat_absorbing", "plate"])
def test_touching_ranges_are_separate_systems(name):
    g, b, bcs, dt, _ = pkg_case(name)
    key = "adj/" + name + "/"
    pr = E[key + "pred"]
    pred = P.FlowState(P.NodalField(g, pr[0]), P.NodalField(g, pr[1]), P.NodalField(g, pr[2]), dt)
    ranges = tuple(tuple(int(v) for v in r) for r in E[key + "ranges"])
    corr, sol = P.apply_correction(pred, b, dt, ranges, bcs)
    ref = E[key + "corr"]
    print(name, rel(corr.hu.values, ref[0]), rel(sol.p_nh.values, ref[2]))
    assert rel(corr.hu.values, ref[0]) < 1e-10
    assert np.abs(corr.hw.values - ref[1]).max() <= 1e-9 * max(np.abs(ref[1]).max(), 1e-9)
    assert np.abs(sol.p_nh.values - ref[2]).max() <= 1e-9 * max(np.abs(ref[2]).max(), 1e-9)
    co = P.assemble_coefficients(pred, b, dt)
    s2 = P.solve_on_ranges(pred, co, ranges, bcs)
    rs = E[key + "solve"]
    assert rel(s2.hu_corrected.values, rs[0]) < 1e-10
    assert np.abs(s2.p_nh.values - rs[1]).max() <= 1e-9 * max(np.abs(rs[1]).max(), 1e-9)
    if name != "plate":   # (the plate at t = 0 has pressure only near its edge)
        # one merged range is a different system: the split matters
        merged = P.solve_on_ranges(pred, co, ((ranges[0][0], ranges[1][1]),) + ranges[2:], bcs)
        assert rel(merged.p_nh.values, rs[1]) > 1e-6
