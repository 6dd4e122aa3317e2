"""Orders p > 1 on the host side (no GPU): the package's GridSpec builds the
reference's m-node operators bit for bit (tests/golden/pm.npz, from the
reference GridSpec, grid.py:71-114), and the nh_pm_member record carries them
in the C layout."""

import os

import numpy as np
import pytest

import paper_2505_17025_b200 as P
from paper_2505_17025_b200 import _device as D, _lib

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "pm.npz"))
FIELDS = ("ref_nodes", "nodes", "sample_nodes", "mass", "stiffness", "deriv_ref", "weak_div",
          "lift_left", "lift_right")


@pytest.mark.parametrize("p", [1, 2, 3])
def test_grid_operators_bitwise_equal_to_reference(p):
    g = P.GridSpec(0.0, 30.0, 48, p)
    for f in FIELDS:
        assert np.array_equal(np.asarray(getattr(g, f)), GOLD[f"grid_p{p}_{f}"]), f


@pytest.mark.parametrize("p", [1, 2, 3])
def test_pm_record_layout(p):
    g = P.GridSpec(0.0, 30.0, 48, p)
    m = p + 1
    r = D.pm_record(g)[0]
    assert r.dtype == _lib.PM_DTYPE and _lib.PM_DTYPE.itemsize == 608
    for f in ("weak_div", "mass", "stiffness", "deriv_ref"):
        assert np.array_equal(r[f][:m * m].reshape(m, m), getattr(g, f))
        assert not r[f][m * m:].any()
    assert np.array_equal(r["lift_left"][:m], g.lift_left)
    # node j = (x_left + dx e) + node_off[j] reproduces GridSpec.nodes exactly
    e = np.arange(g.n_elements)[:, None]
    x = (g.x_left + g.dx * e) + r["node_off"][None, :m]
    assert np.array_equal(x, g.nodes)


def test_p4_and_p1_only_entry_points_rejected():
    with pytest.raises(NotImplementedError):
        D.pm_record(P.GridSpec(0.0, 1.0, 8, 4))
    with pytest.raises(NotImplementedError):
        D.member_record(P.GridSpec(0.0, 1.0, 8, 2), P.FlatBottom(1.0), None, 0.1)
    rec = D.member_record(P.GridSpec(0.0, 1.0, 8, 2), P.FlatBottom(1.0), None, 0.1,
                          any_order=True)
    assert not rec["weak_div"].any() and rec["dx"][0] == 0.125
