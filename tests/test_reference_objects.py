"""Drop-in with the reference's own objects: the mirrored API accepts nhswe's
GridSpec / FlowState / BathymetryModel / BoundaryPair / Criterion instances
(reference bathymetry.py:33-184, grid.py:63-196, hydrostatic.py:29-52,
adaptivity.py:27-44) as they are.  The reference package is imported from
baseline/_ref (or the mounted source); the tests skip where it is absent."""

import numpy as np
import pytest

import paper_2505_17025_b200 as P
from paper_2505_17025_b200 import _device as D
from paper_2505_17025_b200.bathymetry import device_model
from tests.harness.ref_bridge import import_reference

R, WHERE = import_reference()
needs_ref = pytest.mark.skipif(R is None, reason=str(WHERE))


def _pairs():
    mo = (1.5, 0.327, 0.218, 2.218, 2.436)
    return [(R.FlatBottom(10.0), P.FlatBottom(10.0)),
            (R.HammackPlate(0.05, 0.005, 0.6, 0.13), P.HammackPlate(0.05, 0.005, 0.6, 0.13)),
            (R.WhittakerSlide(0.175, 0.026, 0.5, R.SlideMotion(*mo), 5.0),
             P.WhittakerSlide(0.175, 0.026, 0.5, P.SlideMotion(*mo), 5.0))]


@needs_ref
def test_reference_bottoms_map_to_the_same_records():
    g = R.GridSpec(0.0, 20.0, 64)
    bcs = R.BoundaryPair(R.WALL, R.ABSORBING)
    for ref, own in _pairs():
        a = D.member_record(g, ref, bcs, 0.01)
        b = D.member_record(P.GridSpec(0.0, 20.0, 64), own, P.BoundaryPair(P.WALL, P.ABSORBING),
                            0.01)
        assert a.tobytes() == b.tobytes(), type(ref).__name__


@needs_ref
def test_unknown_model_is_a_type_error():
    from nhswe.bathymetry import BathymetryModel, BottomSample

    class Custom(BathymetryModel):
        def _sample(self, x, t):
            z = np.zeros_like(x)
            return BottomSample(z + 1.0, z, z, z, z, z)
    with pytest.raises(TypeError, match="no device evaluation"):
        device_model(Custom())


@needs_ref
@pytest.mark.gpu
@pytest.mark.parametrize("k", [0, 1, 2])
def test_adaptive_step_takes_reference_objects(k):
    """adaptive_step on the reference's own objects equals the same call on
    the package's objects, bit for bit."""
    ref, own = _pairs()[k]
    grid_r = R.GridSpec(0.0, 15.0 if k == 2 else 100.0, 120)
    grid_p = P.GridSpec(grid_r.x_left, grid_r.x_right, 120)
    d = own.sample(grid_p.sample_nodes, 0.0).d
    x = grid_p.nodes
    h = d + 0.01 * np.exp(-((x - x.mean()) / (0.1 * x.max())) ** 2)
    hu = 0.02 * h
    hw = np.zeros_like(h)
    st_r = R.FlowState(R.NodalField(grid_r, h), R.NodalField(grid_r, hu), R.NodalField(grid_r, hw),
                       0.0)
    st_p = P.FlowState(P.NodalField(grid_p, h), P.NodalField(grid_p, hu), P.NodalField(grid_p, hw),
                       0.0)
    dt = 0.2 * grid_p.dx / np.sqrt(9.81 * h.max())
    a = P.adaptive_step(st_r, dt, ref, R.BoundaryPair(R.WALL, R.ABSORBING), mode="adaptive",
                        crit=R.Criterion("eta_over_d", 1e-4, True), cfl_warn=False)
    b = P.adaptive_step(st_p, dt, own, P.BoundaryPair(P.WALL, P.ABSORBING), mode="adaptive",
                        crit=P.Criterion("eta_over_d", 1e-4, True), cfl_warn=False)
    for f in ("h", "hu", "hw"):
        assert np.array_equal(getattr(a.state, f).values, getattr(b.state, f).values), f
    assert np.array_equal(a.mask.flags, b.mask.flags)
