"""Edge cases of the streaming path (the default for every run) against the
oracle: member sizes at the tile boundaries (one-element last tile, a member
smaller than one tile, the minimum N = 2), isolated single-element ranges,
ranges touching both domain ends, and the error records (positivity with the
member, element and step of the reference's exception)."""

import numpy as np
import pytest

import paper_2505_17025_b200 as P
from paper_2505_17025_b200 import _device as D
from oracle import nhswe_oracle as O
from tests.helpers import oracle_member, rel

pytestmark = pytest.mark.gpu

OWN = 120   # elements per streaming tile (csrc/stream_kernels.cuh)


def bump_state(grid, a, x0, w, d0=1.0):
    x = grid.nodes
    eta = a / np.cosh((x - x0) / w) ** 2
    h = d0 + eta
    hu = h * np.sqrt(9.81 / d0) * eta
    return h, hu, np.zeros_like(h)


@pytest.mark.parametrize("n", [2, 3, 7, OWN - 1, OWN, OWN + 1, 2 * OWN + 1, 3 * OWN - 1])
@pytest.mark.parametrize("mode", ["adaptive", "global"])
def test_member_sizes_at_tile_boundaries(n, mode):
    """Two members of n elements (different widths, dt and boundary kinds)
    stepped on the streaming path equal the oracle."""
    L = [10.0, 7.0]
    bcs = [P.BoundaryPair(P.WALL, P.ABSORBING), P.BoundaryPair(P.ABSORBING, P.WALL)]
    grids = [P.GridSpec(0.0, l, n) for l in L]
    dts = [0.05 * grids[0].dx, 0.04 * grids[1].dx]
    recs = np.concatenate([D.member_record(g, P.FlatBottom(1.0), b, dt)
                           for g, b, dt in zip(grids, bcs, dts)])
    st = [bump_state(g, 0.2, 0.4 * g.x_right, 0.8) for g in grids]
    H, Q, W = (np.stack([s[k] for s in st]) for k in range(3))
    steps = 40
    crit = P.Criterion("eta_over_d", 1e-3, True) if mode == "adaptive" else None
    ens = P.Ensemble.from_host(recs, H, Q, W)
    assert ens.choose_path(mode, crit) == "stream"
    ens.advance(steps, mode, crit)
    stt = ens.check()
    for i in range(2):
        o = O.run(oracle_member(grids[i], P.FlatBottom(1.0), bcs[i], dts[i]), H[i], Q[i], W[i],
                  steps, mode=mode, enlarge=True)
        assert rel(ens.h[i].cpu().numpy() - 1.0, o.h - 1.0) <= 1e-9, (n, i)
        assert rel(ens.hu[i].cpu().numpy(), o.hu) <= 1e-9, (n, i)
        assert np.abs(ens.hw[i].cpu().numpy() - o.hw).max() <= 1e-9 * max(np.abs(o.hw).max(),
                                                                            1e-12)
        assert stt["flagged"][i] == round(o.fraction_mean * steps * n), (n, i)


def test_isolated_and_end_touching_ranges():
    """Bumps at both walls and one narrow bump in the middle: single-element and
    domain-end ranges in the same member, checked step by step (flags and
    state) against the oracle."""
    n = 2 * OWN + 17
    grid = P.GridSpec(0.0, 50.0, n)
    x = grid.nodes
    eta = (0.05 / np.cosh(x / 1.0) ** 2 + 0.05 / np.cosh((x - 50.0) / 1.0) ** 2
           + 2.2e-3 / np.cosh((x - 25.1) / 0.12) ** 2)
    h = 1.0 + eta
    hu = np.zeros_like(h)
    hw = np.zeros_like(h)
    bcs = P.BoundaryPair(P.WALL, P.WALL)
    dt = 0.05 * grid.dx
    rec = D.member_record(grid, P.FlatBottom(1.0), bcs, dt)
    mem = oracle_member(grid, P.FlatBottom(1.0), bcs, dt)
    T = D.torch()
    steps = 12
    ens = P.Ensemble.from_host(rec, h[None], hu[None], hw[None])
    bits = T.zeros((steps, 1, (n + 31) // 32), dtype=T.int32, device="cuda")
    ens.advance(steps, "adaptive", P.Criterion("eta_over_d"), flag_bits=bits)
    ens.check()
    flags = D.bits_to_flags(bits.cpu().numpy().view(np.uint32)[:, 0], n)
    oh, oq, ow, t = h, hu, hw, 0.0
    for s in range(steps):
        o = O.step(mem, oh, oq, ow, t, "adaptive", "eta_over_d", 1e-3, False, cfl_warn=False)
        assert np.array_equal(flags[s], o.flags), s
        oh, oq, ow, t = o.h, o.hu, o.hw, t + dt
    runs = P.contiguous_ranges(flags[0])
    assert runs[0][0] == 0 and runs[-1][1] == n - 1
    assert any(a == b for a, b in runs) or any(b - a < 3 for a, b in runs)
    assert rel(ens.h[0].cpu().numpy() - 1.0, oh - 1.0) <= 1e-9
    assert rel(ens.hu[0].cpu().numpy(), oq) <= 1e-9


def test_stream_positivity_error_names_member_element_step():
    """A member that dries at entry raises PositivityError(element, t) for that
    member (hydrostatic.py:101-103) on the streaming path; the others are
    unaffected."""
    n = 300
    grid = P.GridSpec(0.0, 10.0, n)
    dt = 0.05 * grid.dx
    bcs = P.BoundaryPair(P.WALL, P.WALL)
    recs = np.concatenate([D.member_record(grid, P.FlatBottom(1.0), bcs, dt)] * 3)
    H = np.ones((3, n, 2))
    H[1, 187, 1] = -1e-3   # member 1, element 187 dry at entry
    Z = np.zeros_like(H)
    ens = P.Ensemble.from_host(recs, H, Z, Z)
    ens.advance(5, "adaptive", P.Criterion("eta_over_d"))
    st = D.read_status(ens.status)
    err = D.decode_error(st["error_key"][1])
    assert err == (0, 1, 187)   # step 0, code POSITIVITY_ENTRY, element 187
    assert D.decode_error(st["error_key"][0]) is None and D.decode_error(st["error_key"][2]) is None
    with pytest.raises(P.PositivityError) as ei:
        ens.check()
    assert ei.value.element == 187


def test_members_longer_than_the_kernel_caps():
    """The reference has no size limit.  A member longer than the streaming
    path chains (32 x 8 tiles of 120 elements) and than the resident cluster
    kernel holds runs the m-node kernels instead (driver.STREAM_MAX_ELEMENTS,
    hydrostatic.RESIDENT_MAX_ELEMENTS): same results as the oracle, through
    the ensemble loop and through the single-step API."""
    from paper_2505_17025_b200.driver import STREAM_MAX_ELEMENTS
    n = STREAM_MAX_ELEMENTS + 1000
    grid = P.GridSpec(0.0, 400.0, n)
    bcs = P.BoundaryPair(P.WALL, P.ABSORBING)
    dt = 0.05 * grid.dx
    h, hu, hw = bump_state(grid, 0.2, 150.0, 6.0)
    crit = P.Criterion("eta_over_d", 1e-3, True)
    steps = 4
    ens = P.Ensemble.from_host(D.member_record(grid, P.FlatBottom(1.0), bcs, dt), h[None],
                               hu[None], hw[None])
    assert ens.choose_path("adaptive", crit) == "generic"
    ens.advance(steps, "adaptive", crit)
    stt = ens.check()
    o = O.run(oracle_member(grid, P.FlatBottom(1.0), bcs, dt), h, hu, hw, steps, enlarge=True)
    assert rel(ens.h[0].cpu().numpy() - 1.0, o.h - 1.0) <= 1e-9
    assert rel(ens.hu[0].cpu().numpy(), o.hu) <= 1e-9
    assert stt["flagged"][0] == round(o.fraction_mean * steps * n) > 0
    st = P.FlowState(P.NodalField(grid, h), P.NodalField(grid, hu), P.NodalField(grid, hw), 0.0)
    r = P.adaptive_step(st, dt, P.FlatBottom(1.0), bcs, mode="adaptive", crit=crit, cfl_warn=False)
    o1 = O.step(oracle_member(grid, P.FlatBottom(1.0), bcs, dt), h, hu, hw, 0.0, "adaptive",
                "eta_over_d", 1e-3, True)
    assert np.array_equal(r.mask.flags, o1.flags)
    assert rel(r.state.hu.values, o1.hu) <= 1e-12


def test_criterion_at_the_threshold():
    """K_P decides |eta / d| > k_nh without the division wherever the product
    comparison is certain and divides only inside a 2^-49 band around the
    threshold.  Uniform members at rest keep h exactly (zero tendencies), so
    eta / d is controlled to the bit: exactly k_nh (inside the band; not
    flagged, the comparison is strict) and one ulp of h to either side."""
    k = 2.0 ** -10
    n = 130
    grid = P.GridSpec(0.0, 10.0, n)
    bcs = P.BoundaryPair(P.WALL, P.WALL)
    dt = 0.01 * grid.dx
    hs = [1.0 + k, np.nextafter(1.0 + k, 2.0), np.nextafter(1.0 + k, 0.0), 1.0 - k,
          np.nextafter(1.0 - k, 0.0), np.nextafter(1.0 - k, 2.0)]
    recs = np.concatenate([D.member_record(grid, P.FlatBottom(1.0), bcs, dt) for _ in hs])
    H = np.stack([np.full((n, 2), v) for v in hs])
    Z = np.zeros_like(H)
    crit = P.Criterion("eta_over_d", k, False)
    for path in ("stream", "resident"):
        ens = P.Ensemble.from_host(recs, H, Z, Z)
        ens.advance(1, "adaptive", crit, path=path)
        st = ens.check()
        want = []
        for v in hs:
            o = O.step(oracle_member(grid, P.FlatBottom(1.0), bcs, dt), np.full((n, 2), v),
                       Z[0], Z[0], 0.0, "adaptive", "eta_over_d", k, False)
            assert np.array_equal(o.h, np.full((n, 2), v))   # at rest: h exact
            want.append(int(o.flags.sum()))
        assert want == [0, n, 0, 0, n, 0], want
        assert list(st["flagged"]) == want, (path, list(st["flagged"]))
