"""CPU-side checks of the drop-in boundary: the C-ABI library loads and exports
every function include/nhswe_b200.h declares; host packing / decoding logic."""

import ctypes
import os
import re
import sys

import numpy as np
import pytest
from hypothesis import given, strategies as st

import paper_2505_17025_b200 as P
from paper_2505_17025_b200 import _device as D
from paper_2505_17025_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "nhswe_b200.h")


def header_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return set(re.findall(r"^\s*(?:int|size_t|long long|const char\*|void)\s+\**(nh_\w+)\s*\(", txt, flags=re.M))


def test_header_declares_the_exports():
    assert header_functions() == set(_lib.EXPORTS)


def test_library_loads_and_exports_every_symbol():
    lib = _lib.load()
    for name in header_functions():
        assert getattr(lib, name) is not None
    assert lib.nh_abi_version() == _lib.ABI_VERSION == 5


def test_plan_host_logic():
    p = _lib.plan(4096, 4096)
    assert p["cluster"] * p["tile"] >= 4096 and p["threads"] % 32 == 0
    assert p["cluster"] <= 16
    assert _lib.plan(16384, 65536)["cluster"] <= 16
    small = _lib.plan(2000, 1)
    assert small["cluster"] > 1            # single members spread over a cluster
    with pytest.raises(ValueError):
        _lib.plan(1, 1)


def test_struct_layouts():
    assert _lib.MEMBER_DTYPE.itemsize == 312
    assert _lib.STATUS_DTYPE.itemsize == 72
    assert ctypes.sizeof(_lib.Scheme) == 72
    assert ctypes.sizeof(_lib.Outputs) == 48


def test_member_record_copies_reference_constants():
    g = P.GridSpec(0.0, 200.0, 2000)
    r = D.member_record(g, P.FlatBottom(1.0), P.BoundaryPair(P.WALL, P.ABSORBING), 0.01)
    assert r["dx"][0] == g.dx and r["eps"][0] == 1e-9 * g.dx
    assert np.array_equal(r["weak_div"][0], g.weak_div.ravel())
    assert np.array_equal(r["mass"][0], g.mass.ravel())
    assert r["bc_left"][0] == _lib.BC_WALL and r["bc_right"][0] == _lib.BC_ABSORBING
    with pytest.raises(NotImplementedError):
        D.member_record(P.GridSpec(0.0, 1.0, 4, poly_order=2), P.FlatBottom(1.0), None, 0.1)


@given(st.lists(st.booleans(), min_size=1, max_size=200))
def test_flag_bits_roundtrip(bits):
    f = np.array(bits, dtype=bool)
    w = D.flags_to_bits(f[None])
    assert w.dtype == np.uint32 and w.shape == (1, (len(bits) + 31) // 32)
    assert np.array_equal(D.bits_to_flags(w, len(bits))[0], f)
    for e in np.flatnonzero(f):
        assert (int(w[0, e >> 5]) >> (e & 31)) & 1


@given(st.lists(st.booleans(), min_size=0, max_size=80))
def test_contiguous_ranges_roundtrip(bits):
    f = np.array(bits, dtype=bool)
    rebuilt = np.zeros_like(f)
    for e0, e1 in P.contiguous_ranges(f):
        assert e0 <= e1
        rebuilt[e0:e1 + 1] = True
    assert np.array_equal(rebuilt, f)


def test_error_key_decoding_and_exception_mapping():
    key = (7 << 34) | (_lib.ERR_POSITIVITY_ENTRY << 30) | (12 + 1)
    assert D.decode_error(key) == (7, _lib.ERR_POSITIVITY_ENTRY, 12)
    assert D.decode_error(0xFFFFFFFFFFFFFFFF) is None
    st_ = np.zeros(1, dtype=_lib.STATUS_DTYPE)
    st_["error_key"] = key
    with pytest.raises(P.PositivityError) as ei:
        D.raise_for_status(st_, 0.0, 0.1)
    assert ei.value.element == 12
    t = 0.0
    for _ in range(7):
        t += 0.1
    assert ei.value.time == t
    st_["error_key"] = (3 << 34) | (_lib.ERR_POSITIVITY_STAGE2 << 30)
    with pytest.raises(P.PositivityError) as ei:
        D.raise_for_status(st_, 0.0, 0.1)
    assert ei.value.element == -1
    st_["error_key"] = (0 << 34) | (_lib.ERR_SOLVE_NONFINITE << 30) | 5
    with pytest.raises(P.EllipticSolveError):
        D.raise_for_status(st_, 0.0, 0.1)


def test_api_validation_without_gpu():
    g = P.GridSpec(0.0, 10.0, 10)
    d = np.ones((10, 2))
    s = P.FlowState(P.NodalField(g, d), P.NodalField(g, 0 * d), P.NodalField(g, 0 * d), 0.0)
    bcs = P.BoundaryPair(P.WALL, P.WALL)
    with pytest.raises(ValueError):
        P.adaptive_step(s, 0.01, P.FlatBottom(1.0), bcs, mode="magic")
    with pytest.raises(ValueError):
        P.adaptive_step(s, 0.01, P.FlatBottom(1.0), bcs, mode="adaptive")
    with pytest.raises(ValueError):
        P.heun_step(s, -1.0, P.FlatBottom(1.0), bcs)
    with pytest.raises(ValueError):
        P.Criterion("vorticity")
    with pytest.raises(ValueError):
        P.BoundaryCondition("periodic")


def test_gpu_entry_points_fail_loudly_without_cuda():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    g = P.GridSpec(0.0, 10.0, 10)
    d = np.ones((10, 2))
    s = P.FlowState(P.NodalField(g, d), P.NodalField(g, 0 * d), P.NodalField(g, 0 * d), 0.0)
    with pytest.raises(RuntimeError, match="no CUDA device"):
        P.heun_step(s, 0.01, P.FlatBottom(1.0), P.BoundaryPair(P.WALL, P.WALL))


def test_grid_constants_match_reference_fixture():
    from tests.oracle_cases import load_short
    d = load_short()
    xl, xr, n = d["plate/grid"]
    g = P.GridSpec(float(xl), float(xr), int(n))
    for k in ("mass", "mass_inv", "stiffness", "deriv_ref", "weak_div", "lift_left",
              "lift_right", "sample_nodes"):
        assert np.array_equal(getattr(g, k), d["plate/grid_" + k]), k
