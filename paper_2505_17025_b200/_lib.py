"""ctypes binding of the C ABI (include/nhswe_b200.h).

The shared library is built in-tree by ``paper_2505_17025_b200.build``.  There
is no CPU fallback: if the library or a CUDA device is missing, every entry
point raises.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NH_LIB") or os.path.join(_HERE, "_lib", "libnhswe_b200.so")

# ---- constants mirrored from the header
BOTTOM_FLAT, BOTTOM_PLATE, BOTTOM_QUARTIC_SLIDE, BOTTOM_SMOOTH_BOX, BOTTOM_SLOPE_SLIDE = range(5)
BC_ABSORBING, BC_WALL = 0, 1
MODE_HYDROSTATIC, MODE_GLOBAL, MODE_ADAPTIVE, MODE_CORRECT_GIVEN = range(4)
CRIT = {"eta_over_d": 0, "eta_x": 1, "u": 2, "u_x": 3, "w": 4, "w_x": 5}
ERR_POSITIVITY_ENTRY, ERR_POSITIVITY_STAGE1, ERR_POSITIVITY_STAGE2 = 1, 2, 3
ERR_SOLVE_NONFINITE, ERR_SOLVE_PIVOT, ERR_SOLVE_RESIDUAL, ERR_STRUCTURE = 4, 5, 6, 7
E_ARG, E_CUDA, E_UNSUPPORTED = -1, -2, -3
STATUS_OK_KEY = np.uint64(0xFFFFFFFFFFFFFFFF)

# numpy mirrors of the C structs (packed tables are uploaded as raw bytes)
MEMBER_DTYPE = np.dtype([
    ("x_left", "f8"), ("dx", "f8"), ("dt", "f8"), ("eps", "f8"), ("two_over_dx", "f8"),
    ("weak_div", "f8", (4,)), ("lift_left", "f8", (2,)), ("lift_right", "f8", (2,)),
    ("mass", "f8", (4,)), ("stiffness", "f8", (4,)), ("deriv_ref", "f8", (4,)),
    ("bottom", "f8", (12,)),
    ("bc_left", "i4"), ("bc_right", "i4"), ("bottom_kind", "i4"), ("reserved", "i4"),
])
STATUS_DTYPE = np.dtype([("error_key", "u8"), ("cfl_max", "f8"), ("flagged", "i8"),
                         ("steps_done", "i4"), ("any_hw", "i4"), ("resid_max", "f8"),
                         ("resid_acc", "f8", (4,))])
PM_DTYPE = np.dtype([   # nh_pm_member: m-node operators, m <= 4 (row-major, leading dim m)
    ("weak_div", "f8", (16,)), ("lift_left", "f8", (4,)), ("lift_right", "f8", (4,)),
    ("mass", "f8", (16,)), ("stiffness", "f8", (16,)), ("deriv_ref", "f8", (16,)),
    ("node_off", "f8", (4,)),
])
PM_MAX_NODES = 4
assert MEMBER_DTYPE.itemsize == 312 and STATUS_DTYPE.itemsize == 72 and PM_DTYPE.itemsize == 608


class Scheme(ctypes.Structure):
    _fields_ = [("g", ctypes.c_double), ("rho", ctypes.c_double), ("k_nh", ctypes.c_double),
                ("c11", ctypes.c_double), ("c12", ctypes.c_double), ("c22", ctypes.c_double),
                ("mode", ctypes.c_int32), ("criterion", ctypes.c_int32),
                ("enlarge", ctypes.c_int32), ("record_cfl", ctypes.c_int32),
                ("residual_tol", ctypes.c_double)]


class Outputs(ctypes.Structure):
    _fields_ = [("flag_bits", ctypes.c_void_p), ("p_nh", ctypes.c_void_p),
                ("given_flags", ctypes.c_void_p), ("gauge_nodes", ctypes.c_void_p),
                ("gauge_h", ctypes.c_void_p), ("n_gauges", ctypes.c_int32)]


ABI_VERSION = 5   # include/nhswe_b200.h NH_ABI_VERSION

EXPORTS = ("nh_abi_version", "nh_advance", "nh_stream_advance", "nh_stream_workspace_bytes",
           "nh_rhs", "nh_criterion", "nh_mask", "nh_max_wavespeed", "nh_coefficients",
           "nh_ldg_solve", "nh_correct_momentum", "nh_bottom_sample", "nh_plan",
           "nh_last_cuda_error", "nh_stream_graphs", "nh_stream_timing", "nh_stream_kernel_times",
           "nh_launch_count",
           "nh_selftest_arith", "nh_pm_workspace_bytes", "nh_pm_advance", "nh_pm_rhs",
           "nh_pm_criterion", "nh_pm_coefficients", "nh_pm_ldg_solve", "nh_pm_correct_momentum")

_P = ctypes.c_void_p
_I = ctypes.c_int
_D = ctypes.c_double
_SIGS = {
    "nh_abi_version": ([], _I),
    "nh_advance": ([_P, _I, _I, _P, _P, _P, _P, _I, ctypes.POINTER(Scheme),
                    ctypes.POINTER(Outputs), _P, _P], _I),
    "nh_stream_advance": ([_P, _I, _I, _P, _P, _P, _P, _I, ctypes.POINTER(Scheme),
                           ctypes.POINTER(Outputs), _P, _P, ctypes.c_size_t, _P], _I),
    "nh_stream_workspace_bytes": ([_I, _I], ctypes.c_size_t),
    "nh_stream_graphs": ([_I], _I),
    "nh_stream_timing": ([_I], _I),
    "nh_stream_kernel_times": ([_P, _P], _I),
    "nh_launch_count": ([], ctypes.c_longlong),
    "nh_selftest_arith": ([ctypes.c_longlong, ctypes.c_ulonglong, _P, _P], _I),
    "nh_rhs": ([_P, _I, _I, _P, _P, _P, _P, _D, _P, _P, _P, _P, _P], _I),
    "nh_criterion": ([_P, _I, _I, _P, _P, _P, _P, _I, _P, _P], _I),
    "nh_coefficients": ([_P, _I, _I, _P, _P, _P, _P, _D, _D, _P, _P], _I),
    "nh_mask": ([_P, _I, _I, _I, _D, _I, _P, _P], _I),
    "nh_max_wavespeed": ([_P, _P, _I, ctypes.c_longlong, _D, _P, _P], _I),
    "nh_ldg_solve": ([_P, _I, _I, _P, _P, _P, _P, _D, _D, _D, _D, _D, _P, _P, _P, _P], _I),
    "nh_correct_momentum": ([_P, _I, _I, _P, _P, _P, _P, _D, _P, _P, _P], _I),
    "nh_bottom_sample": ([_P, _I, _P, _I, _P, _P, _P], _I),
    "nh_plan": ([_I, _I, ctypes.POINTER(_I), ctypes.POINTER(_I), ctypes.POINTER(_I),
                 ctypes.POINTER(_I)], _I),
    "nh_last_cuda_error": ([], ctypes.c_char_p),
    "nh_pm_workspace_bytes": ([_I, _I, _I], ctypes.c_size_t),
    "nh_pm_advance": ([_P, _P, _I, _I, _I, _P, _P, _P, _P, _I, ctypes.POINTER(Scheme),
                       ctypes.POINTER(Outputs), _P, _P, ctypes.c_size_t, _P], _I),
    "nh_pm_rhs": ([_P, _P, _I, _I, _I, _P, _P, _P, _P, _D, _P, _P, _P, _P, _P], _I),
    "nh_pm_criterion": ([_P, _P, _I, _I, _I, _P, _P, _P, _P, _I, _P, _P], _I),
    "nh_pm_coefficients": ([_P, _P, _I, _I, _I, _P, _P, _P, _P, _D, _D, _P, _P], _I),
    "nh_pm_ldg_solve": ([_P, _P, _I, _I, _I, _P, _P, _P, _P, _D, _D, _D, _D, _D, _P, _P, _P, _P,
                         ctypes.c_size_t, _P], _I),
    "nh_pm_correct_momentum": ([_P, _P, _I, _I, _I, _P, _P, _P, _P, _D, _P, _P, _P], _I),
}

_lib = None


def load(path: str = LIB_PATH):
    """Load (once) and type the shared library; raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"CUDA extension not built: {path} is missing "
                           "(run `python -m paper_2505_17025_b200.build`)")
    lib = ctypes.CDLL(path)
    for name, (args, res) in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if lib.nh_abi_version() != ABI_VERSION:
        raise RuntimeError("ABI version mismatch")
    _lib = lib
    return lib


def check(rc: int, what: str):
    if rc == 0:
        return
    lib = load()
    if rc == E_UNSUPPORTED:
        raise NotImplementedError(f"{what}: configuration not supported by the B200 kernels")
    if rc == E_ARG:
        raise ValueError(f"{what}: invalid arguments")
    raise RuntimeError(f"{what}: CUDA error: {lib.nh_last_cuda_error().decode()}")


def plan(n_elements: int, n_members: int):
    lib = load()
    c, t, th, sm = _I(), _I(), _I(), _I()
    check(lib.nh_plan(n_elements, n_members, ctypes.byref(c), ctypes.byref(t), ctypes.byref(th),
                      ctypes.byref(sm)), "nh_plan")
    return {"cluster": c.value, "tile": t.value, "threads": th.value, "smem": sm.value}
