"""The reference-side binding of the C ABI, as a maintainer of `nhswe` would
add it next to the reference's driver.py.

Only ctypes, numpy and a CUDA allocator (torch here; any allocator works, the
ABI takes raw device pointers) -- nothing from this repository's Python
package.  The struct layouts and constants are the ones in
include/nhswe_b200.h; tests/test_gpu_capi_stub.py runs this file against the
library and checks it equals the package's own path.

    simulate_native(spec, initial, mode, criterion) -> (h, hu, hw, t, status)

replaces the body of the reference's simulate loop (driver.py:79-94) with
one nh_advance call for all spec.n_steps; it takes the reference's own
ScenarioSpec / FlowState / Criterion objects.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

LIB = os.environ.get("NH_LIB") or os.path.join(
    os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))),
    "paper_2505_17025_b200", "_lib", "libnhswe_b200.so")

_C, _I, _P = ctypes.c_double, ctypes.c_int32, ctypes.c_void_p


class Member(ctypes.Structure):          # nh_member (312 B)
    _fields_ = [("x_left", _C), ("dx", _C), ("dt", _C), ("eps", _C), ("two_over_dx", _C),
                ("weak_div", _C * 4), ("lift_left", _C * 2), ("lift_right", _C * 2),
                ("mass", _C * 4), ("stiffness", _C * 4), ("deriv_ref", _C * 4),
                ("bottom", _C * 12), ("bc_left", _I), ("bc_right", _I), ("bottom_kind", _I),
                ("reserved", _I)]


class Scheme(ctypes.Structure):          # nh_scheme (72 B)
    _fields_ = [("g", _C), ("rho", _C), ("k_nh", _C), ("c11", _C), ("c12", _C), ("c22", _C),
                ("mode", _I), ("criterion", _I), ("enlarge", _I), ("record_cfl", _I),
                ("residual_tol", _C)]


class Status(ctypes.Structure):          # nh_status (72 B)
    _fields_ = [("error_key", ctypes.c_uint64), ("cfl_max", _C), ("flagged", ctypes.c_int64),
                ("steps_done", _I), ("any_hw", _I), ("resid_max", _C), ("resid_acc", _C * 4)]


class Outputs(ctypes.Structure):         # nh_outputs
    _fields_ = [("flag_bits", _P), ("p_nh", _P), ("given_flags", _P), ("gauge_nodes", _P),
                ("gauge_h", _P), ("n_gauges", _I)]


MODES = {"hydrostatic": 0, "global": 1, "adaptive": 2}
CRIT = {"eta_over_d": 0, "eta_x": 1, "u": 2, "u_x": 3, "w": 4, "w_x": 5}
OK_KEY = 2 ** 64 - 1


def load(path: str = LIB):
    lib = ctypes.CDLL(path)
    lib.nh_abi_version.restype = ctypes.c_int
    lib.nh_advance.argtypes = [_P, ctypes.c_int, ctypes.c_int, _P, _P, _P, _P, ctypes.c_int,
                               ctypes.POINTER(Scheme), ctypes.POINTER(Outputs), _P, _P]
    lib.nh_advance.restype = ctypes.c_int
    return lib


def bathymetry_kind_and_params(b):
    """Reference bottom models -> (NH_BOTTOM_*, packed parameters); the layout
    of csrc/bathy.cuh's header comment."""
    kind = type(b).__name__
    if kind == "FlatBottom":
        return 0, [b.h0]
    if kind == "HammackPlate":
        return 1, [b.h0, b.zeta0, b.b, b.alpha]          # alpha = 1.11 / t_c (bathymetry.py:102)
    if kind == "WhittakerSlide":
        m = b.motion
        return 2, [b.h0, b.Hs, b.Ls, b.x_start, m.a0, m.u_t, m.t1, m.t2, m.t3, 2.0 / b.Ls]
    raise TypeError(f"no device form for {kind}")


def simulate_native(lib, spec, initial, mode, criterion=None, rho=1000.0, residual_tol=1e-10):
    """simulate() (driver.py:50-103) with the step loop in one nh_advance call."""
    import torch
    g = spec.grid
    m = Member(x_left=g.x_left, dx=g.dx, dt=spec.dt, eps=1e-9 * g.dx, two_over_dx=2.0 / g.dx)
    for name in ("weak_div", "lift_left", "lift_right", "mass", "stiffness", "deriv_ref"):
        getattr(m, name)[:] = np.ravel(getattr(g, name)).tolist()
    m.bottom_kind, params = bathymetry_kind_and_params(spec.bathymetry)
    m.bottom[:len(params)] = params
    m.bc_left = 1 if spec.bcs.left.kind == "wall" else 0
    m.bc_right = 1 if spec.bcs.right.kind == "wall" else 0
    crit = criterion if criterion is not None else type("C", (), {"kind": "eta_over_d",
                                                                  "k_nh": 1e-3,
                                                                  "enlarge": False})()
    sch = Scheme(g=spec.g, rho=rho, k_nh=crit.k_nh, c11=0.5, c12=-0.5, c22=0.0,
                 mode=MODES[mode], criterion=CRIT[crit.kind], enlarge=int(crit.enlarge),
                 record_cfl=1, residual_tol=residual_tol)

    def dev(a):
        return torch.from_numpy(np.ascontiguousarray(a, np.float64)).cuda()

    h, hu, hw = dev(initial.h.values), dev(initial.hu.values), dev(initial.hw.values)
    t = dev([initial.time])
    mem = torch.frombuffer(bytearray(bytes(m)), dtype=torch.uint8).cuda()
    status = torch.frombuffer(bytearray(bytes(Status(error_key=OK_KEY))), dtype=torch.uint8).cuda()
    out = Outputs()
    rc = lib.nh_advance(mem.data_ptr(), 1, g.n_elements, h.data_ptr(), hu.data_ptr(),
                        hw.data_ptr(), t.data_ptr(), spec.n_steps, ctypes.byref(sch),
                        ctypes.byref(out), status.data_ptr(),
                        torch.cuda.current_stream().cuda_stream)
    if rc != 0:
        raise RuntimeError(f"nh_advance failed ({rc})")
    torch.cuda.synchronize()
    st = Status.from_buffer_copy(status.cpu().numpy().tobytes())
    return h.cpu().numpy(), hu.cpu().numpy(), hw.cpu().numpy(), float(t.item()), st


def raise_for(st, t0, dt):
    """The reference exceptions for a device status (header error_key)."""
    if st.error_key == OK_KEY:
        return
    step, code = st.error_key >> 34, (st.error_key >> 30) & 15
    element = (st.error_key & 0x3FFFFFFF) - 1
    t = t0
    for _ in range(step):
        t = t + dt
    if code in (1, 2, 3):
        from nhswe.hydrostatic import PositivityError
        raise PositivityError(element if code == 1 else -1, t if code == 1 else t + dt)
    if code == 7:
        raise AssertionError("structural condition s12 > 0 violated")
    from nhswe.corrector import EllipticSolveError
    raise EllipticSolveError(f"elliptic solve failed on the device (code {code}, "
                             f"residual {st.resid_max:.3e})")
