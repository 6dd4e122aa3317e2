"""Device plumbing: parameter packing, uploads, status decoding.

PyTorch is used only to own device memory and streams; every computation is
one of the library's kernels (``_lib``).  Without a CUDA device every entry
point raises -- there is deliberately no CPU path.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("no CUDA device: the B200 NH-SWE kernels have no CPU fallback")
    return _lib.load()


def stream_ptr():
    return torch().cuda.current_stream().cuda_stream


def dev(a, dtype=np.float64):
    """Host array -> contiguous device tensor."""
    t = torch()
    arr = np.ascontiguousarray(a, dtype=dtype)
    return t.from_numpy(arr).to("cuda", non_blocking=False)


def ptr(x) -> int | None:
    return None if x is None else x.data_ptr()


# ------------------------------------------------------------------ packing

BC_CODE = {"absorbing": _lib.BC_ABSORBING, "wall": _lib.BC_WALL}


def member_record(grid, bathy, bcs, dt: float | None, any_order: bool = False) -> np.ndarray:
    """One nh_member record (include/nhswe_b200.h) for a (grid, bottom, bcs, dt).

    The P1 kernels take their operators from it; for the m-node kernels
    (any_order=True, orders p > 1) its P1 operator arrays stay zero and the
    operators travel in pm_record(grid)."""
    if grid.poly_order != 1 and not any_order:
        raise NotImplementedError("this entry point implements the P1 discretisation only "
                                  "(orders p > 1: heun_step, adaptive_step, apply_correction, "
                                  "simulate, Ensemble, rhs_operator, criterion_values)")
    r = np.zeros(1, dtype=_lib.MEMBER_DTYPE)
    r["x_left"] = grid.x_left
    r["dx"] = grid.dx
    r["dt"] = 0.0 if dt is None else dt
    r["eps"] = 1e-9 * grid.dx
    r["two_over_dx"] = 2.0 / grid.dx
    if grid.poly_order == 1:
        r["weak_div"] = grid.weak_div.ravel()
        r["lift_left"] = grid.lift_left
        r["lift_right"] = grid.lift_right
        r["mass"] = grid.mass.ravel()
        r["stiffness"] = grid.stiffness.ravel()
        r["deriv_ref"] = grid.deriv_ref.ravel()
    from .bathymetry import device_model
    kind, params = device_model(bathy).pack()
    r["bottom_kind"] = kind
    r["bottom"][0, :len(params)] = params
    if bcs is not None:
        r["bc_left"] = BC_CODE[bcs.left.kind]
        r["bc_right"] = BC_CODE[bcs.right.kind]
    return r


def pm_record(grid) -> np.ndarray:
    """One nh_pm_member record: the grid's m-node operators (the reference
    GridSpec values, grid.py:79-114) and node offsets 0.5*dx*(ref + 1)."""
    m = grid.poly_order + 1
    if m > _lib.PM_MAX_NODES:
        raise NotImplementedError(f"poly_order {grid.poly_order}: the kernels take m <= "
                                  f"{_lib.PM_MAX_NODES} nodes per element")
    r = np.zeros(1, dtype=_lib.PM_DTYPE)
    for f in ("weak_div", "mass", "stiffness", "deriv_ref"):
        r[f][0, :m * m] = np.ascontiguousarray(getattr(grid, f)).ravel()
    r["lift_left"][0, :m] = grid.lift_left
    r["lift_right"][0, :m] = grid.lift_right
    r["node_off"][0, :m] = 0.5 * grid.dx * (grid.ref_nodes + 1.0)
    return r


def pm_from_members(records: np.ndarray) -> np.ndarray:
    """nh_pm_member records of P1 members from their nh_member records (the
    same operators, m = 2): the m-node kernels then run a P1 ensemble -- the
    path of an LDG flux outside the alternating family."""
    records = np.atleast_1d(records)
    r = np.zeros(len(records), dtype=_lib.PM_DTYPE)
    for f in ("weak_div", "mass", "stiffness", "deriv_ref"):
        r[f][:, :4] = records[f].reshape(len(records), 4)
    r["lift_left"][:, :2] = records["lift_left"].reshape(len(records), 2)
    r["lift_right"][:, :2] = records["lift_right"].reshape(len(records), 2)
    r["node_off"][:, 1] = records["dx"].reshape(len(records))
    return r


def upload_members(records: np.ndarray):
    """Structured member table -> device byte tensor."""
    raw = np.ascontiguousarray(records).view(np.uint8)
    return dev(raw, dtype=np.uint8)


def new_status(n: int):
    st = np.zeros(n, dtype=_lib.STATUS_DTYPE)
    st["error_key"] = _lib.STATUS_OK_KEY
    return dev(st.view(np.uint8), dtype=np.uint8)


def read_status(t) -> np.ndarray:
    return t.cpu().numpy().view(_lib.STATUS_DTYPE)


def decode_error(key) -> tuple[int, int, int] | None:
    key = int(key)
    if key == 0xFFFFFFFFFFFFFFFF:
        return None
    return key >> 34, (key >> 30) & 15, (key & 0x3FFFFFFF) - 1


def raise_for_status(status: np.ndarray, t0, dt, member: int = 0):
    """Map a device error record to the reference exception types."""
    from .corrector import EllipticSolveError
    from .hydrostatic import PositivityError
    err = decode_error(status["error_key"][member])
    if err is None:
        return
    step, code, element = err
    t = float(np.asarray(t0).ravel()[member]) if np.ndim(t0) else float(t0)
    dtm = float(np.asarray(dt).ravel()[member]) if np.ndim(dt) else float(dt)
    for _ in range(step):          # time accumulates as t + dt (hydrostatic.py:206)
        t = t + dtm
    if code == _lib.ERR_POSITIVITY_ENTRY:
        raise PositivityError(element, t)
    if code in (_lib.ERR_POSITIVITY_STAGE1, _lib.ERR_POSITIVITY_STAGE2):
        raise PositivityError(-1, t + dtm)
    if code == _lib.ERR_SOLVE_PIVOT:
        raise EllipticSolveError(f"singular elliptic system (zero pivot in element {element})")
    if code == _lib.ERR_SOLVE_RESIDUAL:
        raise EllipticSolveError(
            f"elliptic solve residual {float(status['resid_max'][member]):.3e} exceeds the "
            f"residual tolerance at t={t + dtm} (likely ill-conditioned)")
    if code == _lib.ERR_STRUCTURE:
        raise AssertionError("structural condition s12 > 0 violated")
    raise EllipticSolveError("non-finite elliptic solution")


# ------------------------------------------------------------ small kernels

def bottom_sample(model, x: np.ndarray, t: float):
    lib = require_cuda()
    from .bathymetry import device_model
    rec = np.zeros(1, dtype=_lib.MEMBER_DTYPE)
    kind, params = device_model(model).pack()
    rec["bottom_kind"] = kind
    rec["bottom"][0, :len(params)] = params
    m = upload_members(rec)
    xs = dev(np.ravel(x))
    tt = dev(np.array([t], dtype=np.float64))
    out = torch().empty((6, xs.numel()), dtype=torch().float64, device="cuda")
    _lib.check(lib.nh_bottom_sample(ptr(m), 1, ptr(xs), xs.numel(), ptr(tt), ptr(out),
                                    stream_ptr()), "nh_bottom_sample")
    host = out.cpu().numpy()
    shape = np.shape(x)
    return tuple(host[i].reshape(shape) for i in range(6))


def flags_to_bits(flags: np.ndarray) -> np.ndarray:
    """bool [..., N] -> uint32 words [..., ceil(N/32)] (bit e%32 of word e//32)."""
    f = np.asarray(flags, dtype=bool)
    n = f.shape[-1]
    nw = (n + 31) // 32
    pad = np.zeros(f.shape[:-1] + (nw * 32,), dtype=bool)
    pad[..., :n] = f
    b = np.packbits(pad.reshape(f.shape[:-1] + (nw, 4, 8)), axis=-1, bitorder="little")
    return np.ascontiguousarray(b.reshape(f.shape[:-1] + (nw, 4))).view(np.uint32)[..., 0]


def bits_to_flags(bits: np.ndarray, n: int) -> np.ndarray:
    b = np.ascontiguousarray(bits, dtype=np.uint32)
    u8 = b.view(np.uint8)
    f = np.unpackbits(u8.reshape(b.shape[:-1] + (-1,)), axis=-1, bitorder="little")
    return f[..., :n].astype(bool)


def scheme(mode: int, kind: str = "eta_over_d", k_nh: float = 1e-3, enlarge: bool = False,
           flux=None, g: float = 9.81, rho: float = 1000.0, record_cfl: bool = True,
           residual_tol: float = 1e-10):
    s = _lib.Scheme()
    s.residual_tol = residual_tol
    s.g = g
    s.rho = rho
    s.k_nh = k_nh
    s.c11 = 0.5 if flux is None else flux.c11
    s.c12 = -0.5 if flux is None else flux.c12
    s.c22 = 0.0 if flux is None else flux.c22
    s.mode = mode
    s.criterion = _lib.CRIT[kind]
    s.enlarge = 1 if enlarge else 0
    s.record_cfl = 1 if record_cfl else 0
    return s


def _outputs(flag_bits=None, p_out=None, given=None, gauges=None):
    """nh_outputs; gauges = (int32 node indices [G], float64 out [n_steps][B][G]) or None."""
    if gauges is None:
        return _lib.Outputs(ptr(flag_bits), ptr(p_out), ptr(given), None, None, 0)
    nodes, out = gauges
    return _lib.Outputs(ptr(flag_bits), ptr(p_out), ptr(given), ptr(nodes), ptr(out),
                        int(nodes.numel()))


def advance(members, h, hu, hw, time, n_steps, sch, status, flag_bits=None, p_out=None,
            given=None, gauges=None):
    """Enqueue nh_advance (resident cluster kernel) on the current stream, in place."""
    lib = require_cuda()
    B, N = h.shape[0], h.shape[1]
    out = _outputs(flag_bits, p_out, given, gauges)
    rc = lib.nh_advance(ptr(members), B, N, ptr(h), ptr(hu), ptr(hw), ptr(time), int(n_steps),
                        ctypes.byref(sch), ctypes.byref(out), ptr(status), stream_ptr())
    _lib.check(rc, "nh_advance")


_pm_ws = {}


def pm_workspace(m: int, B: int, N: int):
    n = int(require_cuda().nh_pm_workspace_bytes(m, B, N))
    ws = _pm_ws.get("ws")
    if ws is None or ws.numel() < n:
        ws = torch().empty(n, dtype=torch().uint8, device="cuda")
        _pm_ws["ws"] = ws
    return ws


def pm_advance(members, pm, h, hu, hw, time, n_steps, sch, status, flag_bits=None, p_out=None,
               gauges=None, given=None):
    """Enqueue nh_pm_advance (m-node kernels; h, hu, hw CUDA [B][N][m]) in place."""
    lib = require_cuda()
    B, N, m = h.shape[0], h.shape[1], h.shape[2]
    out = _outputs(flag_bits, p_out, given, gauges)
    ws = pm_workspace(m, B, N)
    rc = lib.nh_pm_advance(ptr(members), ptr(pm), m, B, N, ptr(h), ptr(hu), ptr(hw), ptr(time),
                           int(n_steps), ctypes.byref(sch), ctypes.byref(out), ptr(status),
                           ptr(ws), ws.numel(), stream_ptr())
    _lib.check(rc, "nh_pm_advance")


class nvtx_range:
    """NVTX range around a block of launches (shows in Nsight timelines;
    a no-op cost when no profiler is attached)."""

    def __init__(self, name: str):
        self.name = name

    def __enter__(self):
        torch().cuda.nvtx.range_push(self.name)
        return self

    def __exit__(self, *exc):
        torch().cuda.nvtx.range_pop()


def stream_workspace(B: int, N: int):
    lib = require_cuda()
    n = int(lib.nh_stream_workspace_bytes(B, N))
    return torch().empty(n, dtype=torch().uint8, device="cuda")


def stream_advance(members, h, hu, hw, time, n_steps, sch, status, workspace, flag_bits=None,
                   p_out=None, gauges=None):
    """Enqueue nh_stream_advance (tiled streaming kernels) on the current stream, in place."""
    lib = require_cuda()
    B, N = h.shape[0], h.shape[1]
    out = _outputs(flag_bits, p_out, None, gauges)
    rc = lib.nh_stream_advance(ptr(members), B, N, ptr(h), ptr(hu), ptr(hw), ptr(time),
                               int(n_steps), ctypes.byref(sch), ctypes.byref(out), ptr(status),
                               ptr(workspace), workspace.numel(), stream_ptr())
    _lib.check(rc, "nh_stream_advance")


STREAM_KERNELS = ("nh_stream_kp", "nh_stream_ks", "nh_stream_kx", "nh_stream_kc",
                  "nh_stream_kp_finalize", "nh_stream_prep")


def stream_graphs(enable: bool | None = None) -> bool:
    """Query / set whether nh_stream_advance runs its time loop as a CUDA graph."""
    return bool(require_cuda().nh_stream_graphs(-1 if enable is None else int(bool(enable))))


def stream_timing(enable: bool):
    """Arm / disarm per-kernel CUDA-event timing inside nh_stream_advance."""
    _lib.check(require_cuda().nh_stream_timing(1 if enable else 0), "nh_stream_timing")


def stream_kernel_times() -> dict:
    """{kernel: (total ms, launches)} recorded since arming (then cleared)."""
    ms = (ctypes.c_double * len(STREAM_KERNELS))()
    n = (ctypes.c_longlong * len(STREAM_KERNELS))()
    _lib.check(require_cuda().nh_stream_kernel_times(ms, n), "nh_stream_kernel_times")
    return {k: (ms[i], n[i]) for i, k in enumerate(STREAM_KERNELS)}


def launch_count() -> int:
    """Kernels the library has enqueued since it was loaded."""
    return int(require_cuda().nh_launch_count())
