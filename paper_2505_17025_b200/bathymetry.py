"""Bottom models d(x, t) (reference bathymetry.py:15-193) as GPU parameter packs.

Each model is a frozen dataclass whose ``pack()`` returns the device kind and
its parameter vector for ``nh_member.bottom`` (csrc/bathy.cuh evaluates the
six channels in registers, so bathymetry costs no HBM traffic).
``sample(x, t)`` evaluates the channels through the GPU kernel
``nh_bottom_sample`` and returns a ``BottomSample`` of host arrays, like the
reference.  Besides the reference's three models there are the two harness
models the BASELINE configurations need:
``SmoothBoxPlate`` (configs 2 and 4) and ``SlopeGaussianSlide`` (configs 3
and 5).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib

GRAVITY = 9.81
RHO_WATER = 1000.0
CHANNELS = ("d", "d_x", "d_t", "d_tt", "d_xt", "d_xx")


@dataclass(frozen=True)
class BottomSample:
    d: np.ndarray
    d_x: np.ndarray
    d_t: np.ndarray
    d_tt: np.ndarray
    d_xt: np.ndarray
    d_xx: np.ndarray


class BathymetryModel:
    """Base class (reference bathymetry.py:33-63)."""

    def pack(self) -> tuple[int, list]:
        raise NotImplementedError

    def sample(self, x: np.ndarray, t: float) -> BottomSample:
        x = np.asarray(x, dtype=float)
        key = (x.__array_interface__["data"][0], x.shape, x.strides, float(t))
        memo = getattr(self, "_memo", None)
        if memo is None:
            memo = {}
            object.__setattr__(self, "_memo", memo)
        hit = memo.get(key)
        if hit is not None:
            return hit[1]
        from ._device import bottom_sample
        out = BottomSample(*bottom_sample(self, x, t))
        if len(memo) >= 16:
            memo.pop(next(iter(memo)))
        memo[key] = (x, out)
        return out

    def depth(self, x: np.ndarray, t: float) -> np.ndarray:
        return self.sample(x, t).d


@dataclass(frozen=True)
class FlatBottom(BathymetryModel):
    """Constant still depth (reference bathymetry.py:66-79)."""
    h0: float

    def __post_init__(self):
        if self.h0 <= 0:
            raise ValueError("still depth h0 must be positive")

    def pack(self):
        return _lib.BOTTOM_FLAT, [self.h0]


@dataclass(frozen=True)
class HammackPlate(BathymetryModel):
    """Impulsive plate |x| < b (reference bathymetry.py:82-116)."""
    h0: float
    zeta0: float
    b: float
    t_c: float

    def __post_init__(self):
        if self.h0 <= 0 or self.b <= 0 or self.t_c <= 0:
            raise ValueError("h0, b and t_c must be positive")
        if abs(self.zeta0) >= self.h0:
            raise ValueError("|zeta0| must stay below the still depth")

    @property
    def alpha(self) -> float:
        return 1.11 / self.t_c

    def pack(self):
        return _lib.BOTTOM_PLATE, [self.h0, self.zeta0, self.b, self.alpha]


@dataclass(frozen=True)
class SlideMotion:
    """Accelerate / coast / brake / stop (reference bathymetry.py:119-144)."""
    a0: float
    u_t: float
    t1: float
    t2: float
    t3: float

    def __post_init__(self):
        if not 0 < self.t1 < self.t2 < self.t3:
            raise ValueError("require 0 < t1 < t2 < t3")


@dataclass(frozen=True)
class WhittakerSlide(BathymetryModel):
    """Quartic bump sliding on a flat bed (reference bathymetry.py:147-184)."""
    h0: float
    Hs: float
    Ls: float
    motion: SlideMotion
    x_start: float = 0.0

    def __post_init__(self):
        if not self.h0 > self.Hs > 0:
            raise ValueError("require h0 > Hs > 0")
        if self.Ls <= 0:
            raise ValueError("slide length Ls must be positive")

    def pack(self):
        mo = self.motion
        return _lib.BOTTOM_QUARTIC_SLIDE, [self.h0, self.Hs, self.Ls, self.x_start,
                                           mo.a0, mo.u_t, mo.t1, mo.t2, mo.t3, 2.0 / self.Ls]


@dataclass(frozen=True)
class SmoothBoxPlate(BathymetryModel):
    """Box uplift of half-width b at the wall with a tanh edge of width w.

    d = h0 - zeta(t) S(x), zeta = zeta0 (1 - exp(-alpha t)),
    S = (1 - tanh((|x| - b) / w)) / 2  (BASELINE configs 2 and 4).
    """
    h0: float
    zeta0: float
    b: float
    alpha: float
    w: float

    def __post_init__(self):
        if self.h0 <= 0 or self.b <= 0 or self.alpha <= 0 or self.w <= 0:
            raise ValueError("h0, b, alpha and w must be positive")
        if abs(self.zeta0) >= self.h0:
            raise ValueError("|zeta0| must stay below the still depth")

    def pack(self):
        return _lib.BOTTOM_SMOOTH_BOX, [self.h0, self.zeta0, self.b, self.alpha, self.w,
                                        1.0 / self.w, 1.0 / (self.w * self.w)]


@dataclass(frozen=True)
class SlopeGaussianSlide(BathymetryModel):
    """Gaussian mound sliding down a plane slope (BASELINE configs 3 and 5).

    d0(x) = min(d_top + x tan(theta), d_max), G = A exp(-((x - xc)/sigma)^2/2),
    d = d0 - G, xc(t) = x0 + u_t t0 ln cosh(t/t0) until d0(xc) = d_stop.
    """
    d_top: float
    tan_theta: float
    d_max: float
    A: float
    sigma: float
    x0: float
    u_t: float
    t0: float
    d_stop: float

    @property
    def x_stop(self) -> float:
        return (self.d_stop - self.d_top) / self.tan_theta

    @property
    def t_stop(self) -> float:
        arg = (self.x_stop - self.x0) / (self.u_t * self.t0)
        if arg <= 0.0:
            return 0.0
        return self.t0 * (arg + math.log1p(math.sqrt(-math.expm1(-2.0 * arg))))

    def pack(self):
        return _lib.BOTTOM_SLOPE_SLIDE, [self.d_top, self.tan_theta, self.d_max, self.A,
                                         self.sigma, self.x0, self.u_t, self.t0, self.d_stop,
                                         self.x_stop, self.t_stop, 1.0 / self.sigma]


def hammack_time_constant(h0: float, b: float, direction: str, g: float = GRAVITY) -> float:
    """Reference bathymetry.py:187-193."""
    const = {"up": 0.148, "down": 0.093}.get(direction)
    if const is None:
        raise ValueError(f"direction must be 'up' or 'down', got {direction!r}")
    return const * b / np.sqrt(g * h0)


def device_model(bathy) -> BathymetryModel:
    """The device form of a bottom model: this package's models as they are,
    and the reference's own objects (nhswe.FlatBottom, HammackPlate,
    WhittakerSlide, bathymetry.py:66-184 -- interface sample(x, t), no
    pack()) mapped by class and fields onto the same device kinds, so a
    caller can hand reference objects straight to the mirrored API.  Any
    other model has no device evaluation: TypeError, since the kernels
    evaluate the bottom analytically in registers."""
    if hasattr(bathy, "pack"):
        return bathy
    kind = type(bathy).__name__
    try:
        if kind == "FlatBottom":
            return FlatBottom(float(bathy.h0))
        if kind == "HammackPlate":
            return HammackPlate(float(bathy.h0), float(bathy.zeta0), float(bathy.b),
                                float(bathy.t_c))
        if kind == "WhittakerSlide":
            m = bathy.motion
            return WhittakerSlide(float(bathy.h0), float(bathy.Hs), float(bathy.Ls),
                                  SlideMotion(float(m.a0), float(m.u_t), float(m.t1),
                                              float(m.t2), float(m.t3)),
                                  float(bathy.x_start))
    except AttributeError as exc:
        raise TypeError(f"bottom model {kind}: missing field for its device form ({exc})") from exc
    raise TypeError(f"bottom model {kind} has no device evaluation: the B200 kernels evaluate "
                    "FlatBottom, HammackPlate, WhittakerSlide, SmoothBoxPlate and "
                    "SlopeGaussianSlide analytically; a model known only through sample(x, t) "
                    "cannot run on the device")
