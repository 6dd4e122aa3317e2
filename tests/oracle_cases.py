"""Rebuild oracle objects from the golden fixture metadata (tests/golden/short.npz)."""

import os

import numpy as np

from oracle import nhswe_oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
NAMES = ["flat_walls", "flat_absorbing", "plate", "quartic_slide", "smooth_box", "slope_slide"]


def load_short():
    return np.load(os.path.join(GOLDEN, "short.npz"))


def bottom_from(d, name):
    kind = str(d[name + "/bottom_kind"])
    p = d[name + "/bottom"]
    if kind == "flat":
        return O.Flat(p[1])
    if kind == "plate":
        return O.Plate(*p[1:5])
    if kind == "quartic":
        return O.QuarticSlide(p[1], p[2], p[3], O.Motion(*p[4:9]), p[9])
    if kind == "smooth_box":
        return O.SmoothBox(*p[1:6])
    return O.SlopeSlide(*p[1:10])


def member_from(d, name):
    xl, xr, n = d[name + "/grid"]
    g = O.Grid(float(xl), float(xr), int(n))
    bcs = tuple(str(v) for v in d[name + "/bcs"])
    return O.Member(g, bottom_from(d, name), bcs, float(d[name + "/dt"]))


def state_from(d, name):
    return d[name + "/h0"], d[name + "/hu0"], d[name + "/hw0"]
