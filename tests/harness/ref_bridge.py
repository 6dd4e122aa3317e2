"""The reference package itself (nhswe) driven on a BASELINE member.

Used by `bench.py --impl reference` and the bench's `cpu_baseline` leg, and
by the golden-vector scripts.  It imports the UNMODIFIED reference: first the
copy installed by `pip install --target baseline/_ref /root/reference`
(git-ignored, travels to the GPU box), else the mounted source
tree.  The two harness bottoms of configs 2, 3 and 5 (smoothed box uplift,
Gaussian mound on a slope) have no reference class:
the oracle's numpy model is wrapped as a reference `BathymetryModel`
subclass, exactly as tests/golden/make_golden.py does, so the reference's own
step code runs on them.

Test / benchmark harness only -- never imported by the package.
"""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CANDIDATES = (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src")


def import_reference():
    """The reference package `nhswe` and where it came from, or (None, why)."""
    for path in CANDIDATES:
        if os.path.isdir(os.path.join(path, "nhswe")):
            if path not in sys.path:
                sys.path.insert(0, path)
            try:
                import nhswe
                return nhswe, path
            except Exception as exc:   # pragma: no cover - broken install
                return None, f"import nhswe from {path} failed: {exc}"
    return None, "reference package not installed (baseline/_ref) and /root/reference absent"


def reference_member(cfg, i: int):
    """(R, grid, bathymetry, bcs, dt, FlowState at t = 0) of member i as
    reference objects."""
    R, where = import_reference()
    if R is None:
        raise RuntimeError(where)
    from nhswe.bathymetry import BathymetryModel, BottomSample

    from oracle import nhswe_oracle as O
    from tests.helpers import oracle_depth

    class Wrapped(BathymetryModel):
        def __init__(self, model):
            object.__setattr__(self, "model", model)

        def _sample(self, x, t):
            return BottomSample(*self.model.channels(np.asarray(x, dtype=float), t))

    m = cfg.member(i)
    grid = R.GridSpec(m.grid.x_left, m.grid.x_right, m.grid.n_elements)
    b = m.bathymetry
    kind = type(b).__name__
    if kind == "FlatBottom":
        bathy = R.FlatBottom(b.h0)
    elif kind == "SmoothBoxPlate":
        bathy = Wrapped(O.SmoothBox(b.h0, b.zeta0, b.b, b.alpha, b.w))
    elif kind == "SlopeGaussianSlide":
        bathy = Wrapped(O.SlopeSlide(b.d_top, b.tan_theta, b.d_max, b.A, b.sigma, b.x0, b.u_t,
                                     b.t0, b.d_stop))
    else:
        raise TypeError(kind)
    bcs = R.BoundaryPair(R.BoundaryCondition(m.bcs.left.kind),
                         R.BoundaryCondition(m.bcs.right.kind))
    h, hu, hw = cfg.host_state(i, oracle_depth)
    state = R.FlowState(R.NodalField(grid, h), R.NodalField(grid, hu), R.NodalField(grid, hw),
                        0.0)
    return R, grid, bathy, bcs, m.dt, state
