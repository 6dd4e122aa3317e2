"""Generate golden vectors by running the REAL reference package (nhswe).

Run in the build container (the reference is mounted read-only there):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--long]

Writes tests/golden/*.npz.  Short fixtures pin every hot-path function of
the reference on small inputs; --long also runs the BASELINE configs 1-3 to
their final time through the reference's own `simulate` (configs 2 and 3
use the harness bottom models of oracle/nhswe_oracle.py wrapped as reference
BathymetryModel subclasses, so the reference's step logic is what runs).
Nothing here is used at run time on the GPU box; the fixtures are.
"""

from __future__ import annotations

import argparse
import os
import sys
import time
import zlib

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import nhswe as R  # noqa: E402
from nhswe.bathymetry import BathymetryModel, BottomSample  # noqa: E402
from nhswe import corrector as RC, hydrostatic as RH, adaptivity as RA  # noqa: E402

from oracle import nhswe_oracle as O  # noqa: E402


class Wrapped(BathymetryModel):
    """A harness bottom (oracle model) exposed through the reference's interface."""

    def __init__(self, model):
        object.__setattr__(self, "model", model)

    def _sample(self, x, t):
        return BottomSample(*self.model.channels(np.asarray(x, dtype=float), t))


def smooth_state(grid, d0=10.0, amp=0.5, u0=0.2):
    x = grid.nodes
    h = d0 + amp * np.exp(-((x - x.mean()) / 5.0) ** 2)
    hu = u0 * h * np.sin(0.3 * x)
    hw = 0.05 * h * np.cos(0.2 * x)
    return R.FlowState(R.NodalField(grid, h), R.NodalField(grid, hu), R.NodalField(grid, hw), 0.0)


def cases():
    """(name, grid, bathy (reference object), spec-of-bottom for the oracle, bcs, dt, state)."""
    out = []
    g = R.GridSpec(0.0, 100.0, 60)
    out.append(("flat_walls", g, R.FlatBottom(10.0), ("flat", 10.0),
                R.BoundaryPair(R.WALL, R.WALL), 0.05, smooth_state(g)))
    out.append(("flat_absorbing", g, R.FlatBottom(10.0), ("flat", 10.0),
                R.BoundaryPair(R.ABSORBING, R.ABSORBING), 0.05, smooth_state(g)))
    g = R.GridSpec(0.0, 5.0, 100)
    b = R.HammackPlate(0.05, 0.005, 0.6, 0.13)
    d = b.sample(g.sample_nodes, 0.0).d
    z = np.zeros_like(d)
    out.append(("plate", g, b, ("plate", 0.05, 0.005, 0.6, 0.13),
                R.BoundaryPair(R.WALL, R.ABSORBING), 0.004,
                R.FlowState(R.NodalField(g, d), R.NodalField(g, z), R.NodalField(g, z), 0.0)))
    g = R.GridSpec(0.0, 15.0, 120)
    mo = R.SlideMotion(1.5, 0.327, 0.218, 2.218, 2.436)
    b = R.WhittakerSlide(0.175, 0.026, 0.5, mo, 5.0)
    d = b.sample(g.sample_nodes, 0.0).d
    z = np.zeros_like(d)
    out.append(("quartic_slide", g, b, ("quartic", 0.175, 0.026, 0.5, 1.5, 0.327, 0.218, 2.218,
                                        2.436, 5.0),
                R.BoundaryPair(R.ABSORBING, R.ABSORBING), 0.005,
                R.FlowState(R.NodalField(g, d), R.NodalField(g, z), R.NodalField(g, z), 0.0)))
    g = R.GridSpec(0.0, 10.0, 200)
    ob = O.SmoothBox(0.05, 0.005, 0.3, 20.0, 0.01)
    d = ob.channels(g.sample_nodes, 0.0)[0]
    z = np.zeros_like(d)
    out.append(("smooth_box", g, Wrapped(ob), ("smooth_box", 0.05, 0.005, 0.3, 20.0, 0.01),
                R.BoundaryPair(R.WALL, R.ABSORBING), 0.006,
                R.FlowState(R.NodalField(g, d), R.NodalField(g, z), R.NodalField(g, z), 0.0)))
    g = R.GridSpec(0.0, 20.0, 400)
    ob = O.SlopeSlide(0.1, np.tan(np.radians(15.0)), 1.0, 0.05, 0.2, 1.0, 1.0, 0.5, 0.8)
    d = ob.channels(g.sample_nodes, 0.0)[0]
    z = np.zeros_like(d)
    out.append(("slope_slide", g, Wrapped(ob), ("slope_slide", 0.1, float(np.tan(np.radians(15.0))),
                                                1.0, 0.05, 0.2, 1.0, 1.0, 0.5, 0.8),
                R.BoundaryPair(R.WALL, R.ABSORBING), 0.0026,
                R.FlowState(R.NodalField(g, d), R.NodalField(g, z), R.NodalField(g, z), 0.0)))
    return out


def short_fixtures():
    data = {}
    for name, grid, bathy, bspec, bcs, dt, st in cases():
        p = name + "/"
        data[p + "grid"] = np.array([grid.x_left, grid.x_right, grid.n_elements], dtype=float)
        data[p + "bottom"] = np.array([0.0 if isinstance(v, str) else v for v in bspec])
        data[p + "bottom_kind"] = np.array(bspec[0])
        data[p + "bcs"] = np.array([bcs.left.kind, bcs.right.kind])
        data[p + "dt"] = np.array(dt)
        for k in ("mass", "mass_inv", "stiffness", "deriv_ref", "weak_div", "lift_left",
                  "lift_right", "sample_nodes"):
            data[p + "grid_" + k] = getattr(grid, k)
        data[p + "h0"], data[p + "hu0"], data[p + "hw0"] = (st.h.values, st.hu.values,
                                                            st.hw.values)
        t_h, t_hu, t_hw = RH.rhs_operator(st, bathy, bcs)
        data[p + "rhs"] = np.stack([t_h, t_hu, t_hw])
        pred = RH.heun_step(st, dt, bathy, bcs, cfl_warn=False)
        data[p + "heun"] = np.stack([pred.h.values, pred.hu.values, pred.hw.values])
        for kind in RA.CRITERION_KINDS:
            data[p + "crit_" + kind] = RA.criterion_values(pred, bathy, kind)
        co = RC.assemble_coefficients(pred, bathy, dt)
        data[p + "coef"] = np.stack([co.s11, co.s12, co.s22, co.f1, co.f2, co.phi])
        n = grid.n_elements
        ranges = ((2, n // 3), (n // 2, n // 2 + 1), (n - n // 5, n - 1))
        corr, sol = RC.apply_correction(pred, bathy, dt, ranges, bcs)
        data[p + "corr_ranges"] = np.array(ranges)
        data[p + "corr"] = np.stack([corr.hu.values, corr.hw.values, sol.p_nh.values])
        # 12-step trajectories in every mode (adaptive with two criteria)
        for mode, crit in (("hydrostatic", None), ("global", None),
                           ("adaptive", R.Criterion("eta_over_d")),
                           ("adaptive_enl", R.Criterion("eta_over_d", 1e-3, True)),
                           ("adaptive_wx", R.Criterion("w_x"))):
            s = st
            hist = []
            for _ in range(12):
                r = R.adaptive_step(s, dt, bathy, bcs, mode=mode.split("_")[0], crit=crit,
                                    cfl_warn=False)
                s = r.state
                hist.append(r.mask.flags.copy())
            data[p + "traj_" + mode] = np.stack([s.h.values, s.hu.values, s.hw.values])
            data[p + "traj_" + mode + "_flags"] = np.array(hist)
    # manufactured LDG system (reference test_corrector.py manufactured_coefficients)
    n = 48
    grid = R.GridSpec(0.0, 1.0, n)
    x = grid.nodes
    s11 = 0.4 * np.sin(2.0 * np.pi * x)
    s12 = 2.0 + np.cos(x)
    s22 = 1.0 + 0.5 * np.sin(3.0 * x)
    pex, huex = np.sin(np.pi * x), np.cos(2.0 * x) + 2.0
    f1 = np.pi * np.cos(np.pi * x) + s11 * pex + s12 * huex
    f2 = -2.0 * np.sin(2.0 * x) - s11 * huex + s22 * pex
    bottom = R.FlatBottom(1.0).sample(grid.sample_nodes, 0.0)
    co = RC.EllipticCoefficients(grid, s11, s12, -s11, s22, f1, f2, np.zeros_like(x), bottom,
                                 0.1, 1.0)
    p_, hu_ = RC.ldg_solve(co, (3, 40), outer_hu=(huex[2, 1], huex[41, 0]))
    data["manufactured/coef"] = np.stack([s11, s12, s22, f1, f2])
    data["manufactured/solution"] = np.stack([p_, hu_])
    data["manufactured/outer"] = np.array([huex[2, 1], huex[41, 0]])
    np.savez_compressed(os.path.join(HERE, "short.npz"), **data)
    print("short.npz:", len(data), "arrays")


def error_fixtures():
    """The reference's error semantics and adjacent ranges (errors.npz):
    residual gate, non-finite solve, structural asserts, and corrections on
    touching ranges (each range its own block of the batched system)."""
    data = {}
    n = 48
    grid = R.GridSpec(0.0, 1.0, n)
    x = grid.nodes
    s11 = 0.4 * np.sin(2.0 * np.pi * x)
    s12 = 2.0 + np.cos(x)
    s22 = 1.0 + 0.5 * np.sin(3.0 * x)
    f1 = np.cos(np.pi * x) + s12
    f2 = -2.0 * np.sin(2.0 * x) + s22
    z = np.zeros_like(x)
    bottom = R.FlatBottom(1.0).sample(grid.sample_nodes, 0.0)

    def coeffs(**kw):
        base = dict(s11=s11, s12=s12, s21=-s11, s22=s22, f1=f1, f2=f2, phi=z)
        base.update(kw)
        return RC.EllipticCoefficients(grid, base["s11"], base["s12"], base["s21"], base["s22"],
                                       base["f1"], base["f2"], base["phi"], bottom, 0.1, 1.0)

    def outcome(fn):
        try:
            fn()
            return "ok"
        except Exception as exc:   # noqa: BLE001 - the type name is the fixture
            return type(exc).__name__

    co = coeffs()
    data["err/coef"] = np.stack([s11, s12, s22, f1, f2])
    data["err/tol_default"] = np.array(outcome(lambda: RC.ldg_solve(co, (3, 40), (0.2, 0.3))))
    data["err/tol_1e-18"] = np.array(outcome(
        lambda: RC.ldg_solve(co, (3, 40), (0.2, 0.3), residual_tol=1e-18)))
    bad_f1 = f1.copy()
    bad_f1[10, 1] = np.inf
    data["err/nonfinite"] = np.array(outcome(lambda: RC.ldg_solve(coeffs(f1=bad_f1), (3, 40))))
    neg = s12.copy()
    neg[7, 0] = -1.0
    data["err/s12_negative"] = np.array(outcome(lambda: coeffs(s12=neg)))
    data["err/s21_mismatch"] = np.array(outcome(lambda: coeffs(s21=-s11 + 1e-3)))
    data["err/flux_c12_0"] = np.array(outcome(
        lambda: RC.ldg_solve(co, (3, 40), flux=RC.FluxCoefficients(0.5, 0.0, 0.0))))
    # touching ranges: separate systems (solve_on_ranges and apply_correction)
    for name, grid_, bathy, bspec, bcs, dt, st in cases()[:3]:
        pred = RH.heun_step(st, dt, bathy, bcs, cfl_warn=False)
        m = grid_.n_elements
        ranges = ((2, m // 4), (m // 4 + 1, m // 2), (m // 2 + 1, m // 2 + 1), (m - 3, m - 1))
        corr, sol = RC.apply_correction(pred, bathy, dt, ranges, bcs)
        p = "adj/" + name + "/"
        data[p + "pred"] = np.stack([pred.h.values, pred.hu.values, pred.hw.values])
        data[p + "ranges"] = np.array(ranges)
        data[p + "corr"] = np.stack([corr.hu.values, corr.hw.values, sol.p_nh.values])
        co2 = RC.assemble_coefficients(pred, bathy, dt)
        sol2 = RC.solve_on_ranges(pred, co2, ranges, bcs)
        data[p + "solve"] = np.stack([sol2.hu_corrected.values, sol2.p_nh.values])
    np.savez_compressed(os.path.join(HERE, "errors.npz"), **data)
    print("errors.npz:", {k: str(v) for k, v in data.items() if v.dtype.kind == "U"})


def digest(flags: np.ndarray) -> int:
    return zlib.crc32(np.packbits(flags).tobytes())


# config 3: every 5000 steps through the end (windowed parity restarts the
# GPU from each one), plus the step before the first free-running mask flip
# (34652) for the criterion-margin report
CHECKPOINTS = {"config3": (500,) + tuple(range(5000, 112755, 5000)) + (34652,)}


def long_fixture(name, n_steps=None):
    from paper_2505_17025_b200 import configs
    from tests.helpers import oracle_depth
    cfg = configs.get(name)
    m = cfg.member(0)
    h, hu, hw = cfg.host_state(0, oracle_depth)
    grid = R.GridSpec(m.grid.x_left, m.grid.x_right, m.grid.n_elements)
    bk = type(m.bathymetry).__name__
    if bk == "FlatBottom":
        bathy = R.FlatBottom(m.bathymetry.h0)
    elif bk == "SmoothBoxPlate":
        b = m.bathymetry
        bathy = Wrapped(O.SmoothBox(b.h0, b.zeta0, b.b, b.alpha, b.w))
    else:
        b = m.bathymetry
        bathy = Wrapped(O.SlopeSlide(b.d_top, b.tan_theta, b.d_max, b.A, b.sigma, b.x0, b.u_t,
                                     b.t0, b.d_stop))
    bcs = R.BoundaryPair(R.BoundaryCondition(m.bcs.left.kind), R.BoundaryCondition(m.bcs.right.kind))
    steps = n_steps or cfg.n_steps
    spec = R.ScenarioSpec(cfg.name, grid, m.dt, steps * m.dt, bathy, bcs)
    assert spec.n_steps == steps
    init = R.FlowState(R.NodalField(grid, h), R.NodalField(grid, hu), R.NodalField(grid, hw), 0.0)
    data = {"h0": h, "hu0": hu, "hw0": hw, "dt": np.array(m.dt), "n_steps": np.array(steps)}
    ck = set(CHECKPOINTS.get(name, ()))
    for mode in cfg.modes:
        crit = R.Criterion("eta_over_d") if mode == "adaptive" else None
        t0 = time.time()
        # driver.simulate's loop (driver.py:79-94), unrolled here so the
        # reference state can also be saved at checkpoint steps
        state, loop_time, fractions, cnt, dig = init, 0.0, [], [], []
        for step in range(steps):
            s0 = time.perf_counter()
            res = R.adaptive_step(state, spec.dt, spec.bathymetry, spec.bcs, mode=mode, crit=crit,
                                  g=spec.g)
            loop_time += time.perf_counter() - s0
            state = res.state
            fractions.append(res.mask.fraction)
            if mode == "adaptive":
                f = np.zeros(grid.n_elements, bool)
                for e0, e1 in res.mask.ranges:
                    f[e0:e1 + 1] = True
                cnt.append(int(f.sum()))
                dig.append(digest(f))
            if mode == "adaptive" and step + 1 in ck:
                data[f"ck/s{step + 1}"] = np.stack([state.h.values, state.hu.values, state.hw.values])
                data[f"ck/t{step + 1}"] = np.array(state.time)
        fs = state
        data[mode + "/final"] = np.stack([fs.h.values, fs.hu.values, fs.hw.values])
        data[mode + "/loop_time"] = np.array(loop_time)
        data[mode + "/mask_fraction"] = np.array(float(np.mean(fractions)))
        if mode == "adaptive":
            data[mode + "/flag_count"] = np.array(cnt, dtype=np.int32)
            data[mode + "/flag_crc"] = np.array(dig, dtype=np.uint32)
        print(f"{name} {mode}: {steps} steps in {time.time() - t0:.1f}s", flush=True)
    out = os.path.join(HERE, f"{name}_full.npz" if n_steps is None else f"{name}_{steps}.npz")
    np.savez_compressed(out, **data)
    print("wrote", out, flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--long", nargs="*", default=None)
    ap.add_argument("--errors", action="store_true")
    args = ap.parse_args()
    if args.errors:
        error_fixtures()
    elif args.long is None:
        short_fixtures()
    else:
        for name in args.long or ["config1", "config2", "config3"]:
            long_fixture(name)
