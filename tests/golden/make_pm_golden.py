"""Golden vectors for polynomial orders p = 2, 3, produced by
the REAL reference (run in the build container, where it is mounted read-only):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_pm_golden.py

Writes tests/golden/pm.npz.  Per case: the grid / bottom / boundary /
dt parameters, the initial state, the reference's own rhs_operator and
criterion_values (all six kinds) on it, and a short trajectory of the
reference's adaptive_step in one mode (final state, final p_nh, per-step
flagged-element counts).  The GPU tests rebuild the same inputs through the
package's mirrors of the reference constructors.  Nothing here runs on the
GPU box; the .npz travels.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from nhswe.adaptivity import CRITERION_KINDS, Criterion, adaptive_step, criterion_values  # noqa: E402
from nhswe.bathymetry import FlatBottom, HammackPlate  # noqa: E402
from nhswe.grid import FlowState, GridSpec, NodalField  # noqa: E402
from nhswe.hydrostatic import ABSORBING, WALL, BoundaryPair, rhs_operator  # noqa: E402
from nhswe.scenarios import vertical_momentum_from_constraint  # noqa: E402

BCS = {"wall": WALL, "absorbing": ABSORBING}


def bottom_of(spec):
    if spec["bottom"] == "flat":
        return FlatBottom(spec["h0"])
    return HammackPlate(spec["h0"], spec["zeta0"], spec["b"], spec["t_c"])


def initial(spec, grid, bathy):
    x = grid.nodes
    d = bathy.sample(grid.sample_nodes, 0.0).d
    if spec["init"] == "rest":
        return d.copy(), np.zeros_like(d), np.zeros_like(d)
    a, x0, w = spec["a"], spec["x0"], spec["w"]
    eta = a / np.cosh((x - x0) / w) ** 2
    h = d + eta
    hu = h * np.sqrt(9.81 / spec["h0"]) * eta
    hw = vertical_momentum_from_constraint(grid, h, hu, bathy, 0.0)
    return h, hu, hw


CASES = {
    "p2_flat_global": dict(p=2, n=48, xl=0.0, xr=30.0, bottom="flat", h0=1.0, init="bump",
                           a=0.1, x0=12.0, w=2.0, bcs=("wall", "absorbing"), dt=0.01, steps=40,
                           mode="global"),
    "p2_flat_adaptive": dict(p=2, n=48, xl=0.0, xr=30.0, bottom="flat", h0=1.0, init="bump",
                             a=0.1, x0=12.0, w=2.0, bcs=("wall", "absorbing"), dt=0.01,
                             steps=40, mode="adaptive", kind="eta_over_d", k_nh=1e-3,
                             enlarge=False),
    "p3_flat_adaptive_enl": dict(p=3, n=40, xl=0.0, xr=30.0, bottom="flat", h0=1.0,
                                 init="bump", a=0.15, x0=15.0, w=1.5,
                                 bcs=("absorbing", "absorbing"), dt=0.006, steps=40,
                                 mode="adaptive", kind="eta_over_d", k_nh=1e-3, enlarge=True),
    "p2_flat_hydrostatic": dict(p=2, n=48, xl=0.0, xr=30.0, bottom="flat", h0=1.0, init="bump",
                                a=0.1, x0=12.0, w=2.0, bcs=("wall", "wall"), dt=0.01, steps=40,
                                mode="hydrostatic"),
    "p2_plate_adaptive": dict(p=2, n=60, xl=0.0, xr=3.0, bottom="plate", h0=0.05, zeta0=0.005,
                              b=0.3, t_c=0.08, init="rest", bcs=("wall", "absorbing"),
                              dt=0.002, steps=60, mode="adaptive", kind="eta_over_d", k_nh=1e-3,
                              enlarge=False),
    "p3_plate_global": dict(p=3, n=40, xl=0.0, xr=3.0, bottom="plate", h0=0.05, zeta0=0.005,
                            b=0.3, t_c=0.08, init="rest", bcs=("wall", "absorbing"),
                            dt=0.0015, steps=60, mode="global"),
    "p2_plate_wx": dict(p=2, n=60, xl=0.0, xr=3.0, bottom="plate", h0=0.05, zeta0=0.005,
                        b=0.3, t_c=0.08, init="rest", bcs=("wall", "absorbing"), dt=0.002,
                        steps=40, mode="adaptive", kind="w_x", k_nh=1e-3, enlarge=True),
}


CORR = {"p2_flat_adaptive": [(3, 14), (20, 31)], "p3_plate_global": [(0, 9), (15, 39)]}


def run_case(name, spec, out):
    grid = GridSpec(spec["xl"], spec["xr"], spec["n"], spec["p"])
    bathy = bottom_of(spec)
    bcs = BoundaryPair(BCS[spec["bcs"][0]], BCS[spec["bcs"][1]])
    h, hu, hw = initial(spec, grid, bathy)
    st = FlowState(NodalField(grid, h), NodalField(grid, hu), NodalField(grid, hw), 0.0)
    out[f"{name}_spec"] = np.array(json.dumps(spec))
    out[f"{name}_h0"], out[f"{name}_hu0"], out[f"{name}_hw0"] = h, hu, hw
    t1, t2, t3 = rhs_operator(st, bathy, bcs)
    out[f"{name}_rhs"] = np.stack([t1, t2, t3])
    out[f"{name}_crit"] = np.stack([criterion_values(st, bathy, k) for k in CRITERION_KINDS])
    crit = (Criterion(spec["kind"], spec["k_nh"], spec["enlarge"])
            if spec["mode"] == "adaptive" else None)
    counts, p = [], None
    for _ in range(spec["steps"]):
        r = adaptive_step(st, spec["dt"], bathy, bcs, mode=spec["mode"], crit=crit,
                          cfl_warn=False)
        counts.append(int(r.mask.flags.sum()))
        st = r.state
        p = r.p_nh
    out[f"{name}_h"], out[f"{name}_hu"], out[f"{name}_hw"] = (st.h.values, st.hu.values,
                                                             st.hw.values)
    out[f"{name}_t"] = np.float64(st.time)
    out[f"{name}_p"] = p.values if p is not None else np.zeros_like(h)
    out[f"{name}_counts"] = np.array(counts)
    if name in CORR:   # apply_correction on given ranges, the final state as predictor
        from nhswe.corrector import apply_correction
        cst, sol = apply_correction(st, bathy, spec["dt"], CORR[name], bcs)
        out[f"{name}_corr_ranges"] = np.array(CORR[name])
        out[f"{name}_corr_hu"], out[f"{name}_corr_hw"] = cst.hu.values, cst.hw.values
        out[f"{name}_corr_p"] = sol.p_nh.values
        # the coefficient-level functions on the same predictor (corrector.py:100-482)
        from nhswe.corrector import (assemble_coefficients, correct_momentum, ldg_solve,
                                     solve_on_ranges)
        co = assemble_coefficients(st, bathy, spec["dt"])
        out[f"{name}_coef"] = np.stack([co.s11, co.s12, co.s22, co.f1, co.f2, co.phi])
        lo, hi = CORR[name][0][0], CORR[name][-1][1]
        cw = assemble_coefficients(st, bathy, spec["dt"], window=slice(lo, hi + 1))
        out[f"{name}_coefw"] = np.stack([cw.s11, cw.s12, cw.s22, cw.f1, cw.f2, cw.phi])
        e0, e1 = CORR[name][0]
        pl, hl = ldg_solve(co, (e0, e1), outer_hu=(0.0, 0.37))
        out[f"{name}_ldg_p"], out[f"{name}_ldg_hu"] = pl, hl
        sol2 = solve_on_ranges(st, co, CORR[name], bcs)
        out[f"{name}_sor_p"], out[f"{name}_sor_hu"] = sol2.p_nh.values, sol2.hu_corrected.values
        cm = correct_momentum(st, sol2, co)
        out[f"{name}_cm_hw"] = cm.hw.values
    print(f"{name}: {spec['steps']} steps, flagged per step {counts[:3]}...{counts[-3:]}, "
          f"|hw| {np.abs(st.hw.values).max():.3e}")


def grid_ops(out):
    """The reference GridSpec's m-node operators, p = 1..3 (grid.py:71-114)."""
    for p in (1, 2, 3):
        g = GridSpec(0.0, 30.0, 48, p)
        for f in ("ref_nodes", "nodes", "sample_nodes", "mass", "stiffness", "deriv_ref",
                  "weak_div", "lift_left", "lift_right"):
            out[f"grid_p{p}_{f}"] = np.asarray(getattr(g, f))


SIMS = {   # full simulate() runs of the paper scenarios at p = 2, 3 (driver.py:50-103)
    "sim_solitary_p2": dict(scenario="solitary", over=dict(poly_order=2, n_elements=120,
                                                           dt=0.05, t_end=15.0),
                            gauges=(150.0, 260.0), mode="adaptive", kind="eta_over_d",
                            enlarge=True),
    "sim_solitary_p3": dict(scenario="solitary", over=dict(poly_order=3, n_elements=100,
                                                           dt=0.04, t_end=8.0),
                            gauges=(200.0,), mode="global"),
    "sim_hammack_p2": dict(scenario="hammack_up", over=dict(poly_order=2, dx=0.05, dt=0.004,
                                                            t_end=2.0),
                           gauges=(0.61, 1.61), mode="adaptive", kind="eta_over_d",
                           enlarge=False),
}


def sim_case(name, c, out):
    from dataclasses import replace

    from nhswe.driver import simulate
    from nhswe.scenarios import build_scenario
    spec, init = build_scenario(c["scenario"], **c["over"])
    spec = replace(spec, gauges=tuple(c["gauges"]))
    crit = Criterion(c["kind"], 1e-3, c["enlarge"]) if c["mode"] == "adaptive" else None
    r = simulate(spec, init, c["mode"], crit)
    out[f"{name}_cfg"] = np.array(json.dumps(c))
    out[f"{name}_h"], out[f"{name}_hu"], out[f"{name}_hw"] = (r.final_state.h.values,
                                                             r.final_state.hu.values,
                                                             r.final_state.hw.values)
    out[f"{name}_gauge_eta"] = r.gauge_eta
    out[f"{name}_gauge_t"] = r.gauge_times
    out[f"{name}_frac"] = np.float64(r.mask_fraction_mean)
    print(f"{name}: {spec.n_steps} steps, mask fraction {r.mask_fraction_mean:.4f}")


def main():
    out = {"cases": np.array(json.dumps(list(CASES))), "sims": np.array(json.dumps(list(SIMS)))}
    grid_ops(out)
    for name, c in SIMS.items():
        sim_case(name, c, out)
    for name, spec in CASES.items():
        run_case(name, spec, out)
    np.savez_compressed(os.path.join(HERE, "pm.npz"), **out)
    print("wrote", os.path.join(HERE, "pm.npz"))


if __name__ == "__main__":
    main()
