"""Golden vectors for LDG fluxes outside the alternating family, produced by
the REAL reference (FluxCoefficients, corrector.py:40-47, :205-231).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_flux_golden.py

For every flux below and the short-fixture cases of make_golden.cases():
  * ldg_solve on one range with outer traces, solve_on_ranges and
    apply_correction on several ranges (two of them touching);
  * a 12-step adaptive_step trajectory per mode (global, adaptive +
    enlargement) with the flux: final state, p and per-step flagged counts;
  * simulate() of the paper's solitary scenario (60 steps, adaptive) and, at
    polynomial order 2, apply_correction and a 10-step global trajectory.
Writes tests/golden/flux.npz (inputs are the short fixtures of short.npz).
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import nhswe as R  # noqa: E402
from nhswe import corrector as RC, hydrostatic as RH, adaptivity as RA  # noqa: E402

from tests.golden.make_golden import cases, smooth_state  # noqa: E402

FLUXES = {"central": (0.5, 0.0, 0.0), "mixed": (0.3, 0.25, 0.1), "upwind_like": (1.0, -0.25, -0.05)}
CASES = ("flat_walls", "flat_absorbing", "plate", "slope_slide")


def main():
    data = {"fluxes": np.array(list(FLUXES)), "flux_values": np.array(list(FLUXES.values())),
            "cases": np.array(CASES)}
    all_cases = {c[0]: c for c in cases()}
    for fname, (c11, c12, c22) in FLUXES.items():
        flux = RC.FluxCoefficients(c11, c12, c22)
        for name in CASES:
            _, grid, bathy, _, bcs, dt, st = all_cases[name]
            p = f"{fname}/{name}/"
            pred = RH.heun_step(st, dt, bathy, bcs, cfl_warn=False)
            co = RC.assemble_coefficients(pred, bathy, dt)
            n = grid.n_elements
            pr, hr = RC.ldg_solve(co, (3, n // 2), (0.2, -0.3), flux)
            data[p + "ldg_p"], data[p + "ldg_hu"] = pr, hr
            ranges = ((0, n // 4), (n // 4 + 1, n // 2), (n // 2 + 3, n // 2 + 3), (n - 4, n - 1))
            data[p + "ranges"] = np.array(ranges)
            sol = RC.solve_on_ranges(pred, co, ranges, bcs, flux)
            data[p + "sor"] = np.stack([sol.p_nh.values, sol.hu_corrected.values])
            corr, sol2 = RC.apply_correction(pred, bathy, dt, ranges, bcs, flux)
            data[p + "corr"] = np.stack([corr.hu.values, corr.hw.values, sol2.p_nh.values])
            for mode, crit in (("global", None), ("adaptive", RA.Criterion("eta_over_d", 1e-3, True))):
                s, counts, pn = st, [], None
                for _ in range(12):
                    r = RA.adaptive_step(s, dt, bathy, bcs, mode=mode, crit=crit, flux=flux,
                                         cfl_warn=False)
                    s = r.state
                    counts.append(int(r.mask.flags.sum()))
                    pn = r.p_nh
                data[p + mode] = np.stack([s.h.values, s.hu.values, s.hw.values])
                data[p + mode + "_counts"] = np.array(counts)
                if pn is not None:
                    data[p + mode + "_p"] = pn.values
        # the paper's solitary scenario through simulate()
        spec, init = R.build_scenario("solitary")
        spec = R.ScenarioSpec(spec.name, spec.grid, spec.dt, 60 * spec.dt, spec.bathymetry, spec.bcs,
                              spec.gauges, spec.g)
        res = R.simulate(spec, init, "adaptive", RA.Criterion("eta_over_d"), flux=flux)
        fs = res.final_state
        data[f"{fname}/simulate"] = np.stack([fs.h.values, fs.hu.values, fs.hw.values])
        data[f"{fname}/simulate_frac"] = np.array(res.mask_fraction_mean)
        data[f"{fname}/simulate_gauges"] = res.gauge_eta
        # order p = 2
        g2 = R.GridSpec(0.0, 100.0, 40, poly_order=2)
        st2 = smooth_state(g2)
        b2 = R.FlatBottom(10.0)
        bc2 = R.BoundaryPair(R.WALL, R.ABSORBING)
        pred2 = RH.heun_step(st2, 0.05, b2, bc2, cfl_warn=False)
        data[f"{fname}/p2/state0"] = np.stack([st2.h.values, st2.hu.values, st2.hw.values])
        data[f"{fname}/p2/pred"] = np.stack([pred2.h.values, pred2.hu.values, pred2.hw.values])
        r2 = ((1, 12), (13, 20), (30, 39))
        corr, sol = RC.apply_correction(pred2, b2, 0.05, r2, bc2, flux)
        data[f"{fname}/p2/corr"] = np.stack([corr.hu.values, corr.hw.values, sol.p_nh.values])
        s = st2
        for _ in range(10):
            s = RA.adaptive_step(s, 0.05, b2, bc2, mode="global", flux=flux, cfl_warn=False).state
        data[f"{fname}/p2/global"] = np.stack([s.h.values, s.hu.values, s.hw.values])
        print(fname, "done", flush=True)
    np.savez_compressed(os.path.join(HERE, "flux.npz"), **data)
    print("wrote flux.npz")


if __name__ == "__main__":
    main()
