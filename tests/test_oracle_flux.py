"""The CPU oracle with LDG fluxes outside the alternating family against the
REAL reference's outputs (tests/golden/flux.npz, made by
tests/golden/make_flux_golden.py): corrector.py:40-47, :205-231."""

import os

import numpy as np
import pytest

from oracle import nhswe_oracle as O
from tests.oracle_cases import GOLDEN, load_short, member_from, state_from
from tests.test_oracle_golden import close

D = load_short()
F = np.load(os.path.join(GOLDEN, "flux.npz"))
FLUXES = {str(n): tuple(float(x) for x in v) for n, v in zip(F["fluxes"], F["flux_values"])}
CASES = [str(c) for c in F["cases"]]


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("flux", list(FLUXES))
def test_correction_general_flux(flux, case):
    c11, c12, c22 = FLUXES[flux]
    m = member_from(D, case)
    h, hu, hw = state_from(D, case)
    ph, pq, pw = O.heun(m.grid, m.bottom, m.bcs, 9.81, h, hu, hw, 0.0, m.dt, cfl_warn=False)
    key = f"{flux}/{case}/"
    ranges = tuple(tuple(int(v) for v in r) for r in F[key + "ranges"])
    q2, w2, p = O.correction(m.grid, m.bottom, m.bcs, 9.81, 1000.0, ph, pq, pw, m.dt, m.dt,
                             ranges, c11, c12, c22)
    ref = F[key + "corr"]
    assert close(q2, ref[0], 1e-12) and close(w2, ref[1], 1e-12) and close(p, ref[2], 1e-12)


@pytest.mark.parametrize("mode", ["global", "adaptive"])
@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("flux", list(FLUXES))
def test_trajectory_general_flux(flux, case, mode):
    c11, c12, c22 = FLUXES[flux]
    m = member_from(D, case)
    h, hu, hw = state_from(D, case)
    t, counts = 0.0, []
    for _ in range(12):
        o = O.step(m, h, hu, hw, t, mode, "eta_over_d", 1e-3, mode == "adaptive", c11=c11,
                   c12=c12, c22=c22, cfl_warn=False)
        h, hu, hw = o.h, o.hu, o.hw
        t += m.dt
        counts.append(int(o.flags.sum()))
    key = f"{flux}/{case}/{mode}"
    assert counts == list(F[key + "_counts"])
    for a, b in zip((h, hu, hw), F[key]):
        assert close(a, b, 1e-12)
