"""Criterion sweep and paired timing on the GPU (reference
cli.py:259-267 ``with_global``, cli.py:320-382 ``sweep``).

The sweep tables the reference CLI itself wrote (tests/golden/sweep.npz,
tests/golden/make_sweep_golden.py) are the oracle: every (criterion,
enlarge) row's mask fraction, snapshot accuracy and per-gauge RMSE / r must
match the reference's; time_ratio is a wall-clock ratio and is only checked
for sanity (the GPU's numbers are reported)."""

import json
import os

import numpy as np
import pytest

import paper_2505_17025_b200 as P
from tests.harness import paper_cases
from paper_2505_17025_b200 import configs
from tests.harness.sweep import (criterion_sweep, ensemble_time_ratios, paired_run,
                                         write_sweep_csv)

pytestmark = pytest.mark.gpu

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "sweep.npz"))
KINDS = list(P.CRITERION_KINDS)


def scenario_from_argv(argv):
    """The reference CLI's build_run for the sweep's argv (cli.py:91-136)."""
    a = dict(zip(argv[::2], argv[1::2]))
    over = {}
    if "--t-end" in a:
        over["t_end"] = float(a["--t-end"])
    spec, init = paper_cases.build_scenario(a["--scenario"], **over)
    if "--gauges" in a:
        from dataclasses import replace
        spec = replace(spec, gauges=tuple(float(x) for x in a["--gauges"].split(",")))
    return spec, init


@pytest.mark.parametrize("name", ["solitary", "hammack_up"])
def test_sweep_matches_reference_table(name, tmp_path):
    argv = json.loads(str(GOLD[f"sweep_{name}_argv"]))
    spec, init = scenario_from_argv(argv)
    rows = criterion_sweep(spec, init, KINDS, (False, True), 0.001)
    cols = str(GOLD[f"sweep_{name}_numcols"]).split(",")
    ref = GOLD[f"sweep_{name}_values"]
    assert [r["criterion"] for r in rows] == list(GOLD[f"sweep_{name}_criterion"])
    assert ",".join(rows[0]) == str(GOLD[f"sweep_{name}_header"])
    worst = {}
    for i, r in enumerate(rows):
        for j, c in enumerate(cols):
            v, rv = r[c], ref[i, j]
            if c == "time_ratio":   # a timing, not a parity column: positive and finite
                assert 0.0 < v < 100.0
                continue
            if np.isnan(rv):
                assert v == "", (r["criterion"], r["enlarge"], c)
                continue
            err = abs(v - rv) / max(abs(rv), 1e-300)
            worst[c] = max(worst.get(c, 0.0), err)
            tol = 1e-12 if c == "mask_fraction" else 1e-6
            assert err <= tol, (r["criterion"], r["enlarge"], c, v, rv)
    print(f"{name}: worst relative difference per column vs the reference's sweep.csv: "
          + ", ".join(f"{c} {e:.1e}" for c, e in worst.items()))
    print(f"{name}: GPU time ratios " + ", ".join(
        f"{r['criterion']}/{r['enlarge']} {r['time_ratio']:.2f}" for r in rows))
    path = write_sweep_csv(tmp_path / "sweep.csv", rows, name, 0.001, KINDS, (False, True))
    lines = path.read_text().splitlines()
    assert len(lines) == 2 + len(rows)


def test_paired_run_time_ratio():
    spec, init = paper_cases.build_solitary(t_end=5.0)
    local, glob, ratio = paired_run(spec, init, P.Criterion("eta_over_d", 0.001))
    assert ratio == pytest.approx(local.loop_time / glob.loop_time)
    assert glob.mask_fraction_mean == 1.0 and 0.0 < local.mask_fraction_mean < 1.0


def test_ensemble_time_ratios_rows():
    cfg = configs.Config4(n_members=64, n_elements=1024, n_steps=40)
    recs = cfg.records()
    st = [cfg.host_state(i, lambda mdl, x, t: mdl.depth(x, t)) for i in range(cfg.n_members)]
    H, Q, W = (P.driver.D.dev(np.stack([s[k] for s in st])) for k in range(3))
    rows = ensemble_time_ratios(recs, H, Q, W, 40, ["eta_over_d", "u_x", "w_x"], (False, True))
    assert len(rows) == 1 + 3 * 2
    assert rows[0]["criterion"] == "global" and rows[0]["time_ratio"] == 1.0
    assert rows[0]["mask_fraction"] == 1.0
    for r in rows[1:]:
        assert 0.0 <= r["mask_fraction"] <= 1.0 and r["ms_per_step"] > 0.0
        assert r["path"] == "stream"
    # the initial state is left untouched for the next variant
    assert np.array_equal(H.cpu().numpy(), np.stack([s[0] for s in st]))
