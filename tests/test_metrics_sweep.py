"""Host-side metrics and sweep-table plumbing (no GPU): the reference's metric
tests (pkg/tests/test_metrics.py) re-pointed at paper_2505_17025_b200.metrics,
the metrics pinned to the reference's own outputs (tests/golden/sweep.npz),
and the sweep.csv layout of the reference CLI (pkg/tests/test_cli.py:92-108)."""

import json
import os

import numpy as np
import pytest

from tests.harness.metrics import (DegenerateSeriesError, RunReport, SeriesPair,
                                           aligned_pair, pearson, rmse, time_ratio)
from tests.harness.sweep import SWEEP_HEADER, write_sweep_csv

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "sweep.npz"))


def test_rmse_hand_values():
    assert rmse(SeriesPair([1.0, 2.0, 3.0], [1.0, 2.0, 3.0])) == 0.0
    assert rmse(SeriesPair([0.0, 0.0], [0.01, 0.01])) == pytest.approx(0.01)
    assert rmse(SeriesPair([1, 2, 3], [1, 2, 5])) == pytest.approx(np.sqrt(4.0 / 3.0))


def test_pearson_hand_values_and_degenerate():
    a = np.array([1.0, 2.0, 3.0])
    assert pearson(SeriesPair(a, a)) == pytest.approx(1.0)
    assert pearson(SeriesPair(a, -a)) == pytest.approx(-1.0)
    assert pearson(SeriesPair(a, np.array([1.0, 2.0, 4.0]))) == pytest.approx(0.9820, abs=1e-4)
    with pytest.raises(DegenerateSeriesError):
        pearson(SeriesPair([1.0, 1.0, 1.0], [1.0, 2.0, 3.0]))


def test_series_pair_validation():
    for a, b in (([1.0], [1.0]), ([1.0, 2.0], [1.0, 2.0, 3.0]), ([1.0, np.nan], [1.0, 2.0])):
        with pytest.raises(ValueError):
            SeriesPair(a, b)


def test_metrics_match_reference_golden():
    for k in range(8):
        p = SeriesPair(GOLD[f"metrics_a{k}"], GOLD[f"metrics_b{k}"])
        assert rmse(p) == float(GOLD[f"metrics_rmse{k}"])
        assert pearson(p) == float(GOLD[f"metrics_r{k}"])
    ap = aligned_pair(GOLD["metrics_rt"], GOLD["metrics_rv"], GOLD["metrics_ct"],
                      GOLD["metrics_cv"])
    assert np.array_equal(ap.reference, GOLD["metrics_al_ref"])
    assert np.array_equal(ap.candidate, GOLD["metrics_al_cand"])
    with pytest.raises(ValueError, match="overlap"):
        aligned_pair([0.0, 1.0], [0.0, 1.0], [10.0, 11.0], [0.0, 0.0])


def test_time_ratio_and_config_matching():
    cfg = {"scenario": "solitary", "dt": 0.1, "n_elements": 200, "poly_order": 1, "t_end": 30.0}
    local = RunReport(config=cfg, loop_time=1.0, mask_fraction_mean=0.2)
    glob = RunReport(config=dict(cfg), loop_time=4.0, mask_fraction_mean=1.0)
    assert time_ratio(local, glob) == pytest.approx(0.25)
    with pytest.raises(ValueError, match="dt"):
        time_ratio(local, RunReport(config={**cfg, "dt": 0.05}, loop_time=4.0,
                                    mask_fraction_mean=1.0))
    with pytest.raises(ValueError):
        time_ratio(local, RunReport(config=dict(cfg), loop_time=0.0, mask_fraction_mean=1.0))


def test_run_report_json_keys():
    r = RunReport(config={"scenario": "solitary"}, loop_time=1.5, mask_fraction_mean=0.3,
                  gauge_rmse={"eta@1": 0.01}, gauge_r={"eta@1": 0.999}, time_ratio=0.4,
                  extra={"note": 1})
    doc = json.loads(r.to_json())
    assert doc["time_ratio_local_over_global"] == 0.4
    assert doc["loop_time_s"] == 1.5 and doc["note"] == 1
    assert "time_ratio_local_over_global" not in json.loads(
        RunReport(config={}, loop_time=1.0, mask_fraction_mean=0.0).to_json())


def test_sweep_csv_layout(tmp_path):
    """Empty criterion list: echo + header only; otherwise one row per
    (criterion, enlarge), header in the reference's column order."""
    p = write_sweep_csv(tmp_path / "sweep.csv", [], "solitary", 1e-3, [], [False, True])
    lines = p.read_text().splitlines()
    assert len(lines) == 2 and lines[0].startswith("# config ")
    assert lines[1] == ",".join(SWEEP_HEADER)
    rows = [{"criterion": k, "enlarge": e, "time_ratio": 0.5, "mask_fraction": 0.1,
             "rmse": 0.01, "r": 0.99} for k in ("eta_over_d", "u") for e in (0, 1)]
    lines = write_sweep_csv(tmp_path / "s2.csv", rows, "solitary", 1e-3, ["eta_over_d", "u"],
                            [False, True]).read_text().splitlines()
    assert len(lines) == 2 + 4 and lines[1].startswith("criterion,enlarge,time_ratio")
    echo = json.loads(lines[0][len("# config "):])
    assert echo == json.loads(str(GOLD["sweep_solitary_echo"])) | {"criteria": ["eta_over_d", "u"]}
    assert str(GOLD["sweep_solitary_header"]) == ",".join(SWEEP_HEADER)
