"""Paired adaptive/global timing and criterion sweeps on the GPU path
(reference cli.py:259-267 ``with_global`` and cli.py:320-382 ``cmd_sweep``;
the paper's Tables 5-10: t_local / t_global and accuracy per criterion x
enlargement).

* ``paired_run``       : one adaptive run and its matched global run, back to
                         back in this process, with ``time_ratio`` between them.
* ``criterion_sweep``  : the reference's sweep table -- one global run, then
                         every (criterion, enlarge) adaptive run; per row the
                         time ratio, the mean mask fraction and the accuracy
                         (solitary: final snapshot against the closed form;
                         otherwise against the global run's final eta) plus
                         per-gauge RMSE / r against the global run.
                         ``write_sweep_csv`` writes the reference's sweep.csv.
* ``ensemble_time_ratios`` : the same ratio at throughput scale -- one
                         ensemble (e.g. config 4) stepped from the same
                         initial state once per criterion variant and once
                         globally, device-timed per step.

Loop times are CUDA-event device times of the step loop (``RunResult.loop_time``),
the analogue of the reference's loop-only perf_counter (driver.py:79-94).
"""

from __future__ import annotations

import csv
import json
from pathlib import Path

import numpy as np

from paper_2505_17025_b200 import _device as D
from paper_2505_17025_b200.adaptivity import CRITERION_KINDS, Criterion
from paper_2505_17025_b200.driver import Ensemble, RunResult, simulate
from paper_2505_17025_b200.scenarios import ScenarioSpec

from .metrics import DegenerateSeriesError, RunReport, SeriesPair, pearson, rmse, time_ratio
from .paper_cases import solitary_exact

SWEEP_HEADER = ("criterion", "enlarge", "time_ratio", "mask_fraction", "rmse", "r")


def report_of(result: RunResult) -> RunReport:
    return RunReport(config=result.config_echo(), loop_time=result.loop_time,
                     mask_fraction_mean=result.mask_fraction_mean)


def paired_run(spec: ScenarioSpec, initial, criterion: Criterion):
    """Adaptive run + matched global run (reference cli.py:259-267).
    Returns (adaptive RunResult, global RunResult, t_local / t_global)."""
    local = simulate(spec, initial, "adaptive", criterion)
    glob = simulate(spec, initial, "global")
    return local, glob, time_ratio(report_of(local), report_of(glob))


def solitary_field_metrics(result: RunResult) -> tuple[float, float]:
    """Final eta against the closed-form solitary wave (reference cli.py:198-207)."""
    spec = result.spec
    d0 = spec.bathymetry.h0
    x0 = (spec.grid.x_right - spec.grid.x_left) / 4.0
    exact, _ = solitary_exact(spec.grid.nodes, result.final_state.time, d=d0, x0=x0)
    pair = SeriesPair(exact.ravel(), (result.final_state.h.values - d0).ravel())
    return rmse(pair), pearson(pair)


def _sweep_row(spec, kind, enlarge, result: RunResult, gresult: RunResult, greport) -> dict:
    row = {"criterion": kind, "enlarge": int(enlarge),
           "time_ratio": time_ratio(report_of(result), greport),
           "mask_fraction": result.mask_fraction_mean}
    if spec.name == "solitary":
        row["rmse"], row["r"] = solitary_field_metrics(result)
    else:   # accuracy against the matched global run (cli.py:356-362)
        pair = SeriesPair(gresult.final_state.h.values.ravel(),
                          result.final_state.h.values.ravel())
        row["rmse"], row["r"] = rmse(pair), pearson(pair)
    for k, x in enumerate(spec.gauges):
        pair = SeriesPair(gresult.gauge_eta[:, k], result.gauge_eta[:, k])
        row[f"rmse@{x:g}"] = rmse(pair)
        try:
            row[f"r@{x:g}"] = pearson(pair)
        except DegenerateSeriesError:
            row[f"r@{x:g}"] = ""
    return row


def criterion_sweep(spec: ScenarioSpec, initial, criteria=CRITERION_KINDS,
                    enlarge_options=(False, True), k_nh: float = 0.001,
                    keep_results: bool = False):
    """The reference's sweep (cli.py:320-382) on the GPU path.  Returns the
    rows (dicts, reference column order); with keep_results also the
    {(kind, enlarge): RunResult} map and the global RunResult."""
    criteria = list(criteria)
    for kind in criteria:
        if kind not in CRITERION_KINDS:
            raise ValueError(f"unknown criterion {kind!r}")
    rows, results, gresult = [], {}, None
    if criteria:
        gresult = simulate(spec, initial, "global")
        greport = RunReport(config=gresult.config_echo(), loop_time=gresult.loop_time,
                            mask_fraction_mean=0.0)
        for kind in criteria:
            for enlarge in enlarge_options:
                res = simulate(spec, initial, "adaptive", Criterion(kind, float(k_nh), bool(enlarge)))
                rows.append(_sweep_row(spec, kind, enlarge, res, gresult, greport))
                if keep_results:
                    results[(kind, bool(enlarge))] = res
    if keep_results:
        return rows, results, gresult
    return rows


def write_sweep_csv(path, rows, scenario: str, k_nh: float, criteria, enlarge_options) -> Path:
    """sweep.csv in the reference's layout: a '# config {json}' echo line, the
    header, one row per (criterion, enlarge) (cli.py:370-381)."""
    path = Path(path)
    header = list(rows[0]) if rows else list(SWEEP_HEADER)
    echo = {"scenario": scenario, "k_nh": float(k_nh), "criteria": list(criteria),
            "enlarge_options": [int(bool(e)) for e in enlarge_options]}
    with path.open("w", newline="") as fh:
        fh.write("# config " + json.dumps(echo, sort_keys=True) + "\n")
        w = csv.DictWriter(fh, fieldnames=header)
        w.writeheader()
        w.writerows(rows)
    return path


def ensemble_time_ratios(records: np.ndarray, h0, hu0, hw0, n_steps: int,
                         criteria=CRITERION_KINDS, enlarge_options=(False, True),
                         k_nh: float = 0.001, warmup: int = 0, time0=None):
    """t_local / t_global per (criterion, enlarge) for a whole ensemble
    (B members of N cells; h0/hu0/hw0 CUDA (B, N, 2) initial state at the
    member times time0 (CUDA (B,), default 0), all left untouched).  Every
    variant starts from a copy of the same state, runs `warmup` untimed steps, then n_steps timed by CUDA events on the current
    stream.  Returns a list of dicts with ms_per_step, mask_fraction,
    cell_steps_per_s, path and time_ratio (global row first)."""
    T = D.torch()
    B, N = int(h0.shape[0]), int(h0.shape[1])
    variants = [("global", None)] + [("adaptive", Criterion(k, float(k_nh), bool(e)))
                                     for k in criteria for e in enlarge_options]
    rows = []
    for mode, crit in variants:
        ens = Ensemble(records, h0.clone(), hu0.clone(), hw0.clone(),
                       None if time0 is None else time0.clone())
        if warmup:
            ens.advance(warmup, mode, crit)
            ens.reset_status()
        e0, e1 = T.cuda.Event(enable_timing=True), T.cuda.Event(enable_timing=True)
        T.cuda.synchronize()
        e0.record()
        ens.advance(n_steps, mode, crit)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        st = ens.check()
        frac = float(st["flagged"].sum()) / (B * N * n_steps) if n_steps else 0.0
        rows.append({"criterion": crit.kind if crit else "global",
                     "enlarge": int(crit.enlarge) if crit else 0,
                     "path": ens.choose_path(mode, crit),
                     "ms_per_step": ms / n_steps,
                     "cell_steps_per_s": B * N * n_steps / (ms * 1e-3),
                     "mask_fraction": frac})
        del ens
    tg = rows[0]["ms_per_step"]
    for r in rows:
        r["time_ratio"] = r["ms_per_step"] / tg
    return rows
