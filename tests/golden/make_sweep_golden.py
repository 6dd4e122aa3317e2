"""Golden vectors for the metrics and the criterion sweep, produced by the
REAL reference (run in the build container, where it is mounted read-only):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_sweep_golden.py

Writes tests/golden/sweep.npz:
  * metrics_*     : seeded series and the reference's rmse / pearson /
                    aligned_pair outputs on them (reference metrics.py);
  * sweep_<scen>_*: the reference CLI's own sweep table (cli.py:320-382,
                    ``nhswe sweep``) for the solitary scenario at its defaults
                    and hammack_up over a shortened run, every criterion x
                    {off, on}; time_ratio is a wall-clock number and is kept
                    only for the record, the other columns are the oracle.
Nothing here runs on the GPU box; the .npz travels.
"""

from __future__ import annotations

import csv
import io
import json
import os
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from nhswe import metrics as RM  # noqa: E402
from nhswe.cli import main as ref_main  # noqa: E402

CRITERIA = "eta_over_d,eta_x,u,u_x,w,w_x"
SWEEPS = {"solitary": ["--scenario", "solitary"],
          "hammack_up": ["--scenario", "hammack_up", "--t-end", "4",
                         "--gauges", "0.61,1.61,2.5"]}


def metrics_cases(out):
    rng = np.random.default_rng(2505)
    for k in range(8):
        n = int(rng.integers(2, 60))
        a = rng.normal(size=n) * 10 ** rng.uniform(-6, 3)
        b = a + rng.normal(size=n) * 10 ** rng.uniform(-8, 1)
        out[f"metrics_a{k}"], out[f"metrics_b{k}"] = a, b
        p = RM.SeriesPair(a, b)
        out[f"metrics_rmse{k}"] = np.float64(RM.rmse(p))
        out[f"metrics_r{k}"] = np.float64(RM.pearson(p))
    rt = np.sort(rng.uniform(0, 10, 40))
    rv = np.sin(rt)
    ct = np.linspace(1.0, 9.0, 17)
    cv = np.cos(ct)
    ap = RM.aligned_pair(rt, rv, ct, cv)
    out.update(metrics_rt=rt, metrics_rv=rv, metrics_ct=ct, metrics_cv=cv,
               metrics_al_ref=ap.reference, metrics_al_cand=ap.candidate)


def sweep_case(out, name, argv):
    with tempfile.TemporaryDirectory() as d:
        code = ref_main(["sweep", *argv, "--criteria", CRITERIA, "--enlarge-options", "off,on",
                         "--outdir", d])
        assert code == 0
        text = open(os.path.join(d, "sweep.csv")).read()
    lines = text.splitlines()
    echo = json.loads(lines[0][len("# config "):])
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[1:]))))
    cols = list(rows[0])
    out[f"sweep_{name}_argv"] = np.array(json.dumps(argv))
    out[f"sweep_{name}_echo"] = np.array(json.dumps(echo))
    out[f"sweep_{name}_header"] = np.array(",".join(cols))
    out[f"sweep_{name}_criterion"] = np.array([r["criterion"] for r in rows])
    num = [c for c in cols if c != "criterion"]
    out[f"sweep_{name}_numcols"] = np.array(",".join(num))
    out[f"sweep_{name}_values"] = np.array(
        [[float(r[c]) if r[c] != "" else np.nan for c in num] for r in rows])
    print(name, len(rows), "rows;", cols)


def main():
    out = {}
    metrics_cases(out)
    for name, argv in SWEEPS.items():
        sweep_case(out, name, argv)
    np.savez_compressed(os.path.join(HERE, "sweep.npz"), **out)
    print("wrote", os.path.join(HERE, "sweep.npz"))


if __name__ == "__main__":
    main()
