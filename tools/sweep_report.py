"""GPU criterion sweeps (the paper's Tables 5-10 analogue).

  python tools/sweep_report.py [--members 4096] [--cells 4096] [--steps 200] [--warmup 1000]

1. The reference CLI's sweep on its own scenarios (solitary at defaults,
   hammack_up), through paper_2505_17025_b200.criterion_sweep: per
   (criterion, enlarge) the GPU t_local / t_global, mask fraction and
   accuracy columns.
2. The same ratio at throughput scale: a config-4 ensemble stepped from the
   same state (after `warmup` adaptive steps so the waves have formed) once
   globally and once per (criterion, enlarge) -- ensemble_time_ratios.
"""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2505_17025_b200 as P  # noqa: E402
from tests.harness import paper_cases
from paper_2505_17025_b200 import _device as D, configs  # noqa: E402
from tests.harness.sweep import criterion_sweep, ensemble_time_ratios  # noqa: E402


def table(rows, cols):
    out = ["  ".join(f"{c:>13s}" for c in cols)]
    for r in rows:
        out.append("  ".join(f"{r[c]:>13.5g}" if isinstance(r[c], float) else f"{str(r[c]):>13s}"
                             for c in cols))
    return "\n".join(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--members", type=int, default=4096)
    ap.add_argument("--cells", type=int, default=4096)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=1000)
    a = ap.parse_args()
    cols = ["criterion", "enlarge", "time_ratio", "mask_fraction", "rmse", "r"]
    for name, over, gauges in (("solitary", {}, None),
                               ("hammack_up", {"t_end": 4.0}, (0.61, 1.61, 2.5))):
        spec, init = paper_cases.build_scenario(name, **over)
        if gauges:
            from dataclasses import replace
            spec = replace(spec, gauges=gauges)
        criterion_sweep(spec, init, ["eta_over_d"], (False,))    # warm the code paths
        rows = criterion_sweep(spec, init)
        print(f"== {name}: {spec.n_steps} steps of {spec.grid.n_elements} elements "
              f"(reference CLI sweep, GPU path)")
        print(table(rows, cols))
    cfg = configs.Config4(n_members=a.members, n_elements=a.cells)
    recs = cfg.records()
    st = [cfg.host_state(i, lambda m, x, t: m.depth(x, t)) for i in range(cfg.n_members)]
    H, Q, W = (D.dev(np.stack([s[k] for s in st])) for k in range(3))
    t0 = None
    if a.warmup:
        ens = P.Ensemble(recs, H, Q, W)
        ens.advance(a.warmup, "adaptive", P.Criterion("eta_over_d"))
        ens.check()
        H, Q, W, t0 = ens.h, ens.hu, ens.hw, ens.time
    rows = ensemble_time_ratios(recs, H, Q, W, a.steps, time0=t0)
    print(f"== config-4 ensemble {a.members} x {a.cells}, state after {a.warmup} adaptive steps, "
          f"{a.steps} timed steps per variant")
    print(table(rows, ["criterion", "enlarge", "path", "ms_per_step", "cell_steps_per_s",
                       "mask_fraction", "time_ratio"]))


if __name__ == "__main__":
    main()
