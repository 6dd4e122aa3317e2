"""Paper scenarios (one member each) on both step implementations: loop time
of the whole run for the resident cluster kernel and the streaming tiles
(CUDA-graph time loop), global and adaptive.

    python tools/scenario_paths.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2505_17025_b200 as P  # noqa: E402
from tests.harness import paper_cases
from paper_2505_17025_b200 import _device as D  # noqa: E402

from paper_2505_17025_b200 import configs  # noqa: E402
from tests.helpers import oracle_depth  # noqa: E402


def cases():
    for name in ("solitary", "hammack_up", "whittaker"):
        yield (name,) + paper_cases.build_scenario(name) + (("global", "adaptive"),)
    for name in ("config1", "config2", "config3"):
        cfg = configs.get(name)
        m = cfg.member(0)
        h, hu, hw = cfg.host_state(0, oracle_depth)
        spec = P.ScenarioSpec(name, m.grid, m.dt, cfg.n_steps * m.dt, m.bathymetry, m.bcs)
        init = P.FlowState(P.NodalField(m.grid, h), P.NodalField(m.grid, hu),
                           P.NodalField(m.grid, hw), 0.0)
        yield name, spec, init, cfg.modes


for name, spec, init, modes in cases():
    rec = D.member_record(spec.grid, spec.bathymetry, spec.bcs, spec.dt)
    for mode in modes:
        crit = P.Criterion("eta_over_d", 1e-3, enlarge=(name == "whittaker"))
        for path in ("resident", "stream"):
            ts = []
            for rep in range(3 if spec.n_steps < 20000 else 1):
                ens = P.Ensemble.from_host(rec, init.h.values[None], init.hu.values[None],
                                           init.hw.values[None])
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                ens.advance(spec.n_steps, mode, crit, path=path)
                e1.record()
                e1.synchronize()
                ens.check()
                ts.append(e0.elapsed_time(e1))
            print(f"{name:11s} {mode:8s} {path:8s} N={spec.grid.n_elements:5d} steps={spec.n_steps:5d}: "
                  f"{min(ts):8.2f} ms ({1e3 * min(ts) / spec.n_steps:6.2f} us/step)", flush=True)
