"""Config 3, free run: the first step whose GPU mask differs from the
reference's, and the criterion margin of the flipped cells there.

The GPU runs the whole config-3 loop free (simulate); the first differing
step s* comes from the per-step mask CRCs the reference recorded.  The
reference's own state at s* - 1 is rebuilt by the CPU oracle (bit-identical
to the reference's step) from the nearest reference checkpoint at or before
it; one more oracle step gives the reference's criterion values of step s*
(its predictor's |eta/d|).  The margin of a flipped element is
|crit - k_nh| / k_nh of its larger node -- how close the reference itself sat
to the threshold where the GPU's state (1e-10 away after tens of thousands of
steps) landed on the other side.

    python tools/config3_margin.py > profiles/r2_config3_margin.txt
"""

import os
import sys
import zlib

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import paper_2505_17025_b200 as P  # noqa: E402
from oracle import nhswe_oracle as O  # noqa: E402
from paper_2505_17025_b200 import configs  # noqa: E402
from tests.helpers import oracle_member  # noqa: E402

G = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                         "tests", "golden", "config3_full.npz"))


def main():
    cfg = configs.config3()
    m = cfg.member(0)
    n_steps = int(G["n_steps"])
    spec = P.ScenarioSpec(cfg.name, m.grid, m.dt, n_steps * m.dt, m.bathymetry, m.bcs)
    init = P.FlowState(P.NodalField(m.grid, G["h0"]), P.NodalField(m.grid, G["hu0"]),
                       P.NodalField(m.grid, G["hw0"]), 0.0)
    res = P.simulate(spec, init, "adaptive", P.Criterion("eta_over_d"), record_masks=True)
    n = m.grid.n_elements
    gflags = []
    crc = []
    for _, _, ranges in res.mask_history:
        f = np.zeros(n, bool)
        for e0, e1 in ranges:
            f[e0:e1 + 1] = True
        gflags.append(f)
        crc.append(zlib.crc32(np.packbits(f).tobytes()))
    mism = np.flatnonzero(np.array(crc, dtype=np.uint32) != G["adaptive/flag_crc"])
    if mism.size == 0:
        print("config3 free run: every one of", n_steps, "step masks equals the reference's")
        return
    s = int(mism[0])            # mask_history index: the step from step s to s + 1
    cks = sorted(int(k[4:]) for k in G.files if k.startswith("ck/s") and int(k[4:]) <= s)
    c = cks[-1] if cks else 0
    if c:
        h, hu, hw, t = G[f"ck/s{c}"][0], G[f"ck/s{c}"][1], G[f"ck/s{c}"][2], float(G[f"ck/t{c}"])
    else:
        h, hu, hw, t = G["h0"], G["hu0"], G["hw0"], 0.0
    mem = oracle_member(m.grid, m.bathymetry, m.bcs, m.dt)
    for k in range(c, s):
        o = O.step(mem, h, hu, hw, t, "adaptive", cfl_warn=False)
        h, hu, hw, t = o.h, o.hu, o.hw, t + m.dt
        assert zlib.crc32(np.packbits(o.flags).tobytes()) == G["adaptive/flag_crc"][k]
    ph, pq, pw = O.heun(mem.grid, mem.bottom, mem.bcs, mem.g, h, hu, hw, t, m.dt, False)
    crit = O.indicator(mem.grid, mem.bottom, "eta_over_d", ph, pq, pw, t + m.dt).max(axis=1)
    ref_flags = crit > 1e-3
    assert zlib.crc32(np.packbits(ref_flags).tobytes()) == G["adaptive/flag_crc"][s]
    flipped = np.flatnonzero(ref_flags != gflags[s])
    margin = np.abs(crit[flipped] - 1e-3) / 1e-3
    print(f"config3 free run ({n_steps} steps): masks equal to the reference's for steps "
          f"1..{s}; first differing step {s + 1} (t = {t + m.dt:.6f} s)")
    print(f"  flipped elements {flipped.tolist()}: reference criterion "
          f"{crit[flipped].tolist()} vs k_nh = 1e-3")
    print(f"  relative margin |crit - k_nh| / k_nh = {margin.tolist()}")
    print(f"  (reference state rebuilt by the oracle from checkpoint {c}, "
          f"{s - c} steps, every step's mask CRC equal to the reference's)")
    print(f"  mask fraction over the run: GPU {res.mask_fraction_mean:.4f}, reference "
          f"{float(G['adaptive/mask_fraction']):.4f}")


if __name__ == "__main__":
    main()
