"""GPU path against the REAL reference's golden vectors (tests/golden/*.npz,
made by tests/golden/make_golden.py from /root/reference).

Short fixtures: every hot-path function on six scenario families.  Long
fixtures: BASELINE configs 1-3 run to their final time by the reference's own
`simulate`; the GPU runs the same loop in one fused launch and must agree to
1e-9 relative L-inf in eta and hu at the final time, with per-step masks
identical except where the criterion sits within a hair of k_nh (counted and
reported).
"""

import os
import zlib

import numpy as np
import pytest

import paper_2505_17025_b200 as P
from paper_2505_17025_b200 import _device as D_, configs
from tests.oracle_cases import GOLDEN, NAMES, load_short

pytestmark = pytest.mark.gpu
D = load_short()


def pkg_case(name):
    xl, xr, n = D[name + "/grid"]
    g = P.GridSpec(float(xl), float(xr), int(n))
    kind = str(D[name + "/bottom_kind"])
    p = D[name + "/bottom"]
    if kind == "flat":
        b = P.FlatBottom(p[1])
    elif kind == "plate":
        b = P.HammackPlate(*p[1:5])
    elif kind == "quartic":
        b = P.WhittakerSlide(p[1], p[2], p[3], P.SlideMotion(*p[4:9]), p[9])
    elif kind == "smooth_box":
        b = P.SmoothBoxPlate(*p[1:6])
    else:
        b = P.SlopeGaussianSlide(*p[1:10])
    bc = [P.BoundaryCondition(str(k)) for k in D[name + "/bcs"]]
    st = P.FlowState(P.NodalField(g, D[name + "/h0"]), P.NodalField(g, D[name + "/hu0"]),
                     P.NodalField(g, D[name + "/hw0"]), 0.0)
    return g, b, P.BoundaryPair(*bc), float(D[name + "/dt"]), st


def rel(a, b):
    return float(np.abs(np.asarray(a) - b).max() / max(np.abs(b).max(), 1e-300))


@pytest.mark.parametrize("name", NAMES)
def test_functions_vs_reference(name):
    g, b, bcs, dt, st = pkg_case(name)
    pred = P.heun_step(st, dt, b, bcs, cfl_warn=False)
    ref = D[name + "/heun"]
    assert rel(pred.h.values, ref[0]) < 1e-13
    assert np.abs(pred.hu.values - ref[1]).max() < 1e-12 * max(np.abs(ref[1]).max(), 1e-3)
    for kind in P.CRITERION_KINDS:
        v = P.criterion_values(pred, b, kind)
        r = D[name + "/crit_" + kind]
        assert np.abs(v - r).max() <= 1e-10 * max(np.abs(r).max(), 1e-12)
    ranges = tuple(tuple(int(x) for x in r) for r in D[name + "/corr_ranges"])
    predr = P.FlowState(P.NodalField(g, ref[0]), P.NodalField(g, ref[1]),
                        P.NodalField(g, ref[2]), dt)
    corr, sol = P.apply_correction(predr, b, dt, ranges, bcs)
    cr = D[name + "/corr"]
    assert rel(corr.hu.values, cr[0]) < 1e-10
    assert np.abs(corr.hw.values - cr[1]).max() <= 1e-9 * max(np.abs(cr[1]).max(), 1e-9)
    assert np.abs(sol.p_nh.values - cr[2]).max() <= 1e-9 * max(np.abs(cr[2]).max(), 1e-9)


@pytest.mark.parametrize("mode", ["hydrostatic", "global", "adaptive", "adaptive_enl",
                                  "adaptive_wx"])
@pytest.mark.parametrize("name", NAMES)
def test_trajectories_vs_reference(name, mode):
    g, b, bcs, dt, st = pkg_case(name)
    crit = {"adaptive": P.Criterion("eta_over_d"),
            "adaptive_enl": P.Criterion("eta_over_d", 1e-3, True),
            "adaptive_wx": P.Criterion("w_x")}.get(mode)
    flags = []
    for _ in range(12):
        r = P.adaptive_step(st, dt, b, bcs, mode=mode.split("_")[0], crit=crit, cfl_warn=False)
        st = r.state
        flags.append(r.mask.flags)
    ref_flags = D[name + "/traj_" + mode + "_flags"]
    assert np.array_equal(np.array(flags), ref_flags)
    ref = D[name + "/traj_" + mode]
    assert rel(st.h.values, ref[0]) < 1e-12
    assert np.abs(st.hu.values - ref[1]).max() <= 1e-10 * max(np.abs(ref[1]).max(), 1e-6)
    assert np.abs(st.hw.values - ref[2]).max() <= 1e-9 * max(np.abs(ref[2]).max(), 1e-6)


def test_manufactured_solve_vs_reference():
    n = 48
    g = P.GridSpec(0.0, 1.0, n)
    s11, s12, s22, f1, f2 = D["manufactured/coef"]
    z = np.zeros_like(s11)
    co = P.EllipticCoefficients(g, s11, s12, -s11, s22, f1, f2, z, P.BottomSample(*(z,) * 6),
                                0.1, 1.0)
    p, hu = P.ldg_solve(co, (3, 40), outer_hu=tuple(D["manufactured/outer"]))
    ref = D["manufactured/solution"]
    assert rel(p, ref[0]) < 1e-12 and rel(hu, ref[1]) < 1e-12


LONG = [(c, m) for c in ("config1", "config2", "config3")
        for m in configs.get(c).modes]

# Config 3's reference solution is dynamically sensitive after the slide stops
# (t_stop = 1.96 s): a perturbation of the size of one step's solve
# difference (LAPACK's pivoted band LU vs the condensed chain, ~1e-14) grows
# until, tens of thousands of steps later, a near-threshold criterion value
# flips and the run follows another trajectory -- the reference's own
# arithmetic does the same under a 1e-10 kick (config3_kicked.npz).  Parity
# over the whole run is therefore checked in WINDOWS: the GPU restarts from
# every reference checkpoint (make_golden.py saves the state every 5000
# steps) and must reach the next one within 1e-9 with every per-step mask
# equal to the reference's.  The free-running full run is compared exactly up
# to its first flipped mask (test_full_length_config_vs_reference).
CK_WINDOW = 5000


def _config3_windows():
    path = os.path.join(GOLDEN, "config3_full.npz")
    if not os.path.exists(path):
        return []
    G = np.load(path)
    cks = sorted(int(k[4:]) for k in G.files if k.startswith("ck/s") and int(k[4:]) % CK_WINDOW == 0)
    n = int(G["n_steps"])
    starts = [0] + cks
    return [(s0, min(s0 + CK_WINDOW, n)) for s0 in starts if s0 < n]


def _mask_digests(bits, n):
    flags = D_.bits_to_flags(bits, n)
    packed = np.packbits(flags, axis=-1)
    return (np.array([zlib.crc32(packed[s].tobytes()) for s in range(packed.shape[0])],
                     dtype=np.uint32), flags.sum(-1))


@pytest.mark.parametrize("window", _config3_windows(), ids=lambda w: f"{w[0]}-{w[1]}")
def test_config3_windows_vs_reference(window):
    """Config 3 over its whole run, window by window: start at the reference's
    state of step s0, run to s1; eta / hu within 1e-9 of the reference's state
    at s1 (its final state for the last window), every step's mask equal."""
    s0, s1 = window
    G = np.load(os.path.join(GOLDEN, "config3_full.npz"))
    cfg = configs.config3()
    m = cfg.member(0)
    if s0 == 0:
        st0, t0 = np.stack([G["h0"], G["hu0"], G["hw0"]]), 0.0
    else:
        st0, t0 = G[f"ck/s{s0}"], float(G[f"ck/t{s0}"])
    ens = P.Ensemble.from_host(cfg.records(), st0[0][None], st0[1][None], st0[2][None], [t0])
    T = D_.torch()
    n = cfg.n_elements
    bits = T.zeros((s1 - s0, 1, (n + 31) // 32), dtype=T.int32, device="cuda")
    ens.advance(s1 - s0, "adaptive", P.Criterion("eta_over_d"), flag_bits=bits)
    st = ens.check()
    crc, cnt = _mask_digests(bits.cpu().numpy().view(np.uint32)[:, 0], n)
    ref_crc, ref_cnt = G["adaptive/flag_crc"][s0:s1], G["adaptive/flag_count"][s0:s1]
    if s1 == int(G["n_steps"]):
        ref, t_ref = G["adaptive/final"], None
    else:
        ref, t_ref = G[f"ck/s{s1}"], float(G[f"ck/t{s1}"])
    if t_ref is not None:
        assert float(ens.time.item()) == t_ref
    t1 = float(ens.time.item())
    d = m.bathymetry.sample(m.grid.sample_nodes, t1).d
    h, hu = ens.h[0].cpu().numpy(), ens.hu[0].cpu().numpy()
    e_eta, e_hu = rel(h - d, ref[0] - d), rel(hu, ref[1])
    mism = np.flatnonzero(crc != ref_crc)
    print(f"config3 steps {s0}-{s1}: eta {e_eta:.2e} hu {e_hu:.2e}, step masks differing "
          f"{mism.size}, solve residual <= {st['resid_max'][0]:.1e}")
    assert mism.size == 0, f"first differing steps {(mism[:5] + s0).tolist()}"
    assert np.array_equal(cnt, ref_cnt)
    assert e_eta <= 1e-9 and e_hu <= 1e-9


@pytest.mark.parametrize("cfg_name,mode", LONG)
def test_full_length_config_vs_reference(cfg_name, mode):
    path = os.path.join(GOLDEN, f"{cfg_name}_full.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    G = np.load(path)
    cfg = configs.get(cfg_name)
    m = cfg.member(0)
    n_steps = int(G["n_steps"])
    spec = P.ScenarioSpec(cfg.name, m.grid, m.dt, n_steps * m.dt, m.bathymetry, m.bcs)
    init = P.FlowState(P.NodalField(m.grid, G["h0"]), P.NodalField(m.grid, G["hu0"]),
                       P.NodalField(m.grid, G["hw0"]), 0.0)
    crit = P.Criterion("eta_over_d") if mode == "adaptive" else None
    res = P.simulate(spec, init, mode, crit, record_masks=True)
    ref = G[mode + "/final"]
    d = m.bathymetry.sample(m.grid.sample_nodes, res.final_state.time).d
    eta, eta_ref = res.final_state.h.values - d, ref[0] - d
    e_eta = rel(eta, eta_ref)
    e_hu = rel(res.final_state.hu.values, ref[1])
    print(f"{cfg_name} {mode}: eta rel L-inf {e_eta:.3e}, hu rel L-inf {e_hu:.3e}, "
          f"GPU loop {res.loop_time:.3f}s vs reference {float(G[mode + '/loop_time']):.1f}s")
    if cfg_name == "config3":
        # free run: exact masks up to the first flip (then the run follows
        # another trajectory, as the reference's own does under a 1e-10
        # kick); parity over the whole run is test_config3_windows_vs_reference
        cnt = np.array([sum(e1 - e0 + 1 for e0, e1 in r) for _, _, r in res.mask_history])
        crc = []
        for _, _, ranges in res.mask_history:
            f = np.zeros(m.grid.n_elements, bool)
            for e0, e1 in ranges:
                f[e0:e1 + 1] = True
            crc.append(zlib.crc32(np.packbits(f).tobytes()))
        mism = np.flatnonzero(np.array(crc, dtype=np.uint32) != G[mode + "/flag_crc"])
        first = int(mism[0]) if mism.size else n_steps
        K = np.load(os.path.join(GOLDEN, f"{cfg_name}_kicked.npz"))
        print(f"{cfg_name} free run: masks identical to the reference for steps 0..{first - 1} "
              f"of {n_steps}; mask fraction GPU {res.mask_fraction_mean:.4f}, reference "
              f"{float(G[mode + '/mask_fraction']):.4f}, reference kicked by "
              f"{float(K['rel']):.0e} at step {int(K['start'])}: {float(K['mask_fraction']):.4f}")
        assert first > 30000   # past the slide's stop (step ~14740), well into the wave phase
        assert np.array_equal(cnt[:first], G[mode + "/flag_count"][:first])
        assert np.all(np.isfinite(res.final_state.hu.values))
        return
    assert e_eta <= 1e-9 and e_hu <= 1e-9
    if mode == "adaptive":
        cnt = np.array([sum(e1 - e0 + 1 for e0, e1 in r) for _, _, r in res.mask_history])
        crc = []
        for _, _, ranges in res.mask_history:
            f = np.zeros(m.grid.n_elements, bool)
            for e0, e1 in ranges:
                f[e0:e1 + 1] = True
            crc.append(zlib.crc32(np.packbits(f).tobytes()))
        mism = np.flatnonzero(np.array(crc, dtype=np.uint32) != G[mode + "/flag_crc"])
        print(f"{cfg_name}: {mism.size} of {n_steps} step masks differ "
              f"(max count difference {np.abs(cnt - G[mode + '/flag_count']).max()})")
        # every step's mask equals the reference's (no near-threshold flip
        # occurs in these runs; the margin rule of SURVEY H4 would admit one)
        assert mism.size == 0, f"first differing steps {mism[:5]}"
        assert np.array_equal(cnt, G[mode + "/flag_count"])
