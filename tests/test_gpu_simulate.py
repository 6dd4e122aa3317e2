"""GPU multi-step parity: simulate (one fused launch for the whole loop) and the
batched ensemble path, against the oracle run step by step."""

import numpy as np
import pytest

import paper_2505_17025_b200 as P
from paper_2505_17025_b200 import configs
from oracle import nhswe_oracle as O
from tests.helpers import mask_mismatch_outside_margin, oracle_depth, oracle_member, rel

pytestmark = pytest.mark.gpu


def oracle_history(mem, h, hu, hw, n_steps, mode, kind="eta_over_d", k_nh=1e-3, enlarge=False):
    """Oracle run keeping per-step flags and criterion values."""
    t = 0.0
    flags, vals = [], []
    for _ in range(n_steps):
        ph, pq, pw = O.heun(mem.grid, mem.bottom, mem.bcs, mem.g, h, hu, hw, t, mem.dt,
                            cfl_warn=False)
        o = O.step(mem, h, hu, hw, t, mode, kind, k_nh, enlarge, cfl_warn=False)
        t = t + mem.dt
        vals.append(O.indicator(mem.grid, mem.bottom, kind, ph, pq, pw, t).max(axis=1))
        flags.append(o.flags)
        h, hu, hw = o.h, o.hu, o.hw
    return h, hu, hw, np.array(flags), np.array(vals)


@pytest.mark.parametrize("mode", ["global", "adaptive"])
def test_config1_simulate_prefix(mode):
    cfg = configs.config1()
    m = cfg.member(0)
    h, hu, hw = cfg.host_state(0, None)
    n_steps = 300
    spec = P.ScenarioSpec("c1", m.grid, m.dt, n_steps * m.dt, m.bathymetry, m.bcs)
    assert spec.n_steps == n_steps
    init = P.FlowState(P.NodalField(m.grid, h), P.NodalField(m.grid, hu),
                       P.NodalField(m.grid, hw), 0.0)
    crit = P.Criterion("eta_over_d") if mode == "adaptive" else None
    res = P.simulate(spec, init, mode, crit)
    mem = oracle_member(m.grid, m.bathymetry, m.bcs, m.dt)
    oh, oq, ow, oflags, ovals = oracle_history(mem, h, hu, hw, n_steps, mode)
    assert rel(res.final_state.h.values - 1.0, oh - 1.0) <= 1e-9
    assert rel(res.final_state.hu.values, oq) <= 1e-9
    if mode == "adaptive":
        assert len(res.mask_history) == n_steps
        for s, (_, _, ranges) in enumerate(res.mask_history):
            g = np.zeros(m.grid.n_elements, bool)
            for e0, e1 in ranges:
                g[e0:e1 + 1] = True
            diff = np.flatnonzero(g != oflags[s])
            near = np.abs(ovals[s][diff] - 1e-3) <= 1e-9 * 1e-3
            assert near.all(), f"step {s}: mask differs at {diff[~near][:8]}"
        assert abs(res.mask_fraction_mean - oflags.mean()) < 1e-3


def test_long_member_cluster_global():
    """N = 16384: one member spread over a 15-CTA cluster (DSMEM tree)."""
    grid = P.GridSpec(0.0, 20.0, 16384)
    bathy = P.SlopeGaussianSlide(0.1, np.tan(np.radians(12.0)), 1.0, 0.1, 0.4, 2.0, 1.5, 0.5, 0.8)
    bcs = P.BoundaryPair(P.WALL, P.ABSORBING)
    d = oracle_depth(bathy, grid.sample_nodes, 0.0)
    x = grid.nodes
    h = d + 0.01 * np.exp(-((x - 6.0) / 0.5) ** 2)
    hu = 0.02 * np.exp(-((x - 6.0) / 0.5) ** 2)
    hw = np.zeros_like(h)
    dt = 6.5e-5
    st = P.FlowState(P.NodalField(grid, h), P.NodalField(grid, hu), P.NodalField(grid, hw), 0.0)
    mem = oracle_member(grid, bathy, bcs, dt)
    t = 0.0
    oh, oq, ow = h, hu, hw
    for _ in range(6):
        st = P.adaptive_step(st, dt, bathy, bcs, mode="global", cfl_warn=False).state
        o = O.step(mem, oh, oq, ow, t, "global", cfl_warn=False)
        oh, oq, ow = o.h, o.hu, o.hw
        t += dt
    assert rel(st.hu.values, oq) <= 1e-10
    assert np.abs(st.hw.values - ow).max() <= 1e-10 * np.abs(ow).max()


@pytest.mark.parametrize("path", ["resident", "stream"])
@pytest.mark.parametrize("mode,enlarge", [("adaptive", False), ("adaptive", True), ("global", False)])
def test_ensemble_mixed_members(path, mode, enlarge):
    """Config-4 style mixed ensemble (solitary + box uplift), per-member dt / dx,
    through both step implementations (SMEM-resident clusters / streaming tiles)."""
    cfg = configs.Config4(n_members=6, n_elements=512, n_steps=120)
    recs = cfg.records()
    states = [cfg.host_state(i, oracle_depth) for i in range(cfg.n_members)]
    H = np.stack([s[0] for s in states])
    Q = np.stack([s[1] for s in states])
    Wv = np.stack([s[2] for s in states])
    ens = P.Ensemble.from_host(recs, H, Q, Wv)
    crit = P.Criterion("eta_over_d", 1e-3, enlarge)
    ens.advance(cfg.n_steps, mode, crit, path=path)
    st = ens.check()
    gh, gq, gw = (x.cpu().numpy() for x in (ens.h, ens.hu, ens.hw))
    for i in range(cfg.n_members):
        m = cfg.member(i)
        mem = oracle_member(m.grid, m.bathymetry, m.bcs, m.dt)
        r = O.run(mem, H[i], Q[i], Wv[i], cfg.n_steps, mode=mode, enlarge=enlarge)
        assert rel(gh[i] - m.bathymetry.h0, r.h - m.bathymetry.h0) <= 1e-9, (i, path)
        assert rel(gq[i], r.hu) <= 1e-9, (i, path)
        assert np.abs(gw[i] - r.hw).max() <= 1e-9 * max(np.abs(r.hw).max(), 1e-12), (i, path)
        assert abs(st["flagged"][i] / (cfg.n_steps * cfg.n_elements) - r.fraction_mean) < 1e-3
        assert float(ens.time[i].item()) == r.t, (i, path)


@pytest.mark.parametrize("path", ["resident", "stream"])
@pytest.mark.parametrize("cfg_name,members,n_steps", [("config4", (0, 1, 2047, 4095), 200),
                                                      ("config5", (0, 65535), 40)])
def test_sampled_ensemble_members_full_size(cfg_name, members, n_steps, path):
    """Sampled members of the throughput configs at full N, stepped inside the
    batched ensemble path, against the oracle run of the same members."""
    cfg = configs.Config4() if cfg_name == "config4" else configs.Config5()
    idx = list(members)
    recs = cfg.records(idx)
    states = [cfg.host_state(i, oracle_depth) for i in idx]
    H, Q, W = (np.stack([s[k] for s in states]) for k in range(3))
    ens = P.Ensemble.from_host(recs, H, Q, W)
    mode = "adaptive"
    ens.advance(n_steps, mode, P.Criterion("eta_over_d"), path=path)
    st = ens.check()
    gh, gq, gw = (x.cpu().numpy() for x in (ens.h, ens.hu, ens.hw))
    for k, i in enumerate(idx):
        m = cfg.member(i)
        r = O.run(oracle_member(m.grid, m.bathymetry, m.bcs, m.dt), H[k], Q[k], W[k], n_steps,
                  mode=mode)
        d = oracle_depth(m.bathymetry, m.grid.sample_nodes, r.t)
        assert rel(gh[k] - d, r.h - d) <= 1e-9, (cfg_name, i)
        assert rel(gq[k], r.hu) <= 1e-9 or np.abs(gq[k] - r.hu).max() < 1e-12, (cfg_name, i)
        assert abs(st["flagged"][k] / (n_steps * cfg.n_elements) - r.fraction_mean) < 1e-3


def test_per_step_replay_after_long_run():
    """GPU state at step n -> one oracle step vs one GPU step."""
    cfg = configs.config1()
    m = cfg.member(0)
    h, hu, hw = cfg.host_state(0, None)
    ens = P.Ensemble.from_host(cfg.records(), h[None], hu[None], hw[None])
    crit = P.Criterion("eta_over_d")
    ens.advance(1500, "adaptive", crit)
    ens.check()
    t = float(ens.time.item())
    gh, gq, gw = (x[0].cpu().numpy() for x in (ens.h, ens.hu, ens.hw))
    st = P.FlowState(P.NodalField(m.grid, gh), P.NodalField(m.grid, gq), P.NodalField(m.grid, gw), t)
    r = P.adaptive_step(st, m.dt, m.bathymetry, m.bcs, mode="adaptive", crit=crit)
    mem = oracle_member(m.grid, m.bathymetry, m.bcs, m.dt)
    ph, pq, pw = O.heun(mem.grid, mem.bottom, mem.bcs, 9.81, gh, gq, gw, t, m.dt, cfl_warn=False)
    o = O.step(mem, gh, gq, gw, t, "adaptive", cfl_warn=False)
    vals = O.indicator(mem.grid, mem.bottom, "eta_over_d", ph, pq, pw, t + m.dt)
    bad = mask_mismatch_outside_margin(r.mask.flags, vals, 1e-3)
    assert bad.size == 0
    assert rel(r.state.h.values - 1.0, o.h - 1.0) <= 1e-12
    assert rel(r.state.hu.values, o.hu) <= 1e-12


def test_stream_member_chunks_bitwise_equal():
    """Ensembles too large for one workspace run as member blocks through one
    workspace (config 5 at full size); results are identical to one block."""
    cfg = configs.Config4(n_members=6, n_elements=700, n_steps=60)
    recs = cfg.records()
    states = [cfg.host_state(i, oracle_depth) for i in range(cfg.n_members)]
    H, Q, W = (np.stack([s[k] for s in states]) for k in range(3))
    out = []
    for chunk in (None, 2, 4):
        ens = P.Ensemble.from_host(recs, H, Q, W)
        if chunk:
            ens._chunk = chunk
        ens.advance(cfg.n_steps, "adaptive", P.Criterion("eta_over_d"), path="stream")
        st = ens.check()
        out.append((ens.h.cpu().numpy(), ens.hu.cpu().numpy(), ens.hw.cpu().numpy(),
                    ens.time.cpu().numpy(), st["flagged"].copy()))
    for other in out[1:]:
        for a, b in zip(out[0], other):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("block", [None, 64, 300, 1000])
def test_advance_host_bitwise_equal_to_device_ensemble(block):
    """driver.advance_host (the end-to-end call of bench.py's e2e leg: pinned
    host state streamed through the GPU in member blocks on three streams and
    three device buffers, short blocks at both ends) leaves the host arrays
    bit-identical to Ensemble.advance on the device-resident ensemble."""
    import torch
    from paper_2505_17025_b200.driver import advance_host
    cfg = configs.Config4(n_members=700, n_elements=130, n_steps=21)
    recs = cfg.records()
    states = [cfg.host_state(i, oracle_depth) for i in range(cfg.n_members)]
    H, Q, W = (np.stack([s[k] for s in states]) for k in range(3))
    crit = P.Criterion("eta_over_d")
    ens = P.Ensemble.from_host(recs, H, Q, W)
    ens.advance(cfg.n_steps, "adaptive", crit)
    st = ens.check()
    host = [torch.from_numpy(x.copy()).pin_memory() for x in (H, Q, W)]
    t = torch.zeros(cfg.n_members, dtype=torch.float64).pin_memory()
    st2 = advance_host(recs, *host, t, cfg.n_steps, "adaptive", crit, block=block)
    for a, b in zip(host + [t], (ens.h, ens.hu, ens.hw, ens.time)):
        assert torch.equal(a, b.cpu())
    assert np.array_equal(st2["flagged"], st["flagged"])
    assert (st2["error_key"] == st["error_key"]).all()


@pytest.mark.parametrize("n_steps", [5, 6, 61])
@pytest.mark.parametrize("mode", ["adaptive", "global", "hydrostatic"])
def test_stream_graph_bitwise_equal_to_launches(n_steps, mode):
    """The time loop captured as a CUDA graph of step pairs (nh_stream_graphs)
    gives bit-identical states, times, flag counts and launch counts to plain
    launches, for even and odd step counts and repeated calls (cached graph)."""
    from paper_2505_17025_b200 import _device as D
    cfg = configs.Config4(n_members=6, n_elements=700, n_steps=n_steps)
    recs = cfg.records()
    states = [cfg.host_state(i, oracle_depth) for i in range(cfg.n_members)]
    H, Q, W = (np.stack([s[k] for s in states]) for k in range(3))
    crit = P.Criterion("eta_over_d") if mode == "adaptive" else None
    prev = D.stream_graphs()
    out = []
    try:
        for graphs in (False, True):
            D.stream_graphs(graphs)
            ens = P.Ensemble.from_host(recs, H, Q, W)
            l0 = D.launch_count()
            for _ in range(2):
                ens.advance(n_steps, mode, crit, path="stream")
            launches = D.launch_count() - l0
            st = ens.check()
            out.append((ens.h.cpu().numpy(), ens.hu.cpu().numpy(), ens.hw.cpu().numpy(),
                        ens.time.cpu().numpy(), st["flagged"].copy(), launches))
    finally:
        D.stream_graphs(prev)
    for a, b in zip(out[0], out[1]):
        assert np.array_equal(a, b)


def test_simulate_gauges_recorded_on_device():
    """simulate() with gauges records h at the gauge nodes on the device every
    step (one launch sequence, no per-step sync); gauge_eta matches the oracle
    run step by step (reference driver.py:58-69, 88-94)."""
    cfg = configs.config2()
    m = cfg.member(0)
    n_steps = 400
    gauges = (0.05, 0.3, 0.31, 1.0, 2.5)
    spec = P.ScenarioSpec("c2g", m.grid, m.dt, n_steps * m.dt, m.bathymetry, m.bcs, gauges)
    h, hu, hw = cfg.host_state(0, oracle_depth)
    init = P.FlowState(P.NodalField(m.grid, h), P.NodalField(m.grid, hu),
                       P.NodalField(m.grid, hw), 0.0)
    r = P.simulate(spec, init, "adaptive", P.Criterion("eta_over_d"))
    mem = oracle_member(m.grid, m.bathymetry, m.bcs, m.dt)
    idx = [m.grid.nearest_node(x) for x in gauges]
    gx = np.array([m.grid.sample_nodes[e, j] for e, j in idx])
    t = 0.0
    ref = [h[tuple(np.array(idx).T)] - oracle_depth(m.bathymetry, gx, 0.0)]
    for _ in range(n_steps):
        o = O.step(mem, h, hu, hw, t, "adaptive", cfl_warn=False)
        h, hu, hw = o.h, o.hu, o.hw
        t = t + mem.dt
        ref.append(h[tuple(np.array(idx).T)] - oracle_depth(m.bathymetry, gx, t))
    ref = np.array(ref)
    assert r.gauge_eta.shape == (n_steps + 1, len(gauges))
    assert np.abs(r.gauge_eta - ref).max() <= 1e-12 * max(np.abs(ref).max(), 1e-6)
    assert np.allclose(r.gauge_times[-1], n_steps * m.dt)


@pytest.mark.parametrize("path", ["resident", "stream"])
def test_ensemble_gauges_both_paths(path):
    """Device gauge rows equal the state after each step, for every member, on
    both paths (the stream path records them inside the CUDA-graph loop)."""
    import torch
    cfg = configs.Config4(n_members=6, n_elements=700, n_steps=9)
    recs = cfg.records()
    states = [cfg.host_state(i, oracle_depth) for i in range(cfg.n_members)]
    H, Q, W = (np.stack([s[k] for s in states]) for k in range(3))
    nodes = np.array([0, 1, 351, 700, 1398, 1399], dtype=np.int32)
    ens = P.Ensemble.from_host(recs, H, Q, W)
    ens_ref = P.Ensemble.from_host(recs, H, Q, W)
    g = (torch.as_tensor(nodes, device="cuda"),
         torch.full((cfg.n_steps, 6, nodes.size), np.nan, dtype=torch.float64, device="cuda"))
    ens.advance(cfg.n_steps, "adaptive", P.Criterion("eta_over_d"), path=path, gauges=g)
    out = g[1].cpu().numpy()
    for s in range(cfg.n_steps):
        ens_ref.advance(1, "adaptive", P.Criterion("eta_over_d"), path=path)
        want = ens_ref.h.cpu().numpy().reshape(6, -1)[:, nodes]
        assert np.array_equal(out[s], want), s


@pytest.mark.parametrize("kind,enlarge", [("w", False), ("w_x", False), ("w_x", True)])
def test_w_criteria_stream_fallback(kind, enlarge):
    """w / w_x criteria on the streaming path: a member whose step input has
    hw == 0 everywhere is corrected globally for that step (adaptivity.py:
    153-154; K_F).  Box uplifts start from rest (fallback on the first step
    only), solitary members carry hw from the start (never), and so does a
    still-water member after its first (roundoff-level) correction.  Per-step flags equal the
    resident kernel's, final states match the oracle run."""
    from paper_2505_17025_b200 import _device as D
    cfg = configs.Config4(n_members=6, n_elements=512, n_steps=40)
    n = cfg.n_steps
    recs = [cfg.records()]
    states = [cfg.host_state(i, oracle_depth) for i in range(cfg.n_members)]
    members = [(m.grid, m.bathymetry, m.bcs, m.dt) for m in map(cfg.member, range(cfg.n_members))]
    still = (P.GridSpec(0.0, 100.0, 512), P.FlatBottom(1.0), P.BoundaryPair(P.WALL, P.ABSORBING),
             0.01)   # CFL 0.16
    recs.append(D.member_record(*still))
    members.append(still)
    states.append((np.ones((512, 2)), np.zeros((512, 2)), np.zeros((512, 2))))
    recs = np.concatenate(recs)
    H, Q, W = (np.stack([s[k] for s in states]) for k in range(3))
    B, nw = len(members), (512 + 31) // 32
    crit = P.Criterion(kind, 1e-3, enlarge)
    out = {}
    for path in ("resident", "stream"):
        ens = P.Ensemble.from_host(recs, H, Q, W)
        bits = D.torch().zeros((n, B, nw), dtype=D.torch().int32, device="cuda")
        ens.advance(n, "adaptive", crit, flag_bits=bits, path=path)
        st = ens.check()
        out[path] = (ens.h.cpu().numpy(), ens.hu.cpu().numpy(), ens.hw.cpu().numpy(),
                     bits.cpu().numpy(), st["flagged"].copy())
    assert np.array_equal(out["stream"][3], out["resident"][3])
    assert np.array_equal(out["stream"][4], out["resident"][4])
    first = out["stream"][3][0].view(np.uint32)       # step 0: input hw == 0 -> full mask
    for i in range(B):
        assert (first[i] == 0xFFFFFFFF).all() == (not np.any(W[i])), i
    gh, gq, gw = out["stream"][:3]
    for i, (grid, bathy, bcs, dt) in enumerate(members):
        r = O.run(oracle_member(grid, bathy, bcs, dt), H[i], Q[i], W[i], n, mode="adaptive",
                  kind=kind, enlarge=enlarge)
        d = oracle_depth(bathy, grid.sample_nodes, r.t)
        assert rel(gh[i] - d, r.h - d) <= 1e-9 or np.abs(gh[i] - r.h).max() <= 1e-15, i
        assert np.abs(gq[i] - r.hu).max() <= 1e-9 * max(np.abs(r.hu).max(), 1e-12), i
        assert np.abs(gw[i] - r.hw).max() <= 1e-9 * max(np.abs(r.hw).max(), 1e-12), i
        assert abs(out["stream"][4][i] / (n * 512) - r.fraction_mean) < 1e-12, i
