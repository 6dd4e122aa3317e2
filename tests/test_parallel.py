"""Multi-process sharding logic on CPU (gloo, world size 2): the N>1 path has no
collective on the step path, only MAX of the timed region and a final gather."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2505_17025_b200 import parallel


def test_shard_partitions_members():
    for n in (1, 7, 64, 4097):
        for w in (1, 2, 3, 8):
            got = []
            for r in range(w):
                s = parallel.shard(n, w, r)
                got.extend(s)
                assert abs(len(s) - n / w) < 1
            assert got == list(range(n))
    with pytest.raises(ValueError):
        parallel.shard(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import nhswe_oracle as O
    from paper_2505_17025_b200 import configs
    from tests.helpers import oracle_depth, oracle_member
    cfg = configs.Config4(n_members=6, n_elements=64)

    def build(idx):
        return [(i, *cfg.host_state(i, oracle_depth)) for i in idx]

    def advance(state):
        out = []
        for i, h, hu, hw in state:
            m = cfg.member(i)
            r = O.run(oracle_member(m.grid, m.bathymetry, m.bcs, m.dt), h, hu, hw, 20)
            out.append((i, r))
        state[:] = out
        return 10.0 * (rank + 1)          # pretend device milliseconds

    def summarize(state):
        return {"member": np.array([i for i, _ in state]),
                "hu": np.stack([r.hu for _, r in state]),
                "frac": np.array([r.fraction_mean for _, r in state])}

    ms, out = parallel.run_sharded(cfg.n_members, advance, build, summarize)
    q.put((rank, ms, out))
    dist.destroy_process_group()


def test_gloo_sharded_run_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    res.sort(key=lambda x: x[0])
    assert all(ms == 20.0 for _, ms, _ in res)          # MAX over ranks
    assert res[1][2] is None
    out = res[0][2]
    assert list(out["member"]) == list(range(6))
    # the gathered shards equal a single-process run member by member
    from oracle import nhswe_oracle as O
    from paper_2505_17025_b200 import configs
    from tests.helpers import oracle_depth, oracle_member
    cfg = configs.Config4(n_members=6, n_elements=64)
    for i in range(6):
        m = cfg.member(i)
        r = O.run(oracle_member(m.grid, m.bathymetry, m.bcs, m.dt), *cfg.host_state(i, oracle_depth), 20)
        assert np.array_equal(out["hu"][i], r.hu)


def _bench_worker(rank, world, port, q):
    """bench.py's own sharding path (workload_members -> parallel.shard, the
    untimed gather_summaries) under gloo."""
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    assert bench.dist_env() == (rank, world, rank)
    out = {}
    for wl, kw in (("config5", dict(n_members=11, n_elements=64)),
                   ("config4", dict(n_members=10, n_elements=64))):
        cfg, idx, recs = bench.workload_members(wl, rank, world, **kw)
        assert idx == list(parallel.shard(cfg.n_members, world, rank))
        got = parallel.gather_summaries({"member": np.array(idx, dtype=np.int64),
                                         "rec": recs.view(np.uint8).reshape(len(idx), -1)})
        out[wl] = got
    q.put((rank, out))
    dist.destroy_process_group()


def test_gloo_bench_shards_concatenate_to_single_gpu_table():
    """The shards bench.py builds at world size 2 are, member for member, the
    N=1 ensemble (a member's record depends on its index only), so the
    multi-GPU line is strong scaling of one fixed workload."""
    import bench
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_bench_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res[1]["config5"] is None and res[1]["config4"] is None
    for wl, kw in (("config5", dict(n_members=11, n_elements=64)),
                   ("config4", dict(n_members=10, n_elements=64))):
        cfg, idx, recs = bench.workload_members(wl, 0, 1, **kw)
        got = res[0][wl]
        assert list(got["member"]) == idx == list(range(cfg.n_members))
        assert np.array_equal(got["rec"], recs.view(np.uint8).reshape(len(idx), -1)), wl
        # ... and of the full-size workload's first members
        full = bench.get_config(wl)
        want = full.records(range(3))
        small = bench.get_config(wl, n_members=3)
        if wl == "config5":   # the config-5 table is drawn per member index
            assert np.array_equal(small.records(range(3))["bottom"], want["bottom"])
