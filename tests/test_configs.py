"""BASELINE configuration builders (host input generation)."""

import math

import numpy as np

from paper_2505_17025_b200 import configs
from paper_2505_17025_b200.bathymetry import SlopeGaussianSlide, SmoothBoxPlate
from tests.helpers import oracle_depth


def test_config1_matches_survey_numbers():
    c = configs.config1()
    m = c.member(0)
    assert abs(m.dt - 4.6508e-3) < 1e-7 and c.n_steps == 6450
    h, hu, hw = c.host_state(0, None)
    k = math.sqrt(3 * 0.1 / 4.0)
    assert abs(h.max() - 1.1) < 1e-3
    assert np.all(np.isfinite(hw))


def test_config2_and_3_dt_rule():
    c2, c3 = configs.config2(), configs.config3()
    assert c2.n_steps == 13447 and abs(c2.member(0).dt - 5.9493e-4) < 1e-8
    assert c3.n_steps == 112755 and abs(c3.member(0).dt - 1.3303e-4) < 1e-8


def test_config4_members_deterministic_and_mixed():
    a = configs.Config4(n_members=16, n_elements=64)
    b = configs.Config4(n_members=16, n_elements=64)
    ra, rb = a.records(), b.records()
    assert np.array_equal(ra.view(np.uint8), rb.view(np.uint8))
    kinds = ra["bottom_kind"]
    assert set(kinds[0::2]) == {0} and set(kinds[1::2]) == {3}
    for i in range(1, 16, 2):
        m = a.member(i)
        assert isinstance(m.bathymetry, SmoothBoxPlate) and m.bathymetry.h0 == 0.01
        h, hu, hw = a.host_state(i, oracle_depth)
        assert np.all(h == 0.01) and not hu.any() and not hw.any()


def test_config5_table_admissible():
    c = configs.Config5(n_members=64, n_elements=256)
    tab = c.table()
    assert tab.shape == (64, 5)
    tan_t, A, sigma, x0, u_t = tab.T
    assert np.all((np.degrees(np.arctan(tan_t)) >= 5) & (np.degrees(np.arctan(tan_t)) <= 20))
    assert np.all((sigma >= 0.1) & (sigma <= 1.0)) and np.all((u_t >= 0.2) & (u_t <= 2.0))
    rec = c.records(np.arange(4))
    for i in range(4):
        m = c.member(i)
        kind, params = m.bathymetry.pack()
        assert np.allclose(rec["bottom"][i, :len(params)], params, rtol=1e-15)
        d = oracle_depth(m.bathymetry, m.grid.sample_nodes, 0.0)
        assert d.min() >= 0.04


def test_advance_host_block_schedule():
    """driver.block_schedule: the member blocks of the host-pipelined advance
    cover the ensemble exactly, never exceed the workspace's block, and ramp
    up and down at the ends when the ensemble is long enough."""
    from paper_2505_17025_b200.driver import block_schedule
    for n, blk in ((65536, 2048), (100, 2048), (5000, 2048), (4096, 2048), (3100, 1024),
                   (1, 1), (700, 64), (700, 300), (129, 128)):
        s = block_schedule(n, blk)
        assert sum(s) == n and all(0 < v <= min(n, blk) for v in s), (n, blk, s)
    s = block_schedule(65536, 2048)
    assert s[:3] == [512, 1024, 2048] and s[-2:] == [1024, 512]
    assert block_schedule(100, 2048) == [100]
