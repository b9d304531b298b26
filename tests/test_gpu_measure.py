"""Measurement hooks the bench line relies on (bench.py rooflines)."""
import pytest


@pytest.mark.gpu
def test_draw_peak_is_measured():
    """mpcg_debug_draw_peak: splitmix64 draws per second on a full grid (the register compare
    chain's roofline); a B200 does ~1e12."""
    from paper_2209_13643_b200 import api
    v = api.draw_peak(0)
    assert 1e11 < v < 1e14


@pytest.mark.gpu
def test_chain_reg_probe_counts_draws():
    """The register compare chain is probed as its own class with 77 draws per element pair."""
    import numpy as np
    import paper_2209_13643_b200 as mp
    from paper_2209_13643_b200 import api
    s = mp.Session(device=0, n_local=2, seed=3, frac_bits=16)
    n = 50000
    x = s.tensor(np.random.default_rng(0).integers(0, 2**63, size=(2, n), dtype=np.uint64))
    api.probe_start("chain_reg")
    mp.relu_shares(s, x)
    s.sync()
    ms, launches, units = api.probe_stop()
    assert launches == 1 and ms > 0
    assert units == 77.0 * n
