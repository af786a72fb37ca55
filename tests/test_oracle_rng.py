"""Pins for oracle/rng.py (Omega generator, R8)."""
import os
import numpy as np
from oracle.rng import philox4x32_10, gaussian_block

GOLD = os.path.join(os.path.dirname(__file__), "golden", "philox4x32_10_kat.txt")


def test_philox_known_answers():
    rows = [l.split() for l in open(GOLD) if l.strip() and not l.startswith("#")]
    assert len(rows) == 3
    for r in rows:
        v = [int(x, 16) for x in r]
        ctr = np.array(v[0:4], np.uint32).reshape(4, 1)
        key = np.array(v[4:6], np.uint32).reshape(2, 1)
        out = philox4x32_10(ctr, key)[:, 0]
        assert [int(x) for x in out] == v[6:10]


def test_gaussian_moments():
    g = gaussian_block(1, 0, 0, 20000, 0, 16)
    assert abs(g.mean()) < 0.01
    assert abs(g.var() - 1.0) < 0.01
    # fourth moment of N(0,1) is 3
    assert abs((g ** 4).mean() - 3.0) < 0.1
    # columns uncorrelated
    c = np.corrcoef(g.T)
    assert np.max(np.abs(c - np.eye(16))) < 0.05


def test_block_slicing_consistent():
    full = gaussian_block(7, 3, 0, 50, 0, 13)
    part = gaussian_block(7, 3, 10, 20, 3, 7)
    assert np.array_equal(part, full[10:30, 3:10])
    other = gaussian_block(7, 4, 0, 50, 0, 13)
    assert not np.any(other == full)
