"""Pins for oracle/rng.py (Omega generator, R8)."""
import os
import numpy as np
from math import comb
from oracle.rng import philox4x32_10, omega_block

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


def test_omega_distribution_is_centred_binomial():
    """R8: Omega = (Binomial(64, 1/2) - 32) / 4 -- mean 0, variance 1, kurtosis 3 - 2/64."""
    g = omega_block(1, 0, 0, 20000, 0, 16)
    assert np.all(g * 4 == np.round(g * 4)) and np.abs(g).max() <= 8
    assert abs(g.mean()) < 0.01
    assert abs(g.var() - 1.0) < 0.01
    assert abs((g ** 4).mean() - (3.0 - 2.0 / 64)) < 0.1
    c = np.corrcoef(g.T)                       # columns uncorrelated
    assert np.max(np.abs(c - np.eye(16))) < 0.05
    # frequencies against the closed form C(64, k) / 2^64 (chi-square, 3 sigma)
    k = np.round(g.reshape(-1) * 4 + 32).astype(int)
    obs = np.bincount(k, minlength=65)
    p = np.array([comb(64, i) for i in range(65)], dtype=float) / 2.0 ** 64
    exp = p * k.size
    m = exp > 20
    chi2 = np.sum((obs[m] - exp[m]) ** 2 / exp[m])
    dof = m.sum() - 1
    assert chi2 < dof + 3 * np.sqrt(2 * dof)


def test_omega_entries_from_philox_words():
    """Entry (i, 2q) = (popcount(w0) + popcount(w1) - 32)/4 of Philox(ctr=(i,q,stream,0), key=seed)."""
    seed, stream = 0x123456789, 5
    g = omega_block(seed, stream, 40, 3, 6, 4)
    for r in range(3):
        for q in (3, 4):
            w = philox4x32_10(np.array([[40 + r], [q], [stream], [0]], np.uint32),
                              np.array([[seed & 0xFFFFFFFF], [seed >> 32]], np.uint32))[:, 0]
            bits = [bin(int(x)).count("1") for x in w]
            assert g[r, 2 * q - 6] == (bits[0] + bits[1] - 32) / 4
            assert g[r, 2 * q - 5] == (bits[2] + bits[3] - 32) / 4


def test_block_slicing_consistent():
    full = omega_block(7, 3, 0, 50, 0, 13)
    part = omega_block(7, 3, 10, 20, 3, 7)
    assert np.array_equal(part, full[10:30, 3:10])
    other = omega_block(7, 4, 0, 50, 0, 13)
    assert np.mean(other == full) < 0.2
