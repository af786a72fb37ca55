"""Pins for oracle/kernels.py: closed forms of PAPER.md Eq. cov / Eq. ie."""
import os
import numpy as np
from oracle.kernels import kernel_block, pair_dist

GOLD = os.path.join(os.path.dirname(__file__), "golden", "kernel_values.txt")


def test_closed_forms():
    n = 0
    for line in open(GOLD):
        line = line.split("#")[0].split()
        if not line:
            continue
        kind, param, r, expect = line[0], float(line[1]), float(line[2]), float(line[3])
        X = np.array([[0.0, 0.0, 0.0]])
        Y = np.array([[r, 0.0, 0.0]])
        got = kernel_block(kind, param, X, Y)[0, 0]
        assert abs(got - expect) <= 4e-16 * max(1.0, abs(expect)), (kind, r, got, expect)
        n += 1
    assert n == 5


def test_distance_3d_pythagoras():
    X = np.array([[0.0, 0.0, 0.0]])
    Y = np.array([[1.0, 2.0, 2.0]])
    assert pair_dist(X, Y)[0, 0] == 3.0


def test_symmetry_and_ranges():
    rng = np.random.default_rng(3)
    P = rng.random((60, 3))
    for kind, param in (("exp", 0.2), ("helmholtz", 3.0)):
        K = kernel_block(kind, param, P, P)
        assert np.array_equal(K, K.T)
    K = kernel_block("exp", 0.2, P, P)
    assert np.all(K > 0) and np.all(K <= 1) and np.all(np.diag(K) == 1.0)
    assert np.all(np.diag(kernel_block("helmholtz", 3.0, P, P)) == 0.0)
