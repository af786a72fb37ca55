"""Pins for oracle/verify.py (O10 a-posteriori check)."""
import numpy as np
from oracle import geometry, kernels, h2, rng, verify
from synth import uniform_points
from synthetic_h2 import synthetic_h2


def setup(X, leaf):
    tree = geometry.build_cluster_tree(X, leaf)
    part = geometry.build_partition(tree, 0.7)
    om = lambda c0, nc: rng.omega_block(1, 0, 0, tree.n, c0, nc)
    return tree, part, om, rng.omega_block(1, 2, 0, tree.n, 0, 8)


def test_exact_h2_has_zero_estimate():
    X = uniform_points(1024, 3, 3)
    tree, part, om, Oh = setup(X, 64)
    K, _, _ = synthetic_h2(tree, part, lambda t, m: min(m, 8), 3)
    H, e, r, s = verify.build_verified(tree, part, lambda O: K @ O, lambda a, b: K[np.ix_(a, b)], om, Oh, 1e-10)
    assert r == 0 and e < 1e-12


def test_estimate_equals_dense_residual_and_retry_reaches_tol():
    """e equals ||(K_h - K) Om_h|| / ||K Om_h|| with K_h the dense reconstruction (a different
    evaluation path than the matvec); with s = 30 the first build misses tol = 1e-6, and the
    s / 3 rebuilds reach it (s_used = 30 / 3^r)."""
    X = uniform_points(2048, 3, 0)
    tree, part, om, Oh = setup(X, 64)
    op = kernels.KernelOperator("exp", 0.2, X[tree.perm])
    K = op.dense()
    H0 = h2.build(tree, part, op.sampler, op.entry, om, 1e-6, h2.BuildOpts(tol_safety=30.0))
    e0 = verify.a_posteriori_error(lambda Z: h2.matvec(H0, Z), op.sampler, Oh)
    KO = K @ Oh
    assert abs(e0 - np.linalg.norm((h2.to_dense(H0) - K) @ Oh) / np.linalg.norm(KO)) <= 1e-9 * e0
    assert e0 > 1e-6
    H, e, r, s = verify.build_verified(tree, part, op.sampler, op.entry, om, Oh, 1e-6,
                                       h2.BuildOpts(tol_safety=30.0), retries=6)
    assert 1 <= r <= 6 and e <= 1e-6 and abs(s - 30.0 / 3 ** r) <= 1e-12
    # the estimate tracks the true relative error within the probe count's spread
    true = np.linalg.norm(h2.to_dense(H) - K) / np.linalg.norm(K)
    assert 0.2 * true <= e <= 5 * true
