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



def test_power_method_pins():
    """O9: the power-method 2-norm never exceeds the exact 2-norm (a Rayleigh-type
    lower bound), converges to it for a symmetric matrix with a spectral gap, is exactly the 2-norm
    for a rank-one matrix after two iterations, and the error ratio of an exact H^2 is 0."""
    rng = np.random.default_rng(0)
    Q, _ = np.linalg.qr(rng.standard_normal((60, 60)))
    lam = np.concatenate([[5.0, -3.0], rng.uniform(-1, 1, 58)])
    A = (Q * lam) @ Q.T
    x0 = rng.standard_normal(60)
    exact = np.linalg.norm(A, 2)
    for it in (1, 3, 10):
        assert verify.power_2norm(lambda x: A @ x, x0, it) <= exact * (1 + 1e-12)
    assert abs(verify.power_2norm(lambda x: A @ x, x0, 200) - exact) <= 1e-10 * exact
    u = rng.standard_normal(60)
    R1 = np.outer(u, u)
    assert abs(verify.power_2norm(lambda x: R1 @ x, x0, 2) - np.linalg.norm(R1, 2)) <= 1e-12 * np.linalg.norm(R1, 2)
    r, e, k = verify.power_error(lambda x: A @ x, lambda x: A @ x, x0, 5)
    assert r == 0.0 and e == 0.0 and k > 0
    E = 1e-3 * ((Q * rng.uniform(-1, 1, 60)) @ Q.T)       # symmetric difference of known norm
    r, e, k = verify.power_error(lambda x: (A + E) @ x, lambda x: A @ x, x0, 300)
    assert abs(e - np.linalg.norm(E, 2)) <= 1e-6 * np.linalg.norm(E, 2) and abs(k - exact) <= 1e-10 * exact
