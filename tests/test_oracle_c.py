"""Pins for the C oracle (oracle/c/h2oracle.c via oracle/c_h2.py): Algorithm 1 (PAPER.md
L196-263, §III) with every floating-point operation in a stated order.  Pinned to
things other than itself: the Random123 known-answer vectors, LAPACK dgeqp3 pivots, brute-force
dense error, exact recovery of synthetic H^2 matrices of known ranks, closed forms, special
cases, and agreement with the independent numpy oracle (oracle/h2.py, itself pinned in
test_oracle_h2.py)."""
import os

import numpy as np
import pytest
import scipy.linalg as sla

from oracle import geometry, kernels, h2 as oh2, rng, c_h2
from synth import uniform_points, grid_points
from synthetic_h2 import synthetic_h2

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def setup(X, leaf, eta=0.7):
    tree = geometry.build_cluster_tree(X, leaf)
    part = geometry.build_partition(tree, eta)
    return tree, part, c_h2.TreeArrays(tree, part, X)


def test_philox_known_answers_and_omega_stream():
    """Random123 KAT (tests/golden/philox4x32_10_kat.txt) and the Omega stream equal to the
    numpy oracle's generator bitwise."""
    import ctypes as C
    L = c_h2.lib()
    for line in open(os.path.join(GOLDEN, "philox4x32_10_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        w = [int(x, 16) for x in line.split()]
        ctr = np.array(w[:4], np.uint32)
        key = np.array(w[4:6], np.uint32)
        out = np.empty(4, np.uint32)
        L.h2o_philox4x32_10(C.c_void_p(ctr.ctypes.data), C.c_void_p(key.ctypes.data), C.c_void_p(out.ctypes.data))
        assert list(out) == w[6:10]
    assert np.array_equal(c_h2.omega(11, 3, 7, 500, 5, 37), rng.omega_block(11, 3, 7, 500, 5, 37))


def test_rational_kernel_closed_form():
    """K = 1 / (1 + r^2 / l^2): 1 at r = 0, 1/2 at r = l, 1/5 at r = 2l (exact in binary)."""
    tree, part, ta = setup(np.array([[0.0, 0, 0], [0.5, 0, 0], [0.0, 1.0, 0]]), 4)
    K = c_h2.kernel_block(ta, "rational", 0.5, np.arange(3), np.arange(3))
    P = ta.pts
    for i in range(3):
        for j in range(3):
            r2 = float(np.sum((P[i] - P[j]) ** 2))
            assert K[i, j] == {0.0: 1.0, 0.25: 0.5, 1.0: 0.2, 1.25: 1.0 / 6.0}[r2]


@pytest.mark.parametrize("d,m,seed", [(40, 25, 0), (16, 30, 1), (64, 64, 2), (8, 8, 3)])
def test_cpqr_pivots_match_lapack_dgeqp3(d, m, seed):
    rg = np.random.default_rng(seed)
    A = rg.standard_normal((d, m)) * (0.7 ** np.arange(m))[rg.permutation(m)]   # no near-ties
    k, perm, F, cert = c_h2.cpqr(A.T, 0.0)
    _, R2, P2 = sla.qr(A, pivoting=True, mode="economic")
    kk = min(d, m)
    assert k == kk
    assert np.array_equal(perm[:kk], P2[:kk])
    rdiag = np.abs(np.array([F[i, i] for i in range(kk)]))
    assert np.allclose(rdiag, np.abs(np.diag(R2))[:kk], rtol=1e-12, atol=0)
    assert cert[0] > 0                       # gap certificate of a tie-free matrix


@pytest.mark.parametrize("case", ["cov2d_1k", "cov3d_2k", "ie_8cube", "rational_2k"])
def test_whole_build_error_vs_dense(case):
    """BASELINE north_star: relative Frobenius / 2-norm error vs dense K <= tol (brute force),
    identity rows, nested skeletons (L230, L253)."""
    X, kind, p, leaf, tol = {
        "cov2d_1k": (uniform_points(1024, 2, 0), "exp", 0.2, 32, 1e-6),
        "cov3d_2k": (uniform_points(2048, 3, 0), "exp", 0.2, 64, 1e-6),
        "ie_8cube": (grid_points((8, 8, 8), 1 / 8), "helmholtz", 3.0, 16, 1e-4),
        "rational_2k": (uniform_points(2048, 3, 1), "rational", 0.3, 64, 1e-6)}[case]
    tree, part, ta = setup(X, leaf)
    R = c_h2.build(ta, kind, p, tol)
    H = R.to_h2matrix()
    K = c_h2.kernel_block(ta, kind, p, np.arange(tree.n), np.arange(tree.n))
    if kind != "rational":
        assert np.allclose(K, kernels.KernelOperator(kind, p, X[tree.perm]).dense(), rtol=1e-14, atol=1e-14)
    Kh = oh2.to_dense(H)
    assert np.linalg.norm(Kh - K) <= tol * np.linalg.norm(K)
    assert np.linalg.norm(Kh - K, 2) <= tol * np.linalg.norm(K, 2)
    Dl = tree.leaf_depth
    for t in H.rank:
        for c, Xc in enumerate(H.X[t]):
            k = H.rank[t][c]
            if t == Dl:
                ibar = np.arange(tree.begin[t][c], tree.end[t][c])
            else:
                ibar = np.concatenate([H.skel[t + 1][2 * c], H.skel[t + 1][2 * c + 1]])
            J = np.array([np.where(ibar == s)[0][0] for s in H.skel[t][c]], np.int64)
            assert np.array_equal(Xc[J], np.eye(k))
            assert set(H.skel[t][c]) <= set(ibar)


@pytest.mark.parametrize("seed", [0, 1])
def test_known_rank_recovery(seed):
    """Exact recovery of a synthetic H^2 of known ranks (BASELINE north_star): ranks equal,
    error <= 1e-10."""
    X = uniform_points(1024, 3, 10 + seed)
    tree, part, ta = setup(X, 32)
    K, ranks, active = synthetic_h2(tree, part, lambda t, m: min(m, 6 + (t % 3) * 2), seed)
    nu = np.linalg.norm(K, 2)
    R = c_h2.build(ta, "table", 0.0, 1e-12, dense=K, d_init=max(int(r.max()) for r in ranks.values()) + 8,
                   adaptive=False, tol_rule="literal", norm=nu)
    for t in R.rank:
        assert np.array_equal(R.rank[t], np.where(active[t], ranks[t], 0)), t
    assert np.linalg.norm(oh2.to_dense(R.to_h2matrix()) - K) <= 1e-10 * np.linalg.norm(K)


def test_adaptive_round_count_closed_form():
    """Leaf far field of exact rank 12, d_init = d_blk = 8, p_os = 10: the test (R12) passes at
    the first d >= r + 1 + p_os = 23, i.e. d = 24 after 3 tests."""
    X = uniform_points(1024, 3, 3)
    tree, part, ta = setup(X, 64)
    K, ranks, active = synthetic_h2(tree, part, lambda t, m: min(m, 12), 3)
    R = c_h2.build(ta, "table", 0.0, 1e-10, dense=K, d_init=8, d_blk=8, d_max=64, p_os=10)
    Dl = tree.leaf_depth
    assert R.rounds[Dl] == 3
    assert np.all(R.rank[Dl][active[Dl]] == 12)
    with pytest.raises(c_h2.NotConverged):
        c_h2.build(ta, "table", 0.0, 1e-10, dense=K, d_init=8, d_blk=8, d_max=16)


def test_rank_one_zero_and_exact_sketch():
    X = uniform_points(512, 3, 6)
    tree, part, ta = setup(X, 32)
    v = np.random.default_rng(0).standard_normal(512)
    K = np.outer(v, v)
    R = c_h2.build(ta, "table", 0.0, 1e-8, dense=K)
    for t in R.rank:
        assert set(np.unique(R.rank[t])) <= {0, 1}
    assert np.linalg.norm(oh2.to_dense(R.to_h2matrix()) - K) <= 1e-13 * np.linalg.norm(K)
    R0 = c_h2.build(ta, "table", 0.0, 1e-8, dense=np.zeros((512, 512)))
    assert all(np.all(R0.rank[t] == 0) for t in R0.rank)
    # tol = 0, d >= N: every ID exact, H == K to roundoff
    X = uniform_points(256, 3, 2)
    tree, part, ta = setup(X, 16)
    R = c_h2.build(ta, "exp", 0.2, 0.0, d_init=256, adaptive=False)
    K = kernels.KernelOperator("exp", 0.2, X[tree.perm]).dense()
    assert np.linalg.norm(oh2.to_dense(R.to_h2matrix()) - K) <= 1e-12 * np.linalg.norm(K)


@pytest.mark.parametrize("case,adaptive", [("cov2d_1k", True), ("cov2d_1k", False), ("cov3d_3k", True),
                                           ("ie_8cube", True)])
def test_agrees_with_numpy_oracle(case, adaptive):
    """Two independent implementations of Algorithm 1 on the same tree and Omega stream: ranks,
    skeletons and sample counts equal (a pivot may flip only at a near-tie certified by the numpy
    oracle, 1e-7), H^2 matvecs within 1e-10."""
    X, kind, p, leaf, tol = {
        "cov2d_1k": (uniform_points(1024, 2, 0), "exp", 0.2, 32, 1e-6),
        "cov3d_3k": (uniform_points(3000, 3, 4), "exp", 0.2, 64, 1e-6),
        "ie_8cube": (grid_points((8, 8, 8), 1 / 8), "helmholtz", 3.0, 16, 1e-4)}[case]
    tree, part, ta = setup(X, leaf)
    op = kernels.KernelOperator(kind, p, X[tree.perm])
    om = lambda c0, nc: rng.omega_block(1, 0, 0, tree.n, c0, nc)
    opts = dict(adaptive=adaptive) if adaptive else dict(adaptive=False, d_init=64)
    Ho = oh2.build(tree, part, op.sampler, op.entry, om, tol, oh2.BuildOpts(**opts))
    R = c_h2.build(ta, kind, p, tol, **opts)
    Hc = R.to_h2matrix()
    diverged = set()
    mism = 0
    for t in range(Ho.top, tree.leaf_depth + 1):
        for c in range(1 << t):
            if t < tree.leaf_depth and ({(t + 1, 2 * c), (t + 1, 2 * c + 1)} & diverged):
                diverged.add((t, c))
                continue
            if Hc.rank[t][c] != Ho.rank[t][c] or not np.array_equal(Hc.skel[t][c], Ho.skel[t][c]):
                ido = Ho.ids[t][c]
                assert ido.min_gap < 1e-7 or ido.stop_margin < 1e-7, (t, c)
                diverged.add((t, c))
                mism += 1
    if mism == 0:
        assert R.samples == Ho.samples
        x = np.random.default_rng(3).standard_normal((tree.n, 5))
        yc, yo = oh2.matvec(Hc, x), oh2.matvec(Ho, x)
        assert np.linalg.norm(yc - yo) <= 1e-10 * np.linalg.norm(yo)


def test_thread_count_invariance():
    """Each output element is computed by one thread in the stated order: the build is bitwise
    independent of the OpenMP thread count."""
    X = uniform_points(3000, 3, 4)
    tree, part, ta = setup(X, 64)
    R1 = c_h2.build(ta, "exp", 0.2, 1e-6, threads=1)
    R4 = c_h2.build(ta, "exp", 0.2, 1e-6, threads=4)
    assert R1.samples == R4.samples
    for t in R1.rank:
        for a in ("rank", "skel", "basis", "cert", "B"):
            assert np.array_equal(getattr(R1, a)[t], getattr(R4, a)[t])
    assert np.array_equal(R1.D, R4.D)


def test_external_gaussian_omega():
    """An external (here Gaussian) Omega replaces the Philox stream (PAPER.md L203 'a random
    matrix'): the build still meets tol against dense K."""
    X = uniform_points(1024, 2, 0)
    tree, part, ta = setup(X, 32)
    G = np.random.default_rng(9).standard_normal((tree.n, 512))
    R = c_h2.build(ta, "exp", 0.2, 1e-6, omega_ext=G)
    K = kernels.KernelOperator("exp", 0.2, X[tree.perm]).dense()
    assert np.linalg.norm(oh2.to_dense(R.to_h2matrix()) - K) <= 1e-6 * np.linalg.norm(K)
