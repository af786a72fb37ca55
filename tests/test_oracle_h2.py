"""Pins for oracle/h2.py (Algorithm 1, PAPER.md L196-263 / §III)."""
import numpy as np
import pytest
from oracle import geometry, kernels, h2, rng
from oracle.cpqr import row_id
from synth import uniform_points, grid_points
from synthetic_h2 import synthetic_h2


def setup(X, leaf, eta=0.7):
    tree = geometry.build_cluster_tree(X, leaf)
    part = geometry.build_partition(tree, eta)
    om = lambda c0, nc: rng.omega_block(1, 0, 0, tree.n, c0, nc)
    return tree, part, om


def kernel_build(X, kind, param, leaf, tol, **kw):
    tree, part, om = setup(X, leaf)
    op = kernels.KernelOperator(kind, param, X[tree.perm])
    H = h2.build(tree, part, op.sampler, op.entry, om, tol, h2.BuildOpts(**kw))
    return H, op


@pytest.mark.parametrize("case", ["cov2d_1k", "cov3d_2k", "ie_8cube"])
def test_whole_build_error_vs_dense(case):
    """BASELINE north_star: relative Frobenius error vs dense A <= tol on tiny inputs (brute force)."""
    if case == "cov2d_1k":
        X, kind, p, leaf, tol = uniform_points(1024, 2, 0), "exp", 0.2, 32, 1e-6
    elif case == "cov3d_2k":
        X, kind, p, leaf, tol = uniform_points(2048, 3, 0), "exp", 0.2, 64, 1e-6
    else:
        X, kind, p, leaf, tol = grid_points((8, 8, 8), 1 / 8), "helmholtz", 3.0, 16, 1e-4
    H, op = kernel_build(X, kind, p, leaf, tol)
    K = op.dense()
    Kh = h2.to_dense(H)
    assert np.linalg.norm(Kh - K) <= tol * np.linalg.norm(K)
    assert np.linalg.norm(Kh - K, 2) <= tol * np.linalg.norm(K, 2)
    # matvec agrees with the dense reconstruction
    x = np.random.default_rng(1).standard_normal((K.shape[0], 4))
    assert np.linalg.norm(h2.matvec(H, x) - Kh @ x) <= 1e-12 * np.linalg.norm(Kh @ x)
    # identity rows and nested skeletons (L230, L253)
    Dl = H.tree.leaf_depth
    for t in H.rank:
        for c, Xc in enumerate(H.X[t]):
            J = H.ids[t][c].J
            assert np.array_equal(Xc[J], np.eye(len(J)))
            if t == Dl:
                assert set(H.skel[t][c]) <= set(range(H.tree.begin[t][c], H.tree.end[t][c]))
            else:
                assert set(H.skel[t][c]) <= set(H.skel[t + 1][2 * c]) | set(H.skel[t + 1][2 * c + 1])


@pytest.mark.parametrize("seed", [0, 1])
def test_known_rank_recovery(seed):
    """Exact recovery of a synthetic H^2 of known ranks (BASELINE north_star)."""
    X = uniform_points(1024, 3, 10 + seed)
    tree, part, om = setup(X, 32)
    rank_of = lambda t, m: min(m, 6 + (t % 3) * 2)
    K, ranks, active = synthetic_h2(tree, part, rank_of, seed)
    nu = np.linalg.norm(K, 2)
    sampler = lambda O: K @ O
    entry = lambda r, c: K[np.ix_(r, c)]
    H = h2.build(tree, part, sampler, entry, om, 1e-12,
                 h2.BuildOpts(d_init=max(int(r.max()) for r in ranks.values()) + 8, adaptive=False,
                              tol_rule="literal", norm=nu))
    for t in H.rank:
        expect = np.where(active[t], ranks[t], 0)
        assert np.array_equal(H.rank[t], expect), t
    assert np.linalg.norm(h2.to_dense(H) - K) <= 1e-10 * np.linalg.norm(K)


def test_adaptive_round_count_closed_form():
    """Leaf far field of exact rank r: the convergence test (R12) passes at the first
    d >= r + 1 + p_os; with d_init = d_blk = 8, r = 12, p_os = 10: d = 24, i.e. 3 tests."""
    X = uniform_points(1024, 3, 3)
    tree, part, om = setup(X, 64)
    K, ranks, active = synthetic_h2(tree, part, lambda t, m: min(m, 12), 3)
    H = h2.build(tree, part, lambda O: K @ O, lambda r, c: K[np.ix_(r, c)], om, 1e-10,
                 h2.BuildOpts(d_init=8, d_blk=8, d_max=64, p_os=10))
    Dl = tree.leaf_depth
    assert H.rounds[Dl] == 3
    assert np.all(H.rank[Dl][active[Dl]] == 12)


def test_not_converged_reports_level():
    X = uniform_points(1024, 3, 3)
    tree, part, om = setup(X, 64)
    K, _, _ = synthetic_h2(tree, part, lambda t, m: min(m, 30), 4)
    with pytest.raises(h2.NotConverged) as e:
        h2.build(tree, part, lambda O: K @ O, lambda r, c: K[np.ix_(r, c)], om, 1e-10,
                 h2.BuildOpts(d_init=8, d_blk=8, d_max=24))
    assert e.value.depth == tree.leaf_depth


def test_exact_sketch_reproduces_K():
    """tol = 0, d >= N: every ID is exact, so H == K to roundoff."""
    X = uniform_points(256, 3, 2)
    tree, part, om = setup(X, 16)
    op = kernels.KernelOperator("exp", 0.2, X[tree.perm])
    H = h2.build(tree, part, op.sampler, op.entry, om, 0.0, h2.BuildOpts(d_init=256, adaptive=False))
    K = op.dense()
    assert np.linalg.norm(h2.to_dense(H) - K) <= 1e-12 * np.linalg.norm(K)


def test_rank_one_and_zero_operators():
    X = uniform_points(512, 3, 6)
    tree, part, om = setup(X, 32)
    v = np.random.default_rng(0).standard_normal(512)
    K = np.outer(v, v)
    H = h2.build(tree, part, lambda O: K @ O, lambda r, c: K[np.ix_(r, c)], om, 1e-8)
    for t in H.rank:
        assert set(np.unique(H.rank[t])) <= {0, 1}
    assert np.linalg.norm(h2.to_dense(H) - K) <= 1e-13 * np.linalg.norm(K)
    Z = np.zeros((512, 512))
    H0 = h2.build(tree, part, lambda O: Z @ O, lambda r, c: Z[np.ix_(r, c)], om, 1e-8)
    assert all(np.all(H0.rank[t] == 0) for t in H0.rank)
    assert np.all(h2.to_dense(H0) == 0)


def test_all_dense_and_single_leaf():
    X = uniform_points(300, 3, 8)
    tree = geometry.build_cluster_tree(X, 64)
    part = geometry.build_partition(tree, 1e-12)        # eta -> 0: every leaf pair dense
    om = lambda c0, nc: rng.omega_block(1, 0, 0, tree.n, c0, nc)
    op = kernels.KernelOperator("exp", 0.2, X[tree.perm])
    H = h2.build(tree, part, op.sampler, op.entry, om, 1e-6)
    assert np.all(H.rank[tree.leaf_depth] == 0)          # Y^loc == 0 up to roundoff
    assert np.array_equal(h2.to_dense(H), op.dense())
    t1 = geometry.build_cluster_tree(X[:40], 64)
    p1 = geometry.build_partition(t1, 0.7)
    op1 = kernels.KernelOperator("exp", 0.2, X[:40][t1.perm])
    H1 = h2.build(t1, p1, op1.sampler, op1.entry, lambda c0, nc: rng.omega_block(1, 0, 0, 40, c0, nc), 1e-6)
    assert np.array_equal(h2.to_dense(H1), op1.dense())


def test_leaf_subtraction_brute_force():
    """Y^loc_tau = sum_{b not in N_tau} K(I_tau, I_b) Omega_b (SURVEY 8c pin)."""
    X = uniform_points(2048, 3, 1)
    tree, part, om = setup(X, 64)
    op = kernels.KernelOperator("exp", 0.2, X[tree.perm])
    Om = om(0, 16)
    Y = op.sampler(Om)
    Dl = tree.leaf_depth
    D = {(int(s), int(b)): op.entry(np.arange(tree.begin[Dl][s], tree.end[Dl][s]),
                                    np.arange(tree.begin[Dl][b], tree.end[Dl][b])) for s, b in part.near}
    Yl, Ol = h2.leaf_local_samples(tree, part, D, Y, Om)
    K = op.dense()
    for tau in (0, 5, 31):
        I = slice(tree.begin[Dl][tau], tree.end[Dl][tau])
        mask = np.ones(tree.n, bool)
        for b in part.near_of(tau):
            mask[tree.begin[Dl][b]:tree.end[Dl][b]] = False
        ref = K[I][:, mask] @ Om[mask]
        assert np.linalg.norm(Yl[tau] - ref) <= 1e-12 * np.linalg.norm(Y[I])


def test_weak_admissibility_is_hss():
    """eta -> inf: F_tau = {sibling}, N_tau = {tau}; Algorithm 1 reduces to the HSS sketching
    construction it extends: every level is processed and error <= tol."""
    X = uniform_points(512, 1, 0)
    tree = geometry.build_cluster_tree(X, 32)
    part = geometry.build_partition(tree, 1e12)
    om = lambda c0, nc: rng.omega_block(1, 0, 0, tree.n, c0, nc)
    op = kernels.KernelOperator("exp", 0.2, X[tree.perm])
    H = h2.build(tree, part, op.sampler, op.entry, om, 1e-6)
    assert H.top == 1
    K = op.dense()
    assert np.linalg.norm(h2.to_dense(H) - K) <= 1e-6 * np.linalg.norm(K)


def test_deterministic():
    X = uniform_points(1024, 2, 0)
    H1, _ = kernel_build(X, "exp", 0.2, 32, 1e-6)
    H2, _ = kernel_build(X, "exp", 0.2, 32, 1e-6)
    for t in H1.rank:
        assert np.array_equal(H1.rank[t], H2.rank[t])
        for a, b in zip(H1.X[t], H2.X[t]):
            assert np.array_equal(a, b)


def test_eps_decay_schedule_leaf_identity_and_monotone_parent():
    """R31 level schedule: the leaf threshold is unchanged (decay^0), so leaf ranks and skeletons
    equal the uniform build's; one level up the panels are identical, and a smaller threshold
    cannot truncate earlier, so ranks there are >= the uniform build's."""
    X = uniform_points(2048, 3, 0)
    tree, part, om = setup(X, 64)
    op = kernels.KernelOperator("exp", 0.2, X[tree.perm])
    kw = dict(adaptive=False, d_init=160)
    H1 = h2.build(tree, part, op.sampler, op.entry, om, 1e-6, h2.BuildOpts(**kw))
    Hg = h2.build(tree, part, op.sampler, op.entry, om, 1e-6, h2.BuildOpts(eps_decay=0.5, **kw))
    Dl = tree.leaf_depth
    assert np.array_equal(H1.rank[Dl], Hg.rank[Dl])
    assert all(np.array_equal(a, b) for a, b in zip(H1.skel[Dl], Hg.skel[Dl]))
    assert np.all(Hg.rank[Dl - 1] >= H1.rank[Dl - 1]) and Hg.rank[Dl - 1].sum() > H1.rank[Dl - 1].sum()
