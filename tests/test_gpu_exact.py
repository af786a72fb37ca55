"""Exact-order parity (SURVEY §8(c) parity contract 2): libh2 with opts.exact_order = 1 on the
rational test kernel K = 1 / (1 + r^2 / l^2) and the exactly representable Omega stream performs
every floating-point operation of Algorithm 1 in the order the C oracle (oracle/c/h2oracle.c)
states, so ranks, skeletons I~, bases U / [E1; E2], couplings B, dense blocks D, CPQR certificates
and the sample count are BITWISE equal -- the skeleton / index bookkeeping is proven independent
of rounding (PAPER.md L165-173 ID, L283 identity rows, L230 merge).  Both sides consume the same
partition: the oracle's tree imported into libh2 (h2_tree_import).  Run with  pytest -m gpu."""
import numpy as np
import pytest
import torch

from oracle import geometry, c_h2
from synth import uniform_points, grid_points
import paper_2506_16759_b200 as g
from paper_2506_16759_b200 import _lib as L

pytestmark = pytest.mark.gpu

CASES = {
    # 2D, BASELINE configs[0] shape (N = 1024, leaf 32)
    "rat2d_1k": (lambda: uniform_points(1024, 2, 0), 0.3, 32, 1e-6),
    # 3D, ragged leaves (3000 = 46.875 x 64), several levels
    "rat3d_3000": (lambda: uniform_points(3000, 3, 4), 0.3, 64, 1e-6),
    # 3D, N = 4096, the largest exact-order case
    "rat3d_4096": (lambda: uniform_points(4096, 3, 7), 0.4, 64, 1e-7),
    # regular grid (equal coordinates, tie-prone pivots and admissibility)
    "rat_grid16": (lambda: grid_points((16, 16, 16), 1 / 16), 0.3, 64, 1e-5),
}


def imported(X, leaf):
    tree = geometry.build_cluster_tree(X, leaf)
    part = geometry.build_partition(tree, 0.7)
    T = g.Tree.from_partition(X, tree.perm, tree.begin, tree.end, part.near, part.far)
    return tree, part, T


def assert_bitwise(Hg, R, T):
    assert Hg.samples == R.samples
    assert Hg.top_depth == R.top
    for t in range(R.top, T.leaf_depth + 1):
        assert np.array_equal(Hg.rank(t), R.rank[t].astype(np.int64)), t
        assert np.array_equal(Hg._export(L.H2_X_SKEL, t, np.int32), R.skel[t]), t
        assert np.array_equal(Hg._export(L.H2_X_BASIS, t), R.basis[t]), t
        assert np.array_equal(Hg._export(L.H2_X_B, t), R.B[t]), t
        assert np.array_equal(Hg._export(L.H2_X_CERT, t), R.cert[t].reshape(-1)), t
        assert Hg.stats["rounds"][t] == R.rounds[t], t
    assert np.array_equal(Hg._export(L.H2_X_D), R.D)


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("mode", ["adaptive", "fixed", "literal"])
def test_exact_order_bitwise(case, mode):
    mk, l, leaf, tol = CASES[case]
    X = mk()
    tree, part, T = imported(X, leaf)
    ta = c_h2.TreeArrays(tree, part, X)
    opts = {"adaptive": dict(d_init=16, d_blk=16),
            "fixed": dict(adaptive=False, d_init=96),
            "literal": dict(tol_rule="literal", norm=float(len(X)) * 0.05, d_init=16, d_blk=8)}[mode]
    R = c_h2.build(ta, "rational", l, tol, **opts)
    Hg = g.build(T, ("rational", l), tol, exact_order=1, **opts)
    assert Hg.stats["cpqr_variants"] == L.H2_CQ_V_EXACT
    assert_bitwise(Hg, R, T)
    # and the representation is an accurate H^2 of K (bound of the adaptive north star)
    if mode == "adaptive" and len(X) <= 3000:
        K = c_h2.kernel_block(ta, "rational", l, np.arange(tree.n), np.arange(tree.n))
        x = np.random.default_rng(2).standard_normal((tree.n, 8))
        y = Hg.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
        assert np.linalg.norm(y - K @ x) <= 2 * tol * np.linalg.norm(K @ x)


def test_exact_order_sketch_and_tree_import():
    """The exact-order sketch equals the C oracle's sketch bitwise (any Omega, ragged row range),
    and the imported partition exports what the oracle built."""
    X = uniform_points(2500, 3, 9)
    tree, part, T = imported(X, 64)
    ta = c_h2.TreeArrays(tree, part, X)
    assert np.array_equal(T.perm, tree.perm)
    assert np.array_equal(T.near, part.near)
    assert all(np.array_equal(a, b) for a, b in zip(T.far, part.far))
    Om = np.random.default_rng(1).standard_normal((T.n, 37))
    ref = c_h2.dense_sketch(ta, "rational", 0.3, Om, rows=(101, 2222))
    got = g.dense_sketch(T, torch.from_numpy(Om).cuda(), ("rational", 0.3), 101, 2222).cpu().numpy()
    assert np.array_equal(got, ref)


def test_exact_order_deterministic_and_omega_external():
    """External Omega (h2_build_opts.omega_ext): exactly representable values (the stream read
    back) give the bitwise same build as the stream itself."""
    X = uniform_points(2000, 3, 3)
    tree, part, T = imported(X, 64)
    H1 = g.build(T, ("rational", 0.3), 1e-6, exact_order=1)
    Om = g.omega(T.n, 512)
    H2 = g.build(T, ("rational", 0.3), 1e-6, exact_order=1, omega=Om)
    assert H1.samples == H2.samples
    for t in range(H1.top_depth, T.leaf_depth + 1):
        assert np.array_equal(H1._export(L.H2_X_SKEL, t, np.int32), H2._export(L.H2_X_SKEL, t, np.int32))
        for w in (L.H2_X_BASIS, L.H2_X_B):
            assert np.array_equal(H1._export(w, t), H2._export(w, t))
    assert np.array_equal(H1._export(L.H2_X_D), H2._export(L.H2_X_D))


def compare_with_c(Hg, R, T, cert_tol=1e-7):
    """Production kernels vs the C oracle on the same tree and Omega: ranks and skeletons
    bit-exact, a mismatch accepted only where the oracle's CPQR decision was a certified near-tie
    (gap or margin < cert_tol); ancestors of a diverged cluster are compared by error only.
    Returns (#certified, #compared, diverged masks)."""
    Dl = T.leaf_depth
    div = {Dl + 1: np.zeros(1 << (Dl + 1), bool)}
    certified = compared = 0
    for t in range(Dl, R.top - 1, -1):
        rg = Hg.rank(t)
        sg = Hg.skel(t)
        so = np.split(R.skel[t].astype(np.int64), np.cumsum(R.rank[t])[:-1])
        d = np.zeros(1 << t, bool)
        for c in range(1 << t):
            if t < Dl and (div[t + 1][2 * c] or div[t + 1][2 * c + 1]):
                d[c] = True
                continue
            compared += 1
            if rg[c] != R.rank[t][c] or not np.array_equal(sg[c], so[c]):
                gap, margin = R.cert[t][c]
                assert gap < cert_tol or margin < cert_tol, (t, c, gap, margin)
                certified += 1
                d[c] = True
        div[t] = d
    return certified, compared, div


def test_gaussian_omega_external_vs_c_oracle():
    """A Gaussian Omega ("a random matrix"; SURVEY Z8 reading) supplied to both paths
    (h2_build_opts.omega_ext / the C oracle's omega_ext): the production path (FP64 DMMA sketch for
    an arbitrary Omega, tensor-core-free) against the C oracle -- skeletons bit-exact or certified,
    equal samples, D bitwise-close, probe error <= 2 tol."""
    X = uniform_points(4000, 3, 5)
    tree, part, T = imported(X, 64)
    ta = c_h2.TreeArrays(tree, part, X)
    G = np.random.default_rng(13).standard_normal((T.n, 512))
    R = c_h2.build(ta, "exp", 0.2, 1e-6, omega_ext=G)
    Hg = g.build(T, ("exp", 0.2), 1e-6, omega=torch.from_numpy(G).cuda())
    certified, compared, div = compare_with_c(Hg, R, T)
    assert certified <= max(1, compared // 100)
    if certified == 0:
        assert Hg.samples == R.samples
    Dd = Hg._export(L.H2_X_D)
    assert np.abs(Dd - R.D).max() <= 32 * 2.2e-16
    K = c_h2.kernel_block(ta, "exp", 0.2, np.arange(T.n), np.arange(T.n))
    x = np.random.default_rng(2).standard_normal((T.n, 8))
    y = Hg.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.linalg.norm(y - K @ x) <= 2e-6 * np.linalg.norm(K @ x)


def test_literal_norm_by_power_iteration():
    """H2_TOL_LITERAL with norm <= 0: nu = ||K||_2 estimated through the sketch
    within 5 % of LAPACK's 2-norm at N = 4096 (SURVEY §8(c) pin), reported in stats.norm_est; the
    literal-rule build then uses it (same result as passing that nu explicitly)."""
    X = uniform_points(4096, 3, 0)
    T = g.Tree(X, 64)
    tree, part, _ = imported(X, 64)
    ta = c_h2.TreeArrays(tree, part, X)
    K = c_h2.kernel_block(ta, "exp", 0.2, np.arange(T.n), np.arange(T.n))
    nu = float(np.linalg.norm(K, 2))
    H = g.build(T, ("exp", 0.2), 1e-6, tol_rule="literal", norm=0.0, norm_iters=10)
    est = H.stats["norm_est"]
    assert abs(est - nu) <= 0.05 * nu, (est, nu)
    H2 = g.build(T, ("exp", 0.2), 1e-6, tol_rule="literal", norm=est)
    for t in range(H.top_depth, T.leaf_depth + 1):
        assert np.array_equal(H.rank(t), H2.rank(t))
