"""Pins for oracle/h2_nonsym.py (non-symmetric Algorithm 1, PAPER.md L145 / SURVEY §8(f) NEXT #3)."""
import numpy as np
import pytest
from oracle import geometry, kernels, h2, h2_nonsym, rng
from synth import uniform_points
from synthetic_h2 import synthetic_h2_nonsym


def setup(X, leaf, eta=0.7):
    tree = geometry.build_cluster_tree(X, leaf)
    part = geometry.build_partition(tree, eta)
    om = lambda c0, nc: rng.omega_block(1, 0, 0, tree.n, c0, nc)
    ps = lambda c0, nc: rng.omega_block(1, 1, 0, tree.n, c0, nc)
    return tree, part, om, ps


def test_symmetric_input_reduces_to_symmetric_construction():
    """K = K^T and Psi = Omega: Z = Y, both sides run the symmetric construction, so ranks,
    skeletons and the compressed matrix equal those of oracle/h2.build."""
    X = uniform_points(1024, 3, 0)
    tree, part, om, _ = setup(X, 64)
    op = kernels.KernelOperator("exp", 0.2, X[tree.perm])
    Hs = h2.build(tree, part, op.sampler, op.entry, om, 1e-6)
    Hn = h2_nonsym.build_nonsym(tree, part, op.sampler, op.sampler, op.entry, om, om, 1e-6)
    assert Hn.samples == Hs.samples
    for t in Hs.rank:
        assert np.array_equal(Hn.rank_r[t], Hs.rank[t]) and np.array_equal(Hn.rank_c[t], Hs.rank[t])
        for c in range(1 << t):
            assert np.array_equal(Hn.skel_r[t][c], Hs.skel[t][c])
            assert np.array_equal(Hn.skel_c[t][c], Hs.skel[t][c])
    K = h2.to_dense(Hs)
    assert np.linalg.norm(h2_nonsym.to_dense_nonsym(Hn) - K) <= 1e-12 * np.linalg.norm(K)


def _far_rows(tree, part, t, c):
    """Indices of every cluster admissible to c or to an ancestor of c at depth <= t."""
    out = []
    for u in range(part.top_depth(), t + 1):
        a = c >> (t - u)
        for b in part.far_of(u, a):
            out.append(np.arange(tree.begin[u][b], tree.end[u][b]))
    return np.concatenate(out) if out else np.zeros(0, np.int64)


def _numrank(A):
    if A.size == 0:
        return 0
    s = np.linalg.svd(A, compute_uv=False)
    return int(np.sum(s > 1e-9 * s[0])) if s[0] > 0 else 0


def test_exact_nonsym_h2_recovered():
    """A random non-symmetric H^2 matrix with different row and column ranks (5 / 9 at the
    leaves): the non-adaptive build at d > max rank finds, for every cluster c at depth t, row
    rank = numerical rank of K(I_c, far(c)) and column rank = that of K(far(c), I_c) (brute-force
    SVD of the far-field blocks, far(c) = clusters admissible to c or an ancestor), which differ,
    and reproduces K and K x to rounding."""
    X = uniform_points(2048, 2, 2)
    tree, part, om, ps = setup(X, 32)
    K, rr, rc, active = synthetic_h2_nonsym(tree, part, lambda t, m: min(m, 5 if t == tree.leaf_depth else 7),
                                            lambda t, m: min(m, 9 if t == tree.leaf_depth else 11), 5)
    nu = np.linalg.norm(K, 2)
    H = h2_nonsym.build_nonsym(tree, part, lambda O: K @ O, lambda P: K.T @ P,
                               lambda r, c: K[np.ix_(r, c)], om, ps, 1e-12,
                               h2.BuildOpts(d_init=40, adaptive=False, tol_rule="literal", norm=nu))
    differ = False
    for t in H.rank_r:
        for c in range(1 << t):
            I = np.arange(tree.begin[t][c], tree.end[t][c])
            F = _far_rows(tree, part, t, c)
            assert H.rank_r[t][c] == _numrank(K[np.ix_(I, F)]) <= rr[t][c], (t, c)
            assert H.rank_c[t][c] == _numrank(K[np.ix_(F, I)]) <= rc[t][c], (t, c)
            differ |= H.rank_r[t][c] != H.rank_c[t][c]
    assert differ
    Kh = h2_nonsym.to_dense_nonsym(H)
    assert np.linalg.norm(Kh - K) <= 1e-10 * np.linalg.norm(K)
    x = np.random.default_rng(0).standard_normal((K.shape[0], 3))
    assert np.linalg.norm(h2_nonsym.matvec_nonsym(H, x) - K @ x) <= 1e-10 * np.linalg.norm(K @ x)


def test_transposed_input_swaps_sides():
    """Building K^T (sampler and transposed sampler swapped, Omega and Psi swapped) gives the
    column side of K's build as its row side and vice versa; the result is (K_h)^T."""
    X = uniform_points(1024, 2, 4)
    tree, part, om, ps = setup(X, 32)
    K, _, _, _ = synthetic_h2_nonsym(tree, part, lambda t, m: min(m, 4), lambda t, m: min(m, 8), 6)
    kw = dict(opts=h2.BuildOpts(d_init=16, d_blk=16))
    A = h2_nonsym.build_nonsym(tree, part, lambda O: K @ O, lambda P: K.T @ P, lambda r, c: K[np.ix_(r, c)],
                               om, ps, 1e-8, **kw)
    B = h2_nonsym.build_nonsym(tree, part, lambda O: K.T @ O, lambda P: K @ P, lambda r, c: K.T[np.ix_(r, c)],
                               ps, om, 1e-8, **kw)
    for t in A.rank_r:
        assert np.array_equal(A.rank_r[t], B.rank_c[t]) and np.array_equal(A.rank_c[t], B.rank_r[t])
    assert np.allclose(h2_nonsym.to_dense_nonsym(A), h2_nonsym.to_dense_nonsym(B).T, rtol=0, atol=1e-12 * np.abs(K).max())


@pytest.mark.parametrize("v", [0.0, 2.0])
def test_nonsym_kernel_error_vs_dense(v):
    """exp(-|x-y|/l) (1 + v (x_0 - y_0)): a non-symmetric kernel (antisymmetric first-order
    term); the adaptive build meets the BASELINE error bound against dense K."""
    X = uniform_points(2048, 3, 1)
    tree, part, om, ps = setup(X, 64)
    P = X[tree.perm]
    def blk(r, c):
        d = np.sqrt(((P[r][:, None, :] - P[c][None, :, :]) ** 2).sum(-1))
        return np.exp(-d / 0.2) * (1 + v * (P[r][:, None, 0] - P[c][None, :, 0]))
    K = blk(np.arange(tree.n), np.arange(tree.n))
    tol = 1e-6
    H = h2_nonsym.build_nonsym(tree, part, lambda O: K @ O, lambda Q: K.T @ Q, blk, om, ps, tol)
    Kh = h2_nonsym.to_dense_nonsym(H)
    assert np.linalg.norm(Kh - K) <= tol * np.linalg.norm(K)
    if v:
        Dl = tree.leaf_depth
        assert not np.array_equal(H.rank_r[Dl], H.rank_c[Dl]) or any(
            not np.array_equal(H.skel_r[Dl][c], H.skel_c[Dl][c]) for c in range(1 << Dl))
