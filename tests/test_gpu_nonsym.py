"""Non-symmetric construction (h2_build_nonsym) through the
C ABI against oracle/h2_nonsym.py on the same seeded inputs: ranks and skeletons of BOTH sides
bit-exact or certified near-ties, interpolation bound on the oracle's panels, equal sample
counts, D blocks bitwise, probe error against the dense operator."""
import numpy as np
import pytest
import torch

from oracle import geometry, kernels, h2 as oh2, h2_nonsym as ons, rng
from synth import uniform_points
import paper_2506_16759_b200 as g
from gpu_helpers import CERT_TOL

pytestmark = pytest.mark.gpu


def nonsym_kernel(P, v, ell=0.2):
    """exp(-|x-y|/ell) (1 + v (x_0 - y_0)): non-symmetric (antisymmetric first-order term)."""
    d = np.sqrt(((P[:, None, :] - P[None, :, :]) ** 2).sum(-1))
    return np.exp(-d / ell) * (1 + v * (P[:, None, 0] - P[None, :, 0]))


def oracle_nonsym(tree, part, A, tol, seed=1, **opts):
    om = lambda c0, nc: rng.omega_block(seed, 0, 0, tree.n, c0, nc)
    ps = lambda c0, nc: rng.omega_block(seed, 1, 0, tree.n, c0, nc)
    return ons.build_nonsym(tree, part, lambda O: A @ O, lambda Q: A.T @ Q, lambda r, c: A[np.ix_(r, c)],
                            om, ps, tol, oh2.BuildOpts(**opts))


def compare_side(Hg, Ho, side):
    """compare_builds (gpu_helpers) for one side of the non-symmetric build."""
    ids = Ho.ids_c if side else Ho.ids_r
    skel = Ho.skel_c if side else Ho.skel_r
    panels = Ho.panels_c if side else Ho.panels_r
    Dl = Ho.tree.leaf_depth
    assert Hg.top_depth == Ho.top
    diverged = {Dl + 1: np.zeros(1 << (Dl + 1), bool)}
    certified = compared = 0
    for t in range(Dl, Ho.top - 1, -1):
        rg, sg, Xg = Hg.rank(t, side), Hg.skel(t, side), Hg.basis(t, side)
        div = np.zeros(1 << t, bool)
        for c in range(1 << t):
            if t < Dl and (diverged[t + 1][2 * c] or diverged[t + 1][2 * c + 1]):
                div[c] = True
                continue
            compared += 1
            ido = ids[t][c]
            if not (rg[c] == ido.k and np.array_equal(sg[c], skel[t][c])):
                assert ido.min_gap < CERT_TOL or ido.stop_margin < CERT_TOL, (side, t, c, rg[c], ido.k)
                certified += 1
                div[c] = True
                continue
            J = ido.J
            assert np.array_equal(Xg[c][J], np.eye(len(J)))
            P = panels[t][c]
            if P.size:
                res = np.linalg.norm(P - Xg[c] @ P[J])
                bound = np.sqrt(max(P.shape[0] - len(J), 0)) * Ho.eps
                assert res <= 1.01 * bound + 1e-12 * np.linalg.norm(P), (side, t, c, res, bound)
        diverged[t] = div
    return certified, compared


def setup(n, dim, leaf, seed):
    X = uniform_points(n, dim, seed)
    T = g.Tree(X, leaf)
    tree = geometry.build_cluster_tree(X, leaf)
    part = geometry.build_partition(tree, 0.7)
    assert np.array_equal(tree.perm, T.perm)
    return X, T, tree, part


@pytest.mark.parametrize("n,dim,leaf,v", [(2048, 3, 64, 2.0), (3000, 2, 48, 0.5)])
def test_nonsym_dense_operator_parity(n, dim, leaf, v):
    X, T, tree, part = setup(n, dim, leaf, 11)
    A = nonsym_kernel(X[tree.perm], v)
    tol = 1e-6
    Ho = oracle_nonsym(tree, part, A, tol)
    Ad = torch.from_numpy(A).cuda()
    Hg = g.build(T, ("exp", 0.2), tol, dense=Ad, nonsym=True)
    assert Hg.samples == Ho.samples
    tot_c = tot_n = 0
    for side in (0, 1):
        c, m = compare_side(Hg, Ho, side)
        tot_c, tot_n = tot_c + c, tot_n + m
    assert tot_c <= max(2, tot_n // 50)
    # D: every ordered near block, the operator's entries exactly
    D = Hg.D_blocks()
    Dl = tree.leaf_depth
    for (s, b) in list(D)[:64]:
        assert np.array_equal(D[(s, b)], A[tree.begin[Dl][s]:tree.end[Dl][s], tree.begin[Dl][b]:tree.end[Dl][b]])
    # B_{s,b} = A(I~_s, J~_b)
    for t in range(Hg.top_depth, Dl + 1):
        Bb = Hg.B_blocks(t)
        sr, sc = Hg.skel(t, 0), Hg.skel(t, 1)
        for (s, b) in list(Bb)[:32]:
            assert np.array_equal(Bb[(s, b)], A[np.ix_(sr[s], sc[b])])
    # accuracy against the dense operator, and the oracle's matvec of its own result
    P = np.random.default_rng(3).standard_normal((n, 6))
    y = Hg.matvec(torch.from_numpy(P).cuda()).cpu().numpy()
    ref = A @ P
    assert np.linalg.norm(y - ref) <= 2 * tol * np.linalg.norm(ref)
    yo = ons.matvec_nonsym(Ho, P)
    assert np.linalg.norm(y - yo) <= 2 * tol * np.linalg.norm(ref)


def test_nonsym_matvec_vs_oracle_structure():
    """The GPU matvec of a non-symmetric H^2 equals the dense reconstruction from its own
    exported U/E, V/F, B, D (oracle/h2_nonsym.to_dense_nonsym on the exported blocks)."""
    X, T, tree, part = setup(2048, 3, 64, 12)
    A = nonsym_kernel(X[tree.perm], 1.5)
    Hg = g.build(T, ("exp", 0.2), 1e-6, dense=torch.from_numpy(A).cuda(), nonsym=True)
    Dl = tree.leaf_depth
    H = ons.H2NonSym(tree, part, Hg.top_depth)
    for t in range(Hg.top_depth, Dl + 1):
        H.rank_r[t], H.rank_c[t] = Hg.rank(t, 0), Hg.rank(t, 1)
        H.Xr[t], H.Xc[t] = Hg.basis(t, 0), Hg.basis(t, 1)
        H.B[t] = Hg.B_blocks(t)
    H.D = Hg.D_blocks()
    K = ons.to_dense_nonsym(H)
    P = np.random.default_rng(4).standard_normal((tree.n, 5))
    y = Hg.matvec(torch.from_numpy(P).cuda()).cpu().numpy()
    assert np.linalg.norm(y - K @ P) <= 1e-12 * np.linalg.norm(K @ P)


def test_nonsym_builtin_kernel():
    """Built-in (symmetric) exp kernel through h2_build_nonsym: parity with the oracle's
    non-symmetric build of the same kernel (Psi = stream 1), error within tol."""
    X, T, tree, part = setup(2048, 3, 64, 13)
    op = kernels.KernelOperator("exp", 0.2, X[tree.perm])
    tol = 1e-6
    om = lambda c0, nc: rng.omega_block(1, 0, 0, tree.n, c0, nc)
    ps = lambda c0, nc: rng.omega_block(1, 1, 0, tree.n, c0, nc)
    Ho = ons.build_nonsym(tree, part, op.sampler, op.sampler, op.entry, om, ps, tol)
    Hg = g.build(T, ("exp", 0.2), tol, nonsym=True)
    assert Hg.samples == Ho.samples
    for side in (0, 1):
        c, m = compare_side(Hg, Ho, side)
        assert c <= max(2, m // 50)
    K = op.dense()
    P = np.random.default_rng(5).standard_normal((tree.n, 4))
    y = Hg.matvec(torch.from_numpy(P).cuda()).cpu().numpy()
    assert np.linalg.norm(y - K @ P) <= 2 * tol * np.linalg.norm(K @ P)


def test_nonsym_callbacks_exact_h2():
    """Sketch callback with the transpose flag and entry callback (row and column index arrays
    differ) on a random non-symmetric H^2 with row ranks != column ranks: the fixed-sample build
    recovers the oracle's ranks and skeletons on both sides (the oracle's ranks are pinned to the
    brute-force far-field ranks in tests/test_oracle_nonsym.py) and K to rounding."""
    from synthetic_h2 import synthetic_h2_nonsym
    X, T, tree, part = setup(2048, 2, 32, 14)
    Dl = tree.leaf_depth
    K, rr, rc, active = synthetic_h2_nonsym(tree, part, lambda t, m: min(m, 5 if t == Dl else 7),
                                            lambda t, m: min(m, 9 if t == Dl else 11), 5)
    Kd = torch.from_numpy(K).cuda()
    calls = {0: 0, 1: 0}

    def sketch(om, y, col0, r0, r1, transpose=0):
        calls[int(transpose)] += 1
        y.copy_((Kd.T if transpose else Kd)[r0:r1] @ om)

    def entry(b):
        n = b.nblocks
        view = lambda p, dt: g.device_view(p, (n,), (1,), dt)
        m, nc = view(b.m, torch.int32).cpu(), view(b.nc, torch.int32).cpu()
        ro, co = view(b.row_off, torch.int64).cpu(), view(b.col_off, torch.int64).cpu()
        outp = view(b.out, torch.int64).cpu()
        ridx = g.device_view(b.row_idx, (int((ro + m).max()),), (1,), torch.int32).long()
        cidx = g.device_view(b.col_idx, (int((co + nc).max()),), (1,), torch.int32).long()
        for q in range(n):
            rows = ridx[ro[q]:ro[q] + m[q]]
            cols = cidx[co[q]:co[q] + nc[q]]
            out = g.device_view(int(outp[q]), (int(m[q]), int(nc[q])), (int(nc[q]), 1))
            out.copy_(Kd[rows][:, cols])

    nu = float(np.linalg.norm(K, 2))
    opts = dict(d_init=40, adaptive=False, tol_rule=1, norm=nu)
    Hg = g.build(T, ("exp", 0.2), 1e-12, sketch=sketch, entry=entry, nonsym=True, **opts)
    assert calls[0] >= 1 and calls[1] >= 1
    om = lambda c0, nc: rng.omega_block(1, 0, 0, tree.n, c0, nc)
    ps = lambda c0, nc: rng.omega_block(1, 1, 0, tree.n, c0, nc)
    Ho = ons.build_nonsym(tree, part, lambda O: K @ O, lambda Q: K.T @ Q, lambda r, c: K[np.ix_(r, c)], om, ps,
                          1e-12, oh2.BuildOpts(d_init=40, adaptive=False, tol_rule="literal", norm=nu))
    for t in range(Hg.top_depth, Dl + 1):
        assert np.array_equal(Hg.rank(t, 0), Ho.rank_r[t]), t
        assert np.array_equal(Hg.rank(t, 1), Ho.rank_c[t]), t
    assert any(not np.array_equal(Hg.rank(t, 0), Hg.rank(t, 1)) for t in range(Hg.top_depth, Dl + 1))
    P = np.random.default_rng(6).standard_normal((tree.n, 3))
    y = Hg.matvec(torch.from_numpy(P).cuda()).cpu().numpy()
    assert np.linalg.norm(y - K @ P) <= 1e-9 * np.linalg.norm(K @ P)


def test_nonsym_column_exports_refused_on_symmetric():
    X = uniform_points(1024, 3, 1)
    T = g.Tree(X, 64)
    H = g.build(T, ("exp", 0.2), 1e-6)
    with pytest.raises(g.H2Error):
        H.rank(T.leaf_depth, 1)


def test_nonsym_degenerate_inputs():
    """n below one leaf (no admissible pair: D only) and a two-leaf problem: the non-symmetric
    build reproduces the operator exactly (every block is dense)."""
    for n, leaf in ((40, 64), (100, 64)):
        X = uniform_points(n, 3, 3)
        T = g.Tree(X, leaf)
        A = np.random.default_rng(n).standard_normal((n, n))
        Hg = g.build(T, ("exp", 0.2), 1e-6, dense=torch.from_numpy(A).cuda(), nonsym=True)
        P = np.random.default_rng(1).standard_normal((n, 3))
        y = Hg.matvec(torch.from_numpy(P).cuda()).cpu().numpy()
        assert np.allclose(y, A @ P, rtol=0, atol=1e-12 * np.abs(A @ P).max())


def test_nonsym_h2_plus_uvt_update():
    """BASELINE configs[4] with a genuinely non-symmetric update: M = A_H + U V^T (V != U),
    recompressed by h2_build_nonsym from the H^2-matvec + low-rank sketch (Y = A_H Omega +
    U V^T Omega, Z = A_H Psi + V U^T Psi) with entries extracted from A_H's blocks and bases.
    Against the oracle's non-symmetric build of the dense M: ranks / skeletons of both sides
    bit-exact or certified, D and B entries = M's entries, probe error <= 2 tol."""
    X, T, tree, part = setup(2048, 3, 64, 21)
    n = T.n
    Hb = g.build(T, ("exp", 0.2), 1e-9)
    rr = np.random.default_rng(7)
    U = torch.from_numpy(rr.standard_normal((n, 6)) * 0.3).cuda()
    V = torch.from_numpy(rr.standard_normal((n, 6)) * 0.3).cuda()
    I = torch.eye(n, dtype=torch.float64, device="cuda")
    KH = torch.cat([Hb.matvec(I[:, c:c + 64]) for c in range(0, n, 64)], dim=1)
    M = (KH + U @ V.T).cpu().numpy()
    tol = 1e-6
    Hg = g.build(T, ("exp", 0.2), tol, update=(Hb, U, V), nonsym=True)
    Ho = oracle_nonsym(tree, part, M, tol)
    assert Hg.samples == Ho.samples
    for side in (0, 1):
        c, m = compare_side(Hg, Ho, side)
        assert c <= max(2, m // 50)
    Dl = tree.leaf_depth
    D = Hg.D_blocks()
    for (s, b) in list(D)[::7]:
        ref = M[tree.begin[Dl][s]:tree.end[Dl][s], tree.begin[Dl][b]:tree.end[Dl][b]]
        assert np.abs(D[(s, b)] - ref).max() <= 1e-12 * np.abs(M).max()
    for t in range(Hg.top_depth, Dl + 1):
        Bb = Hg.B_blocks(t)
        sr, sc = Hg.skel(t, 0), Hg.skel(t, 1)
        for (s, b) in list(Bb)[::5]:
            assert np.abs(Bb[(s, b)] - M[np.ix_(sr[s], sc[b])]).max() <= 1e-10 * np.abs(M).max(), (t, s, b)
    P = np.random.default_rng(8).standard_normal((n, 6))
    y = Hg.matvec(torch.from_numpy(P).cuda()).cpu().numpy()
    assert np.linalg.norm(y - M @ P) <= 2 * tol * np.linalg.norm(M @ P)
    with pytest.raises(g.H2Error):   # U V^T is non-symmetric: the symmetric build refuses it
        g.build(T, ("exp", 0.2), tol, update=(Hb, U, V))
