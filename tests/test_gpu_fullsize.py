"""Full-size parity at BASELINE configs[1] (N = 2^18 exp covariance, leaf 64, tol 1e-6): the bench
workload in the launch configuration bench.py times (adaptive, d_init = d_blk = 32, 128-column
tensor-core sketch passes).  At this size the oracle cannot build the H^2, so it checks SAMPLED
outputs it computes one by one (Omega entries, sketch rows, D and B blocks, probe rows of K X) and
properties that hold at any size (identity rows of every basis, the convergence test, skeletons
inside their clusters).  DESIGN.md §3."""
import ctypes as C

import numpy as np
import pytest
import torch

from oracle import kernels, rng
from synth import uniform_points
import paper_2506_16759_b200 as g
from paper_2506_16759_b200 import _lib as L

pytestmark = pytest.mark.gpu

N, LEAF, TOL, KERN = 1 << 18, 64, 1e-6, ("exp", 0.2)


@pytest.fixture(scope="module")
def full():
    X = uniform_points(N, 3, 0)
    T = g.Tree(X, LEAF, 0.7)
    H = g.build(T, KERN, TOL, adaptive=True, d_init=32, d_blk=32, d_max=512)
    op = kernels.KernelOperator(KERN[0], KERN[1], X[T.perm])
    return X, T, H, op


def _export_dev(H, what, depth=0):
    cnt = C.c_int64()
    g._lib.check(L.lib.h2_export_size(H._h, what, depth, C.byref(cnt)))
    out = torch.empty(cnt.value, dtype=torch.float64, device="cuda")
    g._lib.check(L.lib.h2_export(H._h, what, depth, C.c_void_p(out.data_ptr())))
    return out


def test_fullsize_omega_sampled_rows_bitwise():
    Om = g.omega(N, 128)
    rows = np.random.default_rng(5).choice(N, 64, replace=False)
    got = Om[torch.from_numpy(rows).cuda()].cpu().numpy()
    want = np.concatenate([rng.omega_block(1, 0, int(r), 1, 0, 128) for r in rows])
    assert np.array_equal(got, want)


@pytest.mark.parametrize("ncols", [160, 128])
def test_fullsize_sketch_rows(full, ncols):
    """The bench's sketch launch: ONE 160-column packed tensor-core pass over all N = 2^18 rows
    (M = 128 slice pairs, 64-row tiles, the j-split chosen for this N, all TMEM drains of
    65536-j chunks), exactly what h2_build issues for the speculative pass (the build above
    reports one sketch launch of 160 columns), vs the oracle's K(rows, :) Omega for 48 sampled
    rows: <= 1e-13 max|Y| (fixed-point rounding of K at 2^-47, R32).  128 columns:
    the 7-slice / Helmholtz pass shape."""
    X, T, H, op = full
    assert H.stats["sketch_columns"] == 160 and H.stats["entries_sketch"] == N * N   # bench launch shape
    Om = g.omega(N, ncols)
    Y = g.dense_sketch(T, Om, KERN, omega_quarters=True)
    rows = np.sort(np.random.default_rng(6 + ncols).choice(N, 48, replace=False))
    rows[0], rows[-1] = 0, N - 1            # first and last row tiles (ragged j-split edges)
    ref = op.sketch_rows(Om.cpu().numpy(), rows)
    got = Y[torch.from_numpy(rows).cuda()].cpu().numpy()
    assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()


def test_fullsize_cpqr_variants(full):
    """Which CPQR kernels the bench's launch configuration runs (h2_build_stats.cpqr_variants);
    each of them is forced on every level of an oracle-parity build in
    test_gpu_parity.py::test_build_parity_each_cpqr_variant."""
    X, T, H, op = full
    cv = H.stats["cpqr_variants"]
    # the bench's launch configuration runs all three CPQR paths at N = 2^18: the warp kernel on
    # the 64-row leaf panels and the CTA kernels (shared / global panel) on the inner levels
    assert cv & g._lib.H2_CQ_V_WARP and cv & (g._lib.H2_CQ_V_SMEM | g._lib.H2_CQ_V_GLOBAL), cv


def test_fullsize_convergence_and_identity_rows(full):
    X, T, H, op = full
    d, pos = H.samples, 10
    for t in range(H.top_depth, T.leaf_depth + 1):
        k = H.rank(t)
        m = H.panel_rows(t)
        assert np.all((m <= d) | (k <= d - 1 - pos)), t          # §III-B test (R12) at exit
        if t in (T.leaf_depth, T.leaf_depth - 3, H.top_depth):
            sk = H.skel(t)
            Xs = H.basis(t)
            if t == T.leaf_depth:
                lo = T.begin[t]
                ibar = [np.arange(T.begin[t][c], T.end[t][c]) for c in range(len(k))]
            else:
                skc = H.skel(t + 1)
                ibar = [np.concatenate([skc[2 * c], skc[2 * c + 1]]) for c in range(len(k))]
            for c in np.random.default_rng(t).choice(len(k), min(16, len(k)), replace=False):
                where = {int(v): i for i, v in enumerate(ibar[c])}
                J = np.array([where[int(v)] for v in sk[c]])          # skeletons are rows of the panel
                assert np.array_equal(Xs[c][J], np.eye(k[c]))       # identity rows, bitwise


def test_fullsize_D_and_B_blocks_sampled(full):
    """Sampled unique D (near) and B (far, at the skeleton indices) blocks vs the oracle's
    entries: <= 4e-15 relative (custom exp / rsqrt vs numpy)."""
    X, T, H, op = full
    Dl = T.leaf_depth
    sz = (T.end[Dl] - T.begin[Dl]).astype(np.int64)
    near = T.near[T.near[:, 0] <= T.near[:, 1]]
    offs = np.concatenate([[0], np.cumsum(sz[near[:, 0]] * sz[near[:, 1]])])
    Dd = _export_dev(H, L.H2_X_D)
    pick = np.random.default_rng(8).choice(len(near), 24, replace=False)
    for q in pick:
        s, b = near[q]
        blk = Dd[offs[q]:offs[q + 1]].cpu().numpy().reshape(sz[s], sz[b])
        ref = op.entry(np.arange(T.begin[Dl][s], T.end[Dl][s]), np.arange(T.begin[Dl][b], T.end[Dl][b]))
        assert np.abs(blk - ref).max() <= 4e-15 * max(1.0, np.abs(ref).max())
    for t in (H.top_depth, (H.top_depth + Dl) // 2, Dl - 1):
        far = T.far[t][T.far[t][:, 0] < T.far[t][:, 1]]
        if len(far) == 0:
            continue
        k = H.rank(t)
        sk = H.skel(t)
        boffs = np.concatenate([[0], np.cumsum(k[far[:, 0]] * k[far[:, 1]])])
        Bd = _export_dev(H, L.H2_X_B, t)
        for q in np.random.default_rng(t).choice(len(far), min(12, len(far)), replace=False):
            s, b = far[q]
            blk = Bd[boffs[q]:boffs[q + 1]].cpu().numpy().reshape(k[s], k[b])
            ref = op.entry(sk[s], sk[b])
            assert np.abs(blk - ref).max() <= 4e-15 * max(1.0, np.abs(ref).max())


def test_fullsize_matvec_sampled_rows_within_2tol(full):
    """North-star accuracy at full size: ||H X - K X|| / ||K X|| <= 2 tol over 96 sampled rows of
    16 Gaussian probes, K X computed row by row by the oracle."""
    X, T, H, op = full
    P = np.random.default_rng(2).standard_normal((N, 16))
    HX = H.matvec(torch.from_numpy(P).cuda()).cpu().numpy()
    rows = np.sort(np.random.default_rng(9).choice(N, 96, replace=False))
    KX = op.sketch_rows(P, rows)
    err = np.linalg.norm(HX[rows] - KX) / np.linalg.norm(KX)
    assert err <= 2 * TOL, err
