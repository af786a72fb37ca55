"""GPU parity: the CUDA path (libh2 through its C ABI) against the oracle on the same seeded
inputs.  Run with  pytest -m gpu  on a B200."""
import numpy as np
import pytest
import torch

from oracle import kernels, rng, h2 as oh2
from synth import uniform_points, grid_points
import paper_2506_16759_b200 as g
from gpu_helpers import oracle_build, compare_builds, compare_blocks, compare_matvec, probe_error

pytestmark = pytest.mark.gpu

CASES = {
    # BASELINE configs[0]: 2D exp covariance, N=1024, leaf 32, tol 1e-6
    "cov2d_1k": (lambda: uniform_points(1024, 2, 0), "exp", 0.2, 32, 1e-6),
    # ragged leaves (39/40 points), several sketch tiles + ragged tail (5000 = 39*128 + 8)
    "cov3d_5000": (lambda: uniform_points(5000, 3, 0), "exp", 0.2, 64, 1e-6),
    # leaves of exactly 64 points (8192 = 64 x 2^7): the leaf subtraction runs on the tensor cores
    # from the kernel itself (launch_near_sketch_tc) instead of the BSR over the stored D blocks
    "cov3d_8192": (lambda: uniform_points(8192, 3, 1), "exp", 0.2, 64, 1e-6),
    # volume IE on a regular grid (BASELINE configs[3] shape, 16^3), tol 1e-4
    "ie_grid16": (lambda: grid_points((16, 16, 16), 1 / 16), "helmholtz", 3.0, 64, 1e-4),
}


def test_omega_matches_oracle_generator():
    Om = g.omega(3000, 37, seed=11, stream_id=3, col0=5).cpu().numpy()
    ref = rng.omega_block(11, 3, 0, 3000, 5, 37)
    assert np.array_equal(Om, ref)          # exactly representable stream: bit-identical


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("quarters", [False, True])
@pytest.mark.parametrize("ncols", [45, 128, 150, 170])
def test_dense_sketch_matches_oracle(case, quarters, ncols):
    """DMMA path (arbitrary Omega) and, with the h2 Omega stream, the int8 tensor-core path
    (sketch_tc.cu): exp (6 slices, 47-bit grid): 45 columns = one 128-row / 64-column pass, 128 =
    one 64-row / 128-column pass, 150 = one 160-column pass, 170 = 160 + a ragged 10-column pass;
    Helmholtz (7 slices): 128-column passes.  Bound 1e-13 max|Y| (the fixed-point grid
    rounding, <= 2^-48 max|K| per entry, stays at the FP64 GEMM's own rounding level)."""
    mk, kind, p, leaf, tol = CASES[case]
    X = mk()
    T = g.Tree(X, leaf)
    Om = rng.omega_block(1, 0, 0, T.n, 0, ncols)
    if not quarters:
        Om = Om + 1e-3 * np.random.default_rng(7).standard_normal(Om.shape)   # generic values
    op = kernels.KernelOperator(kind, p, X[T.perm])
    ref = op.sampler(Om)
    Od = torch.from_numpy(Om).cuda()
    y = g.dense_sketch(T, Od, (kind, p), omega_quarters=quarters).cpu().numpy()
    scale = np.abs(ref).max()
    assert np.abs(y - ref).max() <= 1e-13 * scale
    # row-range variant (multi-GPU row shard)
    r0, r1 = 333, min(T.n, 1777)
    y2 = g.dense_sketch(T, Od, (kind, p), r0, r1, omega_quarters=quarters).cpu().numpy()
    assert np.abs(y2 - ref[r0:r1]).max() <= 1e-13 * scale


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("adaptive", [False, True])
def test_build_parity(case, adaptive):
    mk, kind, p, leaf, tol = CASES[case]
    X = mk()
    opts = dict(adaptive=adaptive) if adaptive else dict(adaptive=False, d_init=64)
    Ho, op = oracle_build(X, kind, p, leaf, tol, **opts)
    T = g.Tree(X, leaf)
    Hg = g.build(T, (kind, p), tol, **opts)
    div = {}
    certified, compared = compare_builds(Hg, Ho, div)
    assert certified <= max(1, compared // 100)
    if case == "cov2d_1k":
        assert certified == 0          # a deterministic case with no near-tie at all
    if certified == 0:
        assert Hg.samples == Ho.samples
    # D blocks always; B blocks of every pair whose clusters kept identical skeletons
    compare_blocks(Hg, Ho, div)
    # accuracy against the dense operator
    K = op.dense()
    err = probe_error(Hg, K)
    bound = 2 * tol if adaptive else 10 * tol
    assert err <= bound, err
    # H^2 matvecs of the two representations: 1e-10 (BASELINE north_star), or bounded by the
    # two error bounds where a certified near-tie made the skeletons diverge
    compare_matvec(Hg, Ho, certified, bound)


@pytest.mark.parametrize("variant", ["warp", "smem", "global", "cluster", "smem2", "global2"])
@pytest.mark.parametrize("case", ["cov3d_5000", "ie_grid16"])
def test_build_parity_each_cpqr_variant(monkeypatch, case, variant):
    """Every CPQR kernel variant (warp per panel / CTA with the panel in shared memory / CTA with
    the panel in global W / a cluster of CTAs with the rows in distributed shared memory, the one
    large inner panels take at N = 2^18; "2": the opt-in cpqr2
    kernel, H2_CQ2=1) forced on every level of an adaptive build: same skeleton / rank / sample
    parity with the oracle, and the stats name the variant that ran."""
    mk, kind, p, leaf, tol = CASES[case]
    X = mk()
    Ho, op = oracle_build(X, kind, p, leaf, tol)
    T = g.Tree(X, leaf)
    if variant.endswith("2"):
        monkeypatch.setenv("H2_CQ2", "1")
        variant = variant[:-1]
    monkeypatch.setenv("H2_CQ_VARIANT", variant)
    Hg = g.build(T, (kind, p), tol)
    bit = {"warp": g._lib.H2_CQ_V_WARP, "smem": g._lib.H2_CQ_V_SMEM, "global": g._lib.H2_CQ_V_GLOBAL,
           "cluster": g._lib.H2_CQ_V_CLUSTER}[variant]
    used = Hg.stats["cpqr_variants"]
    assert used & bit, used
    if variant != "warp":
        assert not used & g._lib.H2_CQ_V_WARP        # forced on the leaf panels too
    if variant in ("global", "cluster"):
        assert used == bit
    div = {}
    certified, compared = compare_builds(Hg, Ho, div)
    assert certified <= max(1, compared // 100)
    if certified == 0:
        assert Hg.samples == Ho.samples
    compare_blocks(Hg, Ho, div)
    err = probe_error(Hg, op.dense())
    assert err <= 2 * tol, err
    compare_matvec(Hg, Ho, certified, 2 * tol)


def test_matvec_alpha_beta_and_linearity():
    X = uniform_points(2048, 3, 4)
    T = g.Tree(X, 64)
    H = g.build(T, ("exp", 0.2), 1e-6)
    x = torch.randn(T.n, 3, dtype=torch.float64, device="cuda")
    y0 = torch.randn(T.n, 3, dtype=torch.float64, device="cuda")
    y1 = H.matvec(x)
    y2 = H.matvec(x, alpha=2.0, beta=0.5, y=y0.clone())
    assert torch.allclose(y2, 2.0 * y1 + 0.5 * y0, rtol=1e-13, atol=1e-12)
    # column-by-column equals the block product
    for j in range(3):
        yj = H.matvec(x[:, j].contiguous())
        assert torch.allclose(yj, y1[:, j], rtol=1e-13, atol=1e-12)


def test_callback_sampler_and_entries_known_rank_recovery():
    """Black-box K_blk and entry evaluator supplied as callbacks: a
    synthetic H^2 of known ranks is recovered exactly (ranks equal, error <= 1e-10)."""
    from synthetic_h2 import synthetic_h2
    from oracle import geometry
    X = uniform_points(1024, 3, 10)
    tree = geometry.build_cluster_tree(X, 32)
    part = geometry.build_partition(tree, 0.7)
    K, ranks, active = synthetic_h2(tree, part, lambda t, m: min(m, 6 + (t % 3) * 2), 0)
    Kd = torch.from_numpy(K).cuda()
    T = g.Tree(X, 32)

    def sketch(om, y, col0, r0, r1):
        y.copy_(Kd[r0:r1] @ om)

    def entry(b):
        n = b.nblocks
        view = lambda p, dt: g.device_view(p, (n,), (1,), dt)
        m, nc = view(b.m, torch.int32).cpu(), view(b.nc, torch.int32).cpu()
        ro, co = view(b.row_off, torch.int64).cpu(), view(b.col_off, torch.int64).cpu()
        outp = view(b.out, torch.int64).cpu()
        total = int(max(ro.max() + m.max(), co.max() + nc.max()))
        ridx = g.device_view(b.row_idx, (total,), (1,), torch.int32).long()
        cidx = g.device_view(b.col_idx, (total,), (1,), torch.int32).long()
        for q in range(n):
            rows = ridx[ro[q]:ro[q] + m[q]]
            cols = cidx[co[q]:co[q] + nc[q]]
            out = g.device_view(int(outp[q]), (int(m[q]), int(nc[q])), (int(nc[q]), 1))
            out.copy_(Kd[rows][:, cols])

    nu = float(np.linalg.norm(K, 2))
    dmax = max(int(r.max()) for r in ranks.values()) + 8
    H = g.build(T, ("exp", 0.2), 1e-12, sketch=sketch, entry=entry, adaptive=False, d_init=dmax,
                tol_rule="literal", norm=nu)
    for t in range(H.top_depth, T.leaf_depth + 1):
        assert np.array_equal(H.rank(t), np.where(active[t], ranks[t], 0)), t
    x = np.random.default_rng(0).standard_normal((T.n, 4))
    y = H.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.linalg.norm(y - K @ x) <= 1e-10 * np.linalg.norm(K @ x)


def test_not_converged_and_callback_errors():
    X = uniform_points(4096, 3, 0)
    T = g.Tree(X, 64)
    with pytest.raises(g.H2Error) as e:
        g.build(T, ("exp", 0.2), 1e-6, d_init=8, d_blk=8, d_max=16)
    assert e.value.status == -6
    def bad(om, y, c0, r0, r1):
        raise ValueError("boom")
    with pytest.raises(g.H2Error) as e:
        g.build(T, ("exp", 0.2), 1e-6, sketch=bad)
    assert e.value.status == -5
    # the library still works afterwards (no leaked state)
    H = g.build(T, ("exp", 0.2), 1e-6)
    assert H.samples >= 32


def test_degenerate_inputs():
    # N <= leaf: one dense block equal to K, no admissible pairs
    X = uniform_points(40, 3, 1)
    T = g.Tree(X, 64)
    H = g.build(T, ("exp", 0.2), 1e-6)
    K = kernels.kernel_block("exp", 0.2, X[T.perm], X[T.perm])
    D = H.D_blocks()[(0, 0)]
    assert np.abs(D - K).max() <= 1e-15
    x = np.random.default_rng(0).standard_normal((40, 2))
    y = H.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.abs(y - K @ x).max() <= 1e-13
    # all-dense partition (eta -> 0): ranks 0 and exact matvec
    X = uniform_points(500, 3, 2)
    T = g.Tree(X, 32, eta=1e-9)
    H = g.build(T, ("exp", 0.2), 1e-6)
    assert np.all(H.rank(T.leaf_depth) == 0)
    K = kernels.kernel_block("exp", 0.2, X[T.perm], X[T.perm])
    y = H.matvec(torch.from_numpy(np.eye(500)[:, :7].copy()).cuda()).cpu().numpy()
    assert np.abs(y - K[:, :7]).max() <= 1e-13


@pytest.mark.parametrize("case", ["cov3d_8192"])
def test_near_field_tensor_core_vs_bsr(case):
    """The leaf subtraction on the tensor cores (H2_NEAR_TC, default) vs the BSR over the stored D
    blocks: the two Y^loc differ only by the fixed-point rounding of the near-field K (<= 2^-48
    max|K| per entry), so ranks / skeletons agree up to certified near-ties and the H^2
    representations agree to the tolerance level (the switch is read once per process)."""
    import subprocess, sys, os, tempfile
    code = "\n".join([
        "import sys, os, numpy as np, torch",
        "sys.path.insert(0, os.environ['ROOT'])",
        "import paper_2506_16759_b200 as g",
        "from synth import uniform_points",
        "T = g.Tree(uniform_points(8192, 3, 1), 64)",
        "H = g.build(T, ('exp', 0.2), 1e-6)",
        "out = [np.array([H.samples], float)]",
        "out += [H.rank(t).astype(float) for t in range(H.top_depth, T.leaf_depth + 1)]",
        "P = np.random.default_rng(3).standard_normal((T.n, 4))",
        "out += [H.matvec(torch.from_numpy(P).cuda()).cpu().numpy().ravel()]",
        "np.save(sys.argv[1], np.concatenate(out))"])
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = []
    for val in ("0", "1"):
        f = tempfile.mktemp(suffix=".npy")
        subprocess.run([sys.executable, "-c", code, f], check=True, env=dict(os.environ, ROOT=root, H2_NEAR_TC=val))
        res.append(np.load(f))
        os.remove(f)
    a, b = res
    assert a.shape == b.shape and a[0] == b[0]          # samples
    nmv = 8192 * 4
    ra, rb = a[1:-nmv], b[1:-nmv]
    assert np.mean(ra != rb) <= 0.01                    # ranks: certified near-ties only
    ya, yb = a[-nmv:], b[-nmv:]
    assert np.linalg.norm(ya - yb) <= 2e-6 * np.linalg.norm(ya)


def test_async_tree_build_bitwise():
    """h2_tree_build_async: h2_build launches the first sketch pass before waiting for the
    partition thread; the H^2 is bitwise the one built on a synchronous tree."""
    X = uniform_points(6000, 3, 5)
    Hs = g.build(g.Tree(X, 64), ("exp", 0.2), 1e-6)
    Ta = g.Tree(X, 64, asynchronous=True)
    Ha = g.build(Ta, ("exp", 0.2), 1e-6)
    assert Hs.samples == Ha.samples
    for t in range(Hs.top_depth, Ta.leaf_depth + 1):
        assert np.array_equal(Hs.rank(t), Ha.rank(t))
        for w in (g._lib.H2_X_BASIS, g._lib.H2_X_B):
            assert np.array_equal(Hs._export(w, t), Ha._export(w, t))
    assert np.array_equal(Hs._export(g._lib.H2_X_D), Ha._export(g._lib.H2_X_D))
    # the one-call result read (h2_export with H2_ALL_DEPTHS) = the per-depth exports concatenated
    rk, sk = Ha.ranks_and_skeletons()
    assert np.array_equal(rk, np.concatenate([Ha.rank(t) for t in range(Ha.top_depth, Ta.leaf_depth + 1)]))
    assert np.array_equal(sk, np.concatenate([np.concatenate(Ha.skel(t)) for t in range(Ha.top_depth, Ta.leaf_depth + 1)]))


def test_deterministic_bitwise():
    X = uniform_points(5000, 3, 0)
    T = g.Tree(X, 64)
    H1 = g.build(T, ("exp", 0.2), 1e-6)
    H2 = g.build(T, ("exp", 0.2), 1e-6)
    for t in range(H1.top_depth, T.leaf_depth + 1):
        assert np.array_equal(H1.rank(t), H2.rank(t))
        assert np.array_equal(H1._export(g._lib.H2_X_BASIS, t), H2._export(g._lib.H2_X_BASIS, t))
        assert np.array_equal(H1._export(g._lib.H2_X_B, t), H2._export(g._lib.H2_X_B, t))
    assert np.array_equal(H1._export(g._lib.H2_X_D), H2._export(g._lib.H2_X_D))


@pytest.mark.parametrize("nc,slices", [(128, "6"), (150, "6"), (160, "6"), (150, "7")])
def test_tc_pass_width_bitwise(monkeypatch, nc, slices):
    """The 160/128-column (M = 64) and 64-column (M = 128) tensor-core passes accumulate the same
    exact integers and sum the byte slices in the same order: bit-identical sketches, for both
    fixed-point formats (6 slices: 47-bit grid, 7: 52-bit)."""
    monkeypatch.setenv("H2_TC_SLICES", slices)
    X = uniform_points(20000, 3, 0)
    T = g.Tree(X, 64)
    Od = torch.from_numpy(rng.omega_block(1, 0, 0, T.n, 0, nc)).cuda()
    monkeypatch.setenv("H2_TC_WIDE", "0")
    y0 = g.dense_sketch(T, Od, ("exp", 0.2), omega_quarters=True)
    monkeypatch.setenv("H2_TC_WIDE", "1")
    y1 = g.dense_sketch(T, Od, ("exp", 0.2), omega_quarters=True)
    assert torch.equal(y0, y1)


@pytest.mark.parametrize("n,nc,kind", [(20001, 128, "exp"), (9000, 100, "exp"), (4100, 70, "exp"),
                                       (8000, 128, "helmholtz")])
def test_tc_pair_kernel_bitwise(monkeypatch, n, nc, kind):
    """The CTA-pair (cta_group::2, M = 128 over two SMs, B split by columns) 128-column pass
    gives the same bits as the single-CTA pass: ragged row tiles (odd tile counts pad the last
    pair), a partial second column half, and the j-split."""
    X = uniform_points(n, 3, 1) if kind == "exp" else grid_points((20, 20, 20), 1.0 / 20)
    kern = ("exp", 0.2) if kind == "exp" else ("helmholtz", 3.0)
    T = g.Tree(X, 64)
    Od = torch.from_numpy(rng.omega_block(1, 0, 0, T.n, 0, nc)).cuda()
    monkeypatch.setenv("H2_TC_PAIR", "0")
    y0 = g.dense_sketch(T, Od, kern, omega_quarters=True)
    monkeypatch.setenv("H2_TC_PAIR", "1")
    y1 = g.dense_sketch(T, Od, kern, omega_quarters=True)
    assert torch.equal(y0, y1)
    Kd = kernels.KernelOperator(*kern, X[T.perm]).dense() if n <= 9000 else None
    if Kd is not None:
        ref = Kd @ Od.cpu().numpy()
        assert np.abs(y1.cpu().numpy() - ref).max() <= 1e-13 * np.abs(ref).max()


def test_speculative_sketch_columns_bitwise(monkeypatch):
    """Speculative 128-column tensor-core passes change how many Omega columns are
    pushed through the sketch, never the samples consumed: the build is bit-identical to one
    drawing exactly d_blk columns per updateSamples."""
    X = uniform_points(5000, 3, 0)
    T = g.Tree(X, 64)
    monkeypatch.setenv("H2_SPEC", "0")
    H0 = g.build(T, ("exp", 0.2), 1e-6, d_init=16, d_blk=16)
    monkeypatch.setenv("H2_SPEC", "1")
    H1 = g.build(T, ("exp", 0.2), 1e-6, d_init=16, d_blk=16)
    assert H0.samples == H1.samples
    assert H0.stats["sketch_columns"] == H0.samples
    assert H1.samples <= H1.stats["sketch_columns"] < H1.samples + 128
    assert H1.stats["entries_sketch"] < H0.stats["entries_sketch"]
    for t in range(H0.top_depth, T.leaf_depth + 1):
        assert np.array_equal(H0.rank(t), H1.rank(t))
        assert all(np.array_equal(a, b) for a, b in zip(H0.skel(t), H1.skel(t)))
        assert np.array_equal(H0._export(g._lib.H2_X_BASIS, t), H1._export(g._lib.H2_X_BASIS, t))
        assert np.array_equal(H0._export(g._lib.H2_X_B, t), H1._export(g._lib.H2_X_B, t))


def test_helmholtz_sketch_with_coincident_points():
    """Coincident points (r_min = 0: no fixed-point scale for the Helmholtz tensor-core sketch)
    take the FP64 DMMA path; K(x, x) = 0 (R20) on every coincident pair.  Matches the oracle."""
    X = grid_points((8, 8, 8), 1 / 8)
    X = np.concatenate([X, X[:37]])            # 37 duplicated points
    T = g.Tree(X, 64)
    Om = rng.omega_block(1, 0, 0, T.n, 0, 40)
    op = kernels.KernelOperator("helmholtz", 3.0, X[T.perm])
    ref = op.sampler(Om)
    y = g.dense_sketch(T, torch.from_numpy(Om).cuda(), ("helmholtz", 3.0), omega_quarters=True).cpu().numpy()
    assert np.abs(y - ref).max() <= 1e-13 * np.abs(ref).max()


@pytest.mark.parametrize("case,opts", [("cov3d_5000", dict(d_init=16, d_blk=16)),
                                       ("cov3d_5000", dict(d_init=32, d_blk=24)),
                                       ("cov3d_5000", dict()),
                                       ("ie_grid16", dict(d_init=16, d_blk=8)),
                                       ("cov2d_1k", dict(d_init=8, d_blk=8, d_max=400))])
def test_eager_sweep_bitwise(monkeypatch, case, opts):
    """Eager sweep: every column of a sketch pass goes up with the panel (one
    BSR / shrink launch per depth over the whole pass) instead of block-by-block updateSamples
    replays -- bitwise the lazy build (ranks, skeletons, bases, B, D, certificates, samples)."""
    mk, kind, p, leaf, tol = CASES[case]
    X = mk()
    T = g.Tree(X, leaf)
    monkeypatch.setenv("H2_EAGER", "0")
    H0 = g.build(T, (kind, p), tol, **opts)
    monkeypatch.setenv("H2_EAGER", "1")
    H1 = g.build(T, (kind, p), tol, **opts)
    assert H0.samples == H1.samples
    assert H0.stats["rounds"] == H1.stats["rounds"]
    for t in range(H0.top_depth, T.leaf_depth + 1):
        assert np.array_equal(H0.rank(t), H1.rank(t))
        assert np.array_equal(H0._export(g._lib.H2_X_SKEL, t, np.int32), H1._export(g._lib.H2_X_SKEL, t, np.int32))
        for w in (g._lib.H2_X_BASIS, g._lib.H2_X_B, g._lib.H2_X_CERT):
            assert np.array_equal(H0._export(w, t), H1._export(w, t)), (t, w)
    assert np.array_equal(H0._export(g._lib.H2_X_D), H1._export(g._lib.H2_X_D))


@pytest.mark.parametrize("env,a,b", [("H2_CQ_REG", "0", "1"), ("H2_CQ_REG", "0", "3"), ("H2_BSR_VAR", "0", "3"), ("H2_BSR_VAR", "0", "1"),
                                     ("H2_BSR2", "0", "1"), ("H2_BSR2", "0", "9"), ("H2_BSR2", "1", "2"), ("H2_BSR2", "1", "3"),
                                     ("H2_BSR2", "1", "4"), ("H2_BSR2", "1", "5"),
                                     ("H2_BSR2", "1", "6"), ("H2_BSR2", "1", "7"),
                                     ("H2_BSR2", "1", "8"), ("H2_BSR2", "1", "9"),
                                     ("H2_BSR2", "1", "11"), ("H2_BSR2", "1", "12")])
def test_kernel_variants_bitwise(monkeypatch, env, a, b):
    """Performance variants that keep every element's operation order: the register-cached CPQR
    update (H2_CQ_REG) and the BSR tilings of wide passes (H2_BSR_VAR: 64-column tiles, 32-column
    tiles in a column-fast grid, 160-column CTAs; H2_BSR2: the round-2 kernel with one shared-memory
    layout for both block orientations vs the round-1 family, and its 64-column / 3-stage forms)
    give bitwise the same H^2 (variants are chosen
    once per process: each side runs in its own subprocess)."""
    import subprocess, sys, os
    code = r'''
import sys, os, numpy as np
sys.path.insert(0, os.environ["ROOT"])
import paper_2506_16759_b200 as g
from synth import uniform_points
T = g.Tree(uniform_points(6000, 3, 2), 64)
H = g.build(T, ("exp", 0.2), 1e-6, d_init=32, d_blk=32)
out = [H._export(g._lib.H2_X_BASIS, t) for t in range(H.top_depth, T.leaf_depth + 1)]
out += [H._export(g._lib.H2_X_B, t) for t in range(H.top_depth, T.leaf_depth + 1)]
np.save(sys.argv[1], np.concatenate(out + [H._export(g._lib.H2_X_D), np.array([H.samples], float)]))
'''
    import tempfile
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = []
    for val in (a, b):
        f = tempfile.mktemp(suffix=".npy")
        subprocess.run([sys.executable, "-c", code, f], check=True, env=dict(os.environ, ROOT=root, **{env: val}))
        res.append(np.load(f))
        os.remove(f)
    assert res[0].shape == res[1].shape and np.array_equal(res[0], res[1])


@pytest.mark.parametrize("hyb", ["110", "200"])
def test_cpqr_hybrid_panel_bitwise(hyb):
    """H2_CQ_HYB: the global-panel CPQR moves the active part of the panel into shared memory once
    it fits and continues there -- the same operations in the same order, so with the global
    variant forced on every block-panel level the H^2 is bitwise the all-global one."""
    import subprocess, sys, os, tempfile
    code = r'''
import sys, os, numpy as np
sys.path.insert(0, os.environ["ROOT"])
import paper_2506_16759_b200 as g
from synth import uniform_points
T = g.Tree(uniform_points(6000, 3, 2), 64)
H = g.build(T, ("exp", 0.2), 1e-6, d_init=32, d_blk=32)
assert H.stats["cpqr_variants"] & g._lib.H2_CQ_V_GLOBAL
out = [H._export(g._lib.H2_X_BASIS, t) for t in range(H.top_depth, T.leaf_depth + 1)]
out += [H._export(g._lib.H2_X_CERT, t) for t in range(H.top_depth, T.leaf_depth + 1)]
out += [H._export(g._lib.H2_X_B, t) for t in range(H.top_depth, T.leaf_depth + 1)]
np.save(sys.argv[1], np.concatenate(out + [np.array([H.samples], float)]))
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = []
    for val in ("0", hyb):
        f = tempfile.mktemp(suffix=".npy")
        env = dict(os.environ, ROOT=root, H2_CQ_VARIANT="global", H2_CQ_HYB=val)
        subprocess.run([sys.executable, "-c", code, f], check=True, env=env)
        res.append(np.load(f))
        os.remove(f)
    assert res[0].shape == res[1].shape and np.array_equal(res[0], res[1])
