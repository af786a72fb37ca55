"""GPU KD ordering of h2_tree_build_async (kd_gpu.cu): the same tree as the host ordering (R4:
median split of the longest axis, key (coordinate, original index)), bit for bit -- permutation,
node ranges, tree-order coordinates, partition -- on uniform 1D/2D/3D points, a regular grid (ties
everywhere), duplicated points and sizes that are not powers of two."""
import numpy as np
import pytest
import torch

from synth import uniform_points, grid_points
import paper_2506_16759_b200 as g

pytestmark = pytest.mark.gpu


def _cases():
    rng = np.random.default_rng(11)
    dup = uniform_points(6000, 3, 2)
    dup[3000:] = dup[:3000]                      # every point twice
    half = uniform_points(9000, 3, 3)
    half[:, 2] = np.round(half[:, 2] * 8) / 8    # heavy ties on one axis
    neg = rng.standard_normal((20000, 2))        # negative coordinates, -0.0
    neg[::97, 0] = -0.0
    neg[1::97, 0] = 0.0
    return {"u3_2^18_bench": (uniform_points(1 << 18, 3, 0), 64),   # the bench's e2e tree (configs[1])
            "u3_2^16": (uniform_points(1 << 16, 3, 0), 64), "u2_50000": (uniform_points(50000, 2, 1), 32),
            "u1_9999": (uniform_points(9999, 1, 4), 16), "grid32": (grid_points((32, 32, 32), 1 / 32), 64),
            "dup": (dup, 40), "ties": (half, 50), "signed": (neg, 24)}


@pytest.mark.parametrize("name", list(_cases()))
def test_gpu_kd_ordering_matches_host(name, monkeypatch):
    X, leaf = _cases()[name]
    Th = g.Tree(X, leaf, 0.7)                              # host ordering (synchronous build)
    Tg = g.Tree(X, leaf, 0.7, asynchronous=True)           # GPU ordering (asynchronous build)
    assert np.array_equal(Th.perm, Tg.perm)
    for t in range(Th.leaf_depth + 1):
        assert np.array_equal(Th.begin[t], Tg.begin[t]) and np.array_equal(Th.end[t], Tg.end[t])
    assert Th.near_nnz == Tg.near_nnz and Th.far_nnz_total == Tg.far_nnz_total and Th.csp == Tg.csp
    assert np.array_equal(Th.near, Tg.near)


def test_gpu_kd_build_bitwise():
    """A build on the GPU-ordered tree is bitwise the build on the host-ordered one."""
    X = uniform_points(1 << 15, 3, 6)
    Hh = g.build(g.Tree(X, 64, 0.7), ("exp", 0.2), 1e-6)
    Hg = g.build(g.Tree(X, 64, 0.7, asynchronous=True), ("exp", 0.2), 1e-6)
    assert Hh.samples == Hg.samples
    L = g._lib
    for t in range(Hh.top_depth, Hh.tree.leaf_depth + 1):
        assert np.array_equal(Hh._export(L.H2_X_SKEL, t, np.int32), Hg._export(L.H2_X_SKEL, t, np.int32))
        assert np.array_equal(Hh._export(L.H2_X_BASIS, t), Hg._export(L.H2_X_BASIS, t))
        assert np.array_equal(Hh._export(L.H2_X_B, t), Hg._export(L.H2_X_B, t))
    x = torch.randn(X.shape[0], 4, dtype=torch.float64, device="cuda")
    assert torch.equal(Hh.matvec(x), Hg.matvec(x))
