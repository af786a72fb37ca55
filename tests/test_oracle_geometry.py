"""Pins for oracle/geometry.py (§II-A; readings R1-R6)."""
import numpy as np
import pytest
from oracle.geometry import (build_cluster_tree, build_partition, admissible, diameter, distance,
                             leaf_depth_for)
from synth import uniform_points, grid_points


def test_power_of_two_tree_shape():
    # n=512, leaf 64 -> 8 leaves of 64, 4 levels
    t = build_cluster_tree(uniform_points(512, 3, 1), 64)
    assert t.nlevels == 4 and t.leaf_depth == 3
    assert np.all(t.end[3] - t.begin[3] == 64)


def test_single_point_and_degenerate():
    t = build_cluster_tree(np.array([[0.5, 0.5, 0.5]]), 64)
    assert t.nlevels == 1
    p = build_partition(t, 0.7)
    assert p.near.tolist() == [[0, 0]] and p.top_depth() is None


@pytest.mark.parametrize("n,leaf", [(1000, 32), (777, 20), (5000, 64), (33, 2)])
def test_tree_invariants(n, leaf):
    X = uniform_points(n, 3, 4)
    t = build_cluster_tree(X, leaf)
    assert sorted(t.perm.tolist()) == list(range(n))                   # bijection
    assert t.leaf_depth == leaf_depth_for(n, leaf)
    assert np.max(t.end[t.leaf_depth] - t.begin[t.leaf_depth]) <= leaf
    for d in range(t.leaf_depth):
        for c in range(1 << d):
            b, e = t.begin[d][c], t.end[d][c]
            l, r = (e - b + 1) // 2, (e - b) // 2
            assert t.begin[d + 1][2 * c] == b and t.end[d + 1][2 * c + 1] == e
            assert t.end[d + 1][2 * c] - b == l and e - t.begin[d + 1][2 * c + 1] == r
    Xt = X[t.perm]
    for d in range(t.nlevels):
        for c in range(1 << d):
            P = Xt[t.begin[d][c]:t.end[d][c]]
            assert np.all(P >= t.lo[d][c]) and np.all(P <= t.hi[d][c])


def test_split_is_median_of_longest_axis():
    X = np.column_stack([np.arange(10.0), np.zeros(10), np.zeros(10)])[::-1].copy()
    t = build_cluster_tree(X, 5)
    Xt = X[t.perm]
    assert np.all(Xt[:5, 0] < Xt[5:, 0].min())


def test_grid_ties_deterministic():
    X = grid_points((8, 8, 4), 1.0 / 8)
    t1 = build_cluster_tree(X, 16)
    t2 = build_cluster_tree(X.copy(), 16)
    assert np.array_equal(t1.perm, t2.perm)


def test_admissibility_closed_form():
    # Eq.(1): unit boxes, centre distance 2 -> (sqrt3 + sqrt3)/2 <= 0.7 * 2 is False; at 3 True
    lo0, hi0 = np.zeros(3), np.ones(3)
    assert diameter(lo0, hi0) == np.sqrt(3.0)
    assert distance(lo0, hi0, lo0 + [2, 0, 0], hi0 + [2, 0, 0]) == 2.0
    assert distance(lo0, hi0, lo0 + [2, 0, 0], hi0 + [2, 0, 0], "box") == 1.0
    assert not (np.sqrt(3.0) <= 0.7 * 2.0)
    assert np.sqrt(3.0) <= 0.7 * 3.0


@pytest.mark.parametrize("rule", ["center", "box"])
def test_partition_tiles_matrix_once(rule):
    X = uniform_points(1500, 3, 9)
    t = build_cluster_tree(X, 32)
    p = build_partition(t, 0.7, rule)
    cover = np.zeros((t.n, t.n), np.int32)
    Dl = t.leaf_depth
    for s, b in p.near:
        cover[t.begin[Dl][s]:t.end[Dl][s], t.begin[Dl][b]:t.end[Dl][b]] += 1
    for d, f in enumerate(p.far):
        for s, b in f:
            cover[t.begin[d][s]:t.end[d][s], t.begin[d][b]:t.end[d][b]] += 1
            # admissible leaves have inadmissible parents
            assert not admissible(t, d - 1, s // 2, b // 2, 0.7, rule)
            assert admissible(t, d, s, b, 0.7, rule)
    assert np.all(cover == 1)
    # symmetry
    ns = set(map(tuple, p.near.tolist()))
    assert all((b, s) in ns for s, b in ns)
    for f in p.far:
        fs = set(map(tuple, f.tolist()))
        assert all((b, s) in fs for s, b in fs)


def test_eta_limits():
    X = uniform_points(1024, 2, 0)
    t = build_cluster_tree(X, 32)
    p0 = build_partition(t, 1e-12)
    assert len(p0.near) == (1 << t.leaf_depth) ** 2 and p0.top_depth() is None     # all dense
    pinf = build_partition(t, 1e12)                     # weak admissibility -> HSS partition
    assert sorted(map(tuple, pinf.near.tolist())) == [(c, c) for c in range(1 << t.leaf_depth)]
    for d in range(1, t.leaf_depth + 1):
        assert sorted(map(tuple, pinf.far[d].tolist())) == sorted(
            [(c, c ^ 1) for c in range(1 << d)])


def test_box_rule_refines_more_than_centre_rule():
    # the box distance is never larger than the centre distance, so it admits fewer pairs
    X = uniform_points(4096, 3, 0)
    t = build_cluster_tree(X, 64)
    pc, pb = build_partition(t, 0.7, "center"), build_partition(t, 0.7, "box")
    assert len(pb.near) > len(pc.near)


def test_smaller_eta_refines():
    # smaller eta -> more refined partition, larger C_sp
    X = uniform_points(4096, 3, 0)
    t = build_cluster_tree(X, 64)
    p5, p7 = build_partition(t, 0.5), build_partition(t, 0.7)
    assert len(p5.near) >= len(p7.near)
    assert sum(len(f) for f in p5.far) + len(p5.near) > sum(len(f) for f in p7.far) + len(p7.near)
