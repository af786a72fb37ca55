"""CPU-only checks of the C-ABI library: it loads, exports every symbol include/h2.h declares,
and its host-side partition (a0: KD-tree + dual traversal -> CSR descriptors) is bit-identical
to the oracle's (integer/index work must be bit-exact)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle import geometry
from synth import uniform_points, grid_points

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "h2.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = set(re.findall(r"\b(h2_[a-z_0-9]+)\s*\(", src))
    return sorted(n for n in names if not n.endswith("_fn"))


def test_library_exports_every_header_symbol():
    from paper_2506_16759_b200 import _lib
    syms = header_symbols()
    assert len(syms) >= 18
    lib = C.CDLL(_lib.LIB_PATH)
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)
    assert b"sm_100a" in _lib.lib.h2_version()


def test_library_is_sm100a_only():
    from paper_2506_16759_b200 import _lib
    out = os.popen(f"cuobjdump --list-elf {_lib.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out.replace("sm_100a", "")), out


@pytest.mark.parametrize("case", ["u3d_5000_64", "u2d_1024_32", "grid_8x8x8_16", "u3d_777_20", "box_rule",
                                  "u1d_300_8"])
def test_partition_bit_identical_to_oracle(case):
    from paper_2506_16759_b200 import Tree
    rule = "center"
    if case == "u3d_5000_64":
        X, leaf = uniform_points(5000, 3, 0), 64
    elif case == "u2d_1024_32":
        X, leaf = uniform_points(1024, 2, 0), 32
    elif case == "grid_8x8x8_16":
        X, leaf = grid_points((8, 8, 8), 1 / 8), 16
    elif case == "u3d_777_20":
        X, leaf = uniform_points(777, 3, 5), 20
    elif case == "u1d_300_8":
        X, leaf = uniform_points(300, 1, 5), 8
    else:
        X, leaf, rule = uniform_points(3000, 3, 1), 48, "box"
    T = Tree(X, leaf, 0.7, rule)
    ot = geometry.build_cluster_tree(X, leaf)
    op = geometry.build_partition(ot, 0.7, rule)
    assert T.leaf_depth == ot.leaf_depth
    assert np.array_equal(T.perm, ot.perm)
    for t in range(ot.nlevels):
        assert np.array_equal(T.begin[t], ot.begin[t]) and np.array_equal(T.end[t], ot.end[t])
        assert np.array_equal(T.far[t], op.far[t]), t
    assert np.array_equal(T.near, op.near)
    assert (T.top_depth if T.top_depth >= 0 else None) == op.top_depth()


def test_tree_errors_are_reported():
    from paper_2506_16759_b200 import Tree, H2Error
    with pytest.raises(H2Error, match="leaf_size"):
        Tree(uniform_points(10, 3, 0), 1)
    bad = uniform_points(10, 3, 0)
    bad[3, 1] = np.nan
    with pytest.raises(H2Error, match="non-finite"):
        Tree(bad, 4)


def test_tree_import_roundtrip_and_validation():
    """h2_tree_import: the oracle's partition imported into libh2 exports back
    unchanged; malformed partitions are refused with INVALID_ARG (host logic, no device)."""
    import paper_2506_16759_b200 as g
    X = uniform_points(3000, 3, 4)
    tree = geometry.build_cluster_tree(X, 64)
    part = geometry.build_partition(tree, 0.7)
    T = g.Tree.from_partition(X, tree.perm, tree.begin, tree.end, part.near, part.far)
    assert np.array_equal(T.perm, tree.perm)
    assert np.array_equal(T.near, part.near)
    assert all(np.array_equal(a, b) for a, b in zip(T.far, part.far))
    assert all(np.array_equal(T.begin[t], tree.begin[t]) for t in range(tree.leaf_depth + 1))
    assert T.top_depth == part.top_depth()
    bad_perm = tree.perm.copy()
    bad_perm[0] = bad_perm[1]
    far_asym = [f.copy() for f in part.far]
    t0 = part.top_depth()
    far_asym[t0] = far_asym[t0][far_asym[t0][:, 0] != far_asym[t0][0, 0]]   # drop one row's pairs
    ends = [e.copy() for e in tree.end]
    ends[1][0] += 1
    for args in [(bad_perm, tree.begin, tree.end, part.near, part.far),
                 (tree.perm, tree.begin, tree.end, part.near, far_asym),
                 (tree.perm, tree.begin, ends, part.near, part.far),
                 (tree.perm, tree.begin, tree.end, part.near[:-1], part.far)]:
        with pytest.raises(g.H2Error) as e:
            g.Tree.from_partition(X, *args)
        assert e.value.status == -1


@pytest.mark.parametrize("case", ["u3d_5000_64", "u2d_1024_32", "grid_8x8x8_16"])
def test_async_tree_matches_sync(case):
    """h2_tree_build_async (the block partition on a host thread, waited for by its first reader)
    yields exactly the synchronous partition; freeing an async tree with its thread still running
    is safe (the destructor joins)."""
    import paper_2506_16759_b200 as g
    X, leaf = {"u3d_5000_64": (uniform_points(5000, 3, 0), 64), "u2d_1024_32": (uniform_points(1024, 2, 0), 32),
               "grid_8x8x8_16": (grid_points((8, 8, 8), 1 / 8), 16)}[case]
    Ts, Ta = g.Tree(X, leaf), g.Tree(X, leaf, asynchronous=True)
    for a in ("leaf_depth", "top_depth", "csp", "near_nnz", "far_nnz_total"):
        assert getattr(Ts, a) == getattr(Ta, a), a
    assert np.array_equal(Ts.perm, Ta.perm)
    assert np.array_equal(Ts.near, Ta.near)
    assert all(np.array_equal(a, b) for a, b in zip(Ts.far, Ta.far))
    for _ in range(3):
        T = g.Tree(X, leaf, asynchronous=True)
        del T
