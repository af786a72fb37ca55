"""Early exit of failing adaptive convergence tests (CpqrArgs::fail_cap / fail_flag, DESIGN.md §6
CPQR): a round whose level is already known to fail (a cluster with m > d still above eps at
step d - p_os - 1) stops every panel of the launch.  The level decision is exact, so the build
must be BITWISE the build without the early exit (H2_CQ_EARLY=0): samples, rounds, ranks,
skeletons, bases, certificates, B and D."""
import os

import numpy as np
import pytest

from synth import uniform_points, grid_points
import paper_2506_16759_b200 as g

pytestmark = pytest.mark.gpu


def _snap(H):
    L = g._lib
    out = {"samples": H.samples, "rounds": dict(H.stats["rounds"])}
    for t in range(H.top_depth, H.tree.leaf_depth + 1):
        for what in (L.H2_X_RANK, L.H2_X_SKEL):
            out[(what, t)] = H._export(what, t, dtype=np.int32).copy()
        for what in (L.H2_X_BASIS, L.H2_X_B, L.H2_X_CERT):
            out[(what, t)] = H._export(what, t).copy()
    out["D"] = H._export(L.H2_X_D).copy()
    return out


@pytest.mark.parametrize("case", [("u3", 8192, "exp", 0.2, 1e-6, {}), ("u3", 16384, "exp", 0.2, 1e-8, {}),
                                  ("u3", 8192, "exp", 0.2, 1e-7, {"tol_rule": "literal", "norm": 0.0, "d_init": 16, "d_blk": 16}),
                                  ("grid", 4096, "helmholtz", 3.0, 1e-4, {}),
                                  ("u3", 8192, "exp", 0.2, 1e-6, {"H2_CQ_VARIANT": "global"})])
def test_early_exit_bitwise(case, monkeypatch):
    kind, n, kern, param, tol, opts = case
    opts = dict(opts)
    variant = opts.pop("H2_CQ_VARIANT", None)
    if variant:
        monkeypatch.setenv("H2_CQ_VARIANT", variant)
    X = uniform_points(n, 3 if kind == "u3" else 2, 5) if kind != "grid" else grid_points((16, 16, 16), 1 / 16)
    T = g.Tree(X, 64)
    monkeypatch.setenv("H2_CQ_EARLY", "0")
    a = _snap(g.build(T, (kern, param), tol, **opts))
    monkeypatch.setenv("H2_CQ_EARLY", "1")
    b = _snap(g.build(T, (kern, param), tol, **opts))
    assert max(a["rounds"].values()) > 1, "case must contain a failing convergence test"
    bad = [k for k in a if not (a[k] == b[k] if k in ("samples", "rounds") else np.array_equal(a[k], b[k]))]
    assert not bad, bad


@pytest.mark.parametrize("case", [(8192, 3, {"H2_CQ_VARIANT": "cluster"}, {"H2_CQ_VARIANT": "global"}),
                                  (65536, 3, {}, {"H2_CQ_CLUSTER": "0"}),
                                  (16384, 2, {"H2_CQ_VARIANT": "cluster"}, {"H2_CQ_VARIANT": "smem"})])
def test_cluster_cpqr_bitwise(case, monkeypatch):
    """The CTA-cluster CPQR (rows in distributed shared memory, retired in place, positions
    tracked) performs each row's arithmetic and each pivot decision exactly as the row-swapping
    one-CTA kernels: builds with it forced on every level, or chosen for the panels that do not
    fit one CTA (default, N = 2^16), are bitwise the builds without it."""
    n, dim, env_a, env_b = case
    X = uniform_points(n, dim, 7)
    T = g.Tree(X, 64)
    out = []
    for env in (env_a, env_b):
        for k in ("H2_CQ_VARIANT", "H2_CQ_CLUSTER"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        H = g.build(T, ("exp", 0.2), 1e-6)
        out.append((_snap(H), H.stats["cpqr_variants"]))
    (a, va), (b, vb) = out
    assert va & g._lib.H2_CQ_V_CLUSTER and not vb & g._lib.H2_CQ_V_CLUSTER, (va, vb)
    bad = [k for k in a if not (a[k] == b[k] if k in ("samples", "rounds") else np.array_equal(a[k], b[k]))]
    assert not bad, bad
