"""Shared helpers of the GPU parity tests: run the oracle and the CUDA path (through the C ABI)
on the same seeded inputs and compare them as DESIGN.md "Parity contract" states."""
import numpy as np
import torch

from oracle import geometry, kernels, h2 as oh2, rng
import paper_2506_16759_b200 as g

# a skeleton mismatch is accepted only where the oracle's own CPQR took a decision within this
# relative distance of a tie (pivot gap) or of the threshold (truncation margin): perturbations
# of Y^loc by rounding (different summation orders, ~1e-14 absolute) move residual norms near
# eps = 1e-7 rho by < 1e-9 relative.
CERT_TOL = 1e-7


def oracle_build(X, kind, param, leaf, tol, eta=0.7, seed=1, **opts):
    tree = geometry.build_cluster_tree(X, leaf)
    part = geometry.build_partition(tree, eta)
    op = kernels.KernelOperator(kind, param, X[tree.perm])
    om = lambda c0, nc: rng.omega_block(seed, 0, 0, tree.n, c0, nc)
    H = oh2.build(tree, part, op.sampler, op.entry, om, tol, oh2.BuildOpts(**opts))
    return H, op


def compare_builds(Hg, Ho, diverged_out=None):
    """Level by level from the leaves: ranks and skeletons bit-exact where comparable; a
    mismatch must be certified by the oracle (near-tie).  Descendants of a diverged cluster
    (its ancestors in the tree) are excluded.  Returns (#certified mismatches, #compared);
    diverged_out (dict) receives depth -> bool mask of the clusters excluded or diverged."""
    Dl = Ho.tree.leaf_depth
    assert Hg.top_depth == Ho.top
    diverged = {Dl + 1: np.zeros(1 << (Dl + 1), bool)}
    certified = compared = 0
    for t in range(Dl, Ho.top - 1, -1):
        rg = Hg.rank(t)
        sg = Hg.skel(t)
        Xg = Hg.basis(t)
        div = np.zeros(1 << t, bool)
        for c in range(1 << t):
            if t < Dl and (diverged[t + 1][2 * c] or diverged[t + 1][2 * c + 1]):
                div[c] = True
                continue
            compared += 1
            ido = Ho.ids[t][c]
            same = rg[c] == ido.k and np.array_equal(sg[c], Ho.skel[t][c])
            if not same:
                near_tie = ido.min_gap < CERT_TOL or ido.stop_margin < CERT_TOL
                assert near_tie, (f"depth {t} cluster {c}: rank {rg[c]} vs {ido.k}, gap {ido.min_gap:.3e}, "
                                  f"margin {ido.stop_margin:.3e}")
                certified += 1
                div[c] = True
                continue
            # identity rows bitwise
            J = ido.J
            assert np.array_equal(Xg[c][J], np.eye(len(J)))
            # interpolation property on the ORACLE's panel: with the same J, the CUDA basis must
            # reproduce Y^loc to the truncation bound ||R3||_F <= sqrt(m-k) eps (Eq.(3)); X itself
            # is only determined to cond(R11) u (T = R11^{-1} R12, cond up to rho/eps ~ 1e7), so it
            # is not compared entrywise
            P = Ho.panels[t][c]
            if P.size:
                res = np.linalg.norm(P - Xg[c] @ P[J])
                res_o = np.linalg.norm(P - Ho.X[t][c] @ P[J])
                bound = np.sqrt(max(P.shape[0] - len(J), 0)) * Ho.eps
                assert res <= 1.01 * bound + 1e-12 * np.linalg.norm(P), (t, c, res, res_o, bound)
        diverged[t] = div
    if diverged_out is not None:
        diverged_out.update({t: diverged[t] for t in range(Ho.top, Dl + 1)})
    return certified, compared


def compare_blocks(Hg, Ho, diverged, tol_b=4e-15, tol_d=3.2e-15):
    """D blocks entrywise (they do not depend on the skeletons: every near pair is compared) and B
    blocks of every far pair whose two clusters have bit-identical skeletons (diverged clusters
    are compared by error instead, see compare_matvec).  Returns the number of B blocks compared."""
    for (s, b), blk in Hg.D_blocks().items():
        ref = Ho.D[(s, b)]
        assert np.abs(blk - ref).max() <= tol_d * max(1.0, np.abs(ref).max()), (s, b)
    nb = 0
    for t in range(Ho.top, Ho.tree.leaf_depth + 1):
        div = diverged[t]
        for (s, b), blk in Hg.B_blocks(t).items():
            if div[s] or div[b]:
                continue
            ref = Ho.B[t][(s, b)]
            assert np.abs(blk - ref).max() <= tol_b * max(1.0, np.abs(ref).max()), (t, s, b)
            nb += 1
    return nb


def compare_matvec(Hg, Ho, certified, err_bound, seed=3, exact_bound=1e-10):
    """H^2 matvecs of both representations: <= 1e-10 relative when every skeleton matched
    (BASELINE north_star); with certified near-tie divergences the two are different valid
    approximations and agree to the sum of their error bounds (each within err_bound of K)."""
    x = np.random.default_rng(seed).standard_normal((Ho.tree.n, 5))
    yg = Hg.matvec(torch.from_numpy(x).cuda()).cpu().numpy()
    yo = oh2.matvec(Ho, x)
    rel = np.linalg.norm(yg - yo) / np.linalg.norm(yo)
    assert rel <= (exact_bound if certified == 0 else 2 * err_bound), rel
    return rel


def probe_error(Hg, K, q=8, seed=2):
    X = np.random.default_rng(seed).standard_normal((K.shape[0], q))
    y = Hg.matvec(torch.from_numpy(X).cuda()).cpu().numpy()
    ref = K @ X
    return np.linalg.norm(y - ref) / np.linalg.norm(ref)
