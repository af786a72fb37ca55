"""Random symmetric H^2 matrix of prescribed ranks on a given tree/partition, assembled
densely by its definition (Eq.(2) nested basis, L143-158) -- written in the test
suite, independently of oracle/h2.py, to pin the oracle's construction."""
import numpy as np


def synthetic_h2(tree, part, rank_of, seed=0):
    """rank_of(depth, size_or_childranks) -> rank.  Returns (K dense, ranks per depth,
    active per depth) where active[t][c] says whether cluster c at depth t or one of its
    ancestors owns an admissible block (so its sampled far field is non-zero)."""
    rng = np.random.default_rng(seed)
    Dl = tree.leaf_depth
    ttop = part.top_depth()
    n = tree.n
    ranks, U = {}, {}
    ranks[Dl] = np.array([rank_of(Dl, tree.size(Dl, c)) for c in range(1 << Dl)])
    U[Dl] = [rng.standard_normal((tree.size(Dl, c), ranks[Dl][c])) for c in range(1 << Dl)]
    for t in range(Dl - 1, (ttop if ttop is not None else Dl) - 1, -1):
        ranks[t] = np.array([rank_of(t, ranks[t + 1][2 * c] + ranks[t + 1][2 * c + 1]) for c in range(1 << t)])
        U[t] = []
        for c in range(1 << t):
            E1 = rng.standard_normal((ranks[t + 1][2 * c], ranks[t][c]))
            E2 = rng.standard_normal((ranks[t + 1][2 * c + 1], ranks[t][c]))
            U[t].append(np.vstack([U[t + 1][2 * c] @ E1, U[t + 1][2 * c + 1] @ E2]))
    K = np.zeros((n, n))
    sl = lambda t, c: slice(tree.begin[t][c], tree.end[t][c])
    for (s, b) in part.near:
        if s <= b:
            blk = rng.standard_normal((tree.size(Dl, s), tree.size(Dl, b)))
            if s == b:
                blk = blk + blk.T
            K[sl(Dl, s), sl(Dl, b)] = blk
            K[sl(Dl, b), sl(Dl, s)] = blk.T
    for t, f in enumerate(part.far):
        for (s, b) in f:
            if s < b:
                Bst = rng.standard_normal((ranks[t][s], ranks[t][b]))
                blk = U[t][s] @ Bst @ U[t][b].T
                K[sl(t, s), sl(t, b)] = blk
                K[sl(t, b), sl(t, s)] = blk.T
    active = {}
    top = ttop if ttop is not None else Dl
    for t in range(top, Dl + 1):
        own = np.zeros(1 << t, bool)
        own[np.unique(part.far[t][:, 0]) if len(part.far[t]) else []] = True
        if t > top:
            own |= np.repeat(active[t - 1], 2)
        active[t] = own
    return K, ranks, active


def _nested(tree, rng, ranks_of, Dl, top):
    ranks, U = {}, {}
    ranks[Dl] = np.array([ranks_of(Dl, tree.size(Dl, c)) for c in range(1 << Dl)])
    U[Dl] = [rng.standard_normal((tree.size(Dl, c), ranks[Dl][c])) for c in range(1 << Dl)]
    for t in range(Dl - 1, top - 1, -1):
        ranks[t] = np.array([ranks_of(t, ranks[t + 1][2 * c] + ranks[t + 1][2 * c + 1]) for c in range(1 << t)])
        U[t] = []
        for c in range(1 << t):
            E1 = rng.standard_normal((ranks[t + 1][2 * c], ranks[t][c]))
            E2 = rng.standard_normal((ranks[t + 1][2 * c + 1], ranks[t][c]))
            U[t].append(np.vstack([U[t + 1][2 * c] @ E1, U[t + 1][2 * c + 1] @ E2]))
    return ranks, U


def synthetic_h2_nonsym(tree, part, row_rank_of, col_rank_of, seed=0):
    """Random NON-symmetric H^2 matrix K = D + U B V^T ("non-symmetric case"):
    independent nested row bases U (ranks row_rank_of) and column bases V (ranks col_rank_of),
    independent random blocks for (s, b) and (b, s).  Returns (K, row ranks, col ranks, active)."""
    rng = np.random.default_rng(seed)
    Dl = tree.leaf_depth
    ttop = part.top_depth()
    top = ttop if ttop is not None else Dl
    rr, U = _nested(tree, rng, row_rank_of, Dl, top)
    rc, V = _nested(tree, rng, col_rank_of, Dl, top)
    K = np.zeros((tree.n, tree.n))
    sl = lambda t, c: slice(tree.begin[t][c], tree.end[t][c])
    for (s, b) in part.near:
        K[sl(Dl, s), sl(Dl, b)] = rng.standard_normal((tree.size(Dl, s), tree.size(Dl, b)))
    for t, f in enumerate(part.far):
        for (s, b) in f:
            K[sl(t, s), sl(t, b)] = U[t][s] @ rng.standard_normal((rr[t][s], rc[t][b])) @ V[t][b].T
    active = {}
    for t in range(top, Dl + 1):
        own = np.zeros(1 << t, bool)
        own[np.unique(part.far[t][:, 0]) if len(part.far[t]) else []] = True
        if t > top:
            own |= np.repeat(active[t - 1], 2)
        active[t] = own
    return K, rr, rc, active
