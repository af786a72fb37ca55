"""Algorithm 1: bottom-up sketching construction of a symmetric H^2
matrix, fixed-sample (§III-A) and adaptive (§III-B), plus the H^2
matvec and dense reconstruction used for verification.  TEST INFRA.

Notation follows the paper: level l = 1 is the leaf level (L204-205); here clusters are
addressed by depth t (root 0, leaves Dl), l = Dl - t + 1.  Per cluster tau:
  Y^l_tau, Omega^l_tau   samples / projected random vectors (L208, L230-236)
  Y^loc_tau              samples of the admissible part only (L213, L240-243)
  J_tau, X_tau           row ID of Y^loc_tau (L221, L250): X = U_tau (leaf) or [E_nu1; E_nu2]
  skel[tau] = I~_tau     skeleton indices (L224, L253), tree-order global indices
  D[(tau,b)], b in N_tau  dense blocks (L212);  B[t][(tau,b)], b in F_tau  couplings (L258)

Readings used: R9 (d_init/d_blk/d_max), R10-R13 (tolerance and convergence test),
R16 (skeleton order), R17 (typos in L250/L252/L334/L341/L361), R26 (NOT_CONVERGED).
"""
from dataclasses import dataclass, field
import numpy as np

from .cpqr import row_id


class NotConverged(RuntimeError):
    def __init__(self, depth):
        super().__init__(f"adaptive sampling reached d_max at depth {depth}")
        self.depth = depth


@dataclass
class BuildOpts:
    d_init: int = 32
    d_blk: int = 32
    d_max: int = 512
    adaptive: bool = True
    tol_rule: str = "rms"        # "rms": eps = s * tol * ||Y||_F / sqrt(N);  "literal": eps = tol * nu
    tol_safety: float = 0.04     # s (leaf depth; R31)
    p_os: int = 10               # oversampling margin in the convergence test (0 in literal mode)
    norm: float = 0.0            # nu for the literal rule
    max_rank: int = None
    eps_decay: float = 1.25      # R31: eps at depth t scaled by eps_decay^(Dl - t)


@dataclass
class H2Matrix:
    tree: object
    part: object
    top: int                                     # coarsest processed depth
    rank: dict = field(default_factory=dict)     # depth -> int array
    skel: dict = field(default_factory=dict)     # depth -> list of int64 arrays
    X: dict = field(default_factory=dict)        # depth -> list of bases (U at leaves, [E1;E2] above)
    ids: dict = field(default_factory=dict)      # depth -> list of RowID (certification data)
    panels: dict = field(default_factory=dict)   # depth -> list of Y^loc_tau (m x d) at commit
    D: dict = field(default_factory=dict)        # (s, b) -> block, leaf depth
    B: dict = field(default_factory=dict)        # depth -> {(s, b): block}
    samples: int = 0
    rounds: dict = field(default_factory=dict)   # depth -> number of convergence tests
    eps: float = 0.0


def _eps(opts, tol, sumsq, n, levels_up=0):
    """R10/R11: eps_l (eps_abs = eps * approximate norm); R31: times
    eps_decay^levels_up (levels_up = Dl - t)."""
    lvl = 1.0 if opts.eps_decay == 1.0 else opts.eps_decay ** levels_up
    if opts.tol_rule == "rms":
        return lvl * (opts.tol_safety * tol * np.sqrt(sumsq / n))
    if opts.tol_rule == "literal":
        return lvl * (tol * opts.norm)
    raise ValueError(opts.tol_rule)


def _converged(opts, m, k, d):
    """R12: converged iff the panel is saturated (m <= d) or k <= d - 1 - p_os."""
    p = opts.p_os if opts.tol_rule == "rms" else 0
    return m <= d or k <= d - 1 - p


def leaf_local_samples(tree, part, D, Yc, Oc):
    """Line 213: Y^loc_tau = Y^1_tau - sum_{b in N_tau} D_{tau,b} Omega^1_b (b ascending),
    Omega^1_tau = Omega(I_tau, :) (line 208).  Returns per-leaf lists (Y^loc, Omega^1)."""
    Dl = tree.leaf_depth
    Yl, Ol = [], []
    for tau in range(1 << Dl):
        I = np.arange(tree.begin[Dl][tau], tree.end[Dl][tau])
        acc = Yc[I].copy()
        for b in part.near_of(tau):
            acc = acc - D[(tau, int(b))] @ Oc[tree.begin[Dl][b]:tree.end[Dl][b]]
        Yl.append(acc)
        Ol.append(Oc[I].copy())
    return Yl, Ol


def build(tree, part, sampler, entry, omega, tol, opts: BuildOpts = None) -> H2Matrix:
    """Algorithm 1.  sampler(Omega) -> K Omega (N x c); entry(rows, cols) -> K(rows, cols);
    omega(col0, ncols) -> columns [col0, col0+ncols) of the random stream (N x ncols)."""
    opts = opts or BuildOpts()
    N, Dl = tree.n, tree.leaf_depth
    ttop = part.top_depth()
    top = Dl if ttop is None else min(ttop, Dl)
    H = H2Matrix(tree, part, top)
    rng_of = lambda t, c: np.arange(tree.begin[t][c], tree.end[t][c])

    # line 1: Y = K_blk(Omega)
    d = opts.d_init
    Om = omega(0, d)
    Y = sampler(Om)

    def block_sumsq(Yb):
        """||Y_block||_F^2 as DESIGN.md R28 reads it: per-leaf partial sums, added in leaf order."""
        tot = 0.0
        for c in range(1 << Dl):
            rows = Yb[tree.begin[Dl][c]:tree.end[Dl][c]]
            tot += float(np.sum(rows * rows))
        return tot

    sumsq = block_sumsq(Y)
    # line 212: D_{tau,b} = K(I_tau, I_b), b in N_tau
    for (s, b) in part.near:
        H.D[(int(s), int(b))] = entry(rng_of(Dl, s), rng_of(Dl, b))

    def leaf_subtract(Yc, Oc):
        return leaf_local_samples(tree, part, H.D, Yc, Oc)

    def inner_subtract(t, Yn, On):
        """lines 230-243 at depth t: merge children (nu1 first) and subtract
        sum_{b in F_nu} B_{nu,b} Omega^l_b for each child nu (depth t+1)."""
        Yl, Ol = [], []
        for tau in range(1 << t):
            parts_y, parts_o = [], []
            for nu in (2 * tau, 2 * tau + 1):
                acc = Yn[nu].copy()
                for b in part.far_of(t + 1, nu):
                    acc = acc - H.B[t + 1][(nu, int(b))] @ On[int(b)]
                parts_y.append(acc)
                parts_o.append(On[nu])
            Yl.append(np.vstack(parts_y))
            Ol.append(np.vstack(parts_o))
        return Yl, Ol

    def commit_up(t, Yl, Ol):
        """lines 222-223 / 251-252: Y^{l+1}_tau = Y^loc_tau(J,:), Omega^{l+1}_tau = X^T Omega^l_tau."""
        Yn = [Yl[c][H.ids[t][c].J] for c in range(1 << t)]
        On = [H.X[t][c].T @ Ol[c] for c in range(1 << t)]
        return Yn, On

    def sweep_new(target, Ybar, Obar):
        """updateSamples (L217, L247, L386): sweep new samples and vectors up the tree with the
        stored D, B, J, U/E of the completed levels until the current level `target`."""
        Yl, Ol = leaf_subtract(Ybar, Obar)
        t = Dl
        while t > target:
            Yn, On = commit_up(t, Yl, Ol)
            t -= 1
            Yl, Ol = inner_subtract(t, Yn, On)
        return Yl, Ol

    Yl, Ol = leaf_subtract(Y, Om)
    for t in range(Dl, top - 1, -1):
        if t < Dl:
            Yl, Ol = inner_subtract(t, Yn, On)
        rounds = 0
        while True:
            eps = _eps(opts, tol, sumsq, N, Dl - t)
            ids = [row_id(Yl[c], eps, opts.max_rank) for c in range(1 << t)]
            rounds += 1
            if not opts.adaptive:
                break
            if all(_converged(opts, Yl[c].shape[0], ids[c].k, d) for c in range(1 << t)):
                break
            if d + opts.d_blk > opts.d_max:
                raise NotConverged(t)
            # lines 216-217 / 246-247: new random block and samples, swept up to this level
            Obar = omega(d, opts.d_blk)
            Ybar = sampler(Obar)
            sumsq += block_sumsq(Ybar)
            nY, nO = sweep_new(t, Ybar, Obar)
            Yl = [np.hstack([Yl[c], nY[c]]) for c in range(1 << t)]
            Ol = [np.hstack([Ol[c], nO[c]]) for c in range(1 << t)]
            d += opts.d_blk
        H.rounds[t] = rounds
        H.eps = eps
        # lines 221-224 / 250-253: ID, skeletons
        H.ids[t] = ids
        H.panels[t] = Yl                          # Y^loc_tau at the final d (verification data)
        H.X[t] = [i.X for i in ids]
        H.rank[t] = np.array([i.k for i in ids], np.int64)
        if t == Dl:
            H.skel[t] = [rng_of(Dl, c)[ids[c].J] for c in range(1 << t)]
        else:
            H.skel[t] = [np.concatenate([H.skel[t + 1][2 * c], H.skel[t + 1][2 * c + 1]])[ids[c].J]
                         for c in range(1 << t)]
        Yn, On = commit_up(t, Yl, Ol)
        # line 258: B_{tau,b} = K(I~_tau, I~_b), b in F_tau
        H.B[t] = {(int(s), int(b)): entry(H.skel[t][s], H.skel[t][b]) for (s, b) in part.far[t]}
    H.samples = d
    return H


def expanded_basis(H: H2Matrix, t: int, c: int) -> np.ndarray:
    """U_tau for a cluster at depth t via the nested-basis recursion Eq.(2):
    U_tau = diag(U_nu1, U_nu2) [E_nu1; E_nu2].  Rows indexed by I_tau (tree order)."""
    Dl = H.tree.leaf_depth
    if t == Dl:
        return H.X[t][c]
    U1 = expanded_basis(H, t + 1, 2 * c)
    U2 = expanded_basis(H, t + 1, 2 * c + 1)
    k1 = U1.shape[1]
    Xc = H.X[t][c]
    return np.vstack([U1 @ Xc[:k1], U2 @ Xc[k1:]])


def matvec(H: H2Matrix, x: np.ndarray) -> np.ndarray:
    """y = K_H x (H^2 matvec: upward pass, coupling, downward pass, dense leaves)."""
    tree, part, Dl = H.tree, H.part, H.tree.leaf_depth
    x = np.asarray(x, np.float64)
    vec = x.ndim == 1
    if vec:
        x = x[:, None]
    q = x.shape[1]
    rng_of = lambda t, c: np.arange(tree.begin[t][c], tree.end[t][c])
    y = np.zeros((tree.n, q))
    xh = {Dl: [H.X[Dl][c].T @ x[rng_of(Dl, c)] for c in range(1 << Dl)]}
    for t in range(Dl - 1, H.top - 1, -1):
        xh[t] = [H.X[t][c].T @ np.vstack([xh[t + 1][2 * c], xh[t + 1][2 * c + 1]]) for c in range(1 << t)]
    yh = {}
    for t in range(H.top, Dl + 1):
        yh[t] = [np.zeros((H.rank[t][c], q)) for c in range(1 << t)]
        for (s, b) in part.far[t]:
            yh[t][s] = yh[t][s] + H.B[t][(int(s), int(b))] @ xh[t][int(b)]
    for t in range(H.top, Dl):
        for c in range(1 << t):
            z = H.X[t][c] @ yh[t][c]
            k1 = H.rank[t + 1][2 * c]
            yh[t + 1][2 * c] = yh[t + 1][2 * c] + z[:k1]
            yh[t + 1][2 * c + 1] = yh[t + 1][2 * c + 1] + z[k1:]
    for c in range(1 << Dl):
        I = rng_of(Dl, c)
        y[I] += H.X[Dl][c] @ yh[Dl][c]
    for (s, b) in part.near:
        y[rng_of(Dl, s)] += H.D[(int(s), int(b))] @ x[rng_of(Dl, b)]
    return y[:, 0] if vec else y


def to_dense(H: H2Matrix) -> np.ndarray:
    """Dense reconstruction block by block: D for near pairs, U_s B U_t^T for far pairs."""
    tree, part, Dl = H.tree, H.part, H.tree.leaf_depth
    n = tree.n
    K = np.zeros((n, n))
    sl = lambda t, c: slice(tree.begin[t][c], tree.end[t][c])
    for (s, b) in part.near:
        K[sl(Dl, s), sl(Dl, b)] = H.D[(int(s), int(b))]
    for t in range(H.top, Dl + 1):
        for (s, b) in part.far[t]:
            Us = expanded_basis(H, t, int(s))
            Ub = expanded_basis(H, t, int(b))
            K[sl(t, s), sl(t, b)] = Us @ H.B[t][(int(s), int(b))] @ Ub.T
    return K
