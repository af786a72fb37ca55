"""Non-symmetric variant of Algorithm 1 ("the extension to
the non-symmetric case ... is straightforward", L268): K ~ D + U B V^T with row bases U from the
sketch Y = K Omega and column bases V from the sketch Z = K^T Psi.  TEST INFRA.

The two constructions run in lockstep level by level (they are coupled through the subtraction
of the compressed far field):
  row side    Y^loc_tau = Y^l_tau - sum_b B_{nu,b} Omega^l_b,   Omega^l_b = V_b^T Omega(I_b)
  column side Z^loc_tau = Z^l_tau - sum_b B_{b,nu}^T Psi^l_b,   Psi^l_b   = U_b^T Psi(I_b)
with B_{s,b} = K(I~_s, J~_b) (row skeletons of s, column skeletons of b) for every ORDERED far
pair and D_{s,b} = K(I_s, I_b) for every ordered near pair.  Each side is exactly the symmetric
construction of oracle/h2.py (same CPQR row ID, same order of operations) applied to its own
samples, with the other side's projected random vectors in the subtraction.  Readings (DESIGN.md
R29): the tolerance scale rho is the RMS row norm of all Y and Z columns together; a level
converges when every cluster of BOTH sides passes the R12 test; new samples are drawn for both
sides together; Psi is the Omega stream with stream id 1.
"""
from dataclasses import dataclass, field
import numpy as np

from .cpqr import row_id
from .h2 import BuildOpts, NotConverged, _converged


@dataclass
class H2NonSym:
    tree: object
    part: object
    top: int
    rank_r: dict = field(default_factory=dict)   # depth -> row ranks
    rank_c: dict = field(default_factory=dict)   # depth -> column ranks
    skel_r: dict = field(default_factory=dict)   # depth -> list of row skeletons I~
    skel_c: dict = field(default_factory=dict)   # depth -> list of column skeletons J~
    Xr: dict = field(default_factory=dict)       # depth -> list of row bases (U / [E1; E2])
    Xc: dict = field(default_factory=dict)       # depth -> list of column bases (V / [F1; F2])
    D: dict = field(default_factory=dict)        # (s, b) ordered near pairs
    B: dict = field(default_factory=dict)        # depth -> {(s, b): K(I~_s, J~_b)} ordered far pairs
    ids_r: dict = field(default_factory=dict)    # depth -> list of RowID (certification data)
    ids_c: dict = field(default_factory=dict)
    panels_r: dict = field(default_factory=dict) # depth -> list of Y^loc_tau at commit
    panels_c: dict = field(default_factory=dict) # depth -> list of Z^loc_tau at commit
    samples: int = 0
    rounds: dict = field(default_factory=dict)
    eps: float = 0.0


def build_nonsym(tree, part, sampler, sampler_t, entry, omega, psi, tol, opts: BuildOpts = None) -> H2NonSym:
    """sampler(Om) -> K Om, sampler_t(Ps) -> K^T Ps, entry(rows, cols) -> K(rows, cols),
    omega / psi(col0, ncols) -> columns of the two random streams."""
    opts = opts or BuildOpts()
    N, Dl = tree.n, tree.leaf_depth
    ttop = part.top_depth()
    top = Dl if ttop is None else min(ttop, Dl)
    H = H2NonSym(tree, part, top)
    rng_of = lambda t, c: np.arange(tree.begin[t][c], tree.end[t][c])
    d = opts.d_init
    Om, Ps = omega(0, d), psi(0, d)
    Y, Z = sampler(Om), sampler_t(Ps)
    sumsq = float(np.sum(Y * Y)) + float(np.sum(Z * Z))
    for (s, b) in part.near:
        H.D[(int(s), int(b))] = entry(rng_of(Dl, s), rng_of(Dl, b))

    def eps_now(t):
        lvl = 1.0 if opts.eps_decay == 1.0 else opts.eps_decay ** (Dl - t)   # R31
        if opts.tol_rule == "rms":
            return lvl * (opts.tol_safety * tol * np.sqrt(sumsq / (2 * N)))
        return lvl * (tol * opts.norm)

    def leaf_subtract(Yc, Zc, Oc, Pc):
        """line 213 for both sides: Y^loc = Y - sum D Omega_b, Z^loc = Z - sum D_{b,tau}^T Psi_b."""
        Yl, Zl, Ol, Pl = [], [], [], []
        for tau in range(1 << Dl):
            I = rng_of(Dl, tau)
            ay, az = Yc[I].copy(), Zc[I].copy()
            for b in part.near_of(tau):
                J = rng_of(Dl, int(b))
                ay = ay - H.D[(tau, int(b))] @ Oc[J]
                az = az - H.D[(int(b), tau)].T @ Pc[J]
            Yl.append(ay)
            Zl.append(az)
            Ol.append(Oc[I].copy())
            Pl.append(Pc[I].copy())
        return Yl, Zl, Ol, Pl

    def inner_subtract(t, Yn, Zn, On, Pn):
        """lines 230-243 at depth t for both sides (children nu1 first)."""
        Yl, Zl, Ol, Pl = [], [], [], []
        for tau in range(1 << t):
            py, pz, po, pp = [], [], [], []
            for nu in (2 * tau, 2 * tau + 1):
                ay, az = Yn[nu].copy(), Zn[nu].copy()
                for b in part.far_of(t + 1, nu):
                    ay = ay - H.B[t + 1][(nu, int(b))] @ On[int(b)]
                    az = az - H.B[t + 1][(int(b), nu)].T @ Pn[int(b)]
                py.append(ay)
                pz.append(az)
                po.append(On[nu])
                pp.append(Pn[nu])
            Yl.append(np.vstack(py))
            Zl.append(np.vstack(pz))
            Ol.append(np.vstack(po))
            Pl.append(np.vstack(pp))
        return Yl, Zl, Ol, Pl

    def commit_up(t, Yl, Zl, Ol, Pl):
        """shrink each side's samples with its own ID; Omega (the K samples' random vectors) is
        projected with the COLUMN bases, Psi with the ROW bases."""
        Yn = [Yl[c][ids_r[t][c].J] for c in range(1 << t)]
        Zn = [Zl[c][ids_c[t][c].J] for c in range(1 << t)]
        On = [H.Xc[t][c].T @ Ol[c] for c in range(1 << t)]
        Pn = [H.Xr[t][c].T @ Pl[c] for c in range(1 << t)]
        return Yn, Zn, On, Pn

    def sweep_new(target, Yb, Zb, Ob, Pb):
        Yl, Zl, Ol, Pl = leaf_subtract(Yb, Zb, Ob, Pb)
        t = Dl
        while t > target:
            Yn, Zn, On, Pn = commit_up(t, Yl, Zl, Ol, Pl)
            t -= 1
            Yl, Zl, Ol, Pl = inner_subtract(t, Yn, Zn, On, Pn)
        return Yl, Zl, Ol, Pl

    ids_r, ids_c = {}, {}
    Yl, Zl, Ol, Pl = leaf_subtract(Y, Z, Om, Ps)
    for t in range(Dl, top - 1, -1):
        if t < Dl:
            Yl, Zl, Ol, Pl = inner_subtract(t, Yn, Zn, On, Pn)
        rounds = 0
        while True:
            eps = eps_now(t)
            ir = [row_id(Yl[c], eps, opts.max_rank) for c in range(1 << t)]
            ic = [row_id(Zl[c], eps, opts.max_rank) for c in range(1 << t)]
            rounds += 1
            if not opts.adaptive:
                break
            if all(_converged(opts, Yl[c].shape[0], ir[c].k, d) and _converged(opts, Zl[c].shape[0], ic[c].k, d)
                   for c in range(1 << t)):
                break
            if d + opts.d_blk > opts.d_max:
                raise NotConverged(t)
            Ob, Pb = omega(d, opts.d_blk), psi(d, opts.d_blk)
            Yb, Zb = sampler(Ob), sampler_t(Pb)
            sumsq += float(np.sum(Yb * Yb)) + float(np.sum(Zb * Zb))
            nY, nZ, nO, nP = sweep_new(t, Yb, Zb, Ob, Pb)
            Yl = [np.hstack([Yl[c], nY[c]]) for c in range(1 << t)]
            Zl = [np.hstack([Zl[c], nZ[c]]) for c in range(1 << t)]
            Ol = [np.hstack([Ol[c], nO[c]]) for c in range(1 << t)]
            Pl = [np.hstack([Pl[c], nP[c]]) for c in range(1 << t)]
            d += opts.d_blk
        H.rounds[t] = rounds
        H.eps = eps
        ids_r[t], ids_c[t] = ir, ic
        H.ids_r[t], H.ids_c[t] = ir, ic
        H.panels_r[t], H.panels_c[t] = Yl, Zl
        H.Xr[t] = [i.X for i in ir]
        H.Xc[t] = [i.X for i in ic]
        H.rank_r[t] = np.array([i.k for i in ir], np.int64)
        H.rank_c[t] = np.array([i.k for i in ic], np.int64)
        if t == Dl:
            H.skel_r[t] = [rng_of(Dl, c)[ir[c].J] for c in range(1 << t)]
            H.skel_c[t] = [rng_of(Dl, c)[ic[c].J] for c in range(1 << t)]
        else:
            H.skel_r[t] = [np.concatenate([H.skel_r[t + 1][2 * c], H.skel_r[t + 1][2 * c + 1]])[ir[c].J]
                           for c in range(1 << t)]
            H.skel_c[t] = [np.concatenate([H.skel_c[t + 1][2 * c], H.skel_c[t + 1][2 * c + 1]])[ic[c].J]
                           for c in range(1 << t)]
        Yn, Zn, On, Pn = commit_up(t, Yl, Zl, Ol, Pl)
        # line 258 (non-symmetric): B_{s,b} = K(I~_s, J~_b) for every ordered far pair
        H.B[t] = {(int(s), int(b)): entry(H.skel_r[t][s], H.skel_c[t][b]) for (s, b) in part.far[t]}
    H.samples = d
    return H


def expanded(X, tree, t, c):
    """Nested basis (Eq.(2)) of cluster c at depth t from per-depth X."""
    Dl = tree.leaf_depth
    if t == Dl:
        return X[t][c]
    A1 = expanded(X, tree, t + 1, 2 * c)
    A2 = expanded(X, tree, t + 1, 2 * c + 1)
    k1 = A1.shape[1]
    return np.vstack([A1 @ X[t][c][:k1], A2 @ X[t][c][k1:]])


def matvec_nonsym(H: H2NonSym, x: np.ndarray) -> np.ndarray:
    """y = (D + U B V^T) x: upward pass with the column bases, couplings, downward pass with the
    row bases, dense near field."""
    tree, part, Dl = H.tree, H.part, H.tree.leaf_depth
    x = np.asarray(x, np.float64)
    vec = x.ndim == 1
    if vec:
        x = x[:, None]
    q = x.shape[1]
    rng_of = lambda t, c: np.arange(tree.begin[t][c], tree.end[t][c])
    y = np.zeros((tree.n, q))
    xh = {Dl: [H.Xc[Dl][c].T @ x[rng_of(Dl, c)] for c in range(1 << Dl)]}
    for t in range(Dl - 1, H.top - 1, -1):
        xh[t] = [H.Xc[t][c].T @ np.vstack([xh[t + 1][2 * c], xh[t + 1][2 * c + 1]]) for c in range(1 << t)]
    yh = {}
    for t in range(H.top, Dl + 1):
        yh[t] = [np.zeros((H.rank_r[t][c], q)) for c in range(1 << t)]
        for (s, b) in part.far[t]:
            yh[t][s] = yh[t][s] + H.B[t][(int(s), int(b))] @ xh[t][int(b)]
    for t in range(H.top, Dl):
        for c in range(1 << t):
            z = H.Xr[t][c] @ yh[t][c]
            k1 = H.rank_r[t + 1][2 * c]
            yh[t + 1][2 * c] = yh[t + 1][2 * c] + z[:k1]
            yh[t + 1][2 * c + 1] = yh[t + 1][2 * c + 1] + z[k1:]
    for c in range(1 << Dl):
        y[rng_of(Dl, c)] += H.Xr[Dl][c] @ yh[Dl][c]
    for (s, b) in part.near:
        y[rng_of(Dl, s)] += H.D[(int(s), int(b))] @ x[rng_of(Dl, b)]
    return y[:, 0] if vec else y


def to_dense_nonsym(H: H2NonSym) -> np.ndarray:
    tree, part, Dl = H.tree, H.part, H.tree.leaf_depth
    K = np.zeros((tree.n, tree.n))
    sl = lambda t, c: slice(tree.begin[t][c], tree.end[t][c])
    for (s, b) in part.near:
        K[sl(Dl, s), sl(Dl, b)] = H.D[(int(s), int(b))]
    for t in range(H.top, Dl + 1):
        for (s, b) in part.far[t]:
            K[sl(t, s), sl(t, b)] = (expanded(H.Xr, tree, t, int(s)) @ H.B[t][(int(s), int(b))]
                                     @ expanded(H.Xc, tree, t, int(b)).T)
    return K
