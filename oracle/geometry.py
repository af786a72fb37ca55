"""Cluster tree, admissibility Eq.(1) and dual-tree traversal (§II-A).  TEST INFRA.

Readings:
  R1  Dist(s,t) = Euclidean distance between bounding-box CENTRES (default, "center");
      "box" = minimum distance between the two axis-aligned boxes (PAPER.md L122 is silent).
  R2  D(tau) = diagonal length of the axis-aligned bounding box of tau's points.
  R3  adm(s,t) = [s != t] and (D(s)+D(t))*0.5 <= eta*Dist(s,t)   (Eq.(1)).
  R4  KD-tree (L447 "KD-tree with a leaf size of 64-256"): complete binary tree, all leaves
      at depth Dl = min{D : ceil(n / 2^D) <= leaf_size}; split the longest bbox axis (ties ->
      lowest axis) at the median of the stable order (coordinate, original index); the lower
      half gets ceil(m/2) points.
  R6  N_tau = leaf-level clusters b with (tau, b) an inadmissible leaf pair (includes tau);
      F_tau (depth t) = clusters b at depth t with (tau, b) admissible and parents inadmissible.
Arithmetic is written with explicit left-to-right sums so the result does not depend on
numpy reduction order.
"""
from dataclasses import dataclass, field
import numpy as np


@dataclass
class ClusterTree:
    n: int
    dim: int
    leaf_size: int
    leaf_depth: int                 # Dl; depth 0 = root; paper level l = Dl - depth + 1
    perm: np.ndarray                # tree index -> original index (int64)
    begin: list                     # per depth: int64 array (2^t,)
    end: list
    lo: list                        # per depth: (2^t, dim) float64
    hi: list

    @property
    def nlevels(self):
        return self.leaf_depth + 1

    def size(self, t, c):
        return int(self.end[t][c] - self.begin[t][c])


@dataclass
class Partition:
    eta: float
    dist_rule: str
    near: np.ndarray                # (nnz, 2) ordered pairs (s, b) at leaf depth, sorted
    far: list = field(default_factory=list)   # per depth: (nnz_t, 2) ordered pairs, sorted

    def near_of(self, s):
        return self.near[self.near[:, 0] == s, 1]

    def far_of(self, t, s):
        f = self.far[t]
        return f[f[:, 0] == s, 1]

    def top_depth(self):
        """Coarsest depth holding an admissible pair (None if there is none)."""
        for t, f in enumerate(self.far):
            if len(f):
                return t
        return None


def leaf_depth_for(n: int, leaf_size: int) -> int:
    d = 0
    while -(-n // (1 << d)) > leaf_size:
        d += 1
    return d


def build_cluster_tree(points: np.ndarray, leaf_size: int) -> ClusterTree:
    """KD-tree per reading R4 (PAPER.md L121 'hierarchically clustering the indices', L447)."""
    X = np.asarray(points, dtype=np.float64)
    if X.ndim != 2 or X.shape[0] < 1 or not np.all(np.isfinite(X)):
        raise ValueError("build_cluster_tree: need finite n x dim points, n >= 1")
    if leaf_size < 2:
        raise ValueError("build_cluster_tree: leaf_size >= 2")
    n, dim = X.shape
    Dl = leaf_depth_for(n, leaf_size)
    perm = np.arange(n, dtype=np.int64)
    begin = [np.array([0], np.int64)]
    end = [np.array([n], np.int64)]
    for t in range(Dl):
        nb, ne = [], []
        for b, e in zip(begin[t], end[t]):
            sub = perm[b:e]
            pts = X[sub]
            ext = pts.max(axis=0) - pts.min(axis=0)
            axis = int(np.argmax(ext))          # first maximum = lowest axis on ties
            order = np.lexsort((sub, pts[:, axis]))  # primary: coordinate, secondary: original index
            perm[b:e] = sub[order]
            m = e - b
            left = (m + 1) // 2
            nb += [b, b + left]
            ne += [b + left, e]
        begin.append(np.array(nb, np.int64))
        end.append(np.array(ne, np.int64))
    Xt = X[perm]
    lo, hi = [], []
    for t in range(Dl + 1):
        l = np.empty((1 << t, dim))
        h = np.empty((1 << t, dim))
        for c in range(1 << t):
            p = Xt[begin[t][c]:end[t][c]]
            l[c] = p.min(axis=0)
            h[c] = p.max(axis=0)
        lo.append(l)
        hi.append(h)
    return ClusterTree(n, dim, leaf_size, Dl, perm, begin, end, lo, hi)


def diameter(lo, hi):
    """R2: bbox diagonal, sqrt(((e0*e0) + e1*e1) + e2*e2)."""
    acc = 0.0
    for d in range(len(lo)):
        e = hi[d] - lo[d]
        acc = acc + e * e
    return np.sqrt(acc)


def distance(lo_s, hi_s, lo_t, hi_t, rule="center"):
    """R1: centre distance (default) or minimum box-box distance."""
    acc = 0.0
    for d in range(len(lo_s)):
        if rule == "center":
            g = (lo_s[d] + hi_s[d]) * 0.5 - (lo_t[d] + hi_t[d]) * 0.5
        elif rule == "box":
            g = max(0.0, lo_t[d] - hi_s[d], lo_s[d] - hi_t[d])
        else:
            raise ValueError(rule)
        acc = acc + g * g
    return np.sqrt(acc)


def admissible(tree: ClusterTree, t: int, s: int, u: int, eta: float, rule="center") -> bool:
    """Eq.(1) with readings R1-R3."""
    if s == u:
        return False
    Ds = diameter(tree.lo[t][s], tree.hi[t][s])
    Du = diameter(tree.lo[t][u], tree.hi[t][u])
    dist = distance(tree.lo[t][s], tree.hi[t][s], tree.lo[t][u], tree.hi[t][u], rule)
    return bool((Ds + Du) * 0.5 <= eta * dist)


def build_partition(tree: ClusterTree, eta: float, rule: str = "center") -> Partition:
    """Dual-tree traversal from (root, root): admissible pair -> admissible
    leaf (F); inadmissible pair of leaves -> dense leaf (N); otherwise recurse on the four
    child pairs.  Pairs are processed depth by depth; outputs are sorted (row, col)."""
    Dl = tree.leaf_depth
    cur = [(0, 0)]
    far = []
    near = []
    for t in range(Dl + 1):
        f, nxt = [], []
        for (s, u) in cur:
            if admissible(tree, t, s, u, eta, rule):
                f.append((s, u))
            elif t == Dl:
                near.append((s, u))
            else:
                for a in (2 * s, 2 * s + 1):
                    for b in (2 * u, 2 * u + 1):
                        nxt.append((a, b))
        far.append(np.array(sorted(f), dtype=np.int64).reshape(-1, 2))
        cur = nxt
    return Partition(eta, rule, np.array(sorted(near), dtype=np.int64).reshape(-1, 2), far)
