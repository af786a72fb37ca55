"""Entry evaluation K(x, y) (§V-A).  TEST INFRA.

  exp:       K(x,y) = exp(-|x-y| / l)                 (Eq. cov; l = 0.2 in L431)
  helmholtz: K(x,y) = cos(k |x-y|) / |x-y|, x != y   (Eq. ie; k = 3 in L439)
             K(x,x) = 0                               (reading R20: the paper excludes x = y)
|x-y| = sqrt(((dx*dx) + dy*dy) + dz*dz) written left to right.
"""
import numpy as np


def pair_dist(X, Y):
    X = np.asarray(X, np.float64)
    Y = np.asarray(Y, np.float64)
    acc = np.zeros((X.shape[0], Y.shape[0]))
    for d in range(X.shape[1]):
        g = X[:, d][:, None] - Y[:, d][None, :]
        acc = acc + g * g
    return np.sqrt(acc)


def kernel_block(kind: str, param: float, X, Y):
    r = pair_dist(X, Y)
    if kind == "exp":
        return np.exp(-r / param)
    if kind == "helmholtz":
        out = np.zeros_like(r)
        nz = r != 0.0
        out[nz] = np.cos(param * r[nz]) / r[nz]
        return out
    raise ValueError(kind)


class KernelOperator:
    """The black-box pair (sampler, entry evaluator) of Algorithm 1's input
    for a kernel matrix on tree-ordered points: sampler(Omega) = K Omega (dense, row-blocked),
    entry(rows, cols) = K(I_rows, I_cols)."""

    def __init__(self, kind, param, points_tree_order, row_block=512):
        self.kind, self.param = kind, param
        self.X = np.asarray(points_tree_order, np.float64)
        self.n = self.X.shape[0]
        self.row_block = row_block

    def entry(self, rows, cols):
        return kernel_block(self.kind, self.param, self.X[rows], self.X[cols])

    def sketch_rows(self, Omega, rows):
        """Y(rows, :) = K(rows, :) Omega."""
        out = np.empty((len(rows), Omega.shape[1]))
        for a in range(0, len(rows), self.row_block):
            r = rows[a:a + self.row_block]
            out[a:a + len(r)] = kernel_block(self.kind, self.param, self.X[r], self.X) @ Omega
        return out

    def sampler(self, Omega):
        return self.sketch_rows(Omega, np.arange(self.n))

    def dense(self):
        return kernel_block(self.kind, self.param, self.X, self.X)
