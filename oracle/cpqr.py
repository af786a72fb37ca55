"""Column-pivoted QR and the row interpolative decomposition (§II-B, Eq.(3)).  TEST INFRA.

Row ID of Y (m x d) = column ID of A = Y^T (d x m):  A P = Q R, R = [R1 R2; 0 R3],
T = R1^{-1} R2, A ~= A(:, S) [I T]  (L171), so  Y ~= X Y(J, :) with X(J[i], :) = e_i and
X(Rhat[j], :) = T(:, j)^T  (L283: U = [T I]^T up to the permutation).

Readings:
  R12 convergence/truncation uses the same CPQR (L361 "QR ... smallest absolute value of the
      diagonal ... less than eps_abs").
  R13 truncation: stop at step i when the largest remaining column norm (= |R_ii| of the next
      pivot) is <= eps (L173 "discarding R3 when its norm becomes small enough").
  R14 pivot = largest residual 2-norm, RECOMPUTED from the updated trailing block each step
      (no downdating), ties -> lowest column index; Householder reflectors in the LAPACK dlarfg
      convention (beta = -sign(alpha) ||x||, sign(0) = +).
  R15 T = R1^{-1} R2 by back substitution, column by column, rows k-1 -> 0.
"""
from dataclasses import dataclass
import numpy as np


@dataclass
class RowID:
    k: int                 # rank
    J: np.ndarray          # skeleton rows, pivot order (int64, k)
    Rhat: np.ndarray       # redundant rows, pivot order (int64, m-k)
    T: np.ndarray          # k x (m-k) interpolation matrix
    X: np.ndarray          # m x k basis, Y ~= X @ Y[J]
    rdiag: np.ndarray      # |R_ii|, i < k
    min_gap: float         # smallest relative gap best/second-best pivot norm over accepted steps
    stop_margin: float     # |maxnorm - eps| / eps at the truncation decision(s) (inf if none)


def cpqr(A: np.ndarray, eps: float, kmax: int = None):
    """CPQR of A (d x m) with recomputed norms (R14) and threshold truncation (R13).

    Returns (k, perm, R (k x m upper trapezoid in pivoted order), rdiag, min_gap, stop_margin).
    """
    A = np.array(A, dtype=np.float64, copy=True)
    d, m = A.shape
    perm = np.arange(m, dtype=np.int64)
    kcap = min(d, m) if kmax is None else min(d, m, kmax)
    rdiag = []
    min_gap = np.inf
    stop_margin = np.inf
    k = 0
    for i in range(kcap):
        sub = A[i:, i:]
        norms = np.sqrt(np.einsum("ij,ij->j", sub, sub))   # recomputed residual column norms
        j = int(np.argmax(norms))                             # lowest index on ties
        best = norms[j]
        if eps > 0:
            stop_margin = min(stop_margin, abs(best - eps) / eps)
        if not best > eps:
            break
        if len(norms) > 1:
            second = np.max(np.delete(norms, j))
            min_gap = min(min_gap, (best - second) / best)
        p = i + j
        if p != i:
            A[:, [i, p]] = A[:, [p, i]]
            perm[[i, p]] = perm[[p, i]]
        # Householder reflector, LAPACK dlarfg convention
        x = A[i:, i].copy()
        alpha = x[0]
        xnorm = np.sqrt(np.dot(x[1:], x[1:])) if len(x) > 1 else 0.0
        if xnorm == 0.0:
            tau = 0.0
            beta = alpha
            v = np.zeros_like(x)
            v[0] = 1.0
        else:
            beta = -np.copysign(np.hypot(alpha, xnorm), alpha) if alpha != 0 else -np.hypot(alpha, xnorm)
            tau = (beta - alpha) / beta
            v = x / (alpha - beta)
            v[0] = 1.0
        A[i, i] = beta
        A[i + 1:, i] = 0.0
        if i + 1 < m and tau != 0.0:
            w = v @ A[i:, i + 1:]
            A[i:, i + 1:] -= tau * np.outer(v, w)
        rdiag.append(abs(beta))
        k = i + 1
    else:
        # loop ran to the cap: record the margin of the next (unused) pivot if one exists
        if k < min(d, m) and eps > 0:
            sub = A[k:, k:]
            nxt = np.sqrt(np.einsum("ij,ij->j", sub, sub)).max()
            stop_margin = min(stop_margin, abs(nxt - eps) / eps)
    return k, perm, np.triu(A[:k, :]), np.array(rdiag), min_gap, stop_margin


def back_substitute(R1: np.ndarray, R2: np.ndarray) -> np.ndarray:
    """T = R1^{-1} R2 (R15): for each column c, rows i = k-1 .. 0:
    T[i,c] = (R2[i,c] - sum_{j>i} R1[i,j] T[j,c]) / R1[i,i], sum in ascending j."""
    k = R1.shape[0]
    T = np.zeros_like(R2)
    for i in range(k - 1, -1, -1):
        s = R2[i, :].copy()
        for j in range(i + 1, k):
            s = s - R1[i, j] * T[j, :]
        T[i, :] = s / R1[i, i]
    return T


def row_id(Y: np.ndarray, eps: float, kmax: int = None) -> RowID:
    """Row ID of Y (m x d) via the column ID of Y^T."""
    Y = np.asarray(Y, dtype=np.float64)
    m = Y.shape[0]
    k, perm, R, rdiag, gap, margin = cpqr(Y.T, eps, kmax)
    J = perm[:k].copy()
    Rhat = perm[k:].copy()
    T = back_substitute(R[:, :k], R[:, k:]) if k > 0 else np.zeros((0, m - k))
    X = np.zeros((m, k))
    X[J, np.arange(k)] = 1.0
    if k > 0 and m > k:
        X[Rhat, :] = T.T
    return RowID(k, J, Rhat, T, X, rdiag, gap, margin)
