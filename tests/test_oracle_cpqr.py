"""Pins for oracle/cpqr.py (§II-B Eq.(3); readings R12-R15)."""
import numpy as np
import pytest
import scipy.linalg as sla
from oracle.cpqr import cpqr, row_id, back_substitute


def graded(d, m, seed, decay=0.7):
    """Random matrix with well separated column scales (no pivot near-ties)."""
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((d, m)) * (decay ** np.arange(m))[rng.permutation(m)]
    return A


@pytest.mark.parametrize("d,m,seed", [(40, 25, 0), (16, 30, 1), (64, 64, 2), (8, 8, 3)])
def test_pivots_match_lapack_dgeqp3(d, m, seed):
    A = graded(d, m, seed)
    k, perm, R, rdiag, gap, _ = cpqr(A, 0.0)
    Q2, R2, P2 = sla.qr(A, pivoting=True, mode="economic")
    kk = min(d, m)
    assert k == kk
    assert np.array_equal(perm[:kk], P2[:kk])
    assert np.allclose(rdiag, np.abs(np.diag(R2))[:kk], rtol=1e-12, atol=0)
    assert np.allclose(np.abs(R[:, :]), np.abs(R2[:kk, :]), rtol=1e-10, atol=1e-13)


def test_rdiag_nonincreasing_and_full_reconstruction():
    A = np.random.default_rng(5).standard_normal((20, 12))
    idd = row_id(A.T, 0.0)
    assert np.all(np.diff(idd.rdiag) <= 1e-12 * idd.rdiag[0])
    # full rank: Y = X Y(J,:) exactly (to roundoff)
    Y = A.T
    assert np.linalg.norm(Y - idd.X @ Y[idd.J]) <= 1e-13 * np.linalg.norm(Y)


def test_special_matrices():
    assert cpqr(np.zeros((8, 8)), 1e-12)[0] == 0
    k, perm, R, rdiag, _, _ = cpqr(np.eye(8), 1e-12)
    assert k == 8 and np.allclose(rdiag, 1.0)
    u = np.arange(1.0, 11.0)
    v = np.linspace(-1, 2, 7)
    idd = row_id(np.outer(u, v), 1e-10)
    assert idd.k == 1 and idd.J[0] == 9        # largest-norm row is the last one
    assert np.allclose(idd.X @ np.outer(u, v)[idd.J], np.outer(u, v), atol=1e-13)


@pytest.mark.parametrize("seed", range(20))
def test_truncated_residual_bound_and_identity_rows(seed):
    # ||Y - X Y(J,:)||_F = ||R3||_F <= sqrt(m-k) eps (every remaining column norm <= eps)
    rng = np.random.default_rng(100 + seed)
    m, d = 20, 12
    U, _ = np.linalg.qr(rng.standard_normal((m, m)))
    V, _ = np.linalg.qr(rng.standard_normal((d, d)))
    s = 10.0 ** (-np.arange(d) * 0.8)
    Y = U[:, :d] @ np.diag(s) @ V.T
    eps = 1e-5
    idd = row_id(Y, eps)
    res = np.linalg.norm(Y - idd.X @ Y[idd.J])
    assert res <= np.sqrt(m - idd.k) * eps * (1 + 1e-10)
    assert np.array_equal(idd.X[idd.J], np.eye(idd.k))               # identity rows, bitwise
    # rank never exceeds the number of singular values above eps / sqrt(...) bound of CPQR
    sv = np.linalg.svd(Y, compute_uv=False)
    assert idd.k >= np.sum(sv > np.sqrt(m * d) * eps) and idd.k <= np.sum(sv > eps / np.sqrt(m)) + 1


def test_back_substitution():
    rng = np.random.default_rng(0)
    R1 = np.triu(rng.standard_normal((6, 6))) + 4 * np.eye(6)
    R2 = rng.standard_normal((6, 3))
    T = back_substitute(R1, R2)
    assert np.allclose(R1 @ T, R2, atol=1e-13)
    assert np.allclose(T, sla.solve_triangular(R1, R2), atol=1e-13)
