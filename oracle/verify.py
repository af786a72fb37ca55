"""A-posteriori check of a constructed H^2 ("the error is
estimated with the sampler"; R30).  TEST INFRASTRUCTURE: imported only by tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline leg.

  e = ||H Om_h - S(Om_h)||_F / ||S(Om_h)||_F   over q held-out stream columns Om_h;
  while e > tol (at most `retries` times): s <- s / 3 and the construction is redone.

The paper's own error measure ("a few iterations of the power method to
approximate the 2-norm of the difference between the constructed hierarchical matrix and the
provided sampler"):  ||H - K_blk||_2 / ||K_blk||_2, each 2-norm by
power iteration on the (symmetric) operator, x <- A x / ||A x||, estimate ||A x|| for unit x.
"""
from dataclasses import replace
import numpy as np

from . import h2


def a_posteriori_error(matvec, sampler, Om_h):
    Yh = sampler(Om_h)
    return float(np.linalg.norm(matvec(Om_h) - Yh) / np.linalg.norm(Yh))


def build_verified(tree, part, sampler, entry, omega, omega_h, tol, opts: h2.BuildOpts = None, retries=2):
    """Returns (H, e, rebuilds, s_used)."""
    opts = opts or h2.BuildOpts()
    s = opts.tol_safety
    for r in range(retries + 1):
        H = h2.build(tree, part, sampler, entry, omega, tol, replace(opts, tol_safety=s))
        e = a_posteriori_error(lambda X: h2.matvec(H, X), sampler, omega_h)
        if not e > tol or r == retries:
            return H, e, r, s
        s /= 3


def power_2norm(apply, x0, iters):
    """||A||_2 of a symmetric operator by `iters` power iterations from x0:
    x = x0 / ||x0||; repeat: y = A x, nu = ||y||, x = y / nu.  Returns the last nu (<= ||A||_2)."""
    x = np.asarray(x0, dtype=np.float64).reshape(-1)
    x = x / np.linalg.norm(x)
    nu = 0.0
    for _ in range(iters):
        y = apply(x)
        nu = float(np.linalg.norm(y))
        if nu == 0.0:
            return 0.0
        x = y / nu
    return nu


def power_error(matvec, sampler, x0, iters=10):
    """(||H - K_blk||_2 / ||K_blk||_2, ||H - K_blk||_2, ||K_blk||_2) by power iterations from the
    same start vector x0; matvec / sampler act on (n,) vectors."""
    e = power_2norm(lambda x: matvec(x) - sampler(x), x0, iters)
    k = power_2norm(sampler, x0, iters)
    return (e / k if k > 0 else e), e, k
