"""A-posteriori check of a constructed H^2 ("the error is
estimated with the sampler"; R30).  TEST INFRASTRUCTURE: imported only by tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline leg.

  e = ||H Om_h - S(Om_h)||_F / ||S(Om_h)||_F   over q held-out stream columns Om_h;
  while e > tol (at most `retries` times): s <- s / 3 and the construction is redone.
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
