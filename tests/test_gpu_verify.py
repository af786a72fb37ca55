"""O10 a-posteriori check (h2_verify / opts.verify_probes, R30) against oracle/verify.py."""
import numpy as np
import pytest
import torch

from oracle import geometry, kernels, h2 as oh2, rng, verify
from synth import uniform_points
import paper_2506_16759_b200 as g

pytestmark = pytest.mark.gpu


def _oracle(X, s, retries):
    tree = geometry.build_cluster_tree(X, 64)
    part = geometry.build_partition(tree, 0.7)
    op = kernels.KernelOperator("exp", 0.2, X[tree.perm])
    om = lambda c0, nc: rng.omega_block(1, 0, 0, tree.n, c0, nc)
    Oh = rng.omega_block(1, 2, 0, tree.n, 0, 8)
    return verify.build_verified(tree, part, op.sampler, op.entry, om, Oh, 1e-6, oh2.BuildOpts(tol_safety=s),
                                 retries=retries)


@pytest.mark.parametrize("s", [0.1, 30.0])
def test_verify_matches_oracle(s):
    X = uniform_points(2048, 3, 0)
    T = g.Tree(X, 64)
    Hg = g.build(T, ("exp", 0.2), 1e-6, tol_safety=s, verify_probes=8, verify_retries=6)
    Ho, e, r, s_used = _oracle(X, s, 6)
    st = Hg.stats
    assert st["verify_rebuilds"] == r
    assert st["tol_safety_used"] == s_used
    assert st["verify_error"] <= 1e-6 and e <= 1e-6
    assert abs(st["verify_error"] - e) <= 0.05 * e
    # the standalone call is the same computation
    assert Hg.verify(q=8) == st["verify_error"]


def test_verify_dense_operator_and_no_retry_when_off():
    X = uniform_points(3000, 3, 5)
    T = g.Tree(X, 64)
    Xt = torch.from_numpy(X[T.perm]).cuda()
    A = torch.exp(-torch.cdist(Xt, Xt) / 0.2)
    H = g.build(T, ("exp", 0.2), 1e-6, dense=A, tol_safety=30.0)
    assert H.stats["verify_rebuilds"] == 0 and H.stats["verify_error"] == 0.0
    e = H.verify(dense=A)
    P = g.omega(T.n, 8, seed=1, stream_id=2)
    ref = A @ P
    direct = (torch.linalg.norm(H.matvec(P) - ref) / torch.linalg.norm(ref)).item()
    assert abs(e - direct) <= 1e-6 * direct


@pytest.mark.parametrize("n,tol,s", [(3000, 1e-6, 0.04), (2048, 1e-4, 3.0)])
def test_power_method_error_matches_oracle_and_dense(n, tol, s):
    """The paper's error measure (h2_verify_2norm): ||H - K||_2 / ||K||_2 by power
    iterations.  Checked against oracle/verify.power_error run on the same operators (the CUDA
    H as a dense matrix, K by plain torch FP64 ops, the same start vector), and against the exact
    2-norms (the estimates are lower bounds that converge)."""
    X = uniform_points(n, 3, 8)
    T = g.Tree(X, 64)
    H = g.build(T, ("exp", 0.2), tol, tol_safety=s)
    r, e, k = H.verify_2norm(("exp", 0.2), iters=40, stream_id=4)
    Xt = torch.from_numpy(X[T.perm]).cuda()
    K = torch.exp(-torch.sqrt(((Xt[:, None, :] - Xt[None, :, :]) ** 2).sum(-1)) / 0.2)   # no expanded-square
    Hd = torch.cat([H.matvec(torch.eye(n, dtype=torch.float64, device="cuda")[:, c:c + 64].contiguous())
                    for c in range(0, n, 64)], dim=1)
    Kh, Hh = K.cpu().numpy(), Hd.cpu().numpy()
    x0 = g.omega(n, 1, seed=1, stream_id=4).cpu().numpy()[:, 0]
    ro, eo, ko = verify.power_error(lambda x: Hh @ x, lambda x: Kh @ x, x0, 40)
    assert abs(k - ko) <= 1e-10 * ko
    # ||H - K|| is ~1e-8 ||K||: H x - K x cancels, and the rounding of K x (DMMA sketch vs numpy)
    # moves the power iterates; the estimates agree to the iteration's own accuracy
    assert abs(e - eo) <= 1e-3 * eo
    ex_e = float(np.linalg.norm(Hh - Kh, 2))
    ex_k = float(np.linalg.norm(Kh, 2))
    assert e <= ex_e * (1 + 1e-8) and e >= 0.5 * ex_e
    assert k <= ex_k * (1 + 1e-12) and k >= (1 - 1e-10) * ex_k
    assert r <= 2 * tol
    # several start vectors side by side: each column the 1-vector iteration, the best kept
    r8, e8, k8 = H.verify_2norm(("exp", 0.2), iters=40, nvec=8, stream_id=4)
    assert e8 >= e * (1 - 1e-12) and e8 <= ex_e * (1 + 1e-8) and abs(k8 - ex_k) <= 1e-10 * ex_k
