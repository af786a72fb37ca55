"""Table I of the paper (BASELINE.md rows "fixed sample / adaptive"): N = 2^18
3D covariance (exp, l = 0.2, uniform points) and IE (cos(3r)/r, 64^3 cell-centred grid), tol 1e-6,
leaf 256 / 128, fixed samples (d = leaf) vs adaptive (d_init = d_blk = 32).  As in the paper the
black-box sampler is an H^2 matvec (an H2Opus H^2 of K): here an H^2 of K built once at
tol 1e-8 with the dense sketch (untimed setup), then the timed construction uses the O(N)
H^2-matvec sketch (S§8(f) NEXT #1).  Reported: build time (CUDA events, median of 3 after a
warm-up), rank range, device memory of the result (GB), samples, and the relative error
against the TRUE K (16 dense probes; the paper reports it against its sampler's H^2).
--literal: the paper's own tolerance reading (eps_abs = tol * ||K||_2 estimate,
nu from 10 block power iterations with the sampler H^2; p_os = 0), and the relative 2-norm error
||H - K||_2 / ||K||_2 (20 power iterations on H_sampler - H) reported beside the probe error.
Usage: python tools/table1.py [cov|ie] [--literal] > out.json"""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2506_16759_b200 as g  # noqa: E402
from synth import uniform_points, grid_points  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "cov"
if which == "cov":
    X, kern = uniform_points(1 << 18, 3, 0), ("exp", 0.2)
else:
    X, kern = grid_points((64, 64, 64), 1.0 / 64), ("helmholtz", 3.0)
tol = 1e-6
literal = "--literal" in sys.argv
rows = []


def power_norm(apply, n, iters, seed=7):
    v = torch.from_numpy(np.random.default_rng(seed).standard_normal((n, 1))).cuda()
    lam = 0.0
    for _ in range(iters):
        v = v / torch.linalg.norm(v)
        w = apply(v)
        lam = float(torch.linalg.norm(w))
        v = w
    return lam

for leaf in (256, 128):
    T = g.Tree(X, leaf, 0.7)
    t0 = time.perf_counter()
    Hb = g.build(T, kern, 1e-8, d_max=1024)
    torch.cuda.synchronize()
    base_s = time.perf_counter() - t0
    Xp = torch.from_numpy(np.random.default_rng(2).standard_normal((T.n, 16))).cuda()
    KX = g.dense_sketch(T, Xp, kern)
    nu = power_norm(Hb.matvec, T.n, 10) if literal else 0.0
    for mode in ("fixed", "adaptive"):
        kw = dict(adaptive=False, d_init=leaf, d_max=max(leaf, 512)) if mode == "fixed" else dict(d_init=32, d_blk=32)
        if literal:
            kw.update(tol_rule="literal", norm=nu)
        times = []
        for r in range(4):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            H = g.build(T, kern, tol, h2_sketch=Hb, **kw)
            e1.record()
            e1.synchronize()
            if r:
                times.append(e0.elapsed_time(e1) / 1e3)
            if r < 3:
                del H
        st = H.stats
        err = float(torch.linalg.norm(H.matvec(Xp) - KX) / torch.linalg.norm(KX))
        err2 = power_norm(lambda v: Hb.matvec(v) - H.matvec(v), T.n, 20) / nu if literal else None
        rows.append({"problem": which, "tol_rule": "literal" if literal else "rms", "nu": nu, "rel_error_2norm": err2,
                     "mode": mode, "leaf": leaf, "build_s": float(np.median(times)),
                     "build_s_all": times, "rank_range": [min(st["rank_min"].values()), max(st["rank_max"].values())],
                     "memory_GB": H.device_bytes() / 1e9, "samples": st["samples"], "rel_error": err,
                     "phase_ms": st["t_phase_ms"], "base_build_s": base_s, "base_samples": Hb.samples})
        print(json.dumps(rows[-1]), flush=True)
        del H
    del Hb
