"""One-off run of a BASELINE workload at full size on one GPU (no oracle): build time per phase,
samples, ranks, memory, and the dense-probe error ||H X - K X||_F / ||K X||_F (16 probes, the
products K X computed by the GPU dense-sketch kernel).

  python tools/run_config.py cov3d_2m [--reps 1] [--s 0.1]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2506_16759_b200 as g
from synth import WORKLOADS

p = argparse.ArgumentParser()
p.add_argument("workload")
p.add_argument("--reps", type=int, default=1)
p.add_argument("--s", type=float, default=None, help="tol_safety (default: the library's, R31)")
p.add_argument("--s-update", type=float, default=None, help="tol_safety of the update build (configs[4]); default --s")
p.add_argument("--d-blk", type=int, default=32)
p.add_argument("--probes", type=int, default=16)
p.add_argument("--p-os", type=int, default=None, help="oversampling margin of the convergence test (R12); "
               "default: the workload's (configs[4]: 32), else 10")
p.add_argument("--bootstrap", type=float, default=None,
               help="S8(f) NEXT #1: build an H^2 of K at this tighter tol (dense sketch, timed separately), "
                    "then the timed build at the workload tol with its O(N) H^2-matvec sketch")
p.add_argument("--nonsym", type=float, default=None,
               help="S8(f) NEXT #3 (dense workloads): operator exp(-r/l)(1 + v (x_0 - y_0)) with this v, "
                    "built with h2_build_nonsym")
p.add_argument("--uvt", action="store_true", help="configs[4] with M = A_H + U V^T (V != U, h2_build_nonsym)")
p.add_argument("--eps-decay", type=float, default=None, help="R31 level schedule eps_t = eps * decay^(Dl-t) (default: the library's)")
a = p.parse_args()
w = dict(WORKLOADS[a.workload])
X = w["points"]()
n = X.shape[0]
kern = (w["kernel"], w["param"])
t0 = time.perf_counter()
T = g.Tree(X, w["leaf"], 0.7)
t_tree = time.perf_counter() - t0
out = {"workload": a.workload, "eps_decay": a.eps_decay, "n": n, "leaf": w["leaf"], "tol": w["tol"], "tree_s": t_tree,
       "leaf_depth": T.leaf_depth, "top_depth": T.top_depth, "near_nnz": T.near_nnz, "far_nnz": T.far_nnz_total,
       "csp": T.csp}
times = []
update = None
if "update_rank" in w:      # configs[4]: base H^2 of A (untimed setup, like PAPER.md L479), then M = A_H + U U^T
    from synth import lowrank_factor
    t0 = time.perf_counter()
    Hbase = g.build(T, kern, w["tol"], d_init=a.d_blk, d_blk=a.d_blk, tol_safety=a.s, eps_decay=a.eps_decay)
    torch.cuda.synchronize()
    out["base_build_s"] = time.perf_counter() - t0
    out["base_samples"] = Hbase.samples
    U = torch.from_numpy(lowrank_factor(n, w["update_rank"])).cuda()
    update = (Hbase, U)
    if a.uvt:
        update = (Hbase, U, torch.from_numpy(lowrank_factor(n, w["update_rank"], seed=4)).cuda())
        out["update"] = "U V^T (nonsym)"
h2sk = None
dense = None
if w.get("dense"):   # NEXT #4: materialise the operator in tree order (row blocks: no n x n temporaries)
    Xt = torch.from_numpy(X[T.perm]).cuda()
    dense = torch.empty((n, n), dtype=torch.float64, device="cuda")
    for r0 in range(0, n, 4096):
        dense[r0:r0 + 4096] = torch.exp(-torch.cdist(Xt[r0:r0 + 4096], Xt) / w["param"])
        if a.nonsym is not None:
            dense[r0:r0 + 4096] *= 1 + a.nonsym * (Xt[r0:r0 + 4096, :1] - Xt[:, 0][None, :])
    if a.nonsym is not None:
        out["nonsym_v"] = a.nonsym
    out["dense_operator_GB"] = dense.numel() * 8 / 1e9
if a.bootstrap is not None:
    t0 = time.perf_counter()
    h2sk = g.build(T, kern, a.bootstrap, d_init=a.d_blk, d_blk=a.d_blk, tol_safety=a.s, d_max=1024)
    torch.cuda.synchronize()
    out["bootstrap_tol"] = a.bootstrap
    out["bootstrap_build_s"] = time.perf_counter() - t0
    out["bootstrap_samples"] = h2sk.samples
for r in range(a.reps):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    H = g.build(T, kern, w["tol"], d_init=a.d_blk, d_blk=a.d_blk, p_os=a.p_os if a.p_os is not None else w.get("p_os", 10),
                tol_safety=a.s if (update is None or a.s_update is None) else a.s_update, update=update, h2_sketch=h2sk, dense=dense,
                d_max=w.get("d_max", 512), nonsym=a.nonsym is not None or a.uvt, eps_decay=a.eps_decay)
    e1.record()
    e1.synchronize()
    times.append(e0.elapsed_time(e1) / 1e3)
    if r < a.reps - 1:
        del H
st = H.stats
out.update({"build_s": times, "samples": st["samples"], "phase_ms": st["t_phase_ms"], "rounds": st["rounds"],
            "ranks": {t: [st["rank_min"][t], st["rank_max"][t], round(st["rank_mean"][t], 1)] for t in st["rank_min"]},
            **({"col_rank_mean": {t: round(float(H.rank(t, 1).mean()), 1)
                                  for t in range(H.top_depth, T.leaf_depth + 1)}} if H.nonsym else {}),
            "entries_D": st["entries_D"], "entries_B": st["entries_B"], "matrix_GB": H.device_bytes() / 1e9,
            "peak_mem_GB": torch.cuda.max_memory_allocated() / 1e9, "launches": st["launches"]})
from paper_2506_16759_b200._lib import lib as _lib  # noqa: E402
out["cache_GB_before_trim"] = _lib.h2_cache_bytes() / 1e9
_lib.h2_cache_trim()
Xp = torch.from_numpy(np.random.default_rng(2).standard_normal((n, a.probes))).cuda()
t0 = time.perf_counter()
if dense is not None:
    KX = dense @ Xp
elif update is not None:      # M X = A_H X + U (U^T X): the operator the update build compresses
    KX = update[0].matvec(Xp) + update[1] @ (update[-1].T @ Xp)
else:
    KX = g.dense_sketch(T, Xp, kern)
HX = H.matvec(Xp)
torch.cuda.synchronize()
out["probe_error"] = float(torch.linalg.norm(HX - KX) / torch.linalg.norm(KX))
out["probe_s"] = time.perf_counter() - t0
free, total = torch.cuda.mem_get_info()
out["device_free_GB_after"] = free / 1e9
print(json.dumps(out))
