"""Microbenchmark of the dense sketch: int8 tensor-core pass widths (H2_TC_WIDE) vs the FP64 DMMA
path (H2_SK_TC=0).  Usage: python tools/bench_sketch.py [n] [ncols] [exp|helmholtz]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2506_16759_b200 as g
from synth import uniform_points, grid_points
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
nc = int(sys.argv[2]) if len(sys.argv) > 2 else 128
kind = sys.argv[3] if len(sys.argv) > 3 else "exp"
if kind == "exp":
    X, kern = uniform_points(n, 3, 0), ("exp", 0.2)
else:   # IE grid (BASELINE configs[3] shape): 2:2:1 box, spacing h
    m = int(round((n / 4) ** (1 / 3)))
    X, kern = grid_points((2 * m, 2 * m, m), 1.0 / (2 * m)), ("helmholtz", 3.0)
    n = X.shape[0]
T = g.Tree(X, 64)
Om = g.omega(n, nc)
ref = None
for label, env in (("tc-128", {"H2_TC_WIDE": "1", "H2_SK_TC": "1"}), ("tc-64", {"H2_TC_WIDE": "0", "H2_SK_TC": "1"}),
                   ("dmma", {"H2_SK_TC": "0"})):
    os.environ.update(env)
    y = g.dense_sketch(T, Om, kern, omega_quarters=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    reps = 2
    for _ in range(reps):
        y = g.dense_sketch(T, Om, kern, omega_quarters=True)
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    if ref is None:
        ref = y.clone()
    dev = ((y - ref).abs().max() / ref.abs().max()).item()
    print(f"{kind} n={n} {label}: {ms:9.2f} ms for {nc} columns  {n*n/ms/1e9:7.3f} T kernel entries/s per pass-equiv "
          f"max rel dev vs tc-128 {dev:.1e}", flush=True)
