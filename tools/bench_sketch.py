"""Microbenchmark of the int8 tensor-core dense sketch: pass width (H2_TC_WIDE) x producer warps
(H2_TC_NPW).  Usage: python tools/bench_sketch.py [n] [ncols]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_16759_b200 as g
from synth import uniform_points
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
nc = int(sys.argv[2]) if len(sys.argv) > 2 else 128
X = uniform_points(n, 3, 0)
T = g.Tree(X, 64)
Om = g.omega(n, nc)
ref = None
for wide, npw, jc in (("1", "16", "128"), ("1", "8", "128"), ("1", "16", "64"), ("0", "16", "64")):
    if True:
        os.environ["H2_TC_WIDE"], os.environ["H2_TC_NPW"], os.environ["H2_TC_JC"] = wide, npw, jc
        y = g.dense_sketch(T, Om, omega_quarters=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(3):
            y = g.dense_sketch(T, Om, omega_quarters=True)
        e1.record(); e1.synchronize()
        ms = e0.elapsed_time(e1) / 3
        if ref is None:
            ref = y.clone()
        same = torch.equal(y, ref)
        print(f"wide={wide} npw={npw} jc={jc}: {ms:8.2f} ms for {nc} columns  {n*n/ms/1e9:7.2f} G kernel entries/s "
              f"(per evaluation)  bitwise-equal={same}", flush=True)
