"""Microbenchmark of the dense-sketch kernel variants (env knobs H2_SK_MB / H2_SK_SPLIT)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2506_16759_b200 as g
from synth import uniform_points
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
X = uniform_points(n, 3, 0)
T = g.Tree(X, 64)
Om = g.omega(n, 32)
ref = None
variants = sys.argv[2].split(",") if len(sys.argv) > 2 else [str(v) for v in range(7)]
splits = sys.argv[3].split(",") if len(sys.argv) > 3 else ["0"]
for mb in variants:
    for sp in splits:
        os.environ["H2_SK_VAR"], os.environ["H2_SK_SPLIT"] = mb, sp
        y = g.dense_sketch(T, Om)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(3):
            y = g.dense_sketch(T, Om)
        e1.record(); e1.synchronize()
        ms = e0.elapsed_time(e1) / 3
        if ref is None:
            ref = y.clone()
        dev = (y - ref).abs().max().item() / ref.abs().max().item()
        print(f"var={mb} split={sp}: {ms:8.2f} ms  {2*n*n*32/ms/1e9:6.2f} TFLOP/s contraction  "
              f"{n*n/ms/1e9:6.2f} Gentries/ms  rel-dev {dev:.1e}", flush=True)
