"""One int8 tensor-core sketch pass for ncu: python tools/ncu_sketch.py [n] [ncols]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_2506_16759_b200 as g
from synth import uniform_points
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
nc = int(sys.argv[2]) if len(sys.argv) > 2 else 128
T = g.Tree(uniform_points(n, 3, 0), 64)
Om = g.omega(n, nc)
for _ in range(2):
    y = g.dense_sketch(T, Om, omega_quarters=True)
torch.cuda.synchronize()
