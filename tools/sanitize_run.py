"""Small builds that exercise every libh2 kernel family for compute-sanitizer:
int8 tensor-core sketch (sketch_tc: mbarrier / tcgen05 pipeline, 160- and 64-column passes, the
j-split combine), D/B generation, BSR (32- and 64-column variants), the three CPQR variants, the
ID and shrink/projection kernels, the exact-order kernels and the H^2 matvec.
  compute-sanitizer --tool {memcheck,racecheck,synccheck} python tools/sanitize_run.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import paper_2506_16759_b200 as g
from synth import uniform_points, grid_points

X = uniform_points(5000, 3, 0)
T = g.Tree(X, 64)
for variant in ("warp", "smem", "global", "cluster"):
    os.environ["H2_CQ_VARIANT"] = variant
    H = g.build(T, ("exp", 0.2), 1e-6, d_init=16, d_blk=16)
    print(variant, "samples", H.samples, "cpqr_variants", H.stats["cpqr_variants"], flush=True)
os.environ.pop("H2_CQ_VARIANT")
x = torch.randn(T.n, 4, dtype=torch.float64, device="cuda")
y = H.matvec(x)
Om = g.omega(T.n, 160)
Y = g.dense_sketch(T, Om, ("exp", 0.2), omega_quarters=True)      # 160-column packed pass
Y2 = g.dense_sketch(T, Om[:, :45].contiguous(), ("exp", 0.2), omega_quarters=True)   # 64-column pass
Tg = g.Tree(grid_points((12, 12, 12), 1 / 12), 64)
Hh = g.build(Tg, ("helmholtz", 3.0), 1e-4)                        # 7-slice Helmholtz pass
He = g.build(g.Tree(uniform_points(1500, 3, 1), 64), ("rational", 0.3), 1e-6, exact_order=1)
Ta = g.Tree(uniform_points(9000, 3, 2), 64, asynchronous=True)     # GPU KD ordering
Ha = g.build(Ta, ("exp", 0.2), 1e-6)
torch.cuda.synchronize()
print("ok", float(y.norm()), float(Y.norm()), float(Y2.norm()), Hh.samples, He.samples, Ha.samples, flush=True)
