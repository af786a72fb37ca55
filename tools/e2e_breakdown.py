"""Host-side pieces of the end-to-end build (bench e2e): tree build, device upload, build, D2H."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2506_16759_b200 as g
from synth import uniform_points
X = uniform_points(1 << 18, 3, 0)
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter(); T = g.Tree(X, 64, 0.7); t1 = time.perf_counter()
    H = g.build(T, ("exp", 0.2), 1e-6); torch.cuda.synchronize(); t2 = time.perf_counter()
    for t in range(H.top_depth, T.leaf_depth + 1):
        H.rank(t); H.skel(t)
    t3 = time.perf_counter()
    print(f"tree {1e3*(t1-t0):.1f} ms  build(+upload) {1e3*(t2-t1):.1f} ms (device {H.stats['t_total_ms']:.1f})  d2h {1e3*(t3-t2):.1f} ms", flush=True)
    del H, T
