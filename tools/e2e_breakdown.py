"""Host-side pieces of the end-to-end build (bench e2e): tree (async partition), build (incl. the
coordinate upload and the overlapped partition wait), the one-call result read."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2506_16759_b200 as g
from synth import uniform_points
X = uniform_points(1 << 18, 3, 0)
Xpin = torch.from_numpy(X).pin_memory()
torch.cuda.synchronize()
for rep in range(int(os.environ.get("REPS", 4))):
    t0 = time.perf_counter(); T = g.Tree(Xpin.numpy(), 64, 0.7, asynchronous=True); t1 = time.perf_counter()
    H = g.build(T, ("exp", 0.2), 1e-6); t2 = time.perf_counter()
    torch.cuda.synchronize(); t3 = time.perf_counter()
    rk, sk = H.ranks_and_skeletons(); t4 = time.perf_counter()
    print(f"tree {1e3*(t1-t0):.1f} ms  build call {1e3*(t2-t1):.1f} ms (device {H.stats['t_total_ms']:.1f}, "
          f"phases {sum(H.stats['t_phase_ms'].values()):.1f})  sync {1e3*(t3-t2):.1f}  d2h {1e3*(t4-t3):.1f}  "
          f"total {1e3*(t4-t0):.1f} ms", flush=True)
    del H, T
