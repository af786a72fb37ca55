"""H^2 matvec timing (32 columns) for H^2 built at several tolerances: python tools/bench_matvec.py [n]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2506_16759_b200 as g
from synth import uniform_points
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
T = g.Tree(uniform_points(n, 3, 0), 64)
x = torch.from_numpy(np.random.default_rng(2).standard_normal((n, 32))).cuda()
for tol in (1e-6, 1e-8, 1e-10):
    H = g.build(T, ("exp", 0.2), tol, d_max=1024)
    if True:
        y = H.matvec(x); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(5):
            y = H.matvec(x)
        e1.record(); e1.synchronize()
        print(f"n={n} tol={tol:g} GB={H.device_bytes()/1e9:.1f} {e0.elapsed_time(e1)/5:.2f} ms per 32-column matvec", flush=True)
    del H
