import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2506_16759_b200 as g
from synth import uniform_points
for n in [int(a) for a in sys.argv[1:]] or [1000, 5000]:
    X = uniform_points(n, 3, 0)
    T = g.Tree(X, 64)
    Om = g.omega(n, 45)
    os.environ["H2_SK_TC"] = "0"
    ref = g.dense_sketch(T, Om, omega_quarters=True)
    os.environ["H2_SK_TC"] = "1"
    y = g.dense_sketch(T, Om, omega_quarters=True)
    torch.cuda.synchronize()
    err = ((y - ref).abs().max() / ref.abs().max()).item()
    ts = {}
    for mode in ("0", "1"):
        os.environ["H2_SK_TC"] = mode
        O32 = Om[:, :32].contiguous()
        g.dense_sketch(T, O32, omega_quarters=True); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(2):
            g.dense_sketch(T, O32, omega_quarters=True)
        e1.record(); e1.synchronize()
        ts[mode] = e0.elapsed_time(e1) / 2
    print(f"n={n}: max rel diff TC vs DMMA {err:.3e}; 32 cols: DMMA {ts['0']:.2f} ms, TC {ts['1']:.2f} ms", flush=True)
