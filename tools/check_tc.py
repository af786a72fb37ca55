"""Tensor-core sketch (int8 tcgen05, omega_quarters) vs the DMMA sketch: max relative difference
for several column counts (32-column and 64-column passes, ragged last pass) and the time of one
32-column and one 64-column pass.

  python tools/check_tc.py [n ...]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_16759_b200 as g
from synth import uniform_points


def timed(T, O, reps=2):
    g.dense_sketch(T, O, omega_quarters=True); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        g.dense_sketch(T, O, omega_quarters=True)
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / reps


for n in [int(a) for a in sys.argv[1:]] or [1000, 5000]:
    X = uniform_points(n, 3, 0)
    T = g.Tree(X, 64)
    Om = g.omega(n, 100)
    errs = []
    for nc in (32, 45, 64, 100):
        O = Om[:, :nc].contiguous()
        os.environ["H2_SK_TC"] = "0"
        ref = g.dense_sketch(T, O, omega_quarters=True)
        os.environ["H2_SK_TC"] = "1"
        y = g.dense_sketch(T, O, omega_quarters=True)
        torch.cuda.synchronize()
        errs.append(f"{nc}:{((y - ref).abs().max() / ref.abs().max()).item():.1e}")
    ts = {}
    for mode in ("0", "1"):
        os.environ["H2_SK_TC"] = mode
        ts[mode, 32] = timed(T, Om[:, :32].contiguous())
        ts[mode, 64] = timed(T, Om[:, :64].contiguous())
    print(f"n={n}: TC vs DMMA max rel diff {' '.join(errs)}; DMMA 32/64 cols {ts['0', 32]:.2f}/{ts['0', 64]:.2f} ms,"
          f" TC {ts['1', 32]:.2f}/{ts['1', 64]:.2f} ms", flush=True)
