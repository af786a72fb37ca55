"""A/B timing of the dense tensor-core sketch pass under environment switches (one subprocess per
variant: the switches are read once per process).
  python tools/ab_sketch.py N NCOL 'H2_TC_HINT=0' 'H2_TC_HINT=1000' ..."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys
sys.path.insert(0, os.environ["ROOT"])
import torch, paper_2506_16759_b200 as g
from synth import uniform_points, grid_points
n, nc = int(sys.argv[1]), int(sys.argv[2])
kind = os.environ.get("AB_KIND", "exp")
if kind == "exp":
    X, kern = uniform_points(n, 3, 0), ("exp", 0.2)
else:   # IE grid (BASELINE configs[3] shape): 2:2:1 box
    m = int(round((n / 4) ** (1 / 3)))
    X, kern = grid_points((2 * m, 2 * m, m), 1.0 / (2 * m)), ("helmholtz", 3.0)
    n = X.shape[0]
T = g.Tree(X, 64)
Om = g.omega(n, nc)
y = g.dense_sketch(T, Om, kern, omega_quarters=True)
torch.cuda.synchronize()
ms = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); y2 = g.dense_sketch(T, Om, kern, omega_quarters=True); e1.record(); e1.synchronize()
    ms.append(e0.elapsed_time(e1))
print(f"{min(ms):8.2f} ms  (runs {', '.join(f'{m:.2f}' for m in ms)})  bitwise-equal {bool(torch.equal(y, y2))}  |y| {float(y.norm()):.12e}")
'''

if __name__ == "__main__":
    n, nc = sys.argv[1], sys.argv[2]
    for spec in sys.argv[3:]:
        env = dict(os.environ, ROOT=ROOT)
        for kv in spec.split():
            k, v = kv.split("=")
            env[k] = v
        out = subprocess.run([sys.executable, "-c", CHILD, n, nc], env=env, capture_output=True, text=True)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-600:]
        print(f"{spec:40s} {line}", flush=True)
