"""One C2 build (BASELINE configs[1], N = 2^18) for launch lists: python tools/one_build.py [n]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2506_16759_b200 as g
from synth import uniform_points
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 18
T = g.Tree(uniform_points(n, 3, 0), 64, 0.7)
H = g.build(T, ("exp", 0.2), 1e-6)
torch.cuda.synchronize()
print("samples", H.samples, "cpqr ms", H.stats["t_phase_ms"]["cpqr"], "variants", H.stats["cpqr_variants"],
      "depth ms", {t: round(v, 2) for t, v in H.stats["t_depth_ms"].items()})
