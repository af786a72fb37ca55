"""The paper's error measure (h2_verify_2norm) at the north-star size (BASELINE
configs[2], N = 2^21, exp(0.2), tol 1e-6, one B200): ||H - K||_2 / ||K||_2 by power iterations
(argv: iters nvec; the one-column FP64 DMMA dense sketch costs ~10 s per iteration at this N)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2506_16759_b200 as g
from synth import uniform_points

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 5
nvec = int(sys.argv[2]) if len(sys.argv) > 2 else 4
T = g.Tree(uniform_points(1 << 21, 3, 0), 64, 0.7)
H = g.build(T, ("exp", 0.2), 1e-6)
torch.cuda.synchronize()
t0 = time.perf_counter()
r, e, k = H.verify_2norm(("exp", 0.2), iters=iters, nvec=nvec)
print(json.dumps({"workload": "cov3d_2m", "n": T.n, "samples": H.samples, "build_s": H.stats["t_total_ms"] / 1e3,
                  "error_2norm": r, "abs_2norm": e, "k_2norm": k, "iters": iters, "nvec": nvec,
                  "verify_s": time.perf_counter() - t0}))
