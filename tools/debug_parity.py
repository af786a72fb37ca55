import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2506_16759_b200 as g
from synth import uniform_points
from gpu_helpers import oracle_build
for adaptive in (False, True):
    X = uniform_points(1024, 2, 0)
    opts = dict(adaptive=adaptive) if adaptive else dict(adaptive=False, d_init=64)
    Ho, op = oracle_build(X, "exp", 0.2, 32, 1e-6, **opts)
    T = g.Tree(X, 32)
    H = g.build(T, ("exp", 0.2), 1e-6, **opts)
    print("adaptive", adaptive, "samples", H.samples, Ho.samples, "eps", H.stats["eps"], Ho.eps)
    for t in range(T.leaf_depth, H.top_depth - 1, -1):
        rg = H.rank(t); sg = H.skel(t); Xg = H.basis(t); cg = H.cert(t)
        for c in range(1 << t):
            o = Ho.ids[t][c]
            same = rg[c] == o.k and np.array_equal(sg[c], Ho.skel[t][c])
            dx = np.abs(Xg[c] - Ho.X[t][c]).max() if same and Xg[c].size else -1
            if not same or dx > 1e-10:
                print(f" t{t} c{c} k {rg[c]}/{o.k} same {same} dX {dx:.2e} maxX {np.abs(Ho.X[t][c]).max() if Ho.X[t][c].size else 0:.2e} gap {o.min_gap:.2e} marg {o.stop_margin:.2e} gpu-cert {cg[c]}")
                if not same:
                    print("   gpu J", sg[c][:12], "\n   ora J", Ho.skel[t][c][:12])
