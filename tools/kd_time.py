import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_2506_16759_b200 as g
from synth import uniform_points
X = uniform_points(1 << 18, 3, 0)
Xp = torch.from_numpy(X).pin_memory()
for _ in range(2):
    T = g.Tree(Xp.numpy(), 64, 0.7, asynchronous=True)
    T.perm
