"""Debug driver for the sharded build on one GPU: python tools/debug_dist.py WORLD N
(spawns WORLD processes on cuda:0 with gloo; each writes gpurun_out/dist_rank<r>.log)."""
import datetime
import os
import sys

import torch
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def worker(rank, world, n):
    sys.path.insert(0, ROOT)
    log = open(os.path.join(ROOT, "gpurun_out", f"dist_rank{rank}.log"), "w", buffering=1)
    sys.stdout = sys.stderr = log
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = "29611"
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=60))
    import numpy as np
    import paper_2506_16759_b200 as g
    from paper_2506_16759_b200.dist import Comm
    from synth import uniform_points
    X = uniform_points(n, 3, 0)
    T = g.Tree(X, 64)
    print("tree", T.n, T.leaf_depth, T.top_depth, flush=True)
    comm = Comm()
    orig = comm._cb
    H = g.build(T, ("exp", 0.2), 1e-6, comm=comm)
    print("built", H.samples, comm.calls, comm.bytes, flush=True)
    H.allgather(comm)
    print("gathered", flush=True)
    H1 = g.build(T, ("exp", 0.2), 1e-6)
    for t in range(H.top_depth, T.leaf_depth + 1):
        print(t, np.array_equal(H.rank(t), H1.rank(t)),
              np.array_equal(H._export(g._lib.H2_X_BASIS, t), H1._export(g._lib.H2_X_BASIS, t)),
              np.array_equal(H._export(g._lib.H2_X_B, t), H1._export(g._lib.H2_X_B, t)), flush=True)
    print("D", np.array_equal(H._export(g._lib.H2_X_D), H1._export(g._lib.H2_X_D)), flush=True)
    for t in range(H.top_depth, T.leaf_depth + 1):
        a, b = H._export(g._lib.H2_X_SKEL, t), H1._export(g._lib.H2_X_SKEL, t)
        bad = np.nonzero(a != b)[0]
        print("skel", t, len(a), len(bad), bad[:5], a[bad[:5]], b[bad[:5]], flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    world, n = int(sys.argv[1]), int(sys.argv[2])
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    mp.spawn(worker, args=(world, n), nprocs=world, join=True)
