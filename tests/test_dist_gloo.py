"""world_size-2 gloo test of the multi-GPU host logic (paper_2506_16759_b200.dist): row sharding
of the sketch and the all-gather reassembly, on CPU with a stand-in shard function."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, nc, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import importlib.util
        import sys
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        spec = importlib.util.spec_from_file_location("h2dist", os.path.join(root, "paper_2506_16759_b200", "dist.py"))
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        K = torch.from_numpy(np.random.default_rng(0).standard_normal((n, n)))
        om = torch.from_numpy(np.random.default_rng(1).standard_normal((n, nc)))
        calls = []

        def shard_fn(o, out, r0, r1):
            calls.append((r0, r1))
            out.copy_(K[r0:r1] @ o)

        sk = mod.ShardedSketch(n, shard_fn)
        y = torch.full((n, nc + 3), np.nan, dtype=torch.float64)[:, 1:1 + nc]   # strided destination
        sk(om, y, 0, 0, n)
        ok = torch.allclose(y, K @ om, rtol=0, atol=1e-12)
        out_q.put((rank, ok, calls, sk.bounds))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [101, 128])
def test_sharded_sketch_gloo_world2(n):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n, 7, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    bounds = res[0][3]
    assert bounds == [0, n // 2, n]
    for rank, ok, calls, _ in res:
        assert ok
        assert calls == [(bounds[rank], bounds[rank + 1])]
