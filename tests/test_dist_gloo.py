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


def _load_dist():
    import importlib.util
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("h2dist", os.path.join(root, "paper_2506_16759_b200", "dist.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _agv_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mod = _load_dist()
        # uneven segments, one empty, not in rank order of displacement, gaps between them
        counts = [5, 0, 9][:world]
        displs = [20, 3, 0][:world]
        buf = torch.full((40,), 255, dtype=torch.uint8)
        c, d = counts[rank], displs[rank]
        buf[d:d + c] = torch.arange(c, dtype=torch.uint8) + 10 * (rank + 1)
        mod.allgatherv_(buf, counts, displs)
        out_q.put((rank, buf.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_allgatherv_gloo(world):
    """The communicator primitive libh2 calls (h2_comm.allgatherv): in-place, per-rank byte
    segments, empty segments allowed; bytes outside the segments untouched."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_agv_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    counts, displs = [5, 0, 9][:world], [20, 3, 0][:world]
    want = [255] * 40
    for r in range(world):
        for i in range(counts[r]):
            want[displs[r] + i] = i + 10 * (r + 1)
    for r in range(world):
        assert res[r] == want


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_owned_ranges_partition_and_subtrees(world):
    """Cluster ownership of the sharded construction (S§8(e)): the ranges tile every depth, the
    library's h2_dist_range agrees with dist.owned_range, and -- for power-of-two world sizes at
    depths with at least `world` clusters (what h2_build_dist requires) -- the children of an
    owned cluster are owned by the same rank (subtree alignment: no cross-rank merge)."""
    import ctypes as C
    from paper_2506_16759_b200 import _lib
    mod = _load_dist()
    for t in range(0, 12):
        n = 1 << t
        prev = 0
        for r in range(world):
            b, e = mod.owned_range(n, r, world)
            lb, le = C.c_int64(), C.c_int64()
            assert _lib.lib.h2_dist_range(n, r, world, C.byref(lb), C.byref(le)) == 0
            assert (lb.value, le.value) == (b, e)
            assert b == prev and e >= b
            prev = e
            for c in range(b, e):
                assert c * world // n == r
                if t < 11 and world & (world - 1) == 0 and n >= world:
                    cb, ce = mod.owned_range(2 * n, r, world)
                    assert cb <= 2 * c and 2 * c + 1 < ce
        assert prev == n
