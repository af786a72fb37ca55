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


def _a2a_worker(rank, world, port, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mod = _load_dist()
        # (1) the primitive: uneven, empty and gapped segments; bytes outside them untouched
        sc = [(3 * rank + 2 * r) % 5 for r in range(world)]          # rank -> r
        sd, o = [], 1
        for c in sc:
            sd.append(o)
            o += c + 2                                                  # gaps of 2
        send = torch.full((o + 3,), 200, dtype=torch.uint8)
        for r in range(world):
            send[sd[r]:sd[r] + sc[r]] = 10 * rank + r
        rc = [(3 * r + 2 * rank) % 5 for r in range(world)]            # what rank r sends me
        rd, o = [], 4
        for c in rc:
            rd.append(o)
            o += c + 1
        recv = torch.full((o + 2,), 255, dtype=torch.uint8)
        mod.alltoallv_(send, sc, sd, recv, rc, rd)
        # (2) the column-split sketch exchange of libh2 (Builder::callback_sketch): rank g computes
        # all n rows of its column slice, segment h = rows of rank h; receives its rows of every slice
        n, nc = 37, 11
        K = torch.from_numpy(np.random.default_rng(0).standard_normal((n, n)))
        om = torch.from_numpy(np.random.default_rng(1).standard_normal((n, nc)))
        cs = [r * nc // world for r in range(world + 1)]
        rb = mod.row_bounds(n, world)
        w, mine = cs[rank + 1] - cs[rank], rb[rank + 1] - rb[rank]
        part = (K @ om[:, cs[rank]:cs[rank + 1]]).contiguous()          # n x w
        sbytes = part.view(torch.uint8).reshape(-1)
        ssc = [(rb[h + 1] - rb[h]) * w * 8 for h in range(world)]
        ssd = [rb[h] * w * 8 for h in range(world)]
        rrc = [mine * (cs[h + 1] - cs[h]) * 8 for h in range(world)]
        rrd = [mine * cs[h] * 8 for h in range(world)]
        rbuf = torch.zeros(max(mine * nc, 1), dtype=torch.float64)
        mod.alltoallv_(sbytes, ssc, ssd, rbuf.view(torch.uint8), rrc, rrd)
        y = torch.empty(mine, nc, dtype=torch.float64)
        for h in range(world):
            wh = cs[h + 1] - cs[h]
            y[:, cs[h]:cs[h + 1]] = rbuf[mine * cs[h]:mine * cs[h] + mine * wh].reshape(mine, wh)
        ok = bool(torch.allclose(y, (K @ om)[rb[rank]:rb[rank + 1]], rtol=0, atol=1e-12))
        out_q.put((rank, recv.tolist(), rc, rd, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4])
def test_alltoallv_gloo_and_column_split(world):
    """The all-to-all libh2 calls for a column-split callback sketch (h2_comm.alltoallv, S§8(e)
    "splitting the sketch's sample columns"): byte segments with gaps / empty ones arrive at the
    receiver's displacements and nothing else is written; and the column-shard -> row-shard
    exchange of Builder::callback_sketch reassembles Y(own rows, all columns) = (K Omega)(rows)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_a2a_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {r[0]: r[1:] for r in (q.get(timeout=120) for _ in procs)}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for me in range(world):
        recv, rc, rd, ok = res[me]
        assert ok
        want = [255] * len(recv)
        for r in range(world):
            for i in range(rc[r]):
                want[rd[r] + i] = 10 * r + me
        assert recv == want
