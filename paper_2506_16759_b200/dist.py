"""Multi-GPU plumbing (one process per GPU, torch.distributed over NCCL/NVLink).

The O(N^2) dense-kernel sketch Y = K Omega (Algorithm 1 line 1; BASELINE
configs[1..2]) shards by rows with no communication of Omega (each rank regenerates the
counter-based stream, R8): rank r computes Y(rows_r, :) and the shards are
all-gathered so that every rank holds the full Y for the (replicated) construction proper.
Arithmetic stays in libh2; this module only partitions rows and moves bytes.

``Comm`` is the communicator of the sharded construction (h2_build_dist, include/h2.h; S§8(e)):
libh2 calls its in-place ``allgatherv`` on device buffers once per level (ranks, skeleton
indices I~, the next level's Omega rows), and its ``alltoallv`` once per draw of a column-split
callback sketch (sketch_split="cols"), and torch.distributed moves the bytes: NCCL over NVLink
on GPU tensors, or gloo through host staging (multi-process tests on one GPU / CPU).
"""
import ctypes as C
import os

import torch
import torch.distributed as dist


def row_bounds(n: int, world: int):
    """Balanced contiguous row ranges [b_r, b_{r+1}) of n rows over `world` ranks."""
    return [n * r // world for r in range(world + 1)]


class ShardedSketch:
    """h2 sketch callback: compute this rank's rows with `shard_fn(omega, out, r0, r1)` and
    all-gather them into y.  Called by h2_build with all N rows of Omega (tree order)."""

    def __init__(self, n: int, shard_fn, rank: int = None, world: int = None, group=None):
        self.n = n
        self.shard_fn = shard_fn
        self.group = group
        self.rank = dist.get_rank(group) if rank is None else rank
        self.world = dist.get_world_size(group) if world is None else world
        self.bounds = row_bounds(n, self.world)
        self.maxrows = max(self.bounds[i + 1] - self.bounds[i] for i in range(self.world))
        self.bytes_moved = 0

    def __call__(self, om, y, col0, row_begin, row_end):
        assert row_begin == 0 and row_end == self.n
        nc = om.shape[1]
        r0, r1 = self.bounds[self.rank], self.bounds[self.rank + 1]
        part = torch.zeros((self.maxrows, nc), dtype=om.dtype, device=om.device)
        self.shard_fn(om, part[: r1 - r0], r0, r1)
        if dist.get_backend(self.group) == "nccl":
            gathered = torch.empty((self.world * self.maxrows, nc), dtype=om.dtype, device=om.device)
            dist.all_gather_into_tensor(gathered, part, group=self.group)
            chunks = [gathered[r * self.maxrows:(r + 1) * self.maxrows] for r in range(self.world)]
        else:
            chunks = [torch.empty_like(part) for _ in range(self.world)]
            dist.all_gather(chunks, part, group=self.group)
        for r in range(self.world):
            a, b = self.bounds[r], self.bounds[r + 1]
            y[a:b].copy_(chunks[r][: b - a])
        self.bytes_moved += part.numel() * part.element_size() * (self.world - 1)


def dense_shard_fn(tree, kernel):
    """shard_fn computing rows [r0, r1) of the built-in dense kernel sketch with libh2."""
    from . import h2 as _h2

    def fn(om, out, r0, r1):
        _h2.dense_sketch(tree, om, kernel, r0, r1, out=out, omega_quarters=True)   # h2 stream Omega
    return fn


def owned_range(n_clusters: int, rank: int, world: int):
    """Clusters [b, e) of a depth with n_clusters clusters owned by `rank` (cluster c belongs to
    rank floor(c * world / n_clusters); mirrors h2_dist_range)."""
    return (rank * n_clusters + world - 1) // world, ((rank + 1) * n_clusters + world - 1) // world


def allgatherv_(buf: torch.Tensor, counts, displs, group=None):
    """In-place all-gather of byte segments of a 1-D uint8 tensor: segment r =
    buf[displs[r] : displs[r] + counts[r]] is valid on rank r on entry and on every rank on
    return.  NCCL (device tensors): one all-gather of max-size segments through a staging
    buffer; otherwise one broadcast per non-empty segment (gloo: host staging)."""
    nccl = dist.get_backend(group) == "nccl"
    me = dist.get_rank(group)
    if nccl and buf.is_cuda:
        # one NCCL all-gather of equal (max) segments, in place in a staging buffer, then the
        # variable segments are copied out (P small device copies instead of P broadcasts)
        P = len(counts)
        mx = max(counts)
        if mx == 0:
            return
        stage = torch.empty(P * mx, dtype=torch.uint8, device=buf.device)
        mine = torch.zeros(mx, dtype=torch.uint8, device=buf.device)
        c, d = counts[me], displs[me]
        if c:
            mine[:c].copy_(buf[d:d + c])
        dist.all_gather_into_tensor(stage, mine, group=group)
        for r in range(P):
            if r != me and counts[r]:
                buf[displs[r]:displs[r] + counts[r]].copy_(stage[r * mx:r * mx + counts[r]])
        return
    for r, (c, d) in enumerate(zip(counts, displs)):
        if c == 0:
            continue
        seg = buf[d:d + c]
        src = dist.get_global_rank(group, r) if group is not None else r
        if nccl or not seg.is_cuda:
            dist.broadcast(seg, src=src, group=group)
        else:
            host = seg.cpu() if r == me else torch.empty(c, dtype=torch.uint8)
            dist.broadcast(host, src=src, group=group)
            if r != me:
                seg.copy_(host)


def alltoallv_(send: torch.Tensor, scounts, sdispls, recv: torch.Tensor, rcounts, rdispls, group=None):
    """All-to-all of byte segments of 1-D uint8 tensors (the column-split sketch exchange,
    include/h2.h h2_alltoallv_fn): send[sdispls[r] : sdispls[r] + scounts[r]] goes to rank r and
    arrives at recv[rdispls[me] : rdispls[me] + rcounts[me]] there.  The segments are packed in rank
    order into a staging tensor and moved by one ``all_to_all_single`` with split sizes (NCCL on
    device tensors; gloo on host copies), then copied out."""
    me = dist.get_rank(group)
    P = len(scounts)
    nccl = dist.get_backend(group) == "nccl"
    dev = send.device
    stage_dev = dev if (nccl or not send.is_cuda) else torch.device("cpu")
    packed = [send[d:d + c] for c, d in zip(scounts, sdispls)]
    sbuf = torch.cat(packed).to(stage_dev) if sum(scounts) else torch.empty(0, dtype=torch.uint8, device=stage_dev)
    rbuf = torch.empty(sum(rcounts), dtype=torch.uint8, device=stage_dev)
    dist.all_to_all_single(rbuf, sbuf, output_split_sizes=list(rcounts), input_split_sizes=list(scounts),
                           group=group)
    o = 0
    for r in range(P):
        c = rcounts[r]
        if c:
            recv[rdispls[r]:rdispls[r] + c].copy_(rbuf[o:o + c])
        o += c
    return me


class Comm:
    """h2_comm over a torch.distributed process group (one process per GPU)."""

    def __init__(self, group=None):
        from . import _lib as L
        from .h2 import device_view
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.calls = 0
        self.bytes = 0

        def _agv(ctx, buf, counts, displs, stream):
            try:
                P = self.world
                cnt = [int(counts[i]) for i in range(P)]
                dsp = [int(displs[i]) for i in range(P)]
                end = max(d + c for c, d in zip(cnt, dsp))
                if os.environ.get("H2_COMM_TRACE"):
                    print(f"[rank {self.rank}] allgatherv #{self.calls} counts {cnt} displs {dsp}", flush=True)
                with torch.cuda.stream(torch.cuda.ExternalStream(stream or 0)):
                    view = device_view(buf, (end,), (1,), dtype=torch.uint8)
                    allgatherv_(view, cnt, dsp, self.group)
                self.calls += 1
                self.bytes += sum(cnt) - cnt[self.rank]
                return 0
            except Exception:
                import traceback
                traceback.print_exc()
                return 1
        def _a2a(ctx, send, scounts, sdispls, recv, rcounts, rdispls, stream):
            try:
                P = self.world
                sc = [int(scounts[i]) for i in range(P)]
                sd = [int(sdispls[i]) for i in range(P)]
                rc = [int(rcounts[i]) for i in range(P)]
                rd = [int(rdispls[i]) for i in range(P)]
                with torch.cuda.stream(torch.cuda.ExternalStream(stream or 0)):
                    sv = device_view(send, (max(d + c for c, d in zip(sc, sd)),), (1,), dtype=torch.uint8)
                    rv = device_view(recv, (max(d + c for c, d in zip(rc, rd)),), (1,), dtype=torch.uint8)
                    alltoallv_(sv, sc, sd, rv, rc, rd, self.group)
                self.a2a_calls += 1
                self.a2a_bytes += sum(sc) - sc[self.rank]
                return 0
            except Exception:
                import traceback
                traceback.print_exc()
                return 1
        self.a2a_calls = 0
        self.a2a_bytes = 0
        self._cb = L.ALLGATHERV_FN(_agv)
        self._cb2 = L.ALLTOALLV_FN(_a2a)
        self.struct = L.h2_comm(self.rank, self.world, self._cb, None, None, self._cb2)


class NcclComm:
    """libh2's in-library NCCL communicator (h2_comm_init; one process per GPU): the 128-byte NCCL
    unique id of rank 0 is broadcast with torch.distributed, every rank initialises NCCL on its
    current device, and the per-level all-gathers of the sharded construction run inside libh2
    as stream-ordered NCCL broadcast groups (no Python callback, no host synchronisation)."""

    def __init__(self, group=None):
        from . import _lib as L
        self._L = L
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        idb = C.create_string_buffer(128)
        if self.rank == 0:
            L.check(L.lib.h2_comm_get_unique_id(idb))
        obj = [bytes(idb.raw) if self.rank == 0 else None]
        src = dist.get_global_rank(group, 0) if group is not None else 0
        dist.broadcast_object_list(obj, src=src, group=group)
        idb = C.create_string_buffer(obj[0], 128)
        p = C.POINTER(L.h2_comm)()
        L.check(L.lib.h2_comm_init(idb, self.rank, self.world, C.byref(p)))
        self._p = p
        self.struct = p.contents

    def allgatherv(self, buf, counts, displs, stream=None):
        """In-place all-gather of byte segments of a CUDA tensor (h2_comm_allgatherv)."""
        import torch
        P = self.world
        cnt = (C.c_int64 * P)(*counts)
        dsp = (C.c_int64 * P)(*displs)
        s = (stream or torch.cuda.current_stream()).cuda_stream
        self._L.check(self._L.lib.h2_comm_allgatherv(self._p, C.c_void_p(buf.data_ptr()), cnt, dsp, C.c_void_p(s)))

    def alltoallv(self, send, scounts, sdispls, recv, rcounts, rdispls, stream=None):
        """All-to-all of byte segments between CUDA tensors (h2_comm_alltoallv: grouped
        ncclSend / ncclRecv inside libh2)."""
        import torch
        P = self.world
        arr = lambda v: (C.c_int64 * P)(*v)
        s = (stream or torch.cuda.current_stream()).cuda_stream
        self._L.check(self._L.lib.h2_comm_alltoallv(self._p, C.c_void_p(send.data_ptr()), arr(scounts), arr(sdispls),
                                                    C.c_void_p(recv.data_ptr()), arr(rcounts), arr(rdispls),
                                                    C.c_void_p(s)))

    def close(self):
        if getattr(self, "_p", None):
            self._L.lib.h2_comm_free(self._p)
            self._p = None

    def __del__(self):
        self.close()
