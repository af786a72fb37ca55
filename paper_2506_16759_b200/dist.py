"""Multi-GPU plumbing (one process per GPU, torch.distributed over NCCL/NVLink).

The O(N^2) dense-kernel sketch Y = K Omega (Algorithm 1 line 1; BASELINE
configs[1..2]) shards by rows with no communication of Omega (each rank regenerates the
counter-based stream, R8): rank r computes Y(rows_r, :) and the shards are
all-gathered so that every rank holds the full Y for the (replicated) construction proper.
This is the path's one exchange step.  Arithmetic stays in libh2; this module
only partitions rows and moves the shards.
"""
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
