"""Data parallelism for the Gaussian path.

Training: the field, grid and transforms are replicated on every rank; each
rank renders its own share of the step's sample points and produces partial
per-Gaussian accumulators (acc10 = {S, T, A6}), per-slice transform
gradients and loss partial sums.  All of these are plain sums over points,
so ONE all-reduce(sum) of a flat buffer per step gives every rank the exact
full-batch totals; every rank then runs the identical (deterministic)
epilogue + Adam, so no parameter broadcast is needed.  Backend: NCCL over
NVLink on GPUs, gloo on CPU (tests).

Inference: z-slab (axis-0) ownership of the output volume, no collective.
"""

from __future__ import annotations

import torch


def shard_range(n: int, rank: int, world: int):
    """Contiguous [lo, hi) share of n items for `rank` (sizes differ by <= 1)."""
    base, rem = divmod(int(n), int(world))
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def slab_ranges(nx: int, world: int):
    """Axis-0 voxel slabs [(i0, i1)] for z-slab sharded inference."""
    return [shard_range(nx, r, world) for r in range(world)]


class FlatAllReduce:
    """One all-reduce(sum) per step over several same-dtype buffers.

    The buffers are packed into a persistent flat tensor (so the collective is
    a single NCCL call of tens of MB, sized for NVLink/NVLS bandwidth rather
    than launch count), reduced, and unpacked in place."""

    def __init__(self, tensors, group=None):
        self.tensors = list(tensors)
        dt = {t.dtype for t in self.tensors}
        if len(dt) != 1:
            raise ValueError("FlatAllReduce needs one dtype per group")
        self.sizes = [t.numel() for t in self.tensors]
        self.flat = torch.empty(sum(self.sizes), dtype=self.tensors[0].dtype, device=self.tensors[0].device)
        self.group = group

    def __call__(self):
        import torch.distributed as dist

        off = 0
        for t, n in zip(self.tensors, self.sizes):
            self.flat[off:off + n].copy_(t.reshape(-1))
            off += n
        dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=self.group)
        off = 0
        for t, n in zip(self.tensors, self.sizes):
            t.view(-1).copy_(self.flat[off:off + n])
            off += n


def allreduce_sum(tensors, group=None):
    """All-reduce(sum) a list of tensors, grouped by dtype into flat buffers."""
    by_dtype = {}
    for t in tensors:
        by_dtype.setdefault(t.dtype, []).append(t)
    for ts in by_dtype.values():
        FlatAllReduce(ts, group)()
