"""Data parallelism for the Gaussian path.

Training: the field, grid and transforms are replicated on every rank; each
rank renders its share of the step's sample points and produces partial
per-Gaussian accumulators (acc10 = {S, T, A6}), NRF gradients, per-slice
transform gradients and loss partial sums.  All of these are plain sums over
points (the smooth-L1 mean divides by the GLOBAL batch size on every rank),
so one in-place all-reduce(sum) of the step's flat buffers gives every rank
the exact global-batch totals; every rank then runs the identical
(deterministic) epilogue + Adam, so no parameter broadcast is needed.

Two ways to share the points (plan_step):
  strong -- every rank draws the SAME global batch from the reference's RNG
            stream and renders a contiguous share of it and of the SSIM
            slice (the reference's own contiguous point chunks,
            render.py:60-77, 296-317); the SSIM slice prediction is
            assembled by one small all-reduce.  N ranks train exactly the
            model one rank (and the reference) trains.
  weak   -- every rank draws its own batch and SSIM slice (own RNG stream):
            the global batch is N x batch_points, the data loss their mean
            and the SSIM loss the mean over the N slices.

Backend: NCCL over NVLink on GPUs (captured in the step's CUDA graph), gloo
for CPU tests and for several ranks sharing one GPU (eager steps).

Inference: z-slab (axis-0) ownership of the output volume, no collective
until the optional gather (volume_slabs).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch


@dataclass(frozen=True)
class StepPlan:
    """Point layout of one step on one rank.

    The pool-index list is [batch share (nbl) | slice pixels [s_lo, s_hi) |
    the whole slice again (target only; strong sharding over >1 rank)]; the
    first nbl + (s_hi - s_lo) points are rendered.  nb_norm is the GLOBAL
    batch size the smooth-L1 mean divides by."""

    nbl: int
    nb_norm: int
    hw: tuple | None = None
    s_lo: int = 0
    s_hi: int = 0
    full_slice: bool = False

    @property
    def render(self):
        return self.nbl + (self.s_hi - self.s_lo)

    @property
    def gather(self):
        return self.render + (self.hw[0] * self.hw[1] if self.full_slice else 0)


def plan_step(idx, pix, hw, rank: int, world: int, shard: str):
    """(pool indices, StepPlan) of one step on `rank` of `world`.

    idx: the batch drawn by this rank (strong: the global batch, identical on
    every rank); pix: pool indices of the SSIM slice's pixels (or None)."""
    idx = np.asarray(idx, dtype=np.int64)
    strong = world > 1 and shard == "strong"
    nb_norm = len(idx) * (world if shard == "weak" else 1)
    if strong:
        lo, hi = shard_range(len(idx), rank, world)
        idx = idx[lo:hi]
    if pix is None:
        return idx, StepPlan(len(idx), nb_norm)
    pix = np.asarray(pix, dtype=np.int64)
    hw = tuple(int(v) for v in hw)
    if strong:
        s_lo, s_hi = shard_range(len(pix), rank, world)
        return np.concatenate([idx, pix[s_lo:s_hi], pix]), StepPlan(len(idx), nb_norm, hw, s_lo, s_hi, True)
    return np.concatenate([idx, pix]), StepPlan(len(idx), nb_norm, hw, 0, len(pix))


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
