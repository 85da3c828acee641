"""Device-resident training step -- drop-in for the hot part of
/root/reference/pkg/src/mgauss/train.py (TrainConfig, losses, AdamState,
progressive_upsample, init_field, Trainer.step / run / render_volume).

One step runs entirely on the B200: Gaussian binning (counting sort) and
activation, point transform + PSF taps + binning, the cell-exact forward
(with H = sum alpha g P d for d_points), smooth-L1 and SSIM gradients,
the Gaussian-major backward (cutoff-culled windows), transform gradients,
the NRF on tensor cores, and one fused kernel for the chain rule +
anisotropy penalty + Adam on the four Gaussian groups.
The host only draws batch indices from the reference's RNG stream
(SeedSequence(seed).spawn(2), train.py:332-335,348-363,408) so batches are
identical to the reference's.  With ``graph=True`` the step is captured
once per lattice level and replayed as a CUDA graph.

Multi-GPU: Gaussians replicated, sample points sharded; the
only exchange is an all-reduce(sum) of the per-Gaussian accumulators, the
transform accumulators and the loss partials.

StrictTrainer (strict_train.py, re-exported here) is the same step on float64
kernels in the reference's operation order, for parity runs.
"""

from __future__ import annotations

from dataclasses import dataclass, field as dc_field, replace  # noqa: F401

import os

import numpy as np
import torch

from . import _device as dv
from . import _native as N
from .core import TransformSet, lattice_node_index, lattice_node_positions  # noqa: F401
from .errors import NonFiniteLoss, ShrinkNotAllowed
from .parallel import StepPlan, plan_step
from .render import SlicePSF, sample_volume_device

DEFAULT_SCHEDULE = ((0, 70), (500, 100), (1000, 130), (2000, 165), (3000, 200))


_GC_FROZEN = False
_STREAMS = {}


def _graph_pool():
    """One private memory pool for every step graph on the device.  Only one
    step graph is alive at a time (a new shape drops the old graph first), so
    a capture reuses the blocks its predecessor released instead of freeing
    them and allocating fresh ones (cudaFree/cudaMalloc: 0.05-0.17 s per
    recapture at the reconstruction's lattice milestones)."""
    key = ("graph_pool", dv.device())
    ent = _STREAMS.get(key)
    if ent is None:
        # a pool lives while some graph captured into it does: a one-op keeper
        # graph holds it across the gaps between step graphs
        h = torch.cuda.graph_pool_handle()
        keeper = torch.cuda.CUDAGraph()
        cs = _stream("capture")
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(cs):
            keeper.capture_begin(pool=h)
            torch.zeros((1,), device=dv.device())
            keeper.capture_end()
        ent = _STREAMS[key] = (h, keeper)
    return ent[0]


def _stream(name):
    """Process-wide side streams (copy / capture / parallel branch), shared by
    all trainers on the device: a fresh stream per trainer pays new cuBLAS
    workspaces and handles on its first use (up to 0.3 s at the NRF switch)."""
    key = (name, dv.device())
    st = _STREAMS.get(key)
    if st is None:
        st = _STREAMS[key] = torch.cuda.Stream(device=dv.device())
    return st


def freeze_gc():
    """Move everything alive now (torch, numpy and the caller's module state:
    several hundred thousand objects) out of the cyclic collector's reach.  A
    full collection over them took 0.1-0.4 s and landed at random inside a
    step loop (measured as 0.3 s stalls in a 0.7 s desk-scale reconstruction).
    Objects created later are collected as usual.  Process-wide, so it is
    opt-in: the bench and reconstruction entry points call it; a Trainer calls
    it at construction only when MGAUSS_GC_FREEZE=1."""
    global _GC_FROZEN
    if _GC_FROZEN:
        return
    import gc

    gc.collect()
    gc.freeze()
    _GC_FROZEN = True


def _freeze_gc_once():
    if os.environ.get("MGAUSS_GC_FREEZE", "0") == "1":
        freeze_gc()


_PERM_PREFETCH_MIN = 1 << 16
_UPD_SORTED = os.environ.get("MGAUSS_UPD_SORTED", "0") == "1"  # A/B: update walking the sorted order  # pools from this size draw epoch permutations ahead


@dataclass
class TrainConfig:
    """Hyperparameters with the reference defaults (train.py:40-66)."""

    lr_position: float = 0.001
    lr_intensity: float = 0.05
    lr_scale: float = 0.005
    lr_rotation: float = 0.001
    lr_nrf: float = 0.0001
    lr_transform: float = 0.0001
    lambda_ssim: float = 0.5
    lambda_aniso: float = 0.1
    lambda_ratio: float = 1.5
    block_radius: int = 5
    resolution_schedule: tuple = DEFAULT_SCHEDULE
    nrf_activation_iter: int = 2000
    total_iters: int = 4000
    batch_points: int = 65536
    adam_beta1: float = 0.9
    adam_beta2: float = 0.999
    adam_eps: float = 1e-8
    seed: int = 0
    use_ssim: bool = True
    use_nrf: bool = True
    use_aniso: bool = True
    use_progressive: bool = True

    def validate(self):
        for name in ("lr_position", "lr_intensity", "lr_scale", "lr_rotation", "lr_nrf", "lr_transform"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be > 0")
        sched = tuple((int(i), int(r)) for i, r in self.resolution_schedule)
        if not sched or sched[0][0] != 0:
            raise ValueError("resolution_schedule must start at iteration 0")
        its = [i for i, _ in sched]
        if any(b <= a for a, b in zip(its, its[1:])):
            raise ValueError("schedule iterations must be strictly increasing")
        res = [r for _, r in sched]
        if any(b < a for a, b in zip(res, res[1:])):
            raise ValueError("schedule resolutions must be non-decreasing")
        if self.batch_points < 1 or self.total_iters < 0:
            raise ValueError("batch_points >= 1 and total_iters >= 0 required")
        return self

    def resolution_at(self, iteration):
        res = self.resolution_schedule[0][1]
        for it, r in self.resolution_schedule:
            if iteration >= it:
                res = r
        return res

    @property
    def final_resolution(self):
        return max(r for _, r in self.resolution_schedule)

    def to_dict(self):
        """JSON-ready dict (train.py:96-99): the schedule as nested lists."""
        d = dict(self.__dict__)
        d["resolution_schedule"] = [list(m) for m in self.resolution_schedule]
        return d

    @classmethod
    def from_dict(cls, d):
        d = dict(d)
        d["resolution_schedule"] = tuple(tuple(m) for m in d["resolution_schedule"])
        return cls(**d).validate()


@dataclass
class LossReport:
    iteration: int
    total: float
    data: float
    ssim: float
    aniso: float
    resolution: int
    nrf_active: bool
    pairs: int = 0

    def to_line(self):
        return (f"iter={self.iteration} total={self.total:.10g} l1={self.data:.10g} ssim={self.ssim:.10g} "
                f"aniso={self.aniso:.10g} res={self.resolution} nrf={int(self.nrf_active)}")


@dataclass
class DeviceField:
    """Learnable Gaussian parameters (float32 device tensors) on an R^3 lattice.
    node_of[(i*R + j)*R + k] = primitive id at lattice node (i, j, k)."""

    positions: torch.Tensor
    quaternions: torch.Tensor
    log_scales: torch.Tensor
    logits: torch.Tensor
    resolution: int
    node_of: torch.Tensor

    @property
    def count(self):
        return int(self.positions.shape[0])

    @property
    def lattice_dims(self):  # GaussianField's name (core.py:250-301)
        return (self.resolution,) * 3

    @property
    def intensity_logits(self):
        return self.logits

    def to_host(self):
        from .core import GaussianField

        r = self.resolution
        node = dv.to_host(self.node_of).astype(np.int64)
        lat = np.empty((self.count, 3), np.int64)
        lat[node] = lattice_node_index(r)
        return GaussianField(dv.to_host(self.positions).astype(np.float64),
                             dv.to_host(self.quaternions).astype(np.float64),
                             dv.to_host(self.log_scales).astype(np.float64),
                             dv.to_host(self.logits).astype(np.float64), (r, r, r), lat)

    @classmethod
    def from_host(cls, field):
        r = int(field.lattice_dims[0])
        li = np.asarray(field.lattice_index, dtype=np.int64)
        node_of = np.empty(field.count, np.int32)
        node_of[(li[:, 0] * r + li[:, 1]) * r + li[:, 2]] = np.arange(field.count, dtype=np.int32)
        return cls(dv.to_dev(field.positions, torch.float32), dv.to_dev(field.quaternions, torch.float32),
                   dv.to_dev(field.log_scales, torch.float32), dv.to_dev(field.intensity_logits, torch.float32),
                   r, dv.to_dev(node_of, torch.int32))


def uniform_lattice_device(r, logits=None):
    """uniform_lattice_field on the device (core.py:318-342)."""
    n = r ** 3
    pos = dv.to_dev(lattice_node_positions(r), torch.float32)
    q = dv.zeros((n, 4), torch.float32)
    q[:, 0] = 1.0
    s = torch.full((n, 3), float(np.log(1.0 / r)), dtype=torch.float32, device=pos.device)
    lg = dv.zeros((n,), torch.float32) if logits is None else logits.to(torch.float32)
    return DeviceField(pos, q, s, lg, r, torch.arange(n, dtype=torch.int32, device=pos.device))


def init_field_device(coords: torch.Tensor, intensities: torch.Tensor, r: int, logit_eps=1e-4):
    """Logit of the mean sample intensity per lattice cell, 0 where empty (train.py:221-236)."""
    return uniform_lattice_device(r, _init_logits(coords, intensities, r, logit_eps))


def _init_logits(coords: torch.Tensor, intensities: torch.Tensor, r: int, logit_eps):
    """float64 (r^3,) logits of the per-cell mean intensity (0 where empty)."""
    n = r ** 3
    keys = dv.empty((coords.shape[0],), torch.int32)
    N.check(N.lib().mg_cell_keys_f64(N.ptr(coords), coords.shape[0], r, N.ptr(keys), dv.sptr()), "cell_keys")
    k = keys.to(torch.int64)
    sums = torch.zeros(n, dtype=torch.float64, device=coords.device).index_add_(0, k, intensities.double())
    cnts = torch.bincount(k, minlength=n).double()
    occ = cnts > 0
    mean = torch.where(occ, sums / cnts.clamp(min=1), torch.full_like(sums, 0.5))
    mean = mean.clamp(logit_eps, 1.0 - logit_eps)
    return torch.where(occ, torch.log(mean) - torch.log1p(-mean), torch.zeros_like(mean))


def progressive_upsample_device(field: DeviceField, new_r: int) -> DeviceField:
    """train.py:157-218 on the device: trilinear logits/log-scales, sign-aligned
    NLERP quaternions, positions reseeded on the new lattice."""
    old_r = field.resolution
    if new_r < old_r:
        raise ShrinkNotAllowed(f"cannot shrink lattice {old_r} -> {new_r}")
    n = new_r ** 3
    pos = dv.empty((n, 3), torch.float32)
    q = dv.empty((n, 4), torch.float32)
    s = dv.empty((n, 3), torch.float32)
    lg = dv.empty((n,), torch.float32)
    N.check(N.lib().mg_upsample(N.ptr(field.quaternions), N.ptr(field.log_scales), N.ptr(field.logits),
                                N.ptr(field.node_of), old_r, new_r, N.ptr(pos), N.ptr(q), N.ptr(s), N.ptr(lg),
                                dv.sptr()), "upsample")
    return DeviceField(pos, q, s, lg, new_r, torch.arange(n, dtype=torch.int32, device=pos.device))


def _hyper_array(cfg):
    """Host hyper-parameter block read by mg_gauss_update (9 doubles)."""
    return np.array([cfg.lr_position, cfg.lr_rotation, cfg.lr_scale, cfg.lr_intensity, cfg.adam_beta1,
                     cfg.adam_beta2, cfg.adam_eps, cfg.lambda_aniso, cfg.lambda_ratio], dtype=np.float64)


class _StepBuffers:
    """Fixed-shape device buffers for one (N, rendered points, taps, K, NRF)
    configuration.  Everything a distributed step all-reduces lives in two
    flat buffers (acc10 + the NRF gradients in float32; the loss partials and
    the per-slice transform gradients in float64), so the collective runs
    in place on them with no copy in or out."""

    def __init__(self, n, g, b_render, b_gather, ntaps, k, nrf_numel=0):
        L = N.lib()
        ns = b_render * ntaps
        self.gkey = dv.empty((n,), torch.int32)
        self.gorder = dv.empty((n,), torch.int32)
        self.ginv = dv.empty((n,), torch.int32)  # sorted position of each Gaussian (coalesced update walk)
        self.gstart = dv.empty((g ** 3 + 1,), torch.int32)
        self.grec = dv.empty((n, 12), torch.float32)
        self.flat32 = dv.empty((10 * n + nrf_numel,), torch.float32)
        self.acc10 = self.flat32[:10 * n].view(n, 10)
        self.nrf_numel = nrf_numel
        self.pkey = dv.empty((ns,), torch.int32)
        self.pinv = dv.empty((ns,), torch.int32)
        self.pstart = dv.empty((g ** 3 + 1,), torch.int32)
        self.prec = dv.empty((ns, 4), torch.float32)
        self.xout = dv.empty((ns, 3), torch.float64)
        self.out4 = dv.empty((ns, 4), torch.float32)
        self.cnt = dv.empty((ns,), torch.int32)
        self.pred = dv.empty((b_render,), torch.float32)
        self.up = dv.empty((b_render,), torch.float32)
        self.dpts = dv.empty((ns, 3), torch.float64)
        self.rot = dv.empty((max(k, 1), 3, 3), torch.float64)
        kk = max(k, 1)
        self.flat64 = dv.zeros((4 + 7 * kk,), torch.float64)
        self.scalars = self.flat64[:4]  # data loss, aniso loss, ssim sum, spare (non-reporting ranks' ssim)
        self.g7 = self.flat64[4:].view(kk, 7)
        self.scratch12 = dv.empty((kk, 12), torch.float64)
        self.err = dv.zeros((1,), torch.int32)
        wsb = max(L.mg_bin_workspace_bytes(n, g), L.mg_points_workspace_bytes(ns, g),
                  L.mg_forward_workspace_bytes(ns), L.mg_backward_workspace_bytes(n, g),
                  L.mg_transform_grads_workspace_bytes(k))
        self.ws = dv.empty((wsb,), torch.uint8)
        self.ws_gauss = None  # side-stream workspaces (Gaussian binning, transform reduction)
        self.ws_tr = None
        self.ssim_ws = None
        self.slice_pred = None  # strong-sharded SSIM: full-slice prediction / upstream
        self.slice_up = None
        self.idx = dv.empty((b_gather,), torch.int64)
        self.coords = dv.empty((b_gather, 3), torch.float64)
        self.sids = dv.empty((b_gather,), torch.int64)
        self.tgt = dv.empty((b_gather,), torch.float32)
        self.pairs = dv.zeros((1,), torch.int64)
        # two pinned index staging slots (a slot is rewritten only after its
        # previous H2D copy has completed)
        self.idx_host = [torch.empty((b_gather,), dtype=torch.int64, pin_memory=True) for _ in range(2)]
        self.idx_done = [None, None]
        self.slot = 0
        # device landing slots for the H2D copies, which run on a copy stream
        # under the previous step; the step itself reads B.idx (a fixed
        # address for the graph), filled by a short D2D copy
        self.idx_stage = [dv.empty((b_gather,), torch.int64) for _ in range(2)]
        self.stage_free = [None, None]
        # two pinned loss-readback slots (pipelined steps read one while the next fills)
        self.scalars_host = [torch.empty((4,), dtype=torch.float64, pin_memory=True) for _ in range(2)]
        self.err_host = [torch.empty((1,), dtype=torch.int32, pin_memory=True) for _ in range(2)]
        self.r_done = [None, None]
        self.rslot = 0

    def nrf_grad_flat(self):
        return self.flat32[self.flat32.numel() - self.nrf_numel:]


class Trainer:
    """Owns the device field, transforms, optimizer state and the batch stream."""

    def __init__(self, cloud, transforms: TransformSet, config: TrainConfig, slice_grids=None,
                 slice_psf: SlicePSF | None = None, graph=False, dist=None, shard="strong"):
        """``dist``: a torch.distributed group (NCCL on GPUs) for data
        parallelism.  ``shard="strong"`` splits every step's global batch and
        SSIM slice into contiguous per-rank shares (all ranks draw the same
        batch from the reference's RNG stream), so N ranks train exactly the
        reference's model; ``"weak"`` gives every rank its own full batch and
        SSIM slice (its own RNG stream; global batch N x batch_points)."""
        config.validate()
        if shard not in ("strong", "weak"):
            raise ValueError("shard must be 'strong' or 'weak'")
        _freeze_gc_once()
        if config.use_ssim and not slice_grids:
            raise ValueError("use_ssim requires slice sample grids")
        self.config = config
        self.psf = slice_psf
        self.graph = graph
        self.dist = dist  # optional torch.distributed group for gradient all-reduce
        self.shard = shard
        if dist is not None:
            import torch.distributed as tdist

            self.rank, self.world = tdist.get_rank(dist), tdist.get_world_size(dist)
        else:
            self.rank, self.world = 0, 1
        self.coords = dv.to_dev(cloud.coords, torch.float64)
        self.intens = dv.to_dev(cloud.intensities, torch.float32)
        self.sids = dv.to_dev(cloud.slice_ids, torch.int64)
        self.m_points = int(self.coords.shape[0])
        self.slice_grids = list(slice_grids or [])
        self._prepare_sources()
        ts = transforms.copy()
        self.k = len(ts)
        self.tq = dv.to_dev(ts.quats, torch.float64, (self.k, 4))
        self.tt = dv.to_dev(ts.translations, torch.float64, (self.k, 3))
        self.tm = dv.zeros((max(self.k, 1), 7), torch.float64)
        self.tv = dv.zeros((max(self.k, 1), 7), torch.float64)
        root = np.random.SeedSequence(config.seed)
        batch_ss, nrf_ss = root.spawn(2)
        if shard == "weak" and self.rank > 0:  # rank 0 keeps the reference stream
            batch_ss = np.random.SeedSequence(batch_ss.entropy, spawn_key=batch_ss.spawn_key + (1 << 20, self.rank))
        self.rng = np.random.default_rng(batch_ss)
        self.nrf = None
        if config.use_nrf:
            from .nrf import ResidualField

            self.nrf = ResidualField.create(np.random.default_rng(nrf_ss))
            self.nrf_m = {k: torch.zeros_like(v) for k, v in self.nrf.parameter_arrays().items()}
            self.nrf_v = {k: torch.zeros_like(v) for k, v in self.nrf.parameter_arrays().items()}
            self.nrf_t = 0
        start = config.resolution_at(0) if config.use_progressive else config.final_resolution
        self.field = init_field_device(self.coords, self.intens, start)
        self._reset_gauss_adam()
        self.counters = dv.zeros((2,), torch.int32)  # [gauss t, transform t]
        self.iteration = 0
        self._perm = None
        self._cursor = 0
        self._permuter = None  # next-epoch permutation prefetch (large pools)
        b = min(config.batch_points, self.m_points)
        if (self.m_points >= _PERM_PREFETCH_MIN and b < self.m_points
                and os.environ.get("MGAUSS_PERM_PREFETCH", "1") != "0"):
            from ._permuter import EpochPermuter

            # spawned now so its interpreter start-up (~0.5 s) overlaps the
            # set-up and warm-up instead of the first epochs
            self._permuter = EpochPermuter(self.m_points)
        self.reports = []
        self._bufs = None
        self._bufs_key = None
        self._graph = None
        self._graph_key = None
        self._hyper = _hyper_array(config)
        if slice_psf is not None:
            self._psf_off = dv.to_dev(np.asarray(slice_psf.offsets, dtype=np.float64), torch.float64)
            self._psf_w = dv.to_dev(np.asarray(slice_psf.weights, dtype=np.float64), torch.float64)
            self._psf_dirs = dv.to_dev(np.asarray(slice_psf.through_dirs, dtype=np.float64).reshape(-1, 3),
                                       torch.float64)

    # -- state --------------------------------------------------------------
    def _reset_gauss_adam(self):
        n = self.field.count
        # Adam moments, structure-of-arrays [11][n] (slots: pos 3, quat 4, log-scale 3, logit 1)
        self.m = dv.zeros((11, n), torch.float32)
        self.v = dv.zeros((11, n), torch.float32)
        if hasattr(self, "counters"):
            self.counters[0].zero_()

    @property
    def nrf_active(self):
        return self.config.use_nrf and self.iteration >= self.config.nrf_activation_iter

    @property
    def ntaps(self):
        return 1 if self.psf is None else self.psf.ntaps

    # -- batching (train.py:348-363) ------------------------------------------
    def _next_batch(self):
        m = self.m_points
        b = min(self.config.batch_points, m)
        if b == m:
            return np.arange(m)
        picked, need, drew = [], b, False
        while need > 0:
            if self._perm is None or self._cursor >= m:
                perm = self._permuter.take(self.rng) if self._permuter is not None else None
                self._perm = perm if perm is not None else self.rng.permutation(m)
                self._cursor = 0
                drew = True
            take = min(need, m - self._cursor)
            picked.append(self._perm[self._cursor:self._cursor + take])
            self._cursor += take
            need -= take
        # copy the batch out before the helper may refill the old slot
        out = np.concatenate(picked) if len(picked) > 1 else picked[0].copy()
        if drew and m >= _PERM_PREFETCH_MIN and os.environ.get("MGAUSS_PERM_PREFETCH", "1") != "0":
            # RNG draws between epoch boundaries: this step's slice pick and one
            # per full step still served by the current permutation; the next
            # epoch starts with cursor b - ((m - cursor) % b)
            ns = [len(self.slice_grids)] if self.config.use_ssim else []
            calls_e = ns * (1 + (m - self._cursor) // b)
            c_next = b - (m - self._cursor) % b
            calls_next = ns * (1 + (m - c_next) // b)
            if self._permuter is None:
                from ._permuter import EpochPermuter

                self._permuter = EpochPermuter(m)
            if self._permuter.chained:  # the next epoch is queued: queue the one after it
                self._permuter.extend(calls_next)
            else:
                self._permuter.start(self.rng, calls_e, calls_next)
        return out

    def _apply_milestones(self):
        if not self.config.use_progressive:
            return
        for it, res in self.config.resolution_schedule:
            if it == self.iteration and res > self.field.resolution:
                self.field = progressive_upsample_device(self.field, res)
                self._reset_gauss_adam()
                self._graph = None

    def _prepare_sources(self):
        """Cloud + every slice grid in one device pool, so a step's points are a
        single index gather (graph-replayable with a fixed index buffer)."""
        cs, ss, ts = [self.coords], [self.sids], [self.intens]
        self._sg_off, self._sg_shape = [], []
        base = self.m_points
        for sg in self.slice_grids:
            c = dv.to_dev(np.asarray(sg.coords, np.float64).reshape(-1, 3), torch.float64)
            t = dv.to_dev(np.asarray(sg.target, np.float64).ravel(), torch.float32)
            cs.append(c)
            ts.append(t)
            ss.append(torch.full((c.shape[0],), int(sg.slice_id), dtype=torch.int64, device=c.device))
            self._sg_off.append(base)
            self._sg_shape.append(tuple(np.asarray(sg.target).shape))
            base += c.shape[0]
        if len(cs) > 1:
            self.src_coords, self.src_sids, self.src_tgt = torch.cat(cs), torch.cat(ss), torch.cat(ts)
        else:
            self.src_coords, self.src_sids, self.src_tgt = self.coords, self.sids, self.intens

    def host_indices(self, idx, slice_j):
        """Pool indices of one step on this rank and its StepPlan: the batch
        (share), then the SSIM slice's pixels (share), then -- strong sharding
        over several ranks -- the whole slice again for the SSIM target."""
        pix, hw = None, None
        if slice_j is not None:
            hw = self._sg_shape[slice_j]
            pix = self._sg_off[slice_j] + np.arange(hw[0] * hw[1], dtype=np.int64)
        return plan_step(idx, pix, hw, self.rank, self.world, self.shard)

    def draw_step(self):
        """Draw the next step's batch and SSIM slice from the host RNG stream
        (train.py:348-363,408) -> (pool indices, StepPlan)."""
        idx = self._next_batch()
        slice_j = int(self.rng.integers(len(self.slice_grids))) if self.config.use_ssim else None
        return self.host_indices(idx, slice_j)

    # -- one optimizer step ----------------------------------------------------
    # -- checkpoint state: the reference Trainer's tree (train.py:514-583) ----
    _GAUSS_GROUPS = (("positions", "p", 0, 3), ("quaternions", "q", 3, 7), ("log_scales", "s", 7, 10),
                     ("intensity_logits", "a", 10, 11))

    def state_dict(self):
        """Checkpoint tree in the reference layout (train.py:516-544), float64
        host arrays from the float32/float64 device state.  Adam groups that
        have not stepped since their last reset are absent, as in AdamState."""
        host = self.field.to_host()
        t_gauss, t_tr = (int(x) for x in dv.to_host(self.counters))
        adam = {}
        if t_gauss > 0:
            m = dv.to_host(self.m).astype(np.float64).T
            v = dv.to_host(self.v).astype(np.float64).T
            for name, key, lo, hi in self._GAUSS_GROUPS:
                cut = (lambda a: np.ascontiguousarray(a[:, lo])) if hi - lo == 1 else \
                    (lambda a: np.ascontiguousarray(a[:, lo:hi]))
                adam[name] = {"t": t_gauss, "m": {key: cut(m)}, "v": {key: cut(v)}}
        if t_tr > 0 and self.k:
            tm, tv = dv.to_host(self.tm)[:self.k], dv.to_host(self.tv)[:self.k]
            adam["transforms"] = {"t": t_tr, "m": {"q": tm[:, :4].copy(), "t": tm[:, 4:].copy()},
                                  "v": {"q": tv[:, :4].copy(), "t": tv[:, 4:].copy()}}
        if self.nrf is not None and self.nrf_t > 0:
            adam["nrf"] = {"t": int(self.nrf_t),
                           "m": {k: dv.to_host(a).astype(np.float64) for k, a in self.nrf_m.items()},
                           "v": {k: dv.to_host(a).astype(np.float64) for k, a in self.nrf_v.items()}}
        state = {
            "config": self.config.to_dict(),
            "iteration": self.iteration,
            "field": {"positions": host.positions, "quaternions": host.quaternions, "log_scales": host.log_scales,
                      "intensity_logits": host.intensity_logits, "lattice_dims": list(host.lattice_dims),
                      "lattice_index": host.lattice_index},
            "transforms": {"quats": dv.to_host(self.tq).reshape(-1, 4)[:self.k].copy(),
                           "translations": dv.to_host(self.tt).reshape(-1, 3)[:self.k].copy()},
            "adam": adam,
            "rng_state": self.rng.bit_generator.state,
            "perm": None if self._perm is None else np.array(self._perm, dtype=np.int64),
            "cursor": self._cursor,
        }
        if self.nrf is not None:
            state["nrf"] = {"frequency_bands": self.nrf.frequency_bands, "layer_widths": list(self.nrf.layer_widths),
                            "weights": [dv.to_host(w).astype(np.float64) for w in self.nrf.weights],
                            "biases": [dv.to_host(b).astype(np.float64) for b in self.nrf.biases]}
        return state

    def load_state_dict(self, state):
        """Resume from a checkpoint tree written by ``state_dict`` (bit-exact
        continuation) or by the reference Trainer (parameters rounded to
        float32).  The trainer must have been built on the same data."""
        from .core import GaussianField

        cfg = TrainConfig.from_dict(state["config"])
        self.config = cfg
        self._hyper = _hyper_array(cfg)  # the fused Gaussian Adam reads the resumed config's values
        f = state["field"]
        dims = tuple(int(d) for d in f["lattice_dims"])
        self.field = DeviceField.from_host(GaussianField(
            np.asarray(f["positions"], np.float64), np.asarray(f["quaternions"], np.float64),
            np.asarray(f["log_scales"], np.float64), np.asarray(f["intensity_logits"], np.float64), dims,
            np.asarray(f["lattice_index"], np.int64)))
        t = state["transforms"]
        q = np.asarray(t["quats"], np.float64).reshape(-1, 4)
        tr = np.asarray(t["translations"], np.float64).reshape(-1, 3)
        if q.shape[0] != self.k:
            raise ValueError(f"checkpoint has {q.shape[0]} slice transforms, trainer has {self.k}")
        self.tq = dv.to_dev(q, torch.float64, (self.k, 4))
        self.tt = dv.to_dev(tr, torch.float64, (self.k, 3))
        adam = state["adam"]
        self._reset_gauss_adam()
        if "positions" in adam:
            m = np.zeros((self.field.count, 11), np.float32)
            v = np.zeros_like(m)
            for name, key, lo, hi in self._GAUSS_GROUPS:
                g = adam[name]
                m[:, lo:hi] = np.asarray(g["m"][key], np.float64).reshape(self.field.count, hi - lo)
                v[:, lo:hi] = np.asarray(g["v"][key], np.float64).reshape(self.field.count, hi - lo)
            self.m.copy_(torch.from_numpy(np.ascontiguousarray(m.T)))
            self.v.copy_(torch.from_numpy(np.ascontiguousarray(v.T)))
            self.counters[0] = int(adam["positions"]["t"])
        self.tm.zero_()
        self.tv.zero_()
        self.counters[1] = 0
        if "transforms" in adam and self.k:
            g = adam["transforms"]
            self.tm[:self.k].copy_(torch.from_numpy(np.concatenate(
                [np.asarray(g["m"]["q"], np.float64), np.asarray(g["m"]["t"], np.float64)], axis=1)))
            self.tv[:self.k].copy_(torch.from_numpy(np.concatenate(
                [np.asarray(g["v"]["q"], np.float64), np.asarray(g["v"]["t"], np.float64)], axis=1)))
            self.counters[1] = int(g["t"])
        if "nrf" in state and cfg.use_nrf:
            from .nrf import ResidualField

            n = state["nrf"]
            self.nrf = ResidualField.from_numpy(n["weights"], n["biases"], int(n["frequency_bands"]))
            g = adam.get("nrf")
            params = self.nrf.parameter_arrays()
            self.nrf_m = {k: (dv.to_dev(np.asarray(g["m"][k]), torch.float32) if g else torch.zeros_like(a))
                          for k, a in params.items()}
            self.nrf_v = {k: (dv.to_dev(np.asarray(g["v"][k]), torch.float32) if g else torch.zeros_like(a))
                          for k, a in params.items()}
            self.nrf_t = int(g["t"]) if g else 0
        self.rng.bit_generator.state = state["rng_state"]
        self.iteration = int(state["iteration"])
        perm = state.get("perm")
        self._perm = None if perm is None else np.array(perm, dtype=np.int64)
        self._cursor = int(state["cursor"])
        self._bufs, self._bufs_key, self._graph = None, None, None
        return self

    def close(self):
        """Stop the permutation helper process (also done at garbage collection)."""
        if self._permuter is not None:
            self._permuter.close()
            self._permuter = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def step(self, sync=True):
        self._apply_milestones()
        all_idx, plan = self.draw_step()
        report = self._device_step(all_idx, plan, sync)
        self.iteration += 1
        self.reports.append(report)
        return report

    def step_pipelined(self):
        """Enqueue one optimizer step and return the LossReport of the step
        enqueued by the previous call (None on the first call; ``flush()``
        returns the last one).  The host-side batch draw and index upload of
        this step overlap the device running the previous step; every step
        still uploads its indices and reads back its losses."""
        self._apply_milestones()
        all_idx, plan = self.draw_step()
        prev = getattr(self, "_pending", None)
        self._device_step(all_idx, plan, sync=False)
        self._pending = self._enqueue_readback(self._bufs, plan)
        self.iteration += 1
        rep = None
        if prev is not None:
            rep = self._resolve(prev)
            self.reports.append(rep)
        return rep

    def flush(self):
        """Report of the last pipelined step (None if nothing is pending)."""
        prev, self._pending = getattr(self, "_pending", None), None
        if prev is None:
            return None
        rep = self._resolve(prev)
        self.reports.append(rep)
        return rep

    def _buffers(self, plan):
        """Step buffers for a StepPlan (or a plain rendered-point count)."""
        if not isinstance(plan, StepPlan):
            plan = StepPlan(int(plan), int(plan))
        g = self.field.resolution
        nrf_numel = self._nrf_numel() if self.nrf is not None else 0
        key = (self.field.count, g, plan.render, plan.gather, self.ntaps, self.k, nrf_numel)
        if self._bufs_key != key:
            self._bufs = None
            self._graph = None
            self._bufs = _StepBuffers(self.field.count, g, plan.render, plan.gather, self.ntaps, self.k, nrf_numel)
            self._bufs_key = key
        return self._bufs

    def load_indices(self, all_idx, plan):
        """Stage one step's pool indices (host array or device tensor) into the
        fixed index buffer, on the current stream."""
        B = self._buffers(plan)
        if isinstance(all_idx, torch.Tensor):
            B.idx.copy_(all_idx, non_blocking=True)
            return B
        k = B.slot
        B.slot ^= 1
        if B.idx_done[k] is not None:
            B.idx_done[k].synchronize()  # the slot's previous H2D copy has landed
        np.copyto(B.idx_host[k].numpy(), all_idx, casting="unsafe")
        cur = torch.cuda.current_stream()
        cs = self._copy_stream()
        if B.stage_free[k] is not None:
            cs.wait_event(B.stage_free[k])  # the D2D that read this landing slot has run
        with torch.cuda.stream(cs):
            B.idx_stage[k].copy_(B.idx_host[k], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
        B.idx_done[k] = ev
        cur.wait_event(ev)
        B.idx.copy_(B.idx_stage[k], non_blocking=True)
        free = torch.cuda.Event()
        free.record(cur)
        B.stage_free[k] = free
        return B

    def _copy_stream(self):
        return _stream("h2d")

    def _body(self, B, plan):
        N.check(N.lib().mg_gather_batch(N.ptr(B.idx), B.idx.numel(), N.ptr(self.src_coords), N.ptr(self.src_sids),
                                        N.ptr(self.src_tgt), N.ptr(B.coords), N.ptr(B.sids), N.ptr(B.tgt),
                                        dv.sptr()), "gather_batch")
        self._launch(B, plan)

    def run_device_step(self, plan):
        """Run one step on the indices already staged by ``load_indices``:
        replay the captured graph of this plan, or enqueue it eagerly."""
        B = self._bufs
        if self._graph is not None and self._graph_key == (plan, self.nrf_active):
            self._graph.replay()
        else:
            self._body(B, plan)

    def _device_step(self, all_idx, plan, sync):
        B = self.load_indices(all_idx, plan)
        # the step (incl. the NCCL all-reduce, whose communicator the eager
        # warm-up step initialises) is captured once per shape and replayed
        # (a gloo group cannot be captured: distributed gloo steps run eagerly)
        use_graph = self.graph and not self._gloo()
        if use_graph:
            key = (plan, self.nrf_active)
            if self._graph is None or self._graph_key != key:
                self._body(B, plan)  # eager warm-up of this shape (also lazily inits kernels)
                torch.cuda.synchronize()
                self._graph = None  # release the previous shape's graph (and its pool) first
                self._graph, self._graph_key = self._capture(lambda: self._body(B, plan)), key
                # the warm-up already performed this step's update; undo nothing: the
                # captured graph is replayed from the next step on.
            else:
                self._graph.replay()
        else:
            self._body(B, plan)
        if not sync:
            return LossReport(self.iteration, float("nan"), float("nan"), float("nan"), float("nan"),
                              self.field.resolution, self.nrf_active)
        return self._resolve(self._enqueue_readback(B, plan))

    def _gloo(self):
        if self.dist is None:
            return False
        import torch.distributed as tdist

        return tdist.get_backend(self.dist) == "gloo"

    def _capture(self, fn):
        """Capture ``fn``'s launches into a CUDA graph on a side stream.

        Not ``torch.cuda.graph``: its ``__enter__`` empties the device and
        pinned-host caching allocators every time (measured 0.1-0.7 s per
        capture after a large prior allocation, i.e. most of a desk-scale
        reconstruction's wall time across its milestone re-captures)."""
        cur = torch.cuda.current_stream()
        cs = _stream("capture")
        cs.wait_stream(cur)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(cs):
            g.capture_begin(pool=_graph_pool())
            try:
                fn()
            finally:
                g.capture_end()
        cur.wait_stream(cs)
        return g

    def _enqueue_readback(self, B, plan):
        """Async D2H of this step's loss sums and error flag into a pinned slot."""
        k = B.rslot
        B.rslot ^= 1
        if B.r_done[k] is not None:
            B.r_done[k].synchronize()
        B.scalars_host[k].copy_(B.scalars, non_blocking=True)
        B.err_host[k].copy_(B.err, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        B.r_done[k] = ev
        return (B, k, ev, self.iteration, plan, self.field.resolution, self.nrf_active)

    def _resolve(self, pending):
        """LossReport of a step whose readback was enqueued (waits for it)."""
        cfg = self.config
        B, k, ev, iteration, plan, res, nrf_on = pending
        ev.synchronize()
        sc = B.scalars_host[k].numpy().copy()
        err = int(B.err_host[k][0])
        if err:
            from .errors import DegenerateQuaternion

            raise DegenerateQuaternion("quaternion norm <= 1e-12 during training")
        data = float(sc[0])
        aniso = float(sc[1]) if cfg.use_aniso else 0.0
        ssim = 0.0
        if plan.hw is not None:
            h, w = plan.hw
            # weak sharding: one slice per rank, the loss is their mean
            nsl = self.world if (self.shard == "weak" and self.dist is not None) else 1
            ssim = 1.0 - float(sc[2]) / (nsl * (h - 10) * (w - 10))
        total = data + cfg.lambda_ssim * ssim + cfg.lambda_aniso * aniso
        if not np.isfinite(total):
            raise NonFiniteLoss(f"non-finite loss at iteration {iteration}")
        return LossReport(iteration, total, data, ssim, aniso, res, nrf_on)

    def _launch(self, B, plan):
        """Enqueue the whole step on the current stream (graph-capturable)."""
        cfg = self.config
        L = N.lib()
        st = dv.sptr()
        f = self.field
        n, g, r = f.count, f.resolution, cfg.block_radius
        bt = plan.render
        nb, hw = plan.nbl, plan.hw
        coords, sids, tgt = B.coords[:bt], B.sids[:bt], B.tgt[:bt]
        t = self.ntaps
        ns = bt * t
        ws = B.ws
        B.scalars.zero_()
        # Two independent chains run as parallel graph branches: the Gaussian
        # chain on a side stream (own workspace) while the main stream
        # transforms and bins the points; joined before the forward.
        main = torch.cuda.current_stream()
        side = self._side_stream()
        side.wait_stream(main)
        ss = N.stream_ptr(side)
        if B.ws_gauss is None:
            B.ws_gauss = dv.empty((L.mg_bin_workspace_bytes(n, g),), torch.uint8)
        # Gaussians: bin + activate (spatial.py:46-66, render.py:122-142)
        N.check(L.mg_bin_f32(N.ptr(f.positions), n, g, N.ptr(B.gkey), N.ptr(B.gorder), N.ptr(B.gstart),
                             N.ptr(B.ws_gauss), B.ws_gauss.numel(), ss), "bin")
        N.check(L.mg_activate(N.ptr(f.positions), N.ptr(f.quaternions), N.ptr(f.log_scales), N.ptr(f.logits), n,
                              N.ptr(B.gorder), N.ptr(B.grec), N.ptr(B.err), ss), "activate")
        N.check(L.mg_invert_permutation(N.ptr(B.gorder), n, N.ptr(B.ginv), ss), "invert_permutation")
        # points: transforms, PSF taps, bin
        if self.k:
            N.check(L.mg_quat_to_rot_f64(N.ptr(self.tq), self.k, N.ptr(B.rot), st))
        off = self._psf_off if self.psf is not None else None
        wts = self._psf_w if self.psf is not None else None
        dirs = self._psf_dirs if self.psf is not None else None
        N.check(L.mg_bin_points(N.ptr(coords), N.ptr(sids), bt, t, N.ptr(off), N.ptr(dirs), N.ptr(B.rot),
                                N.ptr(self.tt), self.k, g, N.ptr(B.pkey), N.ptr(B.pinv), N.ptr(B.pstart),
                                N.ptr(B.prec), N.ptr(B.xout), N.ptr(ws), ws.numel(), st), "bin_points")
        main.wait_stream(side)
        # forward with H (render_points, _kernels.py:24-70)
        N.check(L.mg_forward(N.ptr(B.grec), n, N.ptr(B.gstart), g, r, N.ptr(B.prec), N.ptr(B.pkey), N.ptr(B.pstart),
                             ns, 1, N.ptr(B.out4), N.ptr(B.cnt), N.ptr(ws), ws.numel(), st), "forward")
        N.check(L.mg_forward_finish(N.ptr(B.out4), N.ptr(B.cnt), N.ptr(B.pinv), bt, t, N.ptr(wts), None,
                                    N.ptr(B.pred), None, N.ptr(B.pairs), st), "finish")
        nrf_cache = None
        if self.nrf_active:
            from .nrf import nrf_forward_fused

            xc = self._centre_points(B, bt, t)
            _, nrf_cache = nrf_forward_fused(self.nrf, xc, pred_add=B.pred)  # pred += r in the kernel
        # losses (train.py:424-436): smooth-L1 mean over the GLOBAL batch
        N.check(L.mg_smooth_l1_scaled(N.ptr(B.pred), N.ptr(tgt), nb, 1.0 / plan.nb_norm, N.ptr(B.up),
                                      N.ptr(B.scalars[0:1]), st), "smooth_l1")
        if hw is not None:
            self._ssim(B, plan, tgt, st)
        # backward (render_backward): upstream -> point records, d_points; Gaussian-major pass
        N.check(L.mg_backward_points(None, N.ptr(B.up), bt, t, N.ptr(wts), N.ptr(B.pinv), N.ptr(B.out4),
                                     N.ptr(B.prec), N.ptr(B.dpts), st), "backward_points")
        # the per-slice transform reduction needs only d_points: it runs on the
        # side stream (own workspace) under the Gaussian-major backward
        if self.k:
            side.wait_stream(main)
            if B.ws_tr is None:
                B.ws_tr = dv.empty((L.mg_transform_grads_workspace_bytes(self.k),), torch.uint8)
            N.check(L.mg_transform_grads(N.ptr(B.dpts), N.ptr(coords), N.ptr(sids), bt, t, N.ptr(off), N.ptr(dirs),
                                         N.ptr(self.tq), self.k, N.ptr(B.scratch12), N.ptr(B.g7), 0, N.ptr(B.ws_tr),
                                         B.ws_tr.numel(), ss),
                    "transform_grads")
        N.check(L.mg_backward(N.ptr(B.grec), N.ptr(B.gkey), N.ptr(B.gstart), n, g, r, N.ptr(B.prec),
                              N.ptr(B.pstart), N.ptr(B.acc10), N.ptr(ws), ws.numel(), st), "backward")
        if self.k:
            main.wait_stream(side)
        ng = None
        if nrf_cache is not None:
            from .nrf import nrf_backward_fused

            # gradients land in the step's flat float32 buffer behind acc10
            # (all-reduced in place with it when distributed, then the fused Adam)
            gv = self._nrf_grad_views(B)
            nl = len(self.nrf.weights)
            gws, gbs = [gv[f"w{i}"] for i in range(nl)], [gv[f"b{i}"] for i in range(nl)]
            _, _, dp = nrf_backward_fused(self.nrf, self._centre_x, B.up, nrf_cache, out=(gws, gbs))
            ng = True
            if self.k:
                dp64 = dp.double().contiguous()
                N.check(L.mg_transform_grads(N.ptr(dp64), N.ptr(coords), N.ptr(sids), bt, 1, None, None,
                                             N.ptr(self.tq), self.k, N.ptr(B.scratch12), N.ptr(B.g7), 1,
                                             N.ptr(ws), ws.numel(), st),
                        "nrf_transform_grads")
        if self.dist is not None:
            self._allreduce(B)
        # updates (train.py:461-477): epilogue + aniso + Adam fused; transforms; NRF
        N.check(L.mg_counter_incr(N.ptr(self.counters), 2, st))
        hyper = self._hyper
        upd, perm = (L.mg_gauss_update, B.gorder) if _UPD_SORTED else (L.mg_gauss_update_inv, B.ginv)
        N.check(upd(N.ptr(B.acc10), N.ptr(perm), n, N.ptr(f.positions), N.ptr(f.quaternions),
                                  N.ptr(f.log_scales), N.ptr(f.logits), N.ptr(self.m), N.ptr(self.v),
                                  hyper.ctypes.data_as(N.P), 1 if cfg.use_aniso else 0, N.ptr(self.counters[0:1]),
                                  N.ptr(B.scalars[1:2]), st), "gauss_update")
        if self.k:
            N.check(L.mg_transform_adam(N.ptr(self.tq), N.ptr(self.tt), N.ptr(B.g7), N.ptr(self.tm), N.ptr(self.tv),
                                        self.k, cfg.lr_transform, cfg.adam_beta1, cfg.adam_beta2, cfg.adam_eps,
                                        N.ptr(self.counters[1:2]), st), "transform_adam")
        if ng is not None:
            self._nrf_adam(B)

    def _ssim(self, B, plan, tgt, st):
        """SSIM loss + upstream of the step's slice (ssim.py:59-122).

        Unsharded / weak: this rank rendered the whole slice.  Strong over N
        ranks: each rank rendered pixels [s_lo, s_hi); the full prediction is
        assembled by an all-reduce(sum) of zero-padded shares (exact: one
        non-zero term per pixel), every rank evaluates the identical SSIM
        gradient and keeps its own pixels' upstream; rank 0 alone reports the
        SSIM sum."""
        L = N.lib()
        h, w = plan.hw
        nb = plan.nbl
        need = L.mg_ssim_workspace_bytes(h, w)
        if B.ssim_ws is None or B.ssim_ws.numel() < need:
            B.ssim_ws = dv.empty((need,), torch.uint8)
        weak = self.dist is not None and self.shard == "weak"
        scale = self.config.lambda_ssim / (self.world if weak else 1)
        if not plan.full_slice:
            N.check(L.mg_ssim_loss_grad(N.ptr(B.pred[nb:]), N.ptr(tgt[nb:]), h, w, scale, N.ptr(B.up[nb:]),
                                        N.ptr(B.scalars[2:3]), N.ptr(B.ssim_ws), B.ssim_ws.numel(), st), "ssim")
            return
        import torch.distributed as tdist

        hw_n = h * w
        if B.slice_pred is None or B.slice_pred.numel() != hw_n:
            B.slice_pred = dv.empty((hw_n,), torch.float32)
            B.slice_up = dv.empty((hw_n,), torch.float32)
        B.slice_pred.zero_()
        B.slice_pred[plan.s_lo:plan.s_hi].copy_(B.pred[nb:])
        tdist.all_reduce(B.slice_pred, op=tdist.ReduceOp.SUM, group=self.dist)
        full_tgt = B.tgt[plan.render:plan.render + hw_n]
        acc = B.scalars[2:3] if self.rank == 0 else B.scalars[3:4]
        N.check(L.mg_ssim_loss_grad(N.ptr(B.slice_pred), N.ptr(full_tgt), h, w, scale, N.ptr(B.slice_up),
                                    N.ptr(acc), N.ptr(B.ssim_ws), B.ssim_ws.numel(), st), "ssim")
        B.up[nb:].copy_(B.slice_up[plan.s_lo:plan.s_hi])

    def _side_stream(self):
        return _stream("side")

    def _centre_points(self, B, bt, t):
        """Transformed (un-shifted) sample positions for the NRF (train.py:414-419)."""
        if t == 1:
            x = B.xout.view(bt, 3)
        else:
            c = int(np.argmin(np.abs(np.asarray(self.psf.offsets))))
            x = B.xout.view(bt, t, 3)[:, c, :]
        self._centre_x = x.to(torch.float32).contiguous()
        return self._centre_x

    @property
    def nrf_t(self):
        """NRF Adam step count (kept on the device so the step graph replays it)."""
        t = getattr(self, "_nrf_tdev", None)
        return 0 if t is None else int(t.item())

    @nrf_t.setter
    def nrf_t(self, value):
        self._nrf_tdev = torch.full((), float(value), dtype=torch.float64, device=dv.device())

    def _nrf_numel(self):
        return sum(v.numel() for v in self.nrf.parameter_arrays().values())

    def _nrf_grad_views(self, B):
        """One view per NRF parameter into the tail of B's flat float32 buffer."""
        params = self.nrf.parameter_arrays()
        flat = B.nrf_grad_flat()
        if getattr(B, "nrf_views", None) is None:
            views, off = {}, 0
            for k, v in params.items():
                views[k] = flat[off:off + v.numel()].view(v.shape)
                off += v.numel()
            B.nrf_views = views
        return B.nrf_views

    def _nrf_adam(self, B):
        """AdamState.step("nrf", ...) (train.py:251-271): one launch over all
        NRF tensors, with the device step counter read and advanced in the
        kernel so the update replays inside the graph."""
        import ctypes

        cfg = self.config
        params = self.nrf.parameter_arrays()
        keys = list(params)
        gv = self._nrf_grad_views(B)

        def arr(ts):
            return (ctypes.c_void_p * len(ts))(*[t.data_ptr() for t in ts])

        ps, gs = arr([params[k] for k in keys]), arr([gv[k] for k in keys])
        ms, vs = arr([self.nrf_m[k] for k in keys]), arr([self.nrf_v[k] for k in keys])
        sizes = (ctypes.c_int64 * len(keys))(*[params[k].numel() for k in keys])
        N.check(N.lib().mg_nrf_adam(ctypes.addressof(gs), ctypes.addressof(ps), ctypes.addressof(ms),
                                    ctypes.addressof(vs), ctypes.addressof(sizes), len(keys), N.ptr(self._nrf_tdev),
                                    cfg.lr_nrf, cfg.adam_beta1, cfg.adam_beta2, cfg.adam_eps, dv.sptr()), "nrf_adam")

    def _allreduce(self, B):
        """All-reduce(sum) in place of the step's two flat partial-sum buffers:
        acc10 (+ the NRF gradients while the NRF is active) in float32, the
        loss partials and per-slice transform gradients in float64 (parallel.py)."""
        import torch.distributed as tdist

        n32 = B.flat32.numel() if self.nrf_active else 10 * self.field.count
        tdist.all_reduce(B.flat32[:n32], op=tdist.ReduceOp.SUM, group=self.dist)
        tdist.all_reduce(B.flat64, op=tdist.ReduceOp.SUM, group=self.dist)

    def run(self, iterations=None):
        target = self.config.total_iters if iterations is None else self.iteration + iterations
        while self.iteration < target:
            self.step()
        return self.reports

    # -- inference (train.py:509-512, render.py:379-408) -------------------------
    def render_volume(self, dims, bounds, include_nrf=True, dist=None, gather=True):
        """Inference sampling of the trained field (train.py:509-512,
        render.py:379-408) on a node-inclusive grid, clipped to [0, 1].

        With ``dist`` (a torch.distributed group) every rank
        samples only its z-slab [i0, i1) of axis 0 (parallel.slab_ranges), so
        the sampling has no collective.  ``gather=True`` then all-gathers the
        slabs (one collective of the padded slabs) and every rank returns the
        whole Volume; ``gather=False`` returns this rank's slab as a Volume
        whose origin is the slab's first plane."""
        from .core import Volume
        from .parallel import slab_ranges
        from .render import grid_coordinates

        f = self.field
        g, r = f.resolution, self.config.block_radius
        B = self._buffers(1)
        L = N.lib()
        N.check(L.mg_bin_f32(N.ptr(f.positions), f.count, g, N.ptr(B.gkey), N.ptr(B.gorder), N.ptr(B.gstart),
                             N.ptr(B.ws), B.ws.numel(), dv.sptr()), "bin")
        N.check(L.mg_activate(N.ptr(f.positions), N.ptr(f.quaternions), N.ptr(f.log_scales), N.ptr(f.logits),
                              f.count, N.ptr(B.gorder), N.ptr(B.grec), N.ptr(B.err), dv.sptr()), "activate")
        dims = tuple(int(d) for d in dims)
        axes, spacing = grid_coordinates(dims, bounds)
        rank, world = 0, 1
        if dist is not None:
            import torch.distributed as tdist

            rank, world = tdist.get_rank(dist), tdist.get_world_size(dist)
        slabs = slab_ranges(dims[0], world)
        i0, i1 = slabs[rank]
        res = None
        if include_nrf and self.nrf_active and i1 > i0:
            from .nrf import nrf_forward_device

            gx, gy, gz = np.meshgrid(axes[0][i0:i1], axes[1], axes[2], indexing="ij")
            pts = dv.to_dev(np.stack([gx.ravel(), gy.ravel(), gz.ravel()], 1), torch.float32)
            res = nrf_forward_device(self.nrf, pts).reshape((i1 - i0,) + dims[1:])
        out = sample_volume_device(B.grec, f.count, B.gstart, g, r, dims, bounds, i0=i0, i1=i1, residual=res)
        if world > 1 and gather:
            import torch.distributed as tdist

            pmax = max(b - a for a, b in slabs)
            pad = torch.zeros((pmax,) + dims[1:], dtype=torch.float32, device=out.device)
            pad[:i1 - i0].copy_(out)
            parts = [torch.empty_like(pad) for _ in range(world)]
            tdist.all_gather(parts, pad, group=dist)
            out = torch.cat([parts[q][:b - a] for q, (a, b) in enumerate(slabs)])
            i0 = 0
        origin = np.array([axes[0][min(i0, dims[0] - 1)], axes[1][0], axes[2][0]])
        return Volume(data=dv.to_host(out).astype(np.float64), spacing=spacing, origin=origin)

    def transforms_host(self):
        return TransformSet(dv.to_host(self.tq), dv.to_host(self.tt))


# ---------------------------------------------------------------------------
# host-facing loss helpers (train.py:108-120, ssim.py:82-122), device-computed
# ---------------------------------------------------------------------------


def smooth_l1_loss_grad(pred, target):
    """(mean Huber loss, d/dpred) in float64 on the device (mg_smooth_l1_f64):
    the host-level API takes and returns float64 like the reference."""
    p = dv.to_dev(np.asarray(pred, dtype=np.float64).ravel(), torch.float64)
    t = dv.to_dev(np.asarray(target, dtype=np.float64).ravel(), torch.float64)
    up = dv.empty(p.shape, torch.float64)
    acc = dv.zeros((1,), torch.float64)
    N.check(N.lib().mg_smooth_l1_f64(N.ptr(p), N.ptr(t), p.numel(), N.ptr(up), N.ptr(acc), dv.sptr()),
            "smooth_l1_f64")
    return float(acc.item()), dv.to_host(up)


def ssim_loss_grad(pred, target):
    """(1 - mean SSIM, d/dpred) of an (H, W) slice, float64 on the device
    (ssim.ssim_loss_grad)."""
    from .ssim import ssim_loss_grad as _ssim

    return _ssim(pred, target)


# ---------------------------------------------------------------------------
# The reference's host-level training API (train.py:108-290), same names and
# semantics, computed by the device kernels: float64 numpy in and out.
# ---------------------------------------------------------------------------


@dataclass
class SliceGrid:
    """Full native in-plane sample grid of one acquired slice (train.py:282-290)."""

    coords: np.ndarray  # (H * W, 3), C-order matching target.ravel()
    target: np.ndarray  # (H, W)
    slice_id: int


def smooth_l1(pred, target):
    """Huber loss (delta 1), mean over the batch (train.py:108-113); mg_smooth_l1."""
    return smooth_l1_loss_grad(pred, target)[0]


def smooth_l1_grad(pred, target):
    """d(mean Huber)/dpred (train.py:116-120); mg_smooth_l1."""
    return smooth_l1_loss_grad(pred, target)[1].reshape(np.shape(pred))


def aniso_loss_grad(field, lambda_ratio):
    """(loss, d loss / d log_scales) of the anisotropy hinge (train.py:128-147),
    float64 on the device (mg_aniso_loss_grad_f64)."""
    s = dv.to_dev(np.asarray(field.log_scales, dtype=np.float64).reshape(-1, 3), torch.float64)
    n = s.shape[0]
    grad = dv.empty((n, 3), torch.float64)
    acc = dv.zeros((1,), torch.float64)
    N.check(N.lib().mg_aniso_loss_grad_f64(N.ptr(s), n, float(lambda_ratio), N.ptr(grad), N.ptr(acc), dv.sptr()),
            "aniso_loss_grad")
    return float(acc.item()), dv.to_host(grad)


def aniso_loss(field, lambda_ratio):
    """train.py:123-125."""
    return aniso_loss_grad(field, lambda_ratio)[0]


def progressive_upsample(field, new_resolution):
    """train.py:157-218 on the device (mg_upsample_f64): trilinear logits and
    log-scales, sign-aligned NLERP quaternions, positions on the new lattice,
    in float64 like the reference (the trainer's own float32 state uses
    progressive_upsample_device)."""
    from .core import GaussianField

    new_r = int(new_resolution)
    old_r = int(field.lattice_dims[0])
    if new_r < old_r:
        raise ShrinkNotAllowed(f"cannot shrink lattice {old_r} -> {new_r}")
    li = np.asarray(field.lattice_index, dtype=np.int64)
    node_of = np.empty(field.count, np.int32)
    node_of[(li[:, 0] * old_r + li[:, 1]) * old_r + li[:, 2]] = np.arange(field.count, dtype=np.int32)
    n = new_r ** 3
    out = [dv.empty((n, c), torch.float64) for c in (3, 4, 3, 1)]
    src = [dv.to_dev(field.quaternions, torch.float64), dv.to_dev(field.log_scales, torch.float64),
           dv.to_dev(field.intensity_logits, torch.float64), dv.to_dev(node_of, torch.int32)]
    N.check(N.lib().mg_upsample_f64(*[N.ptr(t) for t in src], old_r, new_r, *[N.ptr(o) for o in out], dv.sptr()),
            "upsample_f64")
    _, q, sc, lg = (dv.to_host(o) for o in out)
    return GaussianField(lattice_node_positions(new_r), q, sc, lg.reshape(n), (new_r, new_r, new_r),
                         lattice_node_index(new_r))


def init_field(cloud, resolution, logit_eps=1e-4):
    """Uniform lattice field with logit(mean sample intensity) per cell
    (train.py:221-236) on the device (mg_cell_keys_f64 + segmented float64
    means)."""
    from .core import GaussianField

    r = int(resolution)
    coords = dv.to_dev(np.asarray(cloud.coords, np.float64).reshape(-1, 3), torch.float64)
    lg = _init_logits(coords, dv.to_dev(np.asarray(cloud.intensities, np.float64).ravel(), torch.float64), r,
                      logit_eps)
    n = r ** 3
    q = np.zeros((n, 4))
    q[:, 0] = 1.0
    return GaussianField(lattice_node_positions(r), q, np.full((n, 3), np.log(1.0 / r)), dv.to_host(lg), (r, r, r),
                         lattice_node_index(r))


class AdamState:
    """Named parameter groups with first/second moments and step counters
    (train.py:239-279).  ``step`` updates the caller's float64 arrays in place;
    the update runs in float64 on the device (mg_adam_f64)."""

    def __init__(self, beta1=0.9, beta2=0.999, eps=1e-8):
        self.beta1, self.beta2, self.eps = beta1, beta2, eps
        self.groups = {}

    def reset_group(self, name):
        self.groups.pop(name, None)

    def step(self, name, params, grads, lr):
        g = self.groups.setdefault(name, {"t": 0, "m": {}, "v": {}})
        g["t"] += 1
        t = g["t"]
        L = N.lib()
        for key, param in params.items():
            if key not in g["m"]:
                g["m"][key] = np.zeros_like(param, dtype=np.float64)
                g["v"][key] = np.zeros_like(param, dtype=np.float64)
            p = dv.to_dev(param, torch.float64)
            gr = dv.to_dev(np.asarray(grads[key], dtype=np.float64), torch.float64)
            m = dv.to_dev(g["m"][key], torch.float64)
            v = dv.to_dev(g["v"][key], torch.float64)
            N.check(L.mg_adam_f64(N.ptr(p), N.ptr(gr), N.ptr(m), N.ptr(v), p.numel(), t, float(lr), self.beta1,
                                  self.beta2, self.eps, dv.sptr()), "adam")
            param[...] = dv.to_host(p).reshape(param.shape)
            g["m"][key][...] = dv.to_host(m).reshape(param.shape)
            g["v"][key][...] = dv.to_host(v).reshape(param.shape)

    def state_dict(self):
        return {name: {"t": g["t"], "m": {k: a.copy() for k, a in g["m"].items()},
                       "v": {k: a.copy() for k, a in g["v"].items()}} for name, g in self.groups.items()}

    def load_state_dict(self, state):
        self.groups = {name: {"t": int(g["t"]), "m": {k: np.array(a, dtype=np.float64) for k, a in g["m"].items()},
                              "v": {k: np.array(a, dtype=np.float64) for k, a in g["v"].items()}}
                       for name, g in state.items()}


from .strict_train import StrictTrainer  # noqa: E402,F401  (strict-float64 parity path)
