"""Strict-float64 training: the reference Trainer's step
(/root/reference/pkg/src/mgauss/train.py:321-491) evaluated by the float64
device kernels in the reference's operation order, so a strict run follows
the reference's trajectory to rounding level over the whole schedule
(progressive upsample, SSIM, NRF, Adam).

This is the parity path, not the fast path: every step stages float64 host
state through the device kernels (mg_block_forward_f64 / _backward_f64,
mg_smooth_l1_f64, mg_ssim_loss_grad_f64, mg_nrf_forward_f64 / _backward_f64,
mg_aniso_loss_grad_f64, mg_adam_f64, mg_upsample_f64, the CSR builder) like
the reference's numpy arrays move through its numba kernels.  The float32
`Trainer` is the production path; the two differ by float32 rounding, which
training amplifies chaotically (DESIGN.md (c), long-run paragraph) -- this
class shows that what remains after removing that rounding is the
reference's own result.
"""

from __future__ import annotations

import contextlib
import time
from types import SimpleNamespace

import numpy as np
import torch

from . import _device as dv
from . import _native as N
from . import render
from .core import TransformSet
from .errors import NonFiniteLoss
from .nrf import ResidualField64, nrf_backward_f64, nrf_forward_cached_f64
from .spatial import build, build_device


@contextlib.contextmanager
def strict_fp64():
    """Select the float64 kernels for the duration of the block."""
    prev = render.get_strict_fp64()
    render.set_strict_fp64(True)
    try:
        yield
    finally:
        render.set_strict_fp64(prev)


class StrictTrainer:
    """Same constructor and `step()` contract as the reference Trainer
    (train.py:321-347, 385-491); state lives in float64 numpy arrays
    (`field`, `transforms`, `nrf`, `adam`) exactly as the reference holds it."""

    def __init__(self, cloud, transforms: TransformSet, config, slice_grids=None):
        from .train import AdamState, init_field

        config.validate()
        if config.use_ssim and not slice_grids:
            raise ValueError("use_ssim requires slice sample grids")
        self.config = config
        self.cloud = cloud
        self.transforms = TransformSet(np.array(transforms.quats, dtype=np.float64),
                                       np.array(transforms.translations, dtype=np.float64))
        self.slice_grids = list(slice_grids or [])
        batch_ss, nrf_ss = np.random.SeedSequence(config.seed).spawn(2)
        self.rng = np.random.default_rng(batch_ss)
        self.nrf = ResidualField64.create(np.random.default_rng(nrf_ss)) if config.use_nrf else None
        start = config.resolution_at(0) if config.use_progressive else config.final_resolution
        with strict_fp64():
            self.field = init_field(cloud, start)
        self.grid = build(self.field, start, config.block_radius)
        self.adam = AdamState(config.adam_beta1, config.adam_beta2, config.adam_eps)
        self.iteration = 0
        self._perm = None
        self._cursor = 0
        self.reports = []

    # the reference's batch stream (train.py:349-366): host PCG64 permutations
    def _next_batch(self):
        m = self.cloud.coords.shape[0]
        b = min(self.config.batch_points, m)
        if b == m:
            return np.arange(m)
        parts, need = [], b
        while need > 0:
            if self._perm is None or self._cursor >= m:
                self._perm = self.rng.permutation(m)
                self._cursor = 0
            take = min(need, m - self._cursor)
            parts.append(self._perm[self._cursor:self._cursor + take])
            self._cursor += take
            need -= take
        return np.concatenate(parts) if len(parts) > 1 else parts[0]

    @property
    def nrf_active(self):
        return self.config.use_nrf and self.iteration >= self.config.nrf_activation_iter

    def _apply_milestones(self):
        from .train import progressive_upsample

        if not self.config.use_progressive:
            return
        for it, res in self.config.resolution_schedule:
            if it == self.iteration and res > self.field.lattice_dims[0]:
                with strict_fp64():
                    self.field = progressive_upsample(self.field, res)
                self.grid = build(self.field, res, self.config.block_radius)
                for group in ("positions", "quaternions", "log_scales", "intensity_logits"):
                    self.adam.reset_group(group)

    @staticmethod
    def _cell_order(coords, g):
        """Stable sort of the batch by flat cell key (train.py:394-399) -- the
        builder's counting sort, bit-identical to numpy's stable argsort."""
        d = build_device(dv.to_dev(coords, torch.float64), g)
        return dv.to_host(d["order"]).astype(np.int64)

    def step(self, sync=True):
        from .train import LossReport, aniso_loss_grad, smooth_l1_loss_grad, ssim_loss_grad

        cfg = self.config
        self._apply_milestones()
        with strict_fp64():
            idx = self._next_batch()
            idx = idx[self._cell_order(self.cloud.coords[idx], self.grid.grid_resolution)]
            batch = np.ascontiguousarray(self.cloud.coords[idx], dtype=np.float64)
            sids = np.ascontiguousarray(self.cloud.slice_ids[idx], dtype=np.int64)
            targets = np.asarray(self.cloud.intensities[idx], dtype=np.float64)
            nb = batch.shape[0]

            prepared = render.activated_parameters(self.field)
            fwd = render.render_points(self.field, self.grid, self.transforms, SimpleNamespace(coords=batch, slice_ids=sids),
                                       prepared=prepared)
            coords_all, sids_all, points_all = batch, sids, fwd.points
            sg = None
            if cfg.use_ssim:
                sg = self.slice_grids[int(self.rng.integers(len(self.slice_grids)))]
                sl_coords = np.ascontiguousarray(np.asarray(sg.coords, dtype=np.float64).reshape(-1, 3))
                sl_sids = np.full(sl_coords.shape[0], sg.slice_id, dtype=np.int64)
                sl_fwd = render.render_points(self.field, self.grid, self.transforms,
                                              SimpleNamespace(coords=sl_coords, slice_ids=sl_sids), prepared=prepared)
                coords_all = np.concatenate([batch, sl_coords])
                sids_all = np.concatenate([sids, sl_sids])
                points_all = np.concatenate([fwd.points, sl_fwd.points])

            residual = cache = None
            if self.nrf_active:
                r_d, cache = nrf_forward_cached_f64(self.nrf, dv.to_dev(points_all, torch.float64))
                residual = dv.to_host(r_d)

            pred = fwd.intensities if residual is None else fwd.intensities + residual[:nb]
            data_loss, upstream = smooth_l1_loss_grad(pred, targets)
            ssim_val = 0.0
            if cfg.use_ssim:
                sl_pred = sl_fwd.intensities if residual is None else sl_fwd.intensities + residual[nb:]
                target = np.asarray(sg.target, dtype=np.float64)
                ssim_val, dslice = ssim_loss_grad(sl_pred.reshape(target.shape), target)
                upstream = np.concatenate([upstream, cfg.lambda_ssim * dslice.ravel()])
            aniso_val, d_aniso = 0.0, None
            if cfg.use_aniso:
                aniso_val, d_aniso = aniso_loss_grad(self.field, cfg.lambda_ratio)
            total = data_loss + cfg.lambda_ssim * ssim_val + cfg.lambda_aniso * aniso_val
            if not np.isfinite(total):
                raise NonFiniteLoss(f"non-finite loss at iteration {self.iteration}")

            grads = render.render_backward(self.field, self.grid, self.transforms,
                                           SimpleNamespace(coords=coords_all, slice_ids=sids_all), upstream,
                                           prepared=prepared)
            d_transform = grads.d_transform_params
            ng = None
            if self.nrf_active:
                dws, dbs, dp = nrf_backward_f64(cache, dv.to_dev(upstream, torch.float64))
                ng = (dws, dbs)
                d_transform = d_transform + render.transform_grads_from_points(self.transforms, coords_all, sids_all,
                                                                               dv.to_host(dp))
            d_log_scales = grads.d_log_scales
            if d_aniso is not None:
                d_log_scales = d_log_scales + cfg.lambda_aniso * d_aniso

            a = self.adam
            a.step("positions", {"p": self.field.positions}, {"p": grads.d_positions}, cfg.lr_position)
            a.step("quaternions", {"q": self.field.quaternions}, {"q": grads.d_quaternions}, cfg.lr_rotation)
            a.step("log_scales", {"s": self.field.log_scales}, {"s": d_log_scales}, cfg.lr_scale)
            a.step("intensity_logits", {"a": self.field.intensity_logits}, {"a": grads.d_intensity_logits},
                   cfg.lr_intensity)
            a.step("transforms", {"q": self.transforms.quats, "t": self.transforms.translations},
                   {"q": d_transform[:, :4], "t": d_transform[:, 4:]}, cfg.lr_transform)
            if ng is not None:
                grads_nrf = {}
                for li, (dw, db) in enumerate(zip(*ng)):
                    grads_nrf[f"w{li}"], grads_nrf[f"b{li}"] = dw, db
                a.step("nrf", self.nrf.parameter_arrays(), grads_nrf, cfg.lr_nrf)

            self.grid = build(self.field, self.grid.grid_resolution, cfg.block_radius)
        rep = LossReport(iteration=self.iteration, total=float(total), data=float(data_loss), ssim=float(ssim_val),
                         aniso=float(aniso_val), resolution=int(self.field.lattice_dims[0]),
                         nrf_active=self.nrf_active)
        self.iteration += 1
        self.reports.append(rep)
        return rep

    def render_volume(self, dims, bounds=((-1.0, -1.0, -1.0), (1.0, 1.0, 1.0)), include_nrf=True, chunk=65536):
        """sample_volume (render.py:379-408) in float64: Gaussian part plus
        the float64 residual, clipped to [0, 1]."""
        from .core import Volume

        dims = tuple(int(d) for d in dims)
        axes, spacing = render.grid_coordinates(dims, bounds)
        gx, gy, gz = np.meshgrid(axes[0], axes[1], axes[2], indexing="ij")
        pts = np.stack([gx.ravel(), gy.ravel(), gz.ravel()], axis=1)
        out = np.empty(pts.shape[0])
        with strict_fp64():
            for c0 in range(0, pts.shape[0], chunk):
                c1 = min(pts.shape[0], c0 + chunk)
                blk = np.ascontiguousarray(pts[c0:c1])
                vals = render.render_points(self.field, self.grid, None, blk).intensities
                if include_nrf and self.nrf is not None and self.nrf_active:
                    r_d, _ = nrf_forward_cached_f64(self.nrf, dv.to_dev(blk, torch.float64))
                    vals = vals + dv.to_host(r_d)
                out[c0:c1] = vals
        return Volume(data=np.clip(out, 0.0, 1.0).reshape(dims), spacing=spacing,
                      origin=np.array([axes[0][0], axes[1][0], axes[2][0]]))

    def close(self):
        pass
