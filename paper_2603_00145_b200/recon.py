"""End-to-end reconstruction on the device trainer: the caller of the hot path
that BASELINE's "recon s to PSNR" measures.

`reconstruct` follows the reference's run_reconstruction
(/root/reference/pkg/src/mgauss/cli.py:111-141) from the devoxelised cloud
on: train for ``total_iters`` steps, sample the reconstruction on the target
grid (``Trainer.render_volume``) and scale it back to stack intensities.
`psnr` is metrics.py:25-37.  The acquisition simulator and devoxeliser are
outside the hot path (SURVEY §8 scope); `load_recon_fixture` reads the cloud
the reference produced for configs/desk64.cfg (tests/golden/make_recon.py).
"""

from __future__ import annotations

import math
import time
from types import SimpleNamespace

import numpy as np


def psnr(pred, gt, peak=1.0):
    """10 log10(peak^2 / MSE) in dB (+inf for identical volumes)."""
    p = np.asarray(pred, dtype=np.float64)
    g = np.asarray(gt, dtype=np.float64)
    if p.shape != g.shape:
        raise ValueError(f"shape mismatch {p.shape} vs {g.shape}")
    mse = float(np.mean((p - g) ** 2))
    return math.inf if mse == 0.0 else 10.0 * math.log10(peak * peak / mse)


def reconstruct(trainer, dims, first, last, intensity_scale, progress=None):
    """Run ``trainer`` to its ``total_iters`` and sample the node-inclusive
    ``dims`` grid from normalised ``first`` to ``last``.

    Returns (world-intensity volume as float32, training seconds, total seconds)."""
    import torch

    t0 = time.perf_counter()
    while trainer.iteration < trainer.config.total_iters:
        rep = trainer.step(sync=progress is not None)
        if progress is not None:
            progress(rep)
    torch.cuda.synchronize()
    t_train = time.perf_counter() - t0
    vol = trainer.render_volume(tuple(int(d) for d in dims), bounds=(tuple(first), tuple(last)))
    out = (vol.data * float(intensity_scale)).astype(np.float32)
    return out, t_train, time.perf_counter() - t0


def load_recon_fixture(path, long_path=None):
    """(cloud, TransformSet, slice grids, TrainConfig, target) from a
    make_recon.py fixture; ``long_path`` (make_recon.py --long) replaces the
    schedule, length and the reference's results with those of the
    4,000-iteration run on the same data."""
    from .core import TransformSet
    from .train import TrainConfig

    z = np.load(path)
    cloud = SimpleNamespace(coords=z["coords"], intensities=z["intensities"], slice_ids=z["slice_ids"])
    grids = []
    for (h, w), sid in zip(z["grid_shapes"], z["grid_ids"]):
        rows = z["slice_ids"] == sid
        grids.append(SimpleNamespace(coords=z["coords"][rows].reshape(int(h), int(w), 3),
                                     target=z["intensities"][rows].reshape(int(h), int(w)), slice_id=int(sid)))
    cfg = TrainConfig(resolution_schedule=tuple((int(i), int(r)) for i, r in z["schedule"]),
                      nrf_activation_iter=int(z["nrf_activation_iter"]), total_iters=int(z["total_iters"]),
                      batch_points=int(z["batch_points"]), seed=int(z["seed"]))
    target = SimpleNamespace(dims=tuple(int(d) for d in z["dims"]), first=z["first"], last=z["last"],
                             intensity_scale=float(z["intensity_scale"]), gt=z["gt"],
                             ref_psnr_db=float(z["psnr_db"]), ref_seconds=float(z["runtime_s"]),
                             ref_threads=int(z["threads"]), ref_losses=z["losses"])
    if long_path is not None:
        zl = np.load(long_path)
        cfg = TrainConfig(resolution_schedule=tuple((int(i), int(r)) for i, r in zl["schedule"]),
                          nrf_activation_iter=int(zl["nrf_activation_iter"]), total_iters=int(zl["total_iters"]),
                          batch_points=int(zl["batch_points"]), seed=int(zl["seed"]))
        target.ref_psnr_db, target.ref_seconds = float(zl["psnr_db"]), float(zl["runtime_s"])
        target.ref_threads, target.ref_losses = int(zl["threads"]), zl["losses"]
    return cloud, TransformSet(z["t_quats"], z["t_trans"]), grids, cfg, target
