"""Reference desk-scale reconstruction (configs/desk64.cfg) -> tests/golden/recon_desk64.npz.

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tests/golden/make_recon.py [threads] [--long]

--long: the same data with the reference's default training length (4,000
iterations, train.py:56) -- lattice 0:16,500:24,1000:32,1800:40,2800:48, NRF
from 1,600 -- written to recon_desk64_long.npz (trajectory, PSNR, runtime and
the reconstructed volume only; the inputs are recon_desk64.npz's, which the
same seed reproduces).

Runs the REFERENCE pipeline exactly as `mgauss reconstruct` does
(cli.py:111-141: simulate, devoxelize, estimated transforms, slice grids,
Trainer for total_iters, render_volume on the target grid, PSNR against the
phantom, cli.py:197-200) and stores its inputs, the phantom, the final PSNR,
the loss trajectory and the runtime.  The slice grids are not stored: with
foreground_threshold = -1 every pixel is a sample, so grid k is the cloud rows
of slice k reshaped to (H, W) (asserted below).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from mgauss import io as mio  # noqa: E402
from mgauss import render  # noqa: E402
from mgauss.cli import _target_grid, simulate_stacks  # noqa: E402
from mgauss.metrics import psnr  # noqa: E402
from mgauss.simdata import build_slice_grids, devoxelize, normalized_transforms  # noqa: E402
from mgauss.train import Trainer  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
CFG = "/root/reference/pkg/configs/desk64.cfg"


LONG = dict(total_iters=4000, resolution_schedule=((0, 16), (500, 24), (1000, 32), (1800, 40), (2800, 48)),
            nrf_activation_iter=1600)


def main():
    import dataclasses

    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    long_run = "--long" in sys.argv
    perturb = None
    if "--perturb" in sys.argv:  # rounding-level perturbation of the samples (tools/recon_ensemble.py's)
        perturb = int(args.pop(-1))
    threads = int(args[0]) if args else 1
    render.set_num_threads(threads)
    bundle = mio.load_config(CFG)
    if long_run:
        bundle = dataclasses.replace(bundle, train=dataclasses.replace(bundle.train, **LONG))
    gt, stacks = simulate_stacks(bundle.sim, bundle.train.seed)
    cloud = devoxelize(stacks, bundle.sim.foreground_threshold)
    ts = normalized_transforms(stacks, cloud.world_map, "estimated")
    grids = build_slice_grids(stacks, cloud.world_map, cloud.intensity_scale)
    if perturb is not None:
        cloud.intensities = cloud.intensities * (1.0 + 1e-7 * np.random.default_rng(perturb).normal(
            size=cloud.intensities.shape))
        for g in grids:
            g.target = cloud.intensities[cloud.slice_ids == g.slice_id].reshape(np.asarray(g.target).shape)
    for g in grids if perturb is None else []:  # grid k == cloud rows of slice k (foreground threshold -1)
        rows = cloud.slice_ids == g.slice_id
        assert np.array_equal(cloud.coords[rows], np.asarray(g.coords).reshape(-1, 3))
        assert np.array_equal(cloud.intensities[rows], np.asarray(g.target).ravel())
    tr = Trainer(cloud, ts, bundle.train, slice_grids=grids)
    losses = []
    t0 = time.perf_counter()
    while tr.iteration < bundle.train.total_iters:
        rep = tr.step()
        losses.append([rep.total, rep.data, rep.ssim, rep.aniso])
        if tr.iteration % 100 == 0:
            print(tr.iteration, rep.to_line(), f"{time.perf_counter() - t0:.1f}s", flush=True)
    runtime = time.perf_counter() - t0
    dims, spacing, origin = _target_grid(stacks, bundle.recon)
    first = cloud.world_map.to_normalized(origin)
    last = cloud.world_map.to_normalized(origin + (np.array(dims) - 1) * spacing)
    vol = tr.render_volume(dims, bounds=(first, last))
    pred = (vol.data * cloud.intensity_scale).astype(np.float32).astype(np.float64)
    db = psnr(pred, gt.data.astype(np.float32).astype(np.float64))
    print(f"PSNR {db:.4f} dB, {runtime:.1f} s on {threads} thread(s)")
    if perturb is not None:
        with open(os.path.join(OUT, "recon_desk64_long_perturbed.txt"), "a") as fh:
            fh.write(f"{perturb} {db:.6f} {runtime:.1f} {threads}\n")
        return
    if long_run:
        np.savez_compressed(
            os.path.join(OUT, "recon_desk64_long.npz"), psnr_db=db, runtime_s=runtime, threads=threads,
            losses=np.array(losses), recon=pred.astype(np.float32), schedule=np.array(LONG["resolution_schedule"]),
            nrf_activation_iter=LONG["nrf_activation_iter"], total_iters=LONG["total_iters"],
            batch_points=bundle.train.batch_points, seed=bundle.train.seed)
        return
    np.savez_compressed(
        os.path.join(OUT, "recon_desk64.npz"),
        coords=cloud.coords, intensities=cloud.intensities, slice_ids=cloud.slice_ids,
        intensity_scale=cloud.intensity_scale, t_quats=ts.quats, t_trans=ts.translations,
        grid_shapes=np.array([np.asarray(g.target).shape for g in grids]),
        grid_ids=np.array([g.slice_id for g in grids]),
        dims=np.array(dims), first=np.asarray(first), last=np.asarray(last),
        gt=gt.data.astype(np.float32), psnr_db=db, runtime_s=runtime, threads=threads,
        losses=np.array(losses), recon=pred.astype(np.float32),
        schedule=np.array(bundle.train.resolution_schedule), nrf_activation_iter=bundle.train.nrf_activation_iter,
        total_iters=bundle.train.total_iters, batch_points=bundle.train.batch_points, seed=bundle.train.seed)


if __name__ == "__main__":
    main()
