"""Generate golden vectors by running the REFERENCE package (this container only).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Writes small ``.npz`` fixtures next to this script.  The reference is
imported read-only from /root/reference (it does not exist on the GPU box;
the fixtures travel instead).  Single-threaded reference = canonical order
(render.py:44-53).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from mgauss import render, spatial, train  # noqa: E402
from mgauss.core import GaussianField, TransformSet, lattice_node_index, uniform_lattice_field  # noqa: E402
from mgauss import nrf as mnrf  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
render.set_num_threads(1)


class Batch:
    def __init__(self, coords, slice_ids):
        self.coords = coords
        self.slice_ids = slice_ids


def random_field(rng, side=3, scale_lo=-2.2, scale_hi=-0.7):
    """Mirrors the reference fixture (tests/conftest.py:26-36)."""
    n = side ** 3
    return GaussianField(
        positions=rng.uniform(-0.8, 0.8, (n, 3)),
        quaternions=rng.normal(0.0, 1.0, (n, 4)) + np.array([2.0, 0, 0, 0]),
        log_scales=rng.uniform(scale_lo, scale_hi, (n, 3)),
        intensity_logits=rng.normal(0.0, 1.5, n),
        lattice_dims=(side, side, side),
        lattice_index=lattice_node_index(side),
    ).validate()


def f32(a):
    """Round to float32 and back: the GPU holds fp32 parameters, so the
    golden case feeds the reference exactly the values the GPU sees."""
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def field_arrays(f):
    return dict(positions=f.positions, quaternions=f.quaternions, log_scales=f.log_scales,
                logits=f.intensity_logits)


def render_case(name, f, g, r, coords, sids, ts, upstream):
    grid = spatial.build(f, g, block_radius=r)
    fwd = render.render_points(f, grid, ts, Batch(coords, sids), radius=r)
    grads = render.render_backward(f, grid, ts, Batch(coords, sids), upstream, radius=r)
    qn, rot, inv_var, prec6, alpha = render.activated_parameters(f)
    tq = ts.quats if ts is not None else np.zeros((0, 4))
    tt = ts.translations if ts is not None else np.zeros((0, 3))
    np.savez_compressed(
        os.path.join(OUT, f"render_{name}.npz"),
        g=g, r=r, **field_arrays(f), coords=coords, sids=sids, t_quats=tq, t_trans=tt,
        upstream=upstream, cell_starts=grid.cell_starts, cell_indices=grid.cell_indices,
        prec6=prec6, alpha=alpha, qn=qn, inv_var=inv_var,
        points=fwd.points, intensities=fwd.intensities, counts=fwd.contributor_counts,
        d_positions=grads.d_positions, d_quaternions=grads.d_quaternions,
        d_log_scales=grads.d_log_scales, d_logits=grads.d_intensity_logits,
        d_transform=grads.d_transform_params, d_points=grads.d_points,
    )


def make_render_cases():
    rng = np.random.default_rng(20260808)
    # (a) tiny random field, full radius, with transforms (tests/test_render.py:177-199 style)
    f = random_field(rng, side=3)
    for a in ("positions", "quaternions", "log_scales", "intensity_logits"):
        setattr(f, a, f32(getattr(f, a)))
    k = 4
    ts = TransformSet(quats=f32(rng.normal(0, 0.1, (k, 4)) + np.array([1.0, 0, 0, 0])),
                      translations=f32(rng.normal(0, 0.05, (k, 3))))
    coords = rng.uniform(-0.9, 0.9, (400, 3))
    sids = rng.integers(-1, k, 400)
    render_case("small_full", f, 5, 5, coords, sids, ts, rng.normal(size=400))
    # (b) same field, truncated neighborhood r=1 at G=8
    render_case("small_r1", f, 8, 1, coords, sids, ts, rng.normal(size=400))
    # (c) lattice field (training geometry: G = R, one primitive per cell)
    R = 12
    lf = uniform_lattice_field(R)
    lf.positions += rng.normal(0, 0.2 / R, lf.positions.shape)
    lf.quaternions += rng.normal(0, 0.1, lf.quaternions.shape)
    lf.log_scales += rng.normal(0, 0.1, lf.log_scales.shape)
    lf.intensity_logits[:] = rng.normal(0, 1.0, lf.count)
    for a in ("positions", "quaternions", "log_scales", "intensity_logits"):
        setattr(lf, a, f32(getattr(lf, a)))
    k = 6
    ts = TransformSet(quats=f32(rng.normal(0, 0.02, (k, 4)) + np.array([1.0, 0, 0, 0])),
                      translations=f32(rng.normal(0, 0.01, (k, 3))))
    coords = rng.uniform(-1.05, 1.05, (3000, 3))
    sids = rng.integers(0, k, 3000)
    render_case("lattice12", lf, R, 5, coords, sids, ts, rng.normal(size=3000) * 1e-3)
    # (d) no transforms, many points per cell, random positions (bench_speedup-like)
    rf = uniform_lattice_field(10)
    rf.positions[:] = rng.uniform(-0.98, 0.98, rf.positions.shape)
    rf.intensity_logits[:] = rng.normal(0.0, 1.0, rf.count)
    rf.log_scales[:] = np.log(1.0 / 14)
    for a in ("positions", "quaternions", "log_scales", "intensity_logits"):
        setattr(rf, a, f32(getattr(rf, a)))
    coords = rng.uniform(-1.0, 1.0, (5000, 3))
    render_case("random14", rf, 14, 3, coords, np.full(5000, -1, np.int64), None,
                rng.normal(size=5000))
    # (e) clamped log-scales (|s| > 20 -> zero log-scale gradient, render.py:334-335)
    cf = random_field(rng, side=2)
    cf.log_scales[0, 1] = 21.0
    cf.log_scales[1, 2] = -20.5
    for a in ("positions", "quaternions", "log_scales", "intensity_logits"):
        setattr(cf, a, f32(getattr(cf, a)))
    coords = rng.uniform(-0.9, 0.9, (200, 3))
    render_case("clamped", cf, 4, 4, coords, np.full(200, -1, np.int64), None,
                rng.normal(size=200))


def make_spatial_cases():
    rng = np.random.default_rng(7)
    pos = rng.uniform(-1.05, 1.05, (6 ** 3, 3))
    grid = spatial.build(pos, 70)
    sweep = np.linspace(-1.2, 1.2, 1201)
    sweep_cells = spatial.cell_index(np.stack([sweep] * 3, axis=1), 16)[:, 0]
    lat = uniform_lattice_field(6)
    lgrid = spatial.build(lat, 6)
    dup = np.zeros((50, 3))
    dgrid = spatial.build(dup, 70)
    np.savez_compressed(
        os.path.join(OUT, "spatial.npz"),
        pos=pos, cell_starts=grid.cell_starts, cell_indices=grid.cell_indices,
        sweep=sweep, sweep_cells=sweep_cells,
        lat_pos=lat.positions, lat_starts=lgrid.cell_starts, lat_indices=lgrid.cell_indices,
        dup_starts=dgrid.cell_starts, dup_indices=dgrid.cell_indices,
        corner_cells=spatial.cell_index(np.array([[-1.0] * 3, [0.0] * 3, [1.0] * 3]), 70),
    )


def make_volume_case():
    rng = np.random.default_rng(11)
    f = random_field(rng, side=3)
    for a in ("positions", "quaternions", "log_scales", "intensity_logits"):
        setattr(f, a, f32(getattr(f, a)))
    f.intensity_logits[:4] = 6.0
    grid = spatial.build(f, 4, block_radius=2)
    dims = (13, 11, 9)
    bounds = ((-0.9, -1.0, -0.8), (0.95, 1.0, 0.7))
    vol = render.sample_volume(f, grid, None, dims, bounds, radius=2)
    np.savez_compressed(os.path.join(OUT, "volume.npz"), **field_arrays(f), g=4, r=2,
                        dims=np.array(dims), lo=np.array(bounds[0]), hi=np.array(bounds[1]),
                        data=vol.data, spacing=vol.spacing, origin=vol.origin)


def make_train_cases():
    rng = np.random.default_rng(3)
    # Adam: three steps on two groups with distinct step counts (train.py:239-271)
    adam = train.AdamState()
    p = rng.normal(size=(5, 3))
    p0 = p.copy()
    grads = [rng.normal(size=(5, 3)) for _ in range(3)]
    for gr in grads:
        adam.step("positions", {"p": p}, {"p": gr}, 0.01)
    # aniso + smooth-L1
    s = rng.normal(0, 0.5, (64, 3))
    s[0] = [0.1, 0.1, 0.1]
    af = uniform_lattice_field(4)
    af.log_scales[:] = s
    aloss, agrad = train.aniso_loss_grad(af, 1.5)
    pred = rng.normal(size=50) * 2.0
    tgt = rng.normal(size=50)
    # upsample 4 -> 7 with drifted field
    uf = uniform_lattice_field(4)
    uf.intensity_logits[:] = rng.normal(size=uf.count)
    uf.log_scales[:] = rng.normal(0, 0.3, (uf.count, 3))
    uf.quaternions[:] = rng.normal(size=(uf.count, 4)) + np.array([1.5, 0, 0, 0])
    uf.quaternions[::3] *= -1.0
    up = train.progressive_upsample(uf, 7)
    # init_field on a small cloud
    from mgauss.simdata import PointCloud, WorldMap
    cc = rng.uniform(-1, 1, (3000, 3))
    ci = rng.uniform(0, 1, 3000)
    cloud = PointCloud(coords=cc, intensities=ci, slice_ids=np.zeros(3000, np.int64),
                       world_map=WorldMap(1.0, np.zeros(3)), intensity_scale=1.0,
                       num_slices=1)
    init = train.init_field(cloud, 5)
    np.savez_compressed(
        os.path.join(OUT, "train_ops.npz"),
        adam_p0=p0, adam_grads=np.stack(grads), adam_p=p,
        adam_m=adam.groups["positions"]["m"]["p"], adam_v=adam.groups["positions"]["v"]["p"],
        aniso_s=s, aniso_loss=aloss, aniso_grad=agrad,
        sl1_pred=pred, sl1_tgt=tgt, sl1=train.smooth_l1(pred, tgt),
        sl1_grad=train.smooth_l1_grad(pred, tgt),
        up_q=uf.quaternions, up_s=uf.log_scales, up_l=uf.intensity_logits,
        up_idx=uf.lattice_index, up_pos=up.positions, up_qo=up.quaternions,
        up_so=up.log_scales, up_lo=up.intensity_logits,
        init_coords=cc, init_int=ci, init_logits=init.intensity_logits,
    )
    # NRF forward/backward (nrf.py:115-182)
    field = mnrf.ResidualField.create(np.random.default_rng(5))
    field.weights[-1][:] = np.random.default_rng(6).normal(0, 0.1, field.weights[-1].shape)
    x = rng.uniform(-1, 1, (64, 3))
    upn = rng.normal(size=64)
    r = mnrf.nrf_forward(field, x)
    ng = mnrf.nrf_backward(field, x, upn)
    arrays = {f"w{i}": w for i, w in enumerate(field.weights)}
    arrays.update({f"b{i}": b for i, b in enumerate(field.biases)})
    arrays.update({f"dw{i}": w for i, w in enumerate(ng.d_weights)})
    arrays.update({f"db{i}": b for i, b in enumerate(ng.d_biases)})
    np.savez_compressed(os.path.join(OUT, "nrf.npz"), x=x, up=upn, r=r, d_points=ng.d_points,
                        **arrays)


def make_trainer_case():
    """A few reference Trainer steps (no SSIM, no NRF) incl. one lattice milestone."""
    from mgauss.cli import simulate_stacks
    from mgauss.io import SimSettings
    from mgauss.simdata import devoxelize, normalized_transforms

    sim = SimSettings(phantom="nested-ellipsoids", phantom_dims=24, phantom_spacing=1.0,
                      in_plane_spacing=1.0, slice_thickness=4.0, motion_sigma=0.5,
                      noise_sigma=0.01, reg_error_sigma=0.0, foreground_threshold=-1.0)
    _, stacks = simulate_stacks(sim, 7)
    cloud = devoxelize(stacks, -1.0)
    ts = normalized_transforms(stacks, cloud.world_map, "estimated")
    cfg = train.TrainConfig(resolution_schedule=((0, 8), (3, 10)), use_nrf=False,
                            use_ssim=False, batch_points=2048, seed=7, total_iters=6)
    tr = train.Trainer(cloud, ts, cfg)
    losses = []
    batches = []
    for _ in range(6):
        # record the batch the trainer draws (same RNG stream) for the GPU replay
        state = tr.rng.bit_generator.state
        perm, cursor = (None if tr._perm is None else tr._perm.copy()), tr._cursor
        idx = tr._next_batch()
        batches.append(idx.copy())
        tr.rng.bit_generator.state = state
        tr._perm, tr._cursor = perm, cursor
        rep = tr.step()
        losses.append([rep.total, rep.data, rep.aniso])
    np.savez_compressed(
        os.path.join(OUT, "trainer.npz"),
        coords=cloud.coords, intensities=cloud.intensities, slice_ids=cloud.slice_ids,
        t_quats0=ts.quats, t_trans0=ts.translations, batches=np.stack(batches),
        losses=np.array(losses), **field_arrays(tr.field), t_quats=tr.transforms.quats,
        t_trans=tr.transforms.translations, lattice_r=tr.field.lattice_dims[0],
    )


def make_ssim_case():
    from mgauss import ssim as mssim

    rng = np.random.default_rng(9)
    tgt = np.clip(rng.uniform(0, 1, (40, 33)), 0, 1)
    pred = np.clip(tgt + rng.normal(0, 0.1, tgt.shape), 0, 1)
    loss, grad = mssim.ssim_loss_grad(pred, tgt)
    np.savez_compressed(os.path.join(OUT, "ssim.npz"), pred=pred, tgt=tgt, loss=loss, grad=grad)


def make_trainer_full_case():
    """Reference Trainer with SSIM + NRF (active from step 2) + a milestone at 3."""
    from mgauss.cli import simulate_stacks
    from mgauss.io import SimSettings
    from mgauss.simdata import build_slice_grids, devoxelize, normalized_transforms

    sim = SimSettings(phantom="nested-ellipsoids", phantom_dims=24, phantom_spacing=1.0,
                      in_plane_spacing=1.0, slice_thickness=4.0, motion_sigma=0.5,
                      noise_sigma=0.01, reg_error_sigma=0.0, foreground_threshold=-1.0)
    _, stacks = simulate_stacks(sim, 7)
    cloud = devoxelize(stacks, -1.0)
    ts = normalized_transforms(stacks, cloud.world_map, "estimated")
    grids = build_slice_grids(stacks, cloud.world_map, cloud.intensity_scale)
    cfg = train.TrainConfig(resolution_schedule=((0, 8), (3, 10)), use_nrf=True, nrf_activation_iter=2,
                            use_ssim=True, batch_points=2048, seed=11, total_iters=6)
    tr = train.Trainer(cloud, ts, cfg, slice_grids=grids)
    losses = []
    for _ in range(6):
        rep = tr.step()
        losses.append([rep.total, rep.data, rep.ssim, rep.aniso])
    sg_coords = np.stack([g.coords for g in grids])
    sg_target = np.stack([g.target for g in grids])
    np.savez_compressed(
        os.path.join(OUT, "trainer_full.npz"),
        coords=cloud.coords, intensities=cloud.intensities, slice_ids=cloud.slice_ids,
        t_quats0=ts.quats, t_trans0=ts.translations, sg_coords=sg_coords, sg_target=sg_target,
        sg_ids=np.array([g.slice_id for g in grids]), losses=np.array(losses), **field_arrays(tr.field),
        t_quats=tr.transforms.quats, t_trans=tr.transforms.translations,
        nrf_w4=tr.nrf.weights[4], nrf_b4=tr.nrf.biases[4], nrf_w0=tr.nrf.weights[0],
    )


def make_io_cases():
    """F4 formats written by the reference writers (io.py:101-145, 213-237):
    two NIfTI volumes, and an MGSS0001 checkpoint of a reference Trainer (SSIM
    + NRF from step 2, lattice milestone 8 -> 10 at step 3) taken after step 3,
    with the losses of the 3 steps that follow it."""
    from mgauss import io as mio
    from mgauss.cli import simulate_stacks
    from mgauss.core import Volume
    from mgauss.simdata import build_slice_grids, devoxelize, normalized_transforms

    rng = np.random.default_rng(21)
    v32 = rng.normal(0, 1, (5, 4, 3))
    v16 = rng.integers(0, 65535, (3, 4, 2)).astype(np.uint16)
    sp, org = np.array([0.8, 0.9, 1.1]), np.array([-1.5, 2.25, 3.0])
    mio.write_volume(os.path.join(OUT, "io_f32.nii"), Volume(data=v32, spacing=sp, origin=org), descrip="golden f32")
    mio.write_volume(os.path.join(OUT, "io_u16.nii"), Volume(data=v16, spacing=sp, origin=org), descrip="golden u16")

    sim = mio.SimSettings(phantom="nested-ellipsoids", phantom_dims=24, phantom_spacing=1.0, in_plane_spacing=1.0,
                          slice_thickness=4.0, motion_sigma=0.5, noise_sigma=0.01, reg_error_sigma=0.0,
                          foreground_threshold=-1.0)
    _, stacks = simulate_stacks(sim, 7)
    cloud = devoxelize(stacks, -1.0)
    ts = normalized_transforms(stacks, cloud.world_map, "estimated")
    grids = build_slice_grids(stacks, cloud.world_map, cloud.intensity_scale)
    cfg = train.TrainConfig(resolution_schedule=((0, 8), (3, 10)), use_nrf=True, nrf_activation_iter=2,
                            use_ssim=True, batch_points=2048, seed=13, total_iters=6)
    tr = train.Trainer(cloud, ts, cfg, slice_grids=grids)
    for _ in range(3):
        tr.step()
    mio.save_checkpoint(os.path.join(OUT, "io_checkpoint.mgss"), {"trainer": tr.state_dict()})
    after = []
    for _ in range(3):
        rep = tr.step()
        after.append([rep.total, rep.data, rep.ssim, rep.aniso])
    np.savez_compressed(
        os.path.join(OUT, "io.npz"), v32=v32, v16=v16, spacing=sp, origin=org,
        coords=cloud.coords, intensities=cloud.intensities, slice_ids=cloud.slice_ids,
        t_quats0=ts.quats, t_trans0=ts.translations, sg_coords=np.stack([g.coords for g in grids]),
        sg_target=np.stack([g.target for g in grids]), sg_ids=np.array([g.slice_id for g in grids]),
        losses_after=np.array(after), **field_arrays(tr.field))


if __name__ == "__main__":
    make_ssim_case()
    make_trainer_full_case()
    make_spatial_cases()
    make_render_cases()
    make_volume_case()
    make_train_cases()
    make_trainer_case()
    make_io_cases()
    for fn in sorted(os.listdir(OUT)):
        if fn.endswith((".npz", ".nii", ".mgss")):
            print(fn, os.path.getsize(os.path.join(OUT, fn)))
