"""Parity at the BENCHMARKED configurations (SURVEY §8(c) tolerances), not
only at fixture sizes: the float32 device kernels on the benchmark's own
fields and point sets against the CPU oracle (float64, oracle/).

  C2: a 97,336-Gaussian field after 30 training steps; 8,192 batch points
      plus a whole 160x160 SSIM slice, 3-tap PSF, forward + backward.
  C4: the 1,000,000-Gaussian (R = 100) level after 200 training steps (the
      drifted, clustered field: ~half the lattice cells empty); 8,192 batch
      points plus a 256x256 slice, 5-tap PSF, forward + backward.
  C5: 512^3 inference from 2,000,376 Gaussians: 4 whole z-planes (262,144
      voxels each) of the jittered lattice AND of a clustered field whose
      tiles overflow the staged shared-memory path (the global-walk fallback).

Counts bit-exact; intensities rel 1e-4; gradients |d| <= 1e-4 |ref| +
1e-6 max|ref| (reference render.py:161-187, 276-354, 379-408).
"""

import os

import numpy as np
import pytest

from conftest import assert_grad_close

pytestmark = pytest.mark.gpu

THREADS = min(32, os.cpu_count() or 1)


class Bt:
    def __init__(self, coords, sids):
        self.coords, self.slice_ids = coords, sids


def _trained(name, steps):
    import bench
    from paper_2603_00145_b200.train import Trainer

    data, cloud, grids, psf, cfg = bench.make_workload(name, 0, final_only=True)
    tr = Trainer(cloud, data.transforms, cfg, slice_grids=grids, slice_psf=psf, graph=True)
    for _ in range(steps):
        tr.step_pipelined()
    tr.flush()
    return tr, data, psf


def _check_step(tr, data, psf, nbatch, seed):
    """Forward + backward of one step's point set (a batch sample + one whole
    slice) through the public API, vs oracle.psf_render / psf_backward."""
    from oracle import oracle as O
    from paper_2603_00145_b200.render import render_backward, render_points
    from paper_2603_00145_b200.spatial import build

    f = tr.field.to_host()
    ts = tr.transforms_host()
    g, r = tr.field.resolution, tr.config.block_radius
    rng = np.random.default_rng(seed)
    idx = rng.choice(data.coords.shape[0], nbatch, replace=False)
    k = int(rng.integers(data.num_slices))
    sc, _ = data.slice_grid(k)
    coords = np.concatenate([data.coords[idx], sc])
    sids = np.concatenate([data.slice_ids[idx], np.full(sc.shape[0], k, np.int64)])
    up = rng.normal(size=coords.shape[0]) * 1e-3
    grid = build(f, g, r)
    out = render_points(f, grid, ts, Bt(coords, sids), slice_psf=psf)
    gr = render_backward(f, grid, ts, Bt(coords, sids), up, slice_psf=psf)
    inten, cnt = O.psf_render(f.positions, f.quaternions, f.log_scales, f.intensity_logits, g, r, coords, sids,
                              ts.quats, ts.translations, psf.offsets, psf.weights, psf.through_dirs, THREADS)
    og = O.psf_backward(f.positions, f.quaternions, f.log_scales, f.intensity_logits, g, r, coords, sids,
                        ts.quats, ts.translations, psf.offsets, psf.weights, psf.through_dirs, up, THREADS)
    np.testing.assert_array_equal(out.contributor_counts, cnt)
    assert int(cnt.sum()) > 0
    np.testing.assert_allclose(out.intensities, inten, rtol=1e-4, atol=1e-12)
    for name in ("d_positions", "d_quaternions", "d_log_scales", "d_intensity_logits"):
        assert_grad_close(getattr(gr, name), getattr(og, name), name=name)
    assert_grad_close(gr.d_points.sum(axis=1), og.d_points, name="d_points")
    # d_transform_params: a slice's entry is a sum over its ~65k points whose
    # terms cancel (the SSIM slice's y-translation: |sum| = 2e-4 while
    # sum|terms| = 88, a 5e5 cancellation): on top of the §8(c) tolerance the
    # error may be float32 unit roundoff (6e-8, x2) of the summed magnitudes,
    # the best any float32 d_points can give
    k = ts.quats.shape[0]
    dp = og.d_points
    s_t = np.zeros((k, 3))
    np.add.at(s_t, sids, np.abs(dp))
    s_q = np.zeros(k)
    np.add.at(s_q, sids, np.linalg.norm(dp, axis=1) * np.linalg.norm(coords, axis=1))
    allow = 1.2e-7 * np.hstack([np.repeat(2.0 * s_q[:, None], 4, axis=1), s_t])
    a, w = gr.d_transform_params, og.d_transform_params
    tol = 1e-4 * np.abs(w) + 1e-6 * np.abs(w).max() + allow
    assert np.all(np.abs(a - w) <= tol), np.max(np.abs(a - w) / tol)
    return int(cnt.sum())


def test_c2_step_parity():
    tr, data, psf = _trained("C2", 30)
    try:
        pairs = _check_step(tr, data, psf, 8192, 1)
        assert pairs > 5e7
    finally:
        tr.close()


def test_c4_drifted_million_parity():
    tr, data, psf = _trained("C4", 200)
    try:
        assert tr.field.count == 1_000_000
        from paper_2603_00145_b200 import _device as dv

        occupied = np.unique(dv.to_host(tr._bufs.gkey[: tr.field.count])).size
        assert occupied < 0.8 * tr.field.count  # drift emptied cells: the clustered regime
        pairs = _check_step(tr, data, psf, 8192, 2)
        assert pairs > 5e7
    finally:
        tr.close()


def _c5_field(clustered):
    from paper_2603_00145_b200.core import lattice_node_positions

    R = 126
    n = R ** 3
    rng = np.random.default_rng(7)
    pos = lattice_node_positions(R) + rng.normal(0, 0.1 / R, (n, 3))
    if clustered:  # squeeze the field into the central eighth: ~8 Gaussians per occupied cell
        pos = pos * 0.5
    q = np.zeros((n, 4))
    q[:, 0] = 1.0
    q += rng.normal(0, 0.1, (n, 4))
    ls = np.log(1.0 / R) + rng.normal(0, 0.1, (n, 3)) + (np.log(0.5) if clustered else 0.0)
    lg = rng.normal(0, 1, n)
    f32 = lambda a: a.astype(np.float32).astype(np.float64)  # noqa: E731  (the device holds float32)
    return f32(pos), f32(q), f32(ls), f32(lg), R


@pytest.mark.parametrize("clustered", [False, True])
def test_c5_volume_planes_parity(clustered):
    import torch

    from oracle import oracle as O
    from paper_2603_00145_b200 import _device as dv
    from paper_2603_00145_b200 import _native as N
    from paper_2603_00145_b200.render import sample_volume_device
    from paper_2603_00145_b200.spatial import build_device

    pos, q, ls, lg, R = _c5_field(clustered)
    n = pos.shape[0]
    L = N.lib()
    pd, qd, sd, ld = (dv.to_dev(a, torch.float32) for a in (pos, q, ls, lg))
    d = build_device(pd, R)
    grec = dv.empty((n, 12), torch.float32)
    err = dv.zeros((1,), torch.int32)
    N.check(L.mg_activate(N.ptr(pd), N.ptr(qd), N.ptr(sd), N.ptr(ld), n, N.ptr(d["order"]), N.ptr(grec), N.ptr(err),
                          dv.sptr()))
    dims = (512, 512, 512)
    bounds = ((-1.0,) * 3, (1.0,) * 3)
    if clustered:  # the staged tile path must overflow somewhere (> 2,304 records in a 12x12x16-cell union)
        cnt = np.diff(dv.to_host(d["starts"]).astype(np.int64)).reshape(R, R, R)
        assert cnt.max() >= 6 and cnt[60:72, 60:72, 55:71].sum() > 2304
    for i0 in (0, 137, 300, 511) if not clustered else (128, 200, 255, 383):
        got = dv.to_host(sample_volume_device(grec, n, d["starts"], R, 5, dims, bounds, i0=i0, i1=i0 + 1))
        want = O.sample_volume(pos, q, ls, lg, R, 5, dims, bounds, threads=THREADS, x_range=(i0, i0 + 1))
        assert np.count_nonzero(want) > 1000
        np.testing.assert_allclose(got.astype(np.float64), want, rtol=1e-4, atol=1e-7, err_msg=f"plane {i0}")
