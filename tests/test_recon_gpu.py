"""End-to-end reconstruction parity (north_star: final PSNR within 0.05 dB of
the CPU reference on the same inputs, seed, batches and schedule): the
reference's desk-scale run (configs/desk64.cfg: 64^3 phantom, 1500 iterations,
lattice 16^3 -> 48^3, NRF from 600, SSIM) was recorded by
tests/golden/make_recon.py; the device trainer replays the same batch stream
on the same cloud and must land on the same PSNR."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden", "recon_desk64.npz")


@pytest.mark.skipif(not os.path.exists(GOLD), reason="recon fixture not generated")
@pytest.mark.parametrize("graph", [False, True])
def test_desk64_reconstruction_psnr_matches_reference(graph):
    from paper_2603_00145_b200.recon import load_recon_fixture, psnr, reconstruct
    from paper_2603_00145_b200.train import Trainer

    cloud, ts, grids, cfg, tgt = load_recon_fixture(GOLD)
    tr = Trainer(cloud, ts, cfg, slice_grids=grids, graph=graph)
    try:
        losses = []
        vol, t_train, _ = reconstruct(tr, tgt.dims, tgt.first, tgt.last, tgt.intensity_scale,
                                      progress=lambda r: losses.append([r.total, r.data, r.ssim, r.aniso]))
    finally:
        tr.close()
    db = psnr(vol.astype(np.float64), tgt.gt.astype(np.float64))
    print(f"PSNR {db:.4f} dB (reference {tgt.ref_psnr_db:.4f} dB), train {t_train:.2f} s "
          f"(reference {tgt.ref_seconds:.0f} s on {tgt.ref_threads} threads)")
    assert abs(db - tgt.ref_psnr_db) <= 0.05
    # early trajectory tracks the reference closely (fp32 vs fp64 drift grows later)
    np.testing.assert_allclose(np.array(losses)[:50], tgt.ref_losses[:50], rtol=2e-3, atol=1e-7)


LONG = os.path.join(os.path.dirname(__file__), "golden", "recon_desk64_long.npz")


PERTURBED = os.path.join(os.path.dirname(__file__), "golden", "recon_desk64_long_perturbed.txt")


def _reference_ensemble():
    """{seed: PSNR} of the reference's own 4,000-iteration runs: seed 0 the
    unperturbed run (recon_desk64_long.npz), seeds >= 1 with the sample
    intensities scaled by (1 + 1e-7 N(0,1)) (make_recon.py --long --perturb s)."""
    import numpy as np

    out = {0: float(np.load(LONG)["psnr_db"])}
    if os.path.exists(PERTURBED):
        for line in open(PERTURBED):
            f = line.split()
            if f:
                out[int(f[0])] = float(f[1])
    return out


def _perturbed(cloud, grids, seed):
    from types import SimpleNamespace

    inten = cloud.intensities
    if seed:
        inten = inten * (1.0 + 1e-7 * np.random.default_rng(seed).normal(size=inten.shape))
    c2 = SimpleNamespace(coords=cloud.coords, intensities=inten, slice_ids=cloud.slice_ids)
    g2 = [SimpleNamespace(coords=g.coords, slice_id=g.slice_id,
                          target=inten[cloud.slice_ids == g.slice_id].reshape(np.asarray(g.target).shape))
          for g in grids]
    return c2, g2


@pytest.mark.skipif(not os.path.exists(LONG), reason="long recon fixture not generated")
def test_desk64_long_reconstruction_psnr_matches_reference():
    """The reference's default training length (4,000 iterations, train.py:56)
    on the desk64 data (lattice 16 -> 48 over 5 levels, NRF from 1,600).

    Training is chaotic at this length: inputs perturbed by 1e-7 relative move
    the reference's own final PSNR by up to 0.12 dB (its ensemble in
    recon_desk64_long_perturbed.txt; the unperturbed run is the ensemble's
    maximum), so one run is one draw.  The float32 trainer, run on the same
    perturbed inputs, must land with its ensemble mean within 0.05 dB of the
    reference ensemble's mean (no run further than 0.25 dB from it); the
    strict-float64 path reproduces the individual
    reference runs (tests/test_strict_train_gpu.py).  Sampling the trained
    field with the strict float64 kernels gives the float32 volume's PSNR to
    1e-3 dB."""
    from paper_2603_00145_b200 import render
    from paper_2603_00145_b200.recon import load_recon_fixture, psnr, reconstruct
    from paper_2603_00145_b200.spatial import build
    from paper_2603_00145_b200.train import Trainer

    ref = _reference_ensemble()
    cloud, ts, grids, cfg, tgt = load_recon_fixture(GOLD, LONG)
    assert cfg.total_iters == 4000
    dbs = {}
    for seed in sorted(ref):
        c2, g2 = _perturbed(cloud, grids, seed)
        tr = Trainer(c2, ts, cfg, slice_grids=g2, graph=True)
        try:
            vol, t_train, _ = reconstruct(tr, tgt.dims, tgt.first, tgt.last, tgt.intensity_scale)
            dbs[seed] = psnr(vol.astype(np.float64), tgt.gt.astype(np.float64))
            print(f"seed {seed}: float32 {dbs[seed]:.4f} dB (reference {ref[seed]:.4f} dB), train {t_train:.2f} s")
            if seed == 0:
                # the same trained field sampled in strict float64 (Gaussian part; the NRF residual is float32)
                f = tr.field.to_host()
                prev = render.get_strict_fp64()
                render.set_strict_fp64(True)
                try:
                    res = tr.nrf if tr.nrf_active else None
                    v64 = render.sample_volume(f, build(f, f.lattice_dims[0], cfg.block_radius), res, tgt.dims,
                                               (tuple(tgt.first), tuple(tgt.last)))
                finally:
                    render.set_strict_fp64(prev)
                db64 = psnr((v64.data * tgt.intensity_scale).astype(np.float32).astype(np.float64),
                            tgt.gt.astype(np.float64))
                print(f"strict float64 sampling of the trained field: {db64:.4f} dB")
                assert abs(db64 - dbs[0]) <= 1e-3
        finally:
            tr.close()
    r = np.array([ref[s] for s in sorted(ref)])
    d = np.array([dbs[s] for s in sorted(ref)])
    print(f"{len(r)} runs: float32 mean {d.mean():.4f} (range {d.min():.4f}-{d.max():.4f}); "
          f"reference mean {r.mean():.4f} (range {r.min():.4f}-{r.max():.4f})")
    assert abs(d.mean() - r.mean()) <= 0.05
    # single draws: no run far outside the chaotic spread (24-seed float32 ensembles reach 0.14 dB below the mean)
    assert np.abs(d - r.mean()).max() <= 0.25
