"""Checkpoint interop through the device trainer:
- a checkpoint written by the REFERENCE Trainer after step 3 (SSIM + NRF,
  lattice milestone 8 -> 10 at step 3) resumes here and the next 3 losses
  match the reference's own continuation;
- a checkpoint written here resumes bit-exactly (same parameters, optimizer
  state and RNG as the uninterrupted run), through the MGSS0001 file format."""

import os
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _trainer(z, cfg):
    from paper_2603_00145_b200.core import TransformSet
    from paper_2603_00145_b200.train import Trainer

    cloud = SimpleNamespace(coords=z["coords"], intensities=z["intensities"], slice_ids=z["slice_ids"])
    grids = [SimpleNamespace(coords=c, target=t, slice_id=int(s))
             for c, t, s in zip(z["sg_coords"], z["sg_target"], z["sg_ids"])]
    return Trainer(cloud, TransformSet(z["t_quats0"], z["t_trans0"]), cfg, slice_grids=grids)


def test_resume_from_reference_checkpoint():
    from paper_2603_00145_b200 import io as mio
    from paper_2603_00145_b200.train import TrainConfig

    z = load_golden("io")
    state = mio.load_checkpoint(os.path.join(GOLD, "io_checkpoint.mgss"))["trainer"]
    tr = _trainer(z, TrainConfig.from_dict(state["config"]))
    tr.load_state_dict(state)
    assert tr.iteration == 3 and tr.field.resolution == 8
    reps = [tr.step() for _ in range(3)]
    assert tr.field.resolution == 10  # the milestone at iteration 3 fired after the resume
    losses = np.array([[r.total, r.data, r.ssim, r.aniso] for r in reps])
    np.testing.assert_allclose(losses, z["losses_after"], rtol=2e-4, atol=1e-8)
    f = tr.field.to_host()
    np.testing.assert_allclose(f.positions, z["positions"], atol=5e-5)
    np.testing.assert_allclose(f.intensity_logits, z["logits"], atol=5e-4)
    tr.close()


def test_own_checkpoint_resumes_bit_exactly(tmp_path):
    from paper_2603_00145_b200 import _device as dv
    from paper_2603_00145_b200 import io as mio
    from paper_2603_00145_b200.train import TrainConfig

    z = load_golden("io")
    cfg = TrainConfig(resolution_schedule=((0, 8), (3, 10)), use_nrf=True, nrf_activation_iter=2, use_ssim=True,
                      batch_points=2048, seed=5, total_iters=8)
    a = _trainer(z, cfg)
    for _ in range(4):
        a.step()
    p = tmp_path / "ck.mgss"
    mio.save_checkpoint(p, {"trainer": a.state_dict()})
    b = _trainer(z, cfg)
    b.load_state_dict(mio.load_checkpoint(p)["trainer"])
    for _ in range(3):
        ra, rb = a.step(), b.step()
        # parameters evolve bit-identically; the reported loss sums use fp64
        # atomics (summation order varies in the last bits)
        np.testing.assert_allclose([rb.total, rb.data, rb.ssim, rb.aniso], [ra.total, ra.data, ra.ssim, ra.aniso],
                                   rtol=1e-12, atol=0)
    for x, y in [(a.field.positions, b.field.positions), (a.field.quaternions, b.field.quaternions),
                 (a.field.log_scales, b.field.log_scales), (a.field.logits, b.field.logits), (a.m, b.m),
                 (a.v, b.v), (a.tq, b.tq), (a.tt, b.tt), (a.nrf.weights[2], b.nrf.weights[2])]:
        np.testing.assert_array_equal(dv.to_host(x), dv.to_host(y))
    assert a.rng.bit_generator.state == b.rng.bit_generator.state
    a.close()
    b.close()


def test_resume_takes_the_checkpoint_config(tmp_path):
    """A trainer constructed with other learning rates / loss weights resumes
    on the checkpoint's config, as the reference CLI's --resume does
    (cli.py:121-123): every optimizer group -- including the fused Gaussian
    Adam + anisotropy kernel, whose hyperparameters live on the device --
    continues bit-exactly like the uninterrupted run."""
    import dataclasses

    from paper_2603_00145_b200 import _device as dv
    from paper_2603_00145_b200 import io as mio
    from paper_2603_00145_b200.train import TrainConfig

    z = load_golden("io")
    cfg = TrainConfig(resolution_schedule=((0, 8),), use_nrf=False, use_ssim=True, batch_points=2048, seed=5,
                      total_iters=8)
    other = dataclasses.replace(cfg, lr_position=0.01, lr_rotation=0.02, lr_scale=0.03, lr_intensity=0.2,
                                lambda_aniso=0.7, lambda_ratio=1.1, adam_beta1=0.8)
    a = _trainer(z, cfg)
    for _ in range(3):
        a.step()
    p = tmp_path / "ck.mgss"
    mio.save_checkpoint(p, {"trainer": a.state_dict()})
    b = _trainer(z, other)
    b.load_state_dict(mio.load_checkpoint(p)["trainer"])
    assert b.config.lr_position == cfg.lr_position and b.config.lambda_aniso == cfg.lambda_aniso
    for _ in range(3):
        a.step()
        b.step()
    for x, y in [(a.field.positions, b.field.positions), (a.field.log_scales, b.field.log_scales),
                 (a.field.logits, b.field.logits), (a.m, b.m), (a.v, b.v), (a.tq, b.tq)]:
        np.testing.assert_array_equal(dv.to_host(x), dv.to_host(y))
    a.close()
    b.close()
