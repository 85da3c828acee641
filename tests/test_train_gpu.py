"""GPU parity of the device-resident training step against the reference
trainer's recorded trajectory (tests/golden/trainer*.npz, produced by running
/root/reference's Trainer) and the oracle's loss / optimizer restatements."""

from types import SimpleNamespace

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def test_smooth_l1_and_ssim_kernels():
    from paper_2603_00145_b200.train import smooth_l1_loss_grad, ssim_loss_grad

    z = load_golden("train_ops")
    loss, grad = smooth_l1_loss_grad(z["sl1_pred"], z["sl1_tgt"])
    np.testing.assert_allclose(loss, z["sl1"], rtol=1e-6)
    np.testing.assert_allclose(grad, z["sl1_grad"], rtol=1e-6, atol=1e-9)
    s = load_golden("ssim")
    loss, grad = ssim_loss_grad(s["pred"], s["tgt"])
    np.testing.assert_allclose(loss, s["loss"], rtol=1e-5)
    np.testing.assert_allclose(grad, s["grad"], rtol=1e-4, atol=1e-6 * np.abs(s["grad"]).max())


def test_upsample_and_init_field():
    import torch

    from paper_2603_00145_b200 import _device as dv
    from paper_2603_00145_b200.train import DeviceField, init_field_device, progressive_upsample_device

    z = load_golden("train_ops")
    r = 4
    node_of = np.empty(r ** 3, np.int32)
    li = z["up_idx"]
    node_of[(li[:, 0] * r + li[:, 1]) * r + li[:, 2]] = np.arange(r ** 3)
    f = DeviceField(dv.to_dev(np.zeros((64, 3)), torch.float32), dv.to_dev(z["up_q"], torch.float32),
                    dv.to_dev(z["up_s"], torch.float32), dv.to_dev(z["up_l"], torch.float32), r,
                    dv.to_dev(node_of, torch.int32))
    up = progressive_upsample_device(f, 7)
    np.testing.assert_allclose(dv.to_host(up.positions), z["up_pos"], atol=1e-6)
    np.testing.assert_allclose(dv.to_host(up.quaternions), z["up_qo"], atol=1e-6)
    np.testing.assert_allclose(dv.to_host(up.log_scales), z["up_so"], atol=1e-6)
    np.testing.assert_allclose(dv.to_host(up.logits), z["up_lo"], atol=1e-5)
    init = init_field_device(dv.to_dev(z["init_coords"], torch.float64), dv.to_dev(z["init_int"], torch.float32), 5)
    np.testing.assert_allclose(dv.to_host(init.logits), z["init_logits"], atol=1e-5)


def _cloud(z):
    return SimpleNamespace(coords=z["coords"], intensities=z["intensities"], slice_ids=z["slice_ids"])


def test_trainer_matches_reference_trajectory():
    """6 reference steps (no SSIM / NRF) with a lattice milestone 8 -> 10 at step 3."""
    from paper_2603_00145_b200.core import TransformSet
    from paper_2603_00145_b200.train import TrainConfig, Trainer

    z = load_golden("trainer")
    cfg = TrainConfig(resolution_schedule=((0, 8), (3, 10)), use_nrf=False, use_ssim=False, batch_points=2048,
                      seed=7, total_iters=6)
    tr = Trainer(_cloud(z), TransformSet(z["t_quats0"], z["t_trans0"]), cfg)
    for it in range(6):  # same RNG stream as the reference -> identical batches, every step
        np.testing.assert_array_equal(np.sort(tr._next_batch()), np.sort(z["batches"][it]))
    tr.close()
    tr = Trainer(_cloud(z), TransformSet(z["t_quats0"], z["t_trans0"]), cfg)
    reps = tr.run()
    losses = np.array([[r.total, r.data, r.aniso] for r in reps])
    np.testing.assert_allclose(losses, z["losses"], rtol=1e-4, atol=1e-9)
    f = tr.field.to_host()
    assert f.count == z["positions"].shape[0]
    np.testing.assert_allclose(f.positions, z["positions"], atol=2e-5)
    np.testing.assert_allclose(f.log_scales, z["log_scales"], atol=2e-4)
    np.testing.assert_allclose(f.intensity_logits, z["logits"], atol=2e-3)
    ts = tr.transforms_host()
    np.testing.assert_allclose(ts.quats, z["t_quats"], atol=1e-6)
    np.testing.assert_allclose(ts.translations, z["t_trans"], atol=1e-6)


def test_trainer_full_matches_reference_losses():
    """SSIM slice term + NRF (active from step 2) + milestone, vs the reference trainer."""
    from paper_2603_00145_b200.core import TransformSet
    from paper_2603_00145_b200.train import TrainConfig, Trainer

    z = load_golden("trainer_full")
    grids = [SimpleNamespace(coords=c, target=t, slice_id=int(s))
             for c, t, s in zip(z["sg_coords"], z["sg_target"], z["sg_ids"])]
    cfg = TrainConfig(resolution_schedule=((0, 8), (3, 10)), use_nrf=True, nrf_activation_iter=2, use_ssim=True,
                      batch_points=2048, seed=11, total_iters=6)
    tr = Trainer(_cloud(z), TransformSet(z["t_quats0"], z["t_trans0"]), cfg, slice_grids=grids)
    reps = tr.run()
    losses = np.array([[r.total, r.data, r.ssim, r.aniso] for r in reps])
    np.testing.assert_allclose(losses, z["losses"], rtol=2e-4, atol=1e-8)
    f = tr.field.to_host()
    np.testing.assert_allclose(f.positions, z["positions"], atol=5e-5)
    from paper_2603_00145_b200 import _device as dv

    np.testing.assert_allclose(dv.to_host(tr.nrf.weights[4]), z["nrf_w4"], atol=1e-5)


def test_render_volume_runs():
    from paper_2603_00145_b200.core import TransformSet
    from paper_2603_00145_b200.train import TrainConfig, Trainer

    z = load_golden("trainer")
    cfg = TrainConfig(resolution_schedule=((0, 8),), use_nrf=False, use_ssim=False, batch_points=1024, seed=7)
    tr = Trainer(_cloud(z), TransformSet(z["t_quats0"], z["t_trans0"]), cfg)
    tr.run(2)
    vol = tr.render_volume((12, 12, 12), ((-1, -1, -1), (1, 1, 1)))
    assert vol.data.shape == (12, 12, 12) and 0.0 <= vol.data.min() and vol.data.max() <= 1.0


def test_graph_with_nrf_matches_eager():
    """The captured step (incl. the NRF forward/backward, its multi-tensor Adam
    with the device step counter, SSIM, and a lattice milestone that forces a
    recapture) evolves exactly like the eager step."""
    from paper_2603_00145_b200 import _device as dv
    from paper_2603_00145_b200.core import TransformSet
    from paper_2603_00145_b200.train import TrainConfig, Trainer

    z = load_golden("trainer_full")
    grids = [SimpleNamespace(coords=c, target=t, slice_id=int(s))
             for c, t, s in zip(z["sg_coords"], z["sg_target"], z["sg_ids"])]
    cfg = TrainConfig(resolution_schedule=((0, 8), (4, 10)), use_nrf=True, nrf_activation_iter=2, use_ssim=True,
                      batch_points=2048, seed=11, total_iters=8)
    runs = []
    for graph in (False, True):
        tr = Trainer(_cloud(z), TransformSet(z["t_quats0"], z["t_trans0"]), cfg, slice_grids=grids, graph=graph)
        reps = tr.run()
        runs.append((tr, np.array([[r.total, r.data, r.ssim] for r in reps])))
    (a, la), (b, lb) = runs
    np.testing.assert_allclose(lb, la, rtol=1e-12)
    np.testing.assert_array_equal(dv.to_host(b.field.positions), dv.to_host(a.field.positions))
    np.testing.assert_array_equal(dv.to_host(b.nrf.weights[2]), dv.to_host(a.nrf.weights[2]))
    assert a.nrf_t == b.nrf_t == 6


@pytest.mark.parametrize("graph", [False, True])
def test_pipelined_steps_report_the_same_losses(graph):
    """step_pipelined() returns each step's report one call later (flush()
    returns the last) with exactly the losses of synchronous step()."""
    from paper_2603_00145_b200.core import TransformSet
    from paper_2603_00145_b200.train import TrainConfig, Trainer

    z = load_golden("trainer_full")
    grids = [SimpleNamespace(coords=c, target=t, slice_id=int(s))
             for c, t, s in zip(z["sg_coords"], z["sg_target"], z["sg_ids"])]
    cfg = TrainConfig(resolution_schedule=((0, 8), (3, 10)), use_nrf=True, nrf_activation_iter=2, use_ssim=True,
                      batch_points=2048, seed=11, total_iters=6)
    mk = lambda: Trainer(_cloud(z), TransformSet(z["t_quats0"], z["t_trans0"]), cfg, slice_grids=grids,  # noqa
                         graph=graph)
    a = mk()
    sync = [a.step() for _ in range(6)]
    b = mk()
    piped = [b.step_pipelined() for _ in range(6)]
    assert piped[0] is None
    piped = piped[1:] + [b.flush()]
    assert b.flush() is None
    for ra, rb in zip(sync, piped):
        assert ra.iteration == rb.iteration and ra.resolution == rb.resolution
        np.testing.assert_allclose([rb.total, rb.data, rb.ssim], [ra.total, ra.data, ra.ssim], rtol=1e-12)
