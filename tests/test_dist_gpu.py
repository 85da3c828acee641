"""The data-parallel training path (parallel.py).

* world size 1 over NCCL (the all-reduce captured in the step's CUDA graph):
  an identity, so the trainer must evolve bit-identically to the plain one;
* world size 2 (two processes sharing the box's one GPU over gloo, eager
  steps, host-side collectives): strong sharding must train the SAME model
  as one rank -- losses and parameters within fp32 reduction-order noise --
  and weak sharding must keep the ranks' replicas identical; the z-slab
  sharded volume must equal the single-rank volume.
"""

import os
import subprocess
import sys
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def _trainer(z, dist):
    from paper_2603_00145_b200.core import TransformSet
    from paper_2603_00145_b200.train import TrainConfig, Trainer

    cfg = TrainConfig(resolution_schedule=((0, 8),), use_nrf=False, use_ssim=True, batch_points=2048, seed=3)
    cloud = SimpleNamespace(coords=z["coords"], intensities=z["intensities"], slice_ids=z["slice_ids"])
    grids = [SimpleNamespace(coords=c, target=t, slice_id=int(s))
             for c, t, s in zip(z["sg_coords"], z["sg_target"], z["sg_ids"])]
    return Trainer(cloud, TransformSet(z["t_quats0"], z["t_trans0"]), cfg, slice_grids=grids, graph=True, dist=dist)


def test_nccl_path_world1_matches_plain_trainer():
    import torch
    import torch.distributed as tdist

    from paper_2603_00145_b200 import _device as dv

    z = load_golden("io")
    if not tdist.is_initialized():
        tdist.init_process_group("nccl", init_method="tcp://127.0.0.1:29541", rank=0, world_size=1,
                                 device_id=torch.device("cuda", 0))
    try:
        a, b = _trainer(z, None), _trainer(z, tdist.group.WORLD)
        for _ in range(5):
            ra, rb = a.step(), b.step()
            np.testing.assert_allclose(rb.total, ra.total, rtol=1e-12)
        assert b._graph is not None  # the NCCL all-reduce was captured with the step
        for x, y in [(a.field.positions, b.field.positions), (a.field.quaternions, b.field.quaternions),
                     (a.field.log_scales, b.field.log_scales), (a.field.logits, b.field.logits), (a.tq, b.tq),
                     (a.tt, b.tt)]:
            np.testing.assert_array_equal(dv.to_host(x), dv.to_host(y))
        a.close()
        b.close()
    finally:
        tdist.destroy_process_group()


def _spawn_world(tmp_path, world, shard, steps, use_nrf):
    port = str(29600 + (os.getpid() % 200))
    out = str(tmp_path / f"{shard}")
    worker = os.path.join(os.path.dirname(os.path.abspath(__file__)), "dist_worker.py")
    procs = [subprocess.Popen([sys.executable, worker, str(r), str(world), port, shard, str(steps),
                               "1" if use_nrf else "0", out]) for r in range(world)]
    for p in procs:
        assert p.wait(timeout=600) == 0
    return [dict(np.load(f"{out}_r{r}.npz")) for r in range(world)]


@pytest.mark.parametrize("use_nrf", [False, True])
def test_strong_sharding_world2_matches_world1(tmp_path, use_nrf):
    """2 ranks x half the batch and half the SSIM slice == 1 rank x the whole
    batch: every loss term (smooth-L1 over the global batch, SSIM of the
    assembled slice, aniso once) and every parameter group, through a lattice
    milestone (step 3) and the NRF switch (step 2)."""
    from dist_worker import make_trainer, snapshot

    z = load_golden("io")
    steps = 5
    ranks = _spawn_world(tmp_path, 2, "strong", steps, use_nrf)
    tr = make_trainer(z, None, "strong", use_nrf)
    ref = snapshot(tr, [tr.step() for _ in range(steps)])
    vol = tr.render_volume((13, 9, 7), ((-1.0,) * 3, (1.0,) * 3)).data
    tr.close()
    for res in ranks:
        np.testing.assert_allclose(res["losses"], ref["losses"], rtol=2e-6, atol=1e-9)
        for name in ("positions", "quaternions", "log_scales", "logits", "tq", "tt"):
            np.testing.assert_allclose(res[name], ref[name], rtol=0, atol=2e-6, err_msg=name)
        if use_nrf:
            np.testing.assert_allclose(res["nrf_w2"], ref["nrf_w2"], rtol=0, atol=2e-6)
        np.testing.assert_allclose(res["volume"], vol, rtol=1e-5, atol=1e-6)
    for name in ("positions", "logits", "tq"):  # replicas stay identical
        np.testing.assert_array_equal(ranks[0][name], ranks[1][name])


def test_weak_sharding_world2_replicas_agree(tmp_path):
    """Weak sharding: own batches per rank, one all-reduce of the partial sums
    -> every rank applies the identical update (no parameter broadcast)."""
    ranks = _spawn_world(tmp_path, 2, "weak", 4, True)
    for name in ("positions", "quaternions", "log_scales", "logits", "tq", "tt", "nrf_w2"):
        np.testing.assert_array_equal(ranks[0][name], ranks[1][name], err_msg=name)
    np.testing.assert_array_equal(ranks[0]["losses"], ranks[1]["losses"])
    assert np.all(np.isfinite(ranks[0]["losses"]))
    assert np.all(ranks[0]["losses"][:, 2] < 1.0)  # mean SSIM loss of the two ranks' slices
