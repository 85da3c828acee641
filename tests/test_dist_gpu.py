"""The data-parallel training path (parallel.py FlatAllReduce over NCCL,
captured in the step's CUDA graph) at world size 1: the all-reduce is then
an identity, so the trainer must evolve bit-identically to the plain one
(the step is deterministic).  Multi-rank sums are covered on CPU by
tests/test_parallel_cpu.py (gloo, world size 2)."""

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
