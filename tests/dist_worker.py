"""Worker of the multi-rank GPU tests (tests/test_dist_gpu.py): one rank of a
gloo group (several ranks share the test box's one GPU; gloo steps run
eagerly and the collectives go through the host, so no rank's kernels wait
on another rank's).  Trains a few steps of the `io` golden cloud and saves
losses + parameters (and a z-slab-sharded volume) for the parent to check."""

import os
import sys
from types import SimpleNamespace

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def make_trainer(z, dist, shard, use_nrf, graph=False, schedule=((0, 8), (3, 10))):
    from paper_2603_00145_b200.core import TransformSet
    from paper_2603_00145_b200.train import TrainConfig, Trainer

    cfg = TrainConfig(resolution_schedule=schedule, use_nrf=use_nrf, nrf_activation_iter=2, use_ssim=True,
                      batch_points=2048, seed=3)
    cloud = SimpleNamespace(coords=z["coords"], intensities=z["intensities"], slice_ids=z["slice_ids"])
    grids = [SimpleNamespace(coords=c, target=t, slice_id=int(s))
             for c, t, s in zip(z["sg_coords"], z["sg_target"], z["sg_ids"])]
    return Trainer(cloud, TransformSet(z["t_quats0"], z["t_trans0"]), cfg, slice_grids=grids, graph=graph,
                   dist=dist, shard=shard)


def snapshot(tr, reports):
    from paper_2603_00145_b200 import _device as dv

    out = {"losses": np.array([[r.total, r.data, r.ssim, r.aniso] for r in reports])}
    for name in ("positions", "quaternions", "log_scales", "logits"):
        out[name] = dv.to_host(getattr(tr.field, name)).astype(np.float64)
    out["tq"], out["tt"] = dv.to_host(tr.tq), dv.to_host(tr.tt)
    if tr.nrf is not None:
        out["nrf_w2"] = dv.to_host(tr.nrf.weights[2]).astype(np.float64)
    return out


def main():
    rank, world, port, shard, steps, use_nrf, out = (int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4],
                                                      int(sys.argv[5]), sys.argv[6] == "1", sys.argv[7])
    import torch
    import torch.distributed as tdist

    from conftest import load_golden

    torch.cuda.set_device(0)
    tdist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    z = load_golden("io")
    tr = make_trainer(z, tdist.group.WORLD, shard, use_nrf)
    reps = [tr.step() for _ in range(steps)]
    res = snapshot(tr, reps)
    vol = tr.render_volume((13, 9, 7), ((-1.0,) * 3, (1.0,) * 3), dist=tdist.group.WORLD)
    res["volume"] = vol.data
    np.savez(f"{out}_r{rank}.npz", **res)
    tr.close()
    tdist.barrier()
    tdist.destroy_process_group()


if __name__ == "__main__":
    main()
