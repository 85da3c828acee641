"""Profiling driver for a TRAINED (drifted) field: runs `--train` graph-replayed
training steps of a config, then `--steps` EAGER steps bracketed by
cudaProfilerStart/Stop, so `ncu --profile-from-start off` captures only the
kernels of steps on the drifted field (not the initial lattice).

    ncu --profile-from-start off --set full -k regex:'forward_kernel|backward_kernel' \
        python tools/profile_drifted.py --config C4 --train 200 --steps 1
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--train", type=int, default=200)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--schedule", action="store_true",
                    help="train through the config's resolution schedule instead of starting at its final level")
    a = ap.parse_args()
    import torch

    from paper_2603_00145_b200.train import Trainer

    data, cloud, grids, psf, cfg = bench.make_workload(a.config, 0, final_only=not a.schedule)
    tr = Trainer(cloud, data.transforms, cfg, slice_grids=grids, slice_psf=psf, graph=True)
    for _ in range(a.train):
        tr.step_pipelined()
    tr.flush()
    torch.cuda.synchronize()
    tr.graph = False
    tr._graph = None
    torch.cuda.cudart().cudaProfilerStart()
    for _ in range(a.steps):
        rep = tr.step(sync=True)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("ok", rep.to_line())
    tr.close()


if __name__ == "__main__":
    main()
