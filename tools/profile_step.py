"""Profiling driver: builds the C2 workload and runs a few EAGER training steps
(no CUDA graph) so ncu sees every kernel launch of the step.

    python tools/profile_step.py [--steps 3] [--config C2]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--config", default="C2")
    a = ap.parse_args()
    import torch

    from paper_2603_00145_b200.train import Trainer

    data, cloud, grids, psf, cfg = bench.make_workload(a.config, 0, final_only=True)
    tr = Trainer(cloud, data.transforms, cfg, slice_grids=grids, slice_psf=psf, graph=False)
    for _ in range(a.steps):
        rep = tr.step(sync=True)
    torch.cuda.synchronize()
    print("ok", rep.to_line())


if __name__ == "__main__":
    main()
