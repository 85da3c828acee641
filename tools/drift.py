"""Kernel times as training proceeds (does the step get more expensive as
Gaussians drift off their lattice cells?):  python tools/drift.py [--config C4]"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--every", type=int, default=200)
    ap.add_argument("--rounds", type=int, default=4)
    a = ap.parse_args()
    import torch

    from paper_2603_00145_b200.train import Trainer

    data, cloud, grids, psf, cfg = bench.make_workload(a.config, 0, final_only=True)
    tr = Trainer(cloud, data.transforms, cfg, slice_grids=grids, slice_psf=psf, graph=True)
    for r in range(a.rounds + 1):
        kt = bench.kernel_times(tr, 5)
        gk = tr._bufs.gkey[: tr.field.count].cpu().numpy().astype(np.int64) if hasattr(tr._bufs, "gkey") else None
        extra = ""
        if gk is not None:
            g = tr.field.resolution
            ca, cb = gk[0:-1:2], gk[1::2]
            d = cb - ca[: cb.size]
            same_col = (ca[: cb.size] % g) + d <= g - 1
            ok = (d >= 0) & (d <= 4) & same_col
            extra = f"pairable {ok.mean():.3f}, occupied cells {np.unique(gk).size / g ** 3:.3f}"
        print(f"after {tr.iteration} steps: fwd {kt['forward_ms']:.3f} ms bwd {kt['backward_ms']:.3f} ms "
              f"pairs {kt['pairs_per_launch']:.4g} {extra}", flush=True)
        for _ in range(a.every if r < a.rounds else 0):
            tr.step_pipelined()
        tr.flush()


if __name__ == "__main__":
    main()
