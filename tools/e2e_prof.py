"""Host-side profile of the e2e loop (Trainer.step_pipelined) on the C2
workload: wall ms per step and a cProfile of 200 steps.

    python tools/e2e_prof.py [--config C2] [--steps 200]
"""
import argparse
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--steps", type=int, default=200)
    a = ap.parse_args()
    import torch

    from paper_2603_00145_b200.train import Trainer

    data, cloud, grids, psf, cfg = bench.make_workload(a.config, 0)
    tr = Trainer(cloud, data.transforms, cfg, slice_grids=grids, slice_psf=psf, graph=True)
    for _ in range(10):
        tr.step_pipelined()
    tr.flush()
    torch.cuda.synchronize()
    for rep in range(3):
        t0 = time.perf_counter()
        win = []
        for i in range(a.steps):
            tr.step_pipelined()
            if i % 25 == 24:
                win.append(round(1e3 * (time.perf_counter() - t0), 1))
        tr.flush()
        torch.cuda.synchronize()
        print(f"e2e wall {1e3 * (time.perf_counter() - t0) / a.steps:.3f} ms/step; cumulative ms every 25 steps {win}")
    prof = cProfile.Profile()
    prof.enable()
    for _ in range(a.steps):
        tr.step_pipelined()
    tr.flush()
    torch.cuda.synchronize()
    prof.disable()
    pstats.Stats(prof).sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()
