"""Kernel micro-benchmark on the C2 training state: times the forward and
backward pair kernels (and the whole eager step) with CUDA events.

    python tools/kbench.py [--reps 10]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--train", type=int, default=3, help="training steps before timing (drifted field)")
    ap.add_argument("--radius", type=int, default=None, help="override the candidate radius (what-if timing only)")
    ap.add_argument("--schedule", action="store_true",
                    help="train through the config's resolution schedule (upsampled fields) instead of its final level")
    a = ap.parse_args()
    import torch

    from paper_2603_00145_b200.train import Trainer

    data, cloud, grids, psf, cfg = bench.make_workload(a.config, 0, final_only=not a.schedule)
    if a.radius is not None:
        import dataclasses

        cfg = dataclasses.replace(cfg, block_radius=a.radius)
    tr = Trainer(cloud, data.transforms, cfg, slice_grids=grids, slice_psf=psf, graph=False)
    for _ in range(max(3, a.train)):
        tr.step(sync=False)
    kt = bench.kernel_times(tr, a.reps)
    steps = [tr.draw_step() for _ in range(a.reps)]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for all_idx, plan in steps:
        B = tr.load_indices(torch.from_numpy(all_idx).cuda(), plan)
        tr._body(B, plan)
    e1.record()
    torch.cuda.synchronize()
    kt["step_ms_eager"] = e0.elapsed_time(e1) / len(steps)
    p = kt["pairs_per_launch"]
    kt["fwd_gpairs_s"] = p / kt["forward_ms"] / 1e6
    kt["bwd_gpairs_s"] = p / kt["backward_ms"] / 1e6
    kt["fwd_frac"] = p * 20 / (kt["forward_ms"] / 1e3) / bench.peak_fp32(148, 1965.0)
    kt["bwd_frac"] = p * 56 / (kt["backward_ms"] / 1e3) / bench.peak_fp32(148, 1965.0)
    print(json.dumps(kt))


if __name__ == "__main__":
    main()
