"""Backward cutoff culling on a TRAINED field: gradients with and without
culling (MGAUSS_BWD_CULL) on the same field, points and upstream must agree to
float32 summation order.  Reports the largest relative deviation per
parameter group and the entries above a threshold.

    python tools/cull_check.py [--config C4] [--train 900] [--points 65536]
"""
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
    ap.add_argument("--train", type=int, default=900)
    ap.add_argument("--points", type=int, default=65536)
    ap.add_argument("--final", action="store_true", help="start at the final level instead of the schedule")
    ap.add_argument("--recon", action="store_true", help="the desk64 4,000-iteration fixture instead of a bench config")
    a = ap.parse_args()
    from types import SimpleNamespace

    from paper_2603_00145_b200.render import render_backward
    from paper_2603_00145_b200.spatial import build
    from paper_2603_00145_b200.train import Trainer

    if a.recon:
        from paper_2603_00145_b200.recon import load_recon_fixture

        gd = os.path.join(ROOT, "tests", "golden")
        cloud, ts0, grids, cfg, _ = load_recon_fixture(os.path.join(gd, "recon_desk64.npz"),
                                                       os.path.join(gd, "recon_desk64_long.npz"))
        psf = None
        tr = Trainer(cloud, ts0, cfg, slice_grids=grids, graph=True)
        a.points = min(a.points, cloud.coords.shape[0])
    else:
        data, cloud, grids, psf, cfg = bench.make_workload(a.config, 0, final_only=a.final)
        tr = Trainer(cloud, data.transforms, cfg, slice_grids=grids, slice_psf=psf, graph=True)
    for _ in range(a.train):
        tr.step_pipelined()
    tr.flush()
    f = tr.field.to_host()
    ts = tr.transforms_host()
    g = f.lattice_dims[0]
    grid = build(f, g, cfg.block_radius)
    rng = np.random.default_rng(3)
    idx = rng.choice(cloud.coords.shape[0], a.points, replace=False)
    batch = SimpleNamespace(coords=cloud.coords[idx], slice_ids=cloud.slice_ids[idx])
    up = rng.normal(size=a.points)
    out = {}
    for cull in ("1", "0"):
        os.environ["MGAUSS_BWD_CULL"] = cull
        gr = render_backward(f, grid, ts, batch, up, slice_psf=psf)
        out[cull] = gr
    os.environ.pop("MGAUSS_BWD_CULL", None)
    print(f"{'desk64' if a.recon else a.config} after {a.train} steps: G={g}, n={f.count}, {a.points} points"
          f"{'' if psf is None else f' x {psf.ntaps} taps'}")
    for name in ("d_positions", "d_quaternions", "d_log_scales", "d_intensity_logits", "d_transform_params"):
        on, off = np.asarray(getattr(out["1"], name)), np.asarray(getattr(out["0"], name))
        scale = np.abs(off).max()
        dev = np.abs(on - off)
        rel = dev / np.maximum(np.abs(off), 1e-30)
        bad = np.argwhere(dev > 1e-4 * np.abs(off) + 1e-6 * scale)
        print(f"  {name}: max|on-off|/max|off| = {dev.max() / scale:.2e}; entries beyond the 8(c) tolerance: "
              f"{len(bad)}; largest rel dev {rel.max():.2e}")
        for b in bad[:5]:
            print("    ", tuple(int(x) for x in b), on[tuple(b)], off[tuple(b)])
    tr.close()


if __name__ == "__main__":
    main()
