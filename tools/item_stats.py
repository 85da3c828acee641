"""Occupancy statistics of the C2 step (points / Gaussians per cell, items):
    python tools/item_stats.py [--config C2]"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def hist(name, cnt):
    occ = cnt[cnt > 0]
    q = np.percentile(occ, [10, 50, 90, 99, 100]) if occ.size else []
    print(f"{name}: occupied cells {occ.size}, mean/occupied {occ.mean():.2f}, p10/50/90/99/max {q}")
    for k in range(1, 9):
        print(f"   ={k}: {np.sum(occ == k)}", end="")
    print(f"   >8: {np.sum(occ > 8)}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    a = ap.parse_args()
    from paper_2603_00145_b200.train import Trainer

    data, cloud, grids, psf, cfg = bench.make_workload(a.config, 0, final_only=True)
    tr = Trainer(cloud, data.transforms, cfg, slice_grids=grids, slice_psf=psf, graph=False)
    for _ in range(3):
        tr.step()
    B = tr._bufs
    ps = B.pstart.cpu().numpy().astype(np.int64)
    gs = B.gstart.cpu().numpy().astype(np.int64)
    pc, gc = np.diff(ps), np.diff(gs)
    g = tr.field.resolution
    print("grid", g, "points", ps[-1], "gaussians", gs[-1])
    hist("points/cell", pc)
    hist("gaussians/cell", gc)
    r = cfg.block_radius
    # candidate Gaussians per point cell (box sum of gc over (2r+1)^3, clamped)
    G3 = gc.reshape(g, g, g)
    cs = np.zeros((g + 1, g + 1, g + 1))
    cs[1:, 1:, 1:] = G3.cumsum(0).cumsum(1).cumsum(2)
    idx = np.arange(g)
    lo, hi = np.clip(idx - r, 0, g), np.clip(idx + r + 1, 0, g)
    box = (cs[hi][:, hi][:, :, hi] - cs[lo][:, hi][:, :, hi] - cs[hi][:, lo][:, :, hi] - cs[hi][:, hi][:, :, lo]
           + cs[lo][:, lo][:, :, hi] + cs[lo][:, hi][:, :, lo] + cs[hi][:, lo][:, :, lo] - cs[lo][:, lo][:, :, lo])
    box = box.reshape(-1)
    pairs = float(np.sum(pc * box))
    occ = pc > 0
    print(f"pairs {pairs:.4g}; candidate Gaussians per occupied point cell mean {box[occ].mean():.1f}")
    for q in (1, 2, 4, 8):
        items = np.sum(np.ceil(pc / q))
        print(f"fwd items at Q={q}: {items:.0f}, mean pts/item {ps[-1] / items:.2f}")
    # k-runs of c adjacent cells merged into one item when their points fit 8 points
    P3 = pc.reshape(g * g, g)
    for c in (2, 4):
        items = 0
        for k0 in range(0, g, c):
            run = P3[:, k0:k0 + c]
            tot = run.sum(1)
            fit = tot <= 8
            items += int(np.sum((tot > 0) & fit)) + int(np.sum(np.ceil(run[~fit] / 8)))
        print(f"fwd items with {c}-cell k-runs (<= 8 pts merged): {items}, mean pts/item {ps[-1] / items:.2f}")


if __name__ == "__main__":
    main()
