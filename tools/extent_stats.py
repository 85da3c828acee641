"""How far each Gaussian's cutoff ellipsoid (d^T P d <= 64, _kernels.py:21)
reaches, in grid cells, over the C4 training schedule: the half-extent along
axis a is 8 sqrt(Sigma_aa) (Sigma = R diag(s^2) R^T), i.e. the cell window a
Gaussian can actually touch, against the Chebyshev window r = 5 the candidate
rule allows.

    python tools/extent_stats.py [--config C4] [--steps 4000]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def reach_cells(field, g):
    """Per Gaussian and axis: the farthest cell offset (in cells, from the
    Gaussian's own cell) its cutoff box touches, on the low and high side."""
    from paper_2603_00145_b200.render import activated_parameters

    _, _, _, p6, _ = activated_parameters(field)  # packed precision (P00, P01, P02, P11, P12, P22)
    P = p6[:, [0, 1, 2, 1, 3, 4, 2, 4, 5]].reshape(-1, 3, 3)
    sig = np.linalg.inv(P)[:, [0, 1, 2], [0, 1, 2]]  # Sigma_aa
    ext = 8.0 * np.sqrt(sig) * (g / 2.0)  # half-extent in cell widths
    u = (np.asarray(field.positions, np.float64) + 1.0) * (g / 2.0)  # position in cell units
    c = np.clip(np.floor(u), 0, g - 1)
    lo = c - np.floor(u - ext)
    hi = np.floor(u + ext) - c
    return ext, np.maximum(lo, hi)


def report(tag, field, g, r=5):
    ext, reach = reach_cells(field, g)
    q = np.percentile(ext, [1, 10, 50, 90, 99, 100])
    rr = np.minimum(reach, r)
    cells = np.prod(2 * rr + 1, axis=1)
    print(f"{tag}: G={g} n={field.count} half-extent (cells) p1/10/50/90/99/max {np.round(q, 2)}; "
          f"reach>=r on some axis: {np.mean(reach.max(axis=1) >= r):.3f}; "
          f"mean box cells {cells.mean():.0f} of {(2 * r + 1) ** 3} ({cells.mean() / (2 * r + 1) ** 3:.2f})")
    for k in range(0, r + 1):
        print(f"   max-axis reach {k}: {np.mean(np.minimum(reach.max(axis=1), r) == k):.3f}", end="")
    print()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--steps", type=int, default=4000)
    a = ap.parse_args()
    from paper_2603_00145_b200.train import Trainer

    data, cloud, grids, psf, cfg = bench.make_workload(a.config, 0)
    tr = Trainer(cloud, data.transforms, cfg, slice_grids=grids, slice_psf=psf, graph=True)
    marks = sorted({it - 1 for it, _ in cfg.resolution_schedule[1:]} | {a.steps - 1, 0, 200})
    while tr.iteration < a.steps:
        tr.step()
        if tr.iteration - 1 in marks:
            f = tr.field.to_host()
            report(f"after {tr.iteration} steps", f, f.lattice_dims[0])
    tr.close()


if __name__ == "__main__":
    main()
