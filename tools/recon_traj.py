"""Per-iteration loss trajectory of the 4,000-iteration desk64 run against the
reference's recorded one (where does float32 training drift from float64?)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_2603_00145_b200.recon import load_recon_fixture
    from paper_2603_00145_b200.train import Trainer, freeze_gc

    freeze_gc()
    g = os.path.join(ROOT, "tests", "golden")
    cloud, ts, grids, cfg, tgt = load_recon_fixture(os.path.join(g, "recon_desk64.npz"),
                                                    os.path.join(g, "recon_desk64_long.npz"))
    tr = Trainer(cloud, ts, cfg, slice_grids=grids, graph=True)
    ours = []
    while tr.iteration < cfg.total_iters:
        r = tr.step(sync=True)
        ours.append([r.total, r.data, r.ssim, r.aniso])
    tr.close()
    ours = np.array(ours)
    ref = np.asarray(tgt.ref_losses)
    rel = np.abs(ours - ref) / np.maximum(np.abs(ref), 1e-12)
    for lo, hi in [(0, 10), (10, 100), (100, 500), (500, 1000), (1000, 1600), (1600, 1700), (1700, 2000),
                   (2000, 2800), (2800, 2900), (2900, 3500), (3500, 4000)]:
        print(f"iters [{lo:4d},{hi:4d}): median rel diff total {np.median(rel[lo:hi, 0]):.2e} "
              f"data {np.median(rel[lo:hi, 1]):.2e} ssim {np.median(rel[lo:hi, 2]):.2e} "
              f"mean total ours/ref {ours[lo:hi, 0].mean() / ref[lo:hi, 0].mean():.5f}")


if __name__ == "__main__":
    main()
