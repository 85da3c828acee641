"""Spread of the final PSNR of the 4,000-iteration desk64 reconstruction under
rounding-level perturbations: the sample intensities scaled by (1 + eps N(0,1))
with eps = 1e-7, K seeds.  Training is chaotic (tools/recon_traj.py: trajectory
differences grow ~10x per 500 iterations), so a single run's PSNR is one draw.

    python tools/recon_ensemble.py [K] [--short]
"""
import os
import sys
from types import SimpleNamespace

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_2603_00145_b200.recon import load_recon_fixture, psnr, reconstruct
    from paper_2603_00145_b200.train import Trainer, freeze_gc

    freeze_gc()
    k = int(sys.argv[1]) if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else 8
    g = os.path.join(ROOT, "tests", "golden")
    long = None if "--short" in sys.argv else os.path.join(g, "recon_desk64_long.npz")
    cloud, ts, grids, cfg, tgt = load_recon_fixture(os.path.join(g, "recon_desk64.npz"), long)
    dbs = []
    for seed in range(k):
        eps = 0.0 if seed == 0 else 1e-7
        f = 1.0 + eps * np.random.default_rng(seed).normal(size=cloud.intensities.shape)
        c2 = SimpleNamespace(coords=cloud.coords, intensities=cloud.intensities * f, slice_ids=cloud.slice_ids)
        tr = Trainer(c2, ts, cfg, slice_grids=grids, graph=True)
        vol, _, _ = reconstruct(tr, tgt.dims, tgt.first, tgt.last, tgt.intensity_scale)
        tr.close()
        dbs.append(psnr(vol.astype(np.float64), tgt.gt.astype(np.float64)))
        print(f"seed {seed}: {dbs[-1]:.4f} dB", flush=True)
    d = np.array(dbs)
    print(f"iters {cfg.total_iters}: PSNR mean {d.mean():.4f} std {d.std(ddof=1):.4f} min {d.min():.4f} "
          f"max {d.max():.4f} over {k} runs; reference {tgt.ref_psnr_db:.4f}")


if __name__ == "__main__":
    main()
