"""PSNR of the 4,000-iteration desk64 reconstruction (tests/golden/recon_desk64_long.npz)
under the current build / switches:  python tools/recon_long.py [--short]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_2603_00145_b200.recon import load_recon_fixture, psnr, reconstruct
    from paper_2603_00145_b200.train import Trainer, freeze_gc

    freeze_gc()
    g = os.path.join(ROOT, "tests", "golden")
    long = None if "--short" in sys.argv else os.path.join(g, "recon_desk64_long.npz")
    cloud, ts, grids, cfg, tgt = load_recon_fixture(os.path.join(g, "recon_desk64.npz"), long)
    tr = Trainer(cloud, ts, cfg, slice_grids=grids, graph=True)
    vol, t_train, _ = reconstruct(tr, tgt.dims, tgt.first, tgt.last, tgt.intensity_scale)
    tr.close()
    db = psnr(vol.astype(np.float64), tgt.gt.astype(np.float64))
    print(f"iters {cfg.total_iters}: PSNR {db:.4f} dB (reference {tgt.ref_psnr_db:.4f}), diff {db - tgt.ref_psnr_db:+.4f}, "
          f"train {t_train:.2f} s")


if __name__ == "__main__":
    main()
