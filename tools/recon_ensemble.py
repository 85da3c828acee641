"""Spread of the final PSNR of the desk64 reconstruction under rounding-level
perturbations: the sample intensities (and the slice targets drawn from them)
scaled by (1 + 1e-7 N(0,1)) with numpy seed s, exactly as
tests/golden/make_recon.py --perturb s does for the reference.  Seed 0 is the
unperturbed run.  Training is chaotic (tools/recon_traj.py: trajectory
differences grow ~10x per 500 iterations), so a single run's PSNR is one draw.

    python tools/recon_ensemble.py [K] [--short] [--strict] [--first S]

--strict trains with train.StrictTrainer (float64, the reference's operation
order): seed s then reproduces the reference's `make_recon.py --long
--perturb s` run, and the ensemble is the reference algorithm's own spread.
"""
import os
import sys
import time
from types import SimpleNamespace

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _arg(name, default):
    return int(sys.argv[sys.argv.index(name) + 1]) if name in sys.argv else default


def main():
    from paper_2603_00145_b200.recon import load_recon_fixture, psnr, reconstruct
    from paper_2603_00145_b200.strict_train import StrictTrainer
    from paper_2603_00145_b200.train import Trainer, freeze_gc

    freeze_gc()
    k = int(sys.argv[1]) if len(sys.argv) > 1 and not sys.argv[1].startswith("--") else 8
    first = _arg("--first", 0)
    strict = "--strict" in sys.argv
    g = os.path.join(ROOT, "tests", "golden")
    long = None if "--short" in sys.argv else os.path.join(g, "recon_desk64_long.npz")
    cloud, ts, grids, cfg, tgt = load_recon_fixture(os.path.join(g, "recon_desk64.npz"), long)
    dbs = []
    for seed in range(first, first + k):
        inten = cloud.intensities
        if seed:
            inten = inten * (1.0 + 1e-7 * np.random.default_rng(seed).normal(size=inten.shape))
        c2 = SimpleNamespace(coords=cloud.coords, intensities=inten, slice_ids=cloud.slice_ids)
        g2 = [SimpleNamespace(coords=sg.coords, slice_id=sg.slice_id,
                              target=inten[cloud.slice_ids == sg.slice_id].reshape(np.asarray(sg.target).shape))
              for sg in grids]
        t0 = time.perf_counter()
        tr = (StrictTrainer if strict else Trainer)(c2, ts, cfg, slice_grids=g2,
                                                    **({} if strict else {"graph": True}))
        vol, _, _ = reconstruct(tr, tgt.dims, tgt.first, tgt.last, tgt.intensity_scale)
        tr.close()
        dbs.append(psnr(vol.astype(np.float64), tgt.gt.astype(np.float64)))
        print(f"seed {seed}: {dbs[-1]:.6f} dB ({time.perf_counter() - t0:.0f} s)", flush=True)
    d = np.array(dbs)
    print(f"{'strict float64' if strict else 'float32'} iters {cfg.total_iters}: PSNR mean {d.mean():.4f} "
          f"std {d.std(ddof=1) if len(d) > 1 else 0.0:.4f} min {d.min():.4f} max {d.max():.4f} over {k} runs; "
          f"reference {tgt.ref_psnr_db:.4f}")


if __name__ == "__main__":
    main()
