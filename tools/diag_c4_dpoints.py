"""Diagnostic: error anatomy of d_points / d_transform_params on the drifted C4
field (float32 device path vs float64 oracle, and the oracle fed points
rounded to float32)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    from test_config_parity_gpu import Bt, _trained
    from oracle import oracle as O
    from paper_2603_00145_b200.render import render_backward
    from paper_2603_00145_b200.spatial import build

    tr, data, psf = _trained("C4", 200)
    f = tr.field.to_host()
    ts = tr.transforms_host()
    g, r = tr.field.resolution, 5
    rng = np.random.default_rng(2)
    idx = rng.choice(data.coords.shape[0], 8192, replace=False)
    k = int(rng.integers(data.num_slices))
    sc, _ = data.slice_grid(k)
    coords = np.concatenate([data.coords[idx], sc])
    sids = np.concatenate([data.slice_ids[idx], np.full(sc.shape[0], k, np.int64)])
    up = rng.normal(size=coords.shape[0]) * 1e-3
    gr = render_backward(f, build(f, g, r), ts, Bt(coords, sids), up, slice_psf=psf)
    og = O.psf_backward(f.positions, f.quaternions, f.log_scales, f.intensity_logits, g, r, coords, sids,
                        ts.quats, ts.translations, psf.offsets, psf.weights, psf.through_dirs, up, 16)
    dp = gr.d_points.sum(axis=1)
    e = np.abs(dp - og.d_points)
    mag = np.abs(og.d_points)
    print("d_points: median rel", np.median(e / (mag + 1e-30)), "p99 rel", np.quantile(e / (mag + 1e-30), 0.99),
          "max abs", e.max(), "max mag", mag.max())
    a, w = gr.d_transform_params, og.d_transform_params
    tol = 1e-4 * np.abs(w) + 1e-6 * np.abs(w).max()
    ratio = np.abs(a - w) / tol
    print("transform: worst ratio", ratio.max(), "bad", (ratio > 1).sum())
    worst = np.unravel_index(np.argmax(ratio), ratio.shape)
    s = worst[0]
    sel = sids == s
    print("worst slice", s, "points", sel.sum(), "row", w[s], "got", a[s])
    # per-point contributions to that slice's translation gradient
    print("sum |dp| over slice", np.abs(og.d_points[sel]).sum(axis=0), "sum dp", og.d_points[sel].sum(axis=0))
    print("err of sum", (dp[sel] - og.d_points[sel]).sum(axis=0))
    tr.close()


if __name__ == "__main__":
    main()
