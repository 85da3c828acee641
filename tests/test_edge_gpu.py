"""Boundary cases of the device path against the oracle: radius 0, a radius
larger than the grid, a one-cell grid, a single Gaussian / single sample,
samples far outside the [-1, 1] cube (clamped cells), samples exactly on
cell boundaries, coincident Gaussians, and through the slice-PSF staged path
(mg_bin_points / mg_forward / mg_backward)."""

import numpy as np
import pytest

from conftest import assert_grad_close

pytestmark = pytest.mark.gpu


def _field(rng, n, spread=0.9, scale=-1.5):
    from paper_2603_00145_b200.core import GaussianField

    f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)  # noqa: E731
    q = rng.normal(size=(n, 4))
    q[:, 0] += 2.0
    return GaussianField(f32(rng.uniform(-spread, spread, (n, 3))), f32(q), f32(rng.normal(scale, 0.3, (n, 3))),
                         f32(rng.normal(0, 1, n)), (n, 1, 1), np.zeros((n, 3), np.int64))


CASES = {
    "r0": dict(n=300, b=400, g=6, r=0),
    "r_gt_g": dict(n=120, b=200, g=3, r=7),
    "g1": dict(n=40, b=50, g=1, r=5),
    "one_gauss": dict(n=1, b=64, g=4, r=1),
    "one_point": dict(n=200, b=1, g=5, r=2),
    "outside": dict(n=150, b=300, g=5, r=2, outside=True),
    "on_boundaries": dict(n=150, b=300, g=8, r=2, boundary=True),
    "coincident": dict(n=64, b=300, g=6, r=2, coincident=True),
}


@pytest.mark.parametrize("name", sorted(CASES))
@pytest.mark.parametrize("psf", [False, True])
def test_edge_case_against_oracle(name, psf):
    from oracle import oracle as O
    from paper_2603_00145_b200.render import SlicePSF, render_backward, render_points
    from paper_2603_00145_b200.spatial import build
    from test_render_gpu import Batch, assert_rel

    c = CASES[name]
    rng = np.random.default_rng(sum(map(ord, name)))
    f = _field(rng, c["n"])
    if c.get("coincident"):
        f.positions[:] = f.positions[0]
    pts = rng.uniform(-0.95, 0.95, (c["b"], 3))
    if c.get("outside"):
        pts = rng.uniform(-3.0, 3.0, (c["b"], 3))
    if c.get("boundary"):
        pts = (rng.integers(0, c["g"] + 1, (c["b"], 3)) / (c["g"] / 2.0)) - 1.0  # exact cell edges
    up = rng.normal(size=c["b"])
    grid = build(f, c["g"], c["r"])
    if not psf:
        got = render_points(f, grid, None, Batch(pts), radius=c["r"])
        _, want_i, want_c = O.render_points(f.positions, f.quaternions, f.log_scales, f.intensity_logits, c["g"],
                                            c["r"], pts)
        np.testing.assert_array_equal(got.contributor_counts, want_c)
        assert_rel(got.intensities, want_i, atol=1e-10, name=name)
        gg = render_backward(f, grid, None, Batch(pts), up, radius=c["r"])
        og = O.render_backward(f.positions, f.quaternions, f.log_scales, f.intensity_logits, c["g"], c["r"], pts, up)
        for k in ("d_positions", "d_quaternions", "d_log_scales", "d_intensity_logits"):
            assert_grad_close(getattr(gg, k), getattr(og, k), name=f"{name}:{k}")
    else:
        # one slice (identity transform) with a 3-tap through-plane profile along z
        from paper_2603_00145_b200.core import TransformSet

        ts = TransformSet(np.array([[1.0, 0, 0, 0]]), np.zeros((1, 3)))
        sids = np.zeros(c["b"], np.int64)
        dirs = np.array([[0.0, 0.0, 1.0]])
        sp = SlicePSF(offsets=np.array([-0.05, 0.0, 0.05]), weights=np.array([0.3, 0.4, 0.3]), through_dirs=dirs)
        got = render_points(f, grid, ts, Batch(pts, sids), radius=c["r"], slice_psf=sp)
        want, wcnt = O.psf_render(f.positions, f.quaternions, f.log_scales, f.intensity_logits, c["g"], c["r"], pts,
                                  sids, ts.quats, ts.translations, sp.offsets, sp.weights, dirs)
        np.testing.assert_array_equal(got.contributor_counts, wcnt)
        assert_rel(got.intensities, want, atol=1e-10, name=name + ":psf")
        gg = render_backward(f, grid, ts, Batch(pts, sids), up, radius=c["r"], slice_psf=sp)
        og = O.psf_backward(f.positions, f.quaternions, f.log_scales, f.intensity_logits, c["g"], c["r"], pts, sids,
                            ts.quats, ts.translations, sp.offsets, sp.weights, dirs, up)
        for k in ("d_positions", "d_quaternions", "d_log_scales", "d_intensity_logits", "d_transform_params"):
            assert_grad_close(getattr(gg, k), getattr(og, k), name=f"{name}:psf:{k}")
