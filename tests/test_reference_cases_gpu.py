"""The reference's own forward / gradient / volume cases
(/root/reference/pkg/tests/test_render.py:59-317, conftest.py:9-38) run against
this package's modules (render, spatial, core swapped in for mgauss.*).

The closed forms, dense-oracle sums and float64 central-difference gradient
checks are stated at the reference's tolerances (atol 1e-12 / 1e-10, FD
rtol 1e-4 atol 1e-8 with step 1e-5), which need float64 pair arithmetic: they
run with ``render.set_strict_fp64(True)`` (mg_block_forward_f64 /
mg_block_backward_f64).  The structural cases (locality bit-identity, exact
zeros, identity transforms) also run on the default float32 kernels.
"""

import numpy as np
import pytest

from conftest import central_difference

pytestmark = pytest.mark.gpu


class Batch:
    def __init__(self, coords, slice_ids=None):
        self.coords = np.asarray(coords, dtype=np.float64)
        self.slice_ids = (np.full(self.coords.shape[0], -1, dtype=np.int64) if slice_ids is None
                          else np.asarray(slice_ids, dtype=np.int64))


def random_field(rng, side=3, scale_lo=-2.2, scale_hi=-0.7):
    """conftest.py:27-38."""
    from paper_2603_00145_b200.core import GaussianField, lattice_node_index

    n = side ** 3
    return GaussianField(positions=rng.uniform(-0.8, 0.8, (n, 3)),
                         quaternions=rng.normal(0.0, 1.0, (n, 4)) + np.array([2.0, 0, 0, 0]),
                         log_scales=rng.uniform(scale_lo, scale_hi, (n, 3)),
                         intensity_logits=rng.normal(0.0, 1.5, n), lattice_dims=(side, side, side),
                         lattice_index=lattice_node_index(side)).validate()


def single_gaussian(alpha=0.8, mu=(0.0, 0.0, 0.0), log_scales=(0.0, 0.0, 0.0)):
    from paper_2603_00145_b200.core import uniform_lattice_field

    f = uniform_lattice_field(1)
    f.positions[0] = mu
    f.log_scales[0] = log_scales
    f.intensity_logits[0] = np.log(alpha / (1.0 - alpha))
    return f


def dense_oracle(field, points):
    """Independent dense sum with a numeric inverse of R S S^T R^T (test_render.py:44-56)."""
    from paper_2603_00145_b200.core import quat_to_rotation, sigmoid

    rot = quat_to_rotation(field.quaternions / np.linalg.norm(field.quaternions, axis=1, keepdims=True))
    alphas = sigmoid(field.intensity_logits)
    out = np.zeros(points.shape[0])
    for i in range(field.count):
        sigma = rot[i] @ np.diag(np.exp(field.log_scales[i]) ** 2) @ rot[i].T
        d = points - field.positions[i]
        out += alphas[i] * np.exp(-0.5 * np.einsum("bi,ij,bj->b", d, np.linalg.inv(sigma), d))
    return out


@pytest.fixture(params=["strict_fp64"])
def strict(request):
    from paper_2603_00145_b200 import render

    prev = render.get_strict_fp64()
    render.set_strict_fp64(True)
    yield
    render.set_strict_fp64(prev)


@pytest.fixture(params=["fp32", "strict_fp64"])
def any_mode(request):
    from paper_2603_00145_b200 import render

    prev = render.get_strict_fp64()
    render.set_strict_fp64(request.param == "strict_fp64")
    yield request.param
    render.set_strict_fp64(prev)


# ---- TestForward (test_render.py:59-144) ------------------------------------

def test_query_at_center(strict):
    from paper_2603_00145_b200.render import render_points
    from paper_2603_00145_b200.spatial import build

    f = single_gaussian(alpha=0.8)
    out = render_points(f, build(f, 1), None, Batch([[0.0, 0.0, 0.0]]))
    np.testing.assert_allclose(out.intensities, [0.8], atol=1e-12)
    assert out.contributor_counts[0] == 1


def test_query_at_mahalanobis_sqrt2(strict):
    from paper_2603_00145_b200.render import render_points
    from paper_2603_00145_b200.spatial import build

    f = single_gaussian(alpha=0.8)
    out = render_points(f, build(f, 1), None, Batch(np.sqrt(2.0) * np.array([[1.0, 0.0, 0.0]])))
    np.testing.assert_allclose(out.intensities, [0.8 * np.exp(-1.0)], atol=1e-12)


def test_matches_dense_oracle_at_full_radius(strict, rng):
    from paper_2603_00145_b200.core import GaussianField
    from paper_2603_00145_b200.render import render_points
    from paper_2603_00145_b200.spatial import build

    f = random_field(rng, side=4)
    f2 = GaussianField(positions=f.positions[:50], quaternions=f.quaternions[:50], log_scales=f.log_scales[:50],
                       intensity_logits=f.intensity_logits[:50], lattice_dims=(50, 1, 1),
                       lattice_index=np.zeros((50, 3), dtype=np.int64))
    pts = rng.uniform(-1, 1, (200, 3))
    got = render_points(f2, build(f2, 8), None, Batch(pts), radius=8).intensities
    np.testing.assert_allclose(got, dense_oracle(f2, pts), atol=1e-10)


def test_empty_neighborhood_yields_zero(any_mode):
    from paper_2603_00145_b200.render import render_points
    from paper_2603_00145_b200.spatial import build

    f = single_gaussian(mu=(0.9, 0.9, 0.9))
    out = render_points(f, build(f, 20), None, Batch([[-0.9, -0.9, -0.9]]), radius=0)
    assert out.intensities[0] == 0.0
    assert out.contributor_counts[0] == 0


def test_inconsistent_grid(any_mode, rng):
    from paper_2603_00145_b200.errors import InconsistentGrid
    from paper_2603_00145_b200.render import render_points
    from paper_2603_00145_b200.spatial import build

    f = random_field(rng, side=3)
    with pytest.raises(InconsistentGrid):
        render_points(f, build(f.positions[:-2], 8), None, Batch(np.zeros((1, 3))))


def test_locality_bit_identical(any_mode, rng):
    from paper_2603_00145_b200.render import render_points
    from paper_2603_00145_b200.spatial import build

    f = random_field(rng, side=3)
    f.positions[:] = rng.uniform(-0.2, 0.2, f.positions.shape)
    f.positions[0] = [0.95, 0.95, 0.95]
    pts = rng.uniform(-0.2, 0.2, (40, 3))
    before = render_points(f, build(f, 16), None, Batch(pts), radius=2).intensities
    f.intensity_logits[0] += 3.0
    f.log_scales[0] += 0.5
    after = render_points(f, build(f, 16), None, Batch(pts), radius=2).intensities
    np.testing.assert_array_equal(before, after)


def test_superposition(strict, rng):
    from paper_2603_00145_b200.core import GaussianField
    from paper_2603_00145_b200.render import render_points
    from paper_2603_00145_b200.spatial import build

    fa, fb = random_field(rng, side=3), random_field(rng, side=3)
    union = GaussianField(positions=np.concatenate([fa.positions, fb.positions]),
                          quaternions=np.concatenate([fa.quaternions, fb.quaternions]),
                          log_scales=np.concatenate([fa.log_scales, fb.log_scales]),
                          intensity_logits=np.concatenate([fa.intensity_logits, fb.intensity_logits]),
                          lattice_dims=(54, 1, 1), lattice_index=np.zeros((54, 3), dtype=np.int64))
    pts = rng.uniform(-1, 1, (60, 3))
    g = 8
    i_u = render_points(union, build(union, g), None, Batch(pts), radius=g).intensities
    i_a = render_points(fa, build(fa, g), None, Batch(pts), radius=g).intensities
    i_b = render_points(fb, build(fb, g), None, Batch(pts), radius=g).intensities
    np.testing.assert_allclose(i_u, i_a + i_b, atol=1e-12)


def test_identity_transforms_match_untransformed(any_mode, rng):
    from paper_2603_00145_b200.core import TransformSet
    from paper_2603_00145_b200.render import render_points
    from paper_2603_00145_b200.spatial import build

    f = random_field(rng, side=3)
    grid = build(f, 6)
    pts = rng.uniform(-1, 1, (30, 3))
    sids = rng.integers(0, 4, 30)
    with_t = render_points(f, grid, TransformSet.identity(4), Batch(pts, sids), radius=6)
    without = render_points(f, grid, None, Batch(pts), radius=6)
    np.testing.assert_array_equal(with_t.intensities, without.intensities)
    np.testing.assert_array_equal(with_t.points, pts)


# ---- TestBackward (test_render.py:147-174) -----------------------------------

def test_zero_upstream(any_mode, rng):
    from paper_2603_00145_b200.render import render_backward
    from paper_2603_00145_b200.spatial import build

    f = random_field(rng, side=3)
    g = render_backward(f, build(f, 6), None, Batch(rng.uniform(-1, 1, (10, 3))), np.zeros(10), radius=6)
    for a in (g.d_positions, g.d_quaternions, g.d_log_scales, g.d_intensity_logits):
        assert np.all(a == 0.0)


def test_position_grad_zero_at_center(any_mode):
    from paper_2603_00145_b200.render import render_backward
    from paper_2603_00145_b200.spatial import build

    f = single_gaussian()
    g = render_backward(f, build(f, 1), None, Batch([[0.0, 0.0, 0.0]]), np.ones(1))
    np.testing.assert_allclose(g.d_positions, 0.0, atol=1e-15)


def test_untouched_primitives_get_exact_zero(any_mode, rng):
    from paper_2603_00145_b200.render import render_backward
    from paper_2603_00145_b200.spatial import build

    f = random_field(rng, side=3)
    f.positions[:] = rng.uniform(-0.2, 0.2, f.positions.shape)
    f.positions[5] = [0.95, 0.95, 0.95]
    g = render_backward(f, build(f, 16), None, Batch(rng.uniform(-0.2, 0.2, (20, 3))), rng.normal(size=20),
                        radius=2)
    assert np.all(g.d_positions[5] == 0.0) and np.all(g.d_quaternions[5] == 0.0)
    assert np.all(g.d_log_scales[5] == 0.0) and g.d_intensity_logits[5] == 0.0


# ---- TestGradientsAgainstFiniteDifferences (test_render.py:177-259) -----------

def make_gradcheck_setup(rng, n_side=2, n_points=8, n_slices=3):
    from paper_2603_00145_b200.core import TransformSet

    field = random_field(rng, side=n_side)
    coords = rng.uniform(-0.7, 0.7, (n_points, 3))
    sids = rng.integers(0, n_slices, n_points)
    ts = TransformSet(quats=rng.normal(0, 0.1, (n_slices, 4)) + np.array([1.0, 0, 0, 0]),
                      translations=rng.normal(0, 0.05, (n_slices, 3)))
    return field, coords, sids, ts, rng.normal(size=n_points)


def render_scalar_loss(field, ts, coords, sids, upstream):
    from paper_2603_00145_b200.render import render_points
    from paper_2603_00145_b200.spatial import build

    g = field.lattice_dims[0] + 2
    out = render_points(field, build(field, g), ts, Batch(coords, sids), radius=g)
    return float(np.sum(upstream * out.intensities))


def analytic_gradients(field, ts, coords, sids, upstream):
    from paper_2603_00145_b200.render import render_backward
    from paper_2603_00145_b200.spatial import build

    g = field.lattice_dims[0] + 2
    return render_backward(field, build(field, g), ts, Batch(coords, sids), upstream, radius=g)


@pytest.mark.parametrize("attr,grad", [("positions", "d_positions"), ("quaternions", "d_quaternions"),
                                       ("log_scales", "d_log_scales"), ("intensity_logits", "d_intensity_logits")])
def test_fd_parameter_group(strict, rng, attr, grad):
    field, coords, sids, ts, upstream = make_gradcheck_setup(rng)
    grads = analytic_gradients(field, ts, coords, sids, upstream)
    fd = central_difference(lambda arr: render_scalar_loss(field, ts, coords, sids, upstream), getattr(field, attr))
    np.testing.assert_allclose(getattr(grads, grad), fd, rtol=1e-4, atol=1e-8)


def test_fd_transform_parameters(strict, rng):
    field, coords, sids, ts, upstream = make_gradcheck_setup(rng)
    grads = analytic_gradients(field, ts, coords, sids, upstream)
    loss = lambda arr: render_scalar_loss(field, ts, coords, sids, upstream)  # noqa: E731
    np.testing.assert_allclose(grads.d_transform_params[:, :4], central_difference(loss, ts.quats),
                               rtol=1e-4, atol=1e-8)
    np.testing.assert_allclose(grads.d_transform_params[:, 4:], central_difference(loss, ts.translations),
                               rtol=1e-4, atol=1e-8)


def test_fd_query_point_gradient(strict, rng):
    field, coords, sids, ts, upstream = make_gradcheck_setup(rng)
    grads = analytic_gradients(field, ts, coords, sids, upstream)
    analytic = np.einsum("bij,bi->bj", ts.rotations()[sids], grads.d_points)
    fd = central_difference(lambda arr: render_scalar_loss(field, ts, coords, sids, upstream), coords)
    np.testing.assert_allclose(analytic, fd, rtol=1e-4, atol=1e-8)


def test_fd_slice_psf_gradients(strict, rng):
    """Extension (A17): FD checks of the PSF-integrated render, same tolerances."""
    from paper_2603_00145_b200.render import SlicePSF, render_backward, render_points
    from paper_2603_00145_b200.spatial import build

    field, coords, sids, ts, upstream = make_gradcheck_setup(rng)
    dirs = rng.normal(size=(3, 3))
    psf = SlicePSF(np.array([-0.03, 0.0, 0.03]), np.array([0.3, 0.4, 0.3]),
                   dirs / np.linalg.norm(dirs, axis=1, keepdims=True))
    g = field.lattice_dims[0] + 2

    def loss(arr):
        out = render_points(field, build(field, g), ts, Batch(coords, sids), radius=g, slice_psf=psf)
        return float(np.sum(upstream * out.intensities))

    gr = render_backward(field, build(field, g), ts, Batch(coords, sids), upstream, radius=g, slice_psf=psf)
    np.testing.assert_allclose(gr.d_positions, central_difference(loss, field.positions), rtol=1e-4, atol=1e-8)
    np.testing.assert_allclose(gr.d_log_scales, central_difference(loss, field.log_scales), rtol=1e-4, atol=1e-8)
    np.testing.assert_allclose(gr.d_transform_params[:, 4:], central_difference(loss, ts.translations),
                               rtol=1e-4, atol=1e-8)


# ---- TestSampleVolume (test_render.py:262-308) + block == dense (:311-317) ----

def test_volume_empty_field(any_mode):
    from paper_2603_00145_b200.core import GaussianField
    from paper_2603_00145_b200.render import sample_volume
    from paper_2603_00145_b200.spatial import build

    f = GaussianField(np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 3)), np.zeros(0), (0, 0, 0),
                      np.zeros((0, 3), dtype=np.int64))
    assert np.all(sample_volume(f, build(f, 4), None, (8, 8, 8)).data == 0.0)


def test_volume_center_gaussian_peak_and_decay(any_mode):
    from paper_2603_00145_b200.render import sample_volume
    from paper_2603_00145_b200.spatial import build

    f = single_gaussian(alpha=0.9, log_scales=(-1.0, -1.0, -1.0))
    vol = sample_volume(f, build(f, 1), None, (33, 33, 33))
    assert vol.data.argmax() == np.ravel_multi_index((16, 16, 16), (33, 33, 33))
    line = vol.data[:, 16, 16]
    assert np.all(np.diff(line[:17]) > 0) and np.all(np.diff(line[16:]) < 0)


def test_volume_subsample_coordinate_identity(strict, rng):
    from paper_2603_00145_b200.render import sample_volume
    from paper_2603_00145_b200.spatial import build

    f = random_field(rng, side=3)
    grid = build(f, 3)
    lo, hi = -1.0, 1.0
    step = (hi - lo) / 63.0
    v64 = sample_volume(f, grid, None, (64, 64, 64), ((lo,) * 3, (hi,) * 3), radius=3)
    v32 = sample_volume(f, grid, None, (32, 32, 32), ((lo,) * 3, (hi - step,) * 3), radius=3)
    np.testing.assert_allclose(v64.data[::2, ::2, ::2], v32.data, atol=1e-12)


def test_volume_out_of_memory_guard(any_mode, rng):
    from paper_2603_00145_b200.errors import OutOfMemoryRequest
    from paper_2603_00145_b200.render import sample_volume
    from paper_2603_00145_b200.spatial import build

    f = random_field(rng, side=2)
    with pytest.raises(OutOfMemoryRequest):
        sample_volume(f, build(f, 2), None, (4096, 4096, 4096))


def test_volume_clamped_to_unit_range(any_mode, rng):
    from paper_2603_00145_b200.render import sample_volume
    from paper_2603_00145_b200.spatial import build

    f = random_field(rng, side=2)
    f.intensity_logits[:] = 6.0
    vol = sample_volume(f, build(f, 2), None, (12, 12, 12), radius=2)
    assert vol.data.max() <= 1.0 and vol.data.min() >= 0.0


def test_dense_reference_matches_block_at_full_radius(strict, rng):
    from paper_2603_00145_b200.render import render_points, render_points_dense
    from paper_2603_00145_b200.spatial import build

    f = random_field(rng, side=3)
    pts = rng.uniform(-1, 1, (100, 3))
    block = render_points(f, build(f, 5), None, Batch(pts), radius=5).intensities
    np.testing.assert_allclose(block, render_points_dense(f, pts), atol=1e-12)


def test_strict_matches_oracle_bitwise_close(strict, rng):
    """Strict kernels vs the C oracle (same float64 op order): counts exact,
    intensities and d_points within 1e-13 relative, accumulators within 1e-12."""
    from oracle import oracle as O
    from paper_2603_00145_b200.core import TransformSet
    from paper_2603_00145_b200.render import render_backward, render_points
    from paper_2603_00145_b200.spatial import build

    f = random_field(rng, side=6)
    k = 4
    ts = TransformSet(rng.normal(0, 0.05, (k, 4)) + [1, 0, 0, 0], rng.normal(0, 0.02, (k, 3)))
    pts = rng.uniform(-1, 1, (3000, 3))
    sids = rng.integers(-1, k, 3000)
    up = rng.normal(size=3000)
    grid = build(f, 12, 3)
    out = render_points(f, grid, ts, Batch(pts, sids))
    gr = render_backward(f, grid, ts, Batch(pts, sids), up)
    x, inten, cnt = O.render_points(f.positions, f.quaternions, f.log_scales, f.intensity_logits, 12, 3, pts, sids,
                                    ts.quats, ts.translations)
    og = O.render_backward(f.positions, f.quaternions, f.log_scales, f.intensity_logits, 12, 3, pts, up, sids,
                           ts.quats, ts.translations)
    np.testing.assert_array_equal(out.contributor_counts, cnt)
    np.testing.assert_allclose(out.intensities, inten, rtol=1e-13, atol=1e-300)
    np.testing.assert_allclose(gr.d_points, og.d_points, rtol=1e-12, atol=1e-14)
    for name in ("d_positions", "d_quaternions", "d_log_scales", "d_intensity_logits", "d_transform_params"):
        a, w = getattr(gr, name), getattr(og, name)
        np.testing.assert_allclose(a, w, rtol=1e-10, atol=1e-12 * np.abs(w).max(), err_msg=name)
