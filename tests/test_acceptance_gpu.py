"""The reference's acceptance suite (/root/reference/pkg/tests/test_acceptance.py),
the criteria that fall on the hot path, run against this package:

1. gradient suite (test_acceptance.py:114-201): central differences
   (step 1e-5, rtol 1e-4, atol 1e-8) of every render parameter group and
   the slice transforms on random side-2 fields with radius = G (strict
   float64 kernels), and of the residual field's weights and biases --
   small networks (2 bands, hidden (8, 8)) fully and the production
   architecture on sampled entries (float64 NRF kernels);
2. query oracle (test_acceptance.py:209-246): query_local against the
   Chebyshev rule for 10,000 queries, radius >= G returning everything, and
   full-radius rendering against an independent dense sum to 1e-10;
6. loss unit values (test_acceptance.py:310-320);
7. block speedup -- tests/test_speedup_gpu.py;
9. per-primitive parameter count (test_acceptance.py:400-420).
Criterion 3 (desk-scale reconstruction) is tests/test_recon_gpu.py and
test_strict_train_gpu.py; 8 (determinism, persistence) is test_checkpoint_gpu.py
and the graph-vs-eager tests; 4 and 5 (ablations, radius sweep) are CLI
experiments outside the hot path.
"""

import numpy as np
import pytest

from conftest import central_difference
from test_reference_cases_gpu import Batch, random_field

pytestmark = pytest.mark.gpu


@pytest.fixture
def strict_mode():
    from paper_2603_00145_b200 import render

    prev = render.get_strict_fp64()
    render.set_strict_fp64(True)
    yield
    render.set_strict_fp64(prev)


def test_criterion_1_render_gradient_suite(strict_mode):
    from paper_2603_00145_b200.core import TransformSet
    from paper_2603_00145_b200.render import render_backward, render_points
    from paper_2603_00145_b200.spatial import build

    rng = np.random.default_rng(101)
    for _ in range(100):  # as the reference
        field = random_field(rng, side=2)
        coords = rng.uniform(-0.7, 0.7, (5, 3))
        sids = rng.integers(0, 2, 5)
        ts = TransformSet(rng.normal(0, 0.1, (2, 4)) + np.array([1.0, 0, 0, 0]), rng.normal(0, 0.05, (2, 3)))
        upstream = rng.normal(size=5)
        g = field.lattice_dims[0] + 2

        def loss(_=None):
            out = render_points(field, build(field, g), ts, Batch(coords, sids), radius=g)
            return float(np.sum(upstream * out.intensities))

        grads = render_backward(field, build(field, g), ts, Batch(coords, sids), upstream, radius=g)
        checks = [(grads.d_positions, field.positions), (grads.d_quaternions, field.quaternions),
                  (grads.d_log_scales, field.log_scales), (grads.d_intensity_logits, field.intensity_logits),
                  (grads.d_transform_params[:, :4], ts.quats), (grads.d_transform_params[:, 4:], ts.translations)]
        for analytic, param in checks:
            fd = central_difference(lambda a: loss(), param)
            np.testing.assert_allclose(analytic, fd, rtol=1e-4, atol=1e-8)


def test_criterion_1_nrf_gradient_suite():
    from paper_2603_00145_b200.nrf import ResidualField64, nrf_backward64, nrf_forward64

    rng = np.random.default_rng(101)
    for _ in range(100):  # small networks, every weight and bias
        f = ResidualField64.create(rng, frequency_bands=2, hidden=(8, 8))
        for w in f.weights:
            w[:] = rng.normal(0, 0.6, w.shape)
        for b in f.biases:
            b[:] = rng.normal(0, 0.3, b.shape)
        x = rng.uniform(-1, 1, (4, 3))
        upstream = rng.normal(size=4)

        def nloss(_=None):
            return float(np.sum(upstream * nrf_forward64(f, x)))

        dws, dbs, _ = nrf_backward64(f, x, upstream)
        for li in range(len(f.weights)):
            np.testing.assert_allclose(dws[li], central_difference(lambda a: nloss(), f.weights[li]), rtol=1e-4,
                                       atol=1e-8)
            np.testing.assert_allclose(dbs[li], central_difference(lambda a: nloss(), f.biases[li]), rtol=1e-4,
                                       atol=1e-8)
    for _ in range(3):  # the production architecture on sampled entries
        f = ResidualField64.create(rng)
        for w in f.weights:
            w[:] = rng.normal(0, 0.3, w.shape)
        x = rng.uniform(-1, 1, (4, 3))
        upstream = rng.normal(size=4)
        dws, _, _ = nrf_backward64(f, x, upstream)

        def nloss(_=None):
            return float(np.sum(upstream * nrf_forward64(f, x)))

        for li in (0, 2, 4):
            w = f.weights[li]
            for _ in range(15):
                i, j = int(rng.integers(w.shape[0])), int(rng.integers(w.shape[1]))
                orig = w[i, j]
                w[i, j] = orig + 1e-5
                fp = nloss()
                w[i, j] = orig - 1e-5
                fm = nloss()
                w[i, j] = orig
                np.testing.assert_allclose(dws[li][i, j], (fp - fm) / 2e-5, rtol=1e-4, atol=1e-8)


def test_criterion_1_nrf_input_gradient():
    """d_points (into the slice transforms) by central differences on x."""
    from paper_2603_00145_b200.nrf import ResidualField64, nrf_backward64, nrf_forward64

    rng = np.random.default_rng(7)
    f = ResidualField64.create(rng)
    for w in f.weights:
        w[:] = rng.normal(0, 0.3, w.shape)
    x = rng.uniform(-1, 1, (6, 3))
    up = rng.normal(size=6)
    _, _, dp = nrf_backward64(f, x, up)
    fd = central_difference(lambda a: float(np.sum(up * nrf_forward64(f, x))), x)
    np.testing.assert_allclose(dp, fd, rtol=1e-4, atol=1e-8)


def test_criterion_2_query_oracle(strict_mode):
    from paper_2603_00145_b200.core import quat_to_rotation
    from paper_2603_00145_b200.render import render_points
    from paper_2603_00145_b200.spatial import build, cell_index, query_local

    rng = np.random.default_rng(202)
    field = random_field(rng, side=11)  # 1331 primitives
    field.positions[:] = rng.uniform(-1.05, 1.05, field.positions.shape)
    g = 16
    grid = build(field, g, block_radius=5)
    cells = cell_index(field.positions, g)
    queries = rng.uniform(-1.1, 1.1, (10000, 3))
    qcells = cell_index(queries, g)
    for q in range(queries.shape[0]):
        cheb = np.max(np.abs(cells - qcells[q][None, :]), axis=1)
        np.testing.assert_array_equal(query_local(grid, queries[q]), np.nonzero(cheb <= 5)[0])
    for q in range(100):
        np.testing.assert_array_equal(query_local(grid, queries[q], radius=g), np.arange(field.count))
    pts = rng.uniform(-1, 1, (300, 3))
    got = render_points(field, grid, None, Batch(pts, np.full(300, -1, dtype=np.int64)), radius=g).intensities
    rot = quat_to_rotation(field.quaternions)
    alphas = 1.0 / (1.0 + np.exp(-field.intensity_logits))
    want = np.zeros(300)
    for i in range(field.count):
        prec = np.linalg.inv(rot[i] @ np.diag(np.exp(field.log_scales[i]) ** 2) @ rot[i].T)
        d = pts - field.positions[i]
        want += alphas[i] * np.exp(-0.5 * np.einsum("bi,ij,bj->b", d, prec, d))
    np.testing.assert_allclose(got, want, atol=1e-10)


def test_criterion_6_loss_unit_values():
    from paper_2603_00145_b200.core import uniform_lattice_field
    from paper_2603_00145_b200.ssim import ssim_loss
    from paper_2603_00145_b200.train import aniso_loss, smooth_l1

    assert smooth_l1(0.0, 0.0) == 0.0
    assert smooth_l1(0.5, 0.0) == 0.125
    assert smooth_l1(2.0, 0.0) == 1.5
    f = uniform_lattice_field(1)
    f.log_scales[0] = np.log([3.0, 1.0, 1.0])
    assert aniso_loss(f, 1.5) == pytest.approx(1.5, abs=1e-12)
    img = np.random.default_rng(6).uniform(0, 1, (24, 24))
    assert abs(ssim_loss(img, img)) < 1e-12


def test_ssim_module_errors():
    from paper_2603_00145_b200.errors import ShapeMismatch, SliceTooSmall
    from paper_2603_00145_b200.ssim import ssim_loss

    with pytest.raises(ShapeMismatch):
        ssim_loss(np.zeros((20, 20)), np.zeros((20, 21)))
    with pytest.raises(SliceTooSmall):
        ssim_loss(np.zeros((10, 20)), np.zeros((10, 20)))


def test_criterion_9_parameter_count(tmp_path):
    """11 learnable parameters per primitive in a saved checkpoint
    (test_acceptance.py:400-420)."""
    from types import SimpleNamespace

    from paper_2603_00145_b200.core import TransformSet
    from paper_2603_00145_b200.io import load_checkpoint, save_checkpoint
    from paper_2603_00145_b200.train import TrainConfig, Trainer

    rng = np.random.default_rng(9)
    cloud = SimpleNamespace(coords=rng.uniform(-0.9, 0.9, (500, 3)), intensities=rng.uniform(0.1, 0.9, 500),
                            slice_ids=np.zeros(500, dtype=np.int64))
    cfg = TrainConfig(resolution_schedule=((0, 5),), total_iters=1, batch_points=128, use_ssim=False)
    tr = Trainer(cloud, TransformSet.identity(1), cfg)
    tr.step()
    path = tmp_path / "c.mgss"
    save_checkpoint(path, {"trainer": tr.state_dict()})
    state = load_checkpoint(path)["trainer"]["field"]
    n = tr.field.count
    per = sum(np.asarray(state[k]).size for k in ("positions", "quaternions", "log_scales", "intensity_logits")) / n
    assert per == 11 == tr.field.to_host().params_per_primitive
    tr.close()
