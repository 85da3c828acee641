"""The reference's module tests for the rest of the hot path --
pkg/tests/test_ssim.py, test_train.py, test_nrf.py and test_spatial.py --
restated against this package (render is tests/test_reference_cases_gpu.py),
at the reference's tolerances.  The float64 host-level API carries the
float64 cases; the production float32 residual field the structural ones.
Out of scope and not restated: the 3-D SSIM metric (metrics), fourier_encode /
silu helpers (the kernels encode internally), the simulator-based fixtures
(the toy cloud below is built directly)."""

from types import SimpleNamespace

import numpy as np
import pytest

from conftest import central_difference
from test_reference_cases_gpu import random_field

pytestmark = pytest.mark.gpu


@pytest.fixture
def rng():
    return np.random.default_rng(20260808)


# --------------------------------------------------------------------------- ssim (test_ssim.py)


def _windowed_ssim(a, b):
    """Per-window SSIM recomputed directly (an oracle independent of the
    separable passes): 11x11 outer-product Gaussian window."""
    from paper_2603_00145_b200.ssim import C1, C2, gaussian_window

    w1 = gaussian_window()
    w2 = np.outer(w1, w1)
    n = w1.size
    out = []
    for i in range(a.shape[0] - n + 1):
        for j in range(a.shape[1] - n + 1):
            pa, pb = a[i:i + n, j:j + n], b[i:i + n, j:j + n]
            ma, mb = np.sum(w2 * pa), np.sum(w2 * pb)
            va, vb = np.sum(w2 * pa * pa) - ma * ma, np.sum(w2 * pb * pb) - mb * mb
            cv = np.sum(w2 * pa * pb) - ma * mb
            out.append(((2 * ma * mb + C1) * (2 * cv + C2)) / ((ma * ma + mb * mb + C1) * (va + vb + C2)))
    return float(np.mean(out))


def test_ssim_closed_forms_and_oracle(rng):
    from paper_2603_00145_b200.ssim import C1, C2, gaussian_window, ssim_loss, ssim_mean

    img = rng.uniform(0, 1, (20, 20))
    assert abs(ssim_loss(img, img)) < 1e-12
    # zero vs one: zero variances leave only the C terms
    np.testing.assert_allclose(ssim_loss(np.zeros((16, 16)), np.ones((16, 16))),
                               1.0 - (C1 * C2) / ((1.0 + C1) * C2), atol=1e-15)
    a = rng.uniform(0, 1, (18, 23))
    b = np.clip(a + rng.normal(0, 0.1, a.shape), 0, 1)
    np.testing.assert_allclose(ssim_mean(a, b), _windowed_ssim(a, b), atol=1e-8)
    w = gaussian_window()
    assert w.shape == (11,)
    np.testing.assert_allclose(w.sum(), 1.0, atol=1e-15)


def test_ssim_gradient(rng):
    from paper_2603_00145_b200.ssim import ssim_loss, ssim_loss_grad

    pred = rng.uniform(0.1, 0.9, (14, 15))
    target = np.clip(pred + rng.normal(0, 0.15, pred.shape), 0, 1)
    _, grad = ssim_loss_grad(pred, target)
    fd = central_difference(lambda arr: ssim_loss_grad(pred, target)[0], pred, step=1e-6)
    np.testing.assert_allclose(grad, fd, rtol=1e-4, atol=1e-9)
    img = rng.uniform(0.2, 0.8, (16, 16))
    loss, grad = ssim_loss_grad(img, img.copy())
    assert abs(loss) < 1e-12
    np.testing.assert_allclose(grad, 0.0, atol=1e-10)
    p, t = rng.uniform(0, 1, (17, 13)), rng.uniform(0, 1, (17, 13))
    np.testing.assert_allclose(ssim_loss_grad(p, t)[0], ssim_loss(p, t), atol=1e-14)


# --------------------------------------------------------------------------- losses, Adam (test_train.py)


def test_smooth_l1(rng):
    from paper_2603_00145_b200.train import smooth_l1, smooth_l1_grad

    assert smooth_l1(0.0, 0.0) == 0.0 and smooth_l1(0.5, 0.0) == 0.125 and smooth_l1(2.0, 0.0) == 1.5
    pred, target = rng.normal(size=100), rng.normal(size=100)
    x = pred - target
    np.testing.assert_allclose(smooth_l1(pred, target), np.mean(np.where(np.abs(x) < 1, 0.5 * x * x, np.abs(x) - 0.5)),
                               atol=1e-15)
    pred, target = rng.normal(size=20) * 2.0, rng.normal(size=20)
    fd = central_difference(lambda a: smooth_l1(pred, target), pred, step=1e-6)
    np.testing.assert_allclose(smooth_l1_grad(pred, target), fd, rtol=1e-6, atol=1e-10)


def test_aniso_loss(rng):
    from paper_2603_00145_b200.core import uniform_lattice_field
    from paper_2603_00145_b200.train import aniso_loss, aniso_loss_grad

    assert aniso_loss(uniform_lattice_field(3), 1.5) == 0.0
    f = uniform_lattice_field(1)
    f.log_scales[0] = np.log([3.0, 1.0, 1.0])
    np.testing.assert_allclose(aniso_loss(f, 1.5), 1.5, atol=1e-12)
    f = random_field(rng, side=4)
    e = np.exp(f.log_scales)
    want = np.mean(np.maximum(0.0, e.max(axis=1) / e.min(axis=1) - 1.5))
    np.testing.assert_allclose(aniso_loss(f, 1.5), want, atol=1e-12)
    f = random_field(rng, side=2)
    _, grad = aniso_loss_grad(f, 1.2)
    fd = central_difference(lambda a: aniso_loss(f, 1.2), f.log_scales, step=1e-7)
    np.testing.assert_allclose(grad, fd, rtol=1e-5, atol=1e-10)


def test_adam(rng):
    from paper_2603_00145_b200.train import AdamState

    adam = AdamState(beta1=0.0, beta2=0.0, eps=1e-8)
    p, g = rng.normal(size=50), rng.normal(size=50)
    p0 = p.copy()
    adam.step("g", {"p": p}, {"p": g}, lr=0.1)
    np.testing.assert_allclose(p, p0 - 0.1 * g / (np.abs(g) + 1e-8), atol=1e-15)
    adam = AdamState(beta1=0.9, beta2=0.999, eps=1e-8)
    p = np.zeros(4)
    for _ in range(3):
        adam.step("g", {"p": p}, {"p": np.ones(4)}, lr=0.01)
    st = adam.state_dict()
    assert st["g"]["t"] == 3
    np.testing.assert_allclose(st["g"]["m"]["p"], 1.0 - 0.9 ** 3, atol=1e-12)
    adam = AdamState()
    p = rng.normal(size=20)
    before = p.copy()
    adam.step("g", {"p": p}, {"p": rng.normal(size=20)}, lr=0.0)
    np.testing.assert_array_equal(p, before)
    adam.reset_group("g")
    assert "g" not in adam.groups
    a = AdamState()
    p = rng.normal(size=6)
    a.step("a", {"p": p}, {"p": rng.normal(size=6)}, lr=0.1)
    b = AdamState()
    b.load_state_dict(a.state_dict())
    p1, p2, g = p.copy(), p.copy(), rng.normal(size=6)
    a.step("a", {"p": p1}, {"p": g}, lr=0.1)
    b.step("a", {"p": p2}, {"p": g}, lr=0.1)
    np.testing.assert_array_equal(p1, p2)


# --------------------------------------------------------------------------- upsample, init (test_train.py)


def test_progressive_upsample_cases(rng):
    from paper_2603_00145_b200.core import normalize_quat, uniform_lattice_field
    from paper_2603_00145_b200.errors import ShrinkNotAllowed
    from paper_2603_00145_b200.train import progressive_upsample

    with pytest.raises(ShrinkNotAllowed):
        progressive_upsample(uniform_lattice_field(4), 3)
    f = uniform_lattice_field(4)  # identity resample of a drifted field
    f.intensity_logits[:] = rng.normal(size=f.count)
    f.log_scales[:] = rng.normal(0, 0.3, (f.count, 3))
    f.quaternions[:] = rng.normal(size=(f.count, 4)) + np.array([1.5, 0, 0, 0])
    f.positions += rng.normal(0, 0.01, f.positions.shape)
    out = progressive_upsample(f, 4)
    np.testing.assert_allclose(out.intensity_logits, f.intensity_logits, atol=1e-12)
    np.testing.assert_allclose(out.log_scales, f.log_scales, atol=1e-12)
    np.testing.assert_allclose(out.quaternions, normalize_quat(f.quaternions), atol=1e-12)
    np.testing.assert_allclose(out.positions, uniform_lattice_field(4).positions)
    f = uniform_lattice_field(3)  # constant field stays constant
    f.intensity_logits[:] = 0.7
    f.log_scales[:] = [-1.0, -1.2, -0.8]
    q = rng.normal(size=4) + np.array([1.0, 0, 0, 0])
    f.quaternions[:] = q
    out = progressive_upsample(f, 7)
    np.testing.assert_allclose(out.intensity_logits, 0.7, atol=1e-12)
    np.testing.assert_allclose(out.log_scales, np.broadcast_to([-1.0, -1.2, -0.8], (343, 3)), atol=1e-12)
    np.testing.assert_allclose(out.quaternions, np.broadcast_to(normalize_quat(q), (343, 4)), atol=1e-12)
    f = uniform_lattice_field(4)  # a logit ramp along x is reproduced at the new nodes
    f.intensity_logits[:] = 0.3 + 1.7 * f.positions[:, 0]
    out = progressive_upsample(f, 8)
    want = 0.3 + 1.7 * np.clip(out.positions[:, 0], f.positions[:, 0].min(), f.positions[:, 0].max())
    np.testing.assert_allclose(out.intensity_logits, want, atol=1e-10)
    q = rng.normal(size=4) * 3.0  # NLERP of equal quaternions
    f = uniform_lattice_field(2)
    f.quaternions[:] = q
    np.testing.assert_allclose(progressive_upsample(f, 5).quaternions,
                               np.broadcast_to(normalize_quat(q), (125, 4)), atol=1e-12)
    f = uniform_lattice_field(2)  # mixed-sign equivalents must not cancel
    q = np.array([0.5, 0.5, 0.5, 0.5])
    f.quaternions[:] = q
    f.quaternions[::2] = -q
    np.testing.assert_allclose(np.abs(progressive_upsample(f, 4).quaternions @ q), 1.0, atol=1e-12)


def _toy_cloud(rng, n=4000):
    coords = rng.uniform(-0.9, 0.9, (n, 3))
    return SimpleNamespace(coords=coords, intensities=np.exp(-np.sum(coords ** 2, axis=1) / 0.3) * 0.8,
                           slice_ids=np.zeros(n, dtype=np.int64))


def _toy_slice_grid():
    axis = np.linspace(-0.9, 0.9, 16)
    gx, gy = np.meshgrid(axis, axis, indexing="ij")
    coords = np.stack([gx.ravel(), gy.ravel(), np.zeros(256)], axis=1)
    return SimpleNamespace(coords=coords, target=np.exp(-(gx ** 2 + gy ** 2) / 0.3) * 0.8, slice_id=0)


def _toy_config(**kw):
    from paper_2603_00145_b200.train import TrainConfig

    base = dict(resolution_schedule=((0, 6), (60, 8)), total_iters=80, nrf_activation_iter=40, batch_points=1024,
                seed=3)
    base.update(kw)
    return TrainConfig(**base)


def test_init_field_seeding(rng):
    from paper_2603_00145_b200.spatial import cell_index
    from paper_2603_00145_b200.train import init_field

    cloud = _toy_cloud(rng)
    f = init_field(cloud, 8)
    assert f.count == 512
    cells = cell_index(cloud.coords, 8)
    flat = (cells[:, 0] * 8 + cells[:, 1]) * 8 + cells[:, 2]
    np.testing.assert_array_equal(f.intensity_logits[np.setdiff1d(np.arange(512), flat)], 0.0)
    mean = np.clip(cloud.intensities[flat == flat[0]].mean(), 1e-4, 1 - 1e-4)
    np.testing.assert_allclose(f.intensity_logits[flat[0]], np.log(mean / (1 - mean)), atol=1e-12)


# --------------------------------------------------------------------------- Trainer contracts (test_train.py)


def _trainer(rng, **kw):
    from paper_2603_00145_b200.core import TransformSet
    from paper_2603_00145_b200.train import Trainer

    cfg = _toy_config(**kw)
    grids = [_toy_slice_grid()] if cfg.use_ssim else None
    return Trainer(_toy_cloud(rng), TransformSet.identity(1), cfg, slice_grids=grids)


def test_trainer_contracts(rng):
    from paper_2603_00145_b200 import _device as dv
    from paper_2603_00145_b200.train import TrainConfig

    tr = _trainer(rng)
    rep = tr.step()  # loss decomposition
    np.testing.assert_allclose(rep.total, rep.data + 0.5 * rep.ssim + 0.1 * rep.aniso, atol=1e-12)
    tr.close()

    tr = _trainer(rng)  # the residual field is untouched before its activation, touched right after
    w0 = [dv.to_host(w).copy() for w in tr.nrf.weights]
    b0 = [dv.to_host(b).copy() for b in tr.nrf.biases]
    cfg = tr.config
    for _ in range(cfg.nrf_activation_iter):
        rep = tr.step()
        assert rep.resolution == cfg.resolution_at(rep.iteration)  # schedule conformance
    for a, w in zip(w0, tr.nrf.weights):
        np.testing.assert_array_equal(a, dv.to_host(w))
    for a, b in zip(b0, tr.nrf.biases):
        np.testing.assert_array_equal(a, dv.to_host(b))
    tr.step()
    assert any(np.any(dv.to_host(b) != a) for a, b in zip(b0, tr.nrf.biases))
    while tr.iteration < cfg.total_iters:
        rep = tr.step()
        assert rep.resolution == cfg.resolution_at(rep.iteration)
    tr.close()

    tr = _trainer(rng, use_progressive=False)  # fixed resolution when progressive is off
    assert tr.field.lattice_dims[0] == tr.config.final_resolution
    tr.step()
    assert tr.field.lattice_dims[0] == tr.config.final_resolution
    tr.close()

    tr = _trainer(rng)  # stored quaternions stay raw (moved by Adam, never renormalised)
    tr.field.quaternions *= 3.0
    before = dv.to_host(tr.field.quaternions).copy()
    tr.step()
    after = dv.to_host(tr.field.quaternions)
    assert not np.allclose(np.linalg.norm(after, axis=1), 1.0)
    assert np.max(np.abs(after - before)) < 0.1
    tr.close()

    tr = _trainer(rng, total_iters=200, resolution_schedule=((0, 6),), nrf_activation_iter=100, use_ssim=False)
    first = tr.step().data  # convergence smoke
    for _ in range(199):
        last = tr.step().data
    assert last < first
    tr.close()

    for bad in (dict(lr_position=0.0), dict(resolution_schedule=((0, 16), (10, 8))),
                dict(resolution_schedule=((5, 16),)), dict(resolution_schedule=((0, 16), (0, 24)))):
        with pytest.raises(ValueError):
            TrainConfig(**bad).validate()


# --------------------------------------------------------------------------- residual field (test_nrf.py)


def _scalar_nrf(field, point):
    """Per-point evaluation with plain Python loops (test_nrf.py:19-34's role)."""
    enc = [float(c) for c in point]
    for k in range(field.frequency_bands):
        f = (2.0 ** k) * np.pi
        enc += [np.sin(f * c) for c in point] + [np.cos(f * c) for c in point]
    h = enc
    for li, (w, b) in enumerate(zip(field.weights, field.biases)):
        z = [sum(h[i] * w[i, j] for i in range(len(h))) + b[j] for j in range(w.shape[1])]
        h = z if li == len(field.weights) - 1 else [v / (1.0 + np.exp(-v)) for v in z]
    return field.output_bound * np.tanh(h[0])


def test_nrf_forward_cases(rng):
    from paper_2603_00145_b200 import _device as dv
    from paper_2603_00145_b200.errors import UninitializedField
    from paper_2603_00145_b200.nrf import ResidualField, ResidualField64, nrf_forward, nrf_forward64

    f = ResidualField.create(np.random.default_rng(0))  # production field, float32 kernels
    assert f.layer_widths == (39, 64, 64, 64, 64, 1) and f.frequency_bands == 6 and f.output_bound == 0.1
    x = rng.uniform(-1, 1, (100, 3))
    np.testing.assert_array_equal(nrf_forward(f, x), 0.0)  # zero last layer: a no-op residual
    for w in f.weights:
        w.zero_()
    np.testing.assert_array_equal(nrf_forward(f, x), 0.0)
    for w in f.weights:
        w.copy_(dv.to_dev(rng.normal(0, 2.0, tuple(w.shape)), w.dtype))
    r = nrf_forward(f, rng.uniform(-1.5, 1.5, (100000, 3)))
    assert np.max(np.abs(r)) <= 0.1
    np.testing.assert_array_equal(nrf_forward(f, x), nrf_forward(f, x))  # deterministic
    with pytest.raises(UninitializedField):
        nrf_forward(ResidualField(), np.zeros((1, 3)))
    f = ResidualField64.create(rng)  # float64: against the scalar evaluation
    for w in f.weights:
        w[:] = rng.normal(0, 0.5, w.shape)
    for b in f.biases:
        b[:] = rng.normal(0, 0.2, b.shape)
    pts = rng.uniform(-1, 1, (20, 3))
    np.testing.assert_allclose(nrf_forward64(f, pts), [_scalar_nrf(f, p) for p in pts], atol=1e-10)


def test_nrf_backward_cases(rng):
    from paper_2603_00145_b200.nrf import ResidualField64, nrf_backward64, nrf_forward64

    f = ResidualField64.create(rng, frequency_bands=3, hidden=(9, 7))
    for w in f.weights:
        w[:] = rng.normal(0, 0.6, w.shape)
    for b in f.biases:
        b[:] = rng.normal(0, 0.3, b.shape)
    x = rng.uniform(-1, 1, (10, 3))
    dws, dbs, dp = nrf_backward64(f, x, np.zeros(10))
    assert all(np.all(d == 0.0) for d in dws + dbs) and np.all(dp == 0.0)
    x1 = rng.uniform(-1, 1, (1, 3))
    r = nrf_forward64(f, x1)
    _, dbs, _ = nrf_backward64(f, x1, np.array([1.7]))
    np.testing.assert_allclose(dbs[-1], [1.7 * f.output_bound * (1.0 - (r[0] / f.output_bound) ** 2)], rtol=1e-10)
    x = rng.uniform(-1, 1, (6, 3))
    up = rng.normal(size=6)

    def loss(_=None):
        return float(np.sum(up * nrf_forward64(f, x)))

    dws, dbs, dp = nrf_backward64(f, x, up)
    for li in range(len(f.weights)):
        np.testing.assert_allclose(dws[li], central_difference(lambda a: loss(), f.weights[li]), rtol=1e-4, atol=1e-8)
        np.testing.assert_allclose(dbs[li], central_difference(lambda a: loss(), f.biases[li]), rtol=1e-4, atol=1e-8)
    np.testing.assert_allclose(dp, central_difference(lambda a: loss(), x), rtol=1e-4, atol=1e-8)


# --------------------------------------------------------------------------- spatial (test_spatial.py)


def _cells(positions, g):
    return np.clip(np.floor((np.asarray(positions, np.float64) + 1.0) * g / 2.0), 0, g - 1).astype(np.int64)


def test_cell_index_and_build(rng):
    from paper_2603_00145_b200.core import uniform_lattice_field
    from paper_2603_00145_b200.spatial import build, cell_index

    np.testing.assert_array_equal(cell_index([-1.0, -1.0, -1.0], 70), [0, 0, 0])
    np.testing.assert_array_equal(cell_index([0.0, 0.0, 0.0], 70), [35, 35, 35])
    np.testing.assert_array_equal(cell_index([1.0, 1.0, 1.0], 70), [69, 69, 69])
    for v in np.linspace(-1.2, 1.2, 1201):
        assert cell_index([v, v, v], 16)[0] == min(max(int(np.floor((v + 1.0) * 16 / 2.0)), 0), 15)
    corners = np.array([[sx, sy, sz] for sx in (-1, 1) for sy in (-1, 1) for sz in (-1, 1)], np.float64) * 0.999
    assert np.all(np.diff(build(corners, 2).cell_starts) == 1)
    grid = build(np.zeros((50, 3)), 70)
    assert len(grid.bucket(35, 35, 35)) == 50 and grid.cell_starts[-1] == 50
    f = random_field(rng, side=6)
    f.positions[:] = rng.uniform(-1.05, 1.05, f.positions.shape)
    grid = build(f, 70)
    c = _cells(f.positions, 70)
    np.testing.assert_array_equal(np.diff(grid.cell_starts),
                                  np.bincount((c[:, 0] * 70 + c[:, 1]) * 70 + c[:, 2], minlength=70 ** 3))
    np.testing.assert_array_equal(np.sort(grid.cell_indices), np.arange(f.count))
    f = random_field(rng, side=4)
    g1, g2 = build(f, 12), build(f, 12)
    np.testing.assert_array_equal(g1.cell_indices, g2.cell_indices)
    np.testing.assert_array_equal(g1.cell_starts, g2.cell_starts)
    assert np.all(np.diff(build(uniform_lattice_field(6), 6).cell_starts) == 1)


def test_query_local_cases(rng):
    from paper_2603_00145_b200.spatial import build, query_local

    f = random_field(rng, side=4)
    np.testing.assert_array_equal(query_local(build(f, 9), rng.uniform(-1, 1, 3), radius=9), np.arange(f.count))
    np.testing.assert_array_equal(query_local(build(np.zeros((1, 3)), 21), np.zeros(3), radius=0), [0])
    f = random_field(rng, side=7)
    f.positions[:] = rng.uniform(-1.02, 1.02, f.positions.shape)
    grid = build(f, 24, block_radius=5)
    cells = _cells(f.positions, 24)
    for _ in range(1000):
        x = rng.uniform(-1.1, 1.1, 3)
        c0 = _cells(x[None, :], 24)[0]
        want = np.nonzero(np.max(np.abs(cells - c0[None, :]), axis=1) <= 5)[0]
        np.testing.assert_array_equal(query_local(grid, x), want)
    f = random_field(rng, side=5)
    grid = build(f, 15)
    for _ in range(50):
        x = rng.uniform(-1, 1, 3)
        prev = set()
        for r in range(16):
            cur = set(query_local(grid, x, radius=r).tolist())
            assert prev <= cur
            prev = cur
        assert prev == set(range(f.count))
    assert query_local(build(np.full((3, 3), 0.9), 20), np.array([-0.9, -0.9, -0.9]), radius=1).size == 0
    f = random_field(rng, side=6)
    grid = build(f, 10, block_radius=3)
    for _ in range(100):
        got = query_local(grid, rng.uniform(-1, 1, 3))
        assert len(np.unique(got)) == len(got)
