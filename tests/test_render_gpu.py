"""GPU parity: the sm_100a path vs the reference's golden vectors and the
CPU oracle on the same inputs (tolerances per SURVEY §8(c)):
  integer outputs (cell CSR, contributor counts)  bit-exact
  transformed points (float64 path)                 1e-15 abs
  intensities                                       rel 1e-4
  gradients   |d| <= 1e-4 |ref| + 1e-6 max|ref|
"""

import numpy as np
import pytest

from conftest import assert_grad_close, load_golden

pytestmark = pytest.mark.gpu

CASES = ["small_full", "small_r1", "lattice12", "random14", "clamped"]


class Batch:
    def __init__(self, coords, slice_ids=None):
        self.coords = np.asarray(coords, dtype=np.float64)
        self.slice_ids = (np.full(self.coords.shape[0], -1, np.int64) if slice_ids is None
                          else np.asarray(slice_ids, dtype=np.int64))


def field_of(z):
    from paper_2603_00145_b200.core import GaussianField

    n = z["positions"].shape[0]
    return GaussianField(z["positions"].copy(), z["quaternions"].copy(), z["log_scales"].copy(),
                         z["logits"].copy(), (n, 1, 1), np.zeros((n, 3), np.int64))


def transforms_of(z):
    from paper_2603_00145_b200.core import TransformSet

    if len(z["t_quats"]) == 0:
        return None
    return TransformSet(z["t_quats"].copy(), z["t_trans"].copy())


def assert_rel(got, want, rtol=1e-4, atol=1e-12, name=""):
    got, want = np.asarray(got), np.asarray(want)
    err = np.abs(got - want)
    tol = rtol * np.abs(want) + atol
    bad = err > tol
    assert not bad.any(), (f"{name}: {bad.sum()}/{bad.size} beyond rtol {rtol}; worst rel "
                           f"{np.max(err / (np.abs(want) + 1e-300)):.3g}")


@pytest.mark.parametrize("case", CASES)
def test_build_bit_exact(case):
    from paper_2603_00145_b200.spatial import build

    z = load_golden("render_" + case)
    grid = build(z["positions"], int(z["g"]), int(z["r"]))
    np.testing.assert_array_equal(grid.cell_starts, z["cell_starts"])
    np.testing.assert_array_equal(grid.cell_indices, z["cell_indices"])


def test_spatial_golden():
    from paper_2603_00145_b200.spatial import build, cell_index

    z = load_golden("spatial")
    np.testing.assert_array_equal(cell_index(np.array([[-1.0] * 3, [0.0] * 3, [1.0] * 3]), 70),
                                  z["corner_cells"])
    sw = z["sweep"]
    np.testing.assert_array_equal(cell_index(np.stack([sw] * 3, 1), 16)[:, 0], z["sweep_cells"])
    for pos, g, cs, ci in ((z["pos"], 70, z["cell_starts"], z["cell_indices"]),
                           (z["lat_pos"], 6, z["lat_starts"], z["lat_indices"]),
                           (np.zeros((50, 3)), 70, z["dup_starts"], z["dup_indices"])):
        grid = build(pos, g)
        np.testing.assert_array_equal(grid.cell_starts, cs)
        np.testing.assert_array_equal(grid.cell_indices, ci)


@pytest.mark.parametrize("case", CASES)
def test_activated_parameters(case):
    from paper_2603_00145_b200.render import activated_parameters

    z = load_golden("render_" + case)
    qn, _, iv, p6, al = activated_parameters(field_of(z))
    np.testing.assert_allclose(qn, z["qn"], rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(iv, z["inv_var"], rtol=1e-13)
    np.testing.assert_allclose(p6, z["prec6"], rtol=1e-10, atol=1e-10 * np.abs(z["prec6"]).max())
    np.testing.assert_allclose(al, z["alpha"], rtol=1e-14)


@pytest.mark.parametrize("case", CASES)
def test_render_points_golden(case):
    from paper_2603_00145_b200.render import render_points
    from paper_2603_00145_b200.spatial import build

    z = load_golden("render_" + case)
    f = field_of(z)
    grid = build(f, int(z["g"]), int(z["r"]))
    out = render_points(f, grid, transforms_of(z), Batch(z["coords"], z["sids"]))
    np.testing.assert_array_equal(out.contributor_counts, z["counts"])
    np.testing.assert_allclose(out.points, z["points"], rtol=0, atol=1e-15)
    assert_rel(out.intensities, z["intensities"], name="intensities")


@pytest.mark.parametrize("case", CASES)
def test_render_backward_golden(case):
    from paper_2603_00145_b200.render import render_backward
    from paper_2603_00145_b200.spatial import build

    z = load_golden("render_" + case)
    f = field_of(z)
    grid = build(f, int(z["g"]), int(z["r"]))
    gr = render_backward(f, grid, transforms_of(z), Batch(z["coords"], z["sids"]), z["upstream"])
    for mine, ref in (("d_positions", "d_positions"), ("d_quaternions", "d_quaternions"),
                      ("d_log_scales", "d_log_scales"), ("d_intensity_logits", "d_logits"),
                      ("d_transform_params", "d_transform"), ("d_points", "d_points")):
        assert_grad_close(getattr(gr, mine), z[ref], name=f"{case}:{mine}")


def test_clamped_scale_gradient_exact_zero():
    from paper_2603_00145_b200.render import render_backward
    from paper_2603_00145_b200.spatial import build

    z = load_golden("render_clamped")
    f = field_of(z)
    gr = render_backward(f, build(f, 4, 4), None, Batch(z["coords"]), z["upstream"])
    assert gr.d_log_scales[0, 1] == 0.0 and gr.d_log_scales[1, 2] == 0.0


def test_prepared_matches_unprepared():
    from paper_2603_00145_b200.render import activated_parameters, render_points
    from paper_2603_00145_b200.spatial import build

    z = load_golden("render_lattice12")
    f = field_of(z)
    grid = build(f, int(z["g"]), 5)
    prep = activated_parameters(f)
    a = render_points(f, grid, transforms_of(z), Batch(z["coords"], z["sids"]), prepared=prep)
    b = render_points(f, grid, transforms_of(z), Batch(z["coords"], z["sids"]))
    np.testing.assert_array_equal(a.intensities, b.intensities)


def test_sample_volume_golden():
    from paper_2603_00145_b200.render import sample_volume
    from paper_2603_00145_b200.spatial import build

    z = load_golden("volume")
    f = field_of(z)
    grid = build(f, int(z["g"]), int(z["r"]))
    vol = sample_volume(f, grid, None, tuple(z["dims"]), (z["lo"], z["hi"]), radius=int(z["r"]))
    assert_rel(vol.data, z["data"], name="volume")
    np.testing.assert_allclose(vol.spacing, z["spacing"], rtol=1e-15)
    np.testing.assert_allclose(vol.origin, z["origin"], rtol=1e-15)


def test_dense_golden():
    from paper_2603_00145_b200.render import render_points_dense

    z = load_golden("render_small_full")
    f = field_of(z)
    pts = z["coords"][z["sids"] < 0]
    want = z["intensities"][z["sids"] < 0]  # full radius: block == dense
    assert_rel(render_points_dense(f, pts), want, name="dense")


def test_inconsistent_grid_raises():
    from paper_2603_00145_b200 import InconsistentGrid
    from paper_2603_00145_b200.render import render_points
    from paper_2603_00145_b200.spatial import build

    z = load_golden("render_small_full")
    f = field_of(z)
    grid = build(z["positions"][:-2], 8)
    with pytest.raises(InconsistentGrid):
        render_points(f, grid, None, Batch(np.zeros((1, 3))))


def test_upstream_length_mismatch_raises():
    from paper_2603_00145_b200.render import render_backward
    from paper_2603_00145_b200.spatial import build

    z = load_golden("render_small_full")
    f = field_of(z)
    with pytest.raises(ValueError):
        render_backward(f, build(f, 5), None, Batch(np.zeros((3, 3))), np.zeros(2))


def test_degenerate_quaternion_raises():
    from paper_2603_00145_b200 import DegenerateQuaternion
    from paper_2603_00145_b200.render import render_points
    from paper_2603_00145_b200.spatial import build

    z = load_golden("render_small_full")
    f = field_of(z)
    f.quaternions[3] = 0.0
    with pytest.raises(DegenerateQuaternion):
        render_points(f, build(f, 5), None, Batch(np.zeros((2, 3))))


def test_out_of_memory_guard():
    from paper_2603_00145_b200 import OutOfMemoryRequest
    from paper_2603_00145_b200.render import sample_volume
    from paper_2603_00145_b200.spatial import build

    z = load_golden("render_small_full")
    f = field_of(z)
    with pytest.raises(OutOfMemoryRequest):
        sample_volume(f, build(f, 2), None, (4096, 4096, 4096))


def test_empty_neighborhood_and_empty_batch():
    from paper_2603_00145_b200.core import uniform_lattice_field
    from paper_2603_00145_b200.render import render_points
    from paper_2603_00145_b200.spatial import build

    f = uniform_lattice_field(1)
    f.positions[0] = (0.9, 0.9, 0.9)
    out = render_points(f, build(f, 20), None, Batch([[-0.9, -0.9, -0.9]]), radius=0)
    assert out.intensities[0] == 0.0 and out.contributor_counts[0] == 0
    out = render_points(f, build(f, 20), None, Batch(np.zeros((0, 3))))
    assert out.intensities.shape == (0,)


def test_closed_form_centre_and_sqrt2():
    from paper_2603_00145_b200.core import uniform_lattice_field
    from paper_2603_00145_b200.render import render_points
    from paper_2603_00145_b200.spatial import build

    f = uniform_lattice_field(1)
    f.positions[0] = 0.0
    f.log_scales[0] = 0.0
    f.intensity_logits[0] = np.log(0.8 / 0.2)
    grid = build(f, 1)
    out = render_points(f, grid, None, Batch([[0.0, 0.0, 0.0], [np.sqrt(2.0), 0.0, 0.0]]))
    np.testing.assert_allclose(out.intensities, [0.8, 0.8 * np.exp(-1.0)], rtol=1e-6)
    assert list(out.contributor_counts) == [1, 1]


def test_psf_matches_composed_oracle():
    from oracle import oracle as O
    from paper_2603_00145_b200.render import SlicePSF, render_backward, render_points
    from paper_2603_00145_b200.spatial import build

    z = load_golden("render_lattice12")
    f = field_of(z)
    k = len(z["t_quats"])
    rng = np.random.default_rng(5)
    dirs = np.zeros((k, 3))
    dirs[np.arange(k), rng.integers(0, 3, k)] = 1.0
    psf = SlicePSF(offsets=np.array([-0.03, 0.0, 0.03]), weights=np.array([0.311, 0.378, 0.311]),
                   through_dirs=dirs)
    grid = build(f, int(z["g"]), 5)
    ts = transforms_of(z)
    out = render_points(f, grid, ts, Batch(z["coords"], z["sids"]), slice_psf=psf)
    want, wcnt = O.psf_render(z["positions"], z["quaternions"], z["log_scales"], z["logits"], int(z["g"]), 5,
                              z["coords"], z["sids"], z["t_quats"], z["t_trans"], psf.offsets, psf.weights, dirs)
    np.testing.assert_array_equal(out.contributor_counts, wcnt)
    assert_rel(out.intensities, want, name="psf")
    gr = render_backward(f, grid, ts, Batch(z["coords"], z["sids"]), z["upstream"], slice_psf=psf)
    og = O.psf_backward(z["positions"], z["quaternions"], z["log_scales"], z["logits"], int(z["g"]), 5,
                        z["coords"], z["sids"], z["t_quats"], z["t_trans"], psf.offsets, psf.weights, dirs,
                        z["upstream"])
    for name in ("d_positions", "d_quaternions", "d_log_scales", "d_intensity_logits", "d_transform_params"):
        assert_grad_close(getattr(gr, name), getattr(og, name), name="psf:" + name)


@pytest.mark.parametrize("seed", [0, 1])
def test_random_config_against_oracle(seed):
    """Denser random configurations than the goldens: many points per cell,
    several Gaussians per cell (exercises the Q>2 / QG>1 kernel paths)."""
    from oracle import oracle as O
    from paper_2603_00145_b200.core import GaussianField, TransformSet
    from paper_2603_00145_b200.render import render_backward, render_points
    from paper_2603_00145_b200.spatial import build

    rng = np.random.default_rng(seed)
    n = 3000
    f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)  # noqa: E731
    f = GaussianField(f32(rng.uniform(-0.95, 0.95, (n, 3))),
                      f32(rng.normal(0, 0.3, (n, 4)) + [1, 0, 0, 0]),
                      f32(np.log(1 / 20) + rng.normal(0, 0.2, (n, 3))), f32(rng.normal(0, 1, n)))
    k = 5
    ts = TransformSet(f32(rng.normal(0, 0.05, (k, 4)) + [1, 0, 0, 0]), f32(rng.normal(0, 0.02, (k, 3))))
    b = 20000
    coords = rng.uniform(-1, 1, (b, 3))
    sids = rng.integers(-1, k, b)
    up = rng.normal(size=b)
    g, r = 12, 3
    grid = build(f, g, r)
    out = render_points(f, grid, ts, Batch(coords, sids))
    x, inten, cnt = O.render_points(f.positions, f.quaternions, f.log_scales, f.intensity_logits, g, r, coords,
                                    sids, ts.quats, ts.translations)
    np.testing.assert_array_equal(out.contributor_counts, cnt)
    assert_rel(out.intensities, inten, name="I")
    gr = render_backward(f, grid, ts, Batch(coords, sids), up)
    og = O.render_backward(f.positions, f.quaternions, f.log_scales, f.intensity_logits, g, r, coords, up,
                           sids, ts.quats, ts.translations, threads=4)
    for name in ("d_positions", "d_quaternions", "d_log_scales", "d_intensity_logits", "d_transform_params",
                 "d_points"):
        assert_grad_close(getattr(gr, name), getattr(og, name), name=name)


def test_sample_volume_lattice_against_oracle():
    """A 20^3-lattice field sampled on a 37x41x29 grid (many voxels per cell:
    exercises the multi-chunk voxel boxes) against the oracle."""
    from oracle import oracle as O
    from paper_2603_00145_b200.core import uniform_lattice_field
    from paper_2603_00145_b200.render import sample_volume
    from paper_2603_00145_b200.spatial import build

    rng = np.random.default_rng(4)
    R = 20
    f = uniform_lattice_field(R)
    f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)  # noqa: E731
    f.positions = f32(f.positions + rng.normal(0, 0.1 / R, f.positions.shape))
    f.quaternions = f32(f.quaternions + rng.normal(0, 0.1, f.quaternions.shape))
    f.log_scales = f32(f.log_scales + rng.normal(0, 0.1, f.log_scales.shape))
    f.intensity_logits = f32(rng.normal(0, 1, f.count))
    dims, bounds = (37, 41, 29), ((-0.97, -1.0, -0.9), (1.0, 0.95, 0.99))
    vol = sample_volume(f, build(f, R, 3), None, dims, bounds, radius=3)
    want = O.sample_volume(f.positions, f.quaternions, f.log_scales, f.intensity_logits, R, 3, dims, bounds,
                           threads=4)
    assert_rel(vol.data, want, name="volume")


@pytest.mark.parametrize("r", [5, 2])
def test_sample_volume_after_larger_call(r):
    """Tiled volume path: a larger call first (it leaves its run tables in the
    reused workspace), then a smaller grid with an odd run count per axis and
    several runs per tile, against the oracle.  Guards the tile counts against
    reading past the last run (stale workspace)."""
    from oracle import oracle as O
    from paper_2603_00145_b200.core import uniform_lattice_field
    from paper_2603_00145_b200.render import sample_volume
    from paper_2603_00145_b200.spatial import build

    big = uniform_lattice_field(40)
    big.intensity_logits = np.random.default_rng(1).normal(0, 1, big.count)
    sample_volume(big, build(big, 40, r), None, (96, 96, 96), ((-1.0,) * 3, (1.0,) * 3), radius=r)
    rng = np.random.default_rng(7)
    R = 15
    f = uniform_lattice_field(R)
    f32 = lambda a: np.asarray(a, np.float32).astype(np.float64)  # noqa: E731
    f.positions = f32(f.positions + rng.normal(0, 0.1 / R, f.positions.shape))
    f.log_scales = f32(f.log_scales + rng.normal(0, 0.1, f.log_scales.shape))
    f.intensity_logits = f32(rng.normal(0, 1, f.count))
    dims, bounds = (23, 19, 31), ((-0.95, -1.0, -0.9), (0.97, 0.93, 1.0))
    vol = sample_volume(f, build(f, R, r), None, dims, bounds, radius=r)
    want = O.sample_volume(f.positions, f.quaternions, f.log_scales, f.intensity_logits, R, r, dims, bounds,
                           threads=4)
    assert_rel(vol.data, want, name="volume")
