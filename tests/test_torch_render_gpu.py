"""torch-facing API (north_star: ``render(gaussians, sample_coords, slice_psf)
-> intensities`` and its backward) against the reference's goldens: forward
intensities, the four Gaussian parameter gradients, the per-slice transform
gradients, and the sample-coordinate gradient R_s^T d_points (render.py:292's
d_points is w.r.t. the transformed point)."""

import numpy as np
import pytest

from conftest import assert_grad_close, load_golden

pytestmark = pytest.mark.gpu

CASES = ["small_full", "small_r1", "lattice12", "random14", "clamped"]


def _leaf(a, dtype):
    import torch

    return torch.tensor(np.asarray(a), dtype=dtype, device="cuda", requires_grad=True)


def _run(z, dtype, psf=None):
    import torch

    from paper_2603_00145_b200.torch_render import render

    P = {k: _leaf(z[k], dtype) for k in ("positions", "quaternions", "log_scales", "logits")}
    coords = _leaf(z["coords"], dtype)
    k = len(z["t_quats"])
    tq = _leaf(z["t_quats"], torch.float64) if k else None
    tt = _leaf(z["t_trans"], torch.float64) if k else None
    out = render(P, coords, slice_psf=psf, slice_ids=torch.tensor(z["sids"]), transforms=(tq, tt) if k else None,
                 grid_resolution=int(z["g"]), radius=int(z["r"]))
    (out * torch.tensor(z["upstream"], dtype=dtype, device="cuda")).sum().backward()
    return out, P, coords, tq, tt


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_torch_render_matches_reference(case, dtype):
    import torch

    from oracle import oracle as O

    dt = getattr(torch, dtype)
    z = load_golden("render_" + case)
    out, P, coords, tq, tt = _run(z, dt)
    assert out.dtype == dt and out.shape == (z["coords"].shape[0],)
    got = out.detach().double().cpu().numpy()
    np.testing.assert_allclose(got, z["intensities"], rtol=1e-4, atol=1e-12)
    for name, key in (("positions", "d_positions"), ("quaternions", "d_quaternions"), ("log_scales", "d_log_scales"),
                      ("logits", "d_logits")):
        assert P[name].grad.dtype == dt
        assert_grad_close(P[name].grad.double().cpu().numpy(), z[key], name=f"{case}:{name}")
    want = z["d_points"].copy()
    if tq is not None:
        assert_grad_close(tq.grad.cpu().numpy(), z["d_transform"][:, :4], name=f"{case}:t_quats")
        assert_grad_close(tt.grad.cpu().numpy(), z["d_transform"][:, 4:], name=f"{case}:t_trans")
        rot = O.quat_to_rotation(O.normalize_quat(z["t_quats"]))
        s = z["sids"]
        m = s >= 0
        want[m] = np.einsum("bij,bi->bj", rot[s[m]], z["d_points"][m])
    assert_grad_close(coords.grad.double().cpu().numpy(), want, name=f"{case}:coords")


def test_torch_render_psf_matches_numpy_api():
    """With a slice PSF the layer equals the (oracle-checked) numpy-API PSF path."""
    import torch

    from paper_2603_00145_b200.render import SlicePSF, render_backward, render_points
    from paper_2603_00145_b200.spatial import build
    from test_render_gpu import Batch, field_of, transforms_of

    z = load_golden("render_lattice12")
    k = len(z["t_quats"])
    rng = np.random.default_rng(5)
    dirs = np.zeros((k, 3))
    dirs[np.arange(k), rng.integers(0, 3, k)] = 1.0
    psf = SlicePSF(offsets=np.array([-0.03, 0.0, 0.03]), weights=np.array([0.311, 0.378, 0.311]), through_dirs=dirs)
    out, P, coords, tq, tt = _run(z, torch.float64, psf)
    f = field_of(z)
    grid = build(f, int(z["g"]), 5)
    ref = render_points(f, grid, transforms_of(z), Batch(z["coords"], z["sids"]), slice_psf=psf)
    np.testing.assert_allclose(out.detach().cpu().numpy(), ref.intensities, rtol=1e-6, atol=1e-14)
    gr = render_backward(f, grid, transforms_of(z), Batch(z["coords"], z["sids"]), z["upstream"], slice_psf=psf)
    assert_grad_close(P["positions"].grad.cpu().numpy(), gr.d_positions, rel=1e-6, name="psf:positions")
    assert_grad_close(tq.grad.cpu().numpy(), gr.d_transform_params[:, :4], rel=1e-6, name="psf:t_quats")


def test_torch_render_errors_and_empty():
    import torch

    from paper_2603_00145_b200.torch_render import render

    z = load_golden("render_small_full")
    P = {k: torch.tensor(z[k], device="cuda") for k in ("positions", "quaternions", "log_scales", "logits")}
    P2 = {k: v[:10] for k, v in P.items()}  # N = 10 is not a cube: the grid side must be given
    with pytest.raises(ValueError):
        render(P2, torch.zeros((3, 3), device="cuda"))
    assert render(P, torch.zeros((0, 3), device="cuda"), grid_resolution=3).shape == (0,)
