"""Pin the CPU oracle (oracle/) against golden vectors produced by the reference.

The fixtures come from tests/golden/make_golden.py, which runs the reference
package itself (single thread, canonical order).  CPU only.
"""

import numpy as np
import pytest

from conftest import assert_grad_close, load_golden
from oracle import oracle as O

RENDER_CASES = ["small_full", "small_r1", "lattice12", "random14", "clamped"]


def _tq(z):
    return (z["t_quats"], z["t_trans"]) if len(z["t_quats"]) else (None, None)


def test_cell_index_golden():
    z = load_golden("spatial")
    np.testing.assert_array_equal(O.cell_index(np.array([[-1.0] * 3, [0.0] * 3, [1.0] * 3]), 70),
                                  z["corner_cells"])
    sweep = z["sweep"]
    got = O.cell_index(np.stack([sweep] * 3, axis=1), 16)[:, 0]
    np.testing.assert_array_equal(got, z["sweep_cells"])


def test_build_golden():
    z = load_golden("spatial")
    cs, ci = O.build(z["pos"], 70)
    np.testing.assert_array_equal(cs, z["cell_starts"])
    np.testing.assert_array_equal(ci, z["cell_indices"])
    cs, ci = O.build(z["lat_pos"], 6)
    np.testing.assert_array_equal(cs, z["lat_starts"])
    np.testing.assert_array_equal(ci, z["lat_indices"])
    cs, ci = O.build(np.zeros((50, 3)), 70)
    np.testing.assert_array_equal(cs, z["dup_starts"])
    np.testing.assert_array_equal(ci, z["dup_indices"])


@pytest.mark.parametrize("case", RENDER_CASES)
def test_activated_parameters_golden(case):
    z = load_golden("render_" + case)
    qn, _, inv_var, prec6, alpha = O.activated_parameters(z["quaternions"], z["log_scales"],
                                                          z["logits"])
    np.testing.assert_allclose(qn, z["qn"], rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(inv_var, z["inv_var"], rtol=1e-14)
    np.testing.assert_allclose(prec6, z["prec6"], rtol=1e-12, atol=1e-12 * np.abs(z["prec6"]).max())
    np.testing.assert_allclose(alpha, z["alpha"], rtol=1e-15)


@pytest.mark.parametrize("case", RENDER_CASES)
def test_render_forward_golden(case):
    z = load_golden("render_" + case)
    tq, tt = _tq(z)
    x, inten, cnt = O.render_points(z["positions"], z["quaternions"], z["log_scales"],
                                    z["logits"], int(z["g"]), int(z["r"]), z["coords"], z["sids"],
                                    tq, tt)
    np.testing.assert_array_equal(cnt, z["counts"])
    np.testing.assert_allclose(x, z["points"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(inten, z["intensities"], rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("case", RENDER_CASES)
@pytest.mark.parametrize("threads", [1, 3])
def test_render_backward_golden(case, threads):
    z = load_golden("render_" + case)
    tq, tt = _tq(z)
    g = O.render_backward(z["positions"], z["quaternions"], z["log_scales"], z["logits"],
                          int(z["g"]), int(z["r"]), z["coords"], z["upstream"], z["sids"], tq, tt,
                          threads=threads)
    for mine, ref in (("d_positions", "d_positions"), ("d_quaternions", "d_quaternions"),
                      ("d_log_scales", "d_log_scales"), ("d_intensity_logits", "d_logits"),
                      ("d_transform_params", "d_transform"), ("d_points", "d_points")):
        assert_grad_close(getattr(g, mine), z[ref], rel=1e-10, abs_frac=1e-12, name=mine)


def test_clamped_log_scale_gradient_is_zero():
    z = load_golden("render_clamped")
    assert z["d_log_scales"][0, 1] == 0.0 and z["d_log_scales"][1, 2] == 0.0


def test_dense_matches_block_at_full_radius():
    z = load_golden("render_small_full")
    _, _, _, prec6, alpha = O.activated_parameters(z["quaternions"], z["log_scales"],
                                                   z["logits"])
    pts = z["coords"][z["sids"] < 0]
    dense = O.dense_forward(pts, z["positions"], prec6, alpha)
    _, inten, _ = O.render_points(z["positions"], z["quaternions"], z["log_scales"], z["logits"],
                                  5, 5, pts)
    np.testing.assert_allclose(inten, dense, atol=1e-12)


def test_sample_volume_golden():
    z = load_golden("volume")
    vol = O.sample_volume(z["positions"], z["quaternions"], z["log_scales"], z["logits"],
                          int(z["g"]), int(z["r"]), tuple(z["dims"]), (z["lo"], z["hi"]))
    np.testing.assert_allclose(vol, z["data"], rtol=1e-12, atol=1e-14)


def test_train_ops_golden():
    z = load_golden("train_ops")
    p = z["adam_p0"].copy()
    m = np.zeros_like(p)
    v = np.zeros_like(p)
    for t, gr in enumerate(z["adam_grads"], start=1):
        O.adam_step(p, gr, m, v, t, 0.01)
    np.testing.assert_allclose(p, z["adam_p"], rtol=1e-15, atol=1e-15)
    np.testing.assert_allclose(m, z["adam_m"], rtol=1e-15, atol=1e-15)
    loss, grad = O.aniso_loss_grad(z["aniso_s"], 1.5)
    np.testing.assert_allclose(loss, z["aniso_loss"], rtol=1e-14)
    np.testing.assert_allclose(grad, z["aniso_grad"], rtol=1e-14, atol=1e-16)
    np.testing.assert_allclose(O.smooth_l1(z["sl1_pred"], z["sl1_tgt"]), z["sl1"], rtol=1e-15)
    np.testing.assert_allclose(O.smooth_l1_grad(z["sl1_pred"], z["sl1_tgt"]), z["sl1_grad"],
                               rtol=1e-15)
    pos, q, s, lg = O.progressive_upsample(z["up_q"], z["up_s"], z["up_l"], z["up_idx"], 4, 7)
    np.testing.assert_allclose(pos, z["up_pos"], atol=1e-15)
    np.testing.assert_allclose(q, z["up_qo"], atol=1e-14)
    np.testing.assert_allclose(s, z["up_so"], atol=1e-14)
    np.testing.assert_allclose(lg, z["up_lo"], atol=1e-14)
    np.testing.assert_allclose(O.init_logits(z["init_coords"], z["init_int"], 5),
                               z["init_logits"], atol=1e-14)


def test_nrf_golden():
    z = load_golden("nrf")
    ws = [z[f"w{i}"] for i in range(5)]
    bs = [z[f"b{i}"] for i in range(5)]
    r, _ = O.nrf_forward(ws, bs, z["x"])
    np.testing.assert_allclose(r, z["r"], rtol=1e-12, atol=1e-15)
    dws, dbs, dp = O.nrf_backward(ws, bs, z["x"], z["up"])
    for i in range(5):
        np.testing.assert_allclose(dws[i], z[f"dw{i}"], rtol=1e-10, atol=1e-14)
        np.testing.assert_allclose(dbs[i], z[f"db{i}"], rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(dp, z["d_points"], rtol=1e-10, atol=1e-14)


def test_ssim_golden():
    z = load_golden("ssim")
    loss, grad = O.ssim_loss_grad(z["pred"], z["tgt"])
    np.testing.assert_allclose(loss, z["loss"], rtol=1e-13)
    np.testing.assert_allclose(grad, z["grad"], rtol=1e-10, atol=1e-15)
