"""The reference's host-level training API (train.py:108-290: smooth_l1,
smooth_l1_grad, aniso_loss(_grad), progressive_upsample, init_field,
AdamState) with this package's device-backed implementations, against the
reference's own outputs (tests/golden/train_ops.npz, make_golden.py)."""

from types import SimpleNamespace

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def test_smooth_l1_and_grad():
    from paper_2603_00145_b200.train import smooth_l1, smooth_l1_grad

    z = load_golden("train_ops")
    np.testing.assert_allclose(smooth_l1(z["sl1_pred"], z["sl1_tgt"]), z["sl1"], rtol=1e-6)
    np.testing.assert_allclose(smooth_l1_grad(z["sl1_pred"], z["sl1_tgt"]), z["sl1_grad"], rtol=1e-6, atol=1e-9)


def test_aniso_loss_grad_float64():
    from paper_2603_00145_b200.core import GaussianField
    from paper_2603_00145_b200.train import aniso_loss, aniso_loss_grad

    z = load_golden("train_ops")
    s = z["aniso_s"]
    n = s.shape[0]
    f = GaussianField(np.zeros((n, 3)), np.tile([1.0, 0, 0, 0], (n, 1)), s.copy(), np.zeros(n), (n, 1, 1),
                      np.zeros((n, 3), np.int64))
    loss, grad = aniso_loss_grad(f, 1.5)
    np.testing.assert_allclose(loss, z["aniso_loss"], rtol=1e-13)
    np.testing.assert_allclose(grad, z["aniso_grad"], rtol=1e-13, atol=1e-300)
    assert aniso_loss(f, 1.5) == loss


def test_adam_state_float64():
    from paper_2603_00145_b200.train import AdamState

    z = load_golden("train_ops")
    p = z["adam_p0"].copy()
    st = AdamState()
    for g in z["adam_grads"]:
        st.step("positions", {"p": p}, {"p": g}, 0.01)
    np.testing.assert_allclose(p, z["adam_p"], rtol=1e-13, atol=1e-16)
    np.testing.assert_allclose(st.groups["positions"]["m"]["p"], z["adam_m"], rtol=1e-13, atol=1e-300)
    np.testing.assert_allclose(st.groups["positions"]["v"]["p"], z["adam_v"], rtol=1e-13, atol=1e-300)
    assert st.groups["positions"]["t"] == len(z["adam_grads"])
    st2 = AdamState()
    st2.load_state_dict(st.state_dict())
    assert st2.groups["positions"]["t"] == st.groups["positions"]["t"]
    st.reset_group("positions")
    assert "positions" not in st.groups


def test_progressive_upsample_and_init_field():
    from paper_2603_00145_b200.core import GaussianField
    from paper_2603_00145_b200.errors import ShrinkNotAllowed
    from paper_2603_00145_b200.train import init_field, progressive_upsample

    z = load_golden("train_ops")
    f = GaussianField(np.zeros((64, 3)), z["up_q"].copy(), z["up_s"].copy(), z["up_l"].copy(), (4, 4, 4),
                      z["up_idx"].copy())
    up = progressive_upsample(f, 7)
    assert up.lattice_dims == (7, 7, 7) and up.count == 343
    np.testing.assert_array_equal(up.positions, z["up_pos"])
    np.testing.assert_allclose(up.quaternions, z["up_qo"], atol=1e-6)
    np.testing.assert_allclose(up.log_scales, z["up_so"], atol=1e-6)
    np.testing.assert_allclose(up.intensity_logits, z["up_lo"], atol=1e-5)
    with pytest.raises(ShrinkNotAllowed):
        progressive_upsample(up, 4)
    cloud = SimpleNamespace(coords=z["init_coords"], intensities=z["init_int"])
    init = init_field(cloud, 5)
    np.testing.assert_allclose(init.intensity_logits, z["init_logits"], atol=1e-5)
    assert init.validate() is init
