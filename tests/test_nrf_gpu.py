"""Fused residual-field kernels (csrc/mg_nrf.cu) against the reference's
ResidualField forward/backward golden (nrf.py:23-182, generated from the
reference) and against the torch-op mirror on a larger ragged batch; the
fused backward must also be bit-reproducible (fixed-order partial sums)."""

import numpy as np
import pytest
import torch

from conftest import assert_grad_close, load_golden

pytestmark = pytest.mark.gpu


def _field(ws, bs):
    from paper_2603_00145_b200.nrf import ResidualField

    return ResidualField.from_numpy([np.asarray(w, np.float64) for w in ws], [np.asarray(b, np.float64) for b in bs])


def _h(t):
    return t.detach().double().cpu().numpy()


def test_fused_nrf_matches_reference_golden():
    from paper_2603_00145_b200.nrf import fused_supported, nrf_backward_fused, nrf_forward_fused

    z = load_golden("nrf")
    f = _field([z[f"w{i}"] for i in range(5)], [z[f"b{i}"] for i in range(5)])
    assert fused_supported(f)
    x = torch.as_tensor(z["x"], dtype=torch.float32, device="cuda")
    up = torch.as_tensor(z["up"], dtype=torch.float32, device="cuda")
    r, cache = nrf_forward_fused(f, x)
    np.testing.assert_allclose(_h(r), z["r"], rtol=1e-4, atol=1e-6 * np.abs(z["r"]).max())
    dws, dbs, dp = nrf_backward_fused(f, x, up, cache)
    for i in range(5):
        assert_grad_close(_h(dws[i]), z[f"dw{i}"], name=f"dw{i}")
        assert_grad_close(_h(dbs[i]), z[f"db{i}"], name=f"db{i}")
    assert_grad_close(_h(dp), z["d_points"], name="d_points")


@pytest.mark.parametrize("n", [1, 63, 5000, 20000, 70001])
def test_fused_nrf_matches_torch_mirror(n):
    """Against the torch-op restatement evaluated in FLOAT64 on the same
    float32 inputs (the truth the float32 kernels approximate; a float32
    mirror carries its own rounding, ~1e-5 at the top Fourier band).  n >= 8192
    makes CTAs of the dW pass take several 128-point chunks (the double-
    buffered cp.async prefetch); 70001 is ragged."""
    from types import SimpleNamespace

    from nrf_mirror import nrf_backward, nrf_forward_cached
    from paper_2603_00145_b200.nrf import nrf_backward_fused, nrf_forward_fused

    rng = np.random.default_rng(n)
    widths = (39, 64, 64, 64, 64, 1)
    ws = [rng.uniform(-1, 1, (a, b)) * np.sqrt(6.0 / (a + b)) for a, b in zip(widths[:-1], widths[1:])]
    bs = [rng.normal(0, 0.1, b) for b in widths[1:]]
    f = _field(ws, bs)
    f64 = SimpleNamespace(frequency_bands=6, output_bound=0.1, weights=[w.double() for w in f.weights],
                          biases=[b.double() for b in f.biases])
    x = torch.as_tensor(rng.uniform(-1, 1, (n, 3)), dtype=torch.float32, device="cuda")
    up = torch.as_tensor(rng.normal(size=n), dtype=torch.float32, device="cuda")
    r0, c0 = nrf_forward_cached(f64, x.double())
    pred = torch.as_tensor(rng.normal(size=n), dtype=torch.float32, device="cuda")
    base = pred.clone()
    _, c1 = nrf_forward_fused(f, x, pred_add=pred)
    np.testing.assert_allclose(_h(pred - base), _h(r0), rtol=1e-4, atol=1e-6)
    g0 = nrf_backward(f64, x.double(), up.double(), c0)
    g1 = nrf_backward_fused(f, x, up, c1)
    for i in range(5):
        assert_grad_close(_h(g1[0][i]), _h(g0[0][i]), name=f"dw{i}")
        assert_grad_close(_h(g1[1][i]), _h(g0[1][i]), name=f"db{i}")
    assert_grad_close(_h(g1[2]), _h(g0[2]), name="d_points")
    # deterministic: a second backward gives the same bits
    g2 = nrf_backward_fused(f, x, up, c1)
    for a, b in zip(g1[0] + g1[1] + [g1[2]], g2[0] + g2[1] + [g2[2]]):
        assert torch.equal(a, b)


@pytest.mark.parametrize("tc", ["0", "1"])
def test_nrf_layer_paths_match_golden(tc):
    """Both layer implementations -- tcgen05 3xTF32 (default) and the SIMT
    FFMA2 kernels (MGAUSS_NRF_TC=0) -- against the reference golden, each in
    its own process (the switch is read once)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, MGAUSS_NRF_TC=tc)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", os.path.abspath(__file__) +
                        "::test_fused_nrf_matches_reference_golden"], env=env, cwd=root, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:]


def test_unsupported_width_raises():
    from paper_2603_00145_b200.errors import UnsupportedResidualField
    from paper_2603_00145_b200.nrf import ResidualField, nrf_forward_device

    f = ResidualField.create(np.random.default_rng(1), hidden=(32, 32))
    with pytest.raises(UnsupportedResidualField):
        nrf_forward_device(f, torch.zeros((4, 3), dtype=torch.float32, device="cuda"))


def test_fused_nrf_empty_batch_zero_grads():
    from paper_2603_00145_b200.nrf import ResidualField, nrf_backward_fused, nrf_forward_fused

    f = ResidualField.create(np.random.default_rng(1))
    x = torch.zeros((0, 3), dtype=torch.float32, device="cuda")
    r, cache = nrf_forward_fused(f, x)
    assert r.numel() == 0
    dws, dbs, dp = nrf_backward_fused(f, x, torch.zeros(0, device="cuda"), cache)
    assert dp.shape == (0, 3)
    assert all(float(t.abs().sum()) == 0.0 for t in dws + dbs)
