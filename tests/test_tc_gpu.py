"""The tcgen05 tensor-core path (mg_tc.cuh: TMEM accumulator, K-major
no-swizzle shared-memory descriptors, kind::tf32 and kind::f16 MMAs) against a
float64 GEMM: 1xTF32 to TF32 precision, 3xTF32 (hi*hi + hi*lo + lo*hi) to
the float32 accumulation floor, bf16x3 (8 products of a three-term bf16
split, what the NRF layers use) likewise."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("split", [0, 1, 2])
def test_tc_selftest_gemm(split):
    import torch

    from paper_2603_00145_b200 import _device as dv
    from paper_2603_00145_b200 import _native as N

    rng = np.random.default_rng(split)
    a = rng.normal(size=(128, 64)).astype(np.float32)
    bt = rng.normal(size=(64, 64)).astype(np.float32)
    A, Bt = dv.to_dev(a, torch.float32), dv.to_dev(bt, torch.float32)
    D = dv.zeros((128, 64), torch.float32)
    N.check(N.lib().mg_tc_selftest(N.ptr(A), N.ptr(Bt), N.ptr(D), split, dv.sptr()), "tc_selftest")
    got = dv.to_host(D).astype(np.float64)
    want = a.astype(np.float64) @ bt.astype(np.float64).T
    err = np.abs(got - want).max() / np.abs(want).max()
    print(f"split={split}: max error / max |D| = {err:.3g}")
    # 3xTF32 and bf16x3 both reach the tensor core's float32 accumulation floor (~7e-7 of max|D| at K = 64)
    assert err < {0: 5e-3, 1: 1.5e-6, 2: 1.5e-6}[split]
