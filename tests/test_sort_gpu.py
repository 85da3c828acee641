"""GPU checks of the binning primitives at production sizes: the cell sort
(counting sort + in-cell rank pass) and CSR against numpy's stable argsort /
bincount / cumsum (the reference's spatial.py:46-66 recipe), including a
crowded cell whose ties must keep ascending index."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [1, 2047, 2048, 2049, 100000, 1 << 20, 3000001])
def test_excl_scan_matches_numpy(n):
    import torch

    from paper_2603_00145_b200 import _native as N

    rng = np.random.default_rng(n)
    a = rng.integers(0, 5, n).astype(np.int32)
    t = torch.from_numpy(a).cuda()
    out = torch.empty_like(t)
    ws = torch.empty(N.lib().mg_scan_workspace_bytes(n), dtype=torch.uint8, device="cuda")
    st = N.stream_ptr()
    N.check(N.lib().mg_excl_scan_i32(N.ptr(t), N.ptr(out), n, N.ptr(ws), ws.numel(), st))
    want = np.concatenate([[0], np.cumsum(a)[:-1]]).astype(np.int64)
    np.testing.assert_array_equal(out.cpu().numpy(), want)
    N.check(N.lib().mg_excl_scan_i32(N.ptr(t), N.ptr(t), n, N.ptr(ws), ws.numel(), st))  # in place
    np.testing.assert_array_equal(t.cpu().numpy(), want)


@pytest.mark.parametrize("n,g", [(1000, 8), (97336, 46), (273408, 46), (300000, 80), (500000, 126)])
def test_bin_matches_numpy_stable(n, g):
    import torch

    from paper_2603_00145_b200.spatial import build_device

    rng = np.random.default_rng(n)
    pos = rng.uniform(-1.02, 1.02, (n, 3))
    pos[: n // 10] = pos[0]  # a crowded cell: ties must keep ascending index
    d = build_device(torch.from_numpy(pos).cuda(), g)
    c = np.clip(np.floor((pos + 1.0) * (g / 2.0)).astype(np.int64), 0, g - 1)
    flat = (c[:, 0] * g + c[:, 1]) * g + c[:, 2]
    order = np.argsort(flat, kind="stable")
    starts = np.zeros(g ** 3 + 1, np.int64)
    np.cumsum(np.bincount(flat, minlength=g ** 3), out=starts[1:])
    np.testing.assert_array_equal(d["order"].cpu().numpy(), order)
    np.testing.assert_array_equal(d["starts"].cpu().numpy(), starts)
    np.testing.assert_array_equal(d["keys"].cpu().numpy().astype(np.int64), flat[order])
