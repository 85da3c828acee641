"""Torch-op restatement of the reference residual field (nrf.py:23-182) used
as a TEST reference for the fused kernels (csrc/mg_nrf.cu): fp32 GEMMs on
cuBLAS through torch.  Not part of the product package."""

import numpy as np
import torch


def _freqs(bands, x):
    return (2.0 ** torch.arange(bands, dtype=x.dtype, device=x.device)) * np.pi


def fourier_encode(x: torch.Tensor, bands: int) -> torch.Tensor:
    """nrf.py:23-36 on device: [x, sin(2^0 pi x), cos(2^0 pi x), sin(2^1 pi x), ...],
    all bands in one broadcast (same column order as the reference)."""
    s = x[:, None, :] * _freqs(bands, x)[None, :, None]  # (B, bands, 3)
    sc = torch.stack((torch.sin(s), torch.cos(s)), dim=2)  # (B, bands, 2, 3)
    return torch.cat((x, sc.reshape(x.shape[0], 6 * bands)), dim=1)


def nrf_forward_cached(field, x: torch.Tensor):
    h = fourier_encode(x, field.frequency_bands)
    pre, post = [], [h]
    depth = len(field.weights)
    for li in range(depth):
        z = torch.addmm(field.biases[li], h, field.weights[li])
        pre.append(z)
        if li < depth - 1:
            h = torch.nn.functional.silu(z)  # z * sigmoid(z), one kernel
            post.append(h)
    t = torch.tanh(pre[-1][:, 0])
    return field.output_bound * t, (t, pre, post)


def _split_k(n_rows, parts=128, min_rows=512):
    q = n_rows // parts
    return (parts, q) if q >= min_rows else (0, 0)


def _tn_matmul(a, b):
    """a^T @ b for tall (K x m), (K x n) operands: split-K over equal row
    chunks as one batched GEMM plus a fixed-order sum (a plain K = 131k GEMM
    with a 64 x 64 output runs on a handful of CTAs)."""
    parts, q = _split_k(a.shape[0])
    if not parts:
        return a.T @ b
    main = parts * q
    out = torch.bmm(a[:main].reshape(parts, q, a.shape[1]).transpose(1, 2),
                    b[:main].reshape(parts, q, b.shape[1])).sum(dim=0)
    if main < a.shape[0]:
        out = out + a[main:].T @ b[main:]
    return out


def _col_sum(a):
    """a.sum(dim=0) as a two-stage reduction over equal row chunks."""
    parts, q = _split_k(a.shape[0])
    if not parts:
        return a.sum(dim=0)
    main = parts * q
    out = a[:main].reshape(parts, q, a.shape[1]).sum(dim=1).sum(dim=0)
    if main < a.shape[0]:
        out = out + a[main:].sum(dim=0)
    return out


def nrf_backward(field, x: torch.Tensor, upstream: torch.Tensor, cache):
    """(d_weights, d_biases, d_points) of sum_b upstream_b r(x_b)."""
    t, pre, post = cache
    depth = len(field.weights)
    dws, dbs = [None] * depth, [None] * depth
    dz = (upstream * field.output_bound * (1.0 - t * t))[:, None]
    d_enc = None
    for li in range(depth - 1, -1, -1):
        dws[li] = _tn_matmul(post[li], dz)
        dbs[li] = _col_sum(dz)
        dh = dz @ field.weights[li].T
        if li > 0:  # dh * s (1 + z (1 - s)), s = sigmoid(z): one fused kernel
            dz = torch.ops.aten.silu_backward(dh, pre[li - 1])
        else:
            d_enc = dh
    bands = field.frequency_bands
    f = _freqs(bands, x)[None, :, None]  # (1, bands, 1)
    s = x[:, None, :] * f
    de = d_enc[:, 3:].reshape(x.shape[0], bands, 2, 3)
    dp = d_enc[:, :3] + (f * (torch.cos(s) * de[:, :, 0] - torch.sin(s) * de[:, :, 1])).sum(dim=1)
    return dws, dbs, dp


