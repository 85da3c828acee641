"""Neural Residual Field on the device (/root/reference/pkg/src/mgauss/nrf.py).

r(x) = 0.1 * tanh(MLP(enc(x))), enc = [x, sin(2^k pi x), cos(2^k pi x)]_{k<6}
(39 dims), hidden widths (64, 64, 64, 64) with SiLU, zero-initialised last
layer.  The four dense layers are plain fp32 GEMMs (cuBLAS through torch);
SURVEY §8(a) A16 allows tensor cores only once ncu shows the MLP is a
dense-contraction bottleneck, and bf16/tf32 would break the 1e-4 parity.
Manual backward identical to nrf.py:147-182 (including d/dx into transforms).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field as dc_field

import numpy as np
import torch

from . import _device as dv
from .errors import UninitializedField

OUTPUT_BOUND = 0.1
DEFAULT_BANDS = 6
DEFAULT_HIDDEN = (64, 64, 64, 64)


@dataclass
class ResidualField:
    frequency_bands: int = DEFAULT_BANDS
    layer_widths: tuple = ()
    weights: list = dc_field(default_factory=list)  # (fan_in, fan_out) float32 device tensors
    biases: list = dc_field(default_factory=list)
    output_bound: float = OUTPUT_BOUND

    @classmethod
    def create(cls, rng=None, frequency_bands=DEFAULT_BANDS, hidden=DEFAULT_HIDDEN):
        """Same initialisation stream as nrf.py:58-83 (uniform +-sqrt(6/(fi+fo)), last layer 0)."""
        rng = np.random.default_rng(rng)
        widths = (3 + 6 * int(frequency_bands),) + tuple(hidden) + (1,)
        ws, bs = [], []
        for li in range(len(widths) - 1):
            fi, fo = widths[li], widths[li + 1]
            if li == len(widths) - 2:
                w = np.zeros((fi, fo))
            else:
                bound = np.sqrt(6.0 / (fi + fo))
                w = rng.uniform(-bound, bound, size=(fi, fo))
            ws.append(dv.to_dev(w, torch.float32))
            bs.append(dv.zeros((fo,), torch.float32))
        return cls(int(frequency_bands), widths, ws, bs)

    @classmethod
    def from_numpy(cls, weights, biases, frequency_bands=DEFAULT_BANDS):
        ws = [dv.to_dev(np.asarray(w), torch.float32) for w in weights]
        bs = [dv.to_dev(np.asarray(b), torch.float32) for b in biases]
        widths = (ws[0].shape[0],) + tuple(w.shape[1] for w in ws)
        return cls(int(frequency_bands), widths, ws, bs)

    def parameter_arrays(self):
        out = {}
        for li, (w, b) in enumerate(zip(self.weights, self.biases)):
            out[f"w{li}"] = w
            out[f"b{li}"] = b
        return out


def _freqs(bands, x):
    return (2.0 ** torch.arange(bands, dtype=x.dtype, device=x.device)) * np.pi


def fourier_encode(x: torch.Tensor, bands: int) -> torch.Tensor:
    """nrf.py:23-36 on device: [x, sin(2^0 pi x), cos(2^0 pi x), sin(2^1 pi x), ...],
    all bands in one broadcast (same column order as the reference)."""
    s = x[:, None, :] * _freqs(bands, x)[None, :, None]  # (B, bands, 3)
    sc = torch.stack((torch.sin(s), torch.cos(s)), dim=2)  # (B, bands, 2, 3)
    return torch.cat((x, sc.reshape(x.shape[0], 6 * bands)), dim=1)


def nrf_forward_cached(field: ResidualField, x: torch.Tensor):
    if not field.weights:
        raise UninitializedField("residual field has no weights")
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


def nrf_forward_device(field: ResidualField, x: torch.Tensor, chunk=1 << 20):
    out = torch.empty(x.shape[0], dtype=torch.float32, device=x.device)
    for lo in range(0, x.shape[0], chunk):
        if fused_supported(field):
            xs = x[lo:lo + chunk].contiguous()
            t = torch.empty(xs.shape[0], dtype=torch.float32, device=x.device)
            _fused_forward(field, xs, None, out[lo:lo + chunk], t, None)
        else:
            out[lo:lo + chunk] = nrf_forward_cached(field, x[lo:lo + chunk])[0]
    return out


# -- fused kernels (csrc/mg_nrf.cu): the reference widths in 4 launches -------
FUSED_WIDTHS = (39, 64, 64, 64, 64, 1)


def fused_supported(field: ResidualField) -> bool:
    """The fused kernels are written for the reference configuration
    (6 bands, hidden 64 x 4, output 1, output bound 0.1)."""
    return (tuple(field.layer_widths) == FUSED_WIDTHS and field.frequency_bands == 6
            and abs(field.output_bound - 0.1) < 1e-12 and all(w.is_contiguous() for w in field.weights))


def _ptr_array(tensors):
    return (ctypes.c_void_p * len(tensors))(*[t.data_ptr() for t in tensors])


def _fused_forward(field, x, pred_add, r_out, t_out, z_out):
    from . import _native as N

    w, b = _ptr_array(field.weights), _ptr_array(field.biases)
    N.check(N.lib().mg_nrf_forward(N.ptr(x), x.shape[0], ctypes.addressof(w), ctypes.addressof(b), N.ptr(pred_add),
                                   N.ptr(r_out), N.ptr(t_out), N.ptr(z_out), dv.sptr()), "nrf_forward")


def nrf_forward_fused(field: ResidualField, x: torch.Tensor, pred_add: torch.Tensor | None = None):
    """nrf_forward_cached on the fused kernel: (r or None, cache).  With
    ``pred_add`` the residual is added into it in place and r is not returned."""
    x = x.contiguous()
    n = x.shape[0]
    t = torch.empty(n, dtype=torch.float32, device=x.device)
    z = torch.empty((4, n, 64), dtype=torch.float32, device=x.device)
    r = None if pred_add is not None else torch.empty(n, dtype=torch.float32, device=x.device)
    _fused_forward(field, x, pred_add, r, t, z)
    return r, ("fused", t, z)


def nrf_backward_fused(field: ResidualField, x: torch.Tensor, upstream: torch.Tensor, cache, out=None):
    """nrf_backward on the fused kernels: (d_weights, d_biases, d_points);
    ``out = (d_weights, d_biases)`` writes the gradients into given tensors."""
    from . import _native as N

    _, t, z = cache
    x = x.contiguous()
    up = upstream[:x.shape[0]].to(torch.float32).contiguous()
    n = x.shape[0]
    L = N.lib()
    if out is not None:
        dws, dbs = list(out[0]), list(out[1])
    else:
        dws = [torch.empty_like(w) for w in field.weights]
        dbs = [torch.empty_like(b) for b in field.biases]
    dp = torch.empty((n, 3), dtype=torch.float32, device=x.device)
    ws = torch.empty((max(1, L.mg_nrf_backward_workspace_bytes(n)),), dtype=torch.uint8, device=x.device)
    w, b = _ptr_array(field.weights), _ptr_array(field.biases)
    gw, gb = _ptr_array(dws), _ptr_array(dbs)
    N.check(L.mg_nrf_backward(N.ptr(x), n, ctypes.addressof(w), ctypes.addressof(b), N.ptr(up), N.ptr(t), N.ptr(z),
                              N.ptr(dp), ctypes.addressof(gw), ctypes.addressof(gb), N.ptr(ws), ws.numel(),
                              dv.sptr()), "nrf_backward")
    return dws, dbs, dp


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


def nrf_backward(field: ResidualField, x: torch.Tensor, upstream: torch.Tensor, cache):
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


def nrf_forward(field: ResidualField, x):
    """Host-facing r(x) (numpy in, numpy out), nrf.py:132-137."""
    xt = dv.to_dev(np.atleast_2d(np.asarray(x, dtype=np.float64)), torch.float32)
    r = dv.to_host(nrf_forward_cached(field, xt)[0]).astype(np.float64)
    return float(r[0]) if np.asarray(x).ndim == 1 else r
