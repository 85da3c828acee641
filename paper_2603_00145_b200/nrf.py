"""Neural Residual Field on the device (/root/reference/pkg/src/mgauss/nrf.py).

r(x) = 0.1 * tanh(MLP(enc(x))), enc = [x, sin(2^k pi x), cos(2^k pi x)]_{k<6}
(39 dims), hidden widths (64, 64, 64, 64) with SiLU, zero-initialised last
layer (nrf.py:23-137).  Forward and the manual backward of nrf.py:147-182
(weight/bias gradients and d/dx into the slice transforms) run in the fused
float32 SIMT kernels of csrc/mg_nrf.cu (4 launches per step).
A16 allows tensor cores only if ncu shows the MLP is a dense-contraction
bottleneck; profiles/r02_nrf.md has the capture and the decision.  Only the
reference configuration (6 bands, 64 x 4 hidden, output bound 0.1) exists on
the device: any other width raises UnsupportedResidualField (no second
backend).  The torch-op restatement used as a test reference lives in
tests/nrf_mirror.py.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field as dc_field

import numpy as np
import torch

from . import _device as dv
from .errors import UninitializedField, UnsupportedResidualField

OUTPUT_BOUND = 0.1
DEFAULT_BANDS = 6
DEFAULT_HIDDEN = (64, 64, 64, 64)


def init_arrays(rng=None, frequency_bands=DEFAULT_BANDS, hidden=DEFAULT_HIDDEN):
    """(widths, weights, biases) as float64 numpy arrays drawn from ``rng`` in
    the reference's order (nrf.py:58-83)."""
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
        ws.append(w)
        bs.append(np.zeros(fo))
    return widths, ws, bs


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
        widths, ws, bs = init_arrays(rng, frequency_bands, hidden)
        return cls(int(frequency_bands), widths, [dv.to_dev(w, torch.float32) for w in ws],
                   [dv.to_dev(b, torch.float32) for b in bs])

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


def _require_fused(field: ResidualField):
    if not field.weights:
        raise UninitializedField("residual field has no weights")
    if not fused_supported(field):
        raise UnsupportedResidualField(
            f"device NRF kernels implement the reference widths {FUSED_WIDTHS} with 6 bands and output bound 0.1; "
            f"got widths {tuple(field.layer_widths)}, {field.frequency_bands} bands")


def nrf_forward_device(field: ResidualField, x: torch.Tensor, chunk=1 << 20):
    _require_fused(field)
    out = torch.empty(x.shape[0], dtype=torch.float32, device=x.device)
    for lo in range(0, x.shape[0], chunk):
        xs = x[lo:lo + chunk].contiguous()
        t = torch.empty(xs.shape[0], dtype=torch.float32, device=x.device)
        _fused_forward(field, xs, None, out[lo:lo + chunk], t, None)
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
    _require_fused(field)
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


def nrf_forward(field: ResidualField, x):
    """Host-facing r(x) (numpy in, numpy out), nrf.py:132-137."""
    xt = dv.to_dev(np.atleast_2d(np.asarray(x, dtype=np.float64)), torch.float32)
    r = dv.to_host(nrf_forward_device(field, xt)).astype(np.float64)
    return float(r[0]) if np.asarray(x).ndim == 1 else r


# ---------------------------------------------------------------------------
# float64 residual field for strict-float64 training (csrc/mg_nrf64.cu)
# ---------------------------------------------------------------------------


@dataclass
class ResidualField64:
    """The residual network with float64 host weights (the reference's own
    representation, nrf.py:49-101), evaluated by the float64 kernels of
    mg_nrf64.cu: any widths <= 64 with <= 8 layers.  Used by
    train.StrictTrainer and the host-level nrf_forward64 / nrf_backward64."""

    frequency_bands: int = DEFAULT_BANDS
    layer_widths: tuple = ()
    weights: list = dc_field(default_factory=list)  # (fan_in, fan_out) float64 numpy
    biases: list = dc_field(default_factory=list)
    output_bound: float = OUTPUT_BOUND

    @classmethod
    def create(cls, rng=None, frequency_bands=DEFAULT_BANDS, hidden=DEFAULT_HIDDEN):
        widths, ws, bs = init_arrays(rng, frequency_bands, hidden)
        return cls(int(frequency_bands), widths, ws, bs)

    def parameter_arrays(self):
        out = {}
        for li, (w, b) in enumerate(zip(self.weights, self.biases)):
            out[f"w{li}"] = w
            out[f"b{li}"] = b
        return out


def _require_f64(field: ResidualField64):
    if not field.weights:
        raise UninitializedField("residual field has no weights")
    w = tuple(int(x) for x in field.layer_widths)
    if (len(w) < 2 or len(w) > 9 or w[0] != 3 + 6 * int(field.frequency_bands) or w[-1] != 1
            or max(w) > 64 or min(w) < 1):
        raise UnsupportedResidualField(
            f"float64 NRF kernels take widths <= 64 and <= 8 layers (input 3 + 6 bands, output 1); got {w}")


class Nrf64Cache:
    """Device-resident forward activations (the reference's ``cache``,
    nrf.py:140-145) plus the uploaded weights, consumed by nrf_backward_f64."""

    def __init__(self, field: ResidualField64, x: torch.Tensor):
        from . import _native as N

        self.x = x
        self.n = int(x.shape[0])
        self.widths = (ctypes.c_int32 * len(field.layer_widths))(*[int(v) for v in field.layer_widths])
        self.depth = len(field.layer_widths) - 1
        self.bands = int(field.frequency_bands)
        self.bound = float(field.output_bound)
        self.w = [dv.to_dev(np.ascontiguousarray(w), torch.float64) for w in field.weights]
        self.b = [dv.to_dev(np.ascontiguousarray(b), torch.float64) for b in field.biases]
        self.ws = torch.empty((max(1, N.lib().mg_nrf_f64_workspace_bytes(self.n)),), dtype=torch.uint8,
                              device=x.device)


def nrf_forward_cached_f64(field: ResidualField64, x: torch.Tensor):
    """(r (n,) float64 device tensor, cache) -- nrf.py:140-145 in float64."""
    _require_f64(field)
    x = x.to(torch.float64).contiguous()
    c = Nrf64Cache(field, x)
    from . import _native as N

    r = torch.empty((c.n,), dtype=torch.float64, device=x.device)
    w, b = _ptr_array(c.w), _ptr_array(c.b)  # kept alive across the call
    N.check(N.lib().mg_nrf_forward_f64(N.ptr(x), c.n, ctypes.addressof(w), ctypes.addressof(b),
                                       ctypes.addressof(c.widths), c.depth, c.bands, c.bound, N.ptr(r), N.ptr(c.ws),
                                       c.ws.numel(), dv.sptr()), "nrf_forward_f64")
    return r, c


def nrf_backward_f64(cache: Nrf64Cache, upstream: torch.Tensor):
    """(d_weights, d_biases as float64 numpy, d_points (n, 3) float64 device)
    of sum_b upstream[b] r(x_b) -- nrf.py:147-182 in float64."""
    up = upstream.to(torch.float64).contiguous()
    if up.numel() != cache.n:
        raise ValueError("upstream length does not match the cached batch")
    dws = [torch.empty_like(w) for w in cache.w]
    dbs = [torch.empty_like(b) for b in cache.b]
    from . import _native as N

    dp = torch.empty((cache.n, 3), dtype=torch.float64, device=up.device)
    w, b, gw, gb = _ptr_array(cache.w), _ptr_array(cache.b), _ptr_array(dws), _ptr_array(dbs)
    N.check(N.lib().mg_nrf_backward_f64(N.ptr(cache.x), cache.n, ctypes.addressof(w), ctypes.addressof(b),
                                        ctypes.addressof(cache.widths), cache.depth, cache.bands, cache.bound,
                                        N.ptr(up), N.ptr(dp), ctypes.addressof(gw), ctypes.addressof(gb),
                                        N.ptr(cache.ws), cache.ws.numel(), dv.sptr()), "nrf_backward_f64")
    return [dv.to_host(w) for w in dws], [dv.to_host(b) for b in dbs], dp


def nrf_forward64(field: ResidualField64, x):
    """Host-facing r(x), float64 numpy in and out (nrf.py:132-137)."""
    xt = dv.to_dev(np.atleast_2d(np.asarray(x, dtype=np.float64)), torch.float64)
    r, _ = nrf_forward_cached_f64(field, xt)
    r = dv.to_host(r)
    return float(r[0]) if np.asarray(x).ndim == 1 else r


def nrf_backward64(field: ResidualField64, x, upstream):
    """(d_weights, d_biases, d_points) of sum_b upstream[b] r(x_b), float64
    numpy (nrf.py:147-182)."""
    xt = dv.to_dev(np.atleast_2d(np.asarray(x, dtype=np.float64)), torch.float64)
    _, cache = nrf_forward_cached_f64(field, xt)
    dws, dbs, dp = nrf_backward_f64(cache, dv.to_dev(np.asarray(upstream, np.float64).reshape(-1), torch.float64))
    return dws, dbs, dv.to_host(dp)
