"""Device-memory plumbing for the host layer: torch tensors as raw HBM
buffers, a reusable per-device workspace, host<->device conversion."""

from __future__ import annotations

import numpy as np
import torch

from . import _native as N

_ws_cache: dict = {}


def device():
    N.lib()  # raises NativeLibraryMissing without a GPU / built library
    return torch.device("cuda", torch.cuda.current_device())


def workspace(nbytes: int, slot: str = "default") -> torch.Tensor:
    """A uint8 scratch buffer of at least nbytes (grown geometrically, reused)."""
    dev = device()
    key = (dev.index, slot)
    buf = _ws_cache.get(key)
    if buf is None or buf.numel() < nbytes:
        size = max(int(nbytes), 1 << 20)
        if buf is not None:
            size = max(size, int(buf.numel() * 1.5))
        buf = torch.empty(size, dtype=torch.uint8, device=dev)
        _ws_cache[key] = buf
    return buf


def to_dev(a, dtype, shape=None):
    """numpy / torch -> contiguous device tensor of dtype (copy only if needed)."""
    dev = device()
    if isinstance(a, torch.Tensor):
        t = a.to(device=dev, dtype=dtype)
    else:
        arr = np.ascontiguousarray(np.asarray(a))
        t = torch.from_numpy(arr).to(device=dev, dtype=dtype, non_blocking=False)
    t = t.contiguous()
    if shape is not None:
        t = t.reshape(shape)
    return t


def empty(shape, dtype):
    return torch.empty(shape, dtype=dtype, device=device())


def zeros(shape, dtype):
    return torch.zeros(shape, dtype=dtype, device=device())


def to_host(t):
    return t.detach().cpu().numpy()


def sptr():
    return N.stream_ptr()
