"""Block partition grid on the device -- drop-in for
/root/reference/pkg/src/mgauss/spatial.py (cell_index, PartitionGrid, build,
query_local).

The bucket assignment is evaluated in float64 exactly as numpy does
(floor((x + 1) * (G / 2)), clamped), and the counting sort's in-cell rank
pass (csrc/mg_sort.cu) keeps ascending primitive order inside a cell, so
``cell_starts`` and ``cell_indices`` are bit-identical to the reference.
"""

from __future__ import annotations

from dataclasses import dataclass, field as dc_field

import numpy as np
import torch

from . import _device as dv
from . import _native as N
from .core import GaussianField


def cell_index(mu, grid_resolution):
    """(…,3) float64 positions -> (…,3) int64 cell coordinates (spatial.py:18-27)."""
    g = int(grid_resolution)
    mu_np = np.asarray(mu, dtype=np.float64)
    shape = mu_np.shape
    pos = dv.to_dev(mu_np.reshape(-1, 3), torch.float64)
    keys = dv.empty((pos.shape[0],), torch.int32)
    N.check(N.lib().mg_cell_keys_f64(N.ptr(pos), pos.shape[0], g, N.ptr(keys), dv.sptr()), "cell_index")
    flat = dv.to_host(keys).astype(np.int64) & 0xFFFFFFFF
    out = np.stack([flat // (g * g), (flat // g) % g, flat % g], axis=1)
    return out.reshape(shape)


@dataclass
class PartitionGrid:
    """Uniform cell grid mapping cell -> primitive indices (CSR, spatial.py:30-43).

    ``cell_starts``/``cell_indices`` are the reference's int64 host arrays;
    ``device`` caches the int32 device CSR (+ sorted keys) the kernels use."""

    grid_resolution: int
    block_radius: int
    count: int
    cell_starts: np.ndarray
    cell_indices: np.ndarray
    device: dict = dc_field(default=None, repr=False, compare=False)

    def bucket(self, i, j, k):
        g = self.grid_resolution
        flat = (i * g + j) * g + k
        return self.cell_indices[self.cell_starts[flat]:self.cell_starts[flat + 1]]


def build_device(positions: torch.Tensor, grid_resolution: int):
    """Device CSR from a (N,3) float32/float64 device tensor.

    Returns dict(keys=uint32-as-int32 (N,), order=int32 (N,), starts=int32 (G^3+1,))."""
    g = int(grid_resolution)
    n = positions.shape[0]
    keys = dv.empty((n,), torch.int32)
    order = dv.empty((n,), torch.int32)
    starts = dv.empty((g ** 3 + 1,), torch.int32)
    ws = dv.workspace(N.lib().mg_bin_workspace_bytes(n, g), "bin")
    fn = N.lib().mg_bin_f32 if positions.dtype == torch.float32 else N.lib().mg_bin_f64
    N.check(fn(N.ptr(positions.contiguous()), n, g, N.ptr(keys), N.ptr(order), N.ptr(starts), N.ptr(ws),
               ws.numel(), dv.sptr()), "build")
    return {"keys": keys, "order": order, "starts": starts}


def build(field, grid_resolution, block_radius=5):
    """Bucket every primitive into a G^3 grid (spatial.py:46-66)."""
    positions = field.positions if isinstance(field, GaussianField) else field
    if isinstance(positions, torch.Tensor):
        pos = positions.detach()
        if pos.device.type != "cuda":
            pos = dv.to_dev(pos, torch.float64)
    else:
        pos = dv.to_dev(np.asarray(positions, dtype=np.float64).reshape(-1, 3), torch.float64)
    g = int(grid_resolution)
    d = build_device(pos, g)
    return PartitionGrid(
        grid_resolution=g,
        block_radius=int(block_radius),
        count=int(pos.shape[0]),
        cell_starts=dv.to_host(d["starts"]).astype(np.int64),
        cell_indices=dv.to_host(d["order"]).astype(np.int64),
        device=d,
    )


def query_local(grid: PartitionGrid, x, radius=None):
    """Sorted primitive ids in the Chebyshev-r cell neighbourhood of x
    (spatial.py:69-95).  Host-side index arithmetic on the grid's CSR."""
    g = grid.grid_resolution
    r = grid.block_radius if radius is None else int(radius)
    c = cell_index(np.asarray(x, dtype=np.float64).reshape(1, 3), g)[0]
    lo = np.maximum(c - r, 0)
    hi = np.minimum(c + r, g - 1)
    chunks = []
    for i in range(lo[0], hi[0] + 1):
        for j in range(lo[1], hi[1] + 1):
            base = (i * g + j) * g
            a, b = grid.cell_starts[base + lo[2]], grid.cell_starts[base + hi[2] + 1]
            if b > a:
                chunks.append(grid.cell_indices[a:b])
    if not chunks:
        return np.empty(0, dtype=np.int64)
    return np.sort(np.concatenate(chunks))
