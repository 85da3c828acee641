"""Forward evaluation of the Gaussian intensity field and its analytic
gradients on B200 -- drop-in for /root/reference/pkg/src/mgauss/render.py.

Same function names, argument meaning, return types and exceptions as the
reference (render.py:80-408); the pair loops run in the sm_100a kernels of
``csrc/`` through the C ABI (include/mgauss_b200.h).  There is no CPU
fallback: without the built library and a CUDA device every call raises
NativeLibraryMissing.

Extension beyond the reference: ``slice_psf`` integrates a
through-plane slice profile, I_psf(p) = sum_t w_t I(T_k(p + off_t * dir_k)).
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as dv
from . import _native as N
from .core import LOG_SCALE_LIMIT, TransformSet, Volume  # noqa: F401  (re-export)
from .errors import DegenerateQuaternion, InconsistentGrid, OutOfMemoryRequest
from .spatial import PartitionGrid

MAX_VOLUME_VOXELS = 2 ** 27  # render.py:35

_num_threads = 1
_strict_fp64 = os.environ.get("MGAUSS_STRICT_FP64", "0") not in ("", "0")


def set_num_threads(n):
    """Worker count of the reference's CPU kernels (render.py:44-55).

    Kept for API compatibility (the reference CLI calls it, cli.py:472-479).
    The device kernels have no host worker threads and their reductions are
    fixed-order, so results do not depend on this value."""
    global _num_threads
    _num_threads = max(1, int(n))


def get_num_threads():
    return _num_threads


def set_strict_fp64(on=True):
    """Select the strict float64 pair kernels (mg_block_forward_f64 /
    mg_block_backward_f64) for render_points, render_backward,
    render_points_dense and sample_volume: every pair in IEEE float64 in the
    reference's operation order (_kernels.py:24-162), ~1e-15 relative to the
    reference.  Default off: the float32 kernels (rel. error ~1e-6, within the
    1e-4 contract) are 10-20x faster.  MGAUSS_STRICT_FP64=1 sets it at import."""
    global _strict_fp64
    _strict_fp64 = bool(on)


def get_strict_fp64():
    return _strict_fp64


@dataclass
class RenderBatch:
    points: np.ndarray  # (B, 3) post-transform query coordinates ((B, T, 3) with a PSF)
    intensities: np.ndarray  # (B,)
    contributor_counts: np.ndarray  # (B,) int64


@dataclass
class RenderGradients:
    d_positions: np.ndarray  # (N, 3)
    d_quaternions: np.ndarray  # (N, 4)
    d_log_scales: np.ndarray  # (N, 3)
    d_intensity_logits: np.ndarray  # (N,)
    d_transform_params: np.ndarray  # (K, 7): 4 quaternion + 3 translation
    d_points: np.ndarray  # (B, 3) w.r.t. transformed query coordinates ((B, T, 3) with a PSF)


@dataclass
class SlicePSF:
    """Through-plane slice profile: tap offsets (T,) in normalized units along
    each slice's through-plane unit vector through_dirs (K, 3), weights (T,)."""

    offsets: np.ndarray
    weights: np.ndarray
    through_dirs: np.ndarray

    @property
    def ntaps(self):
        return int(np.asarray(self.offsets).shape[0])


# ---------------------------------------------------------------------------
# argument normalisation (render.py:97-158)
# ---------------------------------------------------------------------------


def _as_batch(samples):
    if hasattr(samples, "coords"):
        coords = np.ascontiguousarray(samples.coords, dtype=np.float64).reshape(-1, 3)
        sids = getattr(samples, "slice_ids", None)
        if sids is None:
            sids = np.full(coords.shape[0], -1, dtype=np.int64)
        return coords, np.ascontiguousarray(sids, dtype=np.int64).reshape(-1)
    if isinstance(samples, np.ndarray):
        coords = np.ascontiguousarray(samples, dtype=np.float64).reshape(-1, 3)
        return coords, np.full(coords.shape[0], -1, dtype=np.int64)
    coords = np.array([np.asarray(s.coord, dtype=np.float64) for s in samples]).reshape(-1, 3)
    sids = np.array([getattr(s, "slice_id", -1) for s in samples], dtype=np.int64)
    return coords, sids


def _as_transforms(transforms):
    if transforms is None:
        return None
    if isinstance(transforms, TransformSet):
        return transforms
    return TransformSet.from_list(list(transforms))


def _transform_arrays(transforms):
    ts = _as_transforms(transforms)
    if ts is None or len(ts) == 0:
        return np.zeros((1, 3, 3)), np.zeros((1, 3)), 0, ts
    return (np.ascontiguousarray(ts.rotations()),
            np.ascontiguousarray(ts.translations, dtype=np.float64), len(ts), ts)


def _check_grid(field, grid):
    if grid.count != field.count:
        raise InconsistentGrid(f"grid indexes {grid.count} primitives, field holds {field.count}")


# ---------------------------------------------------------------------------
# device staging
# ---------------------------------------------------------------------------


def _activate_dev(field):
    """float64 activated parameters on the device (render.py:122-142)."""
    n = field.count
    q = dv.to_dev(field.quaternions, torch.float64, (n, 4))
    s = dv.to_dev(field.log_scales, torch.float64, (n, 3))
    lg = dv.to_dev(field.intensity_logits, torch.float64, (n,))
    qn = dv.empty((n, 4), torch.float64)
    rot = dv.empty((n, 3, 3), torch.float64)
    iv = dv.empty((n, 3), torch.float64)
    p6 = dv.empty((n, 6), torch.float64)
    al = dv.empty((n,), torch.float64)
    err = dv.zeros((1,), torch.int32)
    N.check(N.lib().mg_activate_f64(N.ptr(q), N.ptr(s), N.ptr(lg), n, N.ptr(qn), N.ptr(rot), N.ptr(iv),
                                    N.ptr(p6), N.ptr(al), N.ptr(err), dv.sptr()), "activate")
    if n and int(err.item()):
        raise DegenerateQuaternion("quaternion norm <= 1e-12")
    return qn, rot, iv, p6, al


def activated_parameters(field):
    """(unit quats, rotations, inverse variances, packed precisions, alphas), float64."""
    return tuple(dv.to_host(t) for t in _activate_dev(field))


def _prepared_dev(field, prepared):
    if prepared is None:
        return _activate_dev(field)
    return tuple(dv.to_dev(a, torch.float64) for a in prepared)


def _grid_dev(grid: PartitionGrid):
    d = grid.device
    if d is not None and "starts64" in d:
        return d
    g = grid.grid_resolution
    cs64 = dv.to_dev(grid.cell_starts, torch.int64, (g ** 3 + 1,))
    ci64 = dv.to_dev(grid.cell_indices, torch.int64, (grid.count,))
    d = dict(d or {})
    d["starts64"], d["order64"] = cs64, ci64
    if "starts" not in d:
        st = dv.empty((g ** 3 + 1,), torch.int32)
        od = dv.empty((grid.count,), torch.int32)
        N.check(N.lib().mg_i64_to_i32(N.ptr(cs64), cs64.numel(), N.ptr(st), dv.sptr()))
        N.check(N.lib().mg_i64_to_i32(N.ptr(ci64), ci64.numel(), N.ptr(od), dv.sptr()))
        d["starts"], d["order"] = st, od
    keys = dv.empty((grid.count,), torch.int32)
    N.check(N.lib().mg_keys_from_csr(N.ptr(d["starts"]), g ** 3, N.ptr(keys), dv.sptr()))
    d["keys_csr"] = keys
    grid.device = d
    return d


def _records(field, gd, prec6, alpha):
    n = field.count
    mu = dv.to_dev(field.positions, torch.float64, (n, 3))
    grec = dv.empty((n, 12), torch.float32)
    N.check(N.lib().mg_pack_records(N.ptr(mu), N.ptr(prec6), N.ptr(alpha), N.ptr(gd["order"]), n, N.ptr(grec),
                                    dv.sptr()), "pack_records")
    return mu, grec


# ---------------------------------------------------------------------------
# render_points / render_backward (render.py:161-187, 276-354)
# ---------------------------------------------------------------------------


def render_points(field, grid, transforms, samples, radius=None, prepared=None, slice_psf=None):
    """Evaluate I at every sample after its slice's rigid transform."""
    _check_grid(field, grid)
    coords, sids = _as_batch(samples)
    rot, trans, k, _ = _transform_arrays(transforms)
    r = grid.block_radius if radius is None else int(radius)
    g = grid.grid_resolution
    b = coords.shape[0]
    _, _, _, p6, al = _prepared_dev(field, prepared)
    gd = _grid_dev(grid)
    L = N.lib()
    st = dv.sptr()
    if _strict_fp64:
        return _strict_render(field, gd, p6, al, coords, sids, rot, trans, k, g, r, slice_psf)
    c_d = dv.to_dev(coords, torch.float64)
    s_d = dv.to_dev(sids, torch.int64)
    rot_d = dv.to_dev(rot, torch.float64)
    tr_d = dv.to_dev(trans, torch.float64)
    if slice_psf is None:
        n = field.count
        mu = dv.to_dev(field.positions, torch.float64, (n, 3))
        out_i = dv.empty((b,), torch.float64)
        out_c = dv.empty((b,), torch.int64)
        out_x = dv.empty((b, 3), torch.float64)
        ws = dv.workspace(L.mg_block_workspace_bytes(b, n, g))
        N.check(L.mg_block_forward(N.ptr(c_d), N.ptr(s_d), b, N.ptr(rot_d), N.ptr(tr_d), k, N.ptr(mu), N.ptr(p6),
                                   N.ptr(al), n, N.ptr(gd["starts64"]), N.ptr(gd["order64"]), g, r, N.ptr(out_i),
                                   N.ptr(out_c), N.ptr(out_x), N.ptr(ws), ws.numel(), st), "block_forward")
        return RenderBatch(points=dv.to_host(out_x), intensities=dv.to_host(out_i),
                           contributor_counts=dv.to_host(out_c))
    stg = _stage_psf(field, gd, p6, al, c_d, s_d, rot_d, tr_d, k, g, slice_psf, with_h=False, radius=r)
    t = slice_psf.ntaps
    return RenderBatch(points=dv.to_host(stg["x"]).reshape(b, t, 3), intensities=dv.to_host(stg["I"]),
                       contributor_counts=dv.to_host(stg["cnt"]))


def _psf_expand(coords, sids, psf):
    """(b*t, 3) tap points p + off_t * dir_k in (b, t) order, as the oracle
    composes them (I_psf = sum_t w_t I(T_k(p + off_t dir_k)))."""
    dirs = np.asarray(psf.through_dirs, dtype=np.float64).reshape(-1, 3)
    shift = dirs[np.clip(sids, 0, None)] * (sids >= 0)[:, None]
    taps = [coords + off * shift for off in np.asarray(psf.offsets, dtype=np.float64)]
    return np.ascontiguousarray(np.stack(taps, axis=1).reshape(-1, 3)), np.repeat(sids, psf.ntaps)


def _strict_call(fn, field, gd, p6, al, coords, sids, rot, trans, k, g, r, up=None, acc=None):
    """One strict float64 kernel call (mg_block_forward_f64 / _backward_f64)."""
    L = N.lib()
    n, b = field.count, coords.shape[0]
    mu = dv.to_dev(field.positions, torch.float64, (n, 3))
    c_d = dv.to_dev(coords, torch.float64)
    s_d = dv.to_dev(sids, torch.int64)
    rot_d = dv.to_dev(rot, torch.float64)
    tr_d = dv.to_dev(trans, torch.float64)
    ws = dv.workspace(L.mg_block_f64_workspace_bytes(b, n, g), "strict")
    if up is None:
        out_i = dv.empty((b,), torch.float64)
        out_c = dv.empty((b,), torch.int64)
        out_x = dv.empty((b, 3), torch.float64)
        N.check(L.mg_block_forward_f64(N.ptr(c_d), N.ptr(s_d), b, N.ptr(rot_d), N.ptr(tr_d), k, N.ptr(mu),
                                       N.ptr(p6), N.ptr(al), n, N.ptr(gd["starts64"]), N.ptr(gd["order64"]), g, r,
                                       N.ptr(out_i), N.ptr(out_c), N.ptr(out_x), N.ptr(ws), ws.numel(), dv.sptr()),
                "block_forward_f64")
        return out_i, out_c, out_x
    d_mu, d_ab, d_al = acc
    u_d = dv.to_dev(up, torch.float64)
    d_pts = dv.empty((b, 3), torch.float64)
    N.check(L.mg_block_backward_f64(N.ptr(c_d), N.ptr(s_d), b, N.ptr(rot_d), N.ptr(tr_d), k, N.ptr(mu), N.ptr(p6),
                                    N.ptr(al), n, N.ptr(gd["starts64"]), N.ptr(gd["order64"]), g, r, N.ptr(u_d),
                                    N.ptr(d_mu), N.ptr(d_ab), N.ptr(d_al), N.ptr(d_pts), N.ptr(ws), ws.numel(),
                                    dv.sptr()), "block_backward_f64")
    return d_pts


def _strict_render(field, gd, p6, al, coords, sids, rot, trans, k, g, r, psf):
    b = coords.shape[0]
    if psf is None:
        out_i, out_c, out_x = _strict_call(None, field, gd, p6, al, coords, sids, rot, trans, k, g, r)
        return RenderBatch(points=dv.to_host(out_x), intensities=dv.to_host(out_i),
                           contributor_counts=dv.to_host(out_c))
    t = psf.ntaps
    xc, xs = _psf_expand(coords, sids, psf)
    out_i, out_c, out_x = _strict_call(None, field, gd, p6, al, xc, xs, rot, trans, k, g, r)
    it = dv.to_host(out_i).reshape(b, t)
    ct = dv.to_host(out_c).reshape(b, t)
    inten = np.zeros(b)
    for j, w in enumerate(np.asarray(psf.weights, dtype=np.float64)):
        inten += w * it[:, j]
    return RenderBatch(points=dv.to_host(out_x).reshape(b, t, 3), intensities=inten,
                       contributor_counts=ct.sum(axis=1))


def _stage_psf(field, gd, p6, al, c_d, s_d, rot_d, tr_d, k, g, psf, with_h, radius):
    """Staged device path with slice-PSF tap expansion (mg_bin_points/forward/finish)."""
    L = N.lib()
    st = dv.sptr()
    b = c_d.shape[0]
    t = psf.ntaps
    ns = b * t
    off = dv.to_dev(np.asarray(psf.offsets, dtype=np.float64), torch.float64)
    wts = dv.to_dev(np.asarray(psf.weights, dtype=np.float64), torch.float64)
    dirs = dv.to_dev(np.asarray(psf.through_dirs, dtype=np.float64).reshape(-1, 3), torch.float64)
    _, grec = _records(field, gd, p6, al)
    pkey = dv.empty((ns,), torch.int32)
    pinv = dv.empty((ns,), torch.int32)
    pstart = dv.empty((g ** 3 + 1,), torch.int32)
    prec = dv.empty((ns, 4), torch.float32)
    x = dv.empty((ns, 3), torch.float64)
    ws = dv.workspace(max(L.mg_points_workspace_bytes(ns, g), L.mg_forward_workspace_bytes(ns),
                          L.mg_backward_workspace_bytes(field.count, g)))
    N.check(L.mg_bin_points(N.ptr(c_d), N.ptr(s_d), b, t, N.ptr(off), N.ptr(dirs), N.ptr(rot_d), N.ptr(tr_d), k, g,
                            N.ptr(pkey), N.ptr(pinv), N.ptr(pstart), N.ptr(prec), N.ptr(x), N.ptr(ws), ws.numel(),
                            st), "bin_points")
    out4 = dv.empty((ns, 4), torch.float32)
    cnt = dv.empty((ns,), torch.int32)
    N.check(L.mg_forward(N.ptr(grec), field.count, N.ptr(gd["starts"]), g, radius, N.ptr(prec), N.ptr(pkey),
                         N.ptr(pstart), ns,
                         1 if with_h else 0, N.ptr(out4), N.ptr(cnt), N.ptr(ws), ws.numel(), st), "forward")
    I = dv.empty((b,), torch.float64)
    c64 = dv.empty((b,), torch.int64)
    N.check(L.mg_forward_finish(N.ptr(out4), N.ptr(cnt), N.ptr(pinv), b, t, N.ptr(wts), N.ptr(I), None, N.ptr(c64),
                                None, st), "forward_finish")
    return dict(grec=grec, pkey=pkey, pinv=pinv, pstart=pstart, prec=prec, x=x, out4=out4, I=I, cnt=c64, off=off,
                wts=wts, dirs=dirs, ws=ws)


def render_points_dense(field, samples, transforms=None):
    """All-primitive evaluation, no spatial truncation (render.py:190-204)."""
    coords, sids = _as_batch(samples)
    if transforms is not None:
        rot, trans, k, _ = _transform_arrays(transforms)
        if k:
            sc = sids.clip(min=0)
            moved = np.einsum("kij,bj->bi", rot[sc], coords) + trans[sc]
            coords = np.where(sids[:, None] >= 0, moved, coords)
    _, _, _, p6, al = _activate_dev(field)
    n = field.count
    if _strict_fp64:  # one cell holding every primitive in index order: all pairs, _kernels.py:147-162
        gd = {"starts64": dv.to_dev(np.array([0, n], np.int64), torch.int64),
              "order64": dv.to_dev(np.arange(n, dtype=np.int64), torch.int64)}
        c = np.ascontiguousarray(coords, dtype=np.float64)
        out_i, _, _ = _strict_call(None, field, gd, p6, al, c, np.full(c.shape[0], -1, np.int64),
                                   np.zeros((1, 3, 3)), np.zeros((1, 3)), 0, 1, 0)
        return dv.to_host(out_i)
    L = N.lib()
    mu = dv.to_dev(field.positions, torch.float64, (n, 3))
    pts = dv.to_dev(coords, torch.float64)
    out = dv.empty((coords.shape[0],), torch.float64)
    ws = dv.workspace(L.mg_dense_workspace_bytes(n), "dense")
    N.check(L.mg_dense_forward(N.ptr(pts), pts.shape[0], N.ptr(mu), N.ptr(p6), N.ptr(al), n, N.ptr(out), N.ptr(ws),
                               ws.numel(), dv.sptr()), "dense_forward")
    return dv.to_host(out)


def transform_grads_from_points(transforms, coords, sids, d_points, slice_psf=None):
    """(K, 7) per-slice [d_quat(4), d_trans(3)] from point gradients (render.py:246-273)."""
    ts = _as_transforms(transforms)
    if ts is None or len(ts) == 0:
        return np.zeros((0, 7))
    k = len(ts)
    c_d = dv.to_dev(np.asarray(coords, dtype=np.float64).reshape(-1, 3), torch.float64)
    s_d = dv.to_dev(np.asarray(sids, dtype=np.int64).reshape(-1), torch.int64)
    h_d = d_points if isinstance(d_points, torch.Tensor) else dv.to_dev(
        np.asarray(d_points, dtype=np.float64).reshape(-1, 3), torch.float64)
    return dv.to_host(_transform_grads_dev(ts, c_d, s_d, h_d, slice_psf))


def _transform_grads_dev(ts, c_d, s_d, h_d, psf=None, off=None, dirs=None):
    k = len(ts)
    tq = dv.to_dev(ts.quats, torch.float64, (k, 4))
    scratch = dv.empty((k, 12), torch.float64)
    out = dv.empty((k, 7), torch.float64)
    t = 1 if psf is None else psf.ntaps
    if psf is not None and off is None:
        off = dv.to_dev(np.asarray(psf.offsets, dtype=np.float64), torch.float64)
        dirs = dv.to_dev(np.asarray(psf.through_dirs, dtype=np.float64).reshape(-1, 3), torch.float64)
    L = N.lib()
    ws = dv.workspace(L.mg_transform_grads_workspace_bytes(k), "transform")
    N.check(L.mg_transform_grads(N.ptr(h_d), N.ptr(c_d), N.ptr(s_d), c_d.shape[0], t, N.ptr(off), N.ptr(dirs),
                                 N.ptr(tq), k, N.ptr(scratch), N.ptr(out), 0, N.ptr(ws), ws.numel(), dv.sptr()),
            "transform_grads")
    return out


def render_backward(field, grid, transforms, samples, upstream, radius=None, prepared=None, slice_psf=None):
    """Gradients of sum_b upstream[b] * I(x_b) for every parameter group."""
    _check_grid(field, grid)
    coords, sids = _as_batch(samples)
    up = np.ascontiguousarray(upstream, dtype=np.float64).reshape(-1)
    if up.shape[0] != coords.shape[0]:
        raise ValueError("upstream length does not match sample count")
    if not _strict_fp64 and up.size and np.abs(up).max() > 1e14:
        # the float32 kernels carry u * 2^79.8 in the point records (exponent-offset cutoff, mg_common.cuh)
        raise ValueError("|upstream| > 1e14 exceeds the float32 kernels' range; use render.set_strict_fp64(True)")
    rot, trans, k, ts = _transform_arrays(transforms)
    r = grid.block_radius if radius is None else int(radius)
    g = grid.grid_resolution
    n = field.count
    b = coords.shape[0]
    _, _, _, p6, al = _prepared_dev(field, prepared)
    gd = _grid_dev(grid)
    L = N.lib()
    st = dv.sptr()
    c_d = dv.to_dev(coords, torch.float64)
    s_d = dv.to_dev(sids, torch.int64)
    rot_d = dv.to_dev(rot, torch.float64)
    tr_d = dv.to_dev(trans, torch.float64)
    u_d = dv.to_dev(up, torch.float64)
    d_mu = dv.zeros((n, 3), torch.float64)
    d_ab = dv.zeros((n, 6), torch.float64)
    d_al = dv.zeros((n,), torch.float64)
    t = 1 if slice_psf is None else slice_psf.ntaps
    off = dirs = None
    if _strict_fp64:
        if slice_psf is None:
            d_pts = _strict_call(None, field, gd, p6, al, coords, sids, rot, trans, k, g, r, up, (d_mu, d_ab, d_al))
        else:
            xc, xs = _psf_expand(coords, sids, slice_psf)
            upt = (up[:, None] * np.asarray(slice_psf.weights, dtype=np.float64)[None, :]).reshape(-1)
            d_pts = _strict_call(None, field, gd, p6, al, xc, xs, rot, trans, k, g, r, upt, (d_mu, d_ab, d_al))
    elif slice_psf is None:
        mu = dv.to_dev(field.positions, torch.float64, (n, 3))
        d_pts = dv.empty((b, 3), torch.float64)
        ws = dv.workspace(L.mg_block_workspace_bytes(b, n, g))
        N.check(L.mg_block_backward(N.ptr(c_d), N.ptr(s_d), b, N.ptr(rot_d), N.ptr(tr_d), k, N.ptr(mu), N.ptr(p6),
                                    N.ptr(al), n, N.ptr(gd["starts64"]), N.ptr(gd["order64"]), g, r, N.ptr(u_d),
                                    N.ptr(d_mu), N.ptr(d_ab), N.ptr(d_al), N.ptr(d_pts), N.ptr(ws), ws.numel(), st),
                "block_backward")
    else:
        stg = _stage_psf(field, gd, p6, al, c_d, s_d, rot_d, tr_d, k, g, slice_psf, with_h=True, radius=r)
        off, dirs = stg["off"], stg["dirs"]
        d_pts = dv.empty((b * t, 3), torch.float64)
        N.check(L.mg_backward_points(N.ptr(u_d), None, b, t, N.ptr(stg["wts"]), N.ptr(stg["pinv"]),
                                     N.ptr(stg["out4"]), N.ptr(stg["prec"]), N.ptr(d_pts), st), "backward_points")
        acc = dv.empty((n, 10), torch.float32)
        ws = stg["ws"]
        N.check(L.mg_backward(N.ptr(stg["grec"]), N.ptr(gd["keys_csr"]), N.ptr(gd["starts"]), n, g, r,
                              N.ptr(stg["prec"]), N.ptr(stg["pstart"]), N.ptr(acc), N.ptr(ws), ws.numel(), st),
                "backward")
        N.check(L.mg_backward_accumulators(N.ptr(acc), N.ptr(gd["order"]), n, N.ptr(al), N.ptr(d_mu), N.ptr(d_ab),
                                           N.ptr(d_al), st), "backward_accumulators")
    if _strict_fp64 and slice_psf is not None and k:
        off = dv.to_dev(np.asarray(slice_psf.offsets, dtype=np.float64), torch.float64)
        dirs = dv.to_dev(np.asarray(slice_psf.through_dirs, dtype=np.float64).reshape(-1, 3), torch.float64)
    q = dv.to_dev(field.quaternions, torch.float64, (n, 4))
    s = dv.to_dev(field.log_scales, torch.float64, (n, 3))
    lg = dv.to_dev(field.intensity_logits, torch.float64, (n,))
    dp, dq, ds, dl = (dv.empty((n, 3), torch.float64), dv.empty((n, 4), torch.float64),
                      dv.empty((n, 3), torch.float64), dv.empty((n,), torch.float64))
    N.check(L.mg_epilogue_f64(N.ptr(d_mu), N.ptr(d_ab), N.ptr(d_al), N.ptr(q), N.ptr(s), N.ptr(lg), n, N.ptr(dp),
                              N.ptr(dq), N.ptr(ds), N.ptr(dl), st), "epilogue")
    if k:
        d_t = dv.to_host(_transform_grads_dev(ts, c_d, s_d, d_pts, slice_psf, off, dirs))
    else:
        d_t = np.zeros((0, 7))
    dpts = dv.to_host(d_pts)
    if slice_psf is not None:
        dpts = dpts.reshape(b, t, 3)
    return RenderGradients(d_positions=dv.to_host(dp), d_quaternions=dv.to_host(dq),
                           d_log_scales=dv.to_host(ds), d_intensity_logits=dv.to_host(dl),
                           d_transform_params=d_t, d_points=dpts)


# ---------------------------------------------------------------------------
# inference (render.py:357-408)
# ---------------------------------------------------------------------------


def grid_coordinates(dims, bounds):
    """Node-inclusive per-axis coordinates (render.py:357-376)."""
    lo = np.asarray(bounds[0], dtype=np.float64)
    hi = np.asarray(bounds[1], dtype=np.float64)
    axes, spacing = [], np.empty(3)
    for a in range(3):
        n = int(dims[a])
        if n == 1:
            axes.append(np.array([0.5 * (lo[a] + hi[a])]))
            spacing[a] = hi[a] - lo[a]
        else:
            spacing[a] = (hi[a] - lo[a]) / (n - 1)
            axes.append(lo[a] + np.arange(n) * spacing[a])
    return axes, spacing


def sample_volume_device(grec, n_gauss, gstart, g, r, dims, bounds, i0=0, i1=None, residual=None):
    """Device slab [i0, i1) of the clipped volume as a float32 (i1-i0, ny, nz) tensor."""
    nx, ny, nz = (int(d) for d in dims)
    i1 = nx if i1 is None else int(i1)
    L = N.lib()
    lo = np.ascontiguousarray(np.asarray(bounds[0], dtype=np.float64).reshape(3))
    hi = np.ascontiguousarray(np.asarray(bounds[1], dtype=np.float64).reshape(3))
    out = dv.empty((i1 - i0, ny, nz), torch.float32)
    ws = dv.workspace(L.mg_volume_workspace_bytes(nx, ny, nz), "volume")
    N.check(L.mg_sample_volume(N.ptr(grec), int(n_gauss), N.ptr(gstart), g, r, nx, ny, nz, lo.ctypes.data_as(N.P),
                               hi.ctypes.data_as(N.P), i0, i1, N.ptr(residual), N.ptr(out), N.ptr(ws), ws.numel(),
                               dv.sptr()), "sample_volume")
    return out


def sample_volume(field, grid, residual, dims, bounds=((-1.0, -1.0, -1.0), (1.0, 1.0, 1.0)), radius=None,
                  max_voxels=MAX_VOLUME_VOXELS, chunk=65536):
    """Evaluate the field (+ optional residual) on a dense node-inclusive grid, clipped to [0, 1]."""
    dims = tuple(int(d) for d in dims)
    if any(d < 1 for d in dims):
        raise ValueError("dims must all be >= 1")
    total = dims[0] * dims[1] * dims[2]
    if total > max_voxels:
        raise OutOfMemoryRequest(f"{total} voxels exceed cap {max_voxels}")
    axes, spacing = grid_coordinates(dims, bounds)
    origin = np.array([axes[0][0], axes[1][0], axes[2][0]])
    _check_grid(field, grid)
    r = grid.block_radius if radius is None else int(radius)
    g = grid.grid_resolution
    if field.count == 0:
        return Volume(data=np.zeros(dims), spacing=spacing, origin=origin)
    _, _, _, p6, al = _activate_dev(field)
    gd = _grid_dev(grid)
    if _strict_fp64:  # render.py:394-408: render_points over voxel chunks, float64
        gx, gy, gz = np.meshgrid(axes[0], axes[1], axes[2], indexing="ij")
        pts = np.stack([gx.ravel(), gy.ravel(), gz.ravel()], axis=1)
        out = np.empty(total)
        for c0 in range(0, total, max(1, int(chunk))):
            c1 = min(total, c0 + max(1, int(chunk)))
            oi, _, _ = _strict_call(None, field, gd, p6, al, np.ascontiguousarray(pts[c0:c1]),
                                    np.full(c1 - c0, -1, np.int64), np.zeros((1, 3, 3)), np.zeros((1, 3)), 0, g, r)
            out[c0:c1] = dv.to_host(oi)
        if residual is not None:
            from .nrf import nrf_forward_device

            out += dv.to_host(nrf_forward_device(residual, dv.to_dev(pts, torch.float32))).astype(np.float64)
        return Volume(data=np.clip(out, 0.0, 1.0).reshape(dims), spacing=spacing, origin=origin)
    _, grec = _records(field, gd, p6, al)
    res_d = None
    if residual is not None:
        from .nrf import nrf_forward_device

        gx, gy, gz = np.meshgrid(axes[0], axes[1], axes[2], indexing="ij")
        pts = dv.to_dev(np.stack([gx.ravel(), gy.ravel(), gz.ravel()], axis=1), torch.float32)
        res_d = nrf_forward_device(residual, pts).reshape(dims)
    lo = np.array(bounds[0], dtype=np.float64)
    hi = np.array(bounds[1], dtype=np.float64)
    out = sample_volume_device(grec, field.count, gd["starts"], g, r, dims, (lo, hi), residual=res_d)
    return Volume(data=dv.to_host(out).astype(np.float64), spacing=spacing, origin=origin)
