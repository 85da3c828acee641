"""torch-facing render API (north_star): ``render(gaussians, sample_coords,
slice_psf) -> intensities`` as a ``torch.autograd.Function`` whose forward and
backward are the reference's render_points / render_backward semantics
(/root/reference/pkg/src/mgauss/render.py:161-187, 276-354).

Everything runs on the device through the C ABI (the same staged calls the
trainer uses): Gaussian binning + activation, per-slice rigid transform and
slice-PSF tap expansion, the block forward (with H for the point gradient),
and on backward the Gaussian-major accumulators, the float64 epilogue and the
deterministic per-slice transform reduction.

Gradients flow to the four Gaussian parameter tensors, to the per-slice
transform quaternions / translations and to the sample coordinates
(``d coords = sum_t R_s^T h_t`` with ``h`` the transformed-point gradient of
render.py:292 ``d_points``).  Parameters are evaluated in float32 on the
device, as in the trainer; intensities and gradients come back in the input
dtype.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device as dv
from . import _native as N
from .errors import DegenerateQuaternion


def _f32(t):
    return t.detach().to(device=dv.device(), dtype=torch.float32).contiguous()


def _f64(t):
    return t.detach().to(device=dv.device(), dtype=torch.float64).contiguous()


class _Render(torch.autograd.Function):
    @staticmethod
    def forward(ctx, positions, quaternions, log_scales, logits, coords, tq, tt, sids, g, r, psf):
        L = N.lib()
        st = dv.sptr()
        n, b = positions.shape[0], coords.shape[0]
        t = 1 if psf is None else psf.ntaps
        ns = b * t
        k = 0 if tq is None else tq.shape[0]
        pos, q, s, lg = _f32(positions), _f32(quaternions), _f32(log_scales), _f32(logits)
        c64 = _f64(coords)
        sid = (sids if sids is not None else torch.full((b,), -1, dtype=torch.int64)).to(
            device=dv.device(), dtype=torch.int64).contiguous()
        tq64 = _f64(tq) if k else dv.zeros((1, 4), torch.float64)
        tt64 = _f64(tt) if k else dv.zeros((1, 3), torch.float64)
        rot = dv.empty((max(k, 1), 3, 3), torch.float64)
        if k:
            N.check(L.mg_quat_to_rot_f64(N.ptr(tq64), k, N.ptr(rot), st), "quat_to_rot")
        if psf is not None:
            off = _f64(torch.as_tensor(np.asarray(psf.offsets, dtype=np.float64)))
            wts = _f64(torch.as_tensor(np.asarray(psf.weights, dtype=np.float64)))
            dirs = _f64(torch.as_tensor(np.asarray(psf.through_dirs, dtype=np.float64).reshape(-1, 3)))
        else:
            off = wts = dirs = None
        ws = dv.workspace(max(L.mg_bin_workspace_bytes(n, g), L.mg_points_workspace_bytes(ns, g),
                              L.mg_forward_workspace_bytes(ns), L.mg_backward_workspace_bytes(n, g),
                              L.mg_transform_grads_workspace_bytes(k)), "torch_render")
        gkey = dv.empty((n,), torch.int32)
        gorder = dv.empty((n,), torch.int32)
        gstart = dv.empty((g ** 3 + 1,), torch.int32)
        N.check(L.mg_bin_f32(N.ptr(pos), n, g, N.ptr(gkey), N.ptr(gorder), N.ptr(gstart), N.ptr(ws), ws.numel(),
                             st), "bin")
        grec = dv.empty((n, 12), torch.float32)
        err = dv.zeros((1,), torch.int32)
        N.check(L.mg_activate(N.ptr(pos), N.ptr(q), N.ptr(s), N.ptr(lg), n, N.ptr(gorder), N.ptr(grec), N.ptr(err),
                              st), "activate")
        pkey = dv.empty((ns,), torch.int32)
        pinv = dv.empty((ns,), torch.int32)
        pstart = dv.empty((g ** 3 + 1,), torch.int32)
        prec = dv.empty((ns, 4), torch.float32)
        xout = dv.empty((ns, 3), torch.float64)
        N.check(L.mg_bin_points(N.ptr(c64), N.ptr(sid), b, t, N.ptr(off), N.ptr(dirs), N.ptr(rot), N.ptr(tt64), k, g,
                                N.ptr(pkey), N.ptr(pinv), N.ptr(pstart), N.ptr(prec), N.ptr(xout), N.ptr(ws),
                                ws.numel(), st), "bin_points")
        need_grad = any(ctx.needs_input_grad[:7])
        out4 = dv.empty((ns, 4), torch.float32)
        cnt = dv.empty((ns,), torch.int32)
        N.check(L.mg_forward(N.ptr(grec), n, N.ptr(gstart), g, r, N.ptr(prec), N.ptr(pkey), N.ptr(pstart), ns,
                             1 if need_grad else 0, N.ptr(out4), N.ptr(cnt), N.ptr(ws), ws.numel(), st), "forward")
        inten = dv.empty((b,), torch.float64)
        N.check(L.mg_forward_finish(N.ptr(out4), N.ptr(cnt), N.ptr(pinv), b, t, N.ptr(wts), N.ptr(inten), None, None,
                                    None, st), "forward_finish")
        if n and int(err.item()):
            raise DegenerateQuaternion("quaternion norm <= 1e-12")
        ctx.meta = (n, b, t, k, g, r)
        ctx.dtypes = (positions.dtype, quaternions.dtype, log_scales.dtype, logits.dtype, coords.dtype,
                      None if tq is None else tq.dtype, None if tt is None else tt.dtype)
        ctx.save_for_backward(q, s, lg, c64, sid, tq64, rot, gkey, gorder, gstart, grec, pinv, pstart, prec, out4)
        ctx.psf = (off, wts, dirs)
        return inten.to(positions.dtype)

    @staticmethod
    def backward(ctx, grad_i):
        L = N.lib()
        st = dv.sptr()
        n, b, t, k, g, r = ctx.meta
        q, s, lg, c64, sid, tq64, rot, gkey, gorder, gstart, grec, pinv, pstart, prec, out4 = ctx.saved_tensors
        off, wts, dirs = ctx.psf
        up = _f64(grad_i).reshape(-1)
        ns = b * t
        ws = dv.workspace(max(L.mg_backward_workspace_bytes(n, g), L.mg_transform_grads_workspace_bytes(k)),
                          "torch_render")
        prec = prec.clone()  # upstream goes into the point records' 4th lane
        d_pts = dv.empty((ns, 3), torch.float64)
        N.check(L.mg_backward_points(N.ptr(up), None, b, t, N.ptr(wts), N.ptr(pinv), N.ptr(out4), N.ptr(prec),
                                     N.ptr(d_pts), st), "backward_points")
        acc = dv.empty((n, 10), torch.float32)
        N.check(L.mg_backward(N.ptr(grec), N.ptr(gkey), N.ptr(gstart), n, g, r, N.ptr(prec), N.ptr(pstart), N.ptr(acc),
                              N.ptr(ws), ws.numel(), st), "backward")
        dp, dq, ds, dl = (dv.empty((n, 3), torch.float64), dv.empty((n, 4), torch.float64),
                          dv.empty((n, 3), torch.float64), dv.empty((n,), torch.float64))
        N.check(L.mg_backward_epilogue(N.ptr(acc), N.ptr(gorder), n, N.ptr(q), N.ptr(s), N.ptr(lg), N.ptr(dp),
                                       N.ptr(dq), N.ptr(ds), N.ptr(dl), st), "backward_epilogue")
        d_tq = d_tt = None
        if k and (ctx.needs_input_grad[5] or ctx.needs_input_grad[6]):
            scratch = dv.empty((k, 12), torch.float64)
            out7 = dv.empty((k, 7), torch.float64)
            N.check(L.mg_transform_grads(N.ptr(d_pts), N.ptr(c64), N.ptr(sid), b, t, N.ptr(off), N.ptr(dirs),
                                         N.ptr(tq64), k, N.ptr(scratch), N.ptr(out7), 0, N.ptr(ws), ws.numel(), st),
                    "transform_grads")
            d_tq, d_tt = out7[:, :4], out7[:, 4:]
        d_c = None
        if ctx.needs_input_grad[4]:
            h = d_pts.view(b, t, 3).sum(1)  # sum over taps: the tap offset does not depend on the coordinate
            if k:
                rs = rot[sid.clamp(min=0)]
                hr = torch.einsum("bij,bi->bj", rs, h)  # R^T h
                h = torch.where((sid >= 0)[:, None], hr, h)
            d_c = h
        dt = ctx.dtypes
        cast = (lambda x, d: None if x is None or d is None else x.to(d))
        return (cast(dp, dt[0]), cast(dq, dt[1]), cast(ds, dt[2]), cast(dl, dt[3]), cast(d_c, dt[4]),
                cast(d_tq, dt[5]), cast(d_tt, dt[6]), None, None, None, None)


def _get(obj, *names):
    for nm in names:
        if isinstance(obj, dict) and nm in obj:
            return obj[nm]
        if hasattr(obj, nm):
            return getattr(obj, nm)
    raise AttributeError(f"gaussians has none of {names}")


def render(gaussians, sample_coords, slice_psf=None, slice_ids=None, transforms=None, grid_resolution=None,
           radius=5):
    """Intensities I(x_b) (B,) of the Gaussian field at every sample, differentiable.

    gaussians: object or dict with ``positions`` (N,3), ``quaternions`` (N,4,
    w-first, unnormalised), ``log_scales`` (N,3) and ``intensity_logits`` (or
    ``logits``) (N,) tensors.  sample_coords: (B,3) normalised coordinates;
    slice_ids: (B,) int (< 0 = untransformed); transforms: ``(quats (K,4),
    translations (K,3))`` tensors or an object with ``quats`` / ``translations``;
    slice_psf: ``render.SlicePSF`` (through-plane taps) or None.
    grid_resolution defaults to the lattice side N^(1/3) when N is a cube.
    """
    pos = _get(gaussians, "positions")
    quat = _get(gaussians, "quaternions")
    ls = _get(gaussians, "log_scales")
    lg = _get(gaussians, "intensity_logits", "logits")
    n = pos.shape[0]
    if grid_resolution is None:
        side = int(round(n ** (1.0 / 3.0)))
        if side ** 3 != n:
            raise ValueError("grid_resolution is required when N is not a cube")
        grid_resolution = side
    tq = tt = None
    if transforms is not None:
        if isinstance(transforms, (tuple, list)):
            tq, tt = transforms
        else:
            tq, tt = transforms.quats, transforms.translations
        tq = torch.as_tensor(tq)
        tt = torch.as_tensor(tt)
        if tq.shape[0] == 0:
            tq = tt = None
    coords = torch.as_tensor(sample_coords)
    if coords.shape[0] == 0:
        return torch.zeros((0,), dtype=pos.dtype, device=coords.device)
    sids = None if slice_ids is None else torch.as_tensor(slice_ids)
    return _Render.apply(pos, quat, ls, lg, coords, tq, tt, sids, int(grid_resolution), int(radius), slice_psf)
