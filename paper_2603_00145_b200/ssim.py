"""Windowed SSIM loss with its analytic gradient on the device -- the 2-D
training path of /root/reference/pkg/src/mgauss/ssim.py:21-122 (11-tap
Gaussian window, sigma 1.5, valid windows, C1 = 0.01^2, C2 = 0.03^2), same
names and errors.  Every function runs the four float64 separable passes of
csrc/mg_ssim.cu on float64 inputs (mg_ssim_loss_grad_f64).  The 3-D form
of ssim_mean is the reconstruction metric (metrics.py), outside the hot path.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _device as dv
from . import _native as N
from .errors import ShapeMismatch, SliceTooSmall

WINDOW_SIZE = 11
WINDOW_SIGMA = 1.5
C1 = 0.01 ** 2
C2 = 0.03 ** 2


def gaussian_window(size=WINDOW_SIZE, sigma=WINDOW_SIGMA):
    """Normalised 1-D Gaussian taps (ssim.py:21-25); the kernels hold the
    default window as constants."""
    offsets = np.arange(size, dtype=np.float64) - (size - 1) / 2.0
    w = np.exp(-(offsets ** 2) / (2.0 * sigma ** 2))
    return w / w.sum()


def _check_pair(a, b):
    if a.shape != b.shape:
        raise ShapeMismatch(f"shapes {a.shape} and {b.shape} differ")
    if min(a.shape) < WINDOW_SIZE:
        raise SliceTooSmall(f"min side {min(a.shape)} < window {WINDOW_SIZE}")


def _device_loss_grad(pred, target, window):
    pred = np.asarray(pred, dtype=np.float64)
    target = np.asarray(target, dtype=np.float64)
    _check_pair(pred, target)
    if pred.ndim != 2:
        raise ValueError("the device SSIM is the 2-D slice loss; the 3-D volume metric is outside the hot path")
    if window is not None and not np.array_equal(np.asarray(window, np.float64), gaussian_window()):
        raise ValueError("the device SSIM uses the default 11-tap sigma-1.5 window")
    h, w = pred.shape
    p = dv.to_dev(pred.ravel(), torch.float64)
    t = dv.to_dev(target.ravel(), torch.float64)
    up = dv.empty(p.shape, torch.float64)
    acc = dv.zeros((1,), torch.float64)
    ws = dv.empty((N.lib().mg_ssim_workspace_bytes(h, w),), torch.uint8)
    N.check(N.lib().mg_ssim_loss_grad_f64(N.ptr(p), N.ptr(t), h, w, 1.0, N.ptr(up), N.ptr(acc), N.ptr(ws), ws.numel(),
                                          dv.sptr()), "ssim")
    mean = float(acc.item()) / ((h - WINDOW_SIZE + 1) * (w - WINDOW_SIZE + 1))
    return mean, dv.to_host(up).reshape(h, w)


def ssim_mean(pred, target, window=None):
    """Mean SSIM over all valid windows (ssim.py:59-74), 2-D."""
    return _device_loss_grad(pred, target, window)[0]


def ssim_loss(pred, target):
    """1 - mean SSIM (ssim.py:77-79)."""
    return 1.0 - ssim_mean(pred, target)


def ssim_loss_grad(pred, target, window=None):
    """(loss, dloss/dpred) for 2-D slices (ssim.py:82-122)."""
    mean, grad = _device_loss_grad(pred, target, window)
    return 1.0 - mean, grad
