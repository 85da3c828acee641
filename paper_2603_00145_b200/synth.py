"""Synthetic thick-slice acquisitions shaped like BASELINE.json's configs.

The reference's simulator (simdata.py) is not available on the GPU box, so
benchmarks use this self-contained generator with the same geometry
conventions: three orthogonal stacks (through axes x, y, z),
voxel-centre sample points, an isotropic world->[-1,1]^3 map whose longest
axis spans [-0.98, 0.98] (simdata.py:392-409), per-slice rigid motion
expressed in normalized units (simdata.py:452-473), and the Gaussian slab
profile of simdata.py:242-251 as the slice PSF.  Intensities come from an
analytic nested-ellipsoid phantom -- synthetic data, not the reference's.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .core import TransformSet, quat_to_rotation

FWHM_TO_SIGMA = 2.0 * np.sqrt(2.0 * np.log(2.0))
CONFIGS = {
    # name: (phantom_dims, phantom_spacing_mm, in_plane_mm, thickness_mm, lattice R, nrf, batch)
    "C1": (64, 1.0, 1.0, 4.0, 22, False, 65536),
    "C2": (160, 0.8, 0.8, 3.0, 46, False, 65536),
    "C3": (256, 1.0, 1.0, 4.0, 80, True, 65536),
    "C4": (256, 1.0, 1.0, 4.0, 100, False, 65536),
}


def slab_kernel(thickness, through_spacing):
    """(offsets_mm, weights): Gaussian with FWHM = thickness sampled at the source
    spacing, truncated at half the thickness (simdata.py:242-251)."""
    n_half = int(np.floor(thickness / 2.0 / through_spacing + 1e-9))
    off = np.arange(-n_half, n_half + 1) * through_spacing
    off = off[np.abs(off) <= thickness / 2.0 + 1e-9]
    sigma = thickness / FWHM_TO_SIGMA
    w = np.exp(-(off ** 2) / (2.0 * sigma ** 2))
    return off, w / w.sum()


def phantom(u):
    """Analytic phantom on normalized coordinates u (...,3) in [-1,1]: an outer
    ellipsoid with a ramp, a thin bright shell, two inner ellipsoids."""
    x, y, z = u[..., 0], u[..., 1], u[..., 2]
    rho = np.sqrt((x / 0.80) ** 2 + (y / 0.72) ** 2 + (z / 0.64) ** 2)
    v = np.where(rho < 1.0, 0.32 + 0.18 * (1.0 - rho), 0.0)
    shell = np.abs(np.sqrt(x * x + y * y + z * z) - 0.46) < 0.035
    v = np.where(shell & (rho < 1.0), 0.95, v)
    inner = ((x - 0.16) / 0.30) ** 2 + ((y + 0.10) / 0.26) ** 2 + ((z - 0.08) / 0.24) ** 2 < 1.0
    v = np.where(inner, 0.72 + 0.08 * np.sin(4.0 * np.pi * x) * np.cos(4.0 * np.pi * y), v)
    deep = ((x + 0.28) / 0.16) ** 2 + ((y - 0.20) / 0.18) ** 2 + ((z + 0.12) / 0.15) ** 2 < 1.0
    return np.where(deep, 0.55, v)


def _quat_from_euler(rx, ry, rz):
    def ax(axis, a):
        q = np.zeros(4)
        q[0] = np.cos(a / 2)
        q[1 + axis] = np.sin(a / 2)
        return q

    def mul(a, b):
        aw, ax_, ay, az = a
        bw, bx, by, bz = b
        return np.array([aw * bw - ax_ * bx - ay * by - az * bz, aw * bx + ax_ * bw + ay * bz - az * by,
                         aw * by - ax_ * bz + ay * bw + az * bx, aw * bz + ax_ * by - ay * bx + az * bw])

    return mul(ax(2, rz), mul(ax(1, ry), ax(0, rx)))


@dataclass
class SynthStacks:
    coords: np.ndarray  # (M, 3) normalized, pre-transform
    intensities: np.ndarray  # (M,)
    slice_ids: np.ndarray  # (M,) int64
    transforms: TransformSet  # (K) normalized rigid transforms
    through_dirs: np.ndarray  # (K, 3) unit through-plane vectors
    slice_shape: tuple  # (H, W) of every slice
    slice_offsets: np.ndarray  # (K+1,) start of each slice's points in coords (C-ordered H*W)
    psf_offsets: np.ndarray  # (T,) normalized through-plane tap offsets
    psf_weights: np.ndarray  # (T,)
    scale: float  # world mm -> normalized

    @property
    def num_slices(self):
        return len(self.transforms)

    def slice_grid(self, k):
        a, b = self.slice_offsets[k], self.slice_offsets[k + 1]
        return self.coords[a:b], self.intensities[a:b].reshape(self.slice_shape)


def make_stacks(dims=64, spacing=1.0, in_plane=1.0, thickness=4.0, motion_sigma=0.5, noise_sigma=0.01, seed=7):
    """Three orthogonal stacks of a cubic dims^3 phantom at `spacing` mm."""
    rng = np.random.default_rng(seed)
    extent = dims * spacing
    n_sl = int(np.floor(extent / thickness + 1e-9))
    n_ip = int(np.floor(extent / in_plane + 1e-9))
    ip_c = (np.arange(n_ip) + 0.5) * in_plane  # world mm, origin at volume corner
    th_c = (np.arange(n_sl) + 0.5) * thickness
    lo = min(ip_c[0], th_c[0])
    hi = max(ip_c[-1], th_c[-1])
    center = 0.5 * (lo + hi)
    scale = 2.0 * 0.98 / (hi - lo)
    off_mm, w = slab_kernel(thickness, spacing)
    coords, inten, sids, quats, trans, dirs, starts = [], [], [], [], [], [], [0]
    ga, gb = np.meshgrid(ip_c, ip_c, indexing="ij")
    sid = 0
    for through in range(3):
        inplane = [a for a in range(3) if a != through]
        for m in range(n_sl):
            pts = np.empty((n_ip, n_ip, 3))
            pts[..., inplane[0]] = ga
            pts[..., inplane[1]] = gb
            pts[..., through] = th_c[m]
            u = ((pts - center) * scale).reshape(-1, 3)
            ang = np.deg2rad(rng.normal(0.0, motion_sigma, 3))
            q = _quat_from_euler(*ang)
            t_n = scale * rng.normal(0.0, motion_sigma, 3)
            rot = quat_to_rotation(q)
            # slab-integrated observation of the moved slice (PSF applied before motion)
            val = np.zeros(u.shape[0])
            for o, ww in zip(off_mm, w):
                p = u.copy()
                p[:, through] += o * scale
                val += ww * phantom(p @ rot.T + t_n)
            val += rng.normal(0.0, noise_sigma, val.shape)
            coords.append(u)
            inten.append(val)
            sids.append(np.full(u.shape[0], sid, np.int64))
            quats.append(q)
            trans.append(t_n)
            d = np.zeros(3)
            d[through] = 1.0
            dirs.append(d)
            starts.append(starts[-1] + u.shape[0])
            sid += 1
    inten = np.concatenate(inten)
    inten = np.clip(inten / inten.max(), 0.0, 1.0)
    return SynthStacks(coords=np.concatenate(coords), intensities=inten, slice_ids=np.concatenate(sids),
                       transforms=TransformSet(np.array(quats), np.array(trans)), through_dirs=np.array(dirs),
                       slice_shape=(n_ip, n_ip), slice_offsets=np.array(starts), psf_offsets=off_mm * scale,
                       psf_weights=w, scale=scale)


def make_config(name, seed=7):
    dims, sp, ip, th, _, _, _ = CONFIGS[name]
    return make_stacks(dims, sp, ip, th, seed=seed)
