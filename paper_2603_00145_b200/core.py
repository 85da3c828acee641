"""Host container types and small host math, mirroring the reference's
domain types (/root/reference/pkg/src/mgauss/core.py) so the drop-in API
reads the same: GaussianField, TransformSet, Volume, RigidTransform.

Arrays are numpy float64 on the host (the reference convention).  The
device-resident training state lives in ``paper_2603_00145_b200.train``.
"""

from __future__ import annotations

from dataclasses import dataclass, field as dc_field

import numpy as np

from .errors import DegenerateQuaternion

QUAT_NORM_EPS = 1e-12  # core.py:16
LOG_SCALE_LIMIT = 20.0  # core.py:17
PARAMS_PER_PRIMITIVE = 11  # core.py:18


def normalize_quat(q):
    """q / ||q|| (w-first); DegenerateQuaternion at ||q|| <= 1e-12 (core.py:36-45)."""
    q = np.asarray(q, dtype=np.float64)
    norm = np.linalg.norm(q, axis=-1, keepdims=True)
    if np.any(norm <= QUAT_NORM_EPS):
        raise DegenerateQuaternion(f"quaternion norm {norm.min():g} <= {QUAT_NORM_EPS:g}")
    return q / norm


def quat_to_rotation(q):
    """Rotation matrices of w-first quaternions (core.py:48-67); host math for
    the K per-slice transforms (tiny), the device does the per-Gaussian ones."""
    qn = normalize_quat(q)
    single = qn.ndim == 1
    qn = np.atleast_2d(qn)
    w, x, y, z = qn.T
    rot = np.empty((qn.shape[0], 3, 3))
    rot[:, 0] = np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], 1)
    rot[:, 1] = np.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], 1)
    rot[:, 2] = np.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], 1)
    return rot[0] if single else rot


def sigmoid(x):
    x = np.asarray(x, dtype=np.float64)
    with np.errstate(over="ignore"):
        return 1.0 / (1.0 + np.exp(-x))


def logit(p):
    p = np.asarray(p, dtype=np.float64)
    return np.log(p) - np.log1p(-p)


@dataclass
class RigidTransform:
    """Per-slice rigid map x -> R(q/||q||) x + t (core.py:138-152)."""

    rotation_quat: np.ndarray
    translation: np.ndarray
    slice_id: int = -1


@dataclass
class TransformSet:
    """Structure-of-arrays per-slice rigid transforms (core.py:182-214)."""

    quats: np.ndarray  # (K, 4) w-first, unnormalized
    translations: np.ndarray  # (K, 3)

    @classmethod
    def identity(cls, count):
        q = np.zeros((count, 4))
        q[:, 0] = 1.0
        return cls(quats=q, translations=np.zeros((count, 3)))

    @classmethod
    def from_list(cls, transforms):
        return cls(quats=np.stack([np.asarray(t.rotation_quat, dtype=np.float64) for t in transforms]),
                   translations=np.stack([np.asarray(t.translation, dtype=np.float64)
                                          for t in transforms]))

    def to_list(self):
        return [RigidTransform(self.quats[k].copy(), self.translations[k].copy(), slice_id=k)
                for k in range(len(self))]

    def rotations(self):
        return quat_to_rotation(self.quats)

    def copy(self):
        return TransformSet(self.quats.copy(), self.translations.copy())

    def __len__(self):
        return self.quats.shape[0]


@dataclass
class Volume:
    """Dense scalar volume (core.py:217-247); voxel (i,j,k) at origin + (i,j,k)*spacing."""

    data: np.ndarray
    spacing: np.ndarray = dc_field(default_factory=lambda: np.ones(3))
    origin: np.ndarray = dc_field(default_factory=lambda: np.zeros(3))
    orientation: str = "RAS"

    @property
    def dims(self):
        return tuple(self.data.shape)


@dataclass
class GaussianField:
    """N Gaussian primitives, 11 learnable parameters each (core.py:250-301)."""

    positions: np.ndarray  # (N, 3)
    quaternions: np.ndarray  # (N, 4) w-first, unnormalized
    log_scales: np.ndarray  # (N, 3)
    intensity_logits: np.ndarray  # (N,)
    lattice_dims: tuple = (0, 0, 0)
    lattice_index: np.ndarray | None = None

    @property
    def count(self):
        return int(np.asarray(self.positions).shape[0])

    @property
    def alphas(self):
        return sigmoid(self.intensity_logits)

    @property
    def params_per_primitive(self):
        return 11  # core.py:18

    def validate(self):
        """Shape checks of core.py:287-301 (N = prod(lattice_dims))."""
        n = self.count
        if n != int(np.prod(self.lattice_dims)):
            raise ValueError("primitive count does not match lattice dims")
        li = self.lattice_index if self.lattice_index is not None else np.zeros((0, 3))
        for arr, shape in ((self.positions, (n, 3)), (self.quaternions, (n, 4)), (self.log_scales, (n, 3)),
                           (self.intensity_logits, (n,)), (li, (n, 3))):
            if np.asarray(arr).shape != shape:
                raise ValueError(f"bad array shape {np.asarray(arr).shape}, expected {shape}")
        return self

    def copy(self):
        return GaussianField(np.array(self.positions), np.array(self.quaternions),
                             np.array(self.log_scales), np.array(self.intensity_logits),
                             tuple(self.lattice_dims),
                             None if self.lattice_index is None else np.array(self.lattice_index))


def lattice_node_positions(resolution):
    """Node centres of an R^3 lattice over [-1,1]^3, C-ordered (core.py:304-309)."""
    r = int(resolution)
    axis = -1.0 + (np.arange(r) + 0.5) * (2.0 / r)
    gx, gy, gz = np.meshgrid(axis, axis, axis, indexing="ij")
    return np.stack([gx.ravel(), gy.ravel(), gz.ravel()], axis=1)


def lattice_node_index(resolution):
    r = int(resolution)
    ii, jj, kk = np.meshgrid(np.arange(r), np.arange(r), np.arange(r), indexing="ij")
    return np.stack([ii.ravel(), jj.ravel(), kk.ravel()], axis=1).astype(np.int64)


def uniform_lattice_field(resolution, intensity_logits=None):
    """Fresh R^3 lattice field: identity quats, log-scale log(1/R) (core.py:318-342)."""
    r = int(resolution)
    n = r ** 3
    q = np.zeros((n, 4))
    q[:, 0] = 1.0
    lg = np.zeros(n) if intensity_logits is None else np.asarray(
        intensity_logits, dtype=np.float64).reshape(n).copy()
    return GaussianField(lattice_node_positions(r), q, np.full((n, 3), np.log(1.0 / r)), lg,
                         (r, r, r), lattice_node_index(r))
