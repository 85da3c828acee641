"""On-disk formats of the reference, produced from (and read into) device state
(SURVEY §8(f) F4): the single-file little-endian NIfTI-1 volume
(/root/reference/pkg/src/mgauss/io.py:101-174) and the ``MGSS0001``
checkpoint container (io.py:177-258).  Files are byte-identical to the
reference writer's for the same content, so the reference CLI can ``--resume``
from a checkpoint written here, ``evaluate`` a volume written here, and vice
versa (tests/test_io_cpu.py compares against bytes written by the reference).

Writes are atomic (temporary file + fsync + rename), as in io.py:88-94.
"""

from __future__ import annotations

import json
import os

import numpy as np

from .core import Volume
from .errors import BadMagic, EndianMismatch, TruncatedPayload, UnsupportedDatatype

NIFTI_HEADER_SIZE = 348
NIFTI_MAGIC = b"n+1\x00"
CHECKPOINT_MAGIC = b"MGSS0001"
_VOX_OFFSET = 352  # header + 4-byte empty extension flag

# NIfTI-1 header (nifti1.h), little-endian
NIFTI_HEADER_DTYPE = np.dtype([
    ("sizeof_hdr", "<i4"), ("data_type", "S10"), ("db_name", "S18"), ("extents", "<i4"),
    ("session_error", "<i2"), ("regular", "S1"), ("dim_info", "u1"), ("dim", "<i2", (8,)),
    ("intent_p1", "<f4"), ("intent_p2", "<f4"), ("intent_p3", "<f4"), ("intent_code", "<i2"),
    ("datatype", "<i2"), ("bitpix", "<i2"), ("slice_start", "<i2"), ("pixdim", "<f4", (8,)),
    ("vox_offset", "<f4"), ("scl_slope", "<f4"), ("scl_inter", "<f4"), ("slice_end", "<i2"),
    ("slice_code", "u1"), ("xyzt_units", "u1"), ("cal_max", "<f4"), ("cal_min", "<f4"),
    ("slice_duration", "<f4"), ("toffset", "<f4"), ("glmax", "<i4"), ("glmin", "<i4"),
    ("descrip", "S80"), ("aux_file", "S24"), ("qform_code", "<i2"), ("sform_code", "<i2"),
    ("quatern_b", "<f4"), ("quatern_c", "<f4"), ("quatern_d", "<f4"),
    ("qoffset_x", "<f4"), ("qoffset_y", "<f4"), ("qoffset_z", "<f4"),
    ("srow_x", "<f4", (4,)), ("srow_y", "<f4", (4,)), ("srow_z", "<f4", (4,)),
    ("intent_name", "S16"), ("magic", "S4"),
])
assert NIFTI_HEADER_DTYPE.itemsize == NIFTI_HEADER_SIZE

_CODE_OF = {np.dtype("<f4"): 16, np.dtype("<u2"): 512}  # NIFTI_TYPE_FLOAT32, NIFTI_TYPE_UINT16
_DTYPE_OF = {v: k for k, v in _CODE_OF.items()}
_SIZEOF_HDR_SWAPPED = int.from_bytes(NIFTI_HEADER_SIZE.to_bytes(4, "little"), "big")


def atomic_write(path, payload: bytes):
    """Write ``payload`` to ``path`` through a synced temporary file and a rename."""
    tmp = f"{path}.tmp-{os.getpid()}"
    with open(tmp, "wb") as fh:
        fh.write(payload)
        fh.flush()
        os.fsync(fh.fileno())
    os.replace(tmp, path)


# ---------------------------------------------------------------------------
# NIfTI-1 volumes
# ---------------------------------------------------------------------------


def nifti_bytes(volume: Volume, descrip=""):
    """The NIfTI-1 file image of ``volume`` (io.py:101-145 semantics): float32
    and uint16 payloads pass through, other dtypes are cast to float32; the
    affine travels in srow (sform_code 1, qform unused); Fortran voxel order."""
    data = np.asarray(volume.data)
    if data.dtype not in (np.dtype(np.float32), np.dtype(np.uint16)):
        data = data.astype(np.float32)
    data = np.ascontiguousarray(data)
    if not np.all(np.isfinite(data.astype(np.float64))):
        raise ValueError("volume data must be finite")
    sp = np.asarray(volume.spacing, dtype=np.float64)
    org = np.asarray(volume.origin, dtype=np.float64)
    h = np.zeros((), dtype=NIFTI_HEADER_DTYPE)
    h["sizeof_hdr"] = NIFTI_HEADER_SIZE
    h["regular"] = b"r"
    h["dim"] = [3, *data.shape, 1, 1, 1, 1]
    h["datatype"] = _CODE_OF[data.dtype.newbyteorder("<")]
    h["bitpix"] = 8 * data.dtype.itemsize
    h["pixdim"] = [1.0, *sp, 0.0, 0.0, 0.0, 0.0]
    h["vox_offset"] = float(_VOX_OFFSET)
    h["scl_slope"] = 1.0
    h["xyzt_units"] = 2  # NIFTI_UNITS_MM
    h["descrip"] = descrip.encode()[:79]
    h["sform_code"] = 1
    h["srow_x"] = [sp[0], 0.0, 0.0, org[0]]
    h["srow_y"] = [0.0, sp[1], 0.0, org[1]]
    h["srow_z"] = [0.0, 0.0, sp[2], org[2]]
    h["magic"] = NIFTI_MAGIC
    return h.tobytes() + bytes(_VOX_OFFSET - NIFTI_HEADER_SIZE) + data.tobytes(order="F")


def write_volume(path, volume: Volume, descrip=""):
    """Write ``volume`` (e.g. ``Trainer.render_volume(...)``) as NIfTI-1."""
    atomic_write(path, nifti_bytes(volume, descrip))


def read_volume(path):
    """(Volume, descrip) from a little-endian float32/uint16 NIfTI-1 file (io.py:148-174)."""
    with open(path, "rb") as fh:
        raw = fh.read()
    if len(raw) < NIFTI_HEADER_SIZE:
        raise TruncatedPayload(f"file holds {len(raw)} bytes, header needs {NIFTI_HEADER_SIZE}")
    h = np.frombuffer(raw, dtype=NIFTI_HEADER_DTYPE, count=1)[0]
    if int(h["sizeof_hdr"]) == _SIZEOF_HDR_SWAPPED:
        raise EndianMismatch("big-endian NIfTI files are not supported")
    magic = bytes(h["magic"]).ljust(4, b"\x00")
    if magic != NIFTI_MAGIC or int(h["sizeof_hdr"]) != NIFTI_HEADER_SIZE:
        raise BadMagic(f"bad NIfTI magic/header: magic={magic!r}")
    code = int(h["datatype"])
    if code not in _DTYPE_OF:
        raise UnsupportedDatatype(f"NIfTI datatype code {code} not supported")
    if int(h["dim"][0]) != 3:
        raise UnsupportedDatatype(f"only 3D volumes supported, got dim[0]={int(h['dim'][0])}")
    dt = _DTYPE_OF[code]
    dims = tuple(int(d) for d in h["dim"][1:4])
    lo = int(h["vox_offset"])
    hi = lo + int(np.prod(dims)) * dt.itemsize
    if len(raw) < hi:
        raise TruncatedPayload(f"file holds {len(raw)} bytes, needs {hi}")
    data = np.frombuffer(raw[lo:hi], dtype=dt).reshape(dims, order="F").copy()
    spacing = np.array(h["pixdim"][1:4], dtype=np.float64)
    origin = np.array([h["srow_x"][3], h["srow_y"][3], h["srow_z"][3]], dtype=np.float64)
    return Volume(data=data, spacing=spacing, origin=origin), h["descrip"].decode(errors="replace")


# ---------------------------------------------------------------------------
# MGSS0001 checkpoint container: magic, u64 header length, JSON header
# {"tree": <state with arrays replaced by {"__array__": i}>, "arrays": [...]},
# then the arrays' little-endian bytes back to back.
# ---------------------------------------------------------------------------


def _flatten(obj, arrays):
    if isinstance(obj, np.ndarray):
        arrays.append(np.ascontiguousarray(obj))
        return {"__array__": len(arrays) - 1}
    if isinstance(obj, dict):
        return {k: _flatten(v, arrays) for k, v in obj.items()}
    if isinstance(obj, (list, tuple)):
        return [_flatten(v, arrays) for v in obj]
    if isinstance(obj, np.integer):
        return int(obj)
    if isinstance(obj, np.floating):
        return float(obj)
    return obj


def _inflate(obj, arrays):
    if isinstance(obj, dict):
        if len(obj) == 1 and "__array__" in obj:
            return arrays[obj["__array__"]]
        return {k: _inflate(v, arrays) for k, v in obj.items()}
    if isinstance(obj, list):
        return [_inflate(v, arrays) for v in obj]
    return obj


def checkpoint_bytes(state):
    """The MGSS0001 file image of a nested dict of scalars, lists and arrays."""
    arrays = []
    tree = _flatten(state, arrays)
    specs, blobs, off = [], [], 0
    for a in arrays:
        le = a.dtype.newbyteorder("<")
        blob = a.astype(le, copy=False).tobytes()
        specs.append({"dtype": le.str, "shape": list(a.shape), "offset": off, "nbytes": len(blob)})
        blobs.append(blob)
        off += len(blob)
    header = json.dumps({"tree": tree, "arrays": specs}).encode()
    return CHECKPOINT_MAGIC + len(header).to_bytes(8, "little") + header + b"".join(blobs)


def save_checkpoint(path, state):
    """Write ``state`` (e.g. ``{"trainer": Trainer.state_dict()}``, as cli.py:161-162 does)."""
    atomic_write(path, checkpoint_bytes(state))


def load_checkpoint(path):
    with open(path, "rb") as fh:
        raw = fh.read()
    if len(raw) < 16 or raw[:8] != CHECKPOINT_MAGIC:
        raise BadMagic(f"not a {CHECKPOINT_MAGIC.decode()} checkpoint")
    hlen = int.from_bytes(raw[8:16], "little")
    if len(raw) < 16 + hlen:
        raise TruncatedPayload("checkpoint header truncated")
    header = json.loads(raw[16:16 + hlen].decode())
    base = 16 + hlen
    arrays = []
    for spec in header["arrays"]:
        lo = base + spec["offset"]
        hi = lo + spec["nbytes"]
        if len(raw) < hi:
            raise TruncatedPayload("checkpoint payload truncated")
        arrays.append(np.frombuffer(raw[lo:hi], dtype=np.dtype(spec["dtype"])).reshape(spec["shape"]).copy())
    return _inflate(header["tree"], arrays)
