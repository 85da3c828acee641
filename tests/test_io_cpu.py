"""F4 on-disk formats: NIfTI-1 volumes and the MGSS0001
checkpoint container must be byte-identical to what the reference writers
produce (tests/golden/io_*.{nii,mgss} were written by /root/reference's
mgauss.io, see make_golden.make_io_cases), and read back what they wrote."""

import os

import numpy as np
import pytest

from paper_2603_00145_b200 import io as mio
from paper_2603_00145_b200.core import Volume
from paper_2603_00145_b200.errors import BadMagic, EndianMismatch, TruncatedPayload, UnsupportedDatatype

from conftest import load_golden

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _raw(name):
    with open(os.path.join(GOLD, name), "rb") as fh:
        return fh.read()


@pytest.mark.parametrize("name,key,descrip", [("io_f32.nii", "v32", "golden f32"), ("io_u16.nii", "v16", "golden u16")])
def test_nifti_bytes_match_reference_writer(name, key, descrip):
    g = load_golden("io")
    vol = Volume(data=g[key], spacing=g["spacing"], origin=g["origin"])
    assert mio.nifti_bytes(vol, descrip) == _raw(name)


@pytest.mark.parametrize("name,key,descrip", [("io_f32.nii", "v32", "golden f32"), ("io_u16.nii", "v16", "golden u16")])
def test_nifti_reads_reference_file(name, key, descrip):
    g = load_golden("io")
    vol, d = mio.read_volume(os.path.join(GOLD, name))
    want = g[key].astype(np.float32) if key == "v32" else g[key]
    np.testing.assert_array_equal(vol.data, want)
    assert vol.data.dtype == want.dtype
    np.testing.assert_array_equal(vol.spacing, g["spacing"].astype(np.float32).astype(np.float64))
    np.testing.assert_array_equal(vol.origin, g["origin"].astype(np.float32).astype(np.float64))
    assert d == descrip


def test_nifti_write_is_atomic_and_round_trips(tmp_path):
    vol = Volume(data=np.arange(24, dtype=np.float64).reshape(2, 3, 4), spacing=np.array([1.0, 2.0, 3.0]),
                 origin=np.array([0.5, -0.5, 0.0]))
    p = tmp_path / "v.nii"
    mio.write_volume(p, vol, "x")
    assert sorted(os.listdir(tmp_path)) == ["v.nii"]  # no temp file left behind
    back, d = mio.read_volume(p)
    np.testing.assert_array_equal(back.data, vol.data.astype(np.float32))
    assert d == "x"


def test_nifti_errors(tmp_path):
    raw = bytearray(_raw("io_f32.nii"))
    p = tmp_path / "t.nii"
    p.write_bytes(bytes(raw[:100]))
    with pytest.raises(TruncatedPayload):
        mio.read_volume(p)
    p.write_bytes(bytes(raw[:-8]))
    with pytest.raises(TruncatedPayload):
        mio.read_volume(p)
    bad = bytearray(raw)
    bad[344:348] = b"ni1\x00"
    p.write_bytes(bytes(bad))
    with pytest.raises(BadMagic):
        mio.read_volume(p)
    swapped = bytearray(raw)
    swapped[0:4] = (348).to_bytes(4, "big")
    p.write_bytes(bytes(swapped))
    with pytest.raises(EndianMismatch):
        mio.read_volume(p)
    dt = bytearray(raw)
    dt[70:72] = (64).to_bytes(2, "little")  # float64 datatype code
    p.write_bytes(bytes(dt))
    with pytest.raises(UnsupportedDatatype):
        mio.read_volume(p)
    with pytest.raises(ValueError):
        mio.nifti_bytes(Volume(data=np.array([[[np.nan]]]), spacing=np.ones(3), origin=np.zeros(3)))


def test_checkpoint_round_trip_is_byte_identical_to_reference():
    raw = _raw("io_checkpoint.mgss")
    state = mio.load_checkpoint(os.path.join(GOLD, "io_checkpoint.mgss"))
    tr = state["trainer"]
    assert tr["iteration"] == 3 and tr["config"]["use_nrf"] is True
    assert set(tr["adam"]) >= {"positions", "quaternions", "log_scales", "intensity_logits", "transforms", "nrf"}
    assert tr["field"]["positions"].dtype == np.float64 and tr["field"]["lattice_index"].dtype == np.int64
    assert mio.checkpoint_bytes(state) == raw


def test_checkpoint_errors(tmp_path):
    raw = _raw("io_checkpoint.mgss")
    p = tmp_path / "c.mgss"
    p.write_bytes(b"XXXX0001" + raw[8:])
    with pytest.raises(BadMagic):
        mio.load_checkpoint(p)
    p.write_bytes(raw[:40])
    with pytest.raises(TruncatedPayload):
        mio.load_checkpoint(p)
    p.write_bytes(raw[:-16])
    with pytest.raises(TruncatedPayload):
        mio.load_checkpoint(p)
    state = {"a": np.arange(5, dtype=">i4"), "b": [1, 2.5, None, "s"], "c": {"d": np.float32(1.5), "e": np.int16(3)}}
    mio.save_checkpoint(tmp_path / "x.mgss", state)
    back = mio.load_checkpoint(tmp_path / "x.mgss")
    np.testing.assert_array_equal(back["a"], np.arange(5))
    assert back["a"].dtype == np.dtype("<i4") and back["b"] == [1, 2.5, None, "s"]
    assert back["c"] == {"d": 1.5, "e": 3}
