"""CPU-side checks of the C ABI: the sm_100a library builds, loads, and
exports every symbol include/mgauss_b200.h declares (no compute without a GPU)."""

import os
import re

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "mgauss_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(mg_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for must in ("mg_block_forward", "mg_block_backward", "mg_bin_f32", "mg_forward", "mg_backward",
                 "mg_sample_volume", "mg_gauss_update"):
        assert must in syms


def test_library_exports_every_declared_symbol():
    from paper_2603_00145_b200 import _build, _native

    _build.build()
    lib = _native.load_library()
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    # and the ctypes table covers exactly the declared ABI
    assert set(_native.SIGNATURES) == set(declared_symbols())
    assert lib.mg_abi_version() == _native.ABI_VERSION == 4


def test_library_is_sm100a():
    import subprocess

    from paper_2603_00145_b200 import _build

    path = _build.build()
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2603_00145_b200 import NativeLibraryMissing
    from paper_2603_00145_b200.spatial import build

    with pytest.raises(NativeLibraryMissing):
        build([[0.0, 0.0, 0.0]], 4)
