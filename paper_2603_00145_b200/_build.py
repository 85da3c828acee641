"""Build the sm_100a shared library in-tree (nvcc, no JIT cache).

    python -m paper_2603_00145_b200._build
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT_DIR = os.path.join(HERE, "_lib")
LIB = os.path.join(OUT_DIR, "libmgauss_b200.so")
SOURCES = ["mg_sort.cu", "mg_render.cu", "mg_train.cu", "mg_volume.cu", "mg_ssim.cu", "mg_nrf.cu", "mg_strict.cu", "mg_nrf_tc.cu", "mg_nrf64.cu", "mg_capi.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off",
    "-diag-suppress", "550",
    "-shared",
]


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "mgauss_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force=False, verbose=False, out=None, defines=()):
    out = out or LIB
    if not force and out == LIB and not needs_build():
        return LIB
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cmd = [NVCC, *FLAGS, *[f"-D{d}" for d in defines], "-o", out + ".tmp",
           *[os.path.join(CSRC, s) for s in SOURCES]]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True, cwd=CSRC)
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
