"""ctypes binding of the C ABI in include/mgauss_b200.h.

The product path has no fallback: if the sm_100a library is absent or no
CUDA device is visible, every call raises NativeLibraryMissing.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import NativeLibraryMissing

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MGAUSS_B200_LIB") or os.path.join(_HERE, "_lib", "libmgauss_b200.so")

P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int32
SZ = ctypes.c_size_t
D = ctypes.c_double

# name -> (restype, argtypes); mirrors include/mgauss_b200.h
SIGNATURES = {
    "mg_abi_version": (ctypes.c_int, []),
    "mg_last_error": (ctypes.c_char_p, []),
    "mg_device_sm_count": (ctypes.c_int, []),
    "mg_launch_count": (ctypes.c_longlong, []),
    "mg_cell_keys_f64": (ctypes.c_int, [P, I64, I64, P, P]),
    "mg_bin_workspace_bytes": (SZ, [I64, I64]),
    "mg_bin_f32": (ctypes.c_int, [P, I64, I64, P, P, P, P, SZ, P]),
    "mg_bin_f64": (ctypes.c_int, [P, I64, I64, P, P, P, P, SZ, P]),
    "mg_i32_to_i64": (ctypes.c_int, [P, I64, P, P]),
    "mg_i64_to_i32": (ctypes.c_int, [P, I64, P, P]),
    "mg_keys_from_csr": (ctypes.c_int, [P, I64, P, P]),
    "mg_scan_workspace_bytes": (SZ, [I64]),
    "mg_excl_scan_i32": (ctypes.c_int, [P, P, I64, P, SZ, P]),
    "mg_activate": (ctypes.c_int, [P, P, P, P, I64, P, P, P, P]),
    "mg_activate_f64": (ctypes.c_int, [P, P, P, I64, P, P, P, P, P, P, P]),
    "mg_points_workspace_bytes": (SZ, [I64, I64]),
    "mg_bin_points": (ctypes.c_int, [P, P, I64, I32, P, P, P, P, I64, I64, P, P, P, P, P, P, SZ, P]),
    "mg_forward_workspace_bytes": (SZ, [I64]),
    "mg_forward": (ctypes.c_int, [P, I64, P, I64, I64, P, P, P, I64, I32, P, P, P, SZ, P]),
    "mg_forward_finish": (ctypes.c_int, [P, P, P, I64, I32, P, P, P, P, P, P]),
    "mg_backward_points": (ctypes.c_int, [P, P, I64, I32, P, P, P, P, P, P]),
    "mg_backward_workspace_bytes": (SZ, [I64, I64]),
    "mg_backward": (ctypes.c_int, [P, P, P, I64, I64, I64, P, P, P, P, SZ, P]),
    "mg_backward_epilogue": (ctypes.c_int, [P, P, I64, P, P, P, P, P, P, P, P]),
    "mg_backward_accumulators": (ctypes.c_int, [P, P, I64, P, P, P, P, P]),
    "mg_epilogue_f64": (ctypes.c_int, [P, P, P, P, P, P, I64, P, P, P, P, P]),
    "mg_pack_records": (ctypes.c_int, [P, P, P, P, I64, P, P]),
    "mg_transform_grads_workspace_bytes": (SZ, [I64]),
    "mg_transform_grads": (ctypes.c_int, [P, P, P, I64, I32, P, P, P, I64, P, P, I32, P, SZ, P]),
    "mg_volume_workspace_bytes": (SZ, [I64, I64, I64]),
    "mg_sample_volume": (ctypes.c_int, [P, I64, P, I64, I64, I64, I64, I64, P, P, I64, I64, P, P, P, SZ, P]),
    "mg_smooth_l1": (ctypes.c_int, [P, P, I64, P, P, P]),
    "mg_smooth_l1_scaled": (ctypes.c_int, [P, P, I64, D, P, P, P]),
    "mg_aniso_loss_grad_f64": (ctypes.c_int, [P, I64, D, P, P, P]),
    "mg_adam_f64": (ctypes.c_int, [P, P, P, P, I64, I64, D, D, D, D, P]),
    "mg_nrf_forward": (ctypes.c_int, [P, I64, P, P, P, P, P, P, P]),
    "mg_nrf_backward_workspace_bytes": (SZ, [I64]),
    "mg_nrf_backward": (ctypes.c_int, [P, I64, P, P, P, P, P, P, P, P, P, SZ, P]),
    "mg_nrf_adam": (ctypes.c_int, [P, P, P, P, P, I32, P, D, D, D, D, P]),
    "mg_ssim_workspace_bytes": (SZ, [I64, I64]),
    "mg_ssim_loss_grad": (ctypes.c_int, [P, P, I64, I64, D, P, P, P, SZ, P]),
    "mg_quat_to_rot_f64": (ctypes.c_int, [P, I64, P, P]),
    "mg_counter_incr": (ctypes.c_int, [P, I32, P]),
    "mg_gather_batch": (ctypes.c_int, [P, I64, P, P, P, P, P, P, P]),
    "mg_gauss_update": (ctypes.c_int, [P, P, I64, P, P, P, P, P, P, P, I32, P, P, P]),
    "mg_gauss_update_inv": (ctypes.c_int, [P, P, I64, P, P, P, P, P, P, P, I32, P, P, P]),
    "mg_invert_permutation": (ctypes.c_int, [P, I64, P, P]),
    "mg_transform_adam": (ctypes.c_int, [P, P, P, P, P, I64, D, D, D, D, P, P]),
    "mg_upsample": (ctypes.c_int, [P, P, P, P, I64, I64, P, P, P, P, P]),
    "mg_smooth_l1_f64": (ctypes.c_int, [P, P, I64, P, P, P]),
    "mg_ssim_loss_grad_f64": (ctypes.c_int, [P, P, I64, I64, D, P, P, P, SZ, P]),
    "mg_upsample_f64": (ctypes.c_int, [P, P, P, P, I64, I64, P, P, P, P, P]),
    "mg_nrf_f64_workspace_bytes": (SZ, [I64]),
    "mg_nrf_forward_f64": (ctypes.c_int, [P, I64, P, P, P, I32, I32, D, P, P, SZ, P]),
    "mg_nrf_backward_f64": (ctypes.c_int, [P, I64, P, P, P, I32, I32, D, P, P, P, P, P, SZ, P]),
    "mg_block_workspace_bytes": (SZ, [I64, I64, I64]),
    "mg_block_forward": (ctypes.c_int, [P, P, I64, P, P, I64, P, P, P, I64, P, P, I64, I64, P, P, P, P, SZ, P]),
    "mg_block_backward": (ctypes.c_int,
                          [P, P, I64, P, P, I64, P, P, P, I64, P, P, I64, I64, P, P, P, P, P, P, SZ, P]),
    "mg_tc_selftest": (ctypes.c_int, [P, P, P, I32, P]),
    "mg_block_f64_workspace_bytes": (SZ, [I64, I64, I64]),
    "mg_block_forward_f64": (ctypes.c_int, [P, P, I64, P, P, I64, P, P, P, I64, P, P, I64, I64, P, P, P, P, SZ, P]),
    "mg_block_backward_f64": (ctypes.c_int,
                              [P, P, I64, P, P, I64, P, P, P, I64, P, P, I64, I64, P, P, P, P, P, P, SZ, P]),
    "mg_dense_workspace_bytes": (SZ, [I64]),
    "mg_dense_forward": (ctypes.c_int, [P, I64, P, P, P, I64, P, P, SZ, P]),
}

_lib = None
_lock = threading.Lock()


ABI_VERSION = 4  # include/mgauss_b200.h MG_ABI_VERSION


def load_library(path=LIB_PATH):
    """dlopen the library and bind every symbol (no CUDA call is made); a
    library built from an older header is rejected, not silently mis-called."""
    if not os.path.exists(path):
        raise NativeLibraryMissing(
            f"{path} is not built; run `python -m paper_2603_00145_b200._build` (nvcc, sm_100a)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.mg_abi_version() != ABI_VERSION:
        raise NativeLibraryMissing(f"{path} has ABI {lib.mg_abi_version()}, expected {ABI_VERSION}: rebuild it")
    return lib


def lib():
    """The bound library; requires a CUDA device (no CPU fallback)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                import torch

                if not torch.cuda.is_available():
                    raise NativeLibraryMissing("no CUDA device: the B200 path has no CPU fallback")
                _lib = load_library()
    return _lib


class NativeError(RuntimeError):
    pass


def check(rc, what=""):
    if rc != 0:
        msg = lib().mg_last_error().decode(errors="replace")
        raise NativeError(f"{what or 'mgauss_b200'} failed ({rc}): {msg}")


def ptr(t):
    """Device pointer of a torch tensor (or None -> NULL)."""
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def stream_ptr(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)
