"""B200-native (sm_100a) M-Gaussian volumetric rendering hot path.

Drop-in host API mirroring /root/reference/pkg/src/mgauss (render, spatial,
train); pair loops, binning, epilogues and the optimizer run in the CUDA
kernels under csrc/, reached through the C ABI in include/mgauss_b200.h.
"""

from .errors import (DegenerateQuaternion, InconsistentGrid, MGaussError, NativeLibraryMissing,  # noqa: F401
                     NonFiniteLoss, OutOfMemoryRequest, ShrinkNotAllowed)

__version__ = "0.1.0"
