"""B200-native (sm_100a) wire-scan depth reconstruction (DAXM), arXiv:2201.13309.

The product path is libdaxm.so (include/daxm.h); this package is a thin ctypes
binding with the same names.  Every step of the reconstruction runs in the
library's CUDA kernels -- there is no CPU fallback: if libdaxm.so is missing or
no CUDA device is present, the calls raise.
"""
from .binding import (DaxmError, Plan, abi_version, create, lib, reconstruct, reconstruct_host,  # noqa: F401
                      EDGE, PIXEL_MODEL, DTYPE)

__all__ = ["DaxmError", "Plan", "create", "reconstruct", "reconstruct_host", "abi_version", "lib"]
