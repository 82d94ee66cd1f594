"""B200-native MPDATA step + slab decomposition + FPM partitioner.

The product is ``libimb_b200.so`` (sm_100a CUDA kernels, C++ runtime, C-ABI
``include/imb_mpdata.h``). This package is its Python host mirror; it loads
the library eagerly and raises if it is missing (no CPU fallback).
"""
from ._lib import (AlignmentError, ConfigError, ContractError, CudaError, DomainError,  # noqa: F401
                   ImbError, IncompatibleModelError, InfeasibleError, InsufficientDataError,
                   NcclError, ParseError, RangeError, TooLargeError, LIB_PATH, load)

load()

from . import fpm, mpdata  # noqa: E402,F401

__version__ = "0.1.0"
