"""B200-native (sm_100a) NNPS hot path of "A GPU accelerated mixed-precision SPH
framework with cell-based relative coordinates" (arXiv 2401.08586).

Cell-linked list (CLL), relative-coordinate link list (RCLL) and all-list
neighbour searches at FP64/FP32/FP16, bit-exact with the reference sphx CPU
implementation, behind the C ABI in include/sphx_cuda.h (lib/libsphx_cuda.so).
The C++ drop-in (include/sphx/*.hpp, module `_core`) sits on the same ABI.
"""
from .capi import (FP16, FP32, FP64, PRECISIONS, Context, GridDesc, SphxCudaError,  # noqa: F401
                   build_lattice, build_random_uniform, grid_init, lib)

__all__ = ["FP16", "FP32", "FP64", "PRECISIONS", "Context", "GridDesc", "SphxCudaError",
           "grid_init", "lib", "build_lattice", "build_random_uniform"]
