# SPDX-License-Identifier: Apache-2.0
"""B200-native block-distributed GEMM path of dMath (arxiv 1611.07819).

The product is libgridmath_b200.so (C++ host runtime + sm_100a CUDA kernels,
C ABI in include/gridmath_b200.h); this package only binds it.
"""
from . import _lib  # noqa: F401
from .gridmath import *  # noqa: F401,F403
