"""xmoe: B200-native (sm_100a) MoE-block hot path of X-MoE (arXiv 2508.13337).

The product is libxmoe.so (CUDA kernels + C-ABI, include/xmoe/xmoe.h) with its
C++ host orchestration; `capi` is a thin ctypes binding used by the tests and
the bench driver."""
__all__ = ["capi", "build"]
