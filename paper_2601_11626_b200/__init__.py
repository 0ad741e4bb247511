"""B200-native (sm_100a) merge-error evaluation for compression-aware matrix
clustering (arXiv 2601.11626).  The product is libcmsvd.so (C ABI in
include/cmsvd.h, CUDA kernels in csrc/); ``cmsvd`` is its thin ctypes
binding.  There is no CPU fallback."""
from .cmsvd import (Context, CmsvdError, load, ALL, WEYL, RESIDUAL, INCREMENTAL, RAW, TRUNC,  # noqa: F401
                    ALG_MAX_NORM, ALG_RESIDUAL, ALG_APPROX, SORT_FROBENIUS, SORT_RESIDUAL, HOST, DEVICE, EXPORTS)
