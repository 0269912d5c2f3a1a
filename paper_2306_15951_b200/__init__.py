"""B200-native C-K-S zero-skipping convolution operators (arXiv 2306.15951).

ConvV2 (forward, filter trimming), KS-deconv-V2 (input gradient by kernel
split into stride^2 dense sub-filters) and Sk-dilated-V2 (weight gradient by
leaping access), as tcgen05/TMA kernels for sm_100a behind the C ABI of
libcks.so (include/cks.h).  ``_lib`` is the ctypes binding (same names as the
C entry points); ``ops`` the torch-tensor helpers; ``dist`` the batch-sharded
multi-GPU step.
"""
from ._lib import CKS_BF16, CKS_TF32, CksError, LIB_PATH  # noqa: F401

__all__ = ["CKS_BF16", "CKS_TF32", "CksError", "LIB_PATH"]
