"""B200-native ReAttention hot path (arXiv 2407.15176): position-agnostic top-k
selection + finite-scope attention as sm_100a CUDA kernels behind a C-ABI
(include/reattn_cuda.h), with the reference's C++ API re-created in include/reattn/.

`native` is the ctypes binding used by tests and bench.py."""
from . import native  # noqa: F401

__all__ = ["native"]
