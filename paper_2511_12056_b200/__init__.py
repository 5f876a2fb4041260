"""paper_2511_12056_b200 -- B200-native PipeSP sequence-parallel attention (PipeDiT, arXiv 2511.12056).

The product is libspa.so (C ABI in include/spa.h, CUDA kernels for sm_100a in csrc/);
`spa` is its thin ctypes binding.  No CPU fallback: the calls raise if the library is
missing or the GPU path fails.
"""
from . import spa  # noqa: F401
from .spa import (Comm, Plan, SpaError, attention, get_unique_id, load)  # noqa: F401

__version__ = "0.1.0"
