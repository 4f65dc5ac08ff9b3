"""DynaExq (arXiv 2511.15015) hybrid-precision MoE layer hot path, B200-native (sm_100a).

The product is the C-ABI library libdx.so (include/dx.h); `dx` is its thin ctypes binding.
"""
from . import dx  # noqa: F401  (raises ImportError when libdx.so is missing: no CPU fallback)
