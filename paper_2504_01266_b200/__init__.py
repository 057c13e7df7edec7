"""B200-native GigaAPI matrix multiply (arXiv 2504.01266): row-split, fp32-accurate GEMM.

The product is ``libgiga.so`` (sm_100a kernels + the C ABI of ``include/giga.h``);
``paper_2504_01266_b200.giga`` is its ctypes binding.
"""
from . import giga  # noqa: F401  (raises if libgiga.so is missing: no fallback path)
from .giga import GigaError  # noqa: F401
