"""B200-native GigaAPI matrix multiply (arXiv 2504.01266): row-split, fp32-accurate GEMM.

The product is ``libgiga.so`` (sm_100a kernels + the C ABI of ``include/giga.h``);
``paper_2504_01266_b200.giga`` is its ctypes binding. Importing ``giga`` raises if
``libgiga.so`` is missing (there is no fallback path); ``paper_2504_01266_b200.build`` builds
it and must stay importable without it.
"""


def __getattr__(name):
    if name == "GigaError":
        from .giga import GigaError
        return GigaError
    raise AttributeError(name)
