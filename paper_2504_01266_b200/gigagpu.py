"""The paper's API object, on top of the C ABI (PAPER.md S4.2.2).

GigaAPI exposes a ``GigaGPU`` object whose methods run the data-parallel operations over the
GPUs of one machine: ``performMatrixMultiplication()``, ``computeDotProduct()`` and
``computeL2Norm()``. This class keeps those names; every call goes straight to
libgiga (``giga_matmul``, ``giga_dot``, ``giga_l2norm``): argument handling only.

    with GigaGPU() as gpu:                       # all visible GPUs (the paper: two)
        C = gpu.performMatrixMultiplication(A, B)   # numpy fp32 in, numpy fp32 out
        d = gpu.computeDotProduct(x, y)
        n = gpu.computeL2Norm(x)
"""
from __future__ import annotations

import numpy as np

from . import giga


class GigaGPU:
    def __init__(self, ngpus: int = 0):
        """Claim GPUs 0..ngpus-1 (0: every visible GPU; PAPER.md:311 fixed two)."""
        giga.init(ngpus)
        self.ngpus = giga.num_devices()
        self._open = True

    # -- S4.2.7, P:285-291 ------------------------------------------------------------------
    def performMatrixMultiplication(self, A, B, C=None, ngpus: int | None = None):
        """C = A @ B over the GPUs: row blocks of A per GPU, B to every GPU, C gathered.
        Host numpy / torch CPU arrays (fp32, C-contiguous) or device tensors on GPU 0."""
        M, K = A.shape
        K2, N = B.shape
        if K != K2:
            raise ValueError(f"shape mismatch {tuple(A.shape)} x {tuple(B.shape)}")
        if C is None:
            if isinstance(A, np.ndarray):
                C = np.empty((M, N), np.float32)
            else:
                import torch
                C = torch.empty((M, N), dtype=torch.float32, device=A.device)
        giga.matmul(A, B, C, M, N, K, self.ngpus if ngpus is None else ngpus)
        return C

    # -- S4.2.8, P:299-303 ------------------------------------------------------------------
    def computeDotProduct(self, x, y, ngpus: int | None = None) -> float:
        n = x.size if isinstance(x, np.ndarray) else x.numel()
        return giga.dot(x, y, n, self.ngpus if ngpus is None else ngpus)

    def computeL2Norm(self, x, ngpus: int | None = None) -> float:
        n = x.size if isinstance(x, np.ndarray) else x.numel()
        return giga.l2norm(x, n, self.ngpus if ngpus is None else ngpus)

    # -- lifetime: "construction/destruction releases all device memory" --------
    def close(self):
        if self._open:
            giga.finalize()
            self._open = False

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
