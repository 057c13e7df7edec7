"""CPU fp64 oracle for GigaAPI's matrix multiply -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package. The product path in
``paper_2504_01266_b200/`` never imports it and shares no code with it.

The arithmetic lives in ``oracle_gemm.c`` (plain C, fp64, i-k-j triple loop); this module
only builds/loads that library and marshals numpy arrays. It computes the plain definition

    C[i, j] = sum_k A[i, k] * B[k, j]        (S4.2.7 Matrix Multiplication)
    S[i, j] = sum_k |A[i, k]| * |B[k, j]|    (scale of the north_star bound 1e-5 * S)

Vector ops (dot, l2norm) follow PAPER.md:294-303 in oracle_dot.c; pins in tests/test_oracle_vec.py.

Pins (tests/test_oracle.py): identity, permutation, all-ones = K, integer rank-1 closed
form, the SPEC.md:282 worked 2x2 example (tests/golden/), exact rational brute force on
tiny shapes, exact integer products vs numpy int64, transpose identity, row independence,
thread-count invariance, S == C for nonnegative inputs, float64 BLAS agreement within the
fp64 error bound, and a negative control for the acceptance checker.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRCS = [os.path.join(_HERE, "oracle_gemm.c"), os.path.join(_HERE, "oracle_dot.c")]
_LIB_PATH = os.path.join(_HERE, "liboracle_gemm.so")
_lib = None
_lock = threading.Lock()

CFLAGS = ["-O2", "-fno-fast-math", "-ffp-contract=off", "-shared", "-fPIC", "-pthread"]


def build(force: bool = False) -> str:
    """Compile oracle_gemm.c with gcc (no GPU involved). Returns the .so path."""
    if force or not os.path.exists(_LIB_PATH) or any(
        os.path.getmtime(_LIB_PATH) < os.path.getmtime(s) for s in _SRCS
    ):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, *_SRCS, "-lm"])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB_PATH)
            i64, p = ctypes.c_int64, ctypes.c_void_p
            lib.oracle_gemm_rows_f64.argtypes = [p, p, p, i64, i64, i64, p, p, ctypes.c_int]
            lib.oracle_gemm_rows_f64.restype = ctypes.c_int
            lib.oracle_gemm_f64.argtypes = [p, p, i64, i64, i64, p, p, ctypes.c_int]
            lib.oracle_gemm_f64.restype = ctypes.c_int
            lib.oracle_dot_f64.argtypes = [p, p, i64, p, p]
            lib.oracle_dot_f64.restype = ctypes.c_int
            lib.oracle_l2norm_f64.argtypes = [p, i64, p]
            lib.oracle_l2norm_f64.restype = ctypes.c_int
            _lib = lib
    return _lib


def default_threads() -> int:
    return len(os.sched_getaffinity(0))


def _f32c(x) -> np.ndarray:
    x = np.asarray(x)
    if x.dtype != np.float32:
        raise TypeError(f"oracle inputs are fp32 (SPEC.md:234 MatrixF32), got {x.dtype}")
    return np.ascontiguousarray(x)


def gemm(A, B, nthreads: int | None = None, want_s: bool = True):
    """Full C = A @ B (fp64) and S = |A| @ |B| (fp64, or None). A: MxK fp32, B: KxN fp32."""
    A, B = _f32c(A), _f32c(B)
    if A.ndim != 2 or B.ndim != 2 or A.shape[1] != B.shape[0]:
        raise ValueError(f"shape mismatch {A.shape} x {B.shape}")
    M, K = A.shape
    N = B.shape[1]
    C = np.empty((M, N), np.float64)
    S = np.empty((M, N), np.float64) if want_s else None
    rc = _load().oracle_gemm_f64(
        A.ctypes.data, B.ctypes.data, M, N, K, C.ctypes.data,
        S.ctypes.data if S is not None else None, nthreads or default_threads())
    if rc != 0:
        raise RuntimeError(f"oracle_gemm_f64 failed rc={rc}")
    return C, S


def gemm_rows(A_rows, B, nthreads: int | None = None, want_s: bool = True):
    """C and S for the given rows of A only (A_rows: R x K fp32 holding those rows).

    Row independence makes this identical to the same rows of ``gemm``;
    tests/test_oracle.py pins that."""
    return gemm(A_rows, B, nthreads=nthreads, want_s=want_s)


def gemm_row_index(A, B, rows, nthreads: int | None = None, want_s: bool = True):
    """Rows ``rows`` (int64 indices into A) of C and S, computed without forming the rest."""
    A, B = _f32c(A), _f32c(B)
    rows = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
    M, K = A.shape
    N = B.shape[1]
    if rows.size and (rows.min() < 0 or rows.max() >= M):
        raise IndexError("row index out of range")
    C = np.empty((rows.size, N), np.float64)
    S = np.empty((rows.size, N), np.float64) if want_s else None
    rc = _load().oracle_gemm_rows_f64(
        A.ctypes.data, B.ctypes.data, rows.ctypes.data, rows.size, N, K, C.ctypes.data,
        S.ctypes.data if S is not None else None, nthreads or default_threads())
    if rc != 0:
        raise RuntimeError(f"oracle_gemm_rows_f64 failed rc={rc}")
    return C, S


# ---- vector operations (S4.2.8) ------------------------

def dot(x, y):
    """(dot, sabs): sum_i x_i y_i and sum_i |x_i y_i| in fp64, ascending i (oracle_dot.c)."""
    x, y = _f32c(x).reshape(-1), _f32c(y).reshape(-1)
    if x.size != y.size:
        raise ValueError(f"length mismatch {x.size} vs {y.size}")
    d, s = ctypes.c_double(), ctypes.c_double()
    rc = _load().oracle_dot_f64(x.ctypes.data, y.ctypes.data, x.size, ctypes.addressof(d),
                                ctypes.addressof(s))
    if rc != 0:
        raise RuntimeError("oracle_dot_f64 failed")
    return d.value, s.value


def l2norm(x):
    """sqrt(dot(x, x)), the square root taken once at the end."""
    x = _f32c(x).reshape(-1)
    r = ctypes.c_double()
    if _load().oracle_l2norm_f64(x.ctypes.data, x.size, ctypes.addressof(r)) != 0:
        raise RuntimeError("oracle_l2norm_f64 failed")
    return r.value
