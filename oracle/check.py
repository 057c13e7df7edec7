"""Acceptance checks against the oracle -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The bound is BASELINE.json north_star's, per element:

    |C_gpu[i,j] - Cref[i,j]| <= tol * S[i,j],   tol = 1e-5,  S = sum_k |A_ik| |B_kj|

with S == 0 forcing C_gpu == 0 exactly, and integer-valued inputs forcing bit-exact
agreement C_gpu == float32(Cref) (compared by value, so +0 == -0). DESIGN.md "Readings"
R5/R8 explain the tolerance form and the "several correct results" reading.
"""
from __future__ import annotations

import numpy as np

TOL = 1e-5


def rel_err(C_gpu, Cref, S):
    """Per-element |C_gpu - Cref| / S (0 where S == 0 and C_gpu == 0, inf where S == 0 else)."""
    C_gpu = np.asarray(C_gpu, dtype=np.float64)
    err = np.abs(C_gpu - Cref)
    with np.errstate(divide="ignore", invalid="ignore"):
        r = np.where(S > 0, err / np.where(S > 0, S, 1.0), np.where(err == 0, 0.0, np.inf))
    return r


def check_close(C_gpu, Cref, S, tol: float = TOL):
    """Return (ok, stats). ok iff every element is within tol*S (and finite)."""
    C_gpu = np.asarray(C_gpu)
    if C_gpu.shape != Cref.shape:
        return False, {"reason": f"shape {C_gpu.shape} != {Cref.shape}"}
    finite = np.isfinite(C_gpu)
    r = rel_err(C_gpu, Cref, S)
    worst = float(np.max(r)) if r.size else 0.0
    n_bad = int(np.count_nonzero(~(r <= tol)) + np.count_nonzero(~finite))
    stats = {"max_rel_err": worst, "mean_rel_err": float(np.mean(r)) if r.size else 0.0,
             "n_bad": n_bad, "n": int(r.size)}
    if n_bad:
        idx = np.unravel_index(int(np.argmax(np.where(np.isfinite(r), r, np.inf))), r.shape)
        stats["worst_index"] = tuple(int(i) for i in idx)
    return n_bad == 0, stats


def check_exact(C_gpu, Cref):
    """Bit-exact by value for integer-valued inputs: C_gpu == float32(Cref)."""
    C_gpu = np.asarray(C_gpu, dtype=np.float32)
    ref32 = Cref.astype(np.float32)
    if not np.array_equal(ref32.astype(np.float64), Cref):
        raise ValueError("reference is not exactly representable in fp32; not an exact case")
    bad = C_gpu != ref32
    stats = {"n_bad": int(np.count_nonzero(bad)), "n": int(C_gpu.size)}
    if stats["n_bad"]:
        stats["first_bad"] = tuple(int(i) for i in np.argwhere(bad)[0])
    return stats["n_bad"] == 0, stats
