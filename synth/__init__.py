"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NO arithmetic of the method (no product, no sum, no split): it only
turns (seed, matrix_id, linear index) into an fp32 value. Both sides receive the same
arrays; neither computes its inputs itself.

Generator: counter-based splitmix64 of

    x = seed XOR (matrix_id << 56) XOR linear_index,   linear_index = row * cols + col

keeping the top 24 bits v of the mixed word. Three distributions (PAPER.md:355 says only
"random numbers ... CUDA random number generator ... same random seed"; the distribution
is unstated, reading R11):

* ``"d1"``  x = (v + 1) * 2^-24            in (0, 1]   (cuRAND-uniform reading; all positive)
* ``"d2"``  x = (v - 2^23) * 2^-23         in [-1, 1)  (zero-mean; used for throughput runs)
* ``"d3"``  x = (v mod 17) - 8             in [-8, 8]  (integers: the bit-exact mode)
* ``"d5"``  x = fp32 RN of (v 2^24 + w + 1) 2^-48 in (0, 1], w the next 24 bits of the word:
            uniform values with FULL 24-bit significands at every magnitude (the others are
            fixed-point grids, whose small values have few significant bits). Elements far
            below 1 keep all their bits -- the inputs on which the 3xFP16 scheme's exception
            path runs at a realistic rate (~2^-20 of the elements).

Every value is an exact dyadic rational, so the numpy (host) and torch (device)
implementations below agree bit for bit (tests/test_synth.py pins that), and any row
subset of a matrix can be regenerated independently (row-sampled parity at full size).
"""
from __future__ import annotations

import numpy as np

SEED = 250401266
MATRIX_A = 1
MATRIX_B = 2
VECTOR_X = 3  # dot / L2 norm operands
VECTOR_Y = 4

_GOLDEN = 0x9E3779B97F4A7C15
_MIX1 = 0xBF58476D1CE4E5B9
_MIX2 = 0x94D049BB133111EB
DISTS = ("d1", "d2", "d3", "d4", "d5")


def gen_vector(n: int, vec_id: int, dist: str = "d4", seed: int = SEED) -> np.ndarray:
    """A length-n fp32 vector (one row of the counter-based generator)."""
    return gen_rows(0, 1, n, vec_id, dist, seed)[0]


def _splitmix64_np(x: np.ndarray) -> np.ndarray:
    z = x + np.uint64(_GOLDEN)
    z = (z ^ (z >> np.uint64(30))) * np.uint64(_MIX1)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(_MIX2)
    return z ^ (z >> np.uint64(31))


def _to_dist_np(v: np.ndarray, dist: str, w=None) -> np.ndarray:
    if dist == "d5":  # 48-bit dyadic in (0, 1], exact in fp64, one RN to fp32
        return ((v.astype(np.float64) * 2.0 ** 24 + w.astype(np.float64) + 1.0) * 2.0 ** -48
                ).astype(np.float32)
    if dist == "d4":  # uniform [-10, 10): the paper's vector benchmark values
        return ((v.astype(np.int64) - (1 << 23)).astype(np.float64) * (10 * 2.0 ** -23)
                ).astype(np.float32)
    if dist == "d1":
        return ((v + 1).astype(np.float64) * 2.0 ** -24).astype(np.float32)
    if dist == "d2":
        return ((v.astype(np.int64) - (1 << 23)).astype(np.float64) * 2.0 ** -23).astype(np.float32)
    if dist == "d3":
        return ((v % 17).astype(np.int64) - 8).astype(np.float32)
    raise ValueError(f"unknown distribution {dist!r}; expected one of {DISTS}")


def gen_rows(row0: int, nrows: int, cols: int, matrix_id: int, dist: str = "d2",
             seed: int = SEED, chunk: int = 1 << 24) -> np.ndarray:
    """Rows [row0, row0 + nrows) of the (., cols) matrix `matrix_id`, fp32, row-major."""
    out = np.empty((nrows, cols), np.float32)
    flat = out.reshape(-1)
    base = np.uint64((seed ^ (matrix_id << 56)) & 0xFFFFFFFFFFFFFFFF)
    start = row0 * cols
    total = nrows * cols
    with np.errstate(over="ignore"):
        for off in range(0, total, chunk):
            n = min(chunk, total - off)
            idx = np.arange(start + off, start + off + n, dtype=np.uint64)
            z = _splitmix64_np(base ^ idx)
            v = z >> np.uint64(40)
            w = (z >> np.uint64(16)) & np.uint64(0xFFFFFF)
            flat[off:off + n] = _to_dist_np(v, dist, w)
    return out


def gen_matrix(rows: int, cols: int, matrix_id: int, dist: str = "d2", seed: int = SEED):
    return gen_rows(0, rows, cols, matrix_id, dist, seed)


def gen_rows_index(row_idx, cols: int, matrix_id: int, dist: str = "d2", seed: int = SEED):
    """Arbitrary (not necessarily contiguous) rows, fp32 (len(row_idx), cols)."""
    row_idx = np.asarray(row_idx, dtype=np.int64)
    out = np.empty((row_idx.size, cols), np.float32)
    for t, r in enumerate(row_idx):
        out[t] = gen_rows(int(r), 1, cols, matrix_id, dist, seed)[0]
    return out


# ---- torch implementation (same bits; used to fill large device buffers quickly) --------

def _i64(u: int) -> int:
    """uint64 constant -> the int64 with the same bits."""
    u &= 0xFFFFFFFFFFFFFFFF
    return u - (1 << 64) if u >= (1 << 63) else u


def _lsr(t, s: int):
    """Logical shift right of int64 bit patterns."""
    return (t >> s) & ((1 << (64 - s)) - 1)


def gen_rows_torch(row0: int, nrows: int, cols: int, matrix_id: int, dist: str = "d2",
                   seed: int = SEED, device="cpu", out=None, chunk: int = 1 << 26):
    """torch twin of ``gen_rows`` (int64 wrap-around arithmetic == uint64 bit patterns).

    Writes into ``out`` (a contiguous fp32 tensor of nrows*cols elements) if given."""
    import torch

    if out is None:
        out = torch.empty((nrows, cols), dtype=torch.float32, device=device)
    flat = out.view(-1)
    base = _i64(seed ^ (matrix_id << 56))
    start = row0 * cols
    total = nrows * cols
    for off in range(0, total, chunk):
        n = min(chunk, total - off)
        idx = torch.arange(start + off, start + off + n, dtype=torch.int64, device=flat.device)
        z = (idx ^ base) + _i64(_GOLDEN)
        z = (z ^ _lsr(z, 30)) * _i64(_MIX1)
        z = (z ^ _lsr(z, 27)) * _i64(_MIX2)
        z = z ^ _lsr(z, 31)
        v = _lsr(z, 40)
        if dist == "d5":
            w = _lsr(z, 16) & 0xFFFFFF
            vals = (v.to(torch.float64) * 2.0 ** 24 + w.to(torch.float64) + 1.0) * 2.0 ** -48
        elif dist == "d4":
            vals = (v - (1 << 23)).to(torch.float64) * (10 * 2.0 ** -23)
        elif dist == "d1":
            vals = (v + 1).to(torch.float64) * 2.0 ** -24
        elif dist == "d2":
            vals = (v - (1 << 23)).to(torch.float64) * 2.0 ** -23
        elif dist == "d3":
            vals = (v % 17 - 8).to(torch.float64)
        else:
            raise ValueError(f"unknown distribution {dist!r}")
        flat[off:off + n] = vals.to(torch.float32)
        del idx, z, v, vals
    return out
