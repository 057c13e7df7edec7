"""Adversarial inputs for the TF32 + BF16 product scheme (test infrastructure).

This module EMULATES the kernel's operand rounding -- hi = tf32(x) rounded to nearest with
ties away from zero, lo = x - hi (exact), the correction operands rounded to bf16 (nearest,
ties to even), one exact TF32 product a_hi*b_hi plus the bf16 products bf16(a_lo)*bf16(b) +
bf16(a_hi)*bf16(b_lo) -- only to FIND inputs on which that split is least
accurate. It never supplies an expected value: the GPU tests compare against the closed form
K*a*b (constant rows / columns) or the fp64 oracle. It shares no code with the CUDA path.

Worst case of the split, per product, relative to |a||b| (derivation in DESIGN.md 6.7): the
four bf16 roundings contribute at most 2^-8|a_lo||b| + 2^-20|a||b| + 2^-8|a_hi||b_lo| +
2^-20|a||b| with |a_lo|, |b_lo| <= 2^-11 of |a|, |b|: <= 3 * 2^-19 = 5.72e-6 (plus terms of
order 2^-27). The bit patterns that reach the top of each term exclude each other in part;
the search below reaches 5.31e-6 with exact > computed, the direction in which the tensor
core's truncating accumulation adds to it.
"""
import numpy as np

U23 = 2.0 ** -23


def rna_tf32(x):
    """fp32 -> tf32 (10 explicit mantissa bits), nearest, ties away from zero (the kernel's
    two-integer-op rounding: add half a tf32 ulp to the magnitude bits, truncate)."""
    b = np.asarray(x, np.float32).view(np.uint32)
    return ((b + np.uint32(0x1000)) & np.uint32(0xFFFFE000)).view(np.float32)


def bf16_rne(x):
    """fp32 -> bf16 (as fp32), nearest, ties to even (cvt.rn.bf16x2.f32)."""
    b = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = ((b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return r.view(np.float32)


def split_product(a, b):
    """The TF32 + BF16 scheme's value of a*b (fp64; every term is exact in fp64)."""
    a = np.asarray(a, np.float32)
    b = np.asarray(b, np.float32)
    ah, bh = rna_tf32(a), rna_tf32(b)
    al, bl = a - ah, b - bh  # exact in fp32
    return (ah.astype(np.float64) * bh + bf16_rne(al).astype(np.float64) * bf16_rne(b)
            + bf16_rne(ah).astype(np.float64) * bf16_rne(bl))


def split_rel_error(a, b):
    """(a*b - split_product(a, b)) / |a*b|: positive when the scheme undershoots."""
    ex = np.asarray(a, np.float32).astype(np.float64) * np.asarray(b, np.float32)
    return (ex - split_product(a, b)) / np.abs(ex)


def search_pairs(top=4):
    """Structured search over significands in [1, 2): a = 1 + ja 2^-10 + la 2^-23 with the
    low part la in the top binade of lo (|lo| in [2^-12, 2^-11)), b likewise. Returns the
    `top` pairs (a, b, error) with the largest positive error, distinct a."""
    best = {}
    la = np.arange(2048, 4096, dtype=np.int64)
    for ja in range(64):
        A = (1 + ja * 2.0 ** -10 + la * U23).astype(np.float32)
        for jb in range(64):
            for lb in (4087, 4081, 4089, 4095, 4071, 4085, 4079):
                bv = np.float32(1 + jb * 2.0 ** -10 + lb * U23)
                e = split_rel_error(A, np.full_like(A, bv))
                k = int(np.argmax(e))
                key = float(A[k])
                if key not in best or e[k] > best[key][2]:
                    best[key] = (float(A[k]), float(bv), float(e[k]))
    return sorted(best.values(), key=lambda t: -t[2])[:top]


# search_pairs(4), committed (tests/test_adversarial_cpu.py re-runs the search and checks it):
# (a, b, emulated relative split error), fp32-exact values.
WORST_PAIRS = [
    (float.fromhex("0x1.011fd0p+0"), float.fromhex("0x1.00dfeep+0"), 5.308396767588313e-06),
    (float.fromhex("0x1.051fd0p+0"), float.fromhex("0x1.00dfeep+0"), 5.239819865824205e-06),
    (float.fromhex("0x1.091fd0p+0"), float.fromhex("0x1.00dfeep+0"), 5.173312239796809e-06),
    (float.fromhex("0x1.0d1fd0p+0"), float.fromhex("0x1.00dfeep+0"), 5.108781622431647e-06),
]


# ---- the 3xFP16 scheme ------------------------------------------------------
# Its split error is largest just above the exception threshold: an element 2^-20 below its
# row's maximum. With the maximum at 1.0 the row is scaled by 2^15 (max' = 2^15), so x' =
# x 2^15; for x' just above 2^-5, hi = RN fp16(x') = 2^-5 and lo = RN fp16(x' - hi) lands on
# fp16's subnormal grid (2^-24), where the fp32 grid of x' is 2^-28. x' = 2^-5 + 2^-25 puts
# r = x' - hi exactly half-way between 0 and 2^-24: RN-even gives lo = 0, the split
# undershoots by 2^-25 = (1 - 2^-20) 2^-20 |x'| -- the largest error an element can have
# without being an exception (the GEMM carries it, not the fix kernels). Both operands at
# this value: every product undershoots by ~2 * 2^-20 (1.9e-6), the same sign as the
# truncating TMEM accumulation.
FP16_ROW_MAX = 1.0
FP16_WORST_X = float(np.float32((2.0 ** -5 + 2.0 ** -25) * 2.0 ** -15))


def split16_rel_error(x, row_max=FP16_ROW_MAX):
    """(x - rep(x)) / |x| of the 3xFP16 split for an element of a row whose maximum is
    row_max (emulated: scale to [2^15, 65504), fp16 RN hi, fp16 RN lo)."""
    mx = np.float64(row_max)
    e = int(np.frexp(mx)[1] - 1) - 15
    if mx * 2.0 ** -e >= 65504.0:
        e += 1
    xs = np.float32(np.float64(np.float32(x)) * 2.0 ** -e)
    hi = np.float16(xs)
    lo = np.float16(np.float32(xs - np.float32(hi)))
    rep = (np.float64(hi) + np.float64(lo)) * 2.0 ** e
    return (np.float64(np.float32(x)) - rep) / abs(np.float64(np.float32(x)))
