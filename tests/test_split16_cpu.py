"""CPU pins of the 3xFP16 split's error analysis (test infrastructure).

This EMULATES the operand split of the 3xFP16 scheme in numpy -- e = ilogb(row max) - 14,
x' = x 2^-e, hi = fp16 RN(x'), lo = fp16 RN(x' - hi) (numpy's float16 conversion rounds to
nearest even, as cvt.rn.f16.f32 does) -- to check the bounds DESIGN.md states, which the
kernel's exception rule relies on. It supplies no expected value to any GPU test; the GPU
tests compare against the fp64 oracle.
"""
import numpy as np


def split16(x):
    """(e, hi, lo, err) of a row (float32 array): err = |x' - hi - lo| in scaled units."""
    x = np.asarray(x, np.float32)
    mx = np.max(np.abs(x))
    e = 0 if mx == 0 else int(np.frexp(np.float64(mx))[1] - 1) - 15
    if mx != 0 and np.float64(mx) * 2.0 ** -e >= 65504.0:
        e += 1
    xs = (x.astype(np.float64) * 2.0 ** -e).astype(np.float32)
    hi = xs.astype(np.float16)
    r = (xs - hi.astype(np.float32)).astype(np.float32)
    lo = r.astype(np.float16)
    err = np.abs(xs.astype(np.float64) - hi.astype(np.float64) - lo.astype(np.float64))
    return e, xs, hi, lo, err


def test_scale_puts_the_row_max_in_its_binade():
    rng = np.random.default_rng(1)
    for p in range(-100, 101, 7):
        x = (rng.uniform(-1, 1, 257) * 2.0 ** p).astype(np.float32)
        e, xs, hi, lo, err = split16(x)
        m = np.max(np.abs(xs))
        assert 2.0 ** 14 <= m < 65504.0
        assert np.isfinite(hi.astype(np.float32)).all()  # no fp16 overflow (max 65504)


def test_normal_range_split_error_bound():
    """|x'| >= 2^-3: |x' - hi - lo| <= 2^-22 |x'| (hi and lo RN to 11 bits, or lo's subnormal
    floor 2^-25 <= 2^-22 |x'|)."""
    rng = np.random.default_rng(2)
    for _ in range(20):
        x = rng.uniform(-1, 1, 4096).astype(np.float32) * np.float32(2.0 ** rng.integers(-60, 60))
        e, xs, hi, lo, err = split16(x)
        big = np.abs(xs) >= 2.0 ** -3
        assert np.all(err[big] <= 2.0 ** -22 * np.abs(xs[big].astype(np.float64)))


def test_exceptions_are_exactly_the_elements_beyond_2_to_minus_20():
    """The kernel's rule (split_f16): an exception iff err > 2^-20 |x'|. Everything else keeps
    its product's split error within 2 * 2^-20 + 2^-22; the exceptions only appear far below
    the row maximum (|x'| < 2^-5, i.e. more than 2^20 below it)."""
    rng = np.random.default_rng(3)
    x = rng.uniform(0, 1, 1 << 16).astype(np.float32)
    x[:64] *= np.float32(2.0 ** -30)
    e, xs, hi, lo, err = split16(x)
    exc = err > 2.0 ** -20 * np.abs(xs.astype(np.float64))
    assert exc[:64].sum() >= 32                    # far-below elements: most are exceptions
    assert np.all(np.abs(xs[exc]) < 2.0 ** -5)     # and only those
    keep = ~exc
    assert np.all(err[keep] <= 2.0 ** -20 * np.abs(xs[keep].astype(np.float64)))


def test_integers_split_exactly():
    """Integer inputs up to 2^11 in magnitude: x' is exact in fp16 after a power-of-two scale,
    lo = 0 -- the reason integer GEMMs are bit-exact under 3xFP16."""
    x = np.arange(-2048, 2049, dtype=np.float32)
    e, xs, hi, lo, err = split16(x)
    assert np.all(err == 0) and np.all(lo == 0)


def test_product_error_of_the_three_terms():
    """a b - (a_lo b_hi + a_hi b_lo + a_hi b_hi) = a_lo b_lo + (representation errors): with
    both operands in the normal range, <= 2 * 2^-22 + 2^-22 relative to |a b| (dropped lo lo)."""
    rng = np.random.default_rng(4)
    a = rng.uniform(0.5, 1, 1 << 14).astype(np.float32)
    b = rng.uniform(0.5, 1, 1 << 14).astype(np.float32)
    ea, xa, ah, al, _ = split16(a)
    eb, xb, bh, bl, _ = split16(b)
    ah, al, bh, bl = (v.astype(np.float64) for v in (ah, al, bh, bl))
    got = (al * bh + ah * bl + ah * bh) * 2.0 ** (ea + eb)
    exact = a.astype(np.float64) * b.astype(np.float64)
    rel = np.abs(got - exact) / np.abs(exact)
    assert rel.max() <= 3 * 2.0 ** -22


def pow2_scale(x, e):
    """Emulation of the epilogue's x 2^e (split16.cuh pow2_scale): two float32 multiplications
    by normal powers of two, 2^clamp(e, -126, 127) then 2^clamp(e - e1, -126, 127)."""
    e1 = np.clip(e, -126, 127)
    e2 = np.clip(e - e1, -126, 127)
    f1 = np.ldexp(np.float32(1), e1).astype(np.float32)
    f2 = np.ldexp(np.float32(1), e2).astype(np.float32)
    with np.errstate(over="ignore", under="ignore"):
        return (x.astype(np.float32) * f1).astype(np.float32) * f2


def test_pow2_scale_matches_ldexp_for_normal_results():
    """The epilogue's scaling equals the correctly rounded x 2^e (numpy's float64 ldexp, then
    one rounding to float32) for every result in float32's normal range, over the exponent
    range scale_exp produces (ea + eb in [-328, 224]) and sums |x| < 2^63; and whenever
    e is itself in [-126, 127] (a single rounding, subnormal results included)."""
    rng = np.random.default_rng(16)
    n = 400000
    x = (rng.uniform(-1, 1, n) * 2.0 ** rng.integers(-149, 63, n)).astype(np.float32)
    e = rng.integers(-328, 225, n)
    got = pow2_scale(x, e)
    with np.errstate(over="ignore", under="ignore"):
        want = np.ldexp(x.astype(np.float64), e).astype(np.float32)
    normal = np.abs(want) >= np.float32(2.0 ** -126)
    single = (e >= -126) & (e <= 127)
    sel = normal | single | (want == 0)
    assert sel.sum() > n // 2
    assert np.array_equal(got[sel].view(np.uint32), want[sel].view(np.uint32))
    # outside: a subnormal result reached through two roundings, within one subnormal ulp
    rest = ~sel
    assert np.all(np.abs(got[rest].astype(np.float64) - want[rest].astype(np.float64))
                  <= 2.0 ** -149)
