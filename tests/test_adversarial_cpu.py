"""CPU checks of the adversarial-input constructor (tests/adversarial.py): its emulation of
the operand roundings on hand-worked values, the committed worst pairs, and the analytic
per-product bound of the TF32 + BF16 split."""
import numpy as np

import adversarial as adv

U = 2.0 ** -23


def test_roundings_on_worked_values():
    f = np.float32
    # tf32: 11 significant bits, ties away from zero
    assert adv.rna_tf32(f(1 + 2 ** -11)) == f(1 + 2 ** -10)
    assert adv.rna_tf32(f(1 + 2 ** -11 - U)) == f(1.0)
    assert adv.rna_tf32(f(-(1 + 2 ** -11))) == f(-(1 + 2 ** -10))
    assert adv.rna_tf32(f(1 + 3 * 2 ** -11)) == f(1 + 2 ** -9)
    # bf16: 8 significant bits, ties to even
    assert adv.bf16_rne(f(1 + 2 ** -8)) == f(1.0)
    assert adv.bf16_rne(f(1 + 3 * 2 ** -8)) == f(1 + 2 ** -6)
    assert adv.bf16_rne(f(1 + 2 ** -8 + U)) == f(1 + 2 ** -7)
    # lo is exact and the split reproduces tf32-exact products exactly
    a = f(1 + 2 ** -10)
    assert adv.split_rel_error(a, a) == 0.0
    x = f(1.2345678)
    assert f(adv.rna_tf32(x)) + (x - adv.rna_tf32(x)) == x


def test_committed_worst_pairs_reproduce():
    found = adv.search_pairs(4)
    assert [(a, b) for a, b, _ in found] == [(a, b) for a, b, _ in adv.WORST_PAIRS]
    for (a, b, e), (_, _, e2) in zip(adv.WORST_PAIRS, found):
        assert abs(e - e2) < 1e-18
        assert abs(adv.split_rel_error(np.float32(a), np.float32(b)) - e) < 1e-18
        assert e > 5.1e-6


def test_split_error_within_analytic_bound():
    """|error| <= 3 * 2^-19 |a||b| + O(2^-27) over random and structured significands."""
    rng = np.random.default_rng(5)
    a = (1 + rng.integers(0, 1 << 23, 1 << 20) * U).astype(np.float32)
    b = (1 + rng.integers(0, 1 << 23, 1 << 20) * U).astype(np.float32)
    e = np.abs(adv.split_rel_error(a, b))
    bound = 3 * 2.0 ** -19 + 2.0 ** -26
    assert e.max() <= bound
    for a0, b0, _ in adv.WORST_PAIRS:
        assert abs(adv.split_rel_error(np.float32(a0), np.float32(b0))) <= bound


def test_fp16_worst_element_is_just_under_the_exception_threshold():
    """The constructed 3xFP16 worst case (tests/adversarial.py): undershoot 2^-25 / x',
    below the 2^-20 exception threshold (so the GEMM carries it, not the fix kernels), and the
    largest error any element of that binade reaches (fp32 grid 2^-28 there in scaled units,
    lo's subnormal grid 2^-24: at most half a step)."""
    e = adv.split16_rel_error(adv.FP16_WORST_X)
    assert e == 2.0 ** -25 / (2.0 ** -5 + 2.0 ** -25)
    assert 0 < e < 2.0 ** -20
    xs = (2.0 ** -5 + np.arange(0, 1 << 12) * 2.0 ** -28) * 2.0 ** -15
    errs = np.array([adv.split16_rel_error(v) for v in xs])
    assert np.abs(errs).max() <= e
