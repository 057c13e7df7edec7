"""Pins for the vector-operation oracle (dot, L2 norm)."""
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth
from golden_io import load

RNG = np.random.default_rng(294)


def test_spec_worked_examples():
    g = load("spec_vector.txt")
    d, s = oracle.dot(g["X"][0], g["Y"][0])
    assert d == float(g["C"][0][0]) and s == 32.0
    assert oracle.l2norm(g["L"][0]) == float(g["R"][0][0])
    z = np.zeros(1024, np.float32)
    assert oracle.dot(z, z) == (0.0, 0.0) and oracle.l2norm(z) == 0.0


@pytest.mark.parametrize("n", [1, 2, 7, 33])
def test_exact_rationals(n):
    x = (RNG.uniform(-1, 1, n) * 2.0 ** RNG.integers(-30, 30, n)).astype(np.float32)
    y = (RNG.uniform(-1, 1, n) * 2.0 ** RNG.integers(-30, 30, n)).astype(np.float32)
    d, s = oracle.dot(x, y)
    exact = sum(Fraction(float(a)) * Fraction(float(b)) for a, b in zip(x, y))
    exact_s = sum(abs(Fraction(float(a)) * Fraction(float(b))) for a, b in zip(x, y))
    u = 2.0 ** -53
    assert abs(Fraction(d) - exact) <= Fraction(n * u) * exact_s
    assert abs(Fraction(s) - exact_s) <= Fraction(n * u) * exact_s


def test_integer_inputs_exact():
    x = synth.gen_vector(100003, synth.VECTOR_X, "d3")
    y = synth.gen_vector(100003, synth.VECTOR_Y, "d3")
    d, s = oracle.dot(x, y)
    xi, yi = x.astype(np.int64), y.astype(np.int64)
    assert d == float(int((xi * yi).sum())) and s == float(int(np.abs(xi * yi).sum()))


def test_closed_forms():
    n = 4097
    ones = np.ones(n, np.float32)
    assert oracle.dot(ones, ones)[0] == n
    x = synth.gen_vector(n, synth.VECTOR_X, "d4")
    for k in (0, 17, n - 1):
        e = np.zeros(n, np.float32)
        e[k] = 1.0
        assert oracle.dot(x, e)[0] == float(x[k]) and oracle.dot(e, x)[0] == float(x[k])
    y = synth.gen_vector(n, synth.VECTOR_Y, "d4")
    assert abs(oracle.dot(x, y)[0]) <= oracle.l2norm(x) * oracle.l2norm(y)  # Cauchy-Schwarz
    assert oracle.l2norm(np.float32(4.0) * x) == 4.0 * oracle.l2norm(x)  # exact power-of-2 scale
    assert oracle.dot(x, y)[0] == oracle.dot(y, x)[0]  # symmetric (same products, same order)
    assert math.isclose(oracle.l2norm(x) ** 2, oracle.dot(x, x)[0], rel_tol=1e-15)


def test_matches_float64_library_dot():
    x = synth.gen_vector(1 << 20, synth.VECTOR_X, "d4")
    y = synth.gen_vector(1 << 20, synth.VECTOR_Y, "d4")
    d, s = oracle.dot(x, y)
    ref = float(np.dot(x.astype(np.float64), y.astype(np.float64)))
    assert abs(d - ref) <= 2 * x.size * 2.0 ** -53 * s
    # SPEC.md:292 example: "random length 2^20 uniform[-10,10] ... within rel. err 1e-5"
    assert abs(d - ref) <= 1e-5 * abs(ref)


def test_d4_distribution_range_and_twin():
    import torch
    x = synth.gen_vector(5000, synth.VECTOR_X, "d4")
    assert x.min() >= -10 and x.max() < 10 and abs(float(x.mean())) < 0.5
    t = synth.gen_rows_torch(0, 1, 5000, synth.VECTOR_X, "d4").numpy()[0]
    assert np.array_equal(x.view(np.uint32), t.view(np.uint32))


def test_bad_arguments():
    with pytest.raises(ValueError):
        oracle.dot(np.ones(3, np.float32), np.ones(4, np.float32))
