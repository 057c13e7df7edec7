"""Pins for the CPU fp64 oracle.

Each test checks the oracle against something other than itself: a closed form, a worked
example printed in SPEC.md, exact rational arithmetic, exact integer arithmetic in numpy,
or float64 BLAS within the fp64 error bound. A dropped term, a wrong sign, a transposed
operand or a wrong index in oracle_gemm.c fails at least one of them.
"""
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle.check import check_close, check_exact
import synth
from golden_io import load

RNG = np.random.default_rng(20250401)


def _rand_f32(shape, lo=-1.0, hi=1.0):
    return RNG.uniform(lo, hi, size=shape).astype(np.float32)


# ---- P5: SPEC.md worked examples (golden fixtures) ------------------------------------

@pytest.mark.parametrize("name", ["spec_2x2.txt", "identity_3x3.txt"])
def test_golden_examples(name):
    g = load(name)
    C, S = oracle.gemm(g["A"], g["B"])
    assert np.array_equal(C, g["C"].astype(np.float64))
    # S for these small examples: every term is a nonneg product when inputs are >= 0
    assert np.all(S >= np.abs(C))


# ---- P1: identity ----------------------------------------------------------------------

@pytest.mark.parametrize("m,k", [(1, 1), (3, 7), (17, 33), (64, 5)])
def test_identity_both_sides(m, k):
    A = _rand_f32((m, k))
    C, _ = oracle.gemm(A, np.eye(k, dtype=np.float32))
    assert np.array_equal(C, A.astype(np.float64))
    C2, _ = oracle.gemm(np.eye(m, dtype=np.float32), A)
    assert np.array_equal(C2, A.astype(np.float64))


# ---- P2: permutations (row/column indexing, non-square) --------------------------------

def test_permutations():
    m, k = 11, 6
    A = _rand_f32((m, k))
    p = RNG.permutation(m)
    P = np.zeros((m, m), np.float32)
    P[np.arange(m), p] = 1.0
    C, _ = oracle.gemm(P, A)  # (P A)[i] = A[p[i]]
    assert np.array_equal(C, A[p].astype(np.float64))
    q = RNG.permutation(k)
    Q = np.zeros((k, k), np.float32)
    Q[q, np.arange(k)] = 1.0  # (A Q)[:, j] = A[:, q[j]]
    C2, _ = oracle.gemm(A, Q)
    assert np.array_equal(C2, A[:, q].astype(np.float64))


# ---- P3: all ones gives K everywhere ---------------------------------------------------

@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (5, 3, 129), (2, 9, 1000)])
def test_all_ones(m, n, k):
    C, S = oracle.gemm(np.ones((m, k), np.float32), np.ones((k, n), np.float32))
    assert np.all(C == k) and np.all(S == k)


# ---- P4: rank-1 closed forms -----------------------------------------------------------

def test_rank1_integer_closed_form():
    m, k, n = 7, 13, 5
    u = RNG.integers(-5, 6, m)
    v = RNG.integers(-5, 6, k)
    w = RNG.integers(-5, 6, k)
    z = RNG.integers(-5, 6, n)
    A = np.outer(u, v).astype(np.float32)
    B = np.outer(w, z).astype(np.float32)
    C, _ = oracle.gemm(A, B)
    expect = float(v @ w) * np.outer(u, z).astype(np.float64)
    assert np.array_equal(C, expect)


def test_k1_outer_product():
    a = _rand_f32((9, 1))
    b = _rand_f32((1, 4))
    C, S = oracle.gemm(a, b)
    # a single product of two fp32 values is exact in fp64
    assert np.array_equal(C, a.astype(np.float64) * b.astype(np.float64))
    assert np.array_equal(S, np.abs(C))


# ---- P6: exact rational brute force on tiny shapes -------------------------------------

@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (2, 3, 4), (6, 5, 6), (3, 6, 2)])
def test_exact_rationals(m, n, k):
    # spread exponents so alignment and cancellation matter
    A = (_rand_f32((m, k)) * np.float32(2.0) ** RNG.integers(-20, 20, (m, k))).astype(np.float32)
    B = (_rand_f32((k, n)) * np.float32(2.0) ** RNG.integers(-20, 20, (k, n))).astype(np.float32)
    C, S = oracle.gemm(A, B)
    u = 2.0 ** -53
    gamma = k * u / (1 - k * u)
    for i in range(m):
        for j in range(n):
            exact = sum(Fraction(float(A[i, t])) * Fraction(float(B[t, j])) for t in range(k))
            exact_s = sum(abs(Fraction(float(A[i, t])) * Fraction(float(B[t, j]))) for t in range(k))
            assert abs(Fraction(C[i, j]) - exact) <= Fraction(gamma) * exact_s
            assert abs(Fraction(S[i, j]) - exact_s) <= Fraction(gamma) * exact_s


# ---- exact integer arithmetic (numpy int64 matmul is exact) ----------------------------

def test_integer_inputs_match_int64():
    A = synth.gen_matrix(37, 300, synth.MATRIX_A, "d3")
    B = synth.gen_matrix(300, 29, synth.MATRIX_B, "d3")
    C, S = oracle.gemm(A, B)
    Ai, Bi = A.astype(np.int64), B.astype(np.int64)
    assert np.array_equal(C, (Ai @ Bi).astype(np.float64))
    assert np.array_equal(S, (np.abs(Ai) @ np.abs(Bi)).astype(np.float64))


# ---- float64 BLAS within the fp64 error bound ------------------------------------------

def test_matches_float64_blas():
    A = synth.gen_matrix(40, 700, synth.MATRIX_A, "d2")
    B = synth.gen_matrix(700, 33, synth.MATRIX_B, "d2")
    C, S = oracle.gemm(A, B)
    ref = A.astype(np.float64) @ B.astype(np.float64)
    bound = 2 * 700 * 2.0 ** -53 * S
    assert np.all(np.abs(C - ref) <= bound)


# ---- S invariants ----------------------------------------------------------------------

def test_s_equals_c_for_nonnegative_and_sign_invariance():
    A = synth.gen_matrix(8, 50, synth.MATRIX_A, "d1")
    B = synth.gen_matrix(50, 6, synth.MATRIX_B, "d1")
    C, S = oracle.gemm(A, B)
    assert np.array_equal(C, S)
    Cn, Sn = oracle.gemm(-A, B)
    assert np.array_equal(Cn, -C) and np.array_equal(Sn, S)
    A2 = synth.gen_matrix(8, 50, synth.MATRIX_A, "d2")
    C2, S2 = oracle.gemm(A2, B)
    assert np.all(S2 >= np.abs(C2))


# ---- P7: transpose identity ------------------------------------------------------------

def test_transpose_identity():
    A = _rand_f32((13, 21))
    B = _rand_f32((21, 8))
    C, S = oracle.gemm(A, B)
    Ct, St = oracle.gemm(np.ascontiguousarray(B.T), np.ascontiguousarray(A.T))
    assert np.array_equal(C.T, Ct) and np.array_equal(S.T, St)


# ---- P8: row independence (the basis of the row partition) -----------------------------

def test_row_independence_and_row_index():
    A = _rand_f32((30, 40))
    B = _rand_f32((40, 12))
    C, S = oracle.gemm(A, B)
    rows = np.array([0, 29, 7, 7, 15])
    Cr, Sr = oracle.gemm_row_index(A, B, rows)
    assert np.array_equal(Cr, C[rows]) and np.array_equal(Sr, S[rows])
    C2, S2 = oracle.gemm_rows(A[10:20], B)
    assert np.array_equal(C2, C[10:20]) and np.array_equal(S2, S[10:20])


# ---- P9: thread-count invariance -------------------------------------------------------

def test_thread_count_invariance():
    A = _rand_f32((23, 64))
    B = _rand_f32((64, 17))
    C1, S1 = oracle.gemm(A, B, nthreads=1)
    C7, S7 = oracle.gemm(A, B, nthreads=7)
    assert np.array_equal(C1, C7) and np.array_equal(S1, S7)


def test_bad_arguments():
    with pytest.raises(ValueError):
        oracle.gemm(np.ones((2, 3), np.float32), np.ones((2, 3), np.float32))
    with pytest.raises(TypeError):
        oracle.gemm(np.ones((2, 2)), np.ones((2, 2)))


# ---- P10: negative controls for the checker --------------------------------------------

def test_checker_negative_controls():
    A = synth.gen_matrix(16, 64, synth.MATRIX_A, "d2")
    B = synth.gen_matrix(64, 16, synth.MATRIX_B, "d2")
    C, S = oracle.gemm(A, B)
    ok, _ = check_close(C.astype(np.float32), C, S)
    assert ok
    ok, _ = check_close(C + 0.5e-5 * S, C, S)
    assert ok
    ok, st = check_close(C + 2e-5 * S, C, S)
    assert not ok and st["n_bad"] == C.size
    bad = C.copy()
    bad[3, 5] += 3e-5 * S[3, 5]
    ok, st = check_close(bad, C, S)
    assert not ok and st["n_bad"] == 1 and st["worst_index"] == (3, 5)
    bad2 = C.copy()
    bad2[0, 0] = np.nan
    assert not check_close(bad2, C, S)[0]
    # exact checker
    Ai = synth.gen_matrix(5, 9, synth.MATRIX_A, "d3")
    Bi = synth.gen_matrix(9, 4, synth.MATRIX_B, "d3")
    Ci, _ = oracle.gemm(Ai, Bi)
    assert check_exact(Ci.astype(np.float32), Ci)[0]
    flip = Ci.astype(np.float32)
    flip[4, 3] += 1.0
    assert not check_exact(flip, Ci)[0]


# ---- the want_s=False path (worker_noS: the gloo schedule tests' reference and the
#      cpu_baseline timing leg) --------------------------------------------------------------

@pytest.mark.parametrize("threads", [1, 3, 8])
def test_without_s_equals_with_s_bitwise(threads):
    """C from the path that skips S is the same bits as C from the pinned path (same loop,
    same ascending k), for full products and for row-index selections."""
    A = _rand_f32((37, 53))
    B = _rand_f32((53, 29))
    C1, S1 = oracle.gemm(A, B, nthreads=threads)
    C0, S0 = oracle.gemm(A, B, nthreads=threads, want_s=False)
    assert S0 is None and S1 is not None
    assert C0.dtype == np.float64 and np.array_equal(C0.view(np.uint64), C1.view(np.uint64))
    rows = np.array([36, 0, 5, 5, 17])
    R1, _ = oracle.gemm_row_index(A, B, rows, nthreads=threads)
    R0, S = oracle.gemm_row_index(A, B, rows, nthreads=threads, want_s=False)
    assert S is None and np.array_equal(R0.view(np.uint64), R1.view(np.uint64))
    assert np.array_equal(R0, C1[rows])


def test_without_s_closed_forms():
    """want_s=False pinned on its own against closed forms: all-ones gives K, identity gives
    A, integer inputs give numpy's exact int64 product."""
    C, _ = oracle.gemm(np.ones((5, 300), np.float32), np.ones((300, 7), np.float32),
                       want_s=False)
    assert np.all(C == 300.0)
    A = _rand_f32((9, 9))
    C, _ = oracle.gemm(A, np.eye(9, dtype=np.float32), want_s=False)
    assert np.array_equal(C, A.astype(np.float64))
    Ai = RNG.integers(-50, 51, (23, 41))
    Bi = RNG.integers(-50, 51, (41, 19))
    C, _ = oracle.gemm(Ai.astype(np.float32), Bi.astype(np.float32), nthreads=4, want_s=False)
    assert np.array_equal(C, (Ai @ Bi).astype(np.float64))
