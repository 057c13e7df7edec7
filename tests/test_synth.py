"""The seeded input generator: published splitmix64 test vectors, ranges, and numpy/torch twin."""
import numpy as np
import pytest
import torch

import synth


def test_splitmix64_reference_vectors():
    # splitmix64 (Steele, Lea, Flood 2014; Vigna's reference C) seeded with state 0 returns
    # 0xE220A8397B1DCDAF then 0x6E789E6AA1B965F4: state advances by the golden gamma before
    # mixing, so output n is mix((n+1)*gamma) and our z = x + gamma maps x = n*gamma to it.
    with np.errstate(over="ignore"):
        x = np.array([0, 0x9E3779B97F4A7C15], dtype=np.uint64)
        out = synth._splitmix64_np(x)
    assert int(out[0]) == 0xE220A8397B1DCDAF
    assert int(out[1]) == 0x6E789E6AA1B965F4


@pytest.mark.parametrize("dist", synth.DISTS)
def test_ranges(dist):
    x = synth.gen_rows(0, 64, 1000, synth.MATRIX_A, dist)
    if dist == "d1":
        assert x.min() > 0 and x.max() <= 1
    elif dist == "d2":
        assert x.min() >= -1 and x.max() < 1 and abs(float(x.mean())) < 0.01
    elif dist == "d4":
        assert x.min() >= -10 and x.max() <= 10 and abs(float(x.mean())) < 0.1
    elif dist == "d5":
        assert x.min() > 0 and x.max() <= 1 and abs(float(x.mean()) - 0.5) < 0.01
        # full significands: small values keep bits below the 2^-24 grid of d1
        small = x[x < 2.0 ** -8]
        assert small.size and np.any(small != np.round(small * 2.0 ** 24) * 2.0 ** -24)
    else:
        assert np.array_equal(x, np.round(x)) and x.min() == -8 and x.max() == 8


def test_row_subsets_reproduce():
    full = synth.gen_matrix(40, 33, synth.MATRIX_B, "d2")
    assert np.array_equal(synth.gen_rows(13, 9, 33, synth.MATRIX_B, "d2"), full[13:22])
    assert np.array_equal(synth.gen_rows_index([39, 0, 5], 33, synth.MATRIX_B, "d2"),
                          full[[39, 0, 5]])
    assert not np.array_equal(full, synth.gen_matrix(40, 33, synth.MATRIX_A, "d2"))


@pytest.mark.parametrize("dist", synth.DISTS)
def test_torch_twin_bit_exact(dist):
    a = synth.gen_rows(5, 17, 301, synth.MATRIX_A, dist)
    t = synth.gen_rows_torch(5, 17, 301, synth.MATRIX_A, dist, chunk=1000).numpy()
    assert np.array_equal(a.view(np.uint32), t.view(np.uint32))
