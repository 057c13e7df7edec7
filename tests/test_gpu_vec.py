"""GPU parity for the vector operations (dot, L2 norm).

Bar: |dot_gpu - dot_oracle| <= 2 n 2^-53 sum_i |x_i y_i| (both accumulate exact fp32 products
in fp64, in different orders); integer-valued inputs exact; the SPEC worked examples exact.
"""
import math

import numpy as np
import pytest

import oracle
import synth
from golden_io import load

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


@pytest.fixture(scope="module")
def giga(torch_cuda):
    from paper_2504_01266_b200 import build
    build.build()
    from paper_2504_01266_b200 import giga as g
    g.finalize()
    g.init(1)
    yield g
    g.finalize()


def _bound(n, s):
    return 2 * n * 2.0 ** -53 * s


def test_spec_examples_exact(giga, torch_cuda):
    g = load("spec_vector.txt")
    assert giga.dot(g["X"][0], g["Y"][0]) == 32.0
    assert giga.l2norm(g["L"][0]) == 5.0
    z = np.zeros(4096, np.float32)
    assert giga.dot(z, z) == 0.0 and giga.l2norm(z) == 0.0


@pytest.mark.parametrize("n", [1, 3, 4, 1023, 4096, (1 << 20) + 3, 1 << 26])
@pytest.mark.parametrize("where", ["host", "device"])
def test_dot_vs_oracle(giga, torch_cuda, n, where):
    torch = torch_cuda
    x = synth.gen_vector(n, synth.VECTOR_X, "d4")
    y = synth.gen_vector(n, synth.VECTOR_Y, "d4")
    ref, s = oracle.dot(x, y)
    if where == "host":
        got = giga.dot(x, y)
    else:
        got = giga.dot(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
    assert abs(got - ref) <= _bound(n, s), (got, ref)


def test_integer_inputs_exact_and_deterministic(giga, torch_cuda):
    torch = torch_cuda
    n = (1 << 22) + 5
    x = synth.gen_vector(n, synth.VECTOR_X, "d3")
    y = synth.gen_vector(n, synth.VECTOR_Y, "d3")
    ref, _ = oracle.dot(x, y)
    dx, dy = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    a, b = giga.dot(dx, dy), giga.dot(dx, dy)
    assert a == ref and b == ref
    # unaligned operands (offset by one element) take the scalar path
    assert giga.dot(dx[1:], dy[1:], n - 1) == oracle.dot(x[1:], y[1:])[0]


def test_l2norm_vs_oracle(giga, torch_cuda):
    n = 1 << 24
    x = synth.gen_vector(n, synth.VECTOR_X, "d4")
    ref = oracle.l2norm(x)
    got = giga.l2norm(x)
    s = oracle.dot(x, x)[1]
    # sqrt is monotone with derivative 1/(2 sqrt): the dot bound maps to this one
    assert abs(got - ref) <= _bound(n, s) / (2 * ref) + 4 * math.ulp(ref)


def test_dot_errors(giga, torch_cuda):
    x = np.ones(8, np.float32)
    with pytest.raises(giga.GigaError) as e:
        giga.dot(x, x, 0)
    assert e.value.status == "GIGA_ERR_INVALID_ARG"
    with pytest.raises(giga.GigaError) as e:
        giga.dot(x, torch_cuda.ones(8, device="cuda"))
    assert e.value.status == "GIGA_ERR_INVALID_ARG"
    with pytest.raises(giga.GigaError) as e:
        giga.dot(x, x, 8, ngpus=2)
    assert e.value.status == "GIGA_ERR_INVALID_ARG"


@pytest.mark.parametrize("force", ["0", "1"])
def test_dot_rank_api(torch_cuda, monkeypatch, force):
    """Rank API at world 1; with GIGA_FORCE_COMM the NCCL all-reduce of the partial runs."""
    torch = torch_cuda
    from paper_2504_01266_b200 import giga as g
    monkeypatch.setenv("GIGA_FORCE_COMM", force)
    g.finalize()
    g.rank_init(0, 1, 0, None)
    try:
        n = (1 << 20) + 7
        x = synth.gen_vector(n, synth.VECTOR_X, "d3")
        y = synth.gen_vector(n, synth.VECTOR_Y, "d3")
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        got = g.dot_rank(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), n, stream=s)
        assert got == oracle.dot(x, y)[0]
    finally:
        g.finalize()
        g.init(1)


def test_paper_worked_examples_and_release(torch_cuda):
    """The SPEC's worked examples through the C ABI (SPEC.md:282 2x2 product, the vector
    examples: dot 32, L2 norm 5), and giga_finalize releasing the
    library's device memory."""
    from paper_2504_01266_b200 import giga as g
    g.finalize()
    free0 = torch_cuda.cuda.mem_get_info()[0]
    g.init(1)
    gold = load("spec_2x2.txt")
    C2 = np.empty_like(gold["C"], dtype=np.float32)
    g.matmul(np.ascontiguousarray(gold["A"], np.float32), np.ascontiguousarray(gold["B"], np.float32),
             C2, 2, 2, 2, 1)
    assert np.array_equal(C2, gold["C"])
    A = synth.gen_matrix(300, 520, synth.MATRIX_A, "d3")
    B = synth.gen_matrix(520, 260, synth.MATRIX_B, "d3")
    dC = torch_cuda.empty((300, 260), device="cuda")
    g.matmul(torch_cuda.from_numpy(A).cuda(), torch_cuda.from_numpy(B).cuda(), dC, 300, 260, 520, 1)
    assert np.array_equal(dC.cpu().numpy().astype(np.float64), oracle.gemm(A, B)[0])
    v = load("spec_vector.txt")
    assert g.dot(np.ascontiguousarray(v["X"][0], np.float32),
                 np.ascontiguousarray(v["Y"][0], np.float32)) == 32.0
    assert g.l2norm(np.ascontiguousarray(v["L"][0], np.float32)) == 5.0
    g.finalize()
    torch_cuda.cuda.synchronize()
    assert torch_cuda.cuda.mem_get_info()[0] >= free0 - (64 << 20)
    g.init(1)
