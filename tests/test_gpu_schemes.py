"""GPU parity of the fp32-accurate schemes of the shard GEMM against the CPU fp64 oracle.

terms = 3: 3xTF32 (the product default, BASELINE north_star (3)).
terms = 2: TF32 + BF16 -- a_hi*b_hi as one kind::tf32 MMA plus both corrections as one K=16
kind::f16 MMA over [bf16(a_lo) | bf16(a_hi)] . [bf16(b) ; bf16(b_lo)] (gemm_3xtf32.cu,
DESIGN.md 6.7). Its split error is <= 2^-18 |a||b| per product with the RN hi (the library
default), inside the 1e-5 * sum|A||B| bound (R5) with the accumulation error on top.
"""
import numpy as np
import pytest

import oracle
from oracle.check import check_close, check_exact
import synth

pytestmark = pytest.mark.gpu

SHAPES = [(1, 4, 4), (130, 260, 20), (255, 256, 16), (257, 512, 36), (600, 1000, 1028),
          (2048, 2048, 512)]


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


def _run(giga, torch, A, B, terms, cta_group=0):
    M, K = A.shape
    N = B.shape[1]
    dA = torch.from_numpy(np.ascontiguousarray(A)).cuda()
    dB = torch.from_numpy(np.ascontiguousarray(B)).cuda()
    dC = torch.full((M, N), float("nan"), device="cuda")
    giga.gemm_3xtf32(dA, None, dB, None, dC, M, N, K, terms=terms, cta_group=cta_group)
    torch.cuda.synchronize()
    return dC.cpu().numpy()


@pytest.mark.parametrize("cta_group", [1, 2])
@pytest.mark.parametrize("M,N,K", SHAPES)
def test_tf32bf16_bit_exact_integers(giga, torch_cuda, M, N, K, cta_group):
    """Integer inputs: hi = x, lo = 0, the correction MMA adds exact zeros; C bit-exact."""
    A = synth.gen_matrix(M, K, synth.MATRIX_A, "d3")
    B = synth.gen_matrix(K, N, synth.MATRIX_B, "d3")
    C = _run(giga, torch_cuda, A, B, 2, cta_group)
    ok, st = check_exact(C, oracle.gemm(A, B)[0])
    assert ok, st


@pytest.mark.parametrize("cta_group", [1, 2])
@pytest.mark.parametrize("M,N,K,dist", [(257, 516, 36, "d4"), (700, 900, 3000, "d1"),
                                        (600, 1000, 1028, "d2"), (1500, 2048, 4100, "d1")])
def test_tf32bf16_tolerance(giga, torch_cuda, M, N, K, dist, cta_group):
    A = synth.gen_matrix(M, K, synth.MATRIX_A, dist)
    B = synth.gen_matrix(K, N, synth.MATRIX_B, dist)
    C = _run(giga, torch_cuda, A, B, 2, cta_group)
    Cref, S = oracle.gemm(A, B)
    ok, st = check_close(C, Cref, S)
    assert ok, st
    # the corrections must be there: plain TF32 (terms = 1) is ~1e-4 off on these inputs
    C1 = _run(giga, torch_cuda, A, B, 1, cta_group)
    _, st1 = check_close(C1, Cref, S)
    assert st["max_rel_err"] < 0.1 * st1["max_rel_err"]


@pytest.mark.parametrize("terms", [3, 2])
def test_coherent_worst_case(giga, torch_cuda, terms):
    """Row i of A constant x_i, column j of B constant y_j: all K products of C[i][j] are the
    same, so the split errors add up coherently instead of averaging out -- the adversarial
    case for the per-product bound (32768 value pairs, K = 2048)."""
    rng = np.random.default_rng(11)
    M, N, K = 128, 256, 2048
    x = rng.uniform(0.5, 2.0, M).astype(np.float32)
    y = rng.uniform(0.5, 2.0, N).astype(np.float32)
    A = np.repeat(x[:, None], K, axis=1)
    B = np.repeat(y[None, :], K, axis=0)
    C = _run(giga, torch_cuda, A, B, terms)
    Cref, S = oracle.gemm(A, B)
    ok, st = check_close(C, Cref, S)
    print(f"terms {terms}: coherent max rel err {st['max_rel_err']:.3e}")
    assert ok, st


def test_scheme_is_selectable_for_the_product_path(tmp_path):
    """GIGA_SCHEME=tf32bf16 routes the product path (giga_matmul_sharded) through terms = 2;
    checked in a child process because the scheme is read once per process."""
    import subprocess
    import sys
    import os
    code = (
        "import numpy as np, torch, oracle, synth\n"
        "from oracle.check import check_close\n"
        "from paper_2504_01266_b200 import giga\n"
        "giga.init(1)\n"
        "M, N, K = 520, 1000, 2000\n"
        "A = synth.gen_matrix(M, K, synth.MATRIX_A, 'd1'); B = synth.gen_matrix(K, N, synth.MATRIX_B, 'd1')\n"
        "dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()\n"
        "dC = torch.full((M, N), float('nan'), device='cuda')\n"
        "giga.matmul_sharded([dA], [dB], [dC], M, N, K)\n"
        "ref, S = oracle.gemm(A, B)\n"
        "ok, st = check_close(dC.cpu().numpy(), ref, S)\n"
        "assert ok, st\n"
        "print('ok', st['max_rel_err'])\n"
        "giga.finalize()\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, GIGA_SCHEME="tf32bf16", PYTHONPATH=root)
    r = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.startswith("ok"), r.stdout + r.stderr
