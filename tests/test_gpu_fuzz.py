"""Seeded shape fuzzing: random (M, N, K) from 1 to ~700 (ragged everywhere: K and N not
multiples of 4 take the padded path, M < tile, tails in every dimension) through every public
entry point, integer inputs (bit-exact against the oracle) and non-integer inputs (within the
1e-5 * sum |A||B| bound), C prefilled with NaN."""
import numpy as np
import pytest

import oracle
from oracle.check import check_exact
import synth

pytestmark = pytest.mark.gpu

RNG = np.random.default_rng(20261017)
SHAPES = [tuple(int(v) for v in RNG.integers(1, 700, 3)) for _ in range(14)] + [
    (1, 1, 1), (1, 700, 3), (700, 1, 5), (2, 3, 1), (257, 255, 4), (513, 4, 1023)]


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


def _inputs(M, N, K):
    A = synth.gen_matrix(M, K, synth.MATRIX_A, "d3")
    B = synth.gen_matrix(K, N, synth.MATRIX_B, "d3")
    ref, _ = oracle.gemm(A, B)
    return A, B, ref


@pytest.mark.parametrize("M,N,K", SHAPES)
def test_fuzz_host_device_sharded(giga, torch_cuda, M, N, K):
    torch = torch_cuda
    A, B, ref = _inputs(M, N, K)
    C = np.full((M, N), np.nan, np.float32)
    giga.matmul(A, B, C, M, N, K, 1)
    assert check_exact(C, ref)[0], "host"
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    dC = torch.full((M, N), float("nan"), device="cuda")
    giga.matmul(dA, dB, dC, M, N, K, 1)
    assert check_exact(dC.cpu().numpy(), ref)[0], "device"
    dC.fill_(float("nan"))
    giga.matmul_sharded([dA], [dB], [dC], M, N, K)
    assert check_exact(dC.cpu().numpy(), ref)[0], "sharded"


@pytest.mark.parametrize("M,N,K", SHAPES[:8] + [(300, 516, 2056), (1000, 260, 4100)])
@pytest.mark.parametrize("dist", ["d2", "d4"])
def test_fuzz_non_integer_within_bound(giga, torch_cuda, M, N, K, dist):
    """Non-integer inputs (the lo terms are live) through the host and device paths, C within
    1e-5 * sum |A||B| of the oracle element by element."""
    from oracle.check import check_close
    torch = torch_cuda
    A = synth.gen_matrix(M, K, synth.MATRIX_A, dist)
    B = synth.gen_matrix(K, N, synth.MATRIX_B, dist)
    ref, S = oracle.gemm(A, B)
    C = np.full((M, N), np.nan, np.float32)
    giga.matmul(A, B, C, M, N, K, 1)
    ok, st = check_close(C, ref, S)
    assert ok, ("host", st)
    dC = torch.full((M, N), float("nan"), device="cuda")
    giga.matmul_sharded([torch.from_numpy(A).cuda()], [torch.from_numpy(B).cuda()], [dC],
                        M, N, K)
    ok, st = check_close(dC.cpu().numpy(), ref, S)
    assert ok, ("sharded", st)


@pytest.mark.parametrize("M,N,K", SHAPES[:10])
def test_fuzz_forced_comm_pipeline(giga, torch_cuda, monkeypatch, M, N, K):
    torch = torch_cuda
    monkeypatch.setenv("GIGA_FORCE_COMM", "1")
    monkeypatch.setenv("GIGA_BCAST_CHUNKS", "4")
    monkeypatch.setenv("GIGA_GATHER_CHUNKS", "3")
    A, B, ref = _inputs(M, N, K)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    dC = torch.full((M, N), float("nan"), device="cuda")
    giga.matmul_sharded([dA], [dB], [dC], M, N, K)
    assert check_exact(dC.cpu().numpy(), ref)[0]


@pytest.mark.parametrize("M,N,K", [s for s in SHAPES if s[1] % 4 == 0 and s[2] % 4 == 0][:6]
                         + [(700, 256, 1024), (5, 8, 520)])
def test_fuzz_p2p_virtual(torch_cuda, monkeypatch, M, N, K):
    torch = torch_cuda
    from paper_2504_01266_b200 import giga as g
    monkeypatch.setenv("GIGA_TRANSPORT", "p2p")
    monkeypatch.setenv("GIGA_BCAST_CHUNKS", "2")
    world = 3
    g.finalize()
    g.init_devices([0] * world)
    try:
        A, B, ref = _inputs(M, N, K)
        shards = []
        for r in range(world):
            r0, rows = g.partition(M, world, r)
            shards.append(torch.from_numpy(np.ascontiguousarray(A[r0:r0 + rows])).cuda()
                          if rows else torch.empty(0, device="cuda"))
        Bs = [torch.from_numpy(B).cuda()] + [torch.empty(K, N, device="cuda")
                                             for _ in range(world - 1)]
        Cs = [torch.full((M, N), float("nan"), device="cuda") for _ in range(world)]
        g.matmul_sharded(shards, Bs, Cs, M, N, K)
        for r in range(world):
            assert check_exact(Cs[r].cpu().numpy(), ref)[0], r
    finally:
        g.finalize()
        g.init(1)


@pytest.mark.parametrize("cta_group", [1, 2])
@pytest.mark.parametrize("M,N,K", [(M, N - N % 4 or 4, K - K % 4 or 4) for M, N, K in SHAPES[:10]])
def test_fuzz_3xfp16_building_block(giga, torch_cuda, M, N, K, cta_group):
    """The 3xFP16 scheme (terms = 4) on the fuzz shapes: integer inputs bit-exact, and d5
    (full-significand floats: scales, exceptions and the fixes all live) within the bound."""
    from oracle.check import check_close
    torch = torch_cuda
    A, B, ref = _inputs(M, N, K)
    dC = torch.full((M, N), float("nan"), device="cuda")
    giga.gemm_3xtf32(torch.from_numpy(A).cuda(), None, torch.from_numpy(B).cuda(), None, dC,
                     M, N, K, terms=4, cta_group=cta_group)
    assert check_exact(dC.cpu().numpy(), ref)[0], "d3"
    A = synth.gen_matrix(M, K, synth.MATRIX_A, "d5")
    B = synth.gen_matrix(K, N, synth.MATRIX_B, "d5")
    A[::7, ::5] *= np.float32(2.0 ** -27)  # exceptions in both operands
    B[::5, ::7] *= np.float32(2.0 ** -27)
    ref, S = oracle.gemm(A, B)
    dC.fill_(float("nan"))
    giga.gemm_3xtf32(torch.from_numpy(A).cuda(), None, torch.from_numpy(B).cuda(), None, dC,
                     M, N, K, terms=4, cta_group=cta_group)
    ok, st = check_close(dC.cpu().numpy(), ref, S)
    assert ok, st


def test_fuzz_3xfp16_forced_ragged_paths(torch_cuda):
    """$GIGA_SCHEME=3xfp16 (a subprocess: the scheme is read once) through the host call and
    the padded path of the ragged fuzz shapes (K, N not multiples of 4)."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, os
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import oracle, synth
from oracle.check import check_exact
from paper_2504_01266_b200 import giga
giga.init(1)
for (M, N, K) in [(700, 301, 523), (33, 517, 1031), (513, 5, 1023), (257, 255, 4), (1, 1, 1)]:
    A = synth.gen_matrix(M, K, synth.MATRIX_A, "d3"); B = synth.gen_matrix(K, N, synth.MATRIX_B, "d3")
    ref, _ = oracle.gemm(A, B)
    C = np.full((M, N), np.nan, np.float32)
    giga.matmul(A, B, C, M, N, K, 1)
    assert check_exact(C, ref)[0], ("host", M, N, K)
    dC = torch.full((M, N), float("nan"), device="cuda")
    giga.matmul_sharded([torch.from_numpy(A).cuda()], [torch.from_numpy(B).cuda()], [dC], M, N, K)
    assert check_exact(dC.cpu().numpy(), ref)[0], ("sharded", M, N, K)
giga.finalize()
print("ok")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root,
                       env=dict(os.environ, GIGA_SCHEME="3xfp16"), capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]
