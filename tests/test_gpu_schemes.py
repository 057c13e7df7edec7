"""GPU parity of the fp32-accurate schemes of the shard GEMM against the CPU fp64 oracle.

terms = 3: 3xTF32 (BASELINE north_star (3); the product scheme for small and skinny launches).
terms = 2: TF32 + BF16 -- a_hi*b_hi as one kind::tf32 MMA plus both corrections as one K=16
kind::f16 MMA over [bf16(a_lo) | bf16(a_hi)] . [bf16(b) ; bf16(b_lo)] (gemm_3xtf32.cu,
DESIGN.md 6.7; the product scheme for large launches, giga_product_scheme). Its split error is <= 3 * 2^-19 |a||b| (5.7e-6) per product with the RN hi
(the library default; 5.3e-6 reached by constructed inputs, tests/test_gpu_fullc.py), inside
the 1e-5 * sum|A||B| bound (R5) with the accumulation error on top.
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


_CHILD = """
import os, numpy as np, torch, oracle, synth
from oracle.check import check_close, check_exact
from paper_2504_01266_b200 import giga
giga.init(1)
M, N, K = 4096, 1040, 2064  # host schedule: 4 late row blocks
dist = os.environ["CHILD_DIST"]
A = synth.gen_matrix(M, K, synth.MATRIX_A, dist); B = synth.gen_matrix(K, N, synth.MATRIX_B, dist)
ref, S = oracle.gemm(A, B)
def check(C, what):
    ok, st = check_exact(C, ref) if dist == "d3" else check_close(C, ref, S)
    assert ok, (what, st)
dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
dC = torch.full((M, N), float("nan"), device="cuda")
giga.matmul_sharded([dA], [dB], [dC], M, N, K)
check(dC.cpu().numpy(), "sharded")
C = np.full((M, N), np.nan, np.float32)
giga.matmul(A, B, C, M, N, K, 1)  # host buffers: K-chunks, then row blocks reusing B's prep
check(C, "host")
giga.finalize()
print("ok")
"""


@pytest.mark.parametrize("dist", ["d1", "d3"])
@pytest.mark.parametrize("env", [{}, {"GIGA_FORCE_COMM": "1", "GIGA_BCAST_CHUNKS": "3",
                                      "GIGA_GATHER_CHUNKS": "3"}, {"GIGA_A_PRE": "0"},
                                 {"GIGA_B_PRE": "0"}])
def test_scheme_through_the_product_paths(dist, env):
    """GIGA_SCHEME=tf32bf16 forces terms = 2 on every product launch: the device-resident
    call, the host-buffer schedule (late row blocks reuse the prepared B: b_prep_reuse) and,
    with GIGA_FORCE_COMM, the NCCL pipeline at world 1 (K-chunks accumulating, the last in row
    chunks reusing B's preparation); also with A' / B' built on chip. Child processes: the
    environment is read once per process."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    penv = dict(os.environ, GIGA_SCHEME="tf32bf16", PYTHONPATH=root, CHILD_DIST=dist, **env)
    r = subprocess.run([sys.executable, "-c", _CHILD], env=penv, cwd=root, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


_CHILD_P2P = """
import os, numpy as np, torch, oracle, synth
from oracle.check import check_close, check_exact
from paper_2504_01266_b200 import giga
giga.init_devices([0, 0, 0])
M, N, K = 1500, 1040, 2064
dist = os.environ["CHILD_DIST"]
A = synth.gen_matrix(M, K, synth.MATRIX_A, dist); B = synth.gen_matrix(K, N, synth.MATRIX_B, dist)
ref, S = oracle.gemm(A, B)
shards, Bs, Cs = [], [], []
for g in range(3):
    r0, rows = giga.partition(M, 3, g)
    shards.append(torch.from_numpy(A[r0:r0 + rows]).cuda())
    Bs.append(torch.from_numpy(B).cuda() if g == 0 else torch.empty((K, N), device="cuda"))
    Cs.append(torch.full((M, N), float("nan"), device="cuda"))
for rep in range(2):
    giga.matmul_sharded(shards, Bs, Cs, M, N, K)
    for g, C in enumerate(Cs):
        C = C.cpu().numpy()
        ok, st = check_exact(C, ref) if dist == "d3" else check_close(C, ref, S)
        assert ok, (rep, g, st)
giga.finalize()
print("ok")
"""


@pytest.mark.parametrize("dist", ["d1", "d3"])
def test_scheme_through_the_p2p_transport(dist):
    """TF32 + BF16 forced on the peer-to-peer transport over 3 virtual GPUs of device 0:
    K-chunked GEMMs accumulating, the last chunk's epilogue loading the local partial and
    storing the final rows into every GPU's C_full (the fused gather), twice."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    penv = dict(os.environ, GIGA_SCHEME="tf32bf16", GIGA_TRANSPORT="p2p", PYTHONPATH=root,
                CHILD_DIST=dist)
    r = subprocess.run([sys.executable, "-c", _CHILD_P2P], env=penv, cwd=root,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


_CHILD_REUSE = """
import numpy as np, torch, oracle, synth
from oracle.check import check_exact
from paper_2504_01266_b200 import giga
giga.init(1)
M, N, K = 4096, 1040, 2064
A = synth.gen_matrix(M, K, synth.MATRIX_A, "d3")
B1 = synth.gen_matrix(K, N, synth.MATRIX_B, "d3")
B2 = synth.gen_matrix(K, N, 7, "d3")
dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B1).cuda()
dC = torch.full((M, N), float("nan"), device="cuda")
for Bh in (B1, B2, B1):
    dB.copy_(torch.from_numpy(Bh))  # same pointer, new contents: B is prepared again
    giga.matmul_sharded([dA], [dB], [dC], M, N, K)
    ok, st = check_exact(dC.cpu().numpy(), oracle.gemm(A, Bh)[0])
    assert ok, st
    C = np.full((M, N), np.nan, np.float32)
    giga.matmul(A, Bh, C, M, N, K, 1)  # host path: B staged into the same device buffer
    ok, st = check_exact(C, oracle.gemm(A, Bh)[0])
    assert ok, st
giga.finalize()
print("ok")
"""


@pytest.mark.parametrize("env", [{}, {"GIGA_FORCE_COMM": "1", "GIGA_BCAST_CHUNKS": "3",
                                      "GIGA_GATHER_CHUNKS": "3"}])
def test_b_preparation_is_not_reused_across_calls(env):
    """B's prepared operands are reused only between launches of one product (row chunks /
    row blocks); a later call with the same B pointer but new contents must prepare again."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    penv = dict(os.environ, GIGA_SCHEME="tf32bf16", PYTHONPATH=root, **env)
    r = subprocess.run([sys.executable, "-c", _CHILD_REUSE], env=penv, cwd=root,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


@pytest.mark.parametrize("M,N,K", [(8192, 8192, 2048), (1536, 1040, 1028)])
def test_rank_api_in_a_cuda_graph(torch_cuda, M, N, K):
    """giga_matmul_rank is stream-ordered, so a step can be captured into a CUDA graph and
    replayed (launch-bound inner loops). One eager call first sizes the library's per-stream
    workspaces; the captured launches then reuse them (8192 x 8192 x 2048 runs the prepared
    TF32 + BF16 scheme, 1536 x 1040 x 1028 3xTF32). Replays with new A contents: bit-exact."""
    torch = torch_cuda
    from paper_2504_01266_b200 import giga as g
    g.finalize()
    g.rank_init(0, 1, 0, None)
    try:
        B = synth.gen_matrix(K, N, synth.MATRIX_B, "d3")
        dB = torch.from_numpy(B).cuda()
        dA = torch.empty((M, K), device="cuda")
        dC = torch.full((M, N), float("nan"), device="cuda")
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        A0 = synth.gen_matrix(M, K, synth.MATRIX_A, "d3")
        dA.copy_(torch.from_numpy(A0))
        torch.cuda.synchronize()
        g.matmul_rank(dA, dB, dC, M, N, K, stream=s)  # eager: workspaces sized
        s.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            g.matmul_rank(dA, dB, dC, M, N, K, stream=s)
        rows = np.array(sorted({0, M - 1, M // 2} | set(range(1, M, max(1, M // 61)))))
        for seed in (3, 5):
            A = synth.gen_matrix(M, K, seed, "d3")
            dA.copy_(torch.from_numpy(A))
            dC.fill_(float("nan"))
            torch.cuda.synchronize()
            graph.replay()
            torch.cuda.synchronize()
            ok, st = check_exact(dC.cpu().numpy()[rows], oracle.gemm(A[rows], B)[0])
            assert ok, (seed, st)
            assert not torch.isnan(dC).any().item()
    finally:
        g.finalize()


def test_graph_survives_workspace_growth(torch_cuda):
    """A graph captured at one shape keeps raw pointers to the per-stream workspaces (TF32 +
    BF16 prepared operands); a later eager call with a larger shape on the same stream grows
    them. The superseded buffers must stay allocated until giga_finalize, so
    replaying the older graph is still correct (the freed memory is scribbled over first)."""
    torch = torch_cuda
    from paper_2504_01266_b200 import giga as g
    g.finalize()
    g.rank_init(0, 1, 0, None)
    try:
        M, N, K = 8192, 8192, 2048
        B = synth.gen_matrix(K, N, synth.MATRIX_B, "d3")
        dB = torch.from_numpy(B).cuda()
        A = synth.gen_matrix(M, K, synth.MATRIX_A, "d3")
        dA = torch.from_numpy(A).cuda()
        dC = torch.full((M, N), float("nan"), device="cuda")
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        torch.cuda.synchronize()
        g.matmul_rank(dA, dB, dC, M, N, K, stream=s)
        s.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            g.matmul_rank(dA, dB, dC, M, N, K, stream=s)
        # a larger product on the same stream grows the prepared-operand scratch
        M2, K2 = 12288, 4096
        dA2 = torch.ones((M2, K2), device="cuda")
        dB2 = torch.ones((K2, N), device="cuda")
        dC2 = torch.empty((M2, N), device="cuda")
        g.matmul_rank(dA2, dB2, dC2, M2, N, K2, stream=s)
        s.synchronize()
        assert float(dC2[0, 0]) == K2
        junk = torch.full((3 << 30,), 7.0, device="cuda")  # reuse any freed memory
        torch.cuda.synchronize()
        dC.fill_(float("nan"))
        torch.cuda.synchronize()
        graph.replay()
        torch.cuda.synchronize()
        del junk
        rows = np.array(sorted({0, M - 1} | set(range(1, M, 97))))
        ok, st = check_exact(dC.cpu().numpy()[rows], oracle.gemm(A[rows], B)[0])
        assert ok, st
    finally:
        g.finalize()
