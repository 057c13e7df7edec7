"""GPU parity of the 3xFP16 scheme (terms = 4) against the CPU fp64 oracle.

The scheme is 3xTF32's split -- x = hi + lo, products a_lo b_hi + a_hi b_lo + a_hi b_hi -- on
the fp16 tensor path: TF32's 11-bit significand is fp16's, and the exponent range fp16 lacks
is moved into exact power-of-two scales per row of A and per column of B. Elements the fp16
split cannot carry to 2^-20 (those far below their row's / column's maximum) are exceptions
whose remainders the fix kernels add exactly. Bars: integer inputs bit-exact; otherwise
|C - C_ref| <= 1e-5 sum_k |A_ik||B_kj| (BASELINE.json north_star), on random data, on
constructed worst cases for the split and on inputs made of exceptions.
"""
import numpy as np
import pytest

import oracle
from oracle.check import check_close, check_exact
import synth

pytestmark = pytest.mark.gpu

SHAPES = [(1, 4, 4), (130, 260, 20), (255, 256, 16), (257, 512, 36), (600, 1000, 1028),
          (2048, 2048, 512), (4096, 4096, 4096), (512, 1536, 2048)]


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


def _run(giga, torch, A, B, cta_group=0, terms=4):
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
def test_3xfp16_bit_exact_integers(giga, torch_cuda, M, N, K, cta_group):
    """Integers in [-8, 8]: hi = x', lo = 0 after an exact power-of-two scale; bit-exact C
    (covers both k-split modes: 4096^3 reduce-adds its last wave, 512 x 1536 x 2048 runs
    workspace parts)."""
    A = synth.gen_matrix(M, K, synth.MATRIX_A, "d3")
    B = synth.gen_matrix(K, N, synth.MATRIX_B, "d3")
    C = _run(giga, torch_cuda, A, B, cta_group)
    ok, st = check_exact(C, oracle.gemm(A, B)[0])
    assert ok, st


@pytest.mark.parametrize("cta_group", [1, 2])
@pytest.mark.parametrize("M,N,K,dist", [(257, 516, 36, "d4"), (700, 900, 3000, "d1"),
                                        (600, 1000, 1028, "d2"), (1500, 2048, 4100, "d1")])
def test_3xfp16_tolerance(giga, torch_cuda, M, N, K, dist, cta_group):
    A = synth.gen_matrix(M, K, synth.MATRIX_A, dist)
    B = synth.gen_matrix(K, N, synth.MATRIX_B, dist)
    C = _run(giga, torch_cuda, A, B, cta_group)
    Cref, S = oracle.gemm(A, B)
    ok, st = check_close(C, Cref, S)
    assert ok, st
    # the corrections are there: a_lo / b_lo carry ~2^-11 of each product (plain TF32 / FP16
    # would be ~1e-4 off); what remains is the truncating TMEM accumulation
    assert st["max_rel_err"] < 2e-6, st


def test_row_and_column_scales_far_apart(giga, torch_cuda):
    """Rows of A and columns of B 2^+-50 apart: each gets its own exponent; the epilogue's
    ldexp undoes it exactly."""
    M, N, K = 512, 520, 1000
    rng = np.random.default_rng(11)
    A = (rng.uniform(-1, 1, (M, K)) * 2.0 ** rng.integers(-50, 50, (M, 1))).astype(np.float32)
    B = (rng.uniform(-1, 1, (K, N)) * 2.0 ** rng.integers(-50, 50, (1, N))).astype(np.float32)
    C = _run(giga, torch_cuda, A, B)
    Cref, S = oracle.gemm(A, B)
    ok, st = check_close(C, Cref, S)
    assert ok, st


def _exception_inputs(M, N, K, seed, a_side=True, b_side=True):
    """Each row of A holds one huge element that meets zeros of B, the rest 2^-30..2^-20 of
    it; each column of B likewise: the products that make up C are all between elements the
    fp16 split cannot carry (exceptions), so C comes from the fix kernels."""
    rng = np.random.default_rng(seed)
    A = rng.uniform(0.5, 1.0, (M, K)).astype(np.float32)
    B = rng.uniform(0.5, 1.0, (K, N)).astype(np.float32)
    if a_side:
        A *= np.float32(2.0 ** -25)
        A[:, 0] = 1.0
        B[0, :] = 0.0
    if b_side:
        B *= np.float32(2.0 ** -22)
        B[1, :] = 1.0
        A[:, 1] = 0.0
    return A, B


@pytest.mark.parametrize("a_side,b_side", [(True, False), (False, True), (True, True)])
@pytest.mark.parametrize("M,N,K", [(300, 520, 260), (1024, 1024, 2048)])
def test_exceptions_fixed(giga, torch_cuda, M, N, K, a_side, b_side):
    A, B = _exception_inputs(M, N, K, 3, a_side, b_side)
    C = _run(giga, torch_cuda, A, B)
    Cref, S = oracle.gemm(A, B)
    ok, st = check_close(C, Cref, S)
    assert ok, st
    # without the fixes these elements would be lost to fp16's subnormal floor (a relative
    # error near 1); the 3xTF32 scheme needs no fix -- both agree within the bound
    C3 = _run(giga, torch_cuda, A, B, terms=3)
    ok3, st3 = check_close(C3, Cref, S)
    assert ok3, st3


def test_sparse_exceptions_mixed_with_normal_data(giga, torch_cuda):
    """~1% of the elements 2^-24..2^-40 of their row / column maximum, scattered: the fix
    kernels handle a few per row / strip among ordinary products."""
    M, N, K = 1000, 1040, 3000
    rng = np.random.default_rng(9)
    A = rng.uniform(-1, 1, (M, K)).astype(np.float32)
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    ma = rng.random((M, K)) < 0.01
    mb = rng.random((K, N)) < 0.01
    A[ma] *= (2.0 ** -rng.integers(24, 40, ma.sum())).astype(np.float32)
    B[mb] *= (2.0 ** -rng.integers(24, 40, mb.sum())).astype(np.float32)
    C = _run(giga, torch_cuda, A, B)
    Cref, S = oracle.gemm(A, B)
    ok, st = check_close(C, Cref, S)
    assert ok, st
    # deterministic: the fixes sum in a fixed order
    C2 = _run(giga, torch_cuda, A, B)
    assert np.array_equal(C.view(np.uint32), C2.view(np.uint32))


def test_split_worst_case_at_the_exception_threshold(giga, torch_cuda):
    """The products a split error can reach without being an exception: row maximum (scaled
    to [2^15, 65504)) meeting a zero of B, the rest 2^-21..2^-18 of it (lo subnormal in fp16,
    rounded to 2^-24 steps: up to 2^-20 relative before an element becomes an exception),
    all positive so the errors add coherently. Must stay inside the bound with margin."""
    M, N, K = 256, 256, 8192
    rng = np.random.default_rng(17)
    A = (rng.uniform(2.0 ** -21, 2.0 ** -18, (M, K))).astype(np.float32)
    B = (rng.uniform(2.0 ** -21, 2.0 ** -18, (K, N))).astype(np.float32)
    A[:, 0] = 1.0
    B[0, :] = 0.0
    B[1, :] = 1.0
    A[:, 1] = 0.0
    C = _run(giga, torch_cuda, A, B)
    Cref, S = oracle.gemm(A, B)
    ok, st = check_close(C, Cref, S)
    assert ok, st
    print(f"3xFP16 threshold worst case: max {st['max_rel_err']:.3e} of the 1e-5 bound")
    assert st["max_rel_err"] < 5e-6, st


def test_non_finite_propagates(giga, torch_cuda):
    M, N, K = 256, 260, 512
    A = synth.gen_matrix(M, K, synth.MATRIX_A, "d2")
    B = synth.gen_matrix(K, N, synth.MATRIX_B, "d2")
    A[3, 7] = np.nan
    A[5, 9] = np.inf
    B[11, 13] = np.nan
    C = _run(giga, torch_cuda, A, B)
    assert np.isnan(C[3]).all()          # NaN * b is NaN for every column
    assert not np.isfinite(C[5]).any()   # Inf * b: +-Inf, or NaN (contract: Inf may turn NaN)
    assert np.isnan(C[:, 13]).all()
    ok_rows = [i for i in range(M) if i not in (3, 5)]
    ok_cols = [j for j in range(N) if j != 13]
    Cref, S = oracle.gemm(A[ok_rows], B[:, ok_cols])
    ok, st = check_close(C[np.ix_(ok_rows, ok_cols)], Cref, S)
    assert ok, st


def test_zero_rows_and_columns(giga, torch_cuda):
    M, N, K = 300, 300, 300
    A = synth.gen_matrix(M, K, synth.MATRIX_A, "d2")
    B = synth.gen_matrix(K, N, synth.MATRIX_B, "d2")
    A[10] = 0.0
    B[:, 20] = 0.0
    C = _run(giga, torch_cuda, A, B)
    assert (C[10] == 0).all() and (C[:, 20] == 0).all()
    Cref, S = oracle.gemm(A, B)
    ok, st = check_close(C, Cref, S)
    assert ok, st


_FORCED = r'''
import sys, os
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import oracle, synth
from oracle.check import check_close, check_exact
from paper_2504_01266_b200 import giga
mode = sys.argv[1]
M, N, K, dist = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
A = synth.gen_matrix(M, K, synth.MATRIX_A, dist)
B = synth.gen_matrix(K, N, synth.MATRIX_B, dist)
world = int(os.environ.get("WORLD", "1"))
giga.init_devices([0] * world)
assert giga.product_scheme(M, N, K) == 4
if mode == "host":
    C = np.full((M, N), np.nan, np.float32)
    giga.matmul(A, B, C, M, N, K, world)
    outs = [C]
else:
    shards = []
    for r in range(world):
        r0, rows = giga.partition(M, world, r)
        shards.append(torch.from_numpy(np.ascontiguousarray(A[r0:r0 + rows])).cuda() if rows
                      else torch.empty(0, device="cuda"))
    Bb = [torch.from_numpy(B).cuda()] + [torch.full((K, N), float("nan"), device="cuda")
                                         for _ in range(world - 1)]
    Cf = [torch.full((M, N), float("nan"), device="cuda") for _ in range(world)]
    giga.matmul_sharded(shards, Bb, Cf, M, N, K)
    outs = [c.cpu().numpy() for c in Cf]
Cref, S = oracle.gemm(A, B)
for C in outs:
    ok, st = check_exact(C, Cref) if dist == "d3" else check_close(C, Cref, S)
    assert ok, st
giga.finalize()
print("ok")
'''


@pytest.mark.parametrize("mode,env,M,N,K,dist", [
    ("sharded", {}, 1000, 1040, 2056, "d2"),
    ("host", {}, 1500, 1028, 4100, "d1"),
    # the N > 1 pipeline at world 1: B broadcast in K-chunks, GEMMs accumulating into C
    ("sharded", {"GIGA_FORCE_COMM": "1", "GIGA_BCAST_CHUNKS": "3", "GIGA_GATHER_CHUNKS": "3"},
     1536, 768, 2560, "d3"),
    ("sharded", {"GIGA_FORCE_COMM": "1", "GIGA_BCAST_CHUNKS": "4"}, 1000, 520, 3000, "d1"),
    # virtual GPUs, p2p transport: the last K-chunk's epilogue loads C, adds, and stores to
    # every peer's C_full (the fix kernels mirror their updates to the peers)
    ("sharded", {"WORLD": "3", "GIGA_TRANSPORT": "p2p", "GIGA_BCAST_CHUNKS": "3"},
     1031, 256, 2064, "d3"),
    ("sharded", {"WORLD": "2", "GIGA_TRANSPORT": "p2p"}, 1000, 520, 1040, "d1"),
])
def test_3xfp16_forced_through_every_path(torch_cuda, tmp_path, mode, env, M, N, K, dist):
    """$GIGA_SCHEME=3xfp16 (read once per process: a subprocess) through the paper's host call,
    the sharded call and the N > 1 orchestrations: accumulate, load-C and peer-store epilogues
    all undo the operand scales."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    e = dict(os.environ, GIGA_SCHEME="3xfp16", **env)
    r = subprocess.run([sys.executable, "-c", _FORCED, mode, str(M), str(N), str(K), dist],
                       cwd=root, env=e, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]


def test_3xfp16_exceptions_with_fused_gather(torch_cuda):
    """Exceptions on virtual GPUs with the fused gather: every GPU's C_full gets the fixed
    values (the fix kernels write the peers' copies too)."""
    import os
    import subprocess
    import sys
    code = r'''
import sys, os
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import oracle
from oracle.check import check_close
from paper_2504_01266_b200 import giga
M, N, K, world = 700, 520, 1040, 2
rng = np.random.default_rng(3)
A = rng.uniform(0.5, 1.0, (M, K)).astype(np.float32) * np.float32(2.0 ** -25)
B = rng.uniform(0.5, 1.0, (K, N)).astype(np.float32) * np.float32(2.0 ** -22)
A[:, 0] = 1.0; B[0, :] = 0.0; B[1, :] = 1.0; A[:, 1] = 0.0
giga.init_devices([0] * world)
shards = []
for r in range(world):
    r0, rows = giga.partition(M, world, r)
    shards.append(torch.from_numpy(np.ascontiguousarray(A[r0:r0 + rows])).cuda())
Bb = [torch.from_numpy(B).cuda()] + [torch.zeros((K, N), device="cuda")]
Cf = [torch.full((M, N), float("nan"), device="cuda") for _ in range(world)]
giga.matmul_sharded(shards, Bb, Cf, M, N, K)
Cref, S = oracle.gemm(A, B)
for c in Cf:
    ok, st = check_close(c.cpu().numpy(), Cref, S)
    assert ok, st
assert torch.equal(Cf[0], Cf[1])
giga.finalize()
print("ok")
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    e = dict(os.environ, GIGA_SCHEME="3xfp16", GIGA_TRANSPORT="p2p", GIGA_BCAST_CHUNKS="2")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=e, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]
