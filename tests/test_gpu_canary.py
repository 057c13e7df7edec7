"""Canary guard bands ("results land only in their slot"): every
C buffer the library writes -- the shard's rows of C_full on each GPU, the peers' copies the
fused gather writes over NVLink, C with a row stride wider than N, host C -- sits inside a
larger allocation whose surrounding rows and columns hold a NaN with a marked payload. After
the call the inner region must hold the oracle's result and every canary word must be
bit-for-bit unchanged; the inputs (A, B and B's receive buffers after the broadcast) must not
be modified either. PAPER.md:291 (S4.2.7): each element is assigned once, in its own slot.
"""
import numpy as np
import pytest

import oracle
from oracle.check import check_close, check_exact
import synth

pytestmark = pytest.mark.gpu
CANARY = 0x7FC0DEAD  # a quiet NaN with a payload no computation produces
G = 8                # guard rows above and below; guard columns when the stride allows


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


@pytest.fixture
def lib(torch_cuda):
    from paper_2504_01266_b200 import build
    build.build()
    from paper_2504_01266_b200 import giga as g
    made = []

    def make(devices):
        g.finalize()
        g.init_devices(devices)
        made.append(devices)
        return g

    yield make
    g.finalize()


def _guarded(torch, rows, cols, ld):
    """(outer buffer filled with the canary, inner rows x cols view with row stride ld)."""
    outer = torch.full(((rows + 2 * G) * ld,), CANARY, dtype=torch.int32, device="cuda")
    inner = outer.view(torch.float32)[G * ld:(G + rows) * ld].view(rows, ld)[:, :cols]
    return outer, inner


def _inner_mask(rows, cols, ld):
    m = np.zeros(((rows + 2 * G), ld), bool)
    m[G:G + rows, :cols] = True
    return m.ravel()


def _check_canary(outer, rows, cols, ld, what):
    bits = outer.cpu().numpy().view(np.uint32)
    guard = bits[~_inner_mask(rows, cols, ld)]
    bad = int(np.count_nonzero(guard != CANARY))
    assert bad == 0, f"{what}: {bad} canary words overwritten"


@pytest.mark.parametrize("M,N,K,dist", [(1000, 520, 1040, "d3"),   # ragged, 1-CTA tiles
                                        (4096, 4096, 4096, "d3"),  # k-split reduce (3 waves + 34)
                                        (512, 1536, 2048, "d2"),   # k-split workspace
                                        (8192, 8192, 2048, "d5")])  # the 3xFP16 product scheme
def test_sharded_one_gpu_guard_rows(lib, torch_cuda, M, N, K, dist):
    torch = torch_cuda
    giga = lib([0])
    A = synth.gen_matrix(M, K, synth.MATRIX_A, dist)
    B = synth.gen_matrix(K, N, synth.MATRIX_B, dist)
    a_out, dA = _guarded(torch, M, K, K)
    b_out, dB = _guarded(torch, K, N, N)
    dA.copy_(torch.from_numpy(A))
    dB.copy_(torch.from_numpy(B))
    a_before, b_before = a_out.clone(), b_out.clone()
    c_out, dC = _guarded(torch, M, N, N)
    giga.matmul_sharded([dA], [dB], [dC], M, N, K)
    torch.cuda.synchronize()
    _check_canary(c_out, M, N, N, "C_full")
    assert torch.equal(a_out, a_before) and torch.equal(b_out, b_before), "inputs modified"
    Cref, S = oracle.gemm(A, B)
    C = dC.cpu().numpy()
    ok, st = check_exact(C, Cref) if dist == "d3" else check_close(C, Cref, S)
    assert ok, st


@pytest.mark.parametrize("terms", [3, 2, 4])
@pytest.mark.parametrize("M,N,K", [(700, 900, 1000), (2048, 2048, 2048)])
def test_gemm_building_block_guard_columns(lib, torch_cuda, terms, M, N, K):
    """giga_gemm_3xtf32_ex with ldc = N + 64: the 64 columns right of C in every row and the
    rows above / below are canaries (the TMA store clips to N columns, M rows)."""
    torch = torch_cuda
    giga = lib([0])
    ldc = N + 64
    A = synth.gen_matrix(M, K, synth.MATRIX_A, "d3")
    B = synth.gen_matrix(K, N, synth.MATRIX_B, "d3")
    c_out, dC = _guarded(torch, M, N, ldc)
    # dC is a strided view (ldc > N): pass its address (the binding takes contiguous tensors)
    giga.gemm_3xtf32(torch.from_numpy(A).cuda(), None, torch.from_numpy(B).cuda(), None,
                     dC.data_ptr(), M, N, K, ldc=ldc, terms=terms)
    torch.cuda.synchronize()
    _check_canary(c_out, M, N, ldc, f"C (terms {terms})")
    Cref, _ = oracle.gemm(A, B)
    ok, st = check_exact(dC.cpu().numpy(), Cref)
    assert ok, st


@pytest.mark.parametrize("world,M,N,K", [(2, 1000, 520, 1040), (3, 1031, 256, 2064),
                                         (4, 2048, 512, 1024)])
def test_fused_gather_guard_rows_every_gpu(lib, torch_cuda, monkeypatch, world, M, N, K):
    """p2p transport on virtual GPUs: each GPU's C_full receives its own rows from its GEMM and
    every other GPU's rows from the peers' epilogues; B's receive buffers get the broadcast."""
    torch = torch_cuda
    monkeypatch.setenv("GIGA_TRANSPORT", "p2p")
    monkeypatch.setenv("GIGA_BCAST_CHUNKS", "3")
    giga = lib([0] * world)
    A = synth.gen_matrix(M, K, synth.MATRIX_A, "d3")
    B = synth.gen_matrix(K, N, synth.MATRIX_B, "d3")
    A_sh, a_guard = [], []
    for r in range(world):
        r0, rows = giga.partition(M, world, r)
        o, v = _guarded(torch, max(rows, 1), K, K)
        if rows:
            v.copy_(torch.from_numpy(np.ascontiguousarray(A[r0:r0 + rows])))
        A_sh.append(v[:rows] if rows else torch.empty(0, device="cuda"))
        a_guard.append((o, o.clone()))
    b_guard, B_bufs = [], []
    for r in range(world):
        o, v = _guarded(torch, K, N, N)
        if r == 0:
            v.copy_(torch.from_numpy(B))
        b_guard.append(o)
        B_bufs.append(v)
    c_guard, C_full = [], []
    for r in range(world):
        o, v = _guarded(torch, M, N, N)
        c_guard.append(o)
        C_full.append(v)
    giga.matmul_sharded(A_sh, B_bufs, C_full, M, N, K)
    torch.cuda.synchronize()
    Cref, _ = oracle.gemm(A, B)
    for r in range(world):
        _check_canary(c_guard[r], M, N, N, f"C_full of GPU {r}")
        _check_canary(b_guard[r], K, N, N, f"B buffer of GPU {r}")
        assert torch.equal(a_guard[r][0], a_guard[r][1]), f"A shard of GPU {r} modified"
        ok, st = check_exact(C_full[r].cpu().numpy(), Cref)
        assert ok, (r, st)


def test_host_api_guard_rows(lib, torch_cuda):
    """giga_matmul with host buffers: C is the middle of a larger host array."""
    giga = lib([0])
    M, N, K = 1000, 516, 1040
    A = synth.gen_matrix(M, K, synth.MATRIX_A, "d3")
    B = synth.gen_matrix(K, N, synth.MATRIX_B, "d3")
    outer = np.full((M + 2 * G) * N, CANARY, np.uint32)
    C = outer.view(np.float32)[G * N:(G + M) * N].reshape(M, N)
    giga.matmul(A, B, C, M, N, K, 1)
    mask = _inner_mask(M, N, N)
    assert int(np.count_nonzero(outer[~mask] != CANARY)) == 0, "host canaries overwritten"
    Cref, _ = oracle.gemm(A, B)
    ok, st = check_exact(C, Cref)
    assert ok, st
