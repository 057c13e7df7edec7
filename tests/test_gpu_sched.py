"""The GEMM beside co-running kernels (VERDICT r1 "make the GEMM correct and fast beside
co-running kernels"; DESIGN.md 6.3 "Dynamic schedule").

In the NCCL pipeline the persistent GEMM is launched on 148 - k SMs while NCCL's CTAs run
beside it; if those CTAs sit on k different TPCs, up to k/2 of the GEMM's CTA pairs cannot be
resident until NCCL finishes. With static round-robin units, every wave then waited for the
missing clusters' units (up to 2 ms per wave). With units claimed dynamically the resident
clusters take all the work. Here an occupier kernel (libgiga_debug.so) holds k SMs for a
while; the GEMM must give bit-identical C and lose no more time than the SMs it was denied.
"""
import ctypes
import os

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def env():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2504_01266_b200 import build
    build.build()
    dbg = ctypes.CDLL(os.path.join(ROOT, "paper_2504_01266_b200", "libgiga_debug.so"))
    dbg.giga_dbg_occupy.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p,
                                    ctypes.c_void_p]
    dbg.giga_dbg_gemm_max_ctas.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                           ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
    return torch, dbg


def _gemm(torch, dbg, A, B, C, terms, max_ctas, stream):
    M, K = A.shape
    N = B.shape[1]
    rc = dbg.giga_dbg_gemm_max_ctas(A.data_ptr(), B.data_ptr(), C.data_ptr(), M, N, K, terms,
                                    max_ctas, stream.cuda_stream)
    assert rc == 0


def _timed_gemm(torch, dbg, A, B, C, terms, max_ctas, stream):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    _gemm(torch, dbg, A, B, C, terms, max_ctas, stream)
    e1.record(stream)
    return e0, e1


@pytest.mark.parametrize("terms,size", [(2, 16384), (3, 8192)])
def test_gemm_beside_an_occupier(env, terms, size):
    torch, dbg = env
    M = N = K = size
    A = synth.gen_rows_torch(0, M, K, synth.MATRIX_A, "d3", device="cuda")
    B = synth.gen_rows_torch(0, K, N, synth.MATRIX_B, "d3", device="cuda")
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    s_gemm, s_occ = torch.cuda.Stream(), torch.cuda.Stream()
    results = {}
    for k in (2, 8, 16):
        max_ctas = nsm - k
        C0 = torch.full((M, N), float("nan"), device="cuda")
        for _ in range(2):  # warm (workspaces, counters), then the unobstructed reference time
            torch.cuda.synchronize()
            e0, e1 = _timed_gemm(torch, dbg, A, B, C0, terms, max_ctas, s_gemm)
            e1.synchronize()
        t0 = e0.elapsed_time(e1)
        C = torch.full((M, N), float("nan"), device="cuda")
        smids = torch.full((k,), -1, dtype=torch.int32, device="cuda")
        occ_ms = 0.6 * t0
        torch.cuda.synchronize()
        # the occupier first (each CTA alone on an SM: 120 KiB of shared memory), then the GEMM
        assert dbg.giga_dbg_occupy(k, 120 * 1024, int(occ_ms * 1e6), smids.data_ptr(),
                                   s_occ.cuda_stream) == 0
        import time
        time.sleep(0.002)
        e0, e1 = _timed_gemm(torch, dbg, A, B, C, terms, max_ctas, s_gemm)
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1)
        sm = smids.cpu().numpy()
        assert (sm >= 0).all()
        tpcs = len(set((sm // 2).tolist()))
        # pairs the GEMM wants vs pairs free while the occupier runs (one CTA pair per TPC)
        want = max_ctas // 2
        lost = max(0, want - (nsm // 2 - tpcs))
        allowed = (t0 + occ_ms * lost / want) * 1.05 + 0.05
        assert torch.equal(C, C0), f"k={k}: C differs from the unobstructed launch"
        results[k] = {"t_unobstructed_ms": round(t0, 3), "t_ms": round(t, 3), "tpcs": tpcs,
                      "lost_pairs": lost, "allowed_ms": round(allowed, 3)}
        assert t <= allowed, results
    print(f"terms={terms} {size}^3:", results)


def test_concurrent_launches_on_two_streams(env):
    """Two GEMMs on two streams of one device at once (virtual GPUs, concurrent callers):
    each launch has its own schedule counters, both results bit-identical to serial runs."""
    torch, dbg = env
    M = N = K = 4096
    A = synth.gen_rows_torch(0, M, K, synth.MATRIX_A, "d3", device="cuda")
    B = synth.gen_rows_torch(0, K, N, synth.MATRIX_B, "d3", device="cuda")
    A2 = synth.gen_rows_torch(0, M, K, 7, "d3", device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    ref1 = torch.empty((M, N), device="cuda")
    ref2 = torch.empty((M, N), device="cuda")
    # the inputs were generated on the default stream; torch's side streams do not wait for it
    torch.cuda.synchronize()
    _gemm(torch, dbg, A, B, ref1, 3, 0, s1)
    _gemm(torch, dbg, A2, B, ref2, 3, 0, s1)
    torch.cuda.synchronize()
    for rep in range(3):
        C1 = torch.full((M, N), float("nan"), device="cuda")
        C2 = torch.full((M, N), float("nan"), device="cuda")
        torch.cuda.synchronize()
        _gemm(torch, dbg, A, B, C1, 3, 0, s1)
        _gemm(torch, dbg, A2, B, C2, 3, 0, s2)
        torch.cuda.synchronize()
        assert torch.equal(C1, ref1) and torch.equal(C2, ref2), rep
    Cref, _ = oracle.gemm(synth.gen_rows(5, 1, K, synth.MATRIX_A, "d3"),
                          synth.gen_rows_torch(0, K, N, synth.MATRIX_B, "d3", device="cpu").numpy())
    assert np.array_equal(ref1[5].cpu().numpy().astype(np.float64), Cref[0])
