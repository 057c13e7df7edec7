"""Whole-C and worst-case parity at the BASELINE sizes ("harden parity").

* Freivalds' check of EVERY element of C at 4096^3, the tall 262144 x 1024^2, 16384^3 and
  32768^3 on integer inputs (synth d3),
  through bench.py's launch path: for random integer vectors r, C r == A (B r) exactly. All
  partial sums are integers below 2^53, so fp64 matrix-vector products are exact whatever
  their summation order; a single wrong element of C changes C r unless r's entry at its
  column is 0 (probability 1/2049 per vector; two vectors are used).
* Constructed worst cases (tests/adversarial.py), each scheme on the inputs where its split
  is least accurate and undershoots, so every product's error has the same sign as the
  truncating TMEM accumulation's: the product path's 3xFP16 (every row of A / column of B:
  its maximum 1.0 meeting a zero of the other operand, every other element at 2^-20 of it
  with a split error just under the exception threshold: ~2 * 2^-20 per product), and the
  TF32 + BF16 and 3xTF32 building blocks (rows / columns constant at the (a, b) pairs of
  largest TF32 + BF16 split error, 5.1-5.3e-6). Expected value: a closed form exact in fp64
  (C_ij = K' a_i b_j, S_ij the same). Asserted <= 1e-5 S; the margins are printed and
  written to gpurun_out/adversarial.json.
"""
import json
import os

import numpy as np
import pytest

import adversarial as adv
import synth

pytestmark = pytest.mark.gpu
OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


def _freivalds(torch, A, B, C, seeds=(11, 12)):
    """max |C r - A (B r)| over the seeded integer vectors r (0 means every element of C is
    consistent with A B). A, B, C fp32 CUDA tensors with integer values; fp64 products in row
    chunks (exact: every partial sum is an integer below 2^53)."""
    K, N = B.shape
    worst = 0.0
    for sd in seeds:
        g = torch.Generator(device="cpu").manual_seed(sd)
        r = torch.randint(-1024, 1025, (N,), generator=g, dtype=torch.int64).to(
            device=C.device, dtype=torch.float64)
        Br = torch.empty(K, dtype=torch.float64, device=C.device)
        for k0 in range(0, K, 4096):
            Br[k0:k0 + 4096] = B[k0:k0 + 4096].double() @ r
        for m0 in range(0, C.shape[0], 4096):
            lhs = C[m0:m0 + 4096].double() @ r
            rhs = A[m0:m0 + 4096].double() @ Br
            worst = max(worst, float((lhs - rhs).abs().max()))
            del lhs, rhs
    return worst


@pytest.mark.parametrize("M,N,K", [(4096, 4096, 4096), (262144, 1024, 1024),
                                   (16384, 16384, 16384), (32768, 32768, 32768)])
def test_freivalds_whole_c_integer_inputs(torch_cuda, M, N, K):
    """Every element of C at full size, through bench.py's path (rank API at world 1 on a
    side stream, device-resident inputs, repeated calls), on d3 integer inputs (bit-exact bar:
    K * 8 * 8 <= 2^21, so every fp32 partial sum is exact)."""
    torch = torch_cuda
    from paper_2504_01266_b200 import giga as g
    g.finalize()
    g.rank_init(0, 1, 0, None)
    try:
        A = synth.gen_rows_torch(0, M, K, synth.MATRIX_A, "d3", device="cuda")
        B = synth.gen_rows_torch(0, K, N, synth.MATRIX_B, "d3", device="cuda")
        C = torch.full((M, N), float("nan"), device="cuda")
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        for _ in range(2):
            g.matmul_rank(A, B, C, M, N, K, stream=s)
        s.synchronize()
        assert not torch.isnan(C).any().item()
        assert g.product_scheme(M, N, K) == 4  # the 3xFP16 product path at every size here
        worst = _freivalds(torch, A, B, C)
        assert worst == 0.0, worst
        # the check itself: one wrong element anywhere must be caught
        C[M - 3, 17] += 1.0
        assert _freivalds(torch, A, B, C) > 0.0
    finally:
        g.finalize()


_ADV_SHAPES = {2048: (8192, 8192, 2048), 8192: (4096, 8192, 8192), 32768: (4096, 8192, 32768)}


@pytest.mark.parametrize("K", sorted(_ADV_SHAPES))
def test_constructed_worst_cases(torch_cuda, K):
    torch = torch_cuda
    from paper_2504_01266_b200 import giga as g
    M, N, _ = _ADV_SHAPES[K]
    assert g.product_scheme(M, N, K) == 4
    out = {}
    # the 3xFP16 product path: A rows [1, 0, x, x, ...], B columns [0, 1, x, x, ...]^T
    x = adv.FP16_WORST_X
    A = torch.full((M, K), x, dtype=torch.float32, device="cuda")
    A[:, 0] = adv.FP16_ROW_MAX
    A[:, 1] = 0.0
    B = torch.full((K, N), x, dtype=torch.float32, device="cuda")
    B[0, :] = 0.0
    B[1, :] = adv.FP16_ROW_MAX
    exact = (K - 2) * float(np.float64(x) * np.float64(x))
    g.finalize()
    g.init(1)
    try:
        C = torch.full((M, N), float("nan"), device="cuda")
        g.matmul_sharded([A], [B], [C], M, N, K)
        torch.cuda.synchronize()
        rel = (C.double() - exact) / exact
        out["product_3xfp16"] = {"max_rel": float(rel.abs().max()),
                                 "mean_signed_rel": float(rel.mean()),
                                 "margin_to_1e-5": 1e-5 - float(rel.abs().max()),
                                 "split_error_emulated": 2 * adv.split16_rel_error(x)}
        del A, B, C, rel
    finally:
        g.finalize()
    pairs = adv.WORST_PAIRS
    avals = torch.tensor([p[0] for p in pairs], dtype=torch.float32, device="cuda")
    b = float(np.float32(pairs[0][1]))
    assert all(float(np.float32(p[1])) == b for p in pairs)
    A = avals[torch.arange(M, device="cuda") % len(pairs)].unsqueeze(1).expand(M, K).contiguous()
    B = torch.full((K, N), b, dtype=torch.float32, device="cuda")
    exact = (K * b) * A[:, :1].double()  # C_ij = K a_i b, exact in fp64; S_ij equal (all > 0)
    g.finalize()
    g.init(1)
    try:
        for label, terms in (("tf32bf16", 2), ("3xtf32", 3)):
            C = torch.full((M, N), float("nan"), device="cuda")
            g.gemm_3xtf32(A, None, B, None, C, M, N, K, terms=terms)
            torch.cuda.synchronize()
            rel = ((C.double() - exact) / exact)
            out[label] = {"max_rel": float(rel.abs().max()), "mean_signed_rel": float(rel.mean()),
                          "margin_to_1e-5": 1e-5 - float(rel.abs().max())}
            del C, rel
    finally:
        g.finalize()
    out["split_error_emulated"] = [p[2] for p in pairs]
    os.makedirs(OUT, exist_ok=True)
    path = os.path.join(OUT, "adversarial.json")
    allres = json.load(open(path)) if os.path.exists(path) else {}
    allres[f"{M}x{N}x{K}"] = out
    with open(path, "w") as f:
        json.dump(allres, f, indent=1)
    print(f"adversarial {M}x{N}x{K}: {out}")
    assert out["product_3xfp16"]["max_rel"] <= 1e-5, out
    assert out["tf32bf16"]["max_rel"] <= 1e-5, out
    assert out["3xtf32"]["max_rel"] <= 1e-5, out
