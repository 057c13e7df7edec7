"""Small GEMM / split / dot calls for compute-sanitizer runs (memcheck, racecheck, synccheck,
initcheck): every scheme (3xTF32, TF32 + BF16, 3xFP16 with exceptions), both tile variants,
the host-buffer path, the dot product and the peer-to-peer transport."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2504_01266_b200 import giga

giga.init(1)
for (M, N, K) in [(300, 260, 1028), (129, 300, 9), (600, 512, 512)]:
    A = synth.gen_matrix(M, K, 1, "d3"); B = synth.gen_matrix(K, N, 2, "d3")
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    dC = torch.full((M, N), float("nan"), device="cuda")
    giga.matmul(dA, dB, dC, M, N, K, 1)
    C = np.empty((M, N), np.float32)
    giga.matmul(A, B, C, M, N, K, 1)
    assert np.array_equal(C, dC.cpu().numpy())
# lo computed in shared memory (transform warps) vs TMA-loaded pre-split lo, both tile
# variants, non-integer inputs (so lo != 0): bit-identical
M, N, K = 520, 516, 1040
dA = torch.from_numpy(synth.gen_matrix(M, K, 1, "d2")).cuda()
dB = torch.from_numpy(synth.gen_matrix(K, N, 2, "d2")).cuda()
dAlo, dBlo = torch.empty_like(dA), torch.empty_like(dB)
giga.split_lo(dA, dAlo); giga.split_lo(dB, dBlo)
for cg in (1, 2):
    C1 = torch.empty((M, N), device="cuda"); C2 = torch.empty((M, N), device="cuda")
    giga.gemm_3xtf32(dA, None, dB, None, C1, M, N, K, cta_group=cg)
    giga.gemm_3xtf32(dA, dAlo, dB, dBlo, C2, M, N, K, cta_group=cg)
    torch.cuda.synchronize()
    assert torch.equal(C1, C2), cg
# TF32 + BF16 scheme: operands prepared in HBM (prep kernels; direct TMA -> MMA barrier), and
# with A' / B' built on chip by the transform warps (GIGA_A_PRE / GIGA_B_PRE are read once,
# so the on-chip variants run in sanitize_t2_onchip.py); integer inputs give exact results
M, N, K = 520, 516, 1040
Ai = synth.gen_matrix(M, K, 1, "d3"); Bi = synth.gen_matrix(K, N, 2, "d3")
dAi, dBi = torch.from_numpy(Ai).cuda(), torch.from_numpy(Bi).cuda()
ref = torch.from_numpy(Ai.astype(np.float64) @ Bi.astype(np.float64)).float().cuda()
for cg in (1, 2):
    C3 = torch.full((M, N), float("nan"), device="cuda")
    giga.gemm_3xtf32(dAi, None, dBi, None, C3, M, N, K, terms=2, cta_group=cg)
    torch.cuda.synchronize()
    assert torch.equal(C3, ref), ("terms 2", cg)
# 3xFP16 (terms 4): scaled fp16 operands prepared in HBM, f16 MMAs, exception bitmaps, the
# B-side fix in the epilogue (per-strip lists) and the A-side fix kernel: integer inputs exact;
# inputs made of exceptions (each row's / column's maximum meets the other operand's zeros)
for cg in (1, 2):
    C4 = torch.full((M, N), float("nan"), device="cuda")
    giga.gemm_3xtf32(dAi, None, dBi, None, C4, M, N, K, terms=4, cta_group=cg)
    torch.cuda.synchronize()
    assert torch.equal(C4, ref), ("terms 4", cg)
rng = np.random.default_rng(3)
Ae = rng.uniform(0.5, 1.0, (M, K)).astype(np.float32) * np.float32(2.0 ** -25)
Be = rng.uniform(0.5, 1.0, (K, N)).astype(np.float32) * np.float32(2.0 ** -22)
Ae[:, 0] = 1.0; Be[0, :] = 0.0; Be[1, :] = 1.0; Ae[:, 1] = 0.0
Be[5:9, 3] *= np.float32(2.0 ** -30)  # a few list entries in strip 0 next to the heavy ones
C4 = torch.full((M, N), float("nan"), device="cuda")
giga.gemm_3xtf32(torch.from_numpy(Ae).cuda(), None, torch.from_numpy(Be).cuda(), None, C4,
                 M, N, K, terms=4)
torch.cuda.synchronize()
ex = Ae.astype(np.float64) @ Be.astype(np.float64)
S = np.abs(Ae.astype(np.float64)) @ np.abs(Be.astype(np.float64))
assert np.all(np.abs(C4.cpu().numpy() - ex) <= 1e-5 * S), "terms 4 exceptions"
x = synth.gen_vector(100003, 3, "d3"); y = synth.gen_vector(100003, 4, "d3")
print("dot", giga.dot(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()))
giga.finalize()
# peer-to-peer transport on 3 virtual GPUs of device 0: copy-engine chain for B, C gather
# fused into the GEMM epilogue (TMA stores into every virtual GPU's C_full)
os.environ["GIGA_TRANSPORT"] = "p2p"
giga.init_devices([0, 0, 0])
M, N, K = 700, 260, 1040
A = synth.gen_matrix(M, K, 1, "d3"); B = synth.gen_matrix(K, N, 2, "d3")
shards, Bs, Cs = [], [], []
for gi in range(3):
    r0, rows = giga.partition(M, 3, gi)
    shards.append(torch.from_numpy(A[r0:r0 + rows]).cuda())
    Bs.append(torch.from_numpy(B).cuda() if gi == 0 else torch.empty((K, N), device="cuda"))
    Cs.append(torch.full((M, N), float("nan"), device="cuda"))
giga.matmul_sharded(shards, Bs, Cs, M, N, K)
ref = torch.from_numpy(A.astype(np.float64) @ B.astype(np.float64)).float()
for C in Cs:
    assert torch.equal(C.cpu(), ref)
# the same with the epilogue's 16-byte store mode ($GIGA_P2P_STORE=vec, the multicast
# gather's code path with one store per peer)
os.environ["GIGA_P2P_STORE"] = "vec"
Cs = [torch.full((M, N), float("nan"), device="cuda") for _ in range(3)]
giga.matmul_sharded(shards, Bs, Cs, M, N, K)
for C in Cs:
    assert torch.equal(C.cpu(), ref)
del os.environ["GIGA_P2P_STORE"]
giga.finalize()
del os.environ["GIGA_TRANSPORT"]
# the fused-gather epilogue's store modes on one device (TMA / st.global / multimem.st given
# an ordinary address), 3xFP16 with exceptions (the fixes write every destination)
dAe, dBe = torch.from_numpy(Ae).cuda(), torch.from_numpy(Be).cuda()
Me_, Ne_ = Ae.shape[0], Be.shape[1]
outs = []
for mode, npeer in ((0, 2), (1, 2), (2, 0)):
    Cm = torch.full((Me_, Ne_), float("nan"), device="cuda")
    peers = [torch.full((Me_, Ne_), float("nan"), device="cuda") for _ in range(npeer)]
    giga.gemm_gather_ex(dAe, dBe, Cm, peers, Me_, Ne_, Ae.shape[1], terms=4, store_mode=mode)
    torch.cuda.synchronize()
    for q in peers:
        assert torch.equal(q, Cm), mode
    outs.append(Cm)
assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])
print("sanitize script ok")
