"""Small GEMM / split / dot calls for compute-sanitizer runs (memcheck, racecheck, synccheck)."""
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
x = synth.gen_vector(100003, 3, "d3"); y = synth.gen_vector(100003, 4, "d3")
print("dot", giga.dot(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()))
giga.finalize()
print("sanitize script ok")
