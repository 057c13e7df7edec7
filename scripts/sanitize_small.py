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
x = synth.gen_vector(100003, 3, "d3"); y = synth.gen_vector(100003, 4, "d3")
print("dot", giga.dot(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()))
giga.finalize()
print("sanitize script ok")
