"""compute-sanitizer target: the TF32 + BF16 GEMM with A' / B' built in shared memory by the
transform warps (GIGA_A_PRE=0 / GIGA_B_PRE=0 set by the caller), both tile variants."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2504_01266_b200 import giga

giga.init(1)
M, N, K = 520, 516, 1040
A = synth.gen_matrix(M, K, 1, "d3"); B = synth.gen_matrix(K, N, 2, "d3")
dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
ref = torch.from_numpy(A.astype(np.float64) @ B.astype(np.float64)).float().cuda()
for cg in (1, 2):
    C = torch.full((M, N), float("nan"), device="cuda")
    giga.gemm_3xtf32(dA, None, dB, None, C, M, N, K, terms=2, cta_group=cg)
    torch.cuda.synchronize()
    assert torch.equal(C, ref), cg
giga.finalize()
print("sanitize script ok")
