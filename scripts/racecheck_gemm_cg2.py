"""compute-sanitizer racecheck target: one small cta_group::2 GEMM launch (lo in smem)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2504_01266_b200 import giga
M, N, K = int(os.environ.get("M", 256)), int(os.environ.get("N", 256)), int(os.environ.get("K", 64))
dA = torch.from_numpy(synth.gen_matrix(M, K, 1, "d2")).cuda()
dB = torch.from_numpy(synth.gen_matrix(K, N, 2, "d2")).cuda()
C = torch.empty((M, N), device="cuda")
giga.gemm_3xtf32(dA, None, dB, None, C, M, N, K, cta_group=2)
torch.cuda.synchronize()
print("cg2 gemm ok", float(C.abs().sum()))
