"""Probe: the GEMM launches rank world-1 issues at world W (giga_rank_compute_only) at S^3, for an
ncu launch list (what the N > 1 per-GPU compute spends its time on)."""
import os, sys, torch
sys.path.insert(0, os.getcwd())
import synth
from paper_2504_01266_b200 import giga
M = N = K = int(os.environ.get("S", "32768")); world = int(os.environ.get("W", "8")); r = world - 1
r0, rows = giga.partition(M, world, r)
B = synth.gen_rows_torch(0, K, N, 2, "d2", device="cuda")
A = synth.gen_rows_torch(r0, rows, K, 1, "d2", device="cuda")
C = torch.empty((M, N), device="cuda")
print(giga.pipeline_plan(M, N, K, world))
for _ in range(3):
    giga.rank_compute_only(A, B, C, M, N, K, world, r)
torch.cuda.synchronize()
