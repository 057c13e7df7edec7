"""Shard-GEMM rate on the shapes the host pipeline issues (device-resident, CUDA events)."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_01266_b200 import giga
shapes = [(32768, 32768, 32768), (20480, 32768, 576), (20480, 32768, 1264), (20480, 32768, 4800),
          (1024, 32768, 32768), (2048, 32768, 32768), (8192, 16384, 1024), (512, 16384, 16384),
          (4096, 4096, 4096), (16384, 1024, 1024)]
out = {}
for (M, N, K) in shapes:
    A = torch.randn(M, K, device="cuda"); B = torch.randn(K, N, device="cuda")
    C = torch.empty(M, N, device="cuda")
    for _ in range(2):
        giga.gemm_3xtf32(A, None, B, None, C, M, N, K)
    torch.cuda.synchronize()
    reps = max(3, int(2e12 / (2 * M * N * K)))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        giga.gemm_3xtf32(A, None, B, None, C, M, N, K)
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    out[f"{M}x{N}x{K}"] = round(2 * M * N * K / ms / 1e9, 1)
    print(f"{M}x{N}x{K}: {ms:.3f} ms {out[f'{M}x{N}x{K}']} TF/s", flush=True)
    del A, B, C
