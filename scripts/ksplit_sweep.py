"""Shard-GEMM time per shape under the k-split schedule in effect ($GIGA_TAIL_SPLIT=0: whole
tiles; $GIGA_KSPLIT_S=s: s parts forced; neither: the planned split). Device-resident, CUDA
events over back-to-back launches. One JSON line: {"setting": ..., "MxNxK": [ms, s], ...}."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2504_01266_b200 import giga

SHAPES = [(512, 512, 512), (1024, 1024, 1024), (512, 1536, 2048), (2048, 4096, 4096),
          (4096, 4096, 4096), (2304, 2304, 1040), (1000, 1284, 3000), (512, 16384, 16384),
          (2048, 16384, 16384), (16384, 16384, 16384)]
if os.environ.get("SHAPES"):
    SHAPES = [tuple(int(v) for v in s.split("x")) for s in os.environ["SHAPES"].split(",")]
setting = ("whole" if os.environ.get("GIGA_TAIL_SPLIT") == "0"
           else f"s={os.environ['GIGA_KSPLIT_S']}" if os.environ.get("GIGA_KSPLIT_S") else "plan")
out = {"setting": setting}
for (M, N, K) in SHAPES:
    A = synth.gen_rows_torch(0, M, K, 1, "d2", device="cuda")
    B = synth.gen_rows_torch(0, K, N, 2, "d2", device="cuda")
    C = torch.empty(M, N, device="cuda")
    for _ in range(3):
        giga.gemm_3xtf32(A, None, B, None, C, M, N, K)
    torch.cuda.synchronize()
    reps = max(5, min(2000, int(4e12 / (2 * M * N * K))))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        giga.gemm_3xtf32(A, None, B, None, C, M, N, K)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    out[f"{M}x{N}x{K}"] = [round(ms, 4), giga.gemm_schedule(M, N, K)["s"]]
    del A, B, C
print(json.dumps(out), flush=True)
