"""Shard-GEMM kernel time vs promotion interval (and tile config, LO=presplit, TERMS=3|2), 1 GPU,
CUDA events."""
import json, os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2504_01266_b200 import giga

M = N = K = int(os.environ.get("SIZE", "16384"))
if os.environ.get("MNK"):
    M, N, K = (int(x) for x in os.environ["MNK"].split(","))
dev = torch.device("cuda", 0)
A = synth.gen_rows_torch(0, M, K, 1, "d2", device=dev)
B = synth.gen_rows_torch(0, K, N, 2, "d2", device=dev)
C = torch.empty((M, N), device=dev)
Alo = Blo = None  # lo computed in the GEMM's shared memory (the product path)
if os.environ.get("LO") == "presplit":  # the pre-split design, for comparison
    Alo, Blo = torch.empty_like(A), torch.empty_like(B)
    giga.split_lo(A, Alo); giga.split_lo(B, Blo)
TERMS = int(os.environ.get("TERMS", "3"))
torch.cuda.synchronize()
res = {}
for pk in [int(x) for x in os.environ.get("PKS", "4,8,16,32").split(",")]:
    for _ in range(2):
        giga.gemm_3xtf32(A, Alo, B, Blo, C, M, N, K, terms=TERMS, promote_kblocks=pk)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        giga.gemm_3xtf32(A, Alo, B, Blo, C, M, N, K, terms=TERMS, promote_kblocks=pk)
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    res[pk] = {"ms": round(ms, 3), "logical_tflops": round(2 * M * N * K / ms / 1e9, 1),
               "tensor_tflops": round((6 if TERMS == 3 else 4) * M * N * K / ms / 1e9, 1)}
    print(pk, res[pk], flush=True)
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/sweep_gemm.json", "w"), indent=1)
