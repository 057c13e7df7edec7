"""Short-K GEMM launches (K-chunks of the N > 1 / host pipelines, the tall c4): event time of a
whole giga_gemm_3xtf32_ex call (operand preparation + GEMM + fixes) per scheme, 1 GPU.
SHAPES="M,N,K;..." TERMS="4,3" REPS=5."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2504_01266_b200 import giga

shapes = [tuple(int(x) for x in s.split(",")) for s in os.environ.get(
    "SHAPES", "16384,32768,1024;16384,32768,2048;16384,32768,4096;262144,1024,1024;"
              "32768,1024,1024;16384,16384,16384").split(";")]
terms_list = [int(t) for t in os.environ.get("TERMS", "4,3").split(",")]
reps = int(os.environ.get("REPS", "5"))
dev = torch.device("cuda", 0)
out = []
for (M, N, K) in shapes:
    A = synth.gen_rows_torch(0, M, K, 1, "d2", device=dev)
    B = synth.gen_rows_torch(0, K, N, 2, "d2", device=dev)
    C = torch.empty((M, N), device=dev)
    for t in terms_list:
        for _ in range(2):
            giga.gemm_3xtf32(A, None, B, None, C, M, N, K, terms=t)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            giga.gemm_3xtf32(A, None, B, None, C, M, N, K, terms=t)
        e1.record(); e1.synchronize()
        ms = e0.elapsed_time(e1) / reps
        r = {"shape": [M, N, K], "terms": t, "ms": round(ms, 4),
             "tflops": round(2 * M * N * K / ms / 1e9, 1)}
        print(json.dumps(r), flush=True)
        out.append(r)
    del A, B, C
    torch.cuda.empty_cache()
os.makedirs("gpurun_out", exist_ok=True)
with open("gpurun_out/shortk_probe.jsonl", "w") as f:
    for r in out:
        f.write(json.dumps(r) + "\n")
