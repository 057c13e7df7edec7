"""Where the N > 1 per-GPU compute time goes at normal clocks: for rank W-1 of W, the event time
of a whole giga_rank_compute_only call against the sum of its launches' own event times
(giga_timing: GEMM launches vs preparation / fix launches). The difference is idle time
between launches. S=16384 W=2,4,8."""
import json, os, sys
import torch
sys.path.insert(0, os.getcwd())
import synth
from paper_2504_01266_b200 import giga

S = int(os.environ.get("S", "16384"))
for W in [int(w) for w in os.environ.get("WS", "1,2,4,8").split(",")]:
    M = N = K = S
    r = W - 1
    r0, rows = giga.partition(M, W, r)
    B = synth.gen_rows_torch(0, K, N, 2, "d2", device="cuda")
    A = synth.gen_rows_torch(r0, rows, K, 1, "d2", device="cuda")
    C = torch.empty((M, N), device="cuda")
    for _ in range(3):
        giga.rank_compute_only(A, B, C, M, N, K, W, r)
    torch.cuda.synchronize()
    reps = 5
    giga.timing_reset(); giga.timing_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        giga.rank_compute_only(A, B, C, M, N, K, W, r)
    e1.record(); e1.synchronize()
    kt = giga.timing_read(); giga.timing_enable(False)
    ms = e0.elapsed_time(e1) / reps
    print(json.dumps({"S": S, "W": W, "call_ms": round(ms, 3),
                      "gemm_ms": round(kt["gemm_ms"] / reps, 3),
                      "prep_ms": round(kt["split_ms"] / reps, 3),
                      "gemm_launches": kt["gemm_launches"] / reps,
                      "prep_launches": kt["split_launches"] / reps}), flush=True)
    del A, B, C
    torch.cuda.empty_cache()
