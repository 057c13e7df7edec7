import os, sys, torch, json
sys.path.insert(0, os.getcwd())
from paper_2504_01266_b200 import giga
M = N = K = 16384
A = torch.zeros(M, K, device="cuda"); B = torch.zeros(K, N, device="cuda"); C = torch.empty(M, N, device="cuda")
for terms in ([2] if os.environ.get("GIGA_DBG_MMA") else [3, 2]):
    for _ in range(2): giga.gemm_3xtf32(A, None, B, None, C, M, N, K, terms=terms)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): giga.gemm_3xtf32(A, None, B, None, C, M, N, K, terms=terms)
    e1.record(); e1.synchronize()
    print(json.dumps({"dbg": os.environ.get("GIGA_DBG_MMA"), "terms": terms, "ms": round(e0.elapsed_time(e1) / 10, 3)}), flush=True)
