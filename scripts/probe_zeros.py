import os, sys, torch, json
sys.path.insert(0, os.getcwd())
from paper_2504_01266_b200 import giga
M = N = K = 16384
for fill in ("randn", "zeros"):
    A = torch.randn(M, K, device="cuda") if fill == "randn" else torch.zeros(M, K, device="cuda")
    B = torch.randn(K, N, device="cuda") if fill == "randn" else torch.zeros(K, N, device="cuda")
    C = torch.empty(M, N, device="cuda")
    for terms in (3, 2):
        for _ in range(2): giga.gemm_3xtf32(A, None, B, None, C, M, N, K, terms=terms)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): giga.gemm_3xtf32(A, None, B, None, C, M, N, K, terms=terms)
        e1.record(); e1.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(json.dumps({"fill": fill, "terms": terms, "ms": round(ms, 3), "tflops": round(2*M*N*K/ms/1e9, 1)}), flush=True)
