"""K-chunk shapes of the host-buffer schedule (Me rows x N x Kc): both schemes (GIGA_SCHEME)."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_01266_b200 import giga
giga.init(1)
for (M, N, K) in [(16384, 32768, 576), (16384, 32768, 1024), (16384, 32768, 1792),
                  (8192, 16384, 1024), (4096, 32768, 768)]:
    A = torch.randn(M, K, device="cuda"); B = torch.randn(K, N, device="cuda")
    C = torch.empty(M, N, device="cuda")
    for _ in range(2):
        giga.matmul_sharded([A], [B], [C], M, N, K)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        giga.matmul_sharded([A], [B], [C], M, N, K)
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(json.dumps({"scheme": os.environ.get("GIGA_SCHEME"), "shape": [M, N, K], "ms": round(ms, 4),
                      "tflops": round(2 * M * N * K / ms / 1e9, 1)}), flush=True)
giga.finalize()
