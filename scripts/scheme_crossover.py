"""Product-path step time (giga_matmul_sharded, 1 GPU, preparation included) over shapes, for
the scheme forced by $GIGA_SCHEME: run once per scheme to place product_terms' crossover."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2504_01266_b200 import giga
giga.init(1)
shapes = [(512, 512, 512), (1024, 1024, 1024), (2048, 2048, 2048), (4096, 4096, 4096),
          (2048, 4096, 4096), (32768, 1024, 1024), (262144, 1024, 1024), (8192, 8192, 2048),
          (8192, 8192, 8192), (2048, 16384, 16384), (4096, 16384, 16384), (8192, 16384, 16384),
          (16384, 16384, 4096), (16384, 32768, 1024), (16384, 32768, 576), (4096, 32768, 32768),
          (16384, 16384, 16384)]
if os.environ.get("XO_SHAPES"):
    shapes = [tuple(int(v) for v in x.split("x")) for x in os.environ["XO_SHAPES"].split(",")]
for (M, N, K) in shapes:
    A = torch.randn(M, K, device="cuda"); B = torch.randn(K, N, device="cuda")
    C = torch.empty(M, N, device="cuda")
    for _ in range(2):
        giga.matmul_sharded([A], [B], [C], M, N, K)
    torch.cuda.synchronize()
    reps = max(3, int(3e13 / (2 * M * N * K)))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        giga.matmul_sharded([A], [B], [C], M, N, K)
    e1.record(); e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(json.dumps({"scheme": os.environ.get("GIGA_SCHEME"), "shape": [M, N, K],
                      "ms": round(ms, 4), "tflops": round(2 * M * N * K / ms / 1e9, 1)}), flush=True)
    del A, B, C
giga.finalize()
