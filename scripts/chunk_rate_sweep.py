"""Rate of one K-chunk GEMM launch (operand preparation included) over the shard shapes the
N-GPU pipeline issues: rows = M / N_gpus, N, Kc. Calibrates make_plan's chunk_gemm_time
(runtime.cpp). One JSON line per (rows, N, Kc, scheme): {"ms", "tflops"}.
Usage: python scripts/chunk_rate_sweep.py [N ...]"""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2504_01266_b200 import giga

giga.init_devices([0])
Ns = [int(x) for x in sys.argv[1:]] or [16384, 32768]
for N in Ns:
    Kmax = 16384
    B = synth.gen_rows_torch(0, Kmax, N, 2, "d2", device="cuda")
    for rows in (2048, 4096, 8192, 16384):
        A = synth.gen_rows_torch(0, rows, Kmax, 1, "d2", device="cuda")
        C = torch.empty((rows, N), device="cuda")
        for Kc in (256, 512, 1024, 2048, 4096, 8192, 16384):
            a, b = A[:, :Kc].contiguous(), B[:Kc].contiguous()
            for terms in (3, 2, 4):
                fl = 2.0 * rows * N * Kc
                reps = max(3, min(50, int(2e12 / fl)))
                for _ in range(2):
                    giga.gemm_3xtf32(a, None, b, None, C, rows, N, Kc, terms=terms)
                torch.cuda.synchronize()
                e0, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
                e0.record()
                for _ in range(reps):
                    giga.gemm_3xtf32(a, None, b, None, C, rows, N, Kc, terms=terms)
                e1.record()
                e1.synchronize()
                ms = e0.elapsed_time(e1) / reps
                print(json.dumps({"rows": rows, "N": N, "Kc": Kc, "terms": terms,
                                  "ms": round(ms, 4), "tflops": round(fl / ms / 1e9, 1)}),
                      flush=True)
            del a, b
        del A, C
    del B
    torch.cuda.empty_cache()
giga.finalize()
