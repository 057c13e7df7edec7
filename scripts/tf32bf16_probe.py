"""Bring-up probe of the TF32 + BF16 scheme (terms = 2): accuracy against the oracle on small
shapes for both tile variants, then GEMM rates of terms 3 and 2 at a few shapes.
Env knobs (read once per process): GIGA_HI_RN, GIGA_BX_LBO, GIGA_BX_SBO.
Prints one JSON line per measurement."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from oracle.check import check_close, check_exact  # noqa: E402
import synth  # noqa: E402
from paper_2504_01266_b200 import giga  # noqa: E402

tag = {k: os.environ.get(k) for k in ("GIGA_HI_RN", "GIGA_BX_LBO", "GIGA_BX_SBO", "GIGA_DBG")}
for cg in ((1, 2) if os.environ.get("PROBE_ACC", "1") == "1" else ()):
    for (M, N, K, dist) in [(256, 256, 16, "d3"), (300, 520, 260, "d3"), (700, 900, 3000, "d1"),
                            (512, 512, 1024, "d2")]:
        A = synth.gen_matrix(M, K, synth.MATRIX_A, dist)
        B = synth.gen_matrix(K, N, synth.MATRIX_B, dist)
        dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
        dC = torch.full((M, N), float("nan"), device="cuda")
        giga.gemm_3xtf32(dA, None, dB, None, dC, M, N, K, terms=2, cta_group=cg)
        torch.cuda.synchronize()
        ref, S = oracle.gemm(A, B)
        C = dC.cpu().numpy()
        ok, st = (check_exact if dist == "d3" else check_close)(C, ref, *([] if dist == "d3" else [S]))
        rel = float(np.nanmax(np.abs(C - ref) / np.maximum(S, 1e-300)))
        print(json.dumps({"probe": "acc", **tag, "cg": cg, "shape": [M, N, K], "dist": dist,
                          "ok": bool(ok), "max_rel": rel,
                          "nan": int(np.isnan(C).sum())}), flush=True)

if os.environ.get("PROBE_TIME", "1") == "1":
    shapes = [(16384, 16384, 16384), (32768, 32768, 32768), (4096, 4096, 4096)]
    if os.environ.get("PROBE_SHAPES"):
        shapes = [tuple(int(v) for v in x.split("x")) for x in os.environ["PROBE_SHAPES"].split(",")]
    for (M, N, K) in shapes:
        A = torch.randn(M, K, device="cuda")
        B = torch.randn(K, N, device="cuda")
        C = torch.empty(M, N, device="cuda")
        for terms in [int(t) for t in os.environ.get("PROBE_TERMS", "3,2").split(",")]:
            for _ in range(2):
                giga.gemm_3xtf32(A, None, B, None, C, M, N, K, terms=terms)
            torch.cuda.synchronize()
            reps = max(3, int(4e13 / (2 * M * N * K)))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                giga.gemm_3xtf32(A, None, B, None, C, M, N, K, terms=terms)
            e1.record()
            e1.synchronize()
            ms = e0.elapsed_time(e1) / reps
            print(json.dumps({"probe": "rate", **tag, "terms": terms, "shape": [M, N, K],
                              "ms": round(ms, 4),
                              "tflops": round(2 * M * N * K / ms / 1e9, 1)}), flush=True)
        del A, B, C
        torch.cuda.empty_cache()
