"""Stress the in-kernel lo protocol (transform warps, async-proxy pair signal): random shapes,
both tile variants; the lo-in-smem result must equal the pre-split result bit for bit and be
identical across repeated launches. Runs for $STRESS_SECONDS (default 300)."""
import os, sys, time, json
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2504_01266_b200 import giga

rng = np.random.default_rng(int(os.environ.get("STRESS_SEED", "1")))
deadline = time.time() + float(os.environ.get("STRESS_SECONDS", "300"))
n = fails = 0
while time.time() < deadline:
    M = int(rng.integers(1, 6000)); N = int(rng.integers(1, 1500)) * 4; K = int(rng.integers(1, 3000)) * 4
    cg = int(rng.integers(1, 3)); dist = ["d1", "d2", "d4"][int(rng.integers(0, 3))]
    A = torch.from_numpy(synth.gen_matrix(M, K, synth.MATRIX_A, dist)).cuda()
    B = torch.from_numpy(synth.gen_matrix(K, N, synth.MATRIX_B, dist)).cuda()
    Alo, Blo = torch.empty_like(A), torch.empty_like(B)
    giga.split_lo(A, Alo); giga.split_lo(B, Blo)
    C1 = torch.full((M, N), float("nan"), device="cuda")
    C2 = torch.full((M, N), float("nan"), device="cuda")
    C3 = torch.full((M, N), float("nan"), device="cuda")
    giga.gemm_3xtf32(A, None, B, None, C1, M, N, K, cta_group=cg)
    giga.gemm_3xtf32(A, Alo, B, Blo, C2, M, N, K, cta_group=cg)
    giga.gemm_3xtf32(A, None, B, None, C3, M, N, K, cta_group=cg)
    torch.cuda.synchronize()
    ok = torch.equal(C1.view(torch.int32), C2.view(torch.int32)) and \
        torch.equal(C1.view(torch.int32), C3.view(torch.int32))
    n += 1
    if not ok:
        fails += 1
        print("MISMATCH", M, N, K, cg, dist, flush=True)
print(json.dumps({"cases": n, "mismatches": fails}))
sys.exit(1 if fails else 0)
