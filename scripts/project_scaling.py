"""Per-GPU compute time of the N-GPU pipeline, measured on ONE B200: giga_rank_compute_only
enqueues exactly the GEMM launches a rank issues at world N (K-chunks accumulating, the last
chunk in row chunks, 140 of 148 SMs) without the communication. With B's broadcast and C's
gather overlapped the N-GPU step cannot be faster than this; the
exposed part of the exchange adds to it. Prints one JSON line per config:
{"config", "N": {"compute_ms", "ratio_to_N1", "t_comm_model_ms", "kchunks", "row_chunks",
"startup_model_ms"}}.
Usage: python scripts/project_scaling.py [c3_16384 c5_32768 c4_tall c2_4096]."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
from paper_2504_01266_b200 import giga

CONFIGS = {"c2_4096": (4096, 4096, 4096), "c3_16384": (16384, 16384, 16384),
           "c4_tall": (262144, 1024, 1024), "c5_32768": (32768, 32768, 32768)}
NV_GBS = 770.0  # per-direction NVLink rate the north_star roofline uses (bench.py)
names = sys.argv[1:] or ["c2_4096", "c3_16384", "c4_tall", "c5_32768"]
for name in names:
    M, N, K = CONFIGS[name]
    out = {"config": name, "M": M, "N": N, "K": K,
           "transport": os.environ.get("GIGA_TRANSPORT", "nccl")}
    B = synth.gen_rows_torch(0, K, N, 2, "d2", device="cuda")
    for world in (1, 2, 4, 8):
        rows = [giga.partition(M, world, r)[1] for r in range(world)]
        r = world - 1  # the last rank holds the remainder: the largest shard
        r0 = giga.partition(M, world, r)[0]
        A = synth.gen_rows_torch(r0, rows[r], K, 1, "d2", device="cuda")
        C = torch.empty((M, N), device="cuda")
        reps = max(3, min(50, int(3e12 / (2 * rows[r] * N * K))))
        for _ in range(2):
            giga.rank_compute_only(A, B, C, M, N, K, world, r)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            giga.rank_compute_only(A, B, C, M, N, K, world, r)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / reps
        t_comm = 4.0 * ((K * N if world > 1 else 0) + (M - min(rows)) * N) / (NV_GBS * 1e6)
        out[str(world)] = {"compute_ms": round(ms, 3), "tflops_per_gpu": round(
            2.0 * rows[r] * N * K / ms / 1e9, 1), "t_comm_model_ms": round(t_comm, 3)}
        kb, rc = giga.pipeline_plan(M, N, K, world)
        out[str(world)]["kchunks"] = [int(b - a) for a, b in zip(kb[:-1], kb[1:])]
        out[str(world)]["row_chunks"] = int(rc)
        # before the first GEMM can start: the first K-chunk of B arrives (one ring pass)
        out[str(world)]["startup_model_ms"] = round(
            4.0 * int(kb[1] - kb[0]) * N / (NV_GBS * 1e6), 3) if world > 1 else 0.0
        del A, C
    for world in (2, 4, 8):
        out[str(world)]["compute_speedup_vs_1"] = round(
            out["1"]["compute_ms"] / out[str(world)]["compute_ms"], 2)
    print(json.dumps(out), flush=True)
    del B
    torch.cuda.empty_cache()
