#!/usr/bin/env python
"""Benchmark of the data-parallel dot product (GigaAPI S4.2.8).

    python bench_vec.py [--n 67108864] [--steps 20] [--warmup 3]

One step = giga_dot_rank on device-resident fp32 vectors (the rank API: this process's GPU,
NCCL all-reduce of the fp64 partial when world > 1) including the 8-byte result read-back.
The kernel is HBM-bound: 8 algorithmic bytes per element (x and y read once). Prints one
JSON line: metric "dot GB/s", whole-call and kernel-only roofline fractions against the
measured HBM copy peak (MEASURED_PEAKS.json), and the oracle's rate on the host.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 26)  # the paper's "actual vector size"
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    import torch
    import synth
    from paper_2504_01266_b200 import giga

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        pg = dist
        obj = [giga.comm_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        giga.rank_init(rank, world, local, obj[0])
    else:
        giga.rank_init(0, 1, local, None)
    n = args.n
    r0, rows = giga.partition(n, world, rank)
    x = synth.gen_rows_torch(0, 1, n, synth.VECTOR_X, "d4", device=dev)[0, r0:r0 + rows].contiguous()
    y = synth.gen_rows_torch(0, 1, n, synth.VECTOR_Y, "d4", device=dev)[0, r0:r0 + rows].contiguous()
    s = torch.cuda.Stream(device=dev)
    s.wait_stream(torch.cuda.current_stream(dev))
    for _ in range(args.warmup):
        giga.dot_rank(x, y, n, stream=s)
    torch.cuda.synchronize()
    if pg:
        pg.barrier()
    # whole call (kernel + all-reduce + 8-byte read-back + host sync), CUDA events on `s`
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(args.steps):
        val = giga.dot_rank(x, y, n, stream=s)
    e1.record(s)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    if pg:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        ms = float(t.item())
    # kernel only: the same kernel, launched back to back through torch's profiler-free path
    kern = []
    for _ in range(5):
        k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        k0.record(s)
        giga.dot_rank(x, y, n, stream=s)
        k1.record(s)
        k1.synchronize()
        kern.append(k0.elapsed_time(k1))
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
    gbs = 8.0 * n / (ms * 1e-3) / 1e9
    per_gpu = gbs / world
    out = None
    if rank == 0:
        import oracle
        xs = synth.gen_vector(min(n, 1 << 24), synth.VECTOR_X, "d4")
        ys = synth.gen_vector(min(n, 1 << 24), synth.VECTOR_Y, "d4")
        t0 = time.perf_counter()
        oracle.dot(xs, ys)
        tcpu = time.perf_counter() - t0
        out = {
            "metric": "dot GB/s (fp32 inputs, fp64 accumulation)", "value": round(gbs, 1),
            "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 5), "higher_is_better": True, "scaling": "strong",
            "dtype": "f32 in, f64 accumulate", "data": "synthetic (synth d4, uniform [-10,10))",
            "config": {"workload": f"dot n={n}", "result": val},
            "roofline": {"bound": "hbm", "achieved": round(per_gpu, 1),
                         "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": round(per_gpu / peaks["hbm_gbs"], 4),
                         "note": "whole call per GPU incl. launch, all-reduce and 8-byte "
                                 "read-back; 8 algorithmic bytes per element",
                         "single_call_ms_median": round(statistics.median(kern), 5)},
            "cpu_baseline": {"value": round(8.0 * xs.size / tcpu / 1e9, 3), "unit": "GB/s",
                             "cores": 1, "kind": "oracle",
                             "sample": f"first {xs.size} elements, sequential fp64 loop"},
        }
        print(json.dumps(out), flush=True)
    giga.finalize()
    if pg:
        pg.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
