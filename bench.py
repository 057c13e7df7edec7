#!/usr/bin/env python
"""Benchmark of the row-split fp32-accurate GEMM (GigaAPI, arXiv 2504.01266) on B200.

    python bench.py --gpus N --steps K --warmup W            (N > 1: under torchrun)
    python bench.py --impl reference ...                      (the CPU fp64 oracle arm)
    python bench.py --workload dot [--n 67108864]             (the N3 dot product, GB/s)

One step = the whole hot path over one synthetic problem: broadcast B from
rank 0 (N > 1), the fp32-accurate tcgen05 shard GEMM (3xTF32 with the hi/lo split on chip,
or for large launches TF32 + BF16 with its operands prepared in HBM: giga_product_scheme),
gather the C row blocks on every rank. Default workload: M = N = K = 32768 (BASELINE.json configs[4], the
problem the north_star's targets are quoted on), strong scaling (the same problem split over
N GPUs); --config picks the others. Inputs are seeded synthetic fp32 (synth "d2", U[-1,1)),
resident in HBM before the timed region; each step is bracketed by CUDA events and the L2 is
flushed between steps.

Prints ONE JSON line (rank 0). Metric: logical TFLOP/s = 2 M N K / t (whole job).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (M, N, K)  -- BASELINE.json configs
    "c1_512": (512, 512, 512),
    "c2_4096": (4096, 4096, 4096),
    "c3_16384": (16384, 16384, 16384),
    "c4_tall": (262144, 1024, 1024),
    "c5_32768": (32768, 32768, 32768),
}
# The north_star's targets are quoted on 32768^3 (>= 60% of the 8-GPU roofline, >= 6.5x from 1
# to 8 GPUs); it fits one GPU, so it is the default workload at every N (strong scaling).
DEFAULT_CONFIG = "c5_32768"
# the shard GEMM's fp32-accurate schemes (giga_product_scheme): MMA instruction times per k8
# step in TF32 units, names, what they compute
SCHEME_WEIGHT = {1: 1.0, 2: 2.0, 3: 3.0, 4: 1.5}
SCHEME_NAME = {1: "TF32", 2: "TF32+BF16", 3: "3xTF32", 4: "3xFP16"}
SCHEME_ARITH = {
    1: "plain TF32 tcgen05 MMAs (not fp32-accurate)",
    2: "TF32 + BF16 tcgen05 MMAs (a_hi b_hi in TF32, a_lo b + a_hi b_lo in one K=16 BF16 MMA; "
       "operands prepared in HBM per call)",
    3: "3xTF32 tcgen05 MMAs",
    4: "3xFP16 tcgen05 MMAs (the 3xTF32 split a_lo b_hi + a_hi b_lo + a_hi b_hi on fp16 "
       "operands of power-of-two scaled rows of A / columns of B, prepared in HBM per call; "
       "exceptions fixed in fp64)"}
FILL_PEAK_GBPS = 12829.1  # profiles/r02_tma_fill_sweep.jsonl (max over the sweep)
METRIC = "GEMM TFLOP/s (fp32-accurate) at 1/2/4/8 B200 and % of TF32 tensor roofline"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "hbm_gbs": 6650.0}, "fallback"


class ClockSampler:
    """NVML clock / throttle-reason sampler running during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int, period: float = 0.1):
        self.index, self.period = index, period
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # noqa: BLE001
            self._err = str(e)
            return self
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for b, name in self.REASONS.items():
                    if bits & b and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(self.period)

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join()
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return world, rank, local


_B_CACHE = {}


def oracle_sample(M, N, K, dist, budget_s, threads):
    """Time the oracle, as it stands, on the first R rows of the workload (~budget_s).
    Input generation is outside the timed region (B is generated once per process)."""
    import numpy as np
    import torch
    import oracle
    import synth

    torch.set_num_threads(threads)
    key = (K, N, dist)
    if key not in _B_CACHE:
        _B_CACHE[key] = synth.gen_rows_torch(0, K, N, synth.MATRIX_B, dist, device="cpu").numpy()
    B = _B_CACHE[key]
    probe = max(1, threads)
    A = synth.gen_rows(0, probe, K, synth.MATRIX_A, dist)
    t0 = time.perf_counter()
    oracle.gemm(A, B, nthreads=threads, want_s=False)
    t_probe = time.perf_counter() - t0
    rows = int(max(probe, min(M, probe * max(1.0, budget_s / max(t_probe, 1e-6)))))
    rows = max(probe, rows // probe * probe)
    A = synth.gen_rows(0, rows, K, synth.MATRIX_A, dist)
    t0 = time.perf_counter()
    oracle.gemm(A, B, nthreads=threads, want_s=False)
    t = time.perf_counter() - t0
    return {"rows": rows, "seconds": t, "tflops": 2.0 * rows * N * K / t / 1e12}


def rank_launches(giga, M, N, K, world, rank):
    """(rows, K depth, terms) of every GEMM launch rank `rank` issues in one step, as the
    library plans them: world 1 one launch; the NCCL pipeline one launch per K-chunk of
    giga_pipeline_plan over the rank's rows, the last K-chunk in row chunks (scheme chosen on
    the rank's rows, the row chunks share B's preparation); the p2p transport one launch per
    K-chunk over the rank's rows."""
    r0, rows = giga.partition(M, world, rank)
    if world == 1:
        return [(M, K, giga.product_scheme(M, N, K))]
    kb, rc = giga.pipeline_plan(M, N, K, world)
    out = []
    p2p = os.environ.get("GIGA_TRANSPORT") == "p2p"
    for c in range(len(kb) - 1):
        kc = kb[c + 1] - kb[c]
        if rows == 0:
            continue
        terms = giga.product_scheme(rows, N, kc)
        if c < len(kb) - 2 or p2p:
            out.append((rows, kc, terms))
            continue
        for q in range(rc):
            _, brows = giga.plan_block(M, world, rc, rank, q)
            if brows > 0:
                out.append((brows, kc, terms))
    return out


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(M, N, K, args, world):
    """The oracle, as it stands, on the host cores (SURVEY 8(d) "oracle timing beside it"):
    a bounded row sample of this workload with every usable core, its extrapolation to the
    whole product (labelled as such), and the 1-thread time of c1 512^3 (the config note's
    "about a second")."""
    import numpy as np
    import oracle
    import synth
    threads = len(os.sched_getaffinity(0))
    try:
        r = oracle_sample(M, N, K, args.dist, args.cpu_budget, threads)
        a1 = synth.gen_matrix(512, 512, synth.MATRIX_A, args.dist)
        b1 = synth.gen_matrix(512, 512, synth.MATRIX_B, args.dist)
        t0 = time.perf_counter()
        oracle.gemm(a1, b1, nthreads=1)
        c1_1t = time.perf_counter() - t0
        del np
        return {"value": round(r["tflops"], 6), "unit": "TFLOP/s", "cores": threads,
                "kind": "oracle", "cpu_model": cpu_model(), "n_gpus_of_this_run": world,
                "sample": f"first {r['rows']} rows of C (of {M}), full N={N}, K={K}: "
                          f"{r['seconds']:.1f} s fp64 i-k-j C triple loop",
                "full_product_s_extrapolated": round(r["seconds"] * M / r["rows"], 3),
                "c1_512cubed_1thread_s": round(c1_1t, 3)}
    except Exception as ex:  # noqa: BLE001
        return {"value": None, "error": repr(ex)[:300]}


def run_reference(args):
    """--impl reference: the CPU fp64 oracle on the host cores, same config and metric."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    M, N, K = CONFIGS[args.config]
    threads = len(os.sched_getaffinity(0))
    per_step = max(1.0, args.ref_budget / max(1, args.steps + args.warmup))
    vals = []
    for i in range(args.warmup + args.steps):
        r = oracle_sample(M, N, K, args.dist, per_step, threads)
        if i >= args.warmup:
            vals.append(r)
    tflops = statistics.median(v["tflops"] for v in vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(tflops, 6), "unit": "TFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * statistics.median(v["seconds"] for v in vals), 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": f"{args.config} M={M} N={N} K={K}",
                                        "dist": args.dist},
        "cpu_baseline": {"value": round(tflops, 6), "unit": "TFLOP/s", "cores": threads,
                         "kind": "oracle", "cpu_model": cpu_model(),
                         "sample": f"first {vals[0]['rows']} rows of C per step "
                                   f"(of {M}), full N and K; fp64 i-k-j C triple loop",
                         "full_product_s_extrapolated": round(
                             statistics.median(v["seconds"] for v in vals) * M
                             / vals[0]["rows"], 3)},
        "e2e": {"value": round(tflops, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_reference_dot(args):
    """--impl reference --workload dot: the fp64 oracle dot product, one host core."""
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    import oracle
    import synth
    n = min(args.n, 1 << 26)
    xs = synth.gen_vector(n, synth.VECTOR_X, "d4")
    ys = synth.gen_vector(n, synth.VECTOR_Y, "d4")
    ts = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        oracle.dot(xs, ys)
        if i >= args.warmup:
            ts.append(time.perf_counter() - t0)
    sec = statistics.median(ts)
    gbs = round(8.0 * n / sec / 1e9, 3)
    print(json.dumps({
        "impl": "reference", "metric": "dot GB/s (fp32 inputs, fp64 accumulation)",
        "value": gbs, "unit": "GB/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(sec * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"dot n={n}"},
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": 1, "kind": "oracle",
                         "sample": f"{n} elements, sequential fp64 loop"},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="giga", choices=["giga", "reference"])
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--dist", default="d2", choices=["d1", "d2", "d3", "d5"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-budget", type=float, default=60.0,
                    help="total seconds of oracle work for --impl reference")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--workload", default="gemm", choices=["gemm", "dot"],
                    help="gemm (the hot path, default) or dot (the N3 dot product)")
    ap.add_argument("--n", type=int, default=1 << 26,
                    help="--workload dot: vector length (the paper's size, P:381)")
    ap.add_argument("--transport", default=os.environ.get("GIGA_TRANSPORT", "nccl"),
                    choices=["nccl", "p2p"],
                    help="N > 1: NCCL pipeline (default) or the peer-to-peer transport "
                         "(copy-engine B chain + gather fused into the GEMM epilogue)")
    ap.add_argument("--gather", default="unicast", choices=["unicast", "mc"],
                    help="--transport p2p, N > 1: the fused gather's stores -- one per peer "
                         "(unicast) or one per piece into an NVLink multicast team of C_full "
                         "buffers (mc; falls back to unicast where the driver refuses "
                         "multicast, noted in config.gather)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    os.environ["GIGA_TRANSPORT"] = args.transport
    if args.impl == "reference":
        return run_reference_dot(args) if args.workload == "dot" else run_reference(args)
    if args.workload == "dot":
        return run_dot(args)

    import torch
    import synth
    from paper_2504_01266_b200 import giga

    world, rank, local = dist_env()
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            print(f"--gpus {args.gpus} needs torchrun with {args.gpus} processes", file=sys.stderr)
            return 2
    # GIGA_BENCH_ONE_DEVICE=1 (tests only): every rank on cuda:0, gloo plumbing, p2p
    # transport -- exercises the N > 1 bench path on a one-GPU box; its numbers mean nothing
    one_dev = os.environ.get("GIGA_BENCH_ONE_DEVICE") == "1" and world > 1
    if one_dev:
        local = 0
        args.transport = os.environ["GIGA_TRANSPORT"] = "p2p"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        if one_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
        pg = dist
        if args.transport == "p2p":
            giga.rank_init(rank, world, local, None)
        else:
            obj = [giga.comm_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            giga.rank_init(rank, world, local, obj[0])
    else:
        giga.rank_init(0, 1, local, None)
    red_dev = torch.device("cpu") if one_dev else dev  # tensor device for max-over-ranks

    M, N, K = CONFIGS[args.config]
    r0, rows = giga.partition(M, world, rank)
    A = synth.gen_rows_torch(r0, rows, K, synth.MATRIX_A, args.dist, device=dev)
    if rank == 0:
        B = synth.gen_rows_torch(0, K, N, synth.MATRIX_B, args.dist, device=dev)
    else:
        B = torch.empty((K, N), dtype=torch.float32, device=dev)
    C = torch.empty((M, N), dtype=torch.float32, device=dev)
    gather_note = None
    if world > 1 and args.transport == "p2p" and args.gather == "mc":
        # C_full bound into one multicast team (giga_rank_mc_*): the epilogue writes each
        # piece once and the NVSwitch fills every rank's copy
        try:
            C = giga.as_float_tensor(giga.rank_mc_alloc(M * N * 4), M * N, dev).view(M, N)
            gather_note = "multicast (one multimem.st per piece)"
        except giga.GigaError as e:
            gather_note = f"unicast (multicast refused: {str(e)[:120]})"
    if world > 1 and args.transport == "p2p":  # register B / C_full with every peer (IPC)
        blobs = [None] * world
        pg.all_gather_object(blobs, giga.p2p_export(B, C))
        giga.p2p_import(blobs)
    stream = torch.cuda.Stream(device=dev)
    stream.wait_stream(torch.cuda.current_stream(dev))  # inputs are produced on torch's stream

    def step():
        giga.matmul_rank(A, B, C, M, N, K, stream=stream)

    def barrier():
        if pg is not None:
            pg.barrier()

    for _ in range(args.warmup):
        step()
    stream.synchronize()
    torch.cuda.synchronize()

    # ---- timed region: K steps, device events on the launching stream around each step;
    #      between steps (outside the events) a 512 MiB write flushes the 126 MB L2 ----
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    giga.timing_enable(True)
    giga.timing_reset()
    clocks = ClockSampler(local).start()
    barrier()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    w0 = time.perf_counter()
    with torch.cuda.stream(stream):
        for e0, e1 in evs:
            flush.fill_(1)
            e0.record(stream)
            step()
            e1.record(stream)
    evs[-1][1].synchronize()
    torch.cuda.synchronize()
    wall_ms = (time.perf_counter() - w0) * 1e3  # host upper bound (includes the L2 flushes)
    barrier()
    clk = clocks.stop()
    step_ms = [e0.elapsed_time(e1) for e0, e1 in evs]
    kt = giga.timing_read()
    giga.timing_enable(False)
    if pg is not None:  # per step, the slowest rank's time
        t = torch.tensor(step_ms, dtype=torch.float64, device=red_dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        step_ms = [float(v) for v in t.cpu()]
    ms_step = statistics.median(step_ms)  # the median over the timed steps
    ms_mean = sum(step_ms) / len(step_ms)
    flops = 2.0 * M * N * K
    tflops = flops / (ms_step * 1e-3) / 1e12

    # ---- roofline of the dominant kernel (the shard GEMM) ----
    peaks, peak_src = load_peaks()
    # TF32 dense peak = measured bf16 x (nominal tf32 / bf16 = 1.1 / 2.25 ~ 0.5). The GEMM is
    # timed inside a seconds-long run of back-to-back steps under the power cap, so the
    # sustained figure is the denominator (B200_PROFILING.md); the burst one is reported too.
    tf32_sustained = 0.5 * peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    tf32_burst = 0.5 * peaks["bf16_tflops"]
    # which measured figure is the denominator (B200_PROFILING.md: burst for a kernel timed
    # alone, sustained for one inside a long step): short steps run above the power-capped
    # clock the sustained figure was measured at -- then the burst figure applies
    sust_mhz = (peaks.get("clocks_under_load") or {}).get("sm_mhz_median")
    run_mhz = (clk or {}).get("sm_mhz")
    peak_kind = ("burst" if sust_mhz and run_mhz and run_mhz > sust_mhz else "sustained")
    tf32_peak = tf32_burst if peak_kind == "burst" else tf32_sustained
    launches = rank_launches(giga, M, N, K, world, rank)
    # algorithmic tensor work per step in TF32-instruction-equivalent flops (MMA instruction
    # times x the TF32 rate): 3xTF32 issues 3 TF32 MMAs per logical product (6 r N K per
    # launch), TF32 + BF16 one TF32 MMA plus one BF16 MMA of twice the depth at twice the rate
    # (4 r N K), 3xFP16 three FP16 MMAs of twice the depth at twice the rate (3 r N K)
    tensor_flops = sum(SCHEME_WEIGHT[t] * 2.0 * r * N * kc for r, kc, t in launches)
    terms_set = sorted({t for _, _, t in launches})
    gemm_ms_step = kt["gemm_ms"] / args.steps  # all of this rank's GEMM launches in a step
    achieved = tensor_flops / (gemm_ms_step * 1e-3) / 1e12 if gemm_ms_step > 0 else None
    scheme = "+".join(SCHEME_NAME[t] for t in terms_set)
    traffic, traffic_src = None, None
    tp = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    if world == 1 and os.path.exists(tp):
        try:
            with open(tp) as f:
                traffic = json.load(f).get(f"{args.config}:{scheme}")
            traffic_src = ("profiles/gemm_traffic.json: dram__bytes_read.sum + "
                           "dram__bytes_write.sum of one launch from an ncu --set full capture "
                           "of this kernel and config (not measured in this run)")
        except Exception:  # noqa: BLE001
            traffic = None
    roof = {"bound": "tensor", "achieved": round(achieved, 2) if achieved else None,
            "peak": round(tf32_peak, 1), "unit": "TFLOP/s", "peak_kind": peak_kind,
            "peak_rule": (f"burst when the median SM clock of the timed steps ({run_mhz} MHz) "
                          f"exceeds the one the sustained figure was measured at ({sust_mhz})"),
            "frac": round(achieved / tf32_peak, 4) if achieved else None,
            "frac_vs_sustained": round(achieved / tf32_sustained, 4) if achieved else None,
            "frac_vs_burst": round(achieved / tf32_burst, 4) if achieved else None,
            "traffic": traffic, "traffic_source": traffic_src,
            "kernel": "gemm_3xtf32_kernel", "launches_per_step": len(launches),
            "kernel_ms_per_step": round(gemm_ms_step, 4),
            "kernel_share_of_step": round(gemm_ms_step / ms_mean, 4) if ms_mean else None,
            "peak_note": f"TF32 dense = 0.5 x {peak_src} cuBLAS bf16 sustained "
                         f"({peaks.get('bf16_tflops_sustained')}; burst {peaks['bf16_tflops']}; "
                         f"nominal tf32:bf16 = 1.1:2.25); achieved = the scheme's "
                         f"TF32-equivalent tensor work (3 or 2 x 2 rows N K per launch) / "
                         f"event time of the GEMM launches of a step",
            "scheme": scheme,
            "limit_note": ("operand feed: 32 KiB of TMA fills per CTA per 2-MMA stage against "
                           "the per-SM fill rate (roofline.feed), and the power cap: DESIGN.md 6.7"
                           if 2 in terms_set else
                           "tensor pipe (three MMAs per k8 step with 3xTF32, per k16 step with "
                           "3xFP16) at the power-capped clock"),
            "prep_ms_per_step": round(kt["split_ms"] / args.steps, 4),
            "prep_launches_per_step": round(kt["split_launches"] / args.steps, 2)}
    if terms_set == [4] and achieved:
        # one scheme, one dtype: state the kernel in its own units -- fp16 tensor flops (three
        # FP16 products per logical product: 6 r N K per launch) against the dense FP16 / BF16
        # peak (the same rate), i.e. the same fraction as the TF32-equivalent accounting
        f16 = 2.0 * achieved
        roof.update({"achieved": round(f16, 2), "peak": round(2 * tf32_peak, 1),
                     "frac": round(f16 / (2 * tf32_peak), 4),
                     "frac_vs_sustained": round(f16 / (2 * tf32_sustained), 4),
                     "frac_vs_burst": round(f16 / (2 * tf32_burst), 4), "dtype": "f16",
                     "peak_note": f"dense FP16 = BF16 rate: {peak_src} cuBLAS bf16 sustained "
                                  f"({peaks.get('bf16_tflops_sustained')}; burst "
                                  f"{peaks['bf16_tflops']}); achieved = 3 FP16 products x 2 rows "
                                  f"N K per launch / event time of the GEMM launches of a step"})
    if 2 in terms_set or 4 in terms_set:
        # the prepared TF32 + BF16 kernel's operand feed: 64 KiB of fills per 256 x 256 pair
        # tile and 16-deep k-block = r N K / 16 bytes per launch, against the measured L2 -> SM
        # TMA fill ceiling (scripts/tma_box_bench.cu: 10.7 TB/s on a 148-SM B200 for every box
        # shape; scripts/tma_mcast_bench.cu: multicast does not raise per-SM ingress)
        # (3xFP16: 64 KiB per pair tile and 32-deep k-block = r N K / 32 bytes per launch)
        feed_bytes = sum(r * N * kc / (16.0 if t == 2 else 32.0)
                         for r, kc, t in launches if t in (2, 4))
        fed_flops = sum(SCHEME_WEIGHT[t] * 2.0 * r * N * kc for r, kc, t in launches
                        if t in (2, 4))
        feed_ms = gemm_ms_step * fed_flops / tensor_flops
        feed_ach = feed_bytes / (feed_ms * 1e-3) / 1e9 if feed_ms > 0 else None
        roof["feed"] = {"bound": "l2_to_smem_tma",
                        "achieved": round(feed_ach, 1) if feed_ach else None,
                        "peak": FILL_PEAK_GBPS, "unit": "GB/s",
                        "frac": round(feed_ach / FILL_PEAK_GBPS, 4) if feed_ach else None,
                        "bytes_per_step": feed_bytes,
                        "peak_source": "highest TMA fill rate measured in isolation "
                                       "(scripts/tma_fill_sweep.cu, "
                                       "profiles/r02_tma_fill_sweep.jsonl: 12.8 TB/s both with 3 "
                                       "CTAs per SM x 2 x 32 KiB stages of 8 KiB boxes and with "
                                       "1 CTA per SM x 3 x 64 KiB stages of 32 KiB boxes)"}

    # ---- whole-step roofline: T_roof / t with T_roof = max(T_comp, T_comm),
    #      T_comp = the scheme's tensor work of the largest shard at the TF32 peak,
    #      T_comm = 4 (K N [g > 1] + (M - r_min) N) / BW_nvlink (north_star)
    rows_all = [giga.partition(M, world, g)[1] for g in range(world)]
    bw_nv = 770e9  # measured NVLink peer-copy GB/s per direction (B200_PROFILING.md)
    t_comm = 4.0 * ((K * N if world > 1 else 0) + (M - min(rows_all)) * N) / bw_nv
    w_max = max(range(world), key=lambda g: rows_all[g])
    tf_max = sum(SCHEME_WEIGHT[t] * 2.0 * r * N * kc
                 for r, kc, t in rank_launches(giga, M, N, K, world, w_max))
    t_comp = tf_max / (tf32_peak * 1e12)
    t_comp3 = 2.0 * max(rows_all) * N * K / (tf32_peak * 1e12 / 3)
    t_roof = max(t_comp, t_comm)
    step_roof = {"definition": "T_roof / t (median step), T_roof = max(T_comp, T_comm); T_comp "
                               "= the scheme's TF32-equivalent tensor work of the largest shard "
                               "at the TF32 peak of roofline.peak_kind, T_comm = 4 (K N [g>1] + "
                               "(M - r_min) "
                               "N) / 770 GB/s",
                 "t_comp_ms": round(t_comp * 1e3, 4), "t_comm_ms": round(t_comm * 1e3, 4),
                 "bound": "tensor" if t_comp >= t_comm else "nvlink",
                 "frac": round(t_roof / (ms_step * 1e-3), 4),
                 "frac_vs_3xtf32_ceiling": round(max(t_comp3, t_comm) / (ms_step * 1e-3), 4),
                 "note": "frac_vs_3xtf32_ceiling is the north_star's reading (P_tf32 / 3 per "
                         "logical product); above 1 when a launch runs a scheme cheaper than "
                         "3xTF32 (TF32 + BF16: 2 MMA times per k8 step, 3xFP16: 1.5)"}

    # ---- end to end: host buffers through the C ABI ----
    e2e = None
    if args.e2e_steps > 0:
        if world == 1:  # a failure here must not cost the device-resident line
            try:
                e2e = measure_e2e(giga, torch, synth, args, M, N, K, world, rank, local, dev,
                                  pg, red_dev, (A, B, C), device_ms=ms_step)
            except Exception as ex:  # noqa: BLE001
                e2e = {"value": None, "error": repr(ex)[:300]}
        else:  # collectives inside: every rank must run it (no per-rank recovery)
            e2e = measure_e2e(giga, torch, synth, args, M, N, K, world, rank, local, dev, pg,
                              red_dev, (A, B, C))

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(M, N, K, args, world)

    # the paper's only number for this metric is 32768^3 on its 2 GPUs
    # (159 s -> 0.443 TFLOP/s derived, 2x Quadro RTX 6000); context, not the target
    vs_base = (round(tflops / 0.443, 1) if (args.config == "c5_32768" and world == 2)
               else None)
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(tflops, 3), "unit": "TFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "ms_per_step_mean": round(ms_mean, 4), "timing": "median of per-step CUDA events "
            "(max over ranks per step)",
            "higher_is_better": True, "scaling": "strong", "vs_baseline": vs_base,
            "wall_ms_per_step": round(wall_ms / args.steps, 4),
            "dtype": "f32",
            "arithmetic": " / ".join(SCHEME_ARITH[t] for t in terms_set)
                          + " + fp32 RN promotion (fp32-accurate: <= 1e-5 sum|A||B|)",
            "data": "synthetic",
            "config": {"workload": f"{args.config} M={M} N={N} K={K}", "dist": args.dist,
                       "parallelism": f"row-split x{world}",
                       "transport": args.transport if world > 1 else "none (1 GPU)",
                       **({"gather": gather_note} if gather_note else {}),
                       "l2": "L2 flushed between timed steps (512 MiB write outside the "
                             "per-step events)"},
            "roofline": roof, "roofline_step": step_roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(kt["gemm_launches"] + kt["split_launches"]),
            "gpu_launches_per_step": round((kt["gemm_launches"] + kt["split_launches"])
                                           / args.steps, 2),
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    giga.finalize()
    if pg is not None:
        pg.destroy_process_group()
    return 0


def run_dot(args):
    """--workload dot: the data-parallel dot product (GigaAPI S4.2.8; SURVEY
    N3). One step = giga_dot_rank on device-resident fp32 vectors (this process's GPU; NCCL
    all-reduce of the fp64 partial when world > 1) including the 8-byte result read-back.
    HBM-bound: 8 algorithmic bytes per element (x and y read once)."""
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
        import oracle  # the cpu_baseline leg
        xs = synth.gen_vector(min(n, 1 << 24), synth.VECTOR_X, "d4")
        ys = synth.gen_vector(min(n, 1 << 24), synth.VECTOR_Y, "d4")
        t0 = time.perf_counter()
        oracle.dot(xs, ys)
        tcpu = time.perf_counter() - t0
        out = {
            "metric": "dot GB/s (fp32 inputs, fp64 accumulation)", "value": round(gbs, 1),
            "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 5), "higher_is_better": True, "scaling": "strong",
            "dtype": "f64", "arithmetic": "f32 inputs, exact products, f64 accumulation",
            "data": "synthetic (synth d4, uniform [-10,10))",
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


def pcie_roofline(torch, dev, h2d, d2h, device_ms, e2e_ms):
    """the host-buffer call moves h2d bytes in and d2h bytes out over this
    GPU's PCIe link beside the device-resident step, on three engines that overlap, so its
    time is at least T_roof = max(h2d / R_h2d, d2h / R_d2h, device step). R = pinned 1 GiB
    copy rates measured here, each direction alone (CUDA events, best of 3)."""
    n = 1 << 28
    hb = torch.empty(n, dtype=torch.float32).pin_memory()
    db = torch.empty(n, dtype=torch.float32, device=dev)

    def rate(fn):
        best = 1e9
        for _ in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            fn()
            e1.record()
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1))
        return 4.0 * n / (best * 1e-3) / 1e9

    r_h2d = rate(lambda: db.copy_(hb, non_blocking=True))
    r_d2h = rate(lambda: hb.copy_(db, non_blocking=True))
    t_h2d, t_d2h = h2d / r_h2d / 1e6, d2h / r_d2h / 1e6  # ms
    terms = {"h2d": t_h2d, "d2h": t_d2h, "device_step": device_ms}
    bound = max(terms, key=terms.get)
    t_roof = terms[bound]
    return {"bound": bound, "t_roof_ms": round(t_roof, 3), "frac": round(t_roof / e2e_ms, 4),
            "h2d_ms_at_link_rate": round(t_h2d, 3), "d2h_ms_at_link_rate": round(t_d2h, 3),
            "device_step_ms": round(device_ms, 3), "h2d_GBps_measured": round(r_h2d, 2),
            "d2h_GBps_measured": round(r_d2h, 2),
            "definition": "max(H2D bytes / R_h2d, D2H bytes / R_d2h, device-resident median "
                          "step) / e2e step; R = pinned 1 GiB copies each direction alone"}


def measure_e2e(giga, torch, synth, args, M, N, K, world, rank, local, dev, pg, red_dev,
                dev_bufs, device_ms=None):
    """Same metric with the inputs in pinned HOST memory: every step copies this rank's A
    rows (and B on rank 0) host->device, runs the hot path and copies this rank's C rows
    back (N = 1: the single giga_matmul host-pointer call of the C ABI)."""
    r0, rows = giga.partition(M, world, rank)
    if world == 1:
        giga.finalize()
        giga.init(1)
        Ah = synth.gen_rows_torch(0, M, K, synth.MATRIX_A, args.dist, device=dev).cpu().pin_memory()
        Bh = synth.gen_rows_torch(0, K, N, synth.MATRIX_B, args.dist, device=dev).cpu().pin_memory()
        Ch = torch.empty((M, N), dtype=torch.float32).pin_memory()
        giga.matmul(Ah, Bh, Ch, M, N, K, 1)  # warm (workspace)
        ts = []
        for _ in range(args.e2e_steps):
            t0 = time.perf_counter()
            giga.matmul(Ah, Bh, Ch, M, N, K, 1)
            ts.append(time.perf_counter() - t0)
        t = statistics.median(ts)
        h2d = 4 * (M * K + K * N)
        d2h = 4 * M * N
        out = {"value": round(2.0 * M * N * K / t / 1e12, 3), "unit": "TFLOP/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": round(t * 1e3, 3),
               "api": "giga_matmul(host pinned A, B, C) blocking, wall clock"}
        out["roofline"] = pcie_roofline(torch, dev, h2d, d2h, device_ms, t * 1e3)
        return out
    # N > 1: each rank stages its own rows; rank 0 stages B
    Ah = torch.empty((rows, K), dtype=torch.float32).pin_memory()
    Ah.copy_(synth.gen_rows_torch(r0, rows, K, synth.MATRIX_A, args.dist, device=dev).cpu())
    Bh = None
    if rank == 0:
        Bh = synth.gen_rows_torch(0, K, N, synth.MATRIX_B, args.dist, device=dev).cpu().pin_memory()
    Ch = torch.empty((rows, N), dtype=torch.float32).pin_memory()
    A, B, C = dev_bufs  # the device buffers of the timed run (registered with peers for p2p)
    s = torch.cuda.Stream(device=dev)
    s.wait_stream(torch.cuda.current_stream(dev))

    def one():
        with torch.cuda.stream(s):
            A.copy_(Ah, non_blocking=True)
            if Bh is not None:
                B.copy_(Bh, non_blocking=True)
            giga.matmul_rank(A, B, C, M, N, K, stream=s)
            Ch.copy_(C[r0:r0 + rows], non_blocking=True)
        s.synchronize()

    one()
    ts = []
    for _ in range(args.e2e_steps):
        pg.barrier()
        t0 = time.perf_counter()
        one()
        t = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=red_dev)
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        ts.append(float(t.item()))
    t = statistics.median(ts)
    return {"value": round(2.0 * M * N * K / t / 1e12, 3), "unit": "TFLOP/s",
            "h2d_bytes_per_step": 4 * (M * K + K * N), "d2h_bytes_per_step": 4 * M * N,
            "ms_per_step": round(t * 1e3, 3),
            "api": "pinned H2D + giga_matmul_rank + D2H per rank, wall clock max over ranks"}


if __name__ == "__main__":
    sys.exit(main())
