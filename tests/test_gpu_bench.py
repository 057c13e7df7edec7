"""bench.py's GPU arm prints one contract line (metric, value, roofline of the dominant kernel,
cpu_baseline, e2e through the C ABI with host buffers, clocks, gpu_launches) for a 3xTF32
workload, a 3xFP16 one (the product scheme at c3 and c5) and a forced TF32 + BF16 one (those
two carry the TMA-feed bound too)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(args, env=None):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=900, cwd=ROOT,
                         env=dict(os.environ, **(env or {})))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [x for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def _common(d, steps, warmup):
    assert d["metric"].startswith("GEMM TFLOP/s (fp32-accurate)")
    assert d["unit"] == "TFLOP/s" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["steps"] == steps and d["warmup"] == warmup and d["n_gpus"] == 1
    assert d["dtype"] == "f32" and d["data"] == "synthetic"
    r = d["roofline"]
    assert r["bound"] == "tensor" and r["unit"] == "TFLOP/s" and 0 < r["frac"] < 1.5
    assert r["kernel"] == "gemm_3xtf32_kernel" and 0 < r["kernel_share_of_step"] <= 1.0
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= steps
    assert d["clocks"]["sm_max_mhz"] > 0
    assert "l2" in d["config"]


def test_bench_line_3xtf32_workload():
    # (c2 runs 3xFP16 by the product rule since the epilogue fix: the scheme is forced)
    d = _line(["--config", "c2_4096", "--steps", "3", "--warmup", "3", "--e2e-steps", "2",
               "--no-cpu-baseline"], env={"GIGA_SCHEME": "3xtf32"})
    _common(d, 3, 3)
    assert d["roofline"]["scheme"] == "3xTF32" and "feed" not in d["roofline"]
    assert d["gpu_launches"] == 3  # one GEMM launch per step, no preparation


def test_bench_line_3xfp16_workload_with_cpu_baseline():
    d = _line(["--config", "c3_16384", "--steps", "3", "--warmup", "3", "--e2e-steps", "1",
               "--cpu-budget", "2"])
    _common(d, 3, 3)
    r = d["roofline"]
    assert r["scheme"] == "3xFP16" and r["dtype"] == "f16"
    # per step: 3 + 1 operand-preparation kernels and 2 exception-fix kernels beside the GEMM
    assert r["prep_launches_per_step"] == 6.0
    assert r["feed"]["bound"] == "l2_to_smem_tma" and 0 < r["feed"]["frac"] < 1.2
    assert d["gpu_launches"] == 21
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] >= 1 and c["value"] > 0


def test_bench_line_tf32bf16_forced():
    d = _line(["--config", "c3_16384", "--steps", "3", "--warmup", "3", "--e2e-steps", "1",
               "--no-cpu-baseline"], env={"GIGA_SCHEME": "tf32bf16"})
    _common(d, 3, 3)
    r = d["roofline"]
    assert r["scheme"] == "TF32+BF16" and r["prep_launches_per_step"] == 2.0
    assert r["feed"]["bound"] == "l2_to_smem_tma" and 0 < r["feed"]["frac"] < 1.2
    assert d["gpu_launches"] == 9  # per step: two preparation launches and the GEMM