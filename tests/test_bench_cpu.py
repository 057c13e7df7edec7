"""bench.py's CPU-side contract: the --impl reference arm (the oracle, timed on host cores)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, env=e, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    return out.stdout.strip()


def test_reference_arm_prints_one_contract_line():
    line = _run(["--impl", "reference", "--config", "c1_512", "--steps", "2", "--warmup", "3",
                 "--ref-budget", "2"])
    lines = [x for x in line.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["metric"].startswith("GEMM TFLOP/s (fp32-accurate)")
    assert d["unit"] == "TFLOP/s" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["steps"] == 2 and d["warmup"] == 3
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert "c1_512" in d["config"]["workload"]


def test_reference_arm_nonzero_ranks_are_silent():
    out = _run(["--impl", "reference", "--config", "c1_512", "--steps", "1"],
               env={"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert out == ""
