"""The host-buffer schedule (giga_host_plan, host_plan.cpp): structure and model, on CPU.

The planner's makespan is re-derived here from the returned plan with an independent
three-queue simulation (copy-in queue, GEMM queue, copy-back queue, each in order; a GEMM
waits for its inputs, a copy-back for its rows), and checked against engine lower bounds.
"""
import math
import os
import subprocess
import sys

import pytest

from paper_2504_01266_b200 import giga

H2D = D2H = 50e9
RATE = {3: 250e12, 2: 265e12, 4: 440e12}  # logical TFLOP/s per scheme (host_plan.h)
PREP = 5e12  # bytes/s of the TF32 + BF16 / 3xFP16 operand preparation, ~12 B per element
CLUSTERS = 74
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def gemm_t(m, n, k, accumulate=False, scheme_rows=0, b_prepared=False):
    """waves x (MMA time at the launch's scheme rate + 2 us per wave) + 10 us per launch;
    accumulate launches x1.1; + the operand preparation of the schemes that have one"""
    if m <= 0:
        return 0.0
    terms = giga.product_scheme(max(m, scheme_rows), n, k)
    tiles = math.ceil(m / 256) * math.ceil(n / 256)
    rate = RATE[terms] * (k / (k + 256) if terms == 4 else 1.0)  # 3xFP16's short-K rate
    wave = 2e-6 + 2 * 256 * 256 * k / (rate / CLUSTERS)
    prep = 12.0 * (m * k + (0 if b_prepared else k * n)) / PREP if terms in (2, 4) else 0.0
    return 10e-6 + prep + math.ceil(tiles / CLUSTERS) * wave * (1.1 if accumulate else 1.0)


def simulate(plan, M, N, K):
    Me, kb, rb = plan["Me"], plan["kb"], plan["rb"]
    t = 0.0
    arrive_k, arrive_r = [], []
    for c in range(len(kb) - 1):
        t += 4 * (Me * (kb[c + 1] - kb[c]) + (kb[c + 1] - kb[c]) * N) / H2D
        arrive_k.append(t)
    for q in range(len(rb) - 1):
        t += 4 * (rb[q + 1] - rb[q]) * K / H2D
        arrive_r.append(t)
    comp = back = 0.0
    if Me > 0:
        for c in range(len(kb) - 1):
            comp = max(comp, arrive_k[c]) + gemm_t(Me, N, kb[c + 1] - kb[c], c > 0)
        back = comp + 4 * Me * N / D2H
    late = rb[-1] - rb[0] if len(rb) > 1 else 0
    for q in range(len(rb) - 1):
        rows = rb[q + 1] - rb[q]
        if rows:
            comp = max(comp, arrive_r[q], arrive_k[-1]) + gemm_t(rows, N, K, False, late, q > 0)
            back = max(back, comp) + 4 * rows * N / D2H
    return max(comp, back)


SHAPES = [(32768, 32768, 32768), (16384, 16384, 16384), (4096, 4096, 4096),
          (262144, 1024, 1024), (512, 512, 512), (1, 1, 1), (1000, 7, 9), (300, 5000, 70000),
          (70000, 300, 5000)]


@pytest.mark.parametrize("M,N,K", SHAPES)
def test_plan_structure_and_model(M, N, K, monkeypatch):
    for k in ("GIGA_HOST_H2D_GBS", "GIGA_HOST_D2H_GBS", "GIGA_HOST_GEMM_TFLOPS"):
        monkeypatch.delenv(k, raising=False)
    p = giga.host_plan(M, N, K)
    kb, rb, Me = p["kb"], p["rb"], p["Me"]
    assert kb[0] == 0 and kb[-1] == K and all(a < b for a, b in zip(kb, kb[1:]))
    assert all(x % 16 == 0 for x in kb[1:-1]) and 1 <= len(kb) - 1 <= 16
    assert 0 <= Me <= M and len(rb) - 1 <= 16
    if Me < M:
        assert rb[0] == Me and rb[-1] == M and all(a < b for a, b in zip(rb, rb[1:]))
    else:
        assert rb == [M]
    if Me == 0:
        assert kb == [0, K]  # no phase 1: B arrives in one piece
    t = simulate(p, M, N, K)
    assert p["t_model"] == pytest.approx(t, rel=1e-9)
    # no schedule beats any single engine's total work
    assert t >= 4 * (M * K + K * N) / H2D * (1 - 1e-12)
    assert t >= 4 * M * N / D2H * (1 - 1e-12)
    assert t >= 2 * M * N * K / max(RATE.values()) * (1 - 1e-12)
    naive = 4 * (M * K + K * N) / H2D + gemm_t(M, N, K) + 4 * M * N / D2H
    assert t <= naive * (1 + 1e-12)  # never worse than copy-in, compute, copy-out


def test_plan_beats_naive_schedules():
    """Better than copying everything in, computing, copying everything out, and than the
    fixed round-1 plan (half the rows early, 8 equal K-chunks, 8 equal row blocks)."""
    for M, N, K in SHAPES[:4]:
        p = giga.host_plan(M, N, K)
        naive = 4 * (M * K + K * N) / H2D + gemm_t(M, N, K) + 4 * M * N / D2H
        Me = min(M, (M // 2 + 255) // 256 * 256)
        fixed = {"Me": Me, "kb": [K * i // 8 // 16 * 16 for i in range(8)] + [K],
                 "rb": [Me + (M - Me) * i // 8 for i in range(9)]}
        assert p["t_model"] < naive
        assert p["t_model"] <= simulate(fixed, M, N, K) * (1 + 1e-9)


def test_rates_come_from_the_environment(monkeypatch):
    base = giga.host_plan(16384, 16384, 16384)["t_model"]
    monkeypatch.setenv("GIGA_HOST_H2D_GBS", "25")
    monkeypatch.setenv("GIGA_HOST_D2H_GBS", "25")
    assert giga.host_plan(16384, 16384, 16384)["t_model"] > 1.5 * base


def test_plan_errors():
    with pytest.raises(giga.GigaError):
        giga.host_plan(0, 4, 4)


def test_build_module_importable_without_library():
    """The builder must import on a fresh checkout; the binding must refuse to load without
    the library (no fallback path)."""
    env = dict(os.environ, GIGA_LIB_PATH="/nonexistent/libgiga.so")
    code = ("import paper_2504_01266_b200.build as b; print('build ok')\n"
            "try:\n    from paper_2504_01266_b200 import giga\nexcept ImportError as e:\n"
            "    print('binding refused:', 'missing' in str(e))\n")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True,
                         text=True, timeout=120).stdout
    assert "build ok" in out and "binding refused: True" in out
