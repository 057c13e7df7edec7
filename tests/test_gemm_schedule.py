"""CPU checks of the GEMM launch schedule (giga_gemm_schedule, include/giga.h): the k-split of
under-filled waves (a deterministic stream-K). The schedule is the launch's own host code,
so these tests pin what the kernel is asked to run: unit coverage, workspace bound, and an
independent round-robin simulation of the persistent clusters showing the split shortens
the launch where the wave count is ragged and leaves full waves alone."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MAX_S = 32
MAX_SLOTS = 8192  # 16 KiB partial slots (128 MiB)


@pytest.fixture(scope="module")
def giga():
    from paper_2504_01266_b200 import build
    build.build()
    from paper_2504_01266_b200 import giga as g
    return g


def units(s):
    """(tile, kb0, kb1, part) of every work unit, as the kernel's unit_coords maps them."""
    out = []
    for u in range(s["units"]):
        if u < s["first_split"]:
            out.append((u, 0, s["n_kb"], -1))
        else:
            v = u - s["first_split"]
            t, q = s["first_split"] + v // s["s"], v % s["s"]
            out.append((t, s["n_kb"] * q // s["s"], s["n_kb"] * (q + 1) // s["s"], q))
    return out


def makespan(s):
    """Round-robin persistent clusters (unit u on cluster u mod clusters), each unit costing
    its k-blocks + 1, plus the k-split combine: 4 k-block times for two halves reduce-added
    into a zeroed C, 14 + 5 s for the workspace partials (write, count, ordered read of s):
    the longest cluster."""
    fix = {0: 0.0, 1: 4.0, 2: 14.0 + 5.0 * s["s"]}[s["mode"]]
    load = [0.0] * s["clusters"]
    for u, (_, kb0, kb1, part) in enumerate(units(s)):
        load[u % s["clusters"]] += kb1 - kb0 + 1
    return max(load) + fix


SHAPES = [(512, 512, 512), (2048, 4096, 4096), (4096, 4096, 4096), (16384, 16384, 16384),
          (32768, 32768, 32768), (32768, 1024, 1024), (2304, 2304, 1040), (4096, 32768, 32768),
          (2048, 16384, 16384), (100, 100, 100), (512, 32768, 18512), (1, 1, 1),
          (257, 4100, 36), (300, 300, 8), (65536, 256, 4096), (1000, 1000, 100000)]


@pytest.mark.parametrize("M,N,K", SHAPES)
def test_units_cover_every_tile_and_k_block_once(giga, M, N, K):
    s = giga.gemm_schedule(M, N, K)
    assert s["units"] == s["first_split"] + (s["tiles"] - s["first_split"]) * s["s"]
    cover = {}
    for t, kb0, kb1, part in units(s):
        assert 0 <= kb0 < kb1 <= s["n_kb"]  # every unit does at least one k-block
        cover.setdefault(t, []).append((kb0, kb1))
    assert sorted(cover) == list(range(s["tiles"]))
    for t, r in cover.items():
        r.sort()
        assert r[0][0] == 0 and r[-1][1] == s["n_kb"]
        assert all(a[1] == b[0] for a, b in zip(r, r[1:]))  # contiguous, no overlap


@pytest.mark.parametrize("M,N,K", SHAPES)
def test_split_bounds(giga, M, N, K):
    s = giga.gemm_schedule(M, N, K)
    assert 1 <= s["s"] <= min(MAX_S, max(1, s["n_kb"]))
    whole = dict(s, first_split=s["tiles"], s=1, units=s["tiles"], mode=0)
    if s["mode"] == 0:
        assert s["s"] == 1 and s["first_split"] == s["tiles"] and s["units"] == s["tiles"]
        return
    assert makespan(s) < makespan(whole)
    if s["mode"] == 1:
        # two halves onto a zeroed C: only the last, at most half-full wave (or a grid under
        # one wave) -- two addends onto zero are order-independent, three would not be
        assert s["s"] == 2
        assert s["first_split"] % s["clusters"] == 0
        assert 2 * (s["tiles"] - s["first_split"]) <= s["clusters"]
    else:
        # workspace partials: grids under one wave, all parts in one part wave
        assert s["mode"] == 2 and s["first_split"] == 0
        assert s["tiles"] < s["clusters"] and s["tiles"] * s["s"] <= s["clusters"]
        assert s["tiles"] * s["s"] * s["cta_group"] * 8 <= MAX_SLOTS


def test_known_schedules(giga):
    # 4096^3: 256 tiles on 74 pairs = 3 waves + 34; the 34 run as halves (3.5 wave times)
    s = giga.gemm_schedule(4096, 4096, 4096)
    assert (s["cta_group"], s["tiles"], s["first_split"], s["s"], s["mode"]) == (2, 256, 222, 2, 1)
    # 24 tiles of 128 x 256 on 148 SMs: parts through the workspace
    s = giga.gemm_schedule(512, 1536, 2048)
    assert s["cta_group"] == 1 and s["mode"] == 2 and s["s"] >= 3 and s["units"] <= 148
    assert makespan(s) <= 0.6 * makespan(dict(s, first_split=24, s=1, units=24, mode=0))
    # a 128-tile shard (1.73 waves): cutting a tail of 54 tiles into parts measured slower
    # than whole tiles on B200 (scripts/ksplit_sweep.py), so it runs whole
    assert giga.gemm_schedule(2048, 4096, 4096)["s"] == 1
    # a last wave more than half full (512 tiles = 6 waves + 68 on 74 pairs): runs whole
    s = giga.gemm_schedule(32768, 1024, 1024)
    assert s["tiles"] % s["clusters"] == 68 and s["s"] == 1


def test_never_worse_than_whole_tiles_on_random_shapes(giga):
    import random
    rng = random.Random(250401266)
    for _ in range(300):
        M, N, K = rng.randint(1, 40000), rng.randint(1, 40000), rng.randint(1, 40000)
        s = giga.gemm_schedule(M, N, K)
        whole = dict(s, first_split=s["tiles"], s=1, units=s["tiles"], mode=0)
        if s["tiles"] > 20000:
            continue  # the simulation is O(units); large grids are covered above
        assert makespan(s) <= makespan(whole), (M, N, K, s)


def test_fewer_sms_changes_the_plan_consistently(giga):
    # the NCCL pipeline leaves SMs to the communication kernels: the plan follows the grid
    s = giga.gemm_schedule(2304, 2304, 1040, 140)
    assert s["clusters"] == 70 and s["tiles"] == 81
    assert (s["first_split"], s["s"], s["mode"]) == (70, 2, 1)


def test_env_disables_split():
    code = ("from paper_2504_01266_b200 import giga; "
            "print(giga.gemm_schedule(4096, 4096, 4096)['s'])")
    env = dict(os.environ, GIGA_TAIL_SPLIT="0")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True,
                         text=True, check=True).stdout.strip()
    assert out == "1"
