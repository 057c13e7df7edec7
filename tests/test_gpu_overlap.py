"""Is parallelism working? (S6.1): the copy engines move B
down the peer-to-peer chain while the tensor cores run GEMMs, on the device's own clock.

$GIGA_TRACE=1 makes the p2p transport stamp %globaltimer right before and after every chain
copy (a one-thread kernel on the copy stream) and record every GEMM launch's CTA start / end
times; the timeline line of each (virtual) GPU carries them under "ns". Three virtual GPUs share
cuda:0 (one clock): GPU 0 owns B and starts its GEMMs at once, GPUs 1 and 2 copy B's K-chunks
from their upstream neighbour. At least one chain copy must run inside the interval of some
GEMM launch, and every GPU's GEMM of K-chunk c must start after its own copy of chunk c ends
(the chain's ordering), with C still exact.
"""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_CODE = r'''
import sys, os
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import oracle, synth
from oracle.check import check_exact
from paper_2504_01266_b200 import giga
world, M, N, K = 3, 6144, 4096, 8192
A = synth.gen_matrix(M, K, synth.MATRIX_A, "d3")
B = synth.gen_matrix(K, N, synth.MATRIX_B, "d3")
giga.init_devices([0] * world)
shards = []
for r in range(world):
    r0, rows = giga.partition(M, world, r)
    shards.append(torch.from_numpy(np.ascontiguousarray(A[r0:r0 + rows])).cuda())
Bb = [torch.from_numpy(B).cuda()] + [torch.zeros((K, N), device="cuda") for _ in range(world - 1)]
Cf = [torch.full((M, N), float("nan"), device="cuda") for _ in range(world)]
for _ in range(2):  # the second call is the traced one that counts (warm workspaces)
    giga.matmul_sharded(shards, Bb, Cf, M, N, K)
Cref, _ = oracle.gemm(A[:64], B)
for c in Cf:
    ok, st = check_exact(c[:64].cpu().numpy(), Cref)
    assert ok, st
giga.finalize()
print("ok")
'''


def test_chain_copies_overlap_gemms():
    env = dict(os.environ, GIGA_TRACE="1", GIGA_TRANSPORT="p2p", GIGA_BCAST_CHUNKS="4")
    r = subprocess.run([sys.executable, "-c", _CODE], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stderr.splitlines()
             if x.startswith("{") and '"trace": "p2p"' in x]
    assert len(lines) >= 6, r.stderr[-2000:]
    last = {}
    for ln in lines:  # keep each GPU's last (second-call) timeline
        last[int(ln["meta"]["rank"])] = ln
    assert sorted(last) == [0, 1, 2]
    gemms, copies = [], []
    for rank, ln in last.items():
        ns = ln["ns"]
        g = ns["gemm_cta"]
        assert len(g) == ln["meta"]["kchunks"] and all(s < e for s, e in g)
        gemms += [(rank, s, e) for s, e in g]
        if rank > 0:
            b, e = ns["copy_begin"], ns["copy_end"]
            assert len(b) == len(e) == ln["meta"]["kchunks"]
            copies += [(rank, c, b0, e0) for c, (b0, e0) in enumerate(zip(b, e))]
            # the chain's ordering: this GPU's GEMM of chunk c starts after its copy of c
            for c, (s, _) in enumerate(g):
                assert s >= e[c], (rank, c, s, e[c])
    overlaps = [(cr, c, gr) for cr, c, b0, e0 in copies for gr, s, e in gemms
                if max(b0, s) < min(e0, e)]
    report = {"gemm_launches": len(gemms), "copies": len(copies),
              "copy_gemm_overlaps": len(overlaps),
              "copy_ns": [e0 - b0 for _, _, b0, e0 in copies],
              "gemm_ns": [e - s for _, s, e in gemms]}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "overlap.json"), "w") as f:
        json.dump({"report": report, "timelines": list(last.values())}, f, indent=1)
    print("overlap:", report)
    assert overlaps, report
