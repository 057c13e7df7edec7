"""The fused gather's store paths (the gather is a concatenation of the row
blocks, PAPER.md:218 S4.2.3 / PAPER.md:291 S4.2.7):

* store_mode 0 -- TMA bulk stores to C and every peer (the p2p transport's default);
* store_mode 1 -- 16-byte st.global stores from the epilogue's staging tile, once per
  destination ($GIGA_P2P_STORE=vec);
* store_mode 2 -- 16-byte multimem.st to the multicast team address, ONCE (giga_mc_alloc /
  giga_rank_mc_bind buffers). On sm_100a multimem.st and st.global assemble to the same
  STG.E.128 (the multicast is in the address), so given an ordinary address the mode writes
  that buffer alone: the tests check its addressing, clipping and the 3xFP16 fixes that way.

This pool refuses cuMulticastCreate (profiles/r02_nvls_probe.jsonl): the team allocators are
checked to fail cleanly (GIGA_ERR_UNSUPPORTED) and the multi-GPU team test skips on one GPU.
"""
import numpy as np
import pytest

import oracle
from oracle.check import check_close, check_exact
import synth

pytestmark = pytest.mark.gpu

CANARY = np.uint32(0x7FC0DEAD)  # a NaN payload no kernel produces


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


@pytest.fixture
def giga(torch_cuda):
    from paper_2504_01266_b200 import build
    build.build()
    from paper_2504_01266_b200 import giga as g
    g.finalize()
    yield g
    g.finalize()


def _canvas(torch, M, ldc, extra_rows=3):
    """A (M + extra_rows) x ldc buffer of canary bits; the product goes into its top-left
    M x N block, everything else must stay untouched."""
    buf = np.full((M + extra_rows, ldc), CANARY, np.uint32).view(np.float32)
    return torch.from_numpy(buf).cuda()


def _check_canvas(t, M, N):
    h = t.cpu().numpy()
    bits = h.view(np.uint32)
    assert (bits[M:] == CANARY).all(), "rows below M written"
    assert (bits[:M, N:] == CANARY).all(), "columns right of N written"
    return np.ascontiguousarray(h[:M, :N])


def _exception_inputs(M, N, K, seed):
    """Rows of A / columns of B whose small elements are 3xFP16 exceptions (the epilogue's
    B-side fix and the A-side fix kernel both run), mixed with ordinary data."""
    rng = np.random.default_rng(seed)
    A = rng.uniform(-1, 1, (M, K)).astype(np.float32)
    B = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    ma = rng.random((M, K)) < 0.01
    mb = rng.random((K, N)) < 0.01
    A[ma] *= (2.0 ** -rng.integers(24, 40, ma.sum())).astype(np.float32)
    B[mb] *= (2.0 ** -rng.integers(24, 40, mb.sum())).astype(np.float32)
    return A, B


CASES = [
    # M, N, K, ldc, terms, inputs
    (300, 260, 520, 264, 3, "d3"),      # ragged rows / columns, CTA-pair or single tiles
    (1000, 1024, 2048, 1024, 3, "d1"),
    (777, 516, 1040, 520, 2, "d1"),     # TF32 + BF16
    (1100, 1040, 3000, 1044, 4, "exc"),  # 3xFP16 with exceptions on both sides
    (2100, 1024, 4096, 1024, 0, "d2"),   # the product path's own scheme choice
    (5, 8, 16, 8, 3, "d3"),              # one partial tile
]


@pytest.mark.parametrize("M,N,K,ldc,terms,dist", CASES)
def test_store_modes_bit_identical(giga, torch_cuda, M, N, K, ldc, terms, dist):
    """Every store mode writes the same bits to every destination, nothing outside M x N."""
    torch = torch_cuda
    if dist == "exc":
        A, B = _exception_inputs(M, N, K, 5)
    else:
        A = synth.gen_matrix(M, K, synth.MATRIX_A, dist)
        B = synth.gen_matrix(K, N, synth.MATRIX_B, dist)
    dA, dB = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
    outs = {}
    for mode, npeer in ((0, 2), (1, 2), (2, 0)):
        C = _canvas(torch, M, ldc)
        peers = [_canvas(torch, M, ldc) for _ in range(npeer)]
        giga.gemm_gather_ex(dA, dB, C, peers, M, N, K, ldc=ldc, terms=terms, store_mode=mode)
        torch.cuda.synchronize()
        res = [_check_canvas(t, M, N) for t in [C] + peers]
        for r in res[1:]:
            assert np.array_equal(r.view(np.uint32), res[0].view(np.uint32)), mode
        outs[mode] = res[0]
    for mode in (1, 2):
        assert np.array_equal(outs[mode].view(np.uint32), outs[0].view(np.uint32)), mode
    Cref, S = oracle.gemm(A, B)
    ok, st = check_exact(outs[0], Cref) if dist == "d3" else check_close(outs[0], Cref, S)
    assert ok, st


def test_store_mode_rejects_bad_arguments(giga, torch_cuda):
    torch = torch_cuda
    a = torch.ones((64, 64), device="cuda")
    c = torch.empty((64, 64), device="cuda")
    with pytest.raises(giga.GigaError) as e:  # multicast mode has no peer list
        giga.gemm_gather_ex(a, a, c, [torch.empty_like(c)], 64, 64, 64, store_mode=2)
    assert e.value.status == "GIGA_ERR_INVALID_ARG"
    with pytest.raises(giga.GigaError) as e:
        giga.gemm_gather_ex(a, a, c, [], 64, 64, 64, store_mode=3)
    assert e.value.status == "GIGA_ERR_INVALID_ARG"


@pytest.mark.parametrize("world,M,N,K,dist", [(2, 1000, 520, 1040, "d3"),
                                               (3, 1031, 256, 2064, "d1"),
                                               (4, 4096, 1024, 2048, "d2")])
def test_p2p_vec_store_fused_gather(giga, torch_cuda, monkeypatch, world, M, N, K, dist):
    """$GIGA_P2P_STORE=vec on virtual GPUs: the transport's last K-chunk writes every peer's
    C_full with 16-byte stores (the multicast gather's code path, one store per peer)."""
    torch = torch_cuda
    monkeypatch.setenv("GIGA_TRANSPORT", "p2p")
    monkeypatch.setenv("GIGA_P2P_STORE", "vec")
    monkeypatch.setenv("GIGA_BCAST_CHUNKS", "3")
    giga.init_devices([0] * world)
    A = synth.gen_matrix(M, K, synth.MATRIX_A, dist)
    B = synth.gen_matrix(K, N, synth.MATRIX_B, dist)
    shards = []
    for r in range(world):
        r0, rows = giga.partition(M, world, r)
        shards.append(torch.from_numpy(np.ascontiguousarray(A[r0:r0 + rows])).cuda())
    Bb = [torch.from_numpy(B).cuda()] + [torch.zeros((K, N), device="cuda")
                                         for _ in range(world - 1)]
    Cf = [torch.full((M, N), float("nan"), device="cuda") for _ in range(world)]
    giga.matmul_sharded(shards, Bb, Cf, M, N, K)
    Cref, S = oracle.gemm(A, B)
    for c in Cf:
        h = c.cpu().numpy()
        ok, st = check_exact(h, Cref) if dist == "d3" else check_close(h, Cref, S)
        assert ok, st
    for c in Cf[1:]:
        assert torch.equal(c, Cf[0])


def test_mc_alloc_on_this_pool(giga, torch_cuda):
    """giga_mc_alloc on one device: a team of one where the driver allows multicast (then the
    buffer is zero-filled device memory the GEMM can write), GIGA_ERR_UNSUPPORTED with the
    driver's reason where it does not (this pool)."""
    torch = torch_cuda
    giga.init(1)
    nbytes = 256 * 256 * 4
    try:
        ptrs = giga.mc_alloc(1, nbytes)
    except giga.GigaError as e:
        assert e.status == "GIGA_ERR_UNSUPPORTED", str(e)
        assert "multicast" in str(e).lower()
        return
    c = giga.as_float_tensor(ptrs[0], 256 * 256, torch.device("cuda", 0)).view(256, 256)
    assert torch.count_nonzero(c).item() == 0
    a = torch.ones((256, 256), device="cuda")
    giga.gemm_gather_ex(a, a, c, [], 256, 256, 256, terms=3, store_mode=0)
    torch.cuda.synchronize()
    assert torch.all(c == 256.0).item()
    giga.mc_free(ptrs[0])


def test_mc_alloc_refuses_repeated_devices(giga, torch_cuda):
    giga.init_devices([0, 0])
    with pytest.raises(giga.GigaError) as e:
        giga.mc_alloc(2, 1 << 20)
    assert e.value.status == "GIGA_ERR_INVALID_ARG"
    with pytest.raises(giga.GigaError) as e:
        giga.mc_free(12345)
    assert e.value.status == "GIGA_ERR_INVALID_ARG"


def test_mc_team_fused_gather_physical(giga, torch_cuda, monkeypatch):
    """The multicast gather across physical GPUs: C_full from giga_mc_alloc, the last
    K-chunk's epilogue writes each piece once to the team address. Needs >= 2 GPUs and a
    driver that creates multicast objects (NVSwitch + fabric manager)."""
    torch = torch_cuda
    world = torch.cuda.device_count()
    if world < 2:
        pytest.skip("one GPU: no multicast team across devices")
    world = min(world, 8)
    monkeypatch.setenv("GIGA_TRANSPORT", "p2p")
    giga.init(world)
    M, N, K = 4100, 2048, 4096
    try:
        ptrs = giga.mc_alloc(world, M * N * 4)
    except giga.GigaError as e:
        if e.status == "GIGA_ERR_UNSUPPORTED":
            pytest.skip(str(e))
        raise
    A = synth.gen_matrix(M, K, synth.MATRIX_A, "d1")
    B = synth.gen_matrix(K, N, synth.MATRIX_B, "d1")
    shards, Bb, Cf = [], [], []
    for r in range(world):
        dev = torch.device("cuda", r)
        r0, rows = giga.partition(M, world, r)
        shards.append(torch.from_numpy(np.ascontiguousarray(A[r0:r0 + rows])).to(dev))
        Bb.append(torch.from_numpy(B).to(dev) if r == 0 else torch.zeros((K, N), device=dev))
        Cf.append(giga.as_float_tensor(ptrs[r], M * N, dev).view(M, N))
    giga.matmul_sharded(shards, Bb, Cf, M, N, K)
    Cref, S = oracle.gemm(A, B)
    ref0 = Cf[0].cpu()
    ok, st = check_close(ref0.numpy(), Cref, S)
    assert ok, st
    for c in Cf[1:]:
        assert torch.equal(c.cpu(), ref0)
    giga.mc_free(ptrs[0])


_RANK_MC = r'''
import os, sys
import torch, torch.distributed as dist
sys.path.insert(0, os.getcwd())
from paper_2504_01266_b200 import giga
rank, world = int(sys.argv[1]), int(sys.argv[2])
dist.init_process_group("gloo", init_method="tcp://127.0.0.1:" + sys.argv[3], rank=rank,
                        world_size=world)
giga.rank_init(rank, world, 0, None)
try:
    p = giga.rank_mc_alloc(1 << 22)
    print("bound", hex(p))
except giga.GigaError as e:
    print("refused", e.status, str(e)[:200])
dist.barrier()
giga.finalize()
dist.destroy_process_group()
'''


def test_rank_mc_alloc_collective_outcome(torch_cuda, tmp_path):
    """The rank API's three-phase team protocol over torch.distributed (two processes on this
    GPU): every rank reaches the same outcome -- all bound, or all refused with the driver's
    reason (this pool) -- and nobody hangs."""
    import os
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, GIGA_TRANSPORT="p2p")
    procs = [subprocess.Popen([sys.executable, "-c", _RANK_MC, str(r), "2", str(port)],
                              cwd=root, env=env, stdout=subprocess.PIPE,
                              stderr=subprocess.PIPE, text=True) for r in range(2)]
    outs = [p.communicate(timeout=300) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e[-2000:]
    words = [o.split()[:2] for o, _ in outs]
    assert words[0][0] == words[1][0] and words[0][0] in ("bound", "refused"), outs
    if words[0][0] == "refused":  # the same status on both ranks (this pool: UNSUPPORTED)
        assert words[0][1] == words[1][1], outs


def test_bench_gather_mc_under_torchrun(torch_cuda):
    """bench.py --transport p2p --gather mc at N = 2 (both ranks on this GPU): the ranks build
    the team collectively or all fall back to the unicast gather, and the line says which."""
    import json
    import os
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    env = dict(os.environ, GIGA_BENCH_ONE_DEVICE="1")
    out = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
         "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2",
         "--steps", "2", "--warmup", "3", "--config", "c2_4096", "--no-cpu-baseline",
         "--e2e-steps", "1", "--transport", "p2p", "--gather", "mc"],
        cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [x for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    g = d["config"]["gather"]
    assert g.startswith("multicast") or g.startswith("unicast (multicast refused"), g
    assert d["value"] > 0
