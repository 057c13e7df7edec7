"""Multi-GPU schedules on "virtual GPUs": giga_init_devices([0, 0, ...]) gives several library
GPUs on one device, each with its own streams, workspace and buffers, so the N > 1 code paths
run unchanged on a one-GPU box (copies become device-local). NCCL refuses repeated devices, so
these exercise the peer-to-peer transport (copy-engine chain broadcast of B + the gather fused
into the GEMM epilogue) and the host-summed dot; the NCCL pipeline itself is covered at world
size 1 in test_gpu.py (GIGA_FORCE_COMM) and by the gloo schedule tests.
"""
import numpy as np
import pytest

import oracle
from oracle.check import check_close, check_exact
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


@pytest.fixture
def giga_virtual(torch_cuda):
    from paper_2504_01266_b200 import build
    build.build()
    from paper_2504_01266_b200 import giga as g
    made = []

    def make(n):
        g.finalize()
        g.init_devices([0] * n)
        made.append(n)
        return g

    yield make
    g.finalize()


def _shards(torch, A, world, giga):
    out = []
    for r in range(world):
        r0, rows = giga.partition(A.shape[0], world, r)
        out.append(torch.from_numpy(np.ascontiguousarray(A[r0:r0 + rows])).cuda()
                   if rows else torch.empty(0, device="cuda"))
    return out


@pytest.mark.parametrize("world,M,N,K,dist", [(2, 1000, 520, 1040, "d3"), (3, 1031, 256, 2064, "d3"),
                                               (4, 4096, 1024, 2048, "d1"), (2, 3, 8, 520, "d3"),
                                               (8, 2048, 512, 1024, "d2")])
def test_p2p_transport_fused_gather(giga_virtual, torch_cuda, monkeypatch, world, M, N, K, dist):
    torch = torch_cuda
    monkeypatch.setenv("GIGA_TRANSPORT", "p2p")
    monkeypatch.setenv("GIGA_BCAST_CHUNKS", "3")
    giga = giga_virtual(world)
    A = synth.gen_matrix(M, K, synth.MATRIX_A, dist)
    B = synth.gen_matrix(K, N, synth.MATRIX_B, dist)
    A_sh = _shards(torch, A, world, giga)
    B_bufs = [torch.from_numpy(B).cuda()] + [torch.full((K, N), float("nan"), device="cuda")
                                             for _ in range(world - 1)]
    C_full = [torch.full((M, N), float("nan"), device="cuda") for _ in range(world)]
    giga.matmul_sharded(A_sh, B_bufs, C_full, M, N, K)
    Cref, S = oracle.gemm(A, B)
    for r in range(world):
        assert torch.equal(B_bufs[r], B_bufs[0]), f"B not distributed to rank {r}"
        C = C_full[r].cpu().numpy()
        ok, st = check_exact(C, Cref) if dist == "d3" else check_close(C, Cref, S)
        assert ok, (r, st)
    # every rank's copy is identical (one writer per block, same bits everywhere)
    for r in range(1, world):
        assert torch.equal(C_full[r], C_full[0])


def test_nccl_with_repeated_devices_is_refused(giga_virtual, torch_cuda, monkeypatch):
    torch = torch_cuda
    monkeypatch.setenv("GIGA_TRANSPORT", "nccl")
    giga = giga_virtual(2)
    M = N = K = 64
    A = torch.ones(M, K, device="cuda")
    bufs = [torch.ones(K, N, device="cuda"), torch.empty(K, N, device="cuda")]
    C = [torch.empty(M, N, device="cuda") for _ in range(2)]
    with pytest.raises(giga.GigaError) as e:
        giga.matmul_sharded([A[:32].contiguous(), A[32:].contiguous()], bufs, C, M, N, K)
    assert e.value.status == "GIGA_ERR_COMM"


@pytest.mark.parametrize("world", [2, 3, 8])
def test_dot_over_virtual_gpus(giga_virtual, torch_cuda, world):
    giga = giga_virtual(world)
    n = (1 << 21) + 13
    x = synth.gen_vector(n, synth.VECTOR_X, "d3")
    y = synth.gen_vector(n, synth.VECTOR_Y, "d3")
    assert giga.dot(x, y, ngpus=world) == oracle.dot(x, y)[0]
    xd, yd = torch_cuda.from_numpy(x).cuda(), torch_cuda.from_numpy(y).cuda()
    assert giga.dot(xd, yd, ngpus=world) == oracle.dot(x, y)[0]


# ---- rank API (one process per rank) with the peer-to-peer transport ----------------------

def _rank_worker(rank, world, port, M, N, K, q, transport="p2p", own_device=False,
                 extra_env=None):
    import os
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update({"GIGA_TRANSPORT": transport, "GIGA_BCAST_CHUNKS": "3",
                       "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    os.environ.update(extra_env or {})
    try:
        import torch
        import torch.distributed as dist
        import oracle
        import synth
        from paper_2504_01266_b200 import giga
        dist.init_process_group("gloo", rank=rank, world_size=world)
        dev = rank if own_device else 0
        torch.cuda.set_device(dev)
        if transport == "nccl":  # the NCCL id travels over the gloo group (plumbing)
            obj = [giga.comm_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            giga.rank_init(rank, world, dev, obj[0])
        else:
            giga.rank_init(rank, world, dev, None)
        r0, rows = giga.partition(M, world, rank)
        A = synth.gen_rows(r0, rows, K, synth.MATRIX_A, "d3")
        Bn = synth.gen_matrix(K, N, synth.MATRIX_B, "d3")
        dA = torch.from_numpy(A).cuda() if rows else torch.empty(0, device="cuda")
        dB = torch.from_numpy(Bn).cuda() if rank == 0 else torch.full((K, N), float("nan"),
                                                                      device="cuda")
        dC = torch.full((M, N), float("nan"), device="cuda")
        if transport == "p2p":
            blob = giga.p2p_export(dB, dC)
            blobs = [None] * world
            dist.all_gather_object(blobs, blob)
            giga.p2p_import(blobs)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        for _ in range(3):  # repeated calls: flag call numbers and back-pressure
            giga.matmul_rank(dA, dB, dC, M, N, K, stream=s)
        s.synchronize()
        Cref, _ = oracle.gemm(synth.gen_matrix(M, K, synth.MATRIX_A, "d3"), Bn)
        ok_c = bool(np.array_equal(dC.cpu().numpy().astype(np.float64), Cref))
        ok_b = bool(np.array_equal(dB.cpu().numpy(), Bn))
        n = 100003
        x = synth.gen_vector(n, synth.VECTOR_X, "d3")
        y = synth.gen_vector(n, synth.VECTOR_Y, "d3")
        x0, xr = giga.partition(n, world, rank)
        xs = torch.from_numpy(x[x0:x0 + xr]).cuda()
        ys = torch.from_numpy(y[x0:x0 + xr]).cuda()
        dots = [giga.dot_rank(xs, ys, n, stream=s) for _ in range(2)]
        ok_d = all(v == oracle.dot(x, y)[0] for v in dots)
        dist.barrier()
        giga.finalize()
        q.put((rank, ok_c, ok_b, ok_d, ""))
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        q.put((rank, False, False, False, repr(e)))


@pytest.mark.parametrize("world,M,N,K,scheme,store", [(2, 1000, 520, 1040, None, None),
                                                      (3, 517, 256, 2064, None, None),
                                                      (2, 1000, 520, 2064, "3xfp16", None),
                                                      (3, 517, 256, 2064, "3xfp16", None),
                                                      (3, 517, 256, 2064, None, "vec"),
                                                      (2, 1000, 520, 2064, "3xfp16", "vec")])
def test_rank_p2p_across_processes(torch_cuda, world, M, N, K, scheme, store):
    """Processes sharing cuda:0 through the rank API, p2p transport; with $GIGA_SCHEME=3xfp16
    the load-C epilogue, the operand scales and the A-side fix's mirror writes go into the
    peers' C_full through CUDA IPC; with $GIGA_P2P_STORE=vec the epilogue writes them with
    16-byte stores (the multicast gather's code path, one store per peer)."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    env = {}
    if scheme:
        env["GIGA_SCHEME"] = scheme
    if store:
        env["GIGA_P2P_STORE"] = store
    procs = [ctx.Process(target=_rank_worker,
                         args=(r, world, port, M, N, K, q, "p2p", False, env))
             for r in range(world)]
    for p in procs:
        p.start()
    try:
        res = sorted(q.get(timeout=240) for _ in range(world))
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for rank, ok_c, ok_b, ok_d, err in res:
        assert ok_c and ok_b and ok_d, (rank, ok_c, ok_b, ok_d, err)


def _rank_worker_changing(rank, world, port, M, N, K, q):
    """Inputs change on every call and each rank reads its C_full between calls on its own
    stream; rank 1 reads late (a long sleep first). Without the started[] flags of the p2p
    transport, rank 0's next call writes its rows into rank 1's C_full before rank 1 has read
    the previous result."""
    import os
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update({"GIGA_TRANSPORT": "p2p", "GIGA_BCAST_CHUNKS": "3",
                       "MASTER_ADDR": "127.0.0.1", "MASTER_PORT": str(port)})
    try:
        import torch
        import torch.distributed as dist
        import oracle
        import synth
        from paper_2504_01266_b200 import giga
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        giga.rank_init(rank, world, 0, None)
        r0, rows = giga.partition(M, world, rank)
        dA = torch.empty((max(rows, 1), K), device="cuda")
        dB = torch.full((K, N), float("nan"), device="cuda")
        dC = torch.full((M, N), float("nan"), device="cuda")
        blobs = [None] * world
        dist.all_gather_object(blobs, giga.p2p_export(dB, dC))
        giga.p2p_import(blobs)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        calls = 4
        As = [synth.gen_matrix(M, K, 10 + c, "d3") for c in range(calls)]
        Bs = [synth.gen_matrix(K, N, 20 + c, "d3") for c in range(calls)]
        snaps = []
        with torch.cuda.stream(s):
            for c in range(calls):
                dA[:rows].copy_(torch.from_numpy(As[c][r0:r0 + rows]))
                if rank == 0:
                    dB.copy_(torch.from_numpy(Bs[c]))
                giga.matmul_rank(dA, dB, dC, M, N, K, stream=s)
                if rank == 1:
                    torch.cuda._sleep(200_000_000)  # a slow consumer of call c's C_full
                snaps.append(dC.clone())
        s.synchronize()
        ok = []
        for c in range(calls):
            Cref, _ = oracle.gemm(As[c], Bs[c])
            ok.append(bool(np.array_equal(snaps[c].cpu().numpy().astype(np.float64), Cref)))
        dist.barrier()
        giga.finalize()
        q.put((rank, all(ok), str(ok)))
        dist.destroy_process_group()
    except Exception as e:  # noqa: BLE001
        q.put((rank, False, repr(e)))


def test_rank_p2p_changing_inputs_slow_consumer(torch_cuda):
    import socket
    import torch.multiprocessing as mp
    world, M, N, K = 2, 1024, 512, 1040
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_worker_changing, args=(r, world, port, M, N, K, q))
             for r in range(world)]
    for p in procs:
        p.start()
    try:
        res = sorted(q.get(timeout=240) for _ in range(world))
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for rank, ok, detail in res:
        assert ok, (rank, detail)


def test_rank_p2p_without_registration_refuses(torch_cuda, monkeypatch):
    """world > 1 over the p2p transport but no giga_rank_p2p_export / import: the call must
    fail, not compute only this rank's rows; the dot likewise."""
    torch = torch_cuda
    from paper_2504_01266_b200 import giga
    monkeypatch.setenv("GIGA_TRANSPORT", "p2p")
    giga.finalize()
    giga.rank_init(0, 2, 0, None)
    try:
        M, N, K = 512, 256, 256
        dA = torch.ones((256, K), device="cuda")
        dB = torch.ones((K, N), device="cuda")
        dC = torch.zeros((M, N), device="cuda")
        with pytest.raises(giga.GigaError) as e:
            giga.matmul_rank(dA, dB, dC, M, N, K)
        assert e.value.status == "GIGA_ERR_NOT_INITIALIZED"
        x = torch.ones(100, device="cuda")
        with pytest.raises(giga.GigaError) as e:
            giga.dot_rank(x, x, 200)
        assert e.value.status == "GIGA_ERR_NOT_INITIALIZED"
        # the transport is fixed at rank_init: changing the variable later changes nothing
        monkeypatch.setenv("GIGA_TRANSPORT", "nccl")
        with pytest.raises(giga.GigaError) as e:
            giga.matmul_rank(dA, dB, dC, M, N, K)
        assert e.value.status == "GIGA_ERR_NOT_INITIALIZED"
    finally:
        giga.finalize()


def test_bench_two_ranks_on_one_device(torch_cuda):
    """bench.py's N > 1 path end to end under torchrun (2 ranks sharing cuda:0, gloo plumbing,
    p2p transport): rank init, IPC registration, max-over-ranks timing, one JSON line."""
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
         "--e2e-steps", "1"], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [x for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["transport"] == "p2p" and d["value"] > 0
    assert d["e2e"]["value"] > 0 and d["gpu_launches"] > 0


@pytest.mark.parametrize("world,M,N,K", [(2, 777, 520, 1040), (4, 1000, 256, 2048)])
def test_host_buffers_p2p_virtual(giga_virtual, torch_cuda, monkeypatch, world, M, N, K):
    """giga_matmul with host buffers over several (virtual) GPUs: per-GPU H2D of the A rows,
    B to GPU 0 then down the copy-engine chain, each GPU copies its own C rows home."""
    monkeypatch.setenv("GIGA_TRANSPORT", "p2p")
    giga = giga_virtual(world)
    A = synth.gen_matrix(M, K, synth.MATRIX_A, "d3")
    B = synth.gen_matrix(K, N, synth.MATRIX_B, "d3")
    C = np.full((M, N), np.nan, np.float32)
    giga.matmul(A, B, C, M, N, K, world)
    Cref, _ = oracle.gemm(A, B)
    ok, st = check_exact(C, Cref)
    assert ok, st


def test_rank_worker_nccl_world1(torch_cuda):
    """The NCCL branch of the rank worker the physical-GPU tests use (unique id over gloo,
    rank_init with the id, pipeline with a communicator: GIGA_FORCE_COMM) at world size 1."""
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_rank_worker, args=(0, 1, port, 1000, 520, 2064, q, "nccl", True,
                                               {"GIGA_FORCE_COMM": "1"}))
    p.start()
    try:
        rank, ok_c, ok_b, ok_d, err = q.get(timeout=240)
    finally:
        p.join(timeout=30)
        if p.is_alive():
            p.kill()
    assert ok_c and ok_b and ok_d, err


# ---- physical GPUs (skipped on a one-GPU box; run as they are on a multi-GPU one) ----------

def _ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


multi = pytest.mark.skipif(_ngpus() < 2, reason="needs at least two physical GPUs")


@multi
@pytest.mark.parametrize("transport", ["nccl", "p2p"])
def test_rank_api_physical_gpus(torch_cuda, transport):
    """One process per GPU on distinct devices: NCCL pipeline or p2p transport (IPC, TMA
    stores into peer memory), repeated calls, B distribution, C gather, dot all-reduce."""
    import socket
    import torch.multiprocessing as mp
    world = min(4, _ngpus())
    M, N, K = 1000 * world + 7, 520, 2064
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_worker, args=(r, world, port, M, N, K, q, transport, True))
             for r in range(world)]
    for p in procs:
        p.start()
    try:
        res = sorted(q.get(timeout=300) for _ in range(world))
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for rank, ok_c, ok_b, ok_d, err in res:
        assert ok_c and ok_b and ok_d, (rank, ok_c, ok_b, ok_d, err)


@multi
@pytest.mark.parametrize("transport", ["nccl", "p2p"])
def test_single_process_physical_gpus(torch_cuda, monkeypatch, transport):
    """giga_init(g) over g distinct devices, device-resident shards: every GPU ends with all of
    C, bit-exact on integer inputs."""
    torch = torch_cuda
    from paper_2504_01266_b200 import giga
    monkeypatch.setenv("GIGA_TRANSPORT", transport)
    world = min(4, _ngpus())
    M, N, K = 777 * world, 516, 1040
    A = synth.gen_matrix(M, K, synth.MATRIX_A, "d3")
    B = synth.gen_matrix(K, N, synth.MATRIX_B, "d3")
    giga.finalize()
    giga.init(world)
    try:
        shards, Bs, Cs = [], [], []
        for r in range(world):
            r0, rows = giga.partition(M, world, r)
            dev = torch.device("cuda", r)
            shards.append(torch.from_numpy(np.ascontiguousarray(A[r0:r0 + rows])).to(dev))
            Bs.append(torch.from_numpy(B).to(dev) if r == 0 else
                      torch.full((K, N), float("nan"), device=dev))
            Cs.append(torch.full((M, N), float("nan"), device=dev))
        giga.matmul_sharded(shards, Bs, Cs, M, N, K)
        Cref, _ = oracle.gemm(A, B)
        for r in range(world):
            assert check_exact(Cs[r].cpu().numpy(), Cref)[0], r
        C = np.empty((M, N), np.float32)
        giga.matmul(A, B, C, M, N, K, world)  # host buffers over the same GPUs
        assert check_exact(C, Cref)[0]
    finally:
        giga.finalize()


@multi
@pytest.mark.parametrize("transport", ["nccl", "p2p"])
def test_bench_physical_gpus(torch_cuda, transport):
    """bench.py under torchrun on two distinct GPUs: one JSON line, max-over-ranks timing."""
    import json
    import os
    import socket
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    out = subprocess.run(
        [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
         "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2",
         "--steps", "3", "--warmup", "3", "--config", "c2_4096", "--no-cpu-baseline",
         "--e2e-steps", "1", "--transport", transport], cwd=root, capture_output=True,
        text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [x for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["transport"] == transport and d["value"] > 0
