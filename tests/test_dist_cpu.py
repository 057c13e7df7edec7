"""Multi-process (gloo, CPU) tests of the N > 1 host logic.

The GPU pipeline (api.cpp run_pipeline) is driven by three pieces of host arithmetic exported
through the C ABI: the row partition (giga_partition), the K-chunk plan of the B broadcast
(giga_pipeline_plan) and the C gather blocks (giga_plan_block). Here world-size 2 and 3 process
groups execute exactly that schedule with gloo collectives standing in for NCCL and the CPU
oracle standing in for the shard GEMM (accumulated K-chunk by K-chunk as the GPU does), and
every rank must end with the full C of the one-shot oracle. This checks that the schedule
covers every row once, that all ranks issue matching collectives in the same order (a
mismatch deadlocks or corrupts), and that the ragged last shard is handled.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, M, N, K, dist_name, env, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(env)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        import synth
        from paper_2504_01266_b200 import giga

        r0, rows = giga.partition(M, world, rank)
        A = synth.gen_rows(r0, rows, K, synth.MATRIX_A, dist_name)
        B = (synth.gen_matrix(K, N, synth.MATRIX_B, dist_name) if rank == 0
             else np.full((K, N), np.nan, np.float32))
        kb, rchunks = giga.pipeline_plan(M, N, K, world)
        assert kb[0] == 0 and kb[-1] == K and all(b > a for a, b in zip(kb, kb[1:]))
        Bt = torch.from_numpy(B)
        C = np.full((M, N), np.nan, np.float64)
        Cs = np.zeros((rows, N), np.float64)
        for c in range(len(kb) - 1):  # broadcast chunk c, then accumulate its product
            dist.broadcast(Bt[kb[c]:kb[c + 1]], src=0)
            if rows:
                part, _ = oracle.gemm(np.ascontiguousarray(A[:, kb[c]:kb[c + 1]]),
                                      np.ascontiguousarray(B[kb[c]:kb[c + 1]]), want_s=False)
                Cs += part
        C[r0:r0 + rows] = Cs
        Ct = torch.from_numpy(C)
        for qq in range(rchunks):  # gather rounds: every owner broadcasts its block
            for o in range(world):
                b0, brows = giga.plan_block(M, world, rchunks, o, qq)
                if brows:
                    dist.broadcast(Ct[b0:b0 + brows], src=o)
        full, _ = oracle.gemm(synth.gen_matrix(M, K, synth.MATRIX_A, dist_name),
                              synth.gen_matrix(K, N, synth.MATRIX_B, dist_name), want_s=False)
        if dist_name == "d3":
            ok = bool(np.array_equal(C, full))
        else:
            ok = bool(np.allclose(C, full, rtol=0, atol=1e-9 * np.abs(full).max()))
        q.put((rank, ok, rchunks, len(kb) - 1))
        dist.destroy_process_group()
    except Exception as e:  # surface the failure to the parent
        q.put((rank, repr(e), None, None))


def _run(world, M, N, K, dist_name, env):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, M, N, K, dist_name, env, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    return sorted(res)


@pytest.mark.parametrize("world,M,N,K,dist_name,env", [
    (2, 520, 64, 1040, "d3", {"GIGA_BCAST_CHUNKS": "3", "GIGA_GATHER_CHUNKS": "2"}),
    (3, 1031, 36, 2048, "d2", {"GIGA_BCAST_CHUNKS": "4", "GIGA_GATHER_CHUNKS": "4"}),
    (2, 7, 12, 40, "d3", {}),
])
def test_pipeline_schedule_reconstructs_c(world, M, N, K, dist_name, env):
    res = _run(world, M, N, K, dist_name, env)
    for rank, ok, rchunks, kchunks in res:
        assert ok is True, (rank, ok)


def test_plan_blocks_cover_every_row_once():
    from paper_2504_01266_b200 import giga
    for M, world in [(1, 1), (5, 8), (16384, 8), (1031, 3), (262144, 8)]:
        for rchunks in (1, 2, 3, 4):
            seen = np.zeros(M, np.int64)
            for o in range(world):
                r0, rows = giga.partition(M, world, o)
                got = 0
                for q in range(rchunks):
                    b0, brows = giga.plan_block(M, world, rchunks, o, q)
                    assert brows >= 0 and r0 <= b0 and b0 + brows <= r0 + rows
                    seen[b0:b0 + brows] += 1
                    got += brows
                assert got == rows
            assert np.all(seen == 1)


def test_plan_knobs_and_limits(monkeypatch):
    from paper_2504_01266_b200 import giga
    monkeypatch.delenv("GIGA_TRANSPORT", raising=False)
    kb, rc = giga.pipeline_plan(16384, 16384, 16384, 8)
    sizes = np.diff(kb)
    # each chunk is a GEMM launch whose rate falls with its depth (3xFP16 ~460 k / (k + 530)
    # TFLOP/s, profiles/r02_chunk_rate_sweep_b.jsonl): c3 at 8 takes 2..6 (the cap) chunks
    assert 3 <= len(kb) <= 7 and rc == 4 and all(b % 16 == 0 for b in kb) and kb[-1] == 16384
    # small first chunk, then growing -- or equal chunks when B's transfer (8 NCCL CTAs,
    # ~400 GB/s modelled) is barely faster than the 3xFP16 shard GEMM consumes it (c3 at 8)
    assert sizes[0] >= 256 and np.all(np.diff(sizes) >= -16)
    kb2, _ = giga.pipeline_plan(32768, 32768, 32768, 8)
    assert np.all(np.diff(np.diff(kb2)) > 0)  # c5 at 8: geometric growth
    blocks = [giga.plan_block(16384, 8, rc, 3, q)[1] for q in range(rc)]
    assert np.all(np.diff(blocks) <= 0) and blocks[-1] < blocks[0]  # largest gather first
    # the p2p chain pays (world - 1) hops of the first chunk: at least as many, smaller chunks
    nccl = giga.pipeline_plan(32768, 32768, 32768, 8)[0]
    monkeypatch.setenv("GIGA_TRANSPORT", "p2p")
    p2p = giga.pipeline_plan(32768, 32768, 32768, 8)[0]
    assert len(p2p) >= len(nccl) and p2p[1] <= nccl[1]
    monkeypatch.delenv("GIGA_TRANSPORT")
    # a small problem (the paper's 4096^3 on two GPUs) takes fewer launches than the caps
    kb, rc = giga.pipeline_plan(4096, 4096, 4096, 2)
    assert 2 <= len(kb) - 1 < 6 and rc < 4
    # the tall-skinny c4: B is 4 MiB (no chunking pays), the 896 MiB gather is row-chunked
    kb, rc = giga.pipeline_plan(262144, 1024, 1024, 8)
    assert kb == [0, 1024] and rc == 4
    monkeypatch.setenv("GIGA_BCAST_CHUNKS", "16")
    monkeypatch.setenv("GIGA_GATHER_CHUNKS", "1")
    kb, rc = giga.pipeline_plan(4096, 4096, 4096, 2)
    assert len(kb) == 17 and rc == 1 and np.all(np.diff(kb) >= 256)  # >= 256 deep per chunk
    kb, rc = giga.pipeline_plan(64, 6, 6, 2)  # unaligned shapes: a single chunk of each
    assert kb == [0, 6] and rc == 1
    with pytest.raises(giga.GigaError):
        giga.plan_block(10, 2, 2, 2, 0)
