// pipeline_nccl.cpp -- the multi-GPU row-split matmul over NCCL:
// B broadcast in K-chunks overlapped with accumulating GEMMs, C row blocks gathered.
#include "runtime.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <functional>

namespace giga {

// ---------------------------------------------------------------------------------------
// NCCL

int nccl_check(ncclResult_t r, const char *what) {
  if (r == ncclSuccess) return GIGA_OK;
  const NcclApi *api = nccl_api(nullptr);
  return fail(GIGA_ERR_COMM, "%s failed: %s", what, api ? api->GetErrorString(r) : "?");
}

// Communicator config: NCCL runs beside a persistent GEMM that leaves $GIGA_COMM_SMS (8) SMs
// free, so its kernels are capped at that many CTAs ($GIGA_NCCL_MAX_CTAS overrides; 0 = NCCL
// default) instead of queueing behind the GEMM's CTAs.
ncclConfig_t comm_config() {
  ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
  const int cap = env_int("GIGA_NCCL_MAX_CTAS", env_int("GIGA_COMM_SMS", 8));
  if (cap > 0) cfg.maxCTAs = cap;
  return cfg;
}

int get_comms(int ngpus, std::vector<ncclComm_t> **out) {
  auto it = g.comms.find(ngpus);
  if (it != g.comms.end()) {
    *out = &it->second;
    return GIGA_OK;
  }
  const char *why = nullptr;
  const NcclApi *api = nccl_api(&why);
  if (!api) return fail(GIGA_ERR_COMM, "NCCL unavailable: %s", why ? why : "?");
  ncclUniqueId id;
  TRY(nccl_check(api->GetUniqueId(&id), "ncclGetUniqueId"));
  std::vector<ncclComm_t> comms(ngpus, nullptr);
  TRY(nccl_check(api->GroupStart(), "ncclGroupStart"));
  for (int i = 0; i < ngpus; ++i) {
    CK(cudaSetDevice(g.devs[i].dev));
    ncclConfig_t cfg = comm_config();
    ncclResult_t r = api->CommInitRankConfig(&comms[i], ngpus, id, i, &cfg);
    if (r != ncclSuccess) {
      api->GroupEnd();
      return nccl_check(r, "ncclCommInitRankConfig");
    }
  }
  TRY(nccl_check(api->GroupEnd(), "ncclGroupEnd(init)"));
  g.comms[ngpus] = comms;
  *out = &g.comms[ngpus];
  return GIGA_OK;
}

// Gather the C row blocks so that every rank's C_full holds all of C. Equal blocks: one
// in-place all-gather; otherwise one broadcast per owner (NCCL all-gather needs equal counts).
int gather_rows(const NcclApi *api, ncclComm_t comm, cudaStream_t st, float *C_full, int64_t M,
                int64_t N, int world, int rank) {
  int64_t r0, rows;
  partition_rows(M, world, rank, &r0, &rows);
  if (M % world == 0) {
    return nccl_check(api->AllGather(C_full + r0 * N, C_full, size_t(rows * N), ncclFloat32,
                                     comm, st),
                      "ncclAllGather(C)");
  }
  for (int o = 0; o < world; ++o) {
    int64_t o0, orows;
    partition_rows(M, world, o, &o0, &orows);
    if (orows == 0) continue;
    TRY(nccl_check(api->Broadcast(C_full + o0 * N, C_full + o0 * N, size_t(orows * N),
                                  ncclFloat32, o, comm, st),
                   "ncclBroadcast(C block)"));
  }
  return GIGA_OK;
}

// The GEMM launches of rank `rank` in the pipeline (compute stream `st`): K-chunk c accumulates
// into the rank's rows of C_full (c > 0: C += A_c B_c); the last K-chunk runs in the plan's row
// chunks. before_chunk(c) runs before chunk c's GEMM is enqueued (wait for B chunk c); after(q)
// after row chunk q's GEMM (q = -1: after an earlier, whole K-chunk).
int rank_gemms(const Plan &plan, const GemmExtra &ex, int64_t M, int64_t N, int64_t K, int world,
               int rank, const float *A, const float *Alo, const float *B, const float *Blo,
               float *C_full, cudaStream_t st, const std::function<int(int)> &before_chunk,
               const std::function<int(int)> &after) {
  int64_t r0, rows;
  partition_rows(M, world, rank, &r0, &rows);
  float *Cs = C_full + r0 * N;
  const int64_t *kb = plan.kb;
  for (int c = 0; c < plan.pb; ++c) {
    const int64_t Kc = kb[c + 1] - kb[c];
    TRY(before_chunk(c));
    GemmExtra e = ex;
    e.accumulate = c > 0;
    const float *Bc = B + kb[c] * N, *Bloc = at(Blo, kb[c] * N);
    if (c < plan.pb - 1) {
      if (rows > 0)
        TRY(gemm_chunk(A + kb[c], at(Alo, kb[c]), Bc, Bloc, Cs, rows, N, Kc, e, st));
      TRY(after(-1));
      continue;
    }
    for (int q = 0; q < plan.pc; ++q) {
      int64_t b0, brows;
      plan_block(M, world, plan.pc, rank, q, &b0, &brows);
      const int64_t q0 = b0 - r0;  // offset inside this rank's shard
      e.b_prep_reuse = q > 0;  // the same B chunk for every row chunk
      e.rows_hint = rows;
      if (brows > 0)
        TRY(gemm_chunk(A + q0 * K + kb[c], at(Alo, q0 * K + kb[c]), Bc, Bloc, Cs + q0 * N, brows,
                       N, Kc, e, st));
      TRY(after(q));
    }
  }
  return GIGA_OK;
}

// The SMs the pipeline's GEMMs may use: all but $GIGA_COMM_SMS (8), left to NCCL's kernels.
int pipeline_max_ctas(int dev) {
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  return std::max(2, nsm - std::max(0, env_int("GIGA_COMM_SMS", 8)));
}

// ---------------------------------------------------------------------------------------
// The multi-GPU pipeline (SURVEY.md 8(a) a3-a7 with 8(e) overlap). Per participant (one per
// GPU in single-process mode; this process's GPU in rank mode):
//   compute stream: split A -> A_lo (overlaps the first broadcast chunk);
//                   for each K-chunk c: wait B chunk c, split it, GEMM over that K range
//                   accumulating into the shard's rows of C (c > 0: C += A_c B_c, an fp32
//                   RN add like the in-kernel promotion); the last K-chunk's GEMM is split
//                   into row chunks q, each publishing an event;
//   comm stream:    NCCL broadcast of B chunk by chunk from rank 0 (contiguous K-row
//                   ranges), then per row chunk q one grouped broadcast per owner of its rows
//                   of C (an all-gather of non-contiguous blocks), overlapping the GEMM of
//                   the next row chunks.
// The persistent GEMM leaves $GIGA_COMM_SMS SMs (default 8) free so NCCL's kernels run
// beside it. Every collective is issued in the same order on every rank (the chunk bounds
// are functions of M, N, K, world only).

int run_pipeline(std::vector<Part> &parts, int world, int64_t M, int64_t N, int64_t K) {
  const char *why = nullptr;
  const NcclApi *api = nccl_api(&why);
  if (!api) return fail(GIGA_ERR_COMM, "NCCL unavailable: %s", why ? why : "?");
  bool aligned = (K % 4 == 0) && (N % 4 == 0);
  for (auto &p : parts) aligned = aligned && aligned16(p.A) && aligned16(p.B) && aligned16(p.C);
  const Plan plan = make_plan(M, N, K, world, aligned);
  const int pb = plan.pb, pc = plan.pc;
  const int64_t *kb = plan.kb;
  GemmExtra ex;
  ex.lda = K;
  ex.ldb = N;
  ex.max_ctas = pipeline_max_ctas(parts[0].d->dev);

  std::vector<Trace> tr;  // $GIGA_TRACE=1: per-GPU timeline of the pipeline
  for (auto &p : parts) {
    tr.emplace_back(*p.d, "nccl_pipeline");
    tr.back().meta("rank", p.rank);
    tr.back().meta("world", world);
    tr.back().meta("kchunks", pb);
    tr.back().meta("rchunks", pc);
  }
  // 0. join the caller's stream, workspace, split A
  for (auto &p : parts) {
    CK(cudaSetDevice(p.d->dev));
    TRY(tr[&p - &parts[0]].start(p.st));
    CK(cudaEventRecord(p.d->ev_start, p.st));
    CK(cudaStreamWaitEvent(p.d->comm, p.d->ev_start, 0));
    int64_t r0, rows;
    partition_rows(M, world, p.rank, &r0, &rows);
    if (aligned) {
      TRY(ws_reserve(*p.d, {{&p.d->A_lo, lo_bytes(std::max<int64_t>(rows, 1) * K)},
                            {&p.d->B_lo, lo_bytes(K * N)}}));
      if (rows > 0) TRY(split(p.A, lo_at(p.d->A_lo), rows * K, p.st));
    }
  }
  // 1. broadcast B from rank 0, K-chunk by K-chunk
  for (int c = 0; c < pb; ++c) {
    TRY(nccl_check(api->GroupStart(), "ncclGroupStart"));
    for (auto &p : parts) {
      CK(cudaSetDevice(p.d->dev));
      float *src = p.B + kb[c] * N;
      ncclResult_t r = api->Broadcast(src, src, size_t((kb[c + 1] - kb[c]) * N), ncclFloat32, 0,
                                      p.comm, p.d->comm);
      if (r != ncclSuccess) {
        api->GroupEnd();
        return nccl_check(r, "ncclBroadcast(B chunk)");
      }
    }
    TRY(nccl_check(api->GroupEnd(), "ncclGroupEnd"));
    for (auto &p : parts) {
      CK(cudaSetDevice(p.d->dev));
      CK(cudaEventRecord(p.d->ev_kchunk[c], p.d->comm));
      TRY(tr[&p - &parts[0]].mark("bcast", p.d->comm, 4.0 * double(kb[c + 1] - kb[c]) * N));
    }
  }
  // 2. compute: K-chunks accumulate into C; the last one in row chunks
  for (auto &p : parts) {
    CK(cudaSetDevice(p.d->dev));
    int64_t r0, rows;
    partition_rows(M, world, p.rank, &r0, &rows);
    float *Cs = p.C + r0 * N;
    if (!aligned) {  // padded single-chunk path (odd shapes / unaligned pointers)
      TRY(shard_compute(*p.d, p.st, p.A, rows, p.B, Cs, N, N, K, p.d->ev_kchunk[0]));
      CK(cudaEventRecord(p.d->ev_rchunk[0], p.st));
      continue;
    }
    const float *Alo = lo_at(p.d->A_lo);
    float *Blo = lo_at(p.d->B_lo);
    Trace &t = tr[&p - &parts[0]];
    TRY(rank_gemms(plan, ex, M, N, K, world, p.rank, p.A, Alo, p.B, Blo, p.C, p.st,
                   [&](int c) -> int {
                     CK(cudaStreamWaitEvent(p.st, p.d->ev_kchunk[c], 0));
                     return split(p.B + kb[c] * N, at(Blo, kb[c] * N), (kb[c + 1] - kb[c]) * N,
                                  p.st);
                   },
                   [&](int q) -> int {
                     if (q < 0) return t.mark("gemm", p.st);
                     CK(cudaEventRecord(p.d->ev_rchunk[q], p.st));
                     return t.mark("gemm_rows", p.st);
                   }));
  }
  // 3. gather C row chunk by row chunk: one broadcast per owner, grouped
  for (int q = 0; q < pc; ++q) {
    for (auto &p : parts) {
      CK(cudaSetDevice(p.d->dev));
      CK(cudaStreamWaitEvent(p.d->comm, p.d->ev_rchunk[q], 0));
    }
    TRY(nccl_check(api->GroupStart(), "ncclGroupStart"));
    for (auto &p : parts) {
      CK(cudaSetDevice(p.d->dev));
      if (pc == 1) {  // whole blocks: in-place all-gather when equal, else per-owner bcast
        const int rc = gather_rows(api, p.comm, p.d->comm, p.C, M, N, world, p.rank);
        if (rc != GIGA_OK) {
          api->GroupEnd();
          return rc;
        }
        continue;
      }
      for (int o = 0; o < world; ++o) {
        int64_t b0, brows;
        plan_block(M, world, pc, o, q, &b0, &brows);
        if (brows <= 0) continue;
        float *blk = p.C + b0 * N;
        ncclResult_t r =
            api->Broadcast(blk, blk, size_t(brows * N), ncclFloat32, o, p.comm, p.d->comm);
        if (r != ncclSuccess) {
          api->GroupEnd();
          return nccl_check(r, "ncclBroadcast(C chunk)");
        }
      }
    }
    TRY(nccl_check(api->GroupEnd(), "ncclGroupEnd"));
    for (auto &p : parts) {
      CK(cudaSetDevice(p.d->dev));
      double rows_in = 0;  // rows of C this GPU receives in round q
      for (int o = 0; o < world; ++o) {
        int64_t b0, brows;
        plan_block(M, world, pc, o, q, &b0, &brows);
        if (o != p.rank && brows > 0) rows_in += double(brows);
      }
      TRY(tr[&p - &parts[0]].mark("gather", p.d->comm, 4.0 * rows_in * N));
    }
  }
  // 4. the caller's stream resumes after the gather
  for (auto &p : parts) {
    CK(cudaSetDevice(p.d->dev));
    CK(cudaEventRecord(p.d->ev_c, p.d->comm));
    CK(cudaStreamWaitEvent(p.st, p.d->ev_c, 0));
  }
  for (auto &t : tr) TRY(t.finish());
  return GIGA_OK;
}

}  // namespace giga
