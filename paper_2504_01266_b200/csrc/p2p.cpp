// p2p.cpp -- the peer-to-peer transport (no NCCL): copy-engine chain for B, C gather fused
// into the GEMM epilogue; single process over several devices, or one process per GPU with
// CUDA IPC and device-side flags.
#include "runtime.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>

namespace giga {

// ---------------------------------------------------------------------------------------
// Peer-to-peer transport (single process, $GIGA_TRANSPORT=p2p): no NCCL, no SMs spent on
// communication.
//   B: a pipelined chain of copy-engine transfers in the plan's K-chunks: GPU i pulls chunk c
//      from GPU i-1 as soon as GPU i-1 has it (each GPU's ingress and egress = one copy of B;
//      latency (pb + g - 2) chunk times); GPU i's GEMM on chunk c starts when it lands.
//   C: the gather is fused into the GEMM epilogue: every 32 x 32 block of a GPU's rows is
//      TMA-stored into its own C_full and into every peer's C_full (NVLink writes), tile by
//      tile while the tensor cores work on the next tile.
//   Completion: each GPU's stream waits for every GPU's last GEMM.
// The devices may repeat (giga_init_devices): "virtual GPUs" on one device run exactly this
// schedule with device-local copies and stores, which is how it is tested on a 1-GPU box.

// The GEMM options of K-chunk c of pb when `ex` carries the peers' C buffers: the partial
// sums stay local (chunk 0 stores, later chunks reduce-add into this GPU's C) and only the
// last chunk, which reads back the local partial and adds its own (load_c), stores the final
// values into every peer -- each C element crosses NVLink once, not once per chunk.
static GemmExtra chunk_extra(const GemmExtra &ex, int c, int pb) {
  GemmExtra e = ex;
  const bool last = c == pb - 1;
  e.accumulate = (c > 0 && !last) ? 1 : 0;
  e.load_c = (c > 0 && last) ? 1 : 0;
  if (!last) {
    e.peer_c = nullptr;
    e.n_peer_c = 0;
    e.mc_c = nullptr;  // earlier chunks stay local (TMA stores / reduce-adds)
    e.vec_store = 0;
  }
  return e;
}

// $GIGA_P2P_STORE=vec: the unicast fused gather with 16-byte st.global stores from the
// epilogue instead of TMA stores -- the multicast mode's code path with one store per peer
// (how that path is exercised where no multicast team can be made).
static bool p2p_vec_store() {
  const char *e = getenv("GIGA_P2P_STORE");
  return e && strcmp(e, "vec") == 0;
}

bool transport_p2p() {
  const char *e = getenv("GIGA_TRANSPORT");
  return e && strcmp(e, "p2p") == 0;
}

// gather = false: no fused gather; each part's GEMM writes only its own rows into C_rows.
int run_p2p(std::vector<Part> &parts, int64_t M, int64_t N, int64_t K, bool gather) {
  const int world = int(parts.size());
  if (world > kMaxCDst)
    return fail(GIGA_ERR_UNSUPPORTED, "p2p transport: at most %d GPUs", kMaxCDst);
  bool aligned = (K % 4 == 0) && (N % 4 == 0);
  for (auto &p : parts)
    aligned = aligned && aligned16(p.A) && aligned16(p.B) &&
              aligned16(gather ? p.C : p.C_rows);
  if (!aligned)
    return fail(GIGA_ERR_UNSUPPORTED, "p2p transport needs K %% 4 == N %% 4 == 0, aligned");
  const Plan plan = make_plan(M, N, K, world, true);
  // $GIGA_TRACE=1: per-GPU timeline; %globaltimer stamps around every chain copy and the CTA
  // intervals of every GEMM launch show the copy engines working under the GEMMs
  std::vector<Trace> tr;
  for (auto &p : parts) {
    tr.emplace_back(*p.d, "p2p");
    tr.back().meta("rank", p.rank);
    tr.back().meta("world", world);
    tr.back().meta("kchunks", plan.pb);
  }
  // 0. join the callers' streams, workspace, split A
  for (auto &p : parts) {
    CK(cudaSetDevice(p.d->dev));
    TRY(tr[&p - &parts[0]].start(p.st));
    CK(cudaEventRecord(p.d->ev_start, p.st));
    CK(cudaStreamWaitEvent(p.d->comm, p.d->ev_start, 0));
    int64_t r0, rows;
    partition_rows(M, world, p.rank, &r0, &rows);
    TRY(ws_reserve(*p.d, {{&p.d->A_lo, lo_bytes(std::max<int64_t>(rows, 1) * K)},
                          {&p.d->B_lo, lo_bytes(K * N)}}));
    if (rows > 0) TRY(split(p.A, lo_at(p.d->A_lo), rows * K, p.st));
  }
  // 1. B down the chain, chunk by chunk (copy engines)
  for (int c = 0; c < plan.pb; ++c) {
    const int64_t off = plan.kb[c] * N, cnt = (plan.kb[c + 1] - plan.kb[c]) * N;
    for (int i = 0; i < world; ++i) {
      Part &p = parts[i];
      CK(cudaSetDevice(p.d->dev));
      if (i > 0) {
        Part &up = parts[i - 1];
        CK(cudaStreamWaitEvent(p.d->comm, up.d->ev_kchunk[c], 0));
        TRY(tr[i].stamp("copy_begin", p.d->comm));
        CK(cudaMemcpyPeerAsync(p.B + off, p.d->dev, up.B + off, up.d->dev, size_t(cnt) * 4,
                               p.d->comm));
        TRY(tr[i].stamp("copy_end", p.d->comm));
      }
      CK(cudaEventRecord(p.d->ev_kchunk[c], p.d->comm));
      TRY(tr[i].mark("bcast", p.d->comm, i > 0 ? 4.0 * double(cnt) : 0.0));
    }
  }
  // 2. GEMMs over the K-chunks; every tile also goes to the peers' C_full: through the
  // multicast team address when the C_full buffers are one giga_mc_alloc team (one store per
  // piece, the switch writes every copy), else one store per peer
  GemmExtra ex;
  ex.lda = K;
  ex.ldb = N;
  float *const mc = gather ? mc_address(parts, M, N) : nullptr;
  for (auto &t : tr) t.meta("gather", mc ? 2 : (gather ? 1 : 0));
  for (auto &p : parts) {
    CK(cudaSetDevice(p.d->dev));
    int64_t r0, rows;
    partition_rows(M, world, p.rank, &r0, &rows);
    float *peer[kMaxCDst];
    int np = 0;
    if (gather && !mc)
      for (auto &q : parts)
        if (&q != &p) peer[np++] = q.C + r0 * N;
    ex.peer_c = peer;
    ex.n_peer_c = np;
    ex.mc_c = mc ? mc + r0 * N : nullptr;
    ex.vec_store = (gather && !mc && p2p_vec_store()) ? 1 : 0;
    float *Cr = gather ? p.C + r0 * N : p.C_rows;
    for (int c = 0; c < plan.pb; ++c) {
      const int64_t Kc = plan.kb[c + 1] - plan.kb[c];
      CK(cudaStreamWaitEvent(p.st, p.d->ev_kchunk[c], 0));
      TRY(split(p.B + plan.kb[c] * N, lo_at(p.d->B_lo, plan.kb[c] * N), Kc * N, p.st));
      if (rows == 0) continue;
      GemmExtra ec = chunk_extra(ex, c, plan.pb);
      ec.cta_ns = tr[&p - &parts[0]].cta_slots("gemm_cta", p.st);
      TRY(gemm_chunk(p.A + plan.kb[c], lo_at(p.d->A_lo, plan.kb[c]), p.B + plan.kb[c] * N,
                     lo_at(p.d->B_lo, plan.kb[c] * N), Cr, rows, N, Kc, ec, p.st));
      TRY(tr[&p - &parts[0]].mark("gemm", p.st));
    }
    CK(cudaEventRecord(p.d->ev_c, p.st));
  }
  if (!gather) {  // every rank only needs its own rows
    for (auto &t : tr) TRY(t.finish());
    return GIGA_OK;
  }
  // 3. a GPU's C_full is complete when every GPU's GEMMs are
  for (auto &p : parts) {
    CK(cudaSetDevice(p.d->dev));
    for (auto &q : parts)
      if (&q != &p) CK(cudaStreamWaitEvent(p.st, q.d->ev_c, 0));
  }
  for (auto &t : tr) TRY(t.finish());
  return GIGA_OK;
}

// ---------------------------------------------------------------------------------------
// The same transport across processes (rank API): peers' B, C_full and flag pages are mapped
// through CUDA IPC; cross-process ordering uses device-side flags written and awaited by the
// streams themselves (cuStreamWriteValue32 / cuStreamWaitValue32), so no host round trip:
//   B chain:  rank r waits ready[c] >= s (upstream holds chunk c of call s) and, before
//             overwriting its own chunk c, pulled[c] >= s-1 (downstream finished reading it in
//             call s-1); copies the chunk from upstream's B; marks upstream's pulled[c] = s and
//             downstream's ready[c] = s.
//   C:        at the start of call s every rank writes started[r] = s into every peer's
//             page on its own stream -- ordered after whatever the caller queued there before
//             the call, i.e. after its consumers of call s-1's C_full. The GEMM that stores
//             into the peers' C_full (the last K-chunk's) first waits started[q] >= s for
//             every peer q, so no rank overwrites a C_full its owner may still be reading.
//             Then cdone[r] = s in every peer's page, and this rank waits cdone[q] >= s.

const DrvApi *drv_api() {
  static DrvApi api;
  static std::once_flag once;
  static bool ok = false;
  std::call_once(once, [] {
    void *a = nullptr, *b = nullptr, *c = nullptr;
    cudaDriverEntryPointQueryResult q{};
    ok = cudaGetDriverEntryPoint("cuStreamWaitValue32", &a, cudaEnableDefault, &q) ==
             cudaSuccess &&
         cudaGetDriverEntryPoint("cuStreamWriteValue32", &b, cudaEnableDefault, &q) ==
             cudaSuccess &&
         cudaGetDriverEntryPoint("cuMemGetAddressRange", &c, cudaEnableDefault, &q) ==
             cudaSuccess &&
         a && b && c;
    api.wait = reinterpret_cast<PFN_cuStreamWaitValue32_v8000>(a);
    api.write = reinterpret_cast<PFN_cuStreamWriteValue32_v8000>(b);
    api.range = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(c);
    cudaGetLastError();
  });
  return ok ? &api : nullptr;
}

uint32_t *flag_ready(uint32_t *page, int c) { return page + c; }
uint32_t *flag_pulled(uint32_t *page, int c) { return page + 16 + c; }
uint32_t *flag_cdone(uint32_t *page, int q) { return page + 32 + q; }
uint32_t *flag_dotdone(uint32_t *page, int q) { return page + 96 + q; }
uint32_t *flag_started(uint32_t *page, int q) { return page + 160 + q; }
// two slot sets by call parity: a peer can run at most one call ahead of this rank
double *dot_part(uint32_t *page, int q, uint32_t s) {
  return reinterpret_cast<double *>(page + 256) + (s & 1) * 64 + q;
}

int wait_flag(cudaStream_t st, uint32_t *addr, uint32_t v) {
  const DrvApi *da = drv_api();
  if (da->wait(reinterpret_cast<CUstream>(st), CUdeviceptr(addr), v, CU_STREAM_WAIT_VALUE_GEQ) !=
      CUDA_SUCCESS)
    return fail(GIGA_ERR_CUDA, "cuStreamWaitValue32 failed");
  return GIGA_OK;
}

int write_flag(cudaStream_t st, uint32_t *addr, uint32_t v) {
  const DrvApi *da = drv_api();
  if (da->write(reinterpret_cast<CUstream>(st), CUdeviceptr(addr), v,
                CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
    return fail(GIGA_ERR_CUDA, "cuStreamWriteValue32 failed");
  return GIGA_OK;
}

int run_p2p_rank(DevCtx &d, cudaStream_t st, const float *A, float *B, float *C, int64_t M,
                 int64_t N, int64_t K) {
  RankP2P &x = g.p2p;
  const int r = g.rank, world = g.world;
  if (world > kMaxCDst)
    return fail(GIGA_ERR_UNSUPPORTED, "p2p transport: at most %d ranks", kMaxCDst);
  if (B != x.B || C != x.C)
    return fail(GIGA_ERR_INVALID_ARG,
                "p2p transport: B / C_full must be the buffers registered with "
                "giga_rank_p2p_export");
  if ((K % 4) || (N % 4) || !aligned16(A) || !aligned16(B) || !aligned16(C))
    return fail(GIGA_ERR_UNSUPPORTED, "p2p transport needs K %% 4 == N %% 4 == 0, aligned");
  // the multicast team address of C_full's rows (checked before the call takes a number)
  float *const mc = rank_mc_address(C, M, N);
  if (rank_mc_buffer(C) && !mc)
    return fail(GIGA_ERR_INVALID_ARG, "p2p transport: M x N exceeds the multicast C_full");
  const uint32_t s = ++x.step;
  const Plan plan = make_plan(M, N, K, world, true);
  int64_t r0, rows;
  partition_rows(M, world, r, &r0, &rows);
  Trace tr(d, "p2p_rank");  // $GIGA_TRACE=1: this rank's timeline
  tr.meta("rank", r);
  tr.meta("world", world);
  tr.meta("kchunks", plan.pb);
  TRY(tr.start(st));
  // "my C_full is free for call s": after the caller's earlier work on st
  for (int q = 0; q < world; ++q)
    if (q != r) TRY(write_flag(st, flag_started(x.peerF[q], r), s));
  CK(cudaEventRecord(d.ev_start, st));
  CK(cudaStreamWaitEvent(d.comm, d.ev_start, 0));
  TRY(ws_reserve(d, {{&d.A_lo, lo_bytes(std::max<int64_t>(rows, 1) * K)},
                     {&d.B_lo, lo_bytes(K * N)}}));
  if (rows > 0) TRY(split(A, lo_at(d.A_lo), rows * K, st));
  // B down the chain (copy engine on the comm stream, ordered by flags)
  for (int c = 0; c < plan.pb; ++c) {
    const int64_t off = plan.kb[c] * N, cnt = (plan.kb[c + 1] - plan.kb[c]) * N;
    if (r > 0) {
      TRY(wait_flag(d.comm, flag_ready(x.flags, c), s));
      if (r < world - 1 && s > 1) TRY(wait_flag(d.comm, flag_pulled(x.flags, c), s - 1));
      CK(cudaMemcpyAsync(B + off, x.peerB[r - 1] + off, size_t(cnt) * 4,
                         cudaMemcpyDeviceToDevice, d.comm));
      TRY(write_flag(d.comm, flag_pulled(x.peerF[r - 1], c), s));
    }
    CK(cudaEventRecord(d.ev_kchunk[c], d.comm));
    TRY(tr.mark("b_chunk", d.comm));
    if (r < world - 1) TRY(write_flag(d.comm, flag_ready(x.peerF[r + 1], c), s));
  }
  // GEMMs over the K-chunks, every tile also stored into the peers' C_full (one multicast
  // store per piece when C_full is this rank's team buffer, else one store per peer)
  float *peer[kMaxCDst];
  int np = 0;
  if (!mc)
    for (int q = 0; q < world; ++q)
      if (q != r) peer[np++] = x.peerC[q] + r0 * N;
  GemmExtra ex;
  ex.lda = K;
  ex.ldb = N;
  ex.peer_c = peer;
  ex.n_peer_c = np;
  ex.mc_c = mc ? mc + r0 * N : nullptr;
  ex.vec_store = (!mc && p2p_vec_store()) ? 1 : 0;
  tr.meta("gather", mc ? 2 : 1);
  for (int c = 0; c < plan.pb; ++c) {
    const int64_t Kc = plan.kb[c + 1] - plan.kb[c];
    CK(cudaStreamWaitEvent(st, d.ev_kchunk[c], 0));
    TRY(split(B + plan.kb[c] * N, lo_at(d.B_lo, plan.kb[c] * N), Kc * N, st));
    if (rows == 0) continue;
    if (c == plan.pb - 1)  // this GEMM writes into the peers' C_full: they must have started s
      for (int q = 0; q < world; ++q)
        if (q != r) TRY(wait_flag(st, flag_started(x.flags, q), s));
    TRY(gemm_chunk(A + plan.kb[c], lo_at(d.A_lo, plan.kb[c]), B + plan.kb[c] * N,
                   lo_at(d.B_lo, plan.kb[c] * N), C + r0 * N, rows, N, Kc,
                   chunk_extra(ex, c, plan.pb), st));
    TRY(tr.mark("gemm", st));
  }
  for (int q = 0; q < world; ++q)
    if (q != r) TRY(write_flag(st, flag_cdone(x.peerF[q], r), s));
  for (int q = 0; q < world; ++q)
    if (q != r) TRY(wait_flag(st, flag_cdone(x.flags, q), s));
  TRY(tr.mark("all_c", st));
  // the comm stream's last copies are done before the call's work is (join it back)
  CK(cudaEventRecord(d.ev_c, d.comm));
  CK(cudaStreamWaitEvent(st, d.ev_c, 0));
  TRY(tr.finish());
  return GIGA_OK;
}

// dot partials all-reduced through the flag pages: every rank writes its fp64 partial into
// slot r of every page, then sums slots 0..world-1 in rank order (deterministic).
int p2p_dot_allreduce(DevCtx &d, cudaStream_t st, double *result) {
  RankP2P &x = g.p2p;
  const uint32_t s = ++x.dot_step;
  for (int q = 0; q < g.world; ++q) {
    uint32_t *page = (q == g.rank) ? x.flags : x.peerF[q];
    CK(cudaMemcpyAsync(dot_part(page, g.rank, s), vec_out(d), sizeof(double),
                       cudaMemcpyDeviceToDevice, st));
    TRY(write_flag(st, flag_dotdone(page, g.rank), s));
  }
  for (int q = 0; q < g.world; ++q) TRY(wait_flag(st, flag_dotdone(x.flags, q), s));
  // the partials in rank order into the pinned slot (room for 8 = kMaxCDst ranks)
  CK(cudaMemcpyAsync(d.res_pinned, dot_part(x.flags, 0, s), sizeof(double) * g.world,
                     cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  double tot = 0.0;
  for (int q = 0; q < g.world; ++q) tot += d.res_pinned[q];
  *result = tot;
  return GIGA_OK;
}

void p2p_release() {
  RankP2P &x = g.p2p;
  for (void *p : x.opened) cudaIpcCloseMemHandle(p);
  if (x.flags) cudaFree(x.flags);
  cudaGetLastError();
  x = RankP2P{};
}

// Device-resident path on GPUs 0..ngpus-1 (B_buf[0] root, C_full[g] all receive full C).
}  // namespace giga
