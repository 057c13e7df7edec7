// api.cpp -- the C ABI declared in include/giga.h: library state, the row-block partitioner,
// the per-GPU workspace cache, and the orchestration of one row-split matrix multiply
// (PAPER.md:285-291): place A row blocks, distribute B (NCCL broadcast), split to TF32
// hi/lo, shard GEMM, gather the C row blocks (NCCL all-gather / per-owner broadcast).
#include "giga.h"

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "kernels.h"
#include "host_plan.h"
#include "nccl_loader.h"

namespace giga {
namespace {

// ---------------------------------------------------------------------------------------
// errors
thread_local std::string t_err;

int fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  t_err = buf;
  return code;
}

int fail_cuda(cudaError_t e, const char *what, int line) {
  cudaGetLastError();  // clear a non-sticky error so the next call starts clean
  const int code = (e == cudaErrorMemoryAllocation) ? GIGA_ERR_OOM : GIGA_ERR_CUDA;
  return fail(code, "%s failed at api.cpp:%d: %s (%s)", what, line, cudaGetErrorName(e),
              cudaGetErrorString(e));
}

#define CK(x)                                                     \
  do {                                                            \
    cudaError_t e_ = (x);                                         \
    if (e_ != cudaSuccess) return fail_cuda(e_, #x, __LINE__);    \
  } while (0)

#define TRY(x)                \
  do {                        \
    int r_ = (x);             \
    if (r_ != GIGA_OK) return r_; \
  } while (0)

// ---------------------------------------------------------------------------------------
// state

struct Buf {
  void *p = nullptr;
  size_t bytes = 0;
};

constexpr int kMaxChunks = 16;  // pipeline chunks per phase (B K-chunks, C row-chunks)

struct DevCtx {
  int dev = -1;
  cudaStream_t compute = nullptr;  // splits + GEMM (+ H2D/D2H in host mode)
  cudaStream_t comm = nullptr;     // broadcast of B, gather of C (host mode: H2D copies)
  cudaStream_t d2h = nullptr;      // host mode: device-to-host copies of finished C rows
  cudaEvent_t ev_b = nullptr;      // B present on this GPU
  cudaEvent_t ev_c = nullptr;      // this GPU's C rows computed
  cudaEvent_t ev_start = nullptr;  // caller-stream entry (rank mode)
  cudaEvent_t ev_last = nullptr;   // rank mode: end of the previous call (workspace reuse)
  bool has_last = false;
  std::vector<cudaEvent_t> ev_kchunk;  // pipeline: B K-chunk c present
  std::vector<cudaEvent_t> ev_rchunk;  // pipeline: C row-chunk q computed
  std::vector<cudaEvent_t> ev_done;    // host pipeline: late row block q computed
  std::vector<cudaEvent_t> ev_trace;   // host pipeline timeline ($GIGA_HOST_TRACE), timing
  Buf A_lo, B_lo, A_pad, B_pad, C_pad, A_h, B_h, C_h;
  Buf vec_ws;  // dot: kDotMaxBlocks fp64 partials, the fp64 result, the ticket (zeroed once)
};

// Rank-mode peer-to-peer state: this rank's registered B / C_full, its flag page, and the
// peers' buffers and flag pages mapped through CUDA IPC (index = rank).
// Flag page (device memory, u32 unless noted): ready[c] @0 (upstream has B chunk c),
// pulled[c] @64 (downstream finished reading my chunk c), cdone[q] @128 (rank q wrote its C
// rows into my C_full), dotdone[q] @384, dot partials (fp64) @1024. Values are call numbers.
constexpr size_t kFlagBytes = 4096;
struct RankP2P {
  bool ready = false;
  uint32_t *flags = nullptr;
  float *B = nullptr, *C = nullptr;
  std::vector<float *> peerB, peerC;
  std::vector<uint32_t *> peerF;
  std::vector<void *> opened;
  uint32_t step = 0, dot_step = 0;
};

struct State {
  std::mutex mu;
  int mode = 0;  // 0 none, 1 single-process, 2 rank
  std::vector<DevCtx> devs;
  std::map<int, std::vector<ncclComm_t>> comms;  // single-process: ngpus -> comms
  ncclComm_t rank_comm = nullptr;
  int rank = 0, world = 1;
  RankP2P p2p;
};
State g;

struct TimeRec {
  int dev;
  int kind;  // 0 gemm, 1 split
  cudaEvent_t a, b;
};
std::mutex g_tmu;
bool g_timing = false;
std::vector<TimeRec> g_tpending;
std::vector<std::pair<int, cudaEvent_t>> g_tpool;
double g_tms[2] = {0, 0};
int64_t g_tcount[2] = {0, 0};

cudaEvent_t pool_event(int dev) {
  for (size_t i = 0; i < g_tpool.size(); ++i)
    if (g_tpool[i].first == dev) {
      cudaEvent_t e = g_tpool[i].second;
      g_tpool.erase(g_tpool.begin() + i);
      return e;
    }
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return e;
}

// Launch `fn` on `st`, bracketed by timing events when timing is enabled.
template <class F>
cudaError_t timed(int kind, cudaStream_t st, F fn) {
  bool on;
  {
    std::lock_guard<std::mutex> lk(g_tmu);
    on = g_timing;
  }
  if (!on) return fn();
  int dev = 0;
  cudaGetDevice(&dev);
  cudaEvent_t a, b;
  {
    std::lock_guard<std::mutex> lk(g_tmu);
    a = pool_event(dev);
    b = pool_event(dev);
  }
  if (a) cudaEventRecord(a, st);
  cudaError_t e = fn();
  if (b) cudaEventRecord(b, st);
  std::lock_guard<std::mutex> lk(g_tmu);
  if (a && b)
    g_tpending.push_back({dev, kind, a, b});
  else {
    if (a) g_tpool.push_back({dev, a});
    if (b) g_tpool.push_back({dev, b});
  }
  return e;
}

bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// ---------------------------------------------------------------------------------------
// workspace: grow-only per-GPU buffers, reserved transactionally so a failed call leaves the
// device memory footprint exactly as it found it.

int ws_reserve(DevCtx &d, std::initializer_list<std::pair<Buf *, size_t>> req) {
  std::vector<std::pair<Buf *, void *>> fresh;
  for (auto &r : req) {
    if (r.first->bytes >= r.second) continue;
    bool dup = false;
    for (auto &f : fresh) dup |= (f.first == r.first);
    if (dup) continue;
    void *p = nullptr;
    cudaError_t e = cudaMalloc(&p, r.second);
    if (e != cudaSuccess) {
      for (auto &f : fresh) cudaFree(f.second);
      return fail_cuda(e, "cudaMalloc(workspace)", __LINE__);
    }
    fresh.push_back({r.first, p});
  }
  for (auto &f : fresh) {
    size_t want = 0;
    for (auto &r : req)
      if (r.first == f.first) want = std::max(want, r.second);
    if (f.first->p) cudaFree(f.first->p);
    f.first->p = f.second;
    f.first->bytes = want;
  }
  return GIGA_OK;
}

void ws_free(DevCtx &d) {
  for (Buf *b :
       {&d.A_lo, &d.B_lo, &d.A_pad, &d.B_pad, &d.C_pad, &d.A_h, &d.B_h, &d.C_h, &d.vec_ws}) {
    if (b->p) cudaFree(b->p);
    b->p = nullptr;
    b->bytes = 0;
  }
}

float *fptr(Buf &b) { return static_cast<float *>(b.p); }

int ctx_create(DevCtx &d, int dev) {
  d.dev = dev;
  CK(cudaSetDevice(dev));
  CK(cudaStreamCreateWithFlags(&d.compute, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&d.comm, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&d.d2h, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&d.ev_b, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&d.ev_c, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&d.ev_start, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&d.ev_last, cudaEventDisableTiming));
  for (auto *v : {&d.ev_kchunk, &d.ev_rchunk, &d.ev_done}) {
    v->assign(kMaxChunks, nullptr);
    for (auto &e : *v) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  return GIGA_OK;
}

void ctx_destroy(DevCtx &d) {
  if (d.dev < 0) return;
  cudaSetDevice(d.dev);
  cudaDeviceSynchronize();
  ws_free(d);
  if (d.compute) cudaStreamDestroy(d.compute);
  if (d.comm) cudaStreamDestroy(d.comm);
  if (d.d2h) cudaStreamDestroy(d.d2h);
  for (cudaEvent_t e : {d.ev_b, d.ev_c, d.ev_start, d.ev_last})
    if (e) cudaEventDestroy(e);
  for (auto *v : {&d.ev_kchunk, &d.ev_rchunk, &d.ev_done, &d.ev_trace})
    for (cudaEvent_t e : *v)
      if (e) cudaEventDestroy(e);
  d = DevCtx{};
}

int check_sm100(int dev) {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10)
    return fail(GIGA_ERR_NO_DEVICE, "device %d is sm_%d%d, this build is sm_100a only", dev,
                prop.major, prop.minor);
  return GIGA_OK;
}

// ---------------------------------------------------------------------------------------
// one shard on one GPU: split A and B into TF32 hi/lo and run the tensor-core GEMM into
// C (rows x N, row stride ldc). If `wait_b` is given, B is only touched after it fires (the
// A split overlaps the distribution of B).

// The lo = x - tf32(x) operands are computed inside the GEMM from the raw tiles (the
// default). GIGA_LO_PRESPLIT=1 restores the pre-split design (split_lo_kernel writes lo
// arrays to HBM, the GEMM TMA-loads them: twice the operand traffic; for comparison).
bool lo_presplit() {
  static const bool v = [] {
    const char *e = getenv("GIGA_LO_PRESPLIT");
    return e && *e == '1';
  }();
  return v;
}
size_t lo_bytes(int64_t elems) { return lo_presplit() ? size_t(elems) * 4 : 0; }
float *lo_at(Buf &b, int64_t off = 0) { return lo_presplit() ? fptr(b) + off : nullptr; }
template <class T>
T *at(T *p, int64_t off) {
  return p ? p + off : nullptr;
}

int split(const float *x, float *lo, int64_t n, cudaStream_t st) {
  if (!lo) return GIGA_OK;  // lo computed in the GEMM
  CK(timed(1, st, [&] { return launch_split_lo(x, lo, n, st); }));
  return GIGA_OK;
}

int gemm(const float *A, const float *Alo, const float *B, const float *Blo, float *C,
         int64_t M, int64_t N, int64_t K, int64_t ldc, cudaStream_t st) {
  CK(timed(0, st, [&] {
    return launch_gemm_3xtf32(A, Alo, B, Blo, C, M, N, K, ldc, 3, -1, st);
  }));
  return GIGA_OK;
}

int shard_compute(DevCtx &d, cudaStream_t st, const float *A, int64_t rows, const float *B,
                  float *C, int64_t ldc, int64_t N, int64_t K, cudaEvent_t wait_b) {
  if (rows <= 0) {
    if (wait_b) CK(cudaStreamWaitEvent(st, wait_b, 0));
    return GIGA_OK;
  }
  const bool direct = (K % 4 == 0) && (N % 4 == 0) && (ldc % 4 == 0) && aligned16(A) &&
                      aligned16(B) && aligned16(C);
  if (direct) {
    TRY(ws_reserve(d, {{&d.A_lo, lo_bytes(rows * K)}, {&d.B_lo, lo_bytes(K * N)}}));
    TRY(split(A, lo_at(d.A_lo), rows * K, st));
    if (wait_b) CK(cudaStreamWaitEvent(st, wait_b, 0));
    TRY(split(B, lo_at(d.B_lo), K * N, st));
    return gemm(A, lo_at(d.A_lo), B, lo_at(d.B_lo), C, rows, N, K, ldc, st);
  }
  // Unaligned shapes (H6): zero-padded copies with K, N rounded up to multiples of 4. Zero
  // columns of A / rows of B add nothing to any dot product.
  const int64_t K4 = (K + 3) / 4 * 4, N4 = (N + 3) / 4 * 4;
  TRY(ws_reserve(d, {{&d.A_pad, size_t(rows * K4) * 4},
                     {&d.B_pad, size_t(K4 * N4) * 4},
                     {&d.C_pad, size_t(rows * N4) * 4},
                     {&d.A_lo, lo_bytes(rows * K4)},
                     {&d.B_lo, lo_bytes(K4 * N4)}}));
  CK(cudaMemsetAsync(d.A_pad.p, 0, size_t(rows * K4) * 4, st));
  CK(cudaMemcpy2DAsync(d.A_pad.p, K4 * 4, A, K * 4, K * 4, rows, cudaMemcpyDeviceToDevice, st));
  TRY(split(fptr(d.A_pad), lo_at(d.A_lo), rows * K4, st));
  if (wait_b) CK(cudaStreamWaitEvent(st, wait_b, 0));
  CK(cudaMemsetAsync(d.B_pad.p, 0, size_t(K4 * N4) * 4, st));
  CK(cudaMemcpy2DAsync(d.B_pad.p, N4 * 4, B, N * 4, N * 4, K, cudaMemcpyDeviceToDevice, st));
  TRY(split(fptr(d.B_pad), lo_at(d.B_lo), K4 * N4, st));
  TRY(gemm(fptr(d.A_pad), lo_at(d.A_lo), fptr(d.B_pad), lo_at(d.B_lo), fptr(d.C_pad), rows, N4,
           K4, N4, st));
  CK(cudaMemcpy2DAsync(C, ldc * 4, d.C_pad.p, N4 * 4, N * 4, rows, cudaMemcpyDeviceToDevice,
                       st));
  return GIGA_OK;
}

// ---------------------------------------------------------------------------------------
// NCCL

int nccl_check(ncclResult_t r, const char *what) {
  if (r == ncclSuccess) return GIGA_OK;
  const NcclApi *api = nccl_api(nullptr);
  return fail(GIGA_ERR_COMM, "%s failed: %s", what, api ? api->GetErrorString(r) : "?");
}

int env_int(const char *name, int dflt);

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

void partition_rows(int64_t M, int ngpus, int gi, int64_t *row0, int64_t *rows) {
  const int64_t base = M / ngpus;
  *row0 = int64_t(gi) * base;
  *rows = (gi == ngpus - 1) ? M - int64_t(ngpus - 1) * base : base;
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

// ---------------------------------------------------------------------------------------
// argument checks

bool overlaps(const void *a, size_t abytes, const void *b, size_t bbytes) {
  const uintptr_t x = reinterpret_cast<uintptr_t>(a), y = reinterpret_cast<uintptr_t>(b);
  return x < y + bbytes && y < x + abytes;
}

int check_dims(int64_t M, int64_t N, int64_t K) {
  if (M < 1 || N < 1 || K < 1)
    return fail(GIGA_ERR_INVALID_ARG, "M, N, K must be >= 1 (got %lld, %lld, %lld)",
                (long long)M, (long long)N, (long long)K);
  const int64_t lim = int64_t(1) << 31;
  if (M >= lim || N >= lim || K >= lim || M > (int64_t(1) << 62) / N ||
      K > (int64_t(1) << 62) / N || M > (int64_t(1) << 62) / K)
    return fail(GIGA_ERR_INVALID_ARG, "matrix dimensions too large");
  return GIGA_OK;
}

// pointer kind: 1 = device (dev set), 0 = host
int pointer_kind(const void *p, int *dev) {
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  if (a.type == cudaMemoryTypeDevice) {
    *dev = a.device;
    return 1;
  }
  return 0;
}

// The single-process calls are blocking ("synchronize and copy back"): they
// start after everything already queued on the participating devices (e.g. the producer of
// A or B on another stream) and return after their own work is done.
int quiesce(int ngpus) {
  for (int i = 0; i < ngpus; ++i) {
    CK(cudaSetDevice(g.devs[i].dev));
    CK(cudaDeviceSynchronize());
  }
  return GIGA_OK;
}

// ---------------------------------------------------------------------------------------
// vector operations: per-GPU fp64 partial of a contiguous index range

constexpr size_t kVecWsBytes = size_t(kDotMaxBlocks) * 8 + 64;

int vec_ws(DevCtx &d) {
  if (d.vec_ws.p) return GIGA_OK;
  TRY(ws_reserve(d, {{&d.vec_ws, kVecWsBytes}}));
  CK(cudaMemset(d.vec_ws.p, 0, kVecWsBytes));  // ticket starts at zero
  return GIGA_OK;
}
double *vec_partials(DevCtx &d) { return static_cast<double *>(d.vec_ws.p); }
double *vec_out(DevCtx &d) { return vec_partials(d) + kDotMaxBlocks; }
unsigned *vec_ticket(DevCtx &d) { return reinterpret_cast<unsigned *>(vec_out(d) + 1); }

int dot_partial(DevCtx &d, const float *x, const float *y, int64_t n, cudaStream_t st) {
  TRY(vec_ws(d));
  CK(launch_dot(x, y, n, vec_partials(d), vec_ticket(d), vec_out(d), st));
  return GIGA_OK;
}

int sync_all(int ngpus) {
  for (int i = 0; i < ngpus; ++i) {
    DevCtx &d = g.devs[i];
    CK(cudaSetDevice(d.dev));
    CK(cudaStreamSynchronize(d.compute));
    CK(cudaStreamSynchronize(d.comm));
  }
  return GIGA_OK;
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

// The chunk plan: B is broadcast in pb K-chunks [kb[c], kb[c+1]) (multiples of 16, at least
// 512 deep); the last K-chunk's GEMM and the C gather run in pc row chunks; chunk q of owner
// o is rows [o0 + orows*q/pc, o0 + orows*(q+1)/pc) of its shard (plan_block). Knobs:
// $GIGA_BCAST_CHUNKS (4), $GIGA_GATHER_CHUNKS (4); unaligned shapes use one chunk of each.
struct Plan {
  int pb = 1, pc = 1;
  int64_t kb[kMaxChunks + 1] = {0};
};

int env_int(const char *name, int dflt) {
  const char *e = getenv(name);
  return (e && *e) ? atoi(e) : dflt;
}

Plan make_plan(int64_t M, int64_t K, int world, bool aligned) {
  Plan pl;
  int64_t rows_max = 0;
  for (int r = 0; r < world; ++r) {
    int64_t r0, rows;
    partition_rows(M, world, r, &r0, &rows);
    rows_max = std::max(rows_max, rows);
  }
  if (aligned) {
    pl.pb = std::min(std::max(env_int("GIGA_BCAST_CHUNKS", 4), 1), kMaxChunks);
    pl.pb = int(std::min<int64_t>(pl.pb, std::max<int64_t>(1, K / 512)));
    pl.pc = std::min(std::max(env_int("GIGA_GATHER_CHUNKS", 4), 1), kMaxChunks);
    pl.pc = int(std::min<int64_t>(pl.pc, std::max<int64_t>(1, rows_max / 256)));
  }
  for (int c = 0; c < pl.pb; ++c) pl.kb[c] = (K * c / pl.pb) / 16 * 16;
  pl.kb[pl.pb] = K;
  return pl;
}

void plan_block(int64_t M, int world, int pc, int owner, int q, int64_t *row0, int64_t *rows) {
  int64_t o0, orows;
  partition_rows(M, world, owner, &o0, &orows);
  const int64_t q0 = orows * q / pc, q1 = orows * (q + 1) / pc;
  *row0 = o0 + q0;
  *rows = q1 - q0;
}

struct Part {
  DevCtx *d;
  ncclComm_t comm;
  int rank;
  const float *A;   // rows_r x K shard
  float *B;         // K x N: source on rank 0, receive buffer elsewhere
  float *C;         // M x N: every rank ends with all of C
  cudaStream_t st;  // compute stream
  float *C_rows = nullptr;  // p2p without gather: this rank's rows only (rows x N)
};

bool force_comm() { return env_int("GIGA_FORCE_COMM", 0) != 0; }

int gemm_chunk(const float *A, const float *Alo, const float *B, const float *Blo, float *C,
               int64_t rows, int64_t N, int64_t Kc, const GemmExtra &ex, cudaStream_t st) {
  CK(timed(0, st, [&] {
    return launch_gemm_3xtf32(A, Alo, B, Blo, C, rows, N, Kc, N, 3, -1, st, 0, &ex);
  }));
  return GIGA_OK;
}

int run_pipeline(std::vector<Part> &parts, int world, int64_t M, int64_t N, int64_t K) {
  const char *why = nullptr;
  const NcclApi *api = nccl_api(&why);
  if (!api) return fail(GIGA_ERR_COMM, "NCCL unavailable: %s", why ? why : "?");
  bool aligned = (K % 4 == 0) && (N % 4 == 0);
  for (auto &p : parts) aligned = aligned && aligned16(p.A) && aligned16(p.B) && aligned16(p.C);
  const Plan plan = make_plan(M, K, world, aligned);
  const int pb = plan.pb, pc = plan.pc;
  const int64_t *kb = plan.kb;
  GemmExtra ex;
  ex.lda = K;
  ex.ldb = N;
  {
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, parts[0].d->dev);
    ex.max_ctas = std::max(2, nsm - std::max(0, env_int("GIGA_COMM_SMS", 8)));
  }

  // 0. join the caller's stream, workspace, split A
  for (auto &p : parts) {
    CK(cudaSetDevice(p.d->dev));
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
    for (int c = 0; c < pb; ++c) {
      const int64_t Kc = kb[c + 1] - kb[c];
      CK(cudaStreamWaitEvent(p.st, p.d->ev_kchunk[c], 0));
      TRY(split(p.B + kb[c] * N, at(Blo, kb[c] * N), Kc * N, p.st));
      GemmExtra e = ex;
      e.accumulate = c > 0;
      const float *Bc = p.B + kb[c] * N, *Bloc = at(Blo, kb[c] * N);
      if (c < pb - 1) {
        if (rows > 0)
          TRY(gemm_chunk(p.A + kb[c], at(Alo, kb[c]), Bc, Bloc, Cs, rows, N, Kc, e, p.st));
        continue;
      }
      for (int q = 0; q < pc; ++q) {
        int64_t b0, brows;
        plan_block(M, world, pc, p.rank, q, &b0, &brows);
        const int64_t q0 = b0 - r0;  // offset inside this rank's shard
        if (brows > 0)
          TRY(gemm_chunk(p.A + q0 * K + kb[c], at(Alo, q0 * K + kb[c]), Bc, Bloc, Cs + q0 * N,
                         brows, N, Kc, e, p.st));
        CK(cudaEventRecord(p.d->ev_rchunk[q], p.st));
      }
    }
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
  }
  // 4. the caller's stream resumes after the gather
  for (auto &p : parts) {
    CK(cudaSetDevice(p.d->dev));
    CK(cudaEventRecord(p.d->ev_c, p.d->comm));
    CK(cudaStreamWaitEvent(p.st, p.d->ev_c, 0));
  }
  return GIGA_OK;
}

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

bool transport_p2p() {
  const char *e = getenv("GIGA_TRANSPORT");
  return e && strcmp(e, "p2p") == 0;
}

// gather = false: no fused gather; each part's GEMM writes only its own rows into C_rows.
int run_p2p(std::vector<Part> &parts, int64_t M, int64_t N, int64_t K, bool gather = true) {
  const int world = int(parts.size());
  if (world > kMaxCDst)
    return fail(GIGA_ERR_UNSUPPORTED, "p2p transport: at most %d GPUs", kMaxCDst);
  bool aligned = (K % 4 == 0) && (N % 4 == 0);
  for (auto &p : parts)
    aligned = aligned && aligned16(p.A) && aligned16(p.B) &&
              aligned16(gather ? p.C : p.C_rows);
  if (!aligned)
    return fail(GIGA_ERR_UNSUPPORTED, "p2p transport needs K %% 4 == N %% 4 == 0, aligned");
  const Plan plan = make_plan(M, K, world, true);
  // 0. join the callers' streams, workspace, split A
  for (auto &p : parts) {
    CK(cudaSetDevice(p.d->dev));
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
        CK(cudaMemcpyPeerAsync(p.B + off, p.d->dev, up.B + off, up.d->dev, size_t(cnt) * 4,
                               p.d->comm));
      }
      CK(cudaEventRecord(p.d->ev_kchunk[c], p.d->comm));
    }
  }
  // 2. GEMMs over the K-chunks; every tile also goes to the peers' C_full
  GemmExtra ex;
  ex.lda = K;
  ex.ldb = N;
  for (auto &p : parts) {
    CK(cudaSetDevice(p.d->dev));
    int64_t r0, rows;
    partition_rows(M, world, p.rank, &r0, &rows);
    float *peer[kMaxCDst];
    int np = 0;
    if (gather)
      for (auto &q : parts)
        if (&q != &p) peer[np++] = q.C + r0 * N;
    ex.peer_c = peer;
    ex.n_peer_c = np;
    float *Cr = gather ? p.C + r0 * N : p.C_rows;
    for (int c = 0; c < plan.pb; ++c) {
      const int64_t Kc = plan.kb[c + 1] - plan.kb[c];
      CK(cudaStreamWaitEvent(p.st, p.d->ev_kchunk[c], 0));
      TRY(split(p.B + plan.kb[c] * N, lo_at(p.d->B_lo, plan.kb[c] * N), Kc * N, p.st));
      if (rows == 0) continue;
      GemmExtra e = ex;
      e.accumulate = c > 0;
      TRY(gemm_chunk(p.A + plan.kb[c], lo_at(p.d->A_lo, plan.kb[c]), p.B + plan.kb[c] * N,
                     lo_at(p.d->B_lo, plan.kb[c] * N), Cr, rows, N, Kc, e, p.st));
    }
    CK(cudaEventRecord(p.d->ev_c, p.st));
  }
  if (!gather) return GIGA_OK;  // every rank only needs its own rows
  // 3. a GPU's C_full is complete when every GPU's GEMMs are
  for (auto &p : parts) {
    CK(cudaSetDevice(p.d->dev));
    for (auto &q : parts)
      if (&q != &p) CK(cudaStreamWaitEvent(p.st, q.d->ev_c, 0));
  }
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
//   C:        the GEMM epilogue writes this rank's rows into every peer's C_full; then
//             cdone[r] = s in every peer's page, and this rank waits cdone[q] >= s for all q.

struct DrvApi {
  PFN_cuStreamWaitValue32_v8000 wait = nullptr;
  PFN_cuStreamWriteValue32_v8000 write = nullptr;
  PFN_cuMemGetAddressRange_v3020 range = nullptr;
};

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
  const uint32_t s = ++x.step;
  const Plan plan = make_plan(M, K, world, true);
  int64_t r0, rows;
  partition_rows(M, world, r, &r0, &rows);
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
    if (r < world - 1) TRY(write_flag(d.comm, flag_ready(x.peerF[r + 1], c), s));
  }
  // GEMMs over the K-chunks, every tile also stored into the peers' C_full
  float *peer[kMaxCDst];
  int np = 0;
  for (int q = 0; q < world; ++q)
    if (q != r) peer[np++] = x.peerC[q] + r0 * N;
  GemmExtra ex;
  ex.lda = K;
  ex.ldb = N;
  ex.peer_c = peer;
  ex.n_peer_c = np;
  for (int c = 0; c < plan.pb; ++c) {
    const int64_t Kc = plan.kb[c + 1] - plan.kb[c];
    CK(cudaStreamWaitEvent(st, d.ev_kchunk[c], 0));
    TRY(split(B + plan.kb[c] * N, lo_at(d.B_lo, plan.kb[c] * N), Kc * N, st));
    if (rows == 0) continue;
    GemmExtra e = ex;
    e.accumulate = c > 0;
    TRY(gemm_chunk(A + plan.kb[c], lo_at(d.A_lo, plan.kb[c]), B + plan.kb[c] * N,
                   lo_at(d.B_lo, plan.kb[c] * N), C + r0 * N, rows, N, Kc, e, st));
  }
  for (int q = 0; q < world; ++q)
    if (q != r) TRY(write_flag(st, flag_cdone(x.peerF[q], r), s));
  for (int q = 0; q < world; ++q)
    if (q != r) TRY(wait_flag(st, flag_cdone(x.flags, q), s));
  // the comm stream's last copies are done before the call's work is (join it back)
  CK(cudaEventRecord(d.ev_c, d.comm));
  CK(cudaStreamWaitEvent(st, d.ev_c, 0));
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
  std::vector<double> parts(g.world);
  CK(cudaMemcpyAsync(parts.data(), dot_part(x.flags, 0, s), sizeof(double) * g.world,
                     cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  double tot = 0.0;
  for (double v : parts) tot += v;
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
int sharded_locked(const float *const *A_shard, float *const *B_buf, float *const *C_full,
                   int64_t M, int64_t N, int64_t K, int ngpus) {
  if (ngpus == 1 && !force_comm()) {
    DevCtx &d = g.devs[0];
    CK(cudaSetDevice(d.dev));
    TRY(shard_compute(d, d.compute, A_shard[0], M, B_buf[0], C_full[0], N, N, K, nullptr));
    return sync_all(1);
  }
  if (transport_p2p()) {
    std::vector<Part> parts;
    for (int i = 0; i < ngpus; ++i)
      parts.push_back({&g.devs[i], nullptr, i, A_shard[i], B_buf[i], C_full[i],
                       g.devs[i].compute});
    TRY(run_p2p(parts, M, N, K));
    return sync_all(ngpus);
  }
  std::vector<ncclComm_t> *comms = nullptr;
  TRY(get_comms(ngpus, &comms));
  const NcclApi *api = nccl_api(nullptr);
  std::vector<Part> parts;
  for (int i = 0; i < ngpus; ++i) {
    int64_t r0, rows;
    partition_rows(M, ngpus, i, &r0, &rows);
    parts.push_back({&g.devs[i], (*comms)[i], i, A_shard[i], B_buf[i], C_full[i],
                     g.devs[i].compute});
  }
  TRY(run_pipeline(parts, ngpus, M, N, K));
  TRY(sync_all(ngpus));
  for (int i = 0; i < ngpus; ++i) {
    ncclResult_t ar = ncclSuccess;
    api->CommGetAsyncError((*comms)[i], &ar);
    TRY(nccl_check(ar, "NCCL async"));
  }
  return GIGA_OK;
}

// Host buffers on one GPU (the paper's call): a two-phase schedule over three
// engines -- host-to-device copies on the comm stream, GEMMs on the compute stream,
// device-to-host copies on the d2h stream -- so that the PCIe transfers hide behind the
// tensor cores instead of preceding them (with pinned host memory). The split into phases,
// K-chunks and row blocks is chosen per shape by host_plan_choose (host_plan.cpp):
//   phase 1, the first `Me` rows: their A columns and the B rows of K-chunk c arrive together
//     and the GEMM of chunk c accumulates into C (C += A_c B_c), so compute starts after the
//     first (small) chunk instead of after all of B;
//   phase 2, the remaining rows in row blocks over the full K (B is complete by then): block
//     q's A rows are copied while q-1 computes, and C goes back to the host -- the early rows
//     first, then block by block -- over the other PCIe direction.
int host_pipeline(DevCtx &d, const float *A, const float *B, float *C, int64_t M, int64_t N,
                  int64_t K) {
  CK(cudaSetDevice(d.dev));
  HostRates rates = host_rates_default();
  int nsm = 0;
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, d.dev));
  rates.clusters = std::max(1, nsm / 2);
  const HostPlan plan = host_plan_choose(M, N, K, rates);
  static_assert(kHostMaxChunks <= kMaxChunks, "event arrays");
  const int64_t Me = plan.Me;
  const int P = plan.P, Q = plan.Q;
  const int64_t *kb = plan.kb;
  TRY(ws_reserve(d, {{&d.A_h, size_t(M * K) * 4},
                     {&d.B_h, size_t(K * N) * 4},
                     {&d.C_h, size_t(M * N) * 4},
                     {&d.A_lo, lo_bytes(M * K)},
                     {&d.B_lo, lo_bytes(K * N)}}));
  float *Ad = fptr(d.A_h), *Bd = fptr(d.B_h), *Cd = fptr(d.C_h), *Alo = lo_at(d.A_lo),
        *Blo = lo_at(d.B_lo);
  // $GIGA_HOST_TRACE=1: timing events after every piece of every engine, printed as one JSON
  // line on stderr (a timeline to compare with the plan's model)
  const bool trace = env_int("GIGA_HOST_TRACE", 0) != 0;
  enum { T0 = 0, TK = 1, TR = TK + kMaxChunks, TG1 = TR + kMaxChunks, TG2 = TG1 + kMaxChunks,
         TDE = TG2 + kMaxChunks, TD = TDE + 1, TN = TD + kMaxChunks };
  if (trace && d.ev_trace.empty()) {
    d.ev_trace.assign(TN, nullptr);
    for (auto &e : d.ev_trace) CK(cudaEventCreate(&e));
  }
  auto mark = [&](int slot, cudaStream_t st) -> int {
    if (trace) CK(cudaEventRecord(d.ev_trace[slot], st));
    return GIGA_OK;
  };
  TRY(mark(T0, d.comm));
  // host -> device: (early A columns, B rows) per K-chunk, then the late A row blocks
  for (int c = 0; c < P; ++c) {
    const int64_t Kc = kb[c + 1] - kb[c];
    if (Me > 0)
      CK(cudaMemcpy2DAsync(Ad + kb[c], size_t(K) * 4, A + kb[c], size_t(K) * 4,
                           size_t(Kc) * 4, size_t(Me), cudaMemcpyHostToDevice, d.comm));
    CK(cudaMemcpyAsync(Bd + kb[c] * N, B + kb[c] * N, size_t(Kc * N) * 4,
                       cudaMemcpyHostToDevice, d.comm));
    CK(cudaEventRecord(d.ev_kchunk[c], d.comm));
    TRY(mark(TK + c, d.comm));
  }
  for (int q = 0; q < Q; ++q) {
    const int64_t q0 = plan.rb[q], q1 = plan.rb[q + 1];
    if (q1 > q0)
      CK(cudaMemcpyAsync(Ad + q0 * K, A + q0 * K, size_t((q1 - q0) * K) * 4,
                         cudaMemcpyHostToDevice, d.comm));
    CK(cudaEventRecord(d.ev_rchunk[q], d.comm));
    TRY(mark(TR + q, d.comm));
  }
  // phase 1: early rows, K-chunk by K-chunk, accumulating in C
  GemmExtra ex;
  ex.lda = K;
  ex.ldb = N;
  for (int c = 0; c < P; ++c) {
    const int64_t Kc = kb[c + 1] - kb[c];
    CK(cudaStreamWaitEvent(d.compute, d.ev_kchunk[c], 0));
    TRY(split(Bd + kb[c] * N, at(Blo, kb[c] * N), Kc * N, d.compute));
    if (Me == 0) continue;
    if (Alo)
      CK(timed(1, d.compute, [&] {
        return launch_split_lo_2d(Ad + kb[c], Alo + kb[c], Me, Kc, K, d.compute);
      }));
    GemmExtra e = ex;
    e.accumulate = c > 0;
    TRY(gemm_chunk(Ad + kb[c], at(Alo, kb[c]), Bd + kb[c] * N, at(Blo, kb[c] * N), Cd, Me, N,
                   Kc, e, d.compute));
    TRY(mark(TG1 + c, d.compute));
  }
  if (Me > 0) {
    CK(cudaEventRecord(d.ev_c, d.compute));
    CK(cudaStreamWaitEvent(d.d2h, d.ev_c, 0));
    CK(cudaMemcpyAsync(C, Cd, size_t(Me * N) * 4, cudaMemcpyDeviceToHost, d.d2h));
    TRY(mark(TDE, d.d2h));
  }
  // phase 2: late row blocks over the full K (phase 1 waited for every K-chunk of B)
  for (int q = 0; q < Q; ++q) {
    const int64_t q0 = plan.rb[q], q1 = plan.rb[q + 1];
    CK(cudaStreamWaitEvent(d.compute, d.ev_rchunk[q], 0));
    if (q1 > q0) {
      TRY(split(Ad + q0 * K, at(Alo, q0 * K), (q1 - q0) * K, d.compute));
      TRY(gemm(Ad + q0 * K, at(Alo, q0 * K), Bd, Blo, Cd + q0 * N, q1 - q0, N, K, N,
               d.compute));
    }
    CK(cudaEventRecord(d.ev_done[q], d.compute));
    TRY(mark(TG2 + q, d.compute));
    CK(cudaStreamWaitEvent(d.d2h, d.ev_done[q], 0));
    if (q1 > q0)
      CK(cudaMemcpyAsync(C + q0 * N, Cd + q0 * N, size_t((q1 - q0) * N) * 4,
                         cudaMemcpyDeviceToHost, d.d2h));
    TRY(mark(TD + q, d.d2h));
  }
  CK(cudaStreamSynchronize(d.d2h));
  CK(cudaStreamSynchronize(d.compute));
  CK(cudaStreamSynchronize(d.comm));
  if (trace) {
    auto ms = [&](int slot) {
      float v = 0;
      cudaEventElapsedTime(&v, d.ev_trace[T0], d.ev_trace[slot]);
      return double(v);
    };
    auto list = [&](int base, int n) {
      std::string o = "[";
      for (int i = 0; i < n; ++i) o += (i ? ", " : "") + std::to_string(ms(base + i));
      return o + "]";
    };
    fprintf(stderr,
            "{\"host_trace\": {\"M\": %lld, \"N\": %lld, \"K\": %lld, \"Me\": %lld, "
            "\"P\": %d, \"Q\": %d, \"model_ms\": %.3f, \"h2d_k\": %s, \"h2d_r\": %s, "
            "\"gemm1\": %s, \"gemm2\": %s, \"d2h_early\": %.3f, \"d2h\": %s}}\n",
            (long long)M, (long long)N, (long long)K, (long long)Me, P, Q, plan.t_model * 1e3,
            list(TK, P).c_str(), list(TR, Q).c_str(), list(TG1, Me > 0 ? P : 0).c_str(),
            list(TG2, Q).c_str(), Me > 0 ? ms(TDE) : 0.0, list(TD, Q).c_str());
  }
  return GIGA_OK;
}

int matmul_locked(const float *A, const float *B, float *C, int64_t M, int64_t N, int64_t K,
                  int ngpus) {
  int da = -1, db = -1, dc = -1;
  const int ka = pointer_kind(A, &da), kb = pointer_kind(B, &db), kc = pointer_kind(C, &dc);
  if (ka != kb || kb != kc)
    return fail(GIGA_ERR_INVALID_ARG, "A, B, C must be all host or all device pointers");
  const bool device = ka == 1;
  if (device && (da != g.devs[0].dev || db != g.devs[0].dev || dc != g.devs[0].dev))
    return fail(GIGA_ERR_INVALID_ARG, "device pointers must all live on GPU %d", g.devs[0].dev);

  if (device && ngpus == 1) {
    DevCtx &d = g.devs[0];
    CK(cudaSetDevice(d.dev));
    TRY(shard_compute(d, d.compute, A, M, B, C, N, N, K, nullptr));
    return sync_all(1);
  }
  if (!device && ngpus == 1 && K % 4 == 0 && N % 4 == 0) return host_pipeline(g.devs[0], A, B, C, M, N, K);

  // Stage: every GPU gets its A row block and a B buffer; GPU 0 gets B.
  for (int i = 0; i < ngpus; ++i) {
    DevCtx &d = g.devs[i];
    CK(cudaSetDevice(d.dev));
    int64_t r0, rows;
    partition_rows(M, ngpus, i, &r0, &rows);
    const bool own_b = !(device && i == 0);
    TRY(ws_reserve(d, {{&d.A_h, size_t(std::max<int64_t>(rows, 1) * K) * 4},
                       {&d.B_h, own_b ? size_t(K * N) * 4 : 0},
                       {&d.C_h, size_t(std::max<int64_t>(rows, 1) * N) * 4}}));
    if (rows > 0)
      CK(cudaMemcpyAsync(d.A_h.p, A + r0 * K, size_t(rows * K) * 4,
                         device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, d.compute));
    if (i == 0 && !device)
      CK(cudaMemcpyAsync(d.B_h.p, B, size_t(K * N) * 4, cudaMemcpyHostToDevice, d.compute));
  }
  const float *B0 = device ? B : fptr(g.devs[0].B_h);
  if (ngpus > 1 && !device && transport_p2p() && K % 4 == 0 && N % 4 == 0) {
    // copy-engine chain for B; each GPU writes only its rows and copies them straight home
    std::vector<Part> parts;
    for (int i = 0; i < ngpus; ++i) {
      DevCtx &d = g.devs[i];
      Part p{&d, nullptr, i, fptr(d.A_h), i == 0 ? const_cast<float *>(B0) : fptr(d.B_h),
             nullptr, d.compute};
      p.C_rows = fptr(d.C_h);
      parts.push_back(p);
    }
    TRY(run_p2p(parts, M, N, K, /*gather=*/false));
    for (int i = 0; i < ngpus; ++i) {
      DevCtx &d = g.devs[i];
      CK(cudaSetDevice(d.dev));
      int64_t r0, rows;
      partition_rows(M, ngpus, i, &r0, &rows);
      if (rows > 0)
        CK(cudaMemcpyAsync(C + r0 * N, d.C_h.p, size_t(rows * N) * 4, cudaMemcpyDeviceToHost,
                           d.compute));
    }
    return sync_all(ngpus);
  }
  if (ngpus > 1) {
    std::vector<ncclComm_t> *comms = nullptr;
    TRY(get_comms(ngpus, &comms));
    const NcclApi *api = nccl_api(nullptr);
    // B must be on GPU 0 before the broadcast reads it
    CK(cudaSetDevice(g.devs[0].dev));
    CK(cudaEventRecord(g.devs[0].ev_start, g.devs[0].compute));
    for (int i = 0; i < ngpus; ++i) {
      CK(cudaSetDevice(g.devs[i].dev));
      CK(cudaStreamWaitEvent(g.devs[i].comm, g.devs[0].ev_start, 0));
    }
    TRY(nccl_check(api->GroupStart(), "ncclGroupStart"));
    for (int i = 0; i < ngpus; ++i) {
      DevCtx &d = g.devs[i];
      CK(cudaSetDevice(d.dev));
      float *dst = (i == 0) ? const_cast<float *>(B0) : fptr(d.B_h);
      ncclResult_t r =
          api->Broadcast(B0, dst, size_t(K * N), ncclFloat32, 0, (*comms)[i], d.comm);
      if (r != ncclSuccess) {
        api->GroupEnd();
        return nccl_check(r, "ncclBroadcast(B)");
      }
    }
    TRY(nccl_check(api->GroupEnd(), "ncclGroupEnd"));
  }
  for (int i = 0; i < ngpus; ++i) {
    DevCtx &d = g.devs[i];
    CK(cudaSetDevice(d.dev));
    int64_t r0, rows;
    partition_rows(M, ngpus, i, &r0, &rows);
    cudaEvent_t wait = nullptr;
    if (ngpus > 1) {
      CK(cudaEventRecord(d.ev_b, d.comm));
      wait = d.ev_b;
    }
    const float *Bi = (i == 0) ? B0 : fptr(d.B_h);
    float *Ci = (device && i == 0) ? C + r0 * N : fptr(d.C_h);
    TRY(shard_compute(d, d.compute, fptr(d.A_h), rows, Bi, Ci, N, N, K, wait));
    if (rows > 0 && !(device && i == 0))
      CK(cudaMemcpyAsync(C + r0 * N, d.C_h.p, size_t(rows * N) * 4,
                         device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, d.compute));
  }
  return sync_all(ngpus);
}

// Library state for the single-process API on the given CUDA ordinals (repeats allowed).
int init_devices_locked(const std::vector<int> &devs) {
  const int n = int(devs.size());
  for (int i = 0; i < n; ++i) TRY(check_sm100(devs[i]));
  if (ensure_tma_encoder() != 0)
    return fail(GIGA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
  g.devs.assign(n, DevCtx{});
  for (int i = 0; i < n; ++i) {
    int rc = ctx_create(g.devs[i], devs[i]);
    if (rc != GIGA_OK) {
      for (auto &d : g.devs) ctx_destroy(d);
      g.devs.clear();
      return rc;
    }
  }
  // peer access so NCCL / copies / epilogue stores use NVLink directly (best effort)
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      if (devs[i] == devs[j]) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, devs[i], devs[j]);
      if (can) {
        cudaSetDevice(devs[i]);
        cudaDeviceEnablePeerAccess(devs[j], 0);
        cudaGetLastError();
      }
    }
  g.mode = 1;
  return GIGA_OK;
}

}  // namespace
}  // namespace giga

using namespace giga;

// =========================================================================================
// C ABI
extern "C" {

const char *giga_last_error(void) { return t_err.c_str(); }

int giga_partition(int64_t M, int ngpus, int gi, int64_t *row0, int64_t *rows) {
  if (M < 0 || ngpus < 1 || gi < 0 || gi >= ngpus || !row0 || !rows)
    return fail(GIGA_ERR_INVALID_ARG, "giga_partition: bad arguments");
  partition_rows(M, ngpus, gi, row0, rows);
  return GIGA_OK;
}

int giga_num_devices(void) {
  std::lock_guard<std::mutex> lk(g.mu);
  return g.mode == 1 ? int(g.devs.size()) : (g.mode == 2 ? 1 : 0);
}

int giga_init(int ngpus_max) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (g.mode != 0) return fail(GIGA_ERR_ALREADY_INITIALIZED, "giga_init: already initialised");
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    return fail(GIGA_ERR_NO_DEVICE, "no CUDA device visible");
  }
  const int n = ngpus_max <= 0 ? count : ngpus_max;
  if (n > count)
    return fail(GIGA_ERR_NO_DEVICE, "asked for %d GPUs, %d visible", ngpus_max, count);
  std::vector<int> devs(n);
  for (int i = 0; i < n; ++i) devs[i] = i;
  return init_devices_locked(devs);
}

int giga_init_devices(const int *devices, int n) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (g.mode != 0)
    return fail(GIGA_ERR_ALREADY_INITIALIZED, "giga_init_devices: already initialised");
  if (!devices || n < 1) return fail(GIGA_ERR_INVALID_ARG, "giga_init_devices: empty list");
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    return fail(GIGA_ERR_NO_DEVICE, "no CUDA device visible");
  }
  for (int i = 0; i < n; ++i)
    if (devices[i] < 0 || devices[i] >= count)
      return fail(GIGA_ERR_NO_DEVICE, "device %d not visible", devices[i]);
  return init_devices_locked(std::vector<int>(devices, devices + n));
}

int giga_finalize(void) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (g.mode == 0) return GIGA_OK;
  const NcclApi *api = nccl_api(nullptr);
  if (api) {
    for (auto &kv : g.comms)
      for (ncclComm_t c : kv.second)
        if (c) api->CommDestroy(c);
    if (g.rank_comm) api->CommDestroy(g.rank_comm);
  }
  g.comms.clear();
  g.rank_comm = nullptr;
  if (!g.devs.empty()) cudaSetDevice(g.devs[0].dev);
  p2p_release();
  for (auto &d : g.devs) ctx_destroy(d);
  g.devs.clear();
  {
    std::lock_guard<std::mutex> tl(g_tmu);
    for (auto &r : g_tpending) {
      cudaEventDestroy(r.a);
      cudaEventDestroy(r.b);
    }
    g_tpending.clear();
    for (auto &p : g_tpool) cudaEventDestroy(p.second);
    g_tpool.clear();
  }
  g.mode = 0;
  return GIGA_OK;
}

int giga_matmul(const float *A, const float *B, float *C, int64_t M, int64_t N, int64_t K,
                int ngpus) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (g.mode != 1) return fail(GIGA_ERR_NOT_INITIALIZED, "giga_matmul: call giga_init first");
  if (!A || !B || !C) return fail(GIGA_ERR_INVALID_ARG, "giga_matmul: NULL pointer");
  TRY(check_dims(M, N, K));
  if (ngpus < 1 || ngpus > int(g.devs.size()))
    return fail(GIGA_ERR_INVALID_ARG, "ngpus=%d outside [1, %d]", ngpus, int(g.devs.size()));
  if (overlaps(C, size_t(M * N) * 4, A, size_t(M * K) * 4) ||
      overlaps(C, size_t(M * N) * 4, B, size_t(K * N) * 4))
    return fail(GIGA_ERR_INVALID_ARG, "C overlaps A or B");
  TRY(quiesce(ngpus));
  return matmul_locked(A, B, C, M, N, K, ngpus);
}

int giga_matmul_sharded(const float *const *A_shard, float *const *B_buf, float *const *C_full,
                        int64_t M, int64_t N, int64_t K, int ngpus) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (g.mode != 1)
    return fail(GIGA_ERR_NOT_INITIALIZED, "giga_matmul_sharded: call giga_init first");
  if (!A_shard || !B_buf || !C_full) return fail(GIGA_ERR_INVALID_ARG, "NULL pointer array");
  TRY(check_dims(M, N, K));
  if (ngpus < 1 || ngpus > int(g.devs.size()))
    return fail(GIGA_ERR_INVALID_ARG, "ngpus=%d outside [1, %d]", ngpus, int(g.devs.size()));
  for (int i = 0; i < ngpus; ++i) {
    int64_t r0, rows;
    partition_rows(M, ngpus, i, &r0, &rows);
    if ((rows > 0 && !A_shard[i]) || !B_buf[i] || !C_full[i])
      return fail(GIGA_ERR_INVALID_ARG, "NULL buffer for GPU %d", i);
    int dv = -1;
    if (pointer_kind(C_full[i], &dv) != 1 || dv != g.devs[i].dev ||
        pointer_kind(B_buf[i], &dv) != 1 || dv != g.devs[i].dev ||
        (rows > 0 && (pointer_kind(A_shard[i], &dv) != 1 || dv != g.devs[i].dev)))
      return fail(GIGA_ERR_INVALID_ARG, "buffers for GPU %d must be device memory on it", i);
    if (overlaps(C_full[i], size_t(M * N) * 4, B_buf[i], size_t(K * N) * 4) ||
        (rows > 0 && overlaps(C_full[i], size_t(M * N) * 4, A_shard[i], size_t(rows * K) * 4)))
      return fail(GIGA_ERR_INVALID_ARG, "C_full[%d] overlaps A or B", i);
  }
  TRY(quiesce(ngpus));
  return sharded_locked(A_shard, B_buf, C_full, M, N, K, ngpus);
}

// ---- multi-process (one process per GPU) ------------------------------------------------

int giga_comm_unique_id(uint8_t id[128]) {
  if (!id) return fail(GIGA_ERR_INVALID_ARG, "NULL id");
  const char *why = nullptr;
  const NcclApi *api = nccl_api(&why);
  if (!api) return fail(GIGA_ERR_COMM, "NCCL unavailable: %s", why ? why : "?");
  ncclUniqueId u;
  TRY(nccl_check(api->GetUniqueId(&u), "ncclGetUniqueId"));
  memcpy(id, u.internal, 128);
  return GIGA_OK;
}

int giga_rank_init(int rank, int world, int device, const uint8_t id[128]) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (g.mode != 0)
    return fail(GIGA_ERR_ALREADY_INITIALIZED, "giga_rank_init: already initialised");
  if (world < 1 || rank < 0 || rank >= world || device < 0 ||
      (world > 1 && !id && !transport_p2p()))
    return fail(GIGA_ERR_INVALID_ARG, "giga_rank_init: bad rank/world/device/id");
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || device >= count) {
    cudaGetLastError();
    return fail(GIGA_ERR_NO_DEVICE, "device %d not visible", device);
  }
  TRY(check_sm100(device));
  if (ensure_tma_encoder() != 0)
    return fail(GIGA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
  g.devs.assign(1, DevCtx{});
  int rc = ctx_create(g.devs[0], device);
  if (rc != GIGA_OK) {
    ctx_destroy(g.devs[0]);
    g.devs.clear();
    return rc;
  }
  // NCCL communicator unless the peer-to-peer transport carries everything (it then also
  // runs several ranks on one device, which NCCL refuses)
  if ((world > 1 && !transport_p2p()) || force_comm()) {  // GIGA_FORCE_COMM: world size 1
    const char *why = nullptr;
    const NcclApi *api = nccl_api(&why);
    if (!api) {
      ctx_destroy(g.devs[0]);
      g.devs.clear();
      return fail(GIGA_ERR_COMM, "NCCL unavailable: %s", why ? why : "?");
    }
    ncclUniqueId u;
    if (id)
      memcpy(u.internal, id, 128);
    else if ((rc = nccl_check(api->GetUniqueId(&u), "ncclGetUniqueId")) != GIGA_OK) {
      ctx_destroy(g.devs[0]);
      g.devs.clear();
      return rc;
    }
    cudaSetDevice(device);
    ncclConfig_t cfg = comm_config();
    rc = nccl_check(api->CommInitRankConfig(&g.rank_comm, world, u, rank, &cfg),
                    "ncclCommInitRankConfig");
    if (rc != GIGA_OK) {
      ctx_destroy(g.devs[0]);
      g.devs.clear();
      return rc;
    }
  }
  g.rank = rank;
  g.world = world;
  g.mode = 2;
  return GIGA_OK;
}

int giga_matmul_rank(const float *A_shard, float *B, float *C_full, int64_t M, int64_t N,
                     int64_t K, void *stream) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (g.mode != 2) return fail(GIGA_ERR_NOT_INITIALIZED, "giga_matmul_rank: not initialised");
  TRY(check_dims(M, N, K));
  int64_t r0, rows;
  partition_rows(M, g.world, g.rank, &r0, &rows);
  if ((rows > 0 && !A_shard) || !B || !C_full)
    return fail(GIGA_ERR_INVALID_ARG, "giga_matmul_rank: NULL pointer");
  DevCtx &d = g.devs[0];
  CK(cudaSetDevice(d.dev));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : d.compute;
  // calls share the rank's workspace: a call starts after the previous one, whatever the
  // caller's streams
  if (d.has_last) CK(cudaStreamWaitEvent(st, d.ev_last, 0));
  int rc;
  if (g.p2p.ready && transport_p2p()) {
    rc = run_p2p_rank(d, st, A_shard, B, C_full, M, N, K);
  } else if (!g.rank_comm) {
    rc = shard_compute(d, st, A_shard, rows, B, C_full + r0 * N, N, N, K, nullptr);
  } else {
    std::vector<Part> parts{{&d, g.rank_comm, g.rank, A_shard, B, C_full, st}};
    rc = run_pipeline(parts, g.world, M, N, K);
  }
  TRY(rc);
  CK(cudaEventRecord(d.ev_last, st));
  d.has_last = true;
  return GIGA_OK;
}

// ---- vector operations -------------------------------------------------

int giga_dot(const float *x, const float *y, int64_t n, int ngpus, double *result) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (g.mode != 1) return fail(GIGA_ERR_NOT_INITIALIZED, "giga_dot: call giga_init first");
  if (!x || !y || !result || n < 1)
    return fail(GIGA_ERR_INVALID_ARG, "giga_dot: NULL pointer or n < 1");
  if (ngpus < 1 || ngpus > int(g.devs.size()))
    return fail(GIGA_ERR_INVALID_ARG, "ngpus=%d outside [1, %d]", ngpus, int(g.devs.size()));
  int dx = -1, dy = -1;
  const int kx = pointer_kind(x, &dx), ky = pointer_kind(y, &dy);
  if (kx != ky) return fail(GIGA_ERR_INVALID_ARG, "x, y must be both host or both device");
  const bool device = kx == 1;
  if (device && (dx != g.devs[0].dev || dy != g.devs[0].dev))
    return fail(GIGA_ERR_INVALID_ARG, "device pointers must live on GPU %d", g.devs[0].dev);
  TRY(quiesce(ngpus));
  // "halving, with remainder going on one", generalised: giga_partition's rule
  for (int i = 0; i < ngpus; ++i) {
    DevCtx &d = g.devs[i];
    CK(cudaSetDevice(d.dev));
    int64_t r0, rows;
    partition_rows(n, ngpus, i, &r0, &rows);
    TRY(vec_ws(d));
    if (device && ngpus == 1) {
      TRY(dot_partial(d, x, y, rows, d.compute));
      continue;
    }
    TRY(ws_reserve(d, {{&d.A_h, size_t(std::max<int64_t>(rows, 1)) * 4},
                       {&d.B_h, size_t(std::max<int64_t>(rows, 1)) * 4}}));
    if (rows > 0) {
      if (device) {
        CK(cudaMemcpyPeerAsync(d.A_h.p, d.dev, x + r0, g.devs[0].dev, size_t(rows) * 4,
                               d.compute));
        CK(cudaMemcpyPeerAsync(d.B_h.p, d.dev, y + r0, g.devs[0].dev, size_t(rows) * 4,
                               d.compute));
      } else {
        CK(cudaMemcpyAsync(d.A_h.p, x + r0, size_t(rows) * 4, cudaMemcpyHostToDevice,
                           d.compute));
        CK(cudaMemcpyAsync(d.B_h.p, y + r0, size_t(rows) * 4, cudaMemcpyHostToDevice,
                           d.compute));
      }
    }
    TRY(dot_partial(d, fptr(d.A_h), fptr(d.B_h), rows, d.compute));
  }
  // the host sums the per-GPU partials in device order, in fp64
  double total = 0.0;
  for (int i = 0; i < ngpus; ++i) {
    DevCtx &d = g.devs[i];
    CK(cudaSetDevice(d.dev));
    double part = 0.0;
    CK(cudaMemcpyAsync(&part, vec_out(d), sizeof(double), cudaMemcpyDeviceToHost, d.compute));
    CK(cudaStreamSynchronize(d.compute));
    total += part;
  }
  *result = total;
  return GIGA_OK;
}

int giga_l2norm(const float *x, int64_t n, int ngpus, double *result) {
  double d2 = 0.0;
  TRY(giga_dot(x, x, n, ngpus, &d2));
  *result = sqrt(d2);  // once, on the host, after the reduction
  return GIGA_OK;
}

int giga_dot_rank(const float *x_shard, const float *y_shard, int64_t n, double *result,
                  void *stream) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (g.mode != 2) return fail(GIGA_ERR_NOT_INITIALIZED, "giga_dot_rank: not initialised");
  int64_t r0, rows;
  if (n < 1) return fail(GIGA_ERR_INVALID_ARG, "giga_dot_rank: n < 1");
  partition_rows(n, g.world, g.rank, &r0, &rows);
  if (!result || (rows > 0 && (!x_shard || !y_shard)))
    return fail(GIGA_ERR_INVALID_ARG, "giga_dot_rank: NULL pointer");
  DevCtx &d = g.devs[0];
  CK(cudaSetDevice(d.dev));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : d.compute;
  TRY(dot_partial(d, x_shard, y_shard, rows, st));
  if (g.p2p.ready && g.world > 1) return p2p_dot_allreduce(d, st, result);
  if (g.rank_comm) {  // every rank gets the sum of the partials
    const NcclApi *api = nccl_api(nullptr);
    TRY(nccl_check(api->AllReduce(vec_out(d), vec_out(d), 1, ncclFloat64, ncclSum, g.rank_comm,
                                  st),
                   "ncclAllReduce(dot)"));
  }
  CK(cudaMemcpyAsync(result, vec_out(d), sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return GIGA_OK;
}

// ---- rank-mode peer-to-peer registration (CUDA IPC) ---------------------------------------

namespace {
struct P2PBlob {
  cudaIpcMemHandle_t hB, hC, hF;
  uint64_t offB, offC;
};
static_assert(sizeof(P2PBlob) <= GIGA_P2P_BLOB_BYTES, "blob too small");

int ipc_handle(const void *p, cudaIpcMemHandle_t *h, uint64_t *off) {
  CUdeviceptr base = 0;
  size_t size = 0;
  if (drv_api()->range(&base, &size, CUdeviceptr(p)) != CUDA_SUCCESS)
    return fail(GIGA_ERR_INVALID_ARG, "not a device allocation: %p", p);
  *off = uint64_t(reinterpret_cast<uintptr_t>(p) - uintptr_t(base));
  CK(cudaIpcGetMemHandle(h, reinterpret_cast<void *>(base)));
  return GIGA_OK;
}
}  // namespace

int giga_rank_p2p_export(const float *B, float *C_full, uint8_t *blob) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (g.mode != 2) return fail(GIGA_ERR_NOT_INITIALIZED, "giga_rank_p2p_export: rank mode only");
  if (!B || !C_full || !blob) return fail(GIGA_ERR_INVALID_ARG, "NULL pointer");
  if (!drv_api()) return fail(GIGA_ERR_UNSUPPORTED, "driver stream-memory ops unavailable");
  DevCtx &d = g.devs[0];
  CK(cudaSetDevice(d.dev));
  RankP2P &x = g.p2p;
  if (!x.flags) {
    void *f = nullptr;
    CK(cudaMalloc(&f, kFlagBytes));
    CK(cudaMemset(f, 0, kFlagBytes));
    x.flags = static_cast<uint32_t *>(f);
  }
  P2PBlob b{};
  TRY(ipc_handle(B, &b.hB, &b.offB));
  TRY(ipc_handle(C_full, &b.hC, &b.offC));
  uint64_t off0 = 0;
  TRY(ipc_handle(x.flags, &b.hF, &off0));
  x.B = const_cast<float *>(B);
  x.C = C_full;
  memset(blob, 0, GIGA_P2P_BLOB_BYTES);
  memcpy(blob, &b, sizeof b);
  return GIGA_OK;
}

int giga_rank_p2p_import(const uint8_t *blobs, int world) {
  std::lock_guard<std::mutex> lk(g.mu);
  if (g.mode != 2) return fail(GIGA_ERR_NOT_INITIALIZED, "giga_rank_p2p_import: rank mode only");
  RankP2P &x = g.p2p;
  if (!blobs || world != g.world || !x.flags)
    return fail(GIGA_ERR_INVALID_ARG, "giga_rank_p2p_import: call export first, world=%d", world);
  DevCtx &d = g.devs[0];
  CK(cudaSetDevice(d.dev));
  for (void *p : x.opened) cudaIpcCloseMemHandle(p);
  x.opened.clear();
  x.peerB.assign(world, nullptr);
  x.peerC.assign(world, nullptr);
  x.peerF.assign(world, nullptr);
  for (int q = 0; q < world; ++q) {
    if (q == g.rank) {
      x.peerB[q] = x.B;
      x.peerC[q] = x.C;
      x.peerF[q] = x.flags;
      continue;
    }
    P2PBlob b;
    memcpy(&b, blobs + size_t(q) * GIGA_P2P_BLOB_BYTES, sizeof b);
    void *pb = nullptr, *pc = nullptr, *pf = nullptr;
    CK(cudaIpcOpenMemHandle(&pb, b.hB, cudaIpcMemLazyEnablePeerAccess));
    x.opened.push_back(pb);
    CK(cudaIpcOpenMemHandle(&pc, b.hC, cudaIpcMemLazyEnablePeerAccess));
    x.opened.push_back(pc);
    CK(cudaIpcOpenMemHandle(&pf, b.hF, cudaIpcMemLazyEnablePeerAccess));
    x.opened.push_back(pf);
    x.peerB[q] = reinterpret_cast<float *>(static_cast<char *>(pb) + b.offB);
    x.peerC[q] = reinterpret_cast<float *>(static_cast<char *>(pc) + b.offC);
    x.peerF[q] = static_cast<uint32_t *>(pf);
  }
  // call numbers stay monotonic across re-registrations: the flag pages keep old values
  x.ready = true;
  return GIGA_OK;
}

// ---- pipeline plan (host arithmetic) -----------------------------------------------------

int giga_pipeline_plan(int64_t M, int64_t N, int64_t K, int world, int *kchunks,
                       int64_t *kbounds, int *rchunks) {
  if (M < 1 || N < 1 || K < 1 || world < 1 || !kchunks || !kbounds || !rchunks)
    return fail(GIGA_ERR_INVALID_ARG, "giga_pipeline_plan: bad arguments");
  const Plan pl = make_plan(M, K, world, (K % 4 == 0) && (N % 4 == 0));
  *kchunks = pl.pb;
  *rchunks = pl.pc;
  for (int c = 0; c <= pl.pb; ++c) kbounds[c] = pl.kb[c];
  return GIGA_OK;
}

int giga_plan_block(int64_t M, int world, int rchunks, int owner, int q, int64_t *row0,
                    int64_t *rows) {
  if (M < 0 || world < 1 || rchunks < 1 || owner < 0 || owner >= world || q < 0 ||
      q >= rchunks || !row0 || !rows)
    return fail(GIGA_ERR_INVALID_ARG, "giga_plan_block: bad arguments");
  plan_block(M, world, rchunks, owner, q, row0, rows);
  return GIGA_OK;
}

int giga_host_plan(int64_t M, int64_t N, int64_t K, int num_sms, int64_t *Me, int *P,
                   int64_t *kb, int *Q, int64_t *rb, double *t_model) {
  if (M < 1 || N < 1 || K < 1 || !Me || !P || !kb || !Q || !rb || !t_model)
    return fail(GIGA_ERR_INVALID_ARG, "giga_host_plan: bad arguments");
  HostRates r = host_rates_default();
  r.clusters = std::max(1, (num_sms > 0 ? num_sms : 148) / 2);
  const HostPlan p = host_plan_choose(M, N, K, r);
  *Me = p.Me;
  *P = p.P;
  *Q = p.Q;
  for (int i = 0; i <= p.P; ++i) kb[i] = p.kb[i];
  for (int i = 0; i <= p.Q; ++i) rb[i] = p.rb[i];
  *t_model = p.t_model;
  return GIGA_OK;
}

// ---- building blocks ---------------------------------------------------------------------

int giga_split_lo(const float *x, float *lo, int64_t n, void *stream) {
  if (!x || !lo || n < 0 || !aligned16(x) || !aligned16(lo))
    return fail(GIGA_ERR_INVALID_ARG, "giga_split_lo: bad arguments");
  return split(x, lo, n, static_cast<cudaStream_t>(stream));
}

int giga_gemm_3xtf32_ex(const float *A, const float *A_lo, const float *B, const float *B_lo,
                        float *C, int64_t M, int64_t N, int64_t K, int64_t ldc, int terms,
                        int promote_kblocks, int cta_group, void *stream) {
  if (cta_group < 0 || cta_group > 2)
    return fail(GIGA_ERR_INVALID_ARG, "giga_gemm_3xtf32_ex: cta_group must be 0, 1 or 2");
  if (!A || !B || !C || (!A_lo) != (!B_lo) || (terms != 1 && terms != 3))
    return fail(GIGA_ERR_INVALID_ARG, "giga_gemm_3xtf32: bad pointers/terms");
  TRY(check_dims(M, N, K));
  if ((K & 3) || (N & 3) || (ldc & 3) || ldc < N || !aligned16(A) || !aligned16(B) ||
      !aligned16(C) || (A_lo && !aligned16(A_lo)) || (B_lo && !aligned16(B_lo)))
    return fail(GIGA_ERR_INVALID_ARG,
                "giga_gemm_3xtf32: needs K%%4 == N%%4 == ldc%%4 == 0, ldc >= N, 16B-aligned");
  if (ensure_tma_encoder() != 0) return fail(GIGA_ERR_CUDA, "TMA encoder unavailable");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  CK(timed(0, st, [&] {
    return launch_gemm_3xtf32(A, A_lo, B, B_lo, C, M, N, K, ldc, terms, promote_kblocks, st,
                              cta_group);
  }));
  return GIGA_OK;
}

int giga_gemm_3xtf32(const float *A, const float *A_lo, const float *B, const float *B_lo,
                     float *C, int64_t M, int64_t N, int64_t K, int64_t ldc, void *stream) {
  return giga_gemm_3xtf32_ex(A, A_lo, B, B_lo, C, M, N, K, ldc, 3, -1, 0, stream);
}

// ---- timing ------------------------------------------------------------------------------

int giga_timing_enable(int on) {
  std::lock_guard<std::mutex> lk(g_tmu);
  g_timing = on != 0;
  return GIGA_OK;
}

int giga_timing_reset(void) {
  std::lock_guard<std::mutex> lk(g_tmu);
  for (auto &r : g_tpending) {
    cudaEventSynchronize(r.b);
    g_tpool.push_back({r.dev, r.a});
    g_tpool.push_back({r.dev, r.b});
  }
  g_tpending.clear();
  g_tms[0] = g_tms[1] = 0;
  g_tcount[0] = g_tcount[1] = 0;
  return GIGA_OK;
}

int giga_timing_read(double *gemm_ms, int64_t *gemm_launches, double *split_ms,
                     int64_t *split_launches) {
  std::lock_guard<std::mutex> lk(g_tmu);
  for (auto &r : g_tpending) {
    cudaError_t e = cudaEventSynchronize(r.b);
    float ms = 0;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, r.a, r.b);
    if (e != cudaSuccess) {
      cudaGetLastError();
    } else {
      g_tms[r.kind] += ms;
      g_tcount[r.kind] += 1;
    }
    g_tpool.push_back({r.dev, r.a});
    g_tpool.push_back({r.dev, r.b});
  }
  g_tpending.clear();
  if (gemm_ms) *gemm_ms = g_tms[0];
  if (gemm_launches) *gemm_launches = g_tcount[0];
  if (split_ms) *split_ms = g_tms[1];
  if (split_launches) *split_launches = g_tcount[1];
  return GIGA_OK;
}

}  // extern "C"
