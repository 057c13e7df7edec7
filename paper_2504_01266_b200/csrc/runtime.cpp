// runtime.cpp -- libgiga's host runtime: errors, library state, kernel timing, the per-GPU
// workspace cache, the row-block partitioner, argument checks and the one-shard compute
// (each GPU multiplies its row block of A by B).
#include "runtime.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cmath>

namespace giga {

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

int fail_cuda(cudaError_t e, const char *what, const char *file, int line) {
  cudaGetLastError();  // clear a non-sticky error so the next call starts clean
  const int code = (e == cudaErrorMemoryAllocation) ? GIGA_ERR_OOM : GIGA_ERR_CUDA;
  const char *base = strrchr(file, '/');
  return fail(code, "%s failed at %s:%d: %s (%s)", what, base ? base + 1 : file, line,
              cudaGetErrorName(e), cudaGetErrorString(e));
}

State g;
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

// ---------------------------------------------------------------------------------------
// workspace: grow-only per-GPU buffers, reserved transactionally so a failed call leaves the
// device memory footprint exactly as it found it.

int ws_reserve(DevCtx & /*d: the buffers carry their device*/,
               std::initializer_list<std::pair<Buf *, size_t>> req) {
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
      return fail_cuda(e, "cudaMalloc(workspace)", __FILE__, __LINE__);
    }
    fresh.push_back({r.first, p});
  }
  for (auto &f : fresh) {
    size_t want = 0;
    for (auto &r : req)
      if (r.first == f.first) want = std::max(want, r.second);
    retire_buffer(f.first->p);  // freed now, or at finalize once a graph has captured work
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
  if (d.res_pinned) cudaFreeHost(d.res_pinned);
  if (d.trace_ns) cudaFree(d.trace_ns);
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
float *lo_at(Buf &b, int64_t off) { return lo_presplit() ? fptr(b) + off : nullptr; }

int split(const float *x, float *lo, int64_t n, cudaStream_t st) {
  if (!lo) return GIGA_OK;  // lo computed in the GEMM
  CK(timed(1, st, [&] { return launch_split_lo(x, lo, n, st); }));
  return GIGA_OK;
}

// One product GEMM with the scheme product_terms picks; for the TF32 + BF16 scheme its operand
// preparation launches first, timed as "split" launches (bench.py's roofline separates them).
int run_gemm(const float *A, const float *Alo, const float *B, const float *Blo, float *C,
             int64_t M, int64_t N, int64_t K, int64_t ldc, const GemmExtra &ex,
             cudaStream_t st) {
  int terms = product_terms(Alo, std::max(M, ex.rows_hint), N, K);
  GemmExtra e = ex;
  TermsPrep tp;
  if (terms == 4) {
    // 3xFP16: scaled fp16 hi / lo operands prepared in HBM
    const int64_t lda = e.lda ? e.lda : K, ldb = e.ldb ? e.ldb : N;
    CK(terms_prep_alloc(M, N, K, st, &tp, 4));
    if (!tp.Bh) {
      if (scheme_forced()) return fail(GIGA_ERR_OOM, "3xFP16 operand scratch unavailable");
      terms = 3;
    } else {
      if (!(e.b_prep_reuse && tp.b_matches(B, ldb, N, K)))
        CK(timed(1, st, [&] { return launch_prep16_b(B, ldb, N, K, &tp, st); },
                 kPrep16BLaunches));
      CK(timed(1, st, [&] { return launch_prep16_a(A, lda, M, K, &tp, st); },
               kPrep16ALaunches));
      e.prep = &tp;
      e.defer_fix = 1;
    }
  }
  if (terms == 2) {
    const int64_t lda = e.lda ? e.lda : K, ldb = e.ldb ? e.ldb : N;
    CK(terms_prep_alloc(M, N, K, st, &tp));
    // no scratch for the prepared operands (OOM, stream capture): 3xTF32, which builds its
    // lo operands on chip and beats the on-chip TF32 + BF16 variant
    if (!tp.Bhi && !scheme_forced()) terms = 3;
  }
  if (terms == 2) {
    const int64_t lda = e.lda ? e.lda : K, ldb = e.ldb ? e.ldb : N;
    if (tp.Bhi && !(e.b_prep_reuse && tp.b_matches(B, ldb, N, K)))
      CK(timed(1, st, [&] { return launch_prep_b(B, ldb, N, K, &tp, st); }));
    if (tp.Ahi) CK(timed(1, st, [&] { return launch_prep_a(A, lda, M, K, &tp, st); }));
    e.prep = &tp;
  }
  CK(timed(0, st, [&] {
    return launch_gemm_3xtf32(A, Alo, B, Blo, C, M, N, K, ldc, terms, -1, st, 0, &e);
  }));
  if (terms == 4) {
    const int64_t lda = e.lda ? e.lda : K, ldb = e.ldb ? e.ldb : N;
    CK(timed(1, st, [&] { return launch_fix16(A, lda, B, ldb, M, N, K, &tp, C, ldc, &e, st); },
             kFix16Launches));
  }
  return GIGA_OK;
}

int gemm(const float *A, const float *Alo, const float *B, const float *Blo, float *C,
         int64_t M, int64_t N, int64_t K, int64_t ldc, cudaStream_t st) {
  return run_gemm(A, Alo, B, Blo, C, M, N, K, ldc, GemmExtra(), st);
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
  // C_pad is fully written by the GEMM's TMA bulk stores; compute-sanitizer's initcheck does
  // not see those as initialising it and flags the copy-out below, so the (cold) padded path
  // zero-fills it first
  CK(cudaMemsetAsync(d.C_pad.p, 0, size_t(rows * N4) * 4, st));
  TRY(gemm(fptr(d.A_pad), lo_at(d.A_lo), fptr(d.B_pad), lo_at(d.B_lo), fptr(d.C_pad), rows, N4,
           K4, N4, st));
  CK(cudaMemcpy2DAsync(C, ldc * 4, d.C_pad.p, N4 * 4, N * 4, rows, cudaMemcpyDeviceToDevice,
                       st));
  return GIGA_OK;
}

// ---------------------------------------------------------------------------------------
// row-block partition (floor split, the remainder to the last GPU)

void partition_rows(int64_t M, int ngpus, int gi, int64_t *row0, int64_t *rows) {
  const int64_t base = M / ngpus;
  *row0 = int64_t(gi) * base;
  *rows = (gi == ngpus - 1) ? M - int64_t(ngpus - 1) * base : base;
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
  if (!d.res_pinned) CK(cudaMallocHost(reinterpret_cast<void **>(&d.res_pinned), 64));
  TRY(ws_reserve(d, {{&d.vec_ws, kVecWsBytes}}));
  CK(cudaMemset(d.vec_ws.p, 0, kVecWsBytes));  // ticket starts at zero
  return GIGA_OK;
}
double *vec_partials(DevCtx &d) { return static_cast<double *>(d.vec_ws.p); }
double *vec_out(DevCtx &d) { return vec_partials(d) + kDotMaxBlocks; }
unsigned *vec_ticket(DevCtx &d) { return reinterpret_cast<unsigned *>(vec_out(d) + 1); }

// The fp64 result on the host: an 8-byte copy into the pinned slot (a pageable destination
// would be staged by the driver), then the stream is awaited.
int read_result(DevCtx &d, cudaStream_t st, double *out) {
  CK(cudaMemcpyAsync(d.res_pinned, vec_out(d), sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  *out = *d.res_pinned;
  return GIGA_OK;
}

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
// pipeline plan and chunked GEMM (shared by the NCCL pipeline, p2p and host paths)

int env_int(const char *name, int dflt) {
  const char *e = getenv(name);
  return (e && *e) ? atoi(e) : dflt;
}

// Geometric chunk bounds: n pieces of [0, total) with weights ratio^i, interior bounds rounded
// to the nearest multiple of `align`; false if a piece would be shorter than `min_piece`.
static bool geometric_bounds(int64_t total, int n, double ratio, int64_t align,
                             int64_t min_piece, int64_t *b) {
  double sum = 0, w = 1;
  for (int i = 0; i < n; ++i, w *= ratio) sum += w;
  double cum = 0;
  w = 1;
  b[0] = 0;
  for (int i = 1; i < n; ++i, w *= ratio) {
    cum += w;
    b[i] = int64_t(double(total) * cum / sum / double(align) + 0.5) * align;
    if (b[i] - b[i - 1] < min_piece) return false;
  }
  b[n] = total;
  return b[n] - b[n - 1] >= min_piece;
}

// The K-chunks of B's distribution grow geometrically: the GEMM starts once the first (small)
// chunk has landed, and each later chunk's transfer hides behind the previous chunk's GEMM as
// long as the growth r stays below (GEMM time per K-row) / (transfer time per K-row)
// = (2 rows_max / R) / (4 / BW) = rows_max BW / (2 R), R ~ 255 TFLOP/s, BW ~ 600 GB/s (NCCL
// broadcast) or 770 GB/s (a copy-engine hop); r = 0.8 of that, at most 4, lowered until every
// chunk is >= 256 deep. The number of chunks pb (<= 6 with NCCL, <= 16 with p2p) minimises
//   startup + pb O,  startup = hops x (first chunk's transfer), hops = 1 (NCCL pipelines its
//   broadcast) or world - 1 (the p2p chain forwards whole chunks),
// O ~ 20 us per extra GEMM launch (launch gap and the partial last wave; measured with
// scripts/project_scaling.py: a 2048 x 4096^2 shard in 6 + 3 launches took 0.45 ms against
// 0.24 ms of work). The row chunks pc (<= 4) of the last K-chunk minimise the end of the last
// gather in a simulation of the two streams (GEMM of row chunk q, then its gather after the
// previous gather): big shards keep 4 chunks, small ones (c2 on 2 GPUs) take fewer launches.
// $GIGA_BCAST_CHUNKS / $GIGA_GATHER_CHUNKS force the counts; $GIGA_LAUNCH_US sets O.
// E.g. 32768^3 on 8 GPUs (NCCL): 6 chunks, 4 row chunks; 4096^3 on 2 GPUs: 3 and 2.
// Modelled time of one K-chunk GEMM launch over `rows` rows, operand preparation included:
// the scheme product_terms picks for it at that scheme's rate for this K -- short chunks pay
// the per-tile fill / epilogue and, for 3xFP16, the preparation of the whole Kc x N chunk of B
// (profiles/r02_chunk_rate_sweep_b.jsonl, after the 3xFP16 epilogue fix: 3xFP16
// ~460 k / (k + 530) TFLOP/s, 3xTF32 ~260 k / (k + 64), TF32 + BF16 ~255 k / (k + 128);
// r02_chunk_rate_sweep.jsonl had 3xFP16 at ~430 k / (k + 900)) -- times the last-wave quantisation of
// its 256 x 256 pair tiles on the 70 pairs the pipeline leaves to the GEMM, plus a launch
// cost O.
static double chunk_gemm_time(int64_t rows, int64_t N, int64_t Kc, double O) {
  if (rows <= 0 || Kc <= 0) return 0.0;
  const int t = product_terms(nullptr, rows, N, Kc);
  const double k = double(Kc);
  const double rate = t == 4 ? 460e12 * k / (k + 530.0)
                      : t == 2 ? 255e12 * k / (k + 128.0)
                               : 260e12 * k / (k + 64.0);
  const double waves = double((rows + 255) / 256) * double((N + 255) / 256) / 70.0;
  const double quant = waves / std::ceil(waves);
  return O + 2.0 * double(rows) * double(N) * k / (rate * quant);
}

Plan make_plan(int64_t M, int64_t N, int64_t K, int world, bool aligned) {
  Plan pl;
  int64_t rows_max = 0;
  for (int r = 0; r < world; ++r) {
    int64_t r0, rows;
    partition_rows(M, world, r, &r0, &rows);
    rows_max = std::max(rows_max, rows);
  }
  pl.kb[0] = 0;
  pl.kb[1] = K;
  if (!aligned) return pl;
  const bool p2p = transport_p2p();
  // transfer rate: the copy-engine chain at the NVLink peer-copy rate (770 GB/s measured,
  // B200_PROFILING.md); NCCL's kernels capped at $GIGA_NCCL_MAX_CTAS (= $GIGA_COMM_SMS, 8) CTAs
  // at an assumed $GIGA_NCCL_CTA_GBPS (50) GB/s each, at most 600 GB/s -- a model input to be
  // calibrated with GIGA_TRACE's per-chunk GB/s on a multi-GPU box.
  const double nccl_ctas = std::max(1, env_int("GIGA_NCCL_MAX_CTAS", env_int("GIGA_COMM_SMS", 8)));
  const double bw = p2p ? 770e9
                        : std::min(600e9, nccl_ctas * std::max(1, env_int("GIGA_NCCL_CTA_GBPS", 50)) * 1e9);
  // the shard GEMM's rate by the scheme its launches run (measured)
  const int terms = product_terms(nullptr, rows_max, N, K);
  const double R = terms == 4 ? 400e12 : terms == 2 ? 265e12 : 250e12;
  const double O = std::max(0, env_int("GIGA_LAUNCH_US", 20)) * 1e-6;
  const double r_max = std::min(4.0, std::max(1.0, 0.8 * double(rows_max) * bw / (2.0 * R)));
  const int hops = p2p ? std::max(1, world - 1) : 1;
  const int pb_env = env_int("GIGA_BCAST_CHUNKS", 0);
  const int pb_cap = int(std::min<int64_t>(
      pb_env > 0 ? std::min(pb_env, kMaxChunks) : (p2p ? kMaxChunks : 6),
      std::max<int64_t>(1, K / 256)));
  double best = 1e300;
  for (int pb = pb_env > 0 ? pb_cap : 1; pb <= pb_cap; ++pb) {
    int64_t b[kMaxChunks + 1];
    double r = r_max;
    while (r > 1.0 && !geometric_bounds(K, pb, r, 16, 256, b)) r = std::max(1.0, r * 0.9);
    if (r <= 1.0 && !geometric_bounds(K, pb, 1.0, 16, 256, b)) {
      for (int c = 0; c < pb; ++c) b[c] = (K * c / pb) / 16 * 16;
      b[pb] = K;
    }
    // the start-up (the first chunk's transfer, down the chain for p2p) plus the chunks'
    // GEMMs: more chunks start sooner but run shorter, slower launches (round 2: with the
    // 3xFP16 GEMM the short first chunks cost more than the start-up they save)
    double cost = hops * 4.0 * double(b[1]) * double(N) / bw;
    for (int c = 0; c + 1 < pb; ++c) cost += chunk_gemm_time(rows_max, N, b[c + 1] - b[c], O);
    // the last chunk runs as row chunks (below; ~4 of 0.7-geometric sizes when rows allow)
    const int64_t kl = K - b[pb - 1];
    const int npc = int(std::min<int64_t>(4, std::max<int64_t>(1, rows_max / 256)));
    int64_t rb[kMaxChunks + 1];
    if (!geometric_bounds(rows_max, npc, 0.7, 256, 256, rb))
      for (int i = 0; i <= npc; ++i) rb[i] = rows_max * i / npc;
    for (int q = 0; q < npc; ++q) cost += chunk_gemm_time(rb[q + 1] - rb[q], N, kl, O);
    if (cost < best) {
      best = cost;
      pl.pb = pb;
      for (int c = 0; c <= pb; ++c) pl.kb[c] = b[c];
    }
  }
  const int64_t Kc = K - pl.kb[pl.pb - 1];
  const int pc_env = env_int("GIGA_GATHER_CHUNKS", 0);
  const int pc_cap = int(std::min<int64_t>(pc_env > 0 ? std::min(pc_env, kMaxChunks) : 4,
                                           std::max<int64_t>(1, rows_max / 256)));
  best = 1e300;
  for (int pc = pc_env > 0 ? pc_cap : 1; pc <= pc_cap; ++pc) {
    int64_t b[kMaxChunks + 1];
    if (!geometric_bounds(rows_max, pc, 0.7, 256, 256, b))
      for (int i = 0; i <= pc; ++i) b[i] = rows_max * i / pc;
    double g_end = 0, x_end = 0;  // GEMM stream, gather stream
    for (int q = 0; q < pc; ++q) {
      const double rq = double(b[q + 1] - b[q]);
      g_end += 2.0 * rq * double(N) * double(Kc) / R + O;
      x_end = std::max(g_end, x_end) + 4.0 * rq * double(N) * double(world - 1) / bw;
    }
    if (x_end < best) {
      best = x_end;
      pl.pc = pc;
    }
  }
  return pl;
}

// Row chunks of the last K-chunk's GEMM, gathered one by one: owner o's rows split with
// weights 0.7^q (largest first, rounded to 256-row tiles) so the gather of the last, exposed
// chunk is small (13% of the rows for 4 chunks instead of 25%) while the first gather still
// starts early; shards too small for that split evenly.
void plan_block(int64_t M, int world, int pc, int owner, int q, int64_t *row0, int64_t *rows) {
  int64_t o0, orows;
  partition_rows(M, world, owner, &o0, &orows);
  int64_t b[kMaxChunks + 1];
  if (pc > kMaxChunks || !geometric_bounds(orows, pc, 0.7, 256, 256, b))
    for (int i = 0; i <= pc && i <= kMaxChunks; ++i) b[i] = orows * i / pc;
  *row0 = o0 + b[q];
  *rows = b[q + 1] - b[q];
}

bool force_comm() { return env_int("GIGA_FORCE_COMM", 0) != 0; }

int gemm_chunk(const float *A, const float *Alo, const float *B, const float *Blo, float *C,
               int64_t rows, int64_t N, int64_t Kc, const GemmExtra &ex, cudaStream_t st) {
  return run_gemm(A, Alo, B, Blo, C, rows, N, Kc, N, ex, st);
}

// ---------------------------------------------------------------------------------------
// timelines ($GIGA_TRACE)

Trace::Trace(DevCtx &d, const char *what) : d_(d), what_(what) {
  on_ = env_int("GIGA_TRACE", 0) != 0;
}

int Trace::start(cudaStream_t st) { return on_ ? mark("", st) : GIGA_OK; }

int Trace::mark(const char *series, cudaStream_t st, double bytes) {
  if (!on_) return GIGA_OK;
  bytes_.push_back(bytes);
  if (n_ >= d_.ev_trace.size()) {
    cudaEvent_t e = nullptr;
    CK(cudaEventCreate(&e));
    d_.ev_trace.push_back(e);
  }
  CK(cudaEventRecord(d_.ev_trace[n_], st));
  marks_.push_back({series, n_++});
  return GIGA_OK;
}

// %globaltimer slots: the device's buffer (allocated on first use, zeroed per Trace), handed
// out in order; a trace that runs out of slots reports what it has.
static uint64_t *ns_take(DevCtx &d, size_t &used, size_t n) {
  if (!d.trace_ns) {
    cudaSetDevice(d.dev);
    if (cudaMalloc(&d.trace_ns, kTraceNsSlots * sizeof(uint64_t)) != cudaSuccess) {
      cudaGetLastError();
      d.trace_ns = nullptr;
      return nullptr;
    }
  }
  if (used + n > kTraceNsSlots) return nullptr;
  uint64_t *p = d.trace_ns + used;
  used += n;
  return p;
}

int Trace::stamp(const char *series, cudaStream_t st) {
  if (!on_) return GIGA_OK;
  const size_t at = ns_used_;
  uint64_t *slot = ns_take(d_, ns_used_, 1);
  if (!slot) return GIGA_OK;
  CK(launch_stamp(slot, st));
  ns_.push_back({series, at});
  return GIGA_OK;
}

uint64_t *Trace::cta_slots(const char *series, cudaStream_t st) {
  if (!on_) return nullptr;
  const size_t at = ns_used_;
  uint64_t *p = ns_take(d_, ns_used_, 2 * size_t(kTraceMaxCtas));
  if (!p) return nullptr;
  if (cudaMemsetAsync(p, 0, 2 * size_t(kTraceMaxCtas) * sizeof(uint64_t), st) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  cta_.push_back({series, at});
  return p;
}

void Trace::meta(const char *key, double v) {
  if (!on_) return;
  char buf[96];
  snprintf(buf, sizeof buf, "%s\"%s\": %.17g", meta_.empty() ? "" : ", ", key, v);
  meta_ += buf;
}

int Trace::finish() {
  if (!on_ || marks_.empty()) return GIGA_OK;
  for (auto &m : marks_) CK(cudaEventSynchronize(d_.ev_trace[m.second]));
  std::map<std::string, std::string> series, rates;
  std::map<std::string, float> last;  // previous mark of each series (ms)
  for (size_t i = 1; i < marks_.size(); ++i) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, d_.ev_trace[marks_[0].second], d_.ev_trace[marks_[i].second]));
    std::string &v = series[marks_[i].first];
    char buf[48];
    snprintf(buf, sizeof buf, "%s%.4f", v.empty() ? "" : ", ", ms);
    v += buf;
    if (bytes_[i] > 0) {  // achieved rate of the interval since this series' previous mark
      const float t0 = last.count(marks_[i].first) ? last[marks_[i].first] : 0.0f;
      std::string &r = rates[marks_[i].first];
      snprintf(buf, sizeof buf, "%s%.1f", r.empty() ? "" : ", ",
               ms > t0 ? bytes_[i] / ((ms - t0) * 1e-3) / 1e9 : 0.0);
      r += buf;
    }
    last[marks_[i].first] = ms;
  }
  std::string out = "{\"trace\": \"" + std::string(what_) + "\", \"device\": " +
                    std::to_string(d_.dev) + ", \"meta\": {" + meta_ + "}, \"ms\": {";
  bool first = true;
  for (auto &kv : series) {
    out += (first ? "\"" : ", \"") + kv.first + "\": [" + kv.second + "]";
    first = false;
  }
  out += "}";
  if (!rates.empty()) {
    out += ", \"GBps\": {";
    first = true;
    for (auto &kv : rates) {
      out += (first ? "\"" : ", \"") + kv.first + "\": [" + kv.second + "]";
      first = false;
    }
    out += "}";
  }
  if (!ns_.empty() || !cta_.empty()) {
    // %globaltimer values (ns, the device's clock): stamps and per-launch CTA intervals
    std::vector<uint64_t> h(ns_used_);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h.data(), d_.trace_ns, ns_used_ * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    std::map<std::string, std::string> ns;
    char buf[64];
    for (auto &s : ns_) {
      std::string &v = ns[s.first];
      snprintf(buf, sizeof buf, "%s%llu", v.empty() ? "" : ", ",
               (unsigned long long)h[s.second]);
      v += buf;
    }
    for (auto &c : cta_) {
      uint64_t lo = ~0ull, hi = 0;
      for (int b = 0; b < kTraceMaxCtas; ++b) {
        const uint64_t s0 = h[c.second + 2 * b], s1 = h[c.second + 2 * b + 1];
        if (s0 == 0 || s1 == 0) continue;  // no such CTA in the grid
        lo = std::min(lo, s0);
        hi = std::max(hi, s1);
      }
      std::string &v = ns[c.first];
      snprintf(buf, sizeof buf, "%s[%llu, %llu]", v.empty() ? "" : ", ", (unsigned long long)lo,
               (unsigned long long)hi);
      v += buf;
    }
    out += ", \"ns\": {";
    first = true;
    for (auto &kv : ns) {
      out += (first ? "\"" : ", \"") + kv.first + "\": [" + kv.second + "]";
      first = false;
    }
    out += "}";
  }
  out += "}\n";
  fputs(out.c_str(), stderr);
  return GIGA_OK;
}

}  // namespace giga
