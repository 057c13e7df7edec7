// runtime.h -- internal interface of libgiga's host runtime, shared by its translation units
// (api.cpp: the C ABI; runtime.cpp: state, workspace, checks, shard compute; pipeline_nccl.cpp:
// the NCCL pipeline; p2p.cpp: the peer-to-peer transport; host_pipeline.cpp: host buffers).
// Not installed: the public interface is include/giga.h.
#pragma once
#include "giga.h"

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <initializer_list>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <functional>
#include <vector>

#include "kernels.h"
#include "nccl_loader.h"

namespace giga {

// ---------------------------------------------------------------------------------------
// errors: every failing call stores a message (giga_last_error) and returns a status
extern thread_local std::string t_err;

#define CK(x)                                                               \
  do {                                                                      \
    cudaError_t e_ = (x);                                                   \
    if (e_ != cudaSuccess) return fail_cuda(e_, #x, __FILE__, __LINE__);    \
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

constexpr size_t kTraceNsSlots = 1 << 15;  // per device: %globaltimer slots of class Trace
constexpr int kTraceMaxCtas = 160;          // >= the SM count: CTA slots per traced launch

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
  std::vector<cudaEvent_t> ev_trace;   // timing events of class Trace ($GIGA_TRACE)
  uint64_t *trace_ns = nullptr;        // Trace's %globaltimer slots (device; kTraceNsSlots)
  Buf A_lo, B_lo, A_pad, B_pad, C_pad, A_h, B_h, C_h;
  Buf vec_ws;  // dot: kDotMaxBlocks fp64 partials, the fp64 result, the ticket (zeroed once)
  double *res_pinned = nullptr;  // dot: pinned host landing slot of the fp64 result
};

// Rank-mode peer-to-peer state: this rank's registered B / C_full, its flag page, and the
// peers' buffers and flag pages mapped through CUDA IPC (index = rank).
// Flag page (device memory, u32 unless noted): ready[c] @0 (upstream has B chunk c),
// pulled[c] @64 (downstream finished reading my chunk c), cdone[q] @128 (rank q wrote its C
// rows into my C_full), dotdone[q] @384, started[q] @640 (rank q began call s: its C_full may
// be written), dot partials (fp64) @1024. Values are call numbers.
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
  bool rank_p2p = false;  // rank mode: $GIGA_TRANSPORT=p2p when giga_rank_init ran (fixed then)
  RankP2P p2p;
};
extern State g;

struct TimeRec {
  int dev;
  int kind;  // 0 gemm, 1 split / operand preparation / exception fixes
  cudaEvent_t a, b;
  int n;     // kernels the bracketed call launched
};
extern std::mutex g_tmu;
extern bool g_timing;
extern std::vector<TimeRec> g_tpending;
extern std::vector<std::pair<int, cudaEvent_t>> g_tpool;
extern double g_tms[2];
extern int64_t g_tcount[2];


cudaEvent_t pool_event(int dev);  // a timing event for `dev` (caller holds g_tmu)

// Launch `fn` on `st`, bracketed by timing events when timing is enabled; `n` = the number of
// kernels fn launches (the launch count bench.py reports).
template <class F>
cudaError_t timed(int kind, cudaStream_t st, F fn, int n = 1) {
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
    g_tpending.push_back({dev, kind, a, b, n});
  else {
    if (a) g_tpool.push_back({dev, a});
    if (b) g_tpool.push_back({dev, b});
  }
  return e;
}

inline bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// The chunk plan (runtime.cpp make_plan / plan_block): B is distributed in pb K-chunks
// [kb[c], kb[c+1]) growing geometrically (multiples of 16, at least 256 deep); the last
// K-chunk's GEMM and the C gather run in pc row chunks per owner, shrinking geometrically.
// The counts (at most 6 / 16 K-chunks with NCCL / p2p, 4 row chunks) trade the exposed first
// transfer and last gather against ~20 us per extra GEMM launch; $GIGA_BCAST_CHUNKS and
// $GIGA_GATHER_CHUNKS force them. Unaligned shapes use one chunk of each.
struct Plan {
  int pb = 1, pc = 1;
  int64_t kb[kMaxChunks + 1] = {0};
};

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

struct DrvApi {
  PFN_cuStreamWaitValue32_v8000 wait = nullptr;
  PFN_cuStreamWriteValue32_v8000 write = nullptr;
  PFN_cuMemGetAddressRange_v3020 range = nullptr;
};

template <class T>
T *at(T *p, int64_t off) {
  return p ? p + off : nullptr;
}

// Timeline of one call on one device ($GIGA_TRACE=1): a timing event after each piece of work
// on each engine, printed as one JSON line on stderr when the call ends ({"trace": what,
// "device": d, "meta": {...}, "ms": {series: [end times since the call's start]}}). Tracing
// synchronises the call's streams before printing; it is off unless the variable is set.
class Trace {
 public:
  Trace(DevCtx &d, const char *what);
  bool on() const { return on_; }
  int start(cudaStream_t st);                  // the zero of the timeline
  // bytes > 0: the bytes the stream moved since its previous mark of this series (or since
  // start); finish() then also reports the achieved GB/s of each such interval
  int mark(const char *series, cudaStream_t st, double bytes = 0);
  // %globaltimer intervals on the device clock (comparable across streams): stamp() writes
  // the time the stream reaches it (a 1-thread kernel) into the series; cta_slots() returns
  // room for one GEMM launch's per-CTA (start, end) pairs (GemmExtra::cta_ns), reported as
  // that launch's [first CTA start, last CTA end]. nullptr when tracing is off or full.
  int stamp(const char *series, cudaStream_t st);
  uint64_t *cta_slots(const char *series, cudaStream_t st);
  void meta(const char *key, double v);
  int finish();                                // waits for the last marks, prints the line

 private:
  DevCtx &d_;
  const char *what_;
  bool on_ = false;
  size_t n_ = 0;
  std::vector<std::pair<std::string, size_t>> marks_;
  std::vector<double> bytes_;
  std::vector<std::pair<std::string, size_t>> ns_;   // (series, first slot), 1 slot each
  std::vector<std::pair<std::string, size_t>> cta_;  // (series, first slot), 2 x kMaxCtas
  size_t ns_used_ = 0;
  std::string meta_;
};

// ---- runtime.cpp ---------------------------------------------------------------------------
int fail(int code, const char *fmt, ...) __attribute__((format(printf, 2, 3)));
int fail_cuda(cudaError_t e, const char *what, const char *file, int line);
// workspace: grow-only per-GPU buffers, reserved transactionally (a failure frees nothing old
// and keeps nothing new)
int ws_reserve(DevCtx &d, std::initializer_list<std::pair<Buf *, size_t>> req);
void ws_free(DevCtx &d);
float *fptr(Buf &b);
int ctx_create(DevCtx &d, int dev);
void ctx_destroy(DevCtx &d);
int check_sm100(int dev);
// 3xTF32 lo operands: in the GEMM's shared memory (default) or pre-split arrays
// ($GIGA_LO_PRESPLIT=1): lo_at / lo_bytes give nullptr / 0 in the default mode
bool lo_presplit();
size_t lo_bytes(int64_t elems);
float *lo_at(Buf &b, int64_t off = 0);
int split(const float *x, float *lo, int64_t n, cudaStream_t st);
int run_gemm(const float *A, const float *Alo, const float *B, const float *Blo, float *C,
             int64_t M, int64_t N, int64_t K, int64_t ldc, const GemmExtra &ex,
             cudaStream_t st);
int gemm(const float *A, const float *Alo, const float *B, const float *Blo, float *C,
         int64_t M, int64_t N, int64_t K, int64_t ldc, cudaStream_t st);
int gemm_chunk(const float *A, const float *Alo, const float *B, const float *Blo, float *C,
               int64_t rows, int64_t N, int64_t Kc, const GemmExtra &ex, cudaStream_t st);
int shard_compute(DevCtx &d, cudaStream_t st, const float *A, int64_t rows, const float *B,
                  float *C, int64_t ldc, int64_t N, int64_t K, cudaEvent_t wait_b);
void partition_rows(int64_t M, int ngpus, int gi, int64_t *row0, int64_t *rows);
bool overlaps(const void *a, size_t abytes, const void *b, size_t bbytes);
int check_dims(int64_t M, int64_t N, int64_t K);
int pointer_kind(const void *p, int *dev);  // 1 = device (*dev set), 0 = host
int quiesce(int ngpus);
int sync_all(int ngpus);
int vec_ws(DevCtx &d);
double *vec_partials(DevCtx &d);
double *vec_out(DevCtx &d);
unsigned *vec_ticket(DevCtx &d);
int dot_partial(DevCtx &d, const float *x, const float *y, int64_t n, cudaStream_t st);
int read_result(DevCtx &d, cudaStream_t st, double *out);  // after dot_partial (+ reduction)
int env_int(const char *name, int dflt);
bool force_comm();
Plan make_plan(int64_t M, int64_t N, int64_t K, int world, bool aligned);
void plan_block(int64_t M, int world, int pc, int owner, int q, int64_t *row0, int64_t *rows);

// ---- pipeline_nccl.cpp ---------------------------------------------------------------------
int nccl_check(ncclResult_t r, const char *what);
ncclConfig_t comm_config();
int get_comms(int ngpus, std::vector<ncclComm_t> **out);
int gather_rows(const NcclApi *api, ncclComm_t comm, cudaStream_t st, float *C_full, int64_t M,
                int64_t N, int world, int rank);
int run_pipeline(std::vector<Part> &parts, int world, int64_t M, int64_t N, int64_t K);
int rank_gemms(const Plan &plan, const GemmExtra &ex, int64_t M, int64_t N, int64_t K, int world,
               int rank, const float *A, const float *Alo, const float *B, const float *Blo,
               float *C_full, cudaStream_t st, const std::function<int(int)> &before_chunk,
               const std::function<int(int)> &after);
int pipeline_max_ctas(int dev);

// ---- p2p.cpp -------------------------------------------------------------------------------
bool transport_p2p();
int run_p2p(std::vector<Part> &parts, int64_t M, int64_t N, int64_t K, bool gather = true);
const DrvApi *drv_api();
uint32_t *flag_ready(uint32_t *page, int c);
uint32_t *flag_pulled(uint32_t *page, int c);
uint32_t *flag_cdone(uint32_t *page, int q);
uint32_t *flag_dotdone(uint32_t *page, int q);
uint32_t *flag_started(uint32_t *page, int q);
double *dot_part(uint32_t *page, int q, uint32_t s);
int wait_flag(cudaStream_t st, uint32_t *addr, uint32_t v);
int write_flag(cudaStream_t st, uint32_t *addr, uint32_t v);
int run_p2p_rank(DevCtx &d, cudaStream_t st, const float *A, float *B, float *C, int64_t M,
                 int64_t N, int64_t K);
int p2p_dot_allreduce(DevCtx &d, cudaStream_t st, double *result);
void p2p_release();

// ---- mcast.cpp: NVLink multicast teams (fused gather with one store per piece) -------------
float *mc_address(const std::vector<Part> &parts, int64_t M, int64_t N);
float *rank_mc_address(const float *C_full, int64_t M, int64_t N);
bool rank_mc_buffer(const float *p);
void mc_release_all();

// ---- host_pipeline.cpp ---------------------------------------------------------------------
int host_pipeline(DevCtx &d, const float *A, const float *B, float *C, int64_t M, int64_t N,
                  int64_t K);

}  // namespace giga
