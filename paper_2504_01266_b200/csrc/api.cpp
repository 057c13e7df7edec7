// api.cpp -- the C ABI declared in include/giga.h: initialisation and teardown, argument
// checking, and the dispatch of one row-split matrix multiply to the
// device-resident, NCCL-pipeline, peer-to-peer or host-buffer paths.
#include "runtime.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include "host_plan.h"

namespace giga {
namespace {

// Failure detection for the rank API (stream-ordered calls never wait for NCCL): a
// communicator that has already failed asynchronously (a peer died, a network error) makes
// the next call fail fast with GIGA_ERR_COMM instead of queueing work behind it.
int rank_comm_healthy() {
  if (!g.rank_comm) return GIGA_OK;
  const NcclApi *api = nccl_api(nullptr);
  ncclResult_t ar = ncclSuccess;
  if (api && api->CommGetAsyncError(g.rank_comm, &ar) == ncclSuccess && ar != ncclSuccess &&
      ar != ncclInProgress)
    return nccl_check(ar, "NCCL communicator (asynchronous error from an earlier call)");
  return GIGA_OK;
}

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
  if (!device && ngpus == 1 && K % 4 == 0 && N % 4 == 0)
    return host_pipeline(g.devs[0], A, B, C, M, N, K);

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
  mc_release_all();
  release_gemm_caches();
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
  g.rank_p2p = false;
  g.rank = 0;
  g.world = 1;
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
  g.rank_p2p = transport_p2p() && world > 1;
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
  TRY(rank_comm_healthy());
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : d.compute;
  // calls share the rank's workspace: a call starts after the previous one, whatever the
  // caller's streams. Inside a CUDA-graph capture an event recorded outside it cannot be
  // waited on: the graph's stream orders its replays, and the caller orders the graph
  // against eager calls.
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  CK(cudaStreamIsCapturing(st, &cs));
  const bool capturing = cs != cudaStreamCaptureStatusNone;
  // the transport was fixed at giga_rank_init; a world > 1 without a communicator or a p2p
  // registration would silently compute only this rank's rows
  if (g.world > 1 && !g.rank_comm && !(g.rank_p2p && g.p2p.ready))
    return g.rank_p2p ? fail(GIGA_ERR_NOT_INITIALIZED,
                             "giga_matmul_rank: p2p transport needs giga_rank_p2p_export/import")
                      : fail(GIGA_ERR_NOT_INITIALIZED,
                             "giga_matmul_rank: no communicator for world %d", g.world);
  if (capturing) {
    // the p2p flag protocol bakes the call number into the captured waits and writes, so
    // replays would not order themselves across processes
    if (g.rank_p2p)
      return fail(GIGA_ERR_UNSUPPORTED,
                  "giga_matmul_rank: CUDA-graph capture is not supported with the p2p transport");
    keep_superseded_buffers();  // the graph keeps workspace pointers: never free them early
  }
  if (d.has_last && !capturing) CK(cudaStreamWaitEvent(st, d.ev_last, 0));
  int rc;
  if (g.rank_p2p) {
    rc = run_p2p_rank(d, st, A_shard, B, C_full, M, N, K);
  } else if (!g.rank_comm) {
    rc = shard_compute(d, st, A_shard, rows, B, C_full + r0 * N, N, N, K, nullptr);
  } else {
    std::vector<Part> parts{{&d, g.rank_comm, g.rank, A_shard, B, C_full, st}};
    rc = run_pipeline(parts, g.world, M, N, K);
  }
  TRY(rc);
  if (!capturing) {
    CK(cudaEventRecord(d.ev_last, st));
    d.has_last = true;
  }
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
    TRY(read_result(d, d.compute, &part));
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
  TRY(rank_comm_healthy());
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : d.compute;
  if (g.world > 1 && !g.rank_comm && !(g.rank_p2p && g.p2p.ready))
    return fail(GIGA_ERR_NOT_INITIALIZED, "giga_dot_rank: no communicator / p2p registration "
                "for world %d", g.world);
  TRY(dot_partial(d, x_shard, y_shard, rows, st));
  if (g.rank_p2p) return p2p_dot_allreduce(d, st, result);
  if (g.rank_comm) {  // every rank gets the sum of the partials
    const NcclApi *api = nccl_api(nullptr);
    TRY(nccl_check(api->AllReduce(vec_out(d), vec_out(d), 1, ncclFloat64, ncclSum, g.rank_comm,
                                  st),
                   "ncclAllReduce(dot)"));
  }
  return read_result(d, st, result);
}

// ---- rank-mode peer-to-peer registration (CUDA IPC) ---------------------------------------

namespace {
struct P2PBlob {
  cudaIpcMemHandle_t hB, hC, hF;
  uint64_t offB, offC;
  uint32_t mc;  // 1: C_full is this rank's multicast team buffer (no IPC handle: the epilogue
                // reaches every peer's copy through the team address)
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
  b.mc = rank_mc_buffer(C_full) ? 1u : 0u;
  if (!b.mc) TRY(ipc_handle(C_full, &b.hC, &b.offC));
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
  // every rank's C_full is a multicast team buffer, or none is
  P2PBlob mine;
  memcpy(&mine, blobs + size_t(g.rank) * GIGA_P2P_BLOB_BYTES, sizeof mine);
  for (int q = 0; q < world; ++q) {
    P2PBlob b;
    memcpy(&b, blobs + size_t(q) * GIGA_P2P_BLOB_BYTES, sizeof b);
    if (b.mc != mine.mc)
      return fail(GIGA_ERR_INVALID_ARG,
                  "giga_rank_p2p_import: rank %d's C_full is %sa multicast team buffer, rank "
                  "%d's is %s",
                  q, b.mc ? "" : "not ", g.rank, mine.mc ? "" : "not");
  }
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
    if (!b.mc) {
      CK(cudaIpcOpenMemHandle(&pc, b.hC, cudaIpcMemLazyEnablePeerAccess));
      x.opened.push_back(pc);
    }
    CK(cudaIpcOpenMemHandle(&pf, b.hF, cudaIpcMemLazyEnablePeerAccess));
    x.opened.push_back(pf);
    x.peerB[q] = reinterpret_cast<float *>(static_cast<char *>(pb) + b.offB);
    x.peerC[q] = pc ? reinterpret_cast<float *>(static_cast<char *>(pc) + b.offC) : nullptr;
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
  const Plan pl = make_plan(M, N, K, world, (K % 4 == 0) && (N % 4 == 0));
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
  if (!A || !B || !C || (!A_lo) != (!B_lo) || terms < 1 || terms > 4 ||
      ((terms == 2 || terms == 4) && A_lo))
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

int giga_gemm_gather_ex(const float *A, const float *B, float *C, float *const *peer_c,
                        int n_peer, int64_t M, int64_t N, int64_t K, int64_t ldc, int terms,
                        int store_mode, void *stream) {
  if (!A || !B || !C || n_peer < 0 || n_peer > kMaxCDst - 1 || (n_peer && !peer_c) ||
      terms < 0 || terms > 4 || store_mode < 0 || store_mode > 2 ||
      (store_mode == 2 && n_peer))
    return fail(GIGA_ERR_INVALID_ARG, "giga_gemm_gather_ex: bad arguments");
  TRY(check_dims(M, N, K));
  if ((K & 3) || (N & 3) || (ldc & 3) || ldc < N || !aligned16(A) || !aligned16(B) ||
      !aligned16(C))
    return fail(GIGA_ERR_INVALID_ARG,
                "giga_gemm_gather_ex: needs K%%4 == N%%4 == ldc%%4 == 0, ldc >= N, 16B-aligned");
  for (int i = 0; i < n_peer; ++i)
    if (!peer_c[i] || !aligned16(peer_c[i]))
      return fail(GIGA_ERR_INVALID_ARG, "giga_gemm_gather_ex: peer %d NULL / misaligned", i);
  if (lo_presplit())
    return fail(GIGA_ERR_UNSUPPORTED, "giga_gemm_gather_ex: not with GIGA_LO_PRESPLIT=1");
  if (ensure_tma_encoder() != 0) return fail(GIGA_ERR_CUDA, "TMA encoder unavailable");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  GemmExtra ex;
  ex.lda = K;
  ex.ldb = N;
  float *peers[kMaxCDst];
  for (int i = 0; i < n_peer; ++i) peers[i] = peer_c[i];
  ex.peer_c = peers;
  ex.n_peer_c = n_peer;
  ex.vec_store = store_mode == 1 ? 1 : 0;
  ex.mc_c = store_mode == 2 ? C : nullptr;
  if (terms == 0) return run_gemm(A, nullptr, B, nullptr, C, M, N, K, ldc, ex, st);
  CK(timed(0, st, [&] {
    return launch_gemm_3xtf32(A, nullptr, B, nullptr, C, M, N, K, ldc, terms, -1, st, 0, &ex);
  }));
  return GIGA_OK;
}

int giga_rank_compute_only(const float *A_shard, const float *B, float *C_full, int64_t M,
                           int64_t N, int64_t K, int world, int rank, void *stream) {
  if (!A_shard || !B || !C_full)
    return fail(GIGA_ERR_INVALID_ARG, "giga_rank_compute_only: NULL pointer");
  TRY(check_dims(M, N, K));
  if (world < 1 || world > 4096 || rank < 0 || rank >= world)
    return fail(GIGA_ERR_INVALID_ARG, "giga_rank_compute_only: rank %d of world %d", rank, world);
  if ((K & 3) || (N & 3) || !aligned16(A_shard) || !aligned16(B) || !aligned16(C_full))
    return fail(GIGA_ERR_INVALID_ARG,
                "giga_rank_compute_only: needs K %% 4 == N %% 4 == 0 and 16-byte aligned pointers");
  if (lo_presplit())
    return fail(GIGA_ERR_UNSUPPORTED, "giga_rank_compute_only: not with GIGA_LO_PRESPLIT=1");
  if (ensure_tma_encoder() != 0) return fail(GIGA_ERR_CUDA, "TMA encoder unavailable");
  int dev = 0;
  CK(cudaGetDevice(&dev));
  const Plan plan = make_plan(M, N, K, world, true);
  GemmExtra ex;
  ex.lda = K;
  ex.ldb = N;
  ex.max_ctas = world > 1 ? pipeline_max_ctas(dev) : 0;
  auto none = [](int) { return int(GIGA_OK); };
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (world == 1)  // the single-GPU path: one whole GEMM on all SMs
    return run_gemm(A_shard, nullptr, B, nullptr, C_full, M, N, K, N, GemmExtra(), st);
  if (transport_p2p()) {
    // the p2p transport's GEMMs (run_p2p_rank): all SMs (copy engines move B), one launch per
    // K-chunk accumulating into the rank's rows, the last one reading the partial back
    // (load-C; its stores into the peers' C_full are left out like every transfer here)
    int64_t r0, rows;
    partition_rows(M, world, rank, &r0, &rows);
    if (rows == 0) return GIGA_OK;
    ex.max_ctas = 0;
    for (int c = 0; c < plan.pb; ++c) {
      GemmExtra e = ex;
      const bool last = c == plan.pb - 1;
      e.accumulate = (c > 0 && !last) ? 1 : 0;
      e.load_c = (c > 0 && last) ? 1 : 0;
      e.rows_hint = rows;
      const int64_t Kc = plan.kb[c + 1] - plan.kb[c];
      TRY(gemm_chunk(A_shard + plan.kb[c], nullptr, B + plan.kb[c] * N, nullptr, C_full + r0 * N,
                     rows, N, Kc, e, st));
    }
    return GIGA_OK;
  }
  return rank_gemms(plan, ex, M, N, K, world, rank, A_shard, nullptr, B, nullptr, C_full, st,
                    none, none);
}

int giga_product_scheme(int64_t M, int64_t N, int64_t K, int *terms) {
  if (!terms) return fail(GIGA_ERR_INVALID_ARG, "giga_product_scheme: NULL terms");
  TRY(check_dims(M, N, K));
  *terms = product_terms(lo_presplit() ? reinterpret_cast<const float *>(1) : nullptr, M, N, K);
  return GIGA_OK;
}

int giga_gemm_schedule(int64_t M, int64_t N, int64_t K, int num_sms, int64_t *out) {
  if (!out) return fail(GIGA_ERR_INVALID_ARG, "giga_gemm_schedule: NULL out");
  TRY(check_dims(M, N, K));
  if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX)
    return fail(GIGA_ERR_INVALID_ARG, "giga_gemm_schedule: dimension above 2^31 - 1");
  const int terms =
      product_terms(lo_presplit() ? reinterpret_cast<const float *>(1) : nullptr, M, N, K);
  const GemmSchedule s = gemm_schedule(M, N, K, num_sms > 0 ? num_sms : 148, 0, true,
                                       default_promote_kblocks(terms), terms == 4 ? 32 : 16);
  const int64_t v[8] = {s.cg,          s.num_tiles, s.nclu,      s.n_kb,
                        s.first_split, s.s,         s.num_units, s.mode};
  for (int i = 0; i < 8; ++i) out[i] = v[i];
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
      g_tcount[r.kind] += r.n;
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
