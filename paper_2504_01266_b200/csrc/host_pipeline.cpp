// host_pipeline.cpp -- giga_matmul on host buffers, one GPU: copies in, GEMMs and copies out
// overlapped on three streams, in the schedule host_plan.cpp chooses.
#include "runtime.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include "host_plan.h"

namespace giga {

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

}  // namespace giga
