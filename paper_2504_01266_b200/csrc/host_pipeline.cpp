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
  HostPlan plan = host_plan_choose(M, N, K, rates);
  // $GIGA_HOST_PLAN = "Me,P,Q" (measurements): that plan with equal K-chunks and row blocks
  if (const char *e = getenv("GIGA_HOST_PLAN")) {
    long long me = 0, pp = 1, qq = 1;
    if (sscanf(e, "%lld,%lld,%lld", &me, &pp, &qq) == 3 && me >= 0 && me <= M && pp >= 1 &&
        pp <= kHostMaxChunks && qq >= 1 && qq <= kHostMaxChunks) {
      HostPlan f;
      f.Me = me;
      f.P = me > 0 ? int(pp) : 1;
      for (int c = 0; c <= f.P; ++c) f.kb[c] = c == f.P ? K : (K * c / f.P) / 16 * 16;
      f.Q = me < M ? int(qq) : 0;
      if (f.Q > 0)
        for (int q = 0; q <= f.Q; ++q) f.rb[q] = me + (M - me) * q / f.Q;
      else
        f.rb[0] = M;
      f.t_model = host_plan_model(f, M, N, K, rates);
      plan = f;
    }
  }
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
  Trace tr(d, "host_pipeline");  // $GIGA_TRACE=1: the measured timeline of the plan
  tr.meta("M", double(M));
  tr.meta("N", double(N));
  tr.meta("K", double(K));
  tr.meta("Me", double(Me));
  tr.meta("model_ms", plan.t_model * 1e3);
  TRY(tr.start(d.comm));
  // host -> device: (early A columns, B rows) per K-chunk, then the late A row blocks
  for (int c = 0; c < P; ++c) {
    const int64_t Kc = kb[c + 1] - kb[c];
    if (Me > 0)
      CK(cudaMemcpy2DAsync(Ad + kb[c], size_t(K) * 4, A + kb[c], size_t(K) * 4,
                           size_t(Kc) * 4, size_t(Me), cudaMemcpyHostToDevice, d.comm));
    CK(cudaMemcpyAsync(Bd + kb[c] * N, B + kb[c] * N, size_t(Kc * N) * 4,
                       cudaMemcpyHostToDevice, d.comm));
    CK(cudaEventRecord(d.ev_kchunk[c], d.comm));
    TRY(tr.mark("h2d_k", d.comm));
  }
  for (int q = 0; q < Q; ++q) {
    const int64_t q0 = plan.rb[q], q1 = plan.rb[q + 1];
    if (q1 > q0)
      CK(cudaMemcpyAsync(Ad + q0 * K, A + q0 * K, size_t((q1 - q0) * K) * 4,
                         cudaMemcpyHostToDevice, d.comm));
    CK(cudaEventRecord(d.ev_rchunk[q], d.comm));
    TRY(tr.mark("h2d_r", d.comm));
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
    TRY(tr.mark("gemm1", d.compute));
  }
  if (Me > 0) {
    CK(cudaEventRecord(d.ev_c, d.compute));
    CK(cudaStreamWaitEvent(d.d2h, d.ev_c, 0));
    CK(cudaMemcpyAsync(C, Cd, size_t(Me * N) * 4, cudaMemcpyDeviceToHost, d.d2h));
    TRY(tr.mark("d2h_early", d.d2h));
  }
  // phase 2: late row blocks over the full K (phase 1 waited for every K-chunk of B)
  for (int q = 0; q < Q; ++q) {
    const int64_t q0 = plan.rb[q], q1 = plan.rb[q + 1];
    CK(cudaStreamWaitEvent(d.compute, d.ev_rchunk[q], 0));
    if (q1 > q0) {
      TRY(split(Ad + q0 * K, at(Alo, q0 * K), (q1 - q0) * K, d.compute));
      GemmExtra e2;
      e2.b_prep_reuse = q > 0;  // every late row block multiplies by the same full B
      e2.rows_hint = M - Me;
      TRY(gemm_chunk(Ad + q0 * K, at(Alo, q0 * K), Bd, Blo, Cd + q0 * N, q1 - q0, N, K, e2,
                     d.compute));
    }
    CK(cudaEventRecord(d.ev_done[q], d.compute));
    TRY(tr.mark("gemm2", d.compute));
    CK(cudaStreamWaitEvent(d.d2h, d.ev_done[q], 0));
    if (q1 > q0)
      CK(cudaMemcpyAsync(C + q0 * N, Cd + q0 * N, size_t((q1 - q0) * N) * 4,
                         cudaMemcpyDeviceToHost, d.d2h));
    TRY(tr.mark("d2h", d.d2h));
  }
  CK(cudaStreamSynchronize(d.d2h));
  CK(cudaStreamSynchronize(d.compute));
  CK(cudaStreamSynchronize(d.comm));
  TRY(tr.finish());
  return GIGA_OK;
}

}  // namespace giga
