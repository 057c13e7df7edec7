// host_plan.cpp -- choosing the schedule of the host-buffer matmul on one GPU.
//
// giga_matmul with host A, B, C (the paper's call: matrices built on the
// host, results copied back) is bound by PCIe as much as by the tensor cores: at 32768^3 the
// 12 GiB of copies take ~230 ms at ~50 GB/s per direction against a ~265 ms GEMM; at 16384^3
// the 3 GiB take ~58 ms against 33 ms. Three engines run concurrently -- host->device copies
// (comm stream), the GEMM (compute stream), device->host copies (d2h stream) -- and the order
// of the pieces decides how much of each hides behind the others:
//   phase 1: the first Me rows. K-chunk c brings A[0:Me, kb[c]:kb[c+1]] (a 2-D copy) and
//            B[kb[c]:kb[c+1], :]; its GEMM accumulates into C[0:Me] (C += A_c B_c). Compute
//            starts after the first (small) chunk instead of after all of B; growing chunks
//            keep the copy engine ahead when the GEMM is faster than the copies.
//   phase 2: the remaining rows in blocks over the full K (B is complete): block q's A rows
//            arrive while q-1 computes, and each block's C rows go back while the next block
//            computes; the early rows' C goes back once phase 1 ends. Shrinking blocks make
//            the last, exposed copy-back short.
// host_plan_model() is a three-queue model of that schedule; host_plan_choose() evaluates a
// few thousand (Me, K-chunking, row-blocking) candidates with it (microseconds of CPU).
#include "host_plan.h"

#include <math.h>

#include "kernels.h"
#include <stdlib.h>

#include <algorithm>

namespace giga {

namespace {

// One launch: waves of 256 x 256 tiles, each wave ~2 us of pipeline fill / epilogue beyond its
// MMAs (measured: a 576-deep 20480 x 32768 chunk runs at 241 TF/s against 248 for 32768^3),
// accumulate-mode launches (TMA reduce-add of C) ~10% slower (measured in the e2e timeline),
// at the rate of the scheme the launch runs (chosen on scheme_rows rows, the rows sharing B's
// preparation), plus the operand preparation of the TF32 + BF16 / 3xFP16 schemes (~12 B per
// element of A, and of B unless b_prepared).
double gemm_time(int64_t m, int64_t n, int64_t k, const HostRates &r, bool accumulate,
                 int64_t scheme_rows, bool b_prepared) {
  if (m <= 0 || n <= 0 || k <= 0) return 0.0;
  const int terms = product_terms(nullptr, std::max(m, scheme_rows), n, k);
  // 3xFP16's short-K launches run below its full rate (shorter tiles, per-tile epilogue and
  // preparation weigh more): measured on 8192 / 16384 x 32768 chunks ~310-340 TFLOP/s at
  // K = 512, ~370-380 at K = 1024, ~400-440 at K = 2048 (profiles/r02_chunk_rate_sweep_b.jsonl)
  const double rate = terms == 4 ? r.gemm4 * double(k) / double(k + 256)
                      : terms == 2 ? r.gemm2
                                   : r.gemm;
  const int64_t tiles = ((m + 255) / 256) * ((n + 255) / 256);
  const int64_t waves = (tiles + r.clusters - 1) / r.clusters;
  const double t_wave = 2e-6 + 2.0 * 256.0 * 256.0 * double(k) / (rate / r.clusters);
  const double prep = (terms == 4 || terms == 2)
                          ? 12.0 * (double(m) * double(k) + (b_prepared ? 0.0 : double(k) * double(n))) /
                                r.prep
                          : 0.0;
  return 10e-6 + prep + double(waves) * t_wave * (accumulate ? 1.1 : 1.0);  // + launch
}

// bounds[0..n]: start .. start + total split into n pieces with weights ratio^i, interior
// bounds rounded down to `align`. False if a piece would be empty.
bool geometric(int64_t start, int64_t total, int n, double ratio, int64_t align,
               int64_t *bounds) {
  double sum = 0, w = 1;
  for (int i = 0; i < n; ++i, w *= ratio) sum += w;
  double cum = 0;
  w = 1;
  bounds[0] = start;
  for (int i = 1; i < n; ++i, w *= ratio) {
    cum += w;
    bounds[i] = start + int64_t(double(total) * cum / sum) / align * align;
    if (bounds[i] <= bounds[i - 1]) return false;
  }
  bounds[n] = start + total;
  return n == 1 || bounds[n] > bounds[n - 1];
}

double env_double(const char *name, double dflt) {
  const char *e = getenv(name);
  if (!e || !*e) return dflt;
  const double v = atof(e);
  return v > 0 ? v : dflt;
}

}  // namespace

HostRates host_rates_default() {
  HostRates r;
  r.h2d = env_double("GIGA_HOST_H2D_GBS", r.h2d / 1e9) * 1e9;
  r.d2h = env_double("GIGA_HOST_D2H_GBS", r.d2h / 1e9) * 1e9;
  r.gemm = env_double("GIGA_HOST_GEMM_TFLOPS", r.gemm / 1e12) * 1e12;
  r.gemm4 = env_double("GIGA_HOST_GEMM4_TFLOPS", r.gemm4 / 1e12) * 1e12;
  return r;
}

double host_plan_model(const HostPlan &p, int64_t /*M: rows are in p.rb*/, int64_t N, int64_t K,
                       const HostRates &r) {
  double th = 0, tc = 0, td = 0;
  double arrive_k[kHostMaxChunks], arrive_r[kHostMaxChunks];
  for (int c = 0; c < p.P; ++c) {
    const int64_t Kc = p.kb[c + 1] - p.kb[c];
    th += 4.0 * double(p.Me * Kc + Kc * N) / r.h2d;
    arrive_k[c] = th;
  }
  for (int q = 0; q < p.Q; ++q) {
    th += 4.0 * double((p.rb[q + 1] - p.rb[q]) * K) / r.h2d;
    arrive_r[q] = th;
  }
  if (p.Me > 0) {
    for (int c = 0; c < p.P; ++c)
      tc = std::max(tc, arrive_k[c]) +
           gemm_time(p.Me, N, p.kb[c + 1] - p.kb[c], r, c > 0, 0, false);
    td = tc + 4.0 * double(p.Me * N) / r.d2h;
  }
  const double b_all = arrive_k[p.P - 1];
  const int64_t late = p.Q > 0 ? p.rb[p.Q] - p.rb[0] : 0;
  for (int q = 0; q < p.Q; ++q) {
    const int64_t rows = p.rb[q + 1] - p.rb[q];
    if (rows <= 0) continue;
    // the late row blocks share B's preparation (GemmExtra::b_prep_reuse, rows_hint)
    tc = std::max({tc, arrive_r[q], b_all}) + gemm_time(rows, N, K, r, false, late, q > 0);
    td = std::max(td, tc) + 4.0 * double(rows * N) / r.d2h;
  }
  return std::max(tc, td);
}

HostPlan host_plan_choose(int64_t M, int64_t N, int64_t K, const HostRates &r) {
  static const int kP[] = {1, 2, 3, 4, 6, 8, 10, 12, 14, 16};
  static const double kRatioK[] = {1.0, 1.15, 1.3, 1.5, 2.0};
  static const int kQ[] = {1, 2, 4, 6, 8, 12, 16};
  static const double kRatioQ[] = {1.0, 0.85, 0.7};
  HostPlan best;
  best.t_model = INFINITY;
  for (int f = 0; f <= 8; ++f) {
    const int64_t Me = std::min<int64_t>(M, (M * f / 8 + 255) / 256 * 256);
    if (f > 0 && Me == 0) continue;
    for (int P : kP) {
      if (Me == 0 && P > 1) break;  // no phase 1: B in one piece
      if (P > 1 && K / P < 256) break;
      for (double rk : kRatioK) {
        if (P == 1 && rk != 1.0) break;
        HostPlan p;
        p.Me = Me;
        p.P = P;
        if (!geometric(0, K, P, rk, 16, p.kb)) continue;
        const int64_t late = M - Me;
        for (int Q : kQ) {
          if (late == 0 && Q > 1) break;
          if (Q > 1 && late / Q < 256) break;
          for (double rq : kRatioQ) {
            if (Q == 1 && rq != 1.0) break;
            p.Q = late == 0 ? 0 : Q;
            if (p.Q > 0 && !geometric(Me, late, Q, rq, 256, p.rb)) continue;
            if (p.Q == 0) p.rb[0] = M;
            p.t_model = host_plan_model(p, M, N, K, r);
            if (p.t_model < best.t_model) best = p;
          }
        }
      }
    }
  }
  return best;
}

}  // namespace giga
