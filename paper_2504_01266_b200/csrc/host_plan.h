// host_plan.h -- schedule of giga_matmul's host-buffer path on one GPU (three engines:
// host->device copies, the GEMM, device->host copies). See host_plan.cpp.
#pragma once
#include <stdint.h>

namespace giga {

constexpr int kHostMaxChunks = 16;

struct HostPlan {
  int64_t Me = 0;                     // early rows (phase 1: K-chunked, accumulating in C)
  int P = 1;                          // K-chunks of phase 1
  int64_t kb[kHostMaxChunks + 1]{};   // K-chunk bounds, kb[0] = 0, kb[P] = K, multiples of 16
  int Q = 1;                          // row blocks of phase 2 (rows Me..M, full K)
  int64_t rb[kHostMaxChunks + 1]{};   // row bounds, rb[0] = Me, rb[Q] = M
  double t_model = 0;                 // modelled makespan, seconds
};

struct HostRates {
  double h2d = 50e9;     // bytes/s host -> device (pinned, measured 55.6 alone, 49 in duplex)
  double d2h = 50e9;     // bytes/s device -> host
  // logical fp32-accurate flop/s of the shard GEMM by the scheme a launch runs
  // (giga_product_scheme; measured): 3xTF32, TF32 + BF16, 3xFP16
  double gemm = 250e12, gemm2 = 265e12, gemm4 = 440e12;
  double prep = 5e12;    // bytes/s of the operand preparation (~12 B per element, HBM-bound)
  int clusters = 74;     // concurrent 256 x 256 tiles (CTA pairs on 148 SMs)
};

// Model of one plan (seconds): the copy engines and the GEMM run concurrently, each in order;
// a GEMM waits for its inputs, a copy-back waits for its rows to be final.
double host_plan_model(const HostPlan &p, int64_t M, int64_t N, int64_t K, const HostRates &r);

// The plan with the smallest modelled makespan over a small family (early-row fraction,
// geometric K-chunks, geometric row blocks). Environment overrides of the rates:
// GIGA_HOST_H2D_GBS, GIGA_HOST_D2H_GBS, GIGA_HOST_GEMM_TFLOPS.
HostPlan host_plan_choose(int64_t M, int64_t N, int64_t K, const HostRates &r);
HostRates host_rates_default();

}  // namespace giga
