// Does TMA multicast raise the per-SM fill rate above the ~10.7 TB/s chip-wide ceiling that
// tma_box_bench.cu measures (measurement tool, not product code)? Every CTA streams 8 KiB
// boxes from an L2-resident buffer into a 6-stage ring of 32 KiB stages, in two halves of 3
// stages: wait for my half-h fills, cluster barrier (every CTA of the cluster has its half-h
// data, so the half can be refilled by anyone), re-arm and issue half h again. With
// multicast each CTA of a cluster issues 1/cs of the boxes to the whole cluster: every SM
// still receives 32 KiB per stage, the L2 is read once per cluster. Without multicast every
// CTA issues all of its boxes (same barriers), so the two differ only in L2 reads.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_mcast_bench tma_mcast_bench.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t su32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

constexpr int kStages = 6, kHalf = 3, kStageBytes = 32768, kBoxBytes = 8192, kBoxes = 4;

__global__ void __launch_bounds__(32, 1) mc_stream(const __grid_constant__ CUtensorMap tm,
                                                   int box_c, int box_r, int ncols, int nrows,
                                                   int rounds, int cs, int mcast) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[kStages];
  uint32_t rank = 0;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm)) : "memory");
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
  const int tiles_c = ncols / box_c, tiles_r = nrows / box_r;
  const uint16_t mask = uint16_t((1u << cs) - 1);
  int t = int(blockIdx.x / cs) * 37;
  uint32_t phase[kStages] = {0, 0, 0, 0, 0, 0};
  for (int r = 0; r < rounds; ++r) {
    const int h = r & 1;
    if (r >= 2) {
      if (threadIdx.x == 0)
        for (int i = 0; i < kHalf; ++i) {
          const int s = h * kHalf + i;
          asm volatile(
              "{\n.reg .pred p;\nW_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
              "@!p bra W_%=;\n}" ::"r"(su32(&full[s])),
              "r"(phase[s])
              : "memory");
          phase[s] ^= 1;
        }
      __syncwarp();
      if (cs > 1)  // every CTA of the cluster holds its half-h data: the half may be refilled
        asm volatile(
            "barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
            ::: "memory");
    }
    if (threadIdx.x == 0)
      for (int i = 0; i < kHalf; ++i) {
        const int s = h * kHalf + i;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                         su32(&full[s])),
                     "r"(kStageBytes)
                     : "memory");
        for (int b = 0; b < kBoxes; ++b, ++t) {
          const int tc = t % tiles_c, tr = (t / tiles_c) % tiles_r;
          const uint32_t dst = su32(smem + s * kStageBytes + b * kBoxBytes);
          if (mcast) {
            if (b % cs != int(rank)) continue;
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
                ".multicast::cluster [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
                "l"(reinterpret_cast<uint64_t>(&tm)), "r"(tc * box_c), "r"(tr * box_r),
                "r"(su32(&full[s])), "h"(mask)
                : "memory");
          } else {
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
                "l"(reinterpret_cast<uint64_t>(&tm)), "r"(tc * box_c), "r"(tr * box_r),
                "r"(su32(&full[s]))
                : "memory");
          }
        }
      }
    __syncwarp();
  }
  if (threadIdx.x == 0)
    for (int s = 0; s < kStages; ++s)
      asm volatile(
          "{\n.reg .pred p;\nW2_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
          "@!p bra W2_%=;\n}" ::"r"(su32(&full[s])),
          "r"(phase[s])
          : "memory");
  __syncwarp();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}

int main() {
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  const size_t bytes = 64ull << 20;
  float *buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 0, bytes);
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const size_t smem = kStages * kStageBytes + 1024;
  cudaFuncSetAttribute(mc_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
  cudaFuncSetAttribute(mc_stream, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  const int ncols = 16384, nrows = int(bytes / 4 / ncols);
  CUtensorMap tm;
  const cuuint64_t dims[2] = {cuuint64_t(ncols), cuuint64_t(nrows)};
  const cuuint64_t strides[1] = {cuuint64_t(ncols) * 4};
  const cuuint32_t box[2] = {16, 128};
  const cuuint32_t es[2] = {1, 1};
  enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, buf, dims, strides, box, es,
      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int rounds = 8000;
  struct Run { int cs, mcast; };
  const Run runs[] = {{1, 0}, {2, 0}, {2, 1}, {4, 0}, {4, 1}, {8, 1}};
  for (int rep = 0; rep < 2; ++rep)
    for (const Run &r : runs) {
      cudaLaunchConfig_t lc = {};
      lc.blockDim = dim3(32);
      lc.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = unsigned(r.cs);
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      lc.gridDim = dim3(unsigned(r.cs * 64));
      int nclu = 0;
      cudaOccupancyMaxActiveClusters(&nclu, mc_stream, &lc);
      if (nclu < 1) nclu = sms / r.cs;
      lc.gridDim = dim3(unsigned(r.cs * nclu));
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaLaunchKernelEx(&lc, mc_stream, tm, 16, 128, ncols, nrows, 100, r.cs, r.mcast);
      cudaEventRecord(e0);
      cudaLaunchKernelEx(&lc, mc_stream, tm, 16, 128, ncols, nrows, rounds, r.cs, r.mcast);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const int ctas = r.cs * nclu;
      const double ingress = double(ctas) * rounds * kHalf * kStageBytes;
      const double l2 = r.mcast ? ingress / r.cs : ingress;
      printf("{\"cluster\": %d, \"multicast\": %d, \"ctas\": %d, \"ingress_GBps\": %.1f, "
             "\"l2_read_GBps\": %.1f, \"ingress_B_per_clk_per_SM_at_max\": %.2f, \"err\": \"%s\"}\n",
             r.cs, r.mcast, ctas, ingress / ms / 1e6, l2 / ms / 1e6,
             ingress / (ms * 1e-3) / ctas / (clk * 1e3), cudaGetErrorString(cudaGetLastError()));
      fflush(stdout);
    }
  return 0;
}
