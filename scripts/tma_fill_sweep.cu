// TMA fill-rate sweep (measurement tool, not product code). Every SM streams boxes from an
// L2-resident buffer into a ring of `stages` x `stage_kib` KiB with a consumer warp that only
// waits for each stage to land and releases it. Varied: ring depth, stage size, box shape,
// cluster size and TMA multicast (each CTA of a cluster issues 1/cs of a stage's boxes with
// the whole cluster as destination, so every SM still receives the full stage but the L2
// is read once per cluster). Question answered: is the ~37 B/clk/SM fill ceiling of
// tma_box_bench.cu a per-SM ingress limit (multicast would not raise per-SM ingress) or an
// L2-slice limit (multicast raises it), and is it latency-limited (depth would raise it)?
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_fill_sweep tma_fill_sweep.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ uint32_t su32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// wait modes: 0 try_wait (may suspend the thread), 1 test_wait spin (never suspends),
// 2 try_wait with a 20 ns suspend-time hint
__device__ int g_wait_mode = 0;
__device__ __forceinline__ void wait_parity(uint32_t bar, uint32_t ph) {
  const int mode = g_wait_mode;
  if (mode == 1) {
    asm volatile(
        "{\n.reg .pred p;\nT_%=: mbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra T_%=;\n}" ::"r"(bar),
        "r"(ph)
        : "memory");
  } else if (mode == 2) {
    asm volatile(
        "{\n.reg .pred p;\nH_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 20;\n"
        "@!p bra H_%=;\n}" ::"r"(bar),
        "r"(ph)
        : "memory");
  } else {
    asm volatile(
        "{\n.reg .pred p;\nW_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra W_%=;\n}" ::"r"(bar),
        "r"(ph)
        : "memory");
  }
}
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void csync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}

constexpr int kMaxStages = 24;

__global__ void __launch_bounds__(64, 1)
    fill(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tm1,
         const __grid_constant__ CUtensorMap tm2, const __grid_constant__ CUtensorMap tm3,
         int ndesc, int box_c, int box_r, int box_bytes,
         int ncols, int nrows, int stages, int stage_bytes, int iters, int cs, int mcast) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full[kMaxStages], empty[kMaxStages];
  const uint32_t rank = cs > 1 ? cta_rank() : 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&empty[s])), "r"(cs));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (cs > 1) csync(); else __syncthreads();
  const int boxes = stage_bytes / box_bytes;
  const int tiles_c = ncols / box_c, tiles_r = nrows / box_r;
  const int cluster = blockIdx.x / cs;
  const uint16_t mask = uint16_t((1u << cs) - 1);
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm1)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm2)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tm3)) : "memory");
    const CUtensorMap *tms[4] = {&tm, &tm1, &tm2, &tm3};
    int t = cluster * 37;
    for (int it = 0; it < iters; ++it) {
      const int s = it % stages;
      if (it >= stages) {  // mcast == 2: no consumer, the producer waits for the fill itself
        if (mcast == 2)
          wait_parity(su32(&full[s]), uint32_t((it / stages - 1) & 1));
        else
          wait_parity(su32(&empty[s]), uint32_t((it / stages - 1) & 1));
      }
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])),
                   "r"(stage_bytes) : "memory");
      for (int b = 0; b < boxes; ++b, ++t) {
        const int tc = t % tiles_c, tr = (t / tiles_c) % tiles_r;
        const uint32_t dst = su32(smem + size_t(s) * stage_bytes + size_t(b) * box_bytes);
        const uint64_t tmp = reinterpret_cast<uint64_t>(tms[b % ndesc]);
        if (mcast == 1 && cs > 1) {
          if (b % cs != int(rank)) continue;
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
              ".multicast::cluster [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
              "l"(tmp), "r"(tc * box_c), "r"(tr * box_r),
              "r"(su32(&full[s])), "h"(mask)
              : "memory");
        } else {
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
              " [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
              "l"(tmp), "r"(tc * box_c), "r"(tr * box_r),
              "r"(su32(&full[s]))
              : "memory");
        }
      }
    }
  } else if (threadIdx.x == 32 && mcast != 2) {
    for (int it = 0; it < iters; ++it) {
      const int s = it % stages;
      wait_parity(su32(&full[s]), uint32_t((it / stages) & 1));
      if (cs == 1) {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
        continue;
      }
      for (int q = 0; q < cs; ++q) {  // release stage s in every CTA of the cluster (relaxed:
        uint32_t ra;                   // a release.cluster arrive per stage is ~0.5 us)
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(su32(&empty[s])), "r"(q));
        asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra)
                     : "memory");
      }
    }
  }
  __syncwarp();
  if (cs > 1) csync();  // no CTA exits while a peer may still write into it
}

int main(int argc, char **argv) {
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  const size_t bytes = 48ull << 20;  // L2-resident
  float *buf;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 0, bytes);
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaFuncSetAttribute(fill, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 + 1024);
  cudaFuncSetAttribute(fill, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  struct Box { int c, r; CUtensorMapSwizzle sw; const char *name; };
  const Box boxes[] = {{16, 128, CU_TENSOR_MAP_SWIZZLE_64B, "16x128 sw64 8KiB"},
                       {32, 64, CU_TENSOR_MAP_SWIZZLE_128B, "32x64 sw128 8KiB"},
                       {32, 128, CU_TENSOR_MAP_SWIZZLE_128B, "32x128 sw128 16KiB"},
                       {32, 256, CU_TENSOR_MAP_SWIZZLE_128B, "32x256 sw128 32KiB"},
                       {32, 16, CU_TENSOR_MAP_SWIZZLE_128B, "32x16 sw128 2KiB"},
                       {32, 32, CU_TENSOR_MAP_SWIZZLE_128B, "32x32 sw128 4KiB"}};
  struct Run { int box, stages, stage_kib, cs, mcast, ndesc = 1; };
  const Run runs[] = {
      // no consumer (the producer waits for its own fills), as tma_box_bench.cu
      {0, 6, 32, 1, 2, 1}, {4, 6, 32, 1, 2, 1}, {3, 6, 32, 1, 2, 1}, {4, 6, 32, 1, 2, 4},
      // the same boxes rotated over 2 / 4 identical descriptors
      {4, 6, 32, 1, 0, 2}, {4, 6, 32, 1, 0, 4}, {5, 6, 32, 1, 0, 4}, {1, 6, 32, 1, 0, 4},
      {0, 6, 32, 1, 0, 4},
      // box count per 32 KiB stage: 16 x 2 KiB, 8 x 4 KiB, 4 x 8 KiB, 2 x 16 KiB, 1 x 32 KiB
      {4, 6, 32, 1, 0}, {5, 6, 32, 1, 0}, {1, 6, 32, 1, 0}, {2, 6, 32, 1, 0}, {3, 6, 32, 1, 0},
      // depth / stage-size sweep, no cluster
      {0, 2, 32, 1, 0}, {0, 4, 32, 1, 0}, {0, 6, 32, 1, 0}, {0, 12, 16, 1, 0}, {0, 24, 8, 1, 0},
      {1, 6, 32, 1, 0}, {2, 6, 32, 1, 0}, {3, 6, 32, 1, 0}, {2, 12, 16, 1, 0}, {3, 3, 64, 1, 0},
      // clusters without multicast (placement effect only)
      {0, 6, 32, 2, 0}, {0, 6, 32, 4, 0},
      // multicast: L2 read once per cluster
      {0, 6, 32, 2, 1}, {0, 6, 32, 4, 1}, {0, 6, 32, 8, 1}, {1, 6, 32, 2, 1}, {1, 6, 32, 4, 1},
      {2, 6, 32, 2, 1}, {2, 6, 32, 4, 1},
  };
  const int iters = argc > 1 ? atoi(argv[1]) : 12000;
  const int mode0 = argc > 3 ? atoi(argv[3]) : 0, mode1 = argc > 4 ? atoi(argv[4]) : 2;
  for (int mode = mode0; mode <= mode1; ++mode)
    for (const Run &r : runs) {
      cudaMemcpyToSymbol(g_wait_mode, &mode, sizeof mode);
      const Box &b = boxes[r.box];
      const int box_bytes = b.c * b.r * 4;
      const int ncols = argc > 2 ? atoi(argv[2]) : 4096;
      const int nrows = int(bytes / 4 / ncols);
      CUtensorMap tm;
      const cuuint64_t dims[2] = {cuuint64_t(ncols), cuuint64_t(nrows)};
      const cuuint64_t strides[1] = {cuuint64_t(ncols) * 4};
      const cuuint32_t box[2] = {cuuint32_t(b.c), cuuint32_t(b.r)};
      const cuuint32_t es[2] = {1, 1};
      if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, buf, dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, b.sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        printf("{\"err\": \"encode %s\"}\n", b.name);
        continue;
      }
      const int stage_bytes = r.stage_kib * 1024;
      const size_t smem = size_t(r.stages) * stage_bytes + 1024;
      // as many clusters as fit (occupancy query), one CTA per SM
      cudaLaunchConfig_t lc = {};
      lc.blockDim = dim3(64);
      lc.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = unsigned(r.cs);
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      lc.gridDim = dim3(unsigned(r.cs * 64));
      CUtensorMap tm1 = tm, tm2 = tm, tm3 = tm;
      int nclu = 0;
      cudaOccupancyMaxActiveClusters(&nclu, fill, &lc);
      if (nclu < 1) nclu = sms / r.cs;
      lc.gridDim = dim3(unsigned(r.cs * nclu));
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaLaunchKernelEx(&lc, fill, tm, tm1, tm2, tm3, r.ndesc, b.c, b.r, box_bytes, ncols, nrows, r.stages, stage_bytes,
                         200, r.cs, r.mcast);
      cudaEventRecord(e0);
      cudaLaunchKernelEx(&lc, fill, tm, tm1, tm2, tm3, r.ndesc, b.c, b.r, box_bytes, ncols, nrows, r.stages, stage_bytes,
                         iters, r.cs, r.mcast);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const int ctas = r.cs * nclu;
      const double ingress = double(ctas) * iters * stage_bytes;  // bytes landed in smem
      const double l2 = r.mcast == 1 ? ingress / r.cs : ingress;        // bytes read from L2
      printf("{\"ndesc\": %d, \"wait_mode\": %d, \"box\": \"%s\", \"stages\": %d, \"stage_kib\": %d, \"cluster\": %d, "
             "\"multicast\": %d, \"ctas\": %d, \"ingress_GBps\": %.1f, \"l2_read_GBps\": %.1f, "
             "\"ingress_B_per_clk_per_SM_at_max\": %.2f, \"err\": \"%s\"}\n",
             r.ndesc, mode, b.name, r.stages, r.stage_kib, r.cs, r.mcast, ctas, ingress / ms / 1e6,
             l2 / ms / 1e6, ingress / (ms * 1e-3) / ctas / (clk * 1e3),
             cudaGetErrorString(cudaGetLastError()));
      fflush(stdout);
    }
  return 0;
}
