// TMA fill rate per box shape (measurement tool, not product code): every SM streams 8 KiB
// boxes from an L2-resident 64 MiB buffer into a 6-deep ring of 32 KiB stages (4 boxes per
// stage), no consumer. Shapes: {16 fp32 x 128 rows, 64B swizzle} (the GEMM's K-major A tile),
// {32 x 64, 128B swizzle}, {256 x 8, no swizzle} (1 KiB rows). Prints GB/s and B/clk/SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_box_bench tma_box_bench.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t su32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(32, 1) stream_boxes(const __grid_constant__ CUtensorMap tm,
                                                      int box_c, int box_r, int ncols,
                                                      int nrows, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                              ~uintptr_t(1023));
  __shared__ uint64_t full[6];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < 6; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
  asm volatile("fence.mbarrier_init.release.cluster;");
  const int tiles_c = ncols / box_c, tiles_r = nrows / box_r;
  uint32_t phase[6] = {0, 0, 0, 0, 0, 0};
  int t = blockIdx.x * 37;
  for (int it = 0; it < iters; ++it) {
    const int s = it % 6;
    if (it >= 6) {  // wait for this stage's previous fill before reusing it
      asm volatile(
          "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
          "@!p bra W;\n}" ::"r"(su32(&full[s])),
          "r"(phase[s]));
      phase[s] ^= 1;
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])),
                 "r"(32768));
    for (int b = 0; b < 4; ++b, ++t) {
      const int tc = t % tiles_c, tr = (t / tiles_c) % tiles_r;
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3}], [%4];" ::"r"(su32(smem + s * 32768 + b * 8192)),
          "l"(reinterpret_cast<uint64_t>(&tm)), "r"(tc * box_c), "r"(tr * box_r),
          "r"(su32(&full[s]))
          : "memory");
    }
  }
  for (int s = 0; s < 6; ++s) {
    asm volatile(
        "{\n.reg .pred p;\nW2: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra W2;\n}" ::"r"(su32(&full[s])),
        "r"(phase[s]));
  }
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
  struct Shape { int c, r; CUtensorMapSwizzle sw; const char *name; };
  const Shape shapes[] = {{16, 128, CU_TENSOR_MAP_SWIZZLE_64B, "16x128 sw64 (64 B rows)"},
                          {32, 64, CU_TENSOR_MAP_SWIZZLE_128B, "32x64 sw128 (128 B rows)"},
                          {256, 8, CU_TENSOR_MAP_SWIZZLE_NONE, "256x8 none (1 KiB rows)"}};
  cudaFuncSetAttribute(stream_boxes, cudaFuncAttributeMaxDynamicSharedMemorySize, 6 * 32768 + 1024);
  for (int rep = 0; rep < 2; ++rep)
    for (const Shape &sh : shapes) {
      // view the buffer as rows of `ncols` fp32 (64 KiB rows for the narrow boxes)
      const int ncols = sh.c == 256 ? 256 : 16384;
      const int nrows = int(bytes / 4 / ncols);
      CUtensorMap tm;
      const cuuint64_t dims[2] = {cuuint64_t(ncols), cuuint64_t(nrows)};
      const cuuint64_t strides[1] = {cuuint64_t(ncols) * 4};
      const cuuint32_t box[2] = {cuuint32_t(sh.c), cuuint32_t(sh.r)};
      const cuuint32_t es[2] = {1, 1};
      if (enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, buf, dims, strides, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, sh.sw, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        printf("encode failed for %s\n", sh.name);
        continue;
      }
      const int iters = 20000;
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      stream_boxes<<<sms, 32, 6 * 32768 + 1024>>>(tm, sh.c, sh.r, ncols, nrows, 200);
      cudaEventRecord(a);
      stream_boxes<<<sms, 32, 6 * 32768 + 1024>>>(tm, sh.c, sh.r, ncols, nrows, iters);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double total = double(sms) * iters * 32768.0;
      printf("{\"box\": \"%s\", \"GBps\": %.1f, \"B_per_clk_per_SM_at_max_clock\": %.1f, \"err\": \"%s\"}\n",
             sh.name, total / ms / 1e6, total / (ms * 1e-3) / sms / (clk * 1e3),
             cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
