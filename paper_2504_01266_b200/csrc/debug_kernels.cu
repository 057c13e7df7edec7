// debug_kernels.cu -- bring-up probes for the sm_100a building blocks (libgiga_debug.so).
// Not part of the product path: tests/ and scripts/ use it to check TMA tile layouts,
// UMMA descriptors and TMEM round trips in isolation.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include "kernels.h"
#include "ptx.cuh"

namespace giga {
namespace dbg {

// Nothing but the pair TMEM allocation the GEMM does (cta_group::2 alloc, cluster sync,
// dealloc): isolates the toolchain's own alloc handshake for compute-sanitizer racecheck.
__global__ void __cluster_dims__(2, 1, 1) tmem_pair_alloc_kernel(int *out) {
  __shared__ uint32_t slot;
  if (threadIdx.x < 32) ptx::tmem_alloc_cg2(&slot, 512);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t base = slot;
  if (threadIdx.x == 0) out[blockIdx.x] = int(base);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  if (threadIdx.x < 32) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_cg2(base, 512);
  }
}

// Occupier: each CTA (one per SM: its shared memory leaves no room for a GEMM CTA beside it)
// records its SM and spins for `ns` nanoseconds of %globaltimer. Takes SMs away from a
// concurrently launched GEMM, the way NCCL's kernels do in the multi-GPU pipeline.
__global__ void occupy_kernel(int64_t ns, int *smids) {
  extern __shared__ uint8_t pad[];
  if (threadIdx.x == 0) {
    uint32_t sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    pad[0] = 1;
    smids[blockIdx.x] = int(sm);
    const uint64_t t0 = ptx::globaltimer_ns();
    while (int64_t(ptx::globaltimer_ns() - t0) < ns) __nanosleep(1000);
  }
}

// TMA one box into smem, dump the raw smem bytes (box_bytes) to out.
__global__ void tma_dump_kernel(const __grid_constant__ CUtensorMap tm, int c0, int c1,
                                uint32_t box_bytes, float *out) {
  extern __shared__ uint8_t raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ptx::mbar_expect_tx(&bar, box_bytes);
    ptx::tma_load_2d(smem, &tm, &bar, c0, c1);
  }
  ptx::mbar_wait(&bar, 0);
  for (uint32_t i = threadIdx.x; i < box_bytes / 4; i += blockDim.x)
    out[i] = reinterpret_cast<float *>(smem)[i];
}

// One UMMA: smem images of A (a_bytes) and B (b_bytes) copied verbatim from global, then
// tcgen05.mma with the given descriptors fields, then TMEM -> D (128 x n, row-major).
__global__ void mma_once_kernel(const float *a_img, uint32_t a_bytes, const float *b_img,
                                uint32_t b_bytes, uint32_t a_lbo, uint32_t a_sbo,
                                uint32_t a_layout, uint32_t b_lbo, uint32_t b_sbo,
                                uint32_t b_layout, uint32_t idesc, int n, float *D) {
  extern __shared__ uint8_t raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  uint8_t *sa = smem;
  uint8_t *sb = smem + ((a_bytes + 1023) & ~1023u);
  for (uint32_t i = threadIdx.x; i < a_bytes / 4; i += blockDim.x)
    reinterpret_cast<float *>(sa)[i] = a_img[i];
  for (uint32_t i = threadIdx.x; i < b_bytes / 4; i += blockDim.x)
    reinterpret_cast<float *>(sb)[i] = b_img[i];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    ptx::mbar_init(&bar, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 0) ptx::tmem_alloc(&slot, 256);
  // generic-proxy smem writes must be visible to the async (tensor core) proxy
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    auto mk = [](uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t lay) {
      uint64_t d = 0;
      d |= uint64_t((addr >> 4) & 0x3FFF);
      d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
      d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
      d |= uint64_t(1) << 46;
      d |= uint64_t(lay & 7) << 61;
      return d;
    };
    const uint64_t da = mk(ptx::smem_u32(sa), a_lbo, a_sbo, a_layout);
    const uint64_t db = mk(ptx::smem_u32(sb), b_lbo, b_sbo, b_layout);
    ptx::mma_tf32(tmem, da, db, idesc, 0);
    ptx::mma_commit(&bar);
  }
  ptx::mbar_wait(&bar, 0);
  ptx::tc_fence_after();
  if (warp < 4) {
    for (int c = 0; c < n; c += 16) {
      float v[16];
      ptx::tmem_ld16_wait(tmem + (uint32_t(warp * 32) << 16) + c, v);
      for (int j = 0; j < 16 && c + j < n; ++j) D[(warp * 32 + lane) * n + c + j] = v[j];
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc(tmem, 256);
  }
}

}  // namespace dbg
}  // namespace giga

using namespace giga;

extern "C" int giga_dbg_tma_dump(const float *A, int64_t rows, int64_t cols, int box_cols,
                                 int box_rows, int swizzle_bytes, int c0, int c1, float *out) {
  if (ensure_tma_encoder() != 0) return -1;
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q{};
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap tm;
  const cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
  const cuuint64_t strides[1] = {cuuint64_t(cols) * 4};
  const cuuint32_t box[2] = {cuuint32_t(box_cols), cuuint32_t(box_rows)};
  const cuuint32_t estr[2] = {1, 1};
  CUtensorMapSwizzle sw = swizzle_bytes == 132  ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B
                          : swizzle_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                          : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                          : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                : CU_TENSOR_MAP_SWIZZLE_NONE;
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(A), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return -2;
  const uint32_t bytes = uint32_t(box_cols) * box_rows * 4;
  cudaFuncSetAttribute(dbg::tma_dump_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       int(bytes + 1024));
  dbg::tma_dump_kernel<<<1, 128, bytes + 1024>>>(tm, c0, c1, bytes, out);
  if (cudaGetLastError() != cudaSuccess) return -3;
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : -4;
}

extern "C" int giga_dbg_mma_once(const float *a_img, int a_bytes, const float *b_img,
                                 int b_bytes, int a_lbo, int a_sbo, int a_layout, int b_lbo,
                                 int b_sbo, int b_layout, unsigned idesc, int n, float *D) {
  const int smem = ((a_bytes + 1023) & ~1023) + b_bytes + 1024;
  cudaFuncSetAttribute(dbg::mma_once_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       smem);
  dbg::mma_once_kernel<<<1, 128, smem>>>(a_img, a_bytes, b_img, b_bytes, a_lbo, a_sbo,
                                         a_layout, b_lbo, b_sbo, b_layout, idesc, n, D);
  if (cudaGetLastError() != cudaSuccess) return -3;
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : -4;
}

extern "C" int giga_dbg_tmem_pair_alloc(int nclusters, int *out) {
  dbg::tmem_pair_alloc_kernel<<<2 * nclusters, 64>>>(out);
  if (cudaGetLastError() != cudaSuccess) return -3;
  return cudaDeviceSynchronize() == cudaSuccess ? 0 : -4;
}

// k occupier CTAs (occupy_kernel) on `stream`, `smem` bytes of shared memory each.
extern "C" int giga_dbg_occupy(int nctas, int smem, int64_t ns, int *smids, void *stream) {
  if (cudaFuncSetAttribute(dbg::occupy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           smem) != cudaSuccess)
    return -2;
  dbg::occupy_kernel<<<nctas, 32, smem, static_cast<cudaStream_t>(stream)>>>(ns, smids);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

// One GEMM launch of the product scheme's kernel with its persistent grid capped at max_ctas
// SMs (the NCCL pipeline's configuration: GemmExtra::max_ctas), on `stream`.
extern "C" int giga_dbg_gemm_max_ctas(const float *A, const float *B, float *C, int64_t M,
                                      int64_t N, int64_t K, int terms, int max_ctas,
                                      void *stream) {
  giga::GemmExtra ex;
  ex.max_ctas = max_ctas;
  return giga::launch_gemm_3xtf32(A, nullptr, B, nullptr, C, M, N, K, N, terms, -1,
                                  static_cast<cudaStream_t>(stream), 0, &ex) == cudaSuccess
             ? 0
             : -3;
}
