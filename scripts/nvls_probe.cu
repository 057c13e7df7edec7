// NVLink multicast (NVLS) probe (measurement tool, not product code): can this box bind a
// buffer into a cuMulticastCreate object, and which store paths reach memory through the
// multicast address -- multimem.st (SIMT), a TMA tensor store (cp.async.bulk.tensor) and a
// plain bulk store (cp.async.bulk) from shared memory? Each path writes a known pattern
// through the multicast VA; the host reads it back through the unicast mapping. Rates are
// for one device in the team (the only case a 1-GPU box allows).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o nvls_probe nvls_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define CK(x)                                                                   \
  do {                                                                          \
    CUresult r_ = (x);                                                          \
    if (r_ != CUDA_SUCCESS) {                                                   \
      const char *s_ = nullptr;                                                 \
      cuGetErrorString(r_, &s_);                                                \
      printf("{\"step\": \"%s\", \"err\": \"%s\"}\n", #x, s_ ? s_ : "?");     \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

__global__ void st_multimem(float *mc, int64_t n4, float base) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n4;
       i += int64_t(gridDim.x) * blockDim.x) {
    float v = base + float(i & 1023);
    asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + 4 * i), "f"(v),
                 "f"(v + 1), "f"(v + 2), "f"(v + 3)
                 : "memory");
  }
}

__global__ void st_plain(float *p, int64_t n4, float base) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n4;
       i += int64_t(gridDim.x) * blockDim.x) {
    float v = base + float(i & 1023);
    reinterpret_cast<float4 *>(p)[i] = make_float4(v, v + 1, v + 2, v + 3);
  }
}

// every CTA fills a 32 KiB smem tile (rows of 64 floats) and stores it with the TMA (tensor
// map over the target) or a bulk copy, over its share of 512-row tiles
__global__ void __launch_bounds__(128) st_tma(const __grid_constant__ CUtensorMap tm, float *dst,
                                              int rows, int cols, float base, int bulk) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  float *tile = reinterpret_cast<float *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                          ~uintptr_t(1023));
  const int tr = 128, tc = 64;  // 32 KiB
  const int ntiles = (rows / tr) * (cols / tc);
  for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int r0 = (t / (cols / tc)) * tr, c0 = (t % (cols / tc)) * tc;
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    __syncthreads();
    for (int e = threadIdx.x; e < tr * tc; e += blockDim.x) {
      const int r = e / tc, c = e % tc;
      tile[e] = base + float(((int64_t(r0 + r) * cols + c0 + c) / 4) & 1023) + float((c0 + c) & 3);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(tile));
      if (bulk) {
        for (int r = 0; r < tr; ++r)
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                           dst + int64_t(r0 + r) * cols + c0),
                       "r"(s + uint32_t(r * tc * 4)), "r"(tc * 4)
                       : "memory");
      } else {
        asm volatile(
            "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                reinterpret_cast<uint64_t>(&tm)),
            "r"(c0), "r"(r0), "r"(s)
            : "memory");
      }
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

static int check(const float *h, int64_t n, float base, const char *what) {
  int64_t bad = 0;
  for (int64_t i = 0; i < n; ++i) {
    const float want = base + float((i / 4) & 1023) + float(i & 3);
    if (h[i] != want) ++bad;
  }
  printf("{\"path\": \"%s\", \"mismatches\": %lld}\n", what, (long long)bad);
  return bad == 0;
}

int main() {
  CK(cuInit(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  CUcontext ctx;
  cudaSetDevice(0);
  cudaFree(0);
  CK(cuCtxGetCurrent(&ctx));
  int mc_sup = 0, ndev = 0;
  cuDeviceGetAttribute(&mc_sup, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev);
  cuDeviceGetCount(&ndev);
  printf("{\"multicast_supported\": %d, \"devices\": %d}\n", mc_sup, ndev);
  if (!mc_sup) return 0;

  const size_t want = 256ull << 20;
  CUmulticastObjectProp mp = {};
  mp.numDevices = 1;
  mp.size = want;
  mp.handleTypes = CU_MEM_HANDLE_TYPE_NONE;
  size_t gran = 0;
  CK(cuMulticastGetGranularity(&gran, &mp, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  const size_t size = (want + gran - 1) / gran * gran;
  mp.size = size;
  printf("{\"mc_granularity\": %zu, \"size\": %zu}\n", gran, size);
  CUmemGenericAllocationHandle mch, memh;
  // creation alone with a team of 2 (never bound: binding would wait for a second device):
  // tells whether a one-device team or multicast as such is what the driver refuses
  for (unsigned nd = 2; nd <= 2; ++nd) {
    CUmulticastObjectProp m2 = mp;
    m2.numDevices = nd;
    const CUmemAllocationHandleType hts2[3] = {CU_MEM_HANDLE_TYPE_NONE,
                                               CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
                                               CU_MEM_HANDLE_TYPE_FABRIC};
    for (int h = 0; h < 3; ++h) {
      m2.handleTypes = hts2[h];
      CUmemGenericAllocationHandle t;
      const CUresult r2 = cuMulticastCreate(&t, &m2);
      const char *es = nullptr;
      cuGetErrorString(r2, &es);
      printf("{\"cuMulticastCreate_team\": %u, \"handle_type\": %d, \"result\": \"%s\"}\n", nd,
             int(hts2[h]), es ? es : "?");
      if (r2 == CUDA_SUCCESS) cuMemRelease(t);
    }
  }
  // the handle type the driver accepts varies by platform: try none, POSIX fd, fabric
  const CUmemAllocationHandleType hts[3] = {CU_MEM_HANDLE_TYPE_NONE,
                                            CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
                                            CU_MEM_HANDLE_TYPE_FABRIC};
  CUresult cr = CUDA_ERROR_INVALID_VALUE;
  for (int h = 0; h < 3 && cr != CUDA_SUCCESS; ++h) {
    mp.handleTypes = hts[h];
    cr = cuMulticastCreate(&mch, &mp);
    const char *es = nullptr;
    cuGetErrorString(cr, &es);
    printf("{\"cuMulticastCreate_handle_type\": %d, \"result\": \"%s\"}\n", int(hts[h]), es ? es : "?");
  }
  if (cr != CUDA_SUCCESS) return 1;
  CK(cuMulticastAddDevice(mch, dev));
  CUmemAllocationProp ap = {};
  ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ap.location.id = 0;
  ap.requestedHandleTypes = static_cast<CUmemAllocationHandleType>(mp.handleTypes);
  size_t ugran = 0;
  CK(cuMemGetAllocationGranularity(&ugran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  CK(cuMemCreate(&memh, size, &ap, 0));
  CK(cuMulticastBindMem(mch, 0, memh, 0, size, 0));
  CUdeviceptr uc = 0, mc = 0;
  CK(cuMemAddressReserve(&uc, size, gran, 0, 0));
  CK(cuMemMap(uc, size, 0, memh, 0));
  CK(cuMemAddressReserve(&mc, size, gran, 0, 0));
  CK(cuMemMap(mc, size, 0, mch, 0));
  CUmemAccessDesc ad = {};
  ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  ad.location.id = 0;
  ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(uc, size, &ad, 1));
  CK(cuMemSetAccess(mc, size, &ad, 1));
  printf("{\"mapped\": true}\n");

  const int64_t n = int64_t(size / 4);
  float *h = static_cast<float *>(malloc(size));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto rate = [&](const char *what) {
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"path\": \"%s\", \"GBps\": %.1f, \"err\": \"%s\"}\n", what, size / ms / 1e6,
           cudaGetErrorString(cudaGetLastError()));
  };
  // 1. plain stores through the unicast VA (reference rate)
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    st_plain<<<148 * 4, 512>>>(reinterpret_cast<float *>(uc), n / 4, 1.0f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
  }
  rate("st.global unicast");
  // 2. multimem.st through the multicast VA
  cudaMemset(reinterpret_cast<void *>(uc), 0, size);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    st_multimem<<<148 * 4, 512>>>(reinterpret_cast<float *>(mc), n / 4, 2.0f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
  }
  rate("multimem.st.v4.f32 multicast");
  cudaMemcpy(h, reinterpret_cast<void *>(uc), size, cudaMemcpyDeviceToHost);
  check(h, n, 2.0f, "multimem.st.v4.f32 multicast");

  // 3./4. TMA tensor store and bulk store through the multicast VA
  void *fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  const int cols = 8192, rows = int(n / cols);
  cudaFuncSetAttribute(st_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 33 * 1024);
  for (int target = 0; target < 2; ++target) {
    const CUdeviceptr base = target ? mc : uc;
    CUtensorMap tm;
    const cuuint64_t dims[2] = {cuuint64_t(cols), cuuint64_t(rows)};
    const cuuint64_t strides[1] = {cuuint64_t(cols) * 4};
    const cuuint32_t box[2] = {64, 128};
    const cuuint32_t es[2] = {1, 1};
    CUresult er = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, reinterpret_cast<void *>(base),
                      dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (er != CUDA_SUCCESS) {
      printf("{\"path\": \"tensormap encode %s\", \"err\": %d}\n", target ? "mc" : "uc", int(er));
      continue;
    }
    for (int bulk = 0; bulk < 2; ++bulk) {
      cudaMemset(reinterpret_cast<void *>(uc), 0, size);
      const float b = 3.0f + target * 2 + bulk;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        st_tma<<<148, 128, 33 * 1024>>>(tm, reinterpret_cast<float *>(base), rows, cols, b, bulk);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
      }
      char what[96];
      snprintf(what, sizeof what, "%s store via %s VA", bulk ? "cp.async.bulk" : "TMA tensor",
               target ? "multicast" : "unicast");
      rate(what);
      cudaMemcpy(h, reinterpret_cast<void *>(uc), size, cudaMemcpyDeviceToHost);
      check(h, n, b, what);
    }
  }
  printf("{\"done\": true}\n");
  return 0;
}
