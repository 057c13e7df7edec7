// vecops.cu -- GigaAPI's data-parallel vector operations (arXiv 2504.01266 S4.2.8,
// PAPER.md:294-303): dot product and L2 norm of fp32 vectors, sm_100a.
//
// The paper's kernel: each thread keeps "a running sum to accumulate the partial dot
// product" over a grid-stride range, a 256-slot shared cache, a halving tree reduction and
// per-block partials summed on the host; L2 = sqrt(dot(x, x)) once on the host
// (P:303). Here: 16-byte vector loads with four in flight per thread (the op is HBM-bound:
// 8 bytes per element), products of two fp32 values formed exactly in fp64 and summed in
// fp64, warp-shuffle + shared-memory block reduction, and the per-block partials summed in
// a fixed order by the last block to finish (an atomic ticket), so one launch returns the
// result in device memory and the result is bit-reproducible for a given grid.
#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.h"

namespace giga {

constexpr int kDotThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__global__ void __launch_bounds__(kDotThreads) dot_kernel(const float *__restrict__ x,
                                                          const float *__restrict__ y,
                                                          int64_t n, double *partials,
                                                          unsigned *ticket, double *out) {
  double acc = 0.0;
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15) == 0;
  int64_t done = 0;
  if (vec) {
    const int64_t n4 = n >> 2;
    const float4 *x4 = reinterpret_cast<const float4 *>(x);
    const float4 *y4 = reinterpret_cast<const float4 *>(y);
    int64_t i = tid;
    for (; i + 3 * stride < n4; i += 4 * stride) {
      float4 a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a[u] = __ldcs(x4 + i + u * stride);
        b[u] = __ldcs(y4 + i + u * stride);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        acc = fma(double(a[u].x), double(b[u].x), acc);
        acc = fma(double(a[u].y), double(b[u].y), acc);
        acc = fma(double(a[u].z), double(b[u].z), acc);
        acc = fma(double(a[u].w), double(b[u].w), acc);
      }
    }
    for (; i < n4; i += stride) {
      const float4 a = __ldcs(x4 + i), b = __ldcs(y4 + i);
      acc = fma(double(a.x), double(b.x), acc);
      acc = fma(double(a.y), double(b.y), acc);
      acc = fma(double(a.z), double(b.z), acc);
      acc = fma(double(a.w), double(b.w), acc);
    }
    done = n4 << 2;
  }
  for (int64_t i = done + tid; i < n; i += stride) acc = fma(double(x[i]), double(y[i]), acc);

  __shared__ double red[kDotThreads / 32];
  __shared__ bool last;
  acc = warp_sum(acc);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[warp] = acc;
  __syncthreads();
  if (warp == 0) {
    double v = lane < kDotThreads / 32 ? red[lane] : 0.0;
    v = warp_sum(v);
    if (lane == 0) {
      partials[blockIdx.x] = v;
      __threadfence();
      last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
  }
  __syncthreads();
  if (!last) return;
  // The last block sums the partials in a fixed order (thread t: partials t, t + 256, ... in
  // sequence; then the same shuffle / shared-memory tree as above): deterministic for a given
  // grid, and ~5 dependent loads per thread instead of one thread walking all of them.
  __threadfence();
  double s = 0.0;
  volatile const double *vp = partials;
  for (unsigned b = threadIdx.x; b < gridDim.x; b += kDotThreads) s += vp[b];
  s = warp_sum(s);
  if (lane == 0) red[warp] = s;
  __syncthreads();
  if (warp == 0) {
    double v = lane < kDotThreads / 32 ? red[lane] : 0.0;
    v = warp_sum(v);
    if (lane == 0) {
      *out = v;
      *ticket = 0;  // ready for the next launch on this workspace
    }
  }
}

int dot_grid(int64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t blocks = (n / 4 + kDotThreads - 1) / kDotThreads;
  int64_t cap = int64_t(sms) * 8;
  if (cap > kDotMaxBlocks) cap = kDotMaxBlocks;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  return int(blocks);
}

cudaError_t launch_dot(const float *x, const float *y, int64_t n, double *partials,
                       unsigned *ticket, double *out, cudaStream_t st) {
  if (n < 0) return cudaErrorInvalidValue;
  const int grid = dot_grid(n);
  dot_kernel<<<grid, kDotThreads, 0, st>>>(x, y, n, partials, ticket, out);
  return cudaGetLastError();
}

}  // namespace giga
