// prep16.cu -- the 3xFP16 scheme's operand preparation and A-side exception fix (DESIGN.md
// 6.8), sm_100a: per-row / per-column power-of-two scales, fp16 hi / lo operands, exception
// bitmaps and lists, then (after the GEMM) C += (a - rep(a)) rep(b) for A's exceptions. The
// GEMM itself and its epilogue's B-side fix are in gemm_3xtf32.cu.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <algorithm>

#include "kernels.h"
#include "ptx.cuh"
#include "split16.cuh"

namespace giga {

// A: TPR threads per row (512: one row per block for long rows, whose second read then hits
// L2; 32: one warp per row), row groups grid-strided; padding rows (M <= m < m_pad) only write
// their exponent 0 (ea is padded to whole tiles). Pass 1: max |a| of the row (bit patterns:
// NaN > Inf > finite); pass 2 re-reads the row and writes A_hi / A_lo (fp16, row stride ldh)
// and the row's exceptions. 4 B read (+ the re-read), 4 B written per element.
template <int TPR>
__global__ void __launch_bounds__(512) prep16_a_kernel(const float *__restrict__ A, int64_t lda,
                                                       int M, int m_pad, int K,
                                                       uint16_t *__restrict__ Ah,
                                                       uint16_t *__restrict__ Al, int64_t ldh,
                                                       int *__restrict__ ea,
                                                       unsigned *__restrict__ bits, int wa,
                                                       unsigned *__restrict__ summ, int w2,
                                                       int *__restrict__ flag) {
  constexpr int RPB = 512 / TPR;
  __shared__ uint32_t red[16];
  const int t = int(threadIdx.x) % TPR, rsub = int(threadIdx.x) / TPR;
  const int k4 = K >> 2;
  for (int g = blockIdx.x; g * RPB < m_pad; g += gridDim.x) {
    const int m = g * RPB + rsub;
    const bool live = m < M;
    const float *row = A + int64_t(live ? m : 0) * lda;
    uint32_t mx = 0;
    if (live) {
      // 8 loads in flight per thread
      for (int i0 = t; i0 < k4; i0 += 8 * TPR) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          v[u] = i0 + u * TPR < k4 ? __ldg(reinterpret_cast<const float4 *>(row) + i0 + u * TPR)
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int u = 0; u < 8; ++u)
          mx = max(mx, max(max(__float_as_uint(v[u].x) & 0x7fffffffu,
                               __float_as_uint(v[u].y) & 0x7fffffffu),
                           max(__float_as_uint(v[u].z) & 0x7fffffffu,
                               __float_as_uint(v[u].w) & 0x7fffffffu)));
      }
      for (int k = (k4 << 2) + t; k < K; k += TPR) mx = max(mx, __float_as_uint(row[k]) & 0x7fffffffu);
    }
    mx = __reduce_max_sync(0xffffffffu, mx);
    if (TPR > 32) {
      if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
      __syncthreads();
      if (threadIdx.x < 32) {
        uint32_t v = threadIdx.x < (TPR >> 5) ? red[threadIdx.x] : 0u;
        v = __reduce_max_sync(0xffffffffu, v);
        if (threadIdx.x == 0) red[0] = v;
      }
      __syncthreads();
      mx = red[0];
      __syncthreads();  // red is reused by the next row group
    }
    if (m >= m_pad) continue;
    const int e = live ? scale_exp(mx) : 0;
    if (t == 0) ea[m] = e;
    if (!live) continue;
    uint16_t *hd = Ah + int64_t(m) * ldh, *ld = Al + int64_t(m) * ldh;
    for (int i0 = t; i0 < k4; i0 += 4 * TPR) {
      float4 vv[4];  // 4 loads in flight per thread (the row is L2-resident from pass 1)
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i0 + u * TPR < k4) vv[u] = __ldg(reinterpret_cast<const float4 *>(row) + i0 + u * TPR);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * TPR;
      if (i >= k4) break;
      const float4 v = vv[u];
      uint16_t h[4], l[4];
      const bool x0 = split_f16(v.x, e, h[0], l[0]);
      const bool x1 = split_f16(v.y, e, h[1], l[1]);
      const bool x2 = split_f16(v.z, e, h[2], l[2]);
      const bool x3 = split_f16(v.w, e, h[3], l[3]);
      if (x0 | x1 | x2 | x3) {
        const unsigned nib =
            unsigned(x0) | unsigned(x1) << 1 | unsigned(x2) << 2 | unsigned(x3) << 3;
        const int k = 4 * i, w = k >> 5;
        mark_exception(bits, int64_t(m) * wa + w, nib << (k & 31), summ, int64_t(m) * w2 + (w >> 5),
                       w & 31, flag + m);
      }
      __stcs(reinterpret_cast<uint2 *>(hd) + i,
             make_uint2(h[0] | uint32_t(h[1]) << 16, h[2] | uint32_t(h[3]) << 16));
      __stcs(reinterpret_cast<uint2 *>(ld) + i,
             make_uint2(l[0] | uint32_t(l[1]) << 16, l[2] | uint32_t(l[3]) << 16));
      }
    }
    for (int k = (k4 << 2) + t; k < K; k += TPR) {
      uint16_t h, l;
      if (split_f16(row[k], e, h, l))
        mark_exception(bits, int64_t(m) * wa + (k >> 5), 1u << (k & 31), summ,
                       int64_t(m) * w2 + (k >> 10), (k >> 5) & 31, flag + m);
      hd[k] = h;
      ld[k] = l;
    }
  }
}

// B pass 1: per-column max |b| bits into bmax (zeroed before): a block covers 1024 columns
// (256 threads x 4: every row it reads is one 4 KiB contiguous stretch) and `rows` rows (8 in
// flight per thread), one atomicMax per column per block. rows is chosen so the grid is ~8
// blocks per SM.
__global__ void __launch_bounds__(256) prep16_bmax_kernel(const float *__restrict__ B, int64_t ldb,
                                                          int K, int N, int rows,
                                                          unsigned *__restrict__ bmax) {
  const int n = (blockIdx.x * 256 + int(threadIdx.x)) * 4;
  if (n >= N) return;
  const int r0 = blockIdx.y * rows;
  const int r1 = min(K, r0 + rows);
  uint4 mx = make_uint4(0, 0, 0, 0);
  auto take = [&](float4 v) {
    mx.x = max(mx.x, __float_as_uint(v.x) & 0x7fffffffu);
    mx.y = max(mx.y, __float_as_uint(v.y) & 0x7fffffffu);
    mx.z = max(mx.z, __float_as_uint(v.z) & 0x7fffffffu);
    mx.w = max(mx.w, __float_as_uint(v.w) & 0x7fffffffu);
  };
  if (n + 3 < N) {
    int r = r0;
    for (; r + 8 <= r1; r += 8) {
      float4 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        v[u] = __ldg(reinterpret_cast<const float4 *>(B + int64_t(r + u) * ldb + n));
#pragma unroll
      for (int u = 0; u < 8; ++u) take(v[u]);
    }
    for (; r < r1; ++r) take(__ldg(reinterpret_cast<const float4 *>(B + int64_t(r) * ldb + n)));
  } else {
    for (int r = r0; r < r1; ++r) {
      const float *src = B + int64_t(r) * ldb + n;
      take(make_float4(src[0], n + 1 < N ? src[1] : 0.f, n + 2 < N ? src[2] : 0.f, 0.f));
    }
  }
  atomicMax(bmax + n, mx.x);
  if (n + 1 < N) atomicMax(bmax + n + 1, mx.y);
  if (n + 2 < N) atomicMax(bmax + n + 2, mx.z);
  if (n + 3 < N) atomicMax(bmax + n + 3, mx.w);
}

// B pass 4 (after the writes): the exception list of every strip of 32 columns, one warp per
// strip: for each flagged column (ascending) its exceptions in ascending k, as (k, column in
// the strip, b - rep(b) in fp64), up to kBList entries; bcnt = the strip's total (a total above
// kBList sends the epilogue to the bitmap scan instead).
__global__ void __launch_bounds__(256) compact16_b_kernel(
    const float *__restrict__ B, int64_t ldb, int N, int K, const uint16_t *__restrict__ Bh,
    const uint16_t *__restrict__ Bl, int64_t ldbh, const int *__restrict__ eb,
    const unsigned *__restrict__ bits, const unsigned *__restrict__ summ, int w2,
    const int *__restrict__ flag, int *__restrict__ bcnt, int4 *__restrict__ blist) {
  const int lane = threadIdx.x & 31;
  const int strip = blockIdx.x * 8 + int(threadIdx.x >> 5);
  if (strip * 32 >= N) return;
  const int j = strip * 32 + lane;
  unsigned cols = __ballot_sync(0xffffffffu, j < N && flag[j] != 0);
  const unsigned *S = summ + int64_t(strip) * w2;
  const unsigned *L = bits + int64_t(strip) * K;
  int4 *out = blist + int64_t(strip) * kBList;
  int n = 0;
  while (cols) {
    const int jb = __ffs(cols) - 1;
    cols &= cols - 1;
    const int jj = strip * 32 + jb;
    const int e = eb[jj];
    for (int c0 = 0; c0 < w2; c0 += 32) {
      const unsigned sw = c0 + lane < w2 ? S[c0 + lane] : 0u;
      unsigned nz = __ballot_sync(0xffffffffu, sw != 0u);
      while (nz) {
        const int src = __ffs(nz) - 1;
        nz &= nz - 1;
        const unsigned swv = __shfl_sync(0xffffffffu, sw, src);
        const int k = (c0 + src) * 32 + lane;
        const bool hit = ((swv >> lane) & 1u) && k < K && ((L[k] >> jb) & 1u);
        const unsigned hits = __ballot_sync(0xffffffffu, hit);
        if (hit) {
          const int pos = n + __popc(hits & ((1u << lane) - 1u));
          if (pos < kBList) {
            const int64_t o = int64_t(k) * ldbh + jj;
            const double d = double(B[int64_t(k) * ldb + jj]) -
                             ldexp(double(__half2float(__ushort_as_half(Bh[o]))) +
                                       double(__half2float(__ushort_as_half(Bl[o]))), e);
            out[pos] = make_int4(k, jb, __double2loint(d), __double2hiint(d));
          }
        }
        n += __popc(hits);
      }
    }
  }
  if (lane == 0) bcnt[strip] = n;
}

// B pass 2: eb[j] for every padded column (bmax of padding columns is 0 -> exponent 0).
__global__ void prep16_bexp_kernel(const unsigned *__restrict__ bmax, int n_pad,
                                   int *__restrict__ eb) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < n_pad) eb[j] = scale_exp(bmax[j]);
}

// B pass 3: B_hi / B_lo (fp16, K x N row-major, row stride ldh) and B's exceptions. A block
// covers 1024 columns (256 threads x 4: every row it touches is one 4 KiB stretch in, two 2 KiB
// stretches out) and `rows` rows, RIF rows' loads in flight per thread (the pass-1 layout),
// MINB blocks per SM.
__device__ __forceinline__ void prep16_b_put(const float4 v, int k, int n, int K, int4 e,
                                             uint16_t *__restrict__ Bh,
                                             uint16_t *__restrict__ Bl, int64_t ldh,
                                             unsigned *__restrict__ bits,
                                             unsigned *__restrict__ summ, int w2,
                                             int *__restrict__ flag) {
  uint16_t h[4], l[4];
  const bool x0 = split_f16(v.x, e.x, h[0], l[0]);
  const bool x1 = split_f16(v.y, e.y, h[1], l[1]);
  const bool x2 = split_f16(v.z, e.z, h[2], l[2]);
  const bool x3 = split_f16(v.w, e.w, h[3], l[3]);
  if (x0 | x1 | x2 | x3) {
    const unsigned nib = unsigned(x0) | unsigned(x1) << 1 | unsigned(x2) << 2 | unsigned(x3) << 3;
    atomicOr(bits + int64_t(n >> 5) * K + k, nib << (n & 31));
    atomicOr(summ + int64_t(n >> 5) * w2 + (k >> 5), 1u << (k & 31));
    volatile int *f = flag + n;
    if (x0) f[0] = 1;
    if (x1) f[1] = 1;
    if (x2) f[2] = 1;
    if (x3) f[3] = 1;
  }
  __stcs(reinterpret_cast<uint2 *>(Bh + int64_t(k) * ldh + n),
         make_uint2(h[0] | uint32_t(h[1]) << 16, h[2] | uint32_t(h[3]) << 16));
  __stcs(reinterpret_cast<uint2 *>(Bl + int64_t(k) * ldh + n),
         make_uint2(l[0] | uint32_t(l[1]) << 16, l[2] | uint32_t(l[3]) << 16));
}

template <int RIF, int MINB>
__global__ void __launch_bounds__(256, MINB) prep16_b_kernel(const float *__restrict__ B, int64_t ldb,
                                                       int K, int N, int rows,
                                                       const int *__restrict__ eb,
                                                       uint16_t *__restrict__ Bh,
                                                       uint16_t *__restrict__ Bl, int64_t ldh,
                                                       unsigned *__restrict__ bits,
                                                       unsigned *__restrict__ summ, int w2,
                                                       int *__restrict__ flag) {
  const int n = (blockIdx.x * 256 + int(threadIdx.x)) * 4;
  if (n >= N) return;
  const int r0 = blockIdx.y * rows;
  const int r1 = min(K, r0 + rows);
  const int4 e = *reinterpret_cast<const int4 *>(eb + n);  // eb is padded to 256 columns
  if (n + 3 < N) {
    int r = r0;
    for (; r + RIF <= r1; r += RIF) {
      float4 v[RIF];
#pragma unroll
      for (int u = 0; u < RIF; ++u)
        v[u] = __ldcs(reinterpret_cast<const float4 *>(B + int64_t(r + u) * ldb + n));
#pragma unroll
      for (int u = 0; u < RIF; ++u) prep16_b_put(v[u], r + u, n, K, e, Bh, Bl, ldh, bits, summ, w2, flag);
    }
    for (; r < r1; ++r)
      prep16_b_put(__ldcs(reinterpret_cast<const float4 *>(B + int64_t(r) * ldb + n)), r, n, K,
                   e, Bh, Bl, ldh, bits, summ, w2, flag);
    return;
  }
  // the last, partial group of columns: scalar
  const int ev[4] = {e.x, e.y, e.z, e.w};
  for (int r = r0; r < r1; ++r)
    for (int q = 0; q < 4 && n + q < N; ++q) {
      uint16_t h, l;
      if (split_f16(B[int64_t(r) * ldb + n + q], ev[q], h, l))
        mark_exception(bits, int64_t((n + q) >> 5) * K + r, 1u << ((n + q) & 31), summ,
                       int64_t((n + q) >> 5) * w2 + (r >> 5), r & 31, flag + n + q);
      Bh[int64_t(r) * ldh + n + q] = h;
      Bl[int64_t(r) * ldh + n + q] = l;
    }
}

// ---- 3xFP16 exceptions: C += the remainders the split could not carry -----------------------
// a b = rep(a) rep(b) + (a - rep(a)) rep(b) + a (b - rep(b)) exactly, rep(x) = 2^e (hi + lo).
// The GEMM computes rep(a) rep(b) and, in its epilogue, adds a (b - rep(b)) for the exceptions
// of B in each block's columns (fix_b_list from compact16_b's lists, fix_b_block when a strip
// overflows them: C is still on chip, the A reads overlap the next tile's MMAs); fix16_a
// (after the GEMM) adds (a - rep(a)) rep(b) for those of A row by row
// (rep(b) rows are contiguous). Both sum in fp64 in ascending k and round once into C
// (deterministic); fix16_a mirrors the new values to the peers' copies when the epilogue also
// wrote those (fused gather), and skips rows without exceptions -- the common case: float
// data has ~1e-6 of its elements more than 2^20 below their row / column maximum (synth d5
// has them at that rate; d1-d4, fixed-point grids, have none).
struct PeerC {
  float *p[kMaxCDst - 1];
  int n;
  float *mc;  // non-null: the multicast address of C's rows (C and every peer in one store)
};
constexpr int kFixCap = 1024;  // exceptions staged in shared memory per pass

// Warp 0's staging of exceptions in ascending order. L: level-1 bitmap words, S: their
// summary (bit w % 32 of S[w / 32] set iff L[w] != 0). Starting at summary word s0 it walks the
// non-zero summary words (granules: 32 level-1 words, at most 1024 exceptions = kFixCap) in
// order and emits every set bit (emit(pos, word, bit), pos = its slot in the staging buffer)
// while the buffer has room for the whole granule. Returns (staged count, next summary word;
// n2 when done) to every lane.
template <class Emit>
__device__ __forceinline__ int2 stage_exceptions(const unsigned *__restrict__ S, int n2,
                                                 const unsigned *__restrict__ L, int n1, int s0,
                                                 Emit emit) {
  const int lane = threadIdx.x & 31;
  int n = 0;
  for (int c0 = s0; c0 < n2; c0 += 32) {
    const unsigned sw = c0 + lane < n2 ? S[c0 + lane] : 0u;
    unsigned nz = __ballot_sync(0xffffffffu, sw != 0u);
    while (nz) {
      const int src = __ffs(nz) - 1;
      nz &= nz - 1;
      const int g = c0 + src;
      const unsigned swv = __shfl_sync(0xffffffffu, sw, src);
      const int wi = g * 32 + lane;
      const unsigned word = ((swv >> lane) & 1u) && wi < n1 ? L[wi] : 0u;
      const int c = __popc(word);
      int incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int total = __shfl_sync(0xffffffffu, incl, 31);
      if (n + total > kFixCap) return make_int2(n, g);  // apply what is staged first
      int pos = n + incl - c;
      for (unsigned b = word; b; b &= b - 1) emit(pos++, wi, __ffs(b) - 1);
      n += total;
    }
  }
  return make_int2(n, n2);
}

// Blocks take 32-row windows of A (grid-strided), find the rows flagged with exceptions in
// one parallel read of their flags and process those rows one by one: warp 0 stages the row's
// exceptions in ascending k through the summary words, then all threads add
// sum_k delta_k rep(B[k][j]) to C[i][j] for every column j.
__global__ void __launch_bounds__(256) fix16_a_kernel(
    const float *__restrict__ A, int64_t lda, int M, int N, const uint16_t *__restrict__ Ah,
    const uint16_t *__restrict__ Al, int64_t ldh, const int *__restrict__ ea,
    const uint16_t *__restrict__ Bh, const uint16_t *__restrict__ Bl, int64_t ldbh,
    const int *__restrict__ eb, const unsigned *__restrict__ bits, int wa,
    const unsigned *__restrict__ summ, int w2, const int *__restrict__ flag,
    float *__restrict__ C, int64_t ldc, const PeerC peers) {
  __shared__ int ks[kFixCap];
  __shared__ double ds[kFixCap];
  __shared__ int n_sh, s_sh, nrows;
  __shared__ int rows[32];  // the flagged rows of the current 32-row window
  // this block's columns: chunk blockIdx.y of gridDim.y (multiples of 4)
  const int chunk = ((N + int(gridDim.y) - 1) / int(gridDim.y) + 3) & ~3;
  const int jlo = int(blockIdx.y) * chunk, jhi = min(N, jlo + chunk);
  for (int base = blockIdx.x * 32; base < M; base += gridDim.x * 32) {
    // the flags of 256 rows at once; the rows holding exceptions (any order: rows are
    // independent)
    __syncthreads();
    if (threadIdx.x == 0) nrows = 0;
    __syncthreads();
    if (threadIdx.x < 32) {
      const int r = base + int(threadIdx.x);
      const bool f = r < M && flag[r] != 0;
      const unsigned bal = __ballot_sync(0xffffffffu, f);
      int wofs = 0;
      if ((threadIdx.x & 31) == 0 && bal) wofs = atomicAdd(&nrows, __popc(bal));
      wofs = __shfl_sync(0xffffffffu, wofs, 0);
      if (f) rows[wofs + __popc(bal & ((1u << (threadIdx.x & 31)) - 1u))] = r;
    }
    __syncthreads();
    const int nr = nrows;
    for (int ri = 0; ri < nr; ++ri) {
      const int i = rows[ri];
      const int e = ea[i];
      for (int s = 0; s < w2;) {
        if (threadIdx.x < 32) {
          const int2 r = stage_exceptions(
              summ + int64_t(i) * w2, w2, bits + int64_t(i) * wa, wa, s,
              [&](int pos, int wi, int bit) {
                const int k = wi * 32 + bit;
                const int64_t o = int64_t(i) * ldh + k;
                ks[pos] = k;
                ds[pos] = double(A[int64_t(i) * lda + k]) - rep16(Ah[o], Al[o], e);
              });
          if (threadIdx.x == 0) {
            n_sh = r.x;
            s_sh = r.y;
          }
        }
        __syncthreads();
        const int n = n_sh;
        s = s_sh;
        // 4 columns per thread and step (N, ldc, ldbh are multiples of 4: float4 / 8-byte
        // loads), all loads of a step issued before the stores
        float *__restrict__ crow = C + int64_t(i) * ldc;
        for (int j = jlo + 4 * int(threadIdx.x); j < jhi && n > 0; j += 4 * int(blockDim.x)) {
          const int4 ev = *reinterpret_cast<const int4 *>(eb + j);
          double t0 = 0.0, t1 = 0.0, t2 = 0.0, t3 = 0.0;
          for (int q = 0; q < n; ++q) {
            const int64_t o = int64_t(ks[q]) * ldbh + j;
            const uint2 h = *reinterpret_cast<const uint2 *>(Bh + o);
            const uint2 l = *reinterpret_cast<const uint2 *>(Bl + o);
            const double d = ds[q];
            t0 = fma(d, rep16(uint16_t(h.x), uint16_t(l.x), ev.x), t0);
            t1 = fma(d, rep16(uint16_t(h.x >> 16), uint16_t(l.x >> 16), ev.y), t1);
            t2 = fma(d, rep16(uint16_t(h.y), uint16_t(l.y), ev.z), t2);
            t3 = fma(d, rep16(uint16_t(h.y >> 16), uint16_t(l.y >> 16), ev.w), t3);
          }
          const float4 c = *reinterpret_cast<const float4 *>(crow + j);
          const float4 v = make_float4(float(double(c.x) + t0), float(double(c.y) + t1),
                                       float(double(c.z) + t2), float(double(c.w) + t3));
          if (peers.mc) {  // the switch writes it into C and every peer's copy
            ptx::multimem_st_v4(peers.mc + int64_t(i) * ldc + j, v);
          } else {
            *reinterpret_cast<float4 *>(crow + j) = v;
            for (int pi = 0; pi < peers.n; ++pi)
              *reinterpret_cast<float4 *>(peers.p[pi] + int64_t(i) * ldc + j) = v;
          }
        }
        __syncthreads();  // the next pass overwrites the staged exceptions
      }
    }
  }
}

// ---- host side ----------------------------------------------------------------------------
static int64_t sms_for_grids() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

// Passes 1-4 of B's preparation into tp (see the kernels above): column maxima, exponents,
// fp16 hi / lo with exception bitmaps, per-strip exception lists.
cudaError_t prep16_b_kernels(const float *B, int64_t ldb, int64_t N, int64_t K,
                             const TermsPrep *tp, cudaStream_t st) {
  const int64_t n_pad = (N + 255) / 256 * 256;
  cudaError_t e = cudaMemsetAsync(tp->bmax, 0, size_t(n_pad) * 4, st);
  if (e == cudaSuccess)  // exception bitmap + column flags (contiguous)
    e = cudaMemsetAsync(tp->xb, 0,
                        size_t(K) * tp->wb * 4 + size_t(tp->wb) * tp->w2b * 4 + size_t(n_pad) * 4,
                        st);
  if (e != cudaSuccess) return e;
  const int64_t bx = (N + 1023) / 1024;
  const int64_t by = std::max<int64_t>(1, std::min<int64_t>((K + 7) / 8,
                                                            int64_t(sms_for_grids()) * 8 / bx));
  const int64_t rows = ((K + by - 1) / by + 7) / 8 * 8;
  const dim3 g1(unsigned(bx), unsigned((K + rows - 1) / rows));
  prep16_bmax_kernel<<<g1, 256, 0, st>>>(B, ldb, int(K), int(N), int(rows), tp->bmax);
  prep16_bexp_kernel<<<unsigned((n_pad + 255) / 256), 256, 0, st>>>(
      tp->bmax, int(n_pad), const_cast<int *>(tp->eb));
  // the same grid as pass 1 (1024-column blocks x row ranges, ~8 blocks per SM)
  // 4 rows in flight per thread at 4 blocks per SM (64 registers): ~15% faster than 8 rows at
  // 2 blocks per SM (latency-bound at 25% occupancy, 4.7 TB/s; ncu A/B at 16384 x 32768)
  auto kern = prep16_b_kernel<4, 4>;
  kern<<<g1, 256, 0, st>>>(B, ldb, int(K), int(N), int(rows), tp->eb,
                                     const_cast<uint16_t *>(tp->Bh), const_cast<uint16_t *>(tp->Bl),
                                     tp->ldbh, tp->xb, tp->sb2, tp->w2b, tp->fb);
  compact16_b_kernel<<<unsigned((tp->wb + 7) / 8), 256, 0, st>>>(
      B, ldb, int(N), int(K), tp->Bh, tp->Bl, tp->ldbh, tp->eb, tp->xb, tp->sb2, tp->w2b, tp->fb,
      tp->bcnt, tp->blist);
  return cudaGetLastError();
}

cudaError_t launch_prep16_a(const float *A, int64_t lda, int64_t M, int64_t K, TermsPrep *tp,
                            cudaStream_t st) {
  const int64_t m_pad = (M + 255) / 256 * 256;
  cudaError_t e = cudaMemsetAsync(
      tp->xa, 0, size_t(M) * tp->wa * 4 + size_t(M) * tp->w2a * 4 + size_t(m_pad) * 4, st);
  if (e != cudaSuccess) return e;
  const int64_t cap = int64_t(sms_for_grids()) * 4;
  if (K >= 8192) {
    prep16_a_kernel<512><<<unsigned(std::min(m_pad, cap)), 512, 0, st>>>(
        A, lda, int(M), int(m_pad), int(K), const_cast<uint16_t *>(tp->Ah),
        const_cast<uint16_t *>(tp->Al), tp->ldah, const_cast<int *>(tp->ea), tp->xa, tp->wa,
        tp->sa2, tp->w2a, tp->fa);
  } else {
    prep16_a_kernel<32><<<unsigned(std::min((m_pad + 15) / 16, cap)), 512, 0, st>>>(
        A, lda, int(M), int(m_pad), int(K), const_cast<uint16_t *>(tp->Ah),
        const_cast<uint16_t *>(tp->Al), tp->ldah, const_cast<int *>(tp->ea), tp->xa, tp->wa,
        tp->sa2, tp->w2a, tp->fa);
  }
  return cudaGetLastError();
}

// The exception fixes of one 3xFP16 launch (after its GEMM, same stream).
cudaError_t launch_fix16(const float *A, int64_t lda, const float *B, int64_t ldb,
                                int64_t M, int64_t N, int64_t K, const TermsPrep *tp, float *C,
                                int64_t ldc, const GemmExtra *ex, cudaStream_t st) {
  PeerC peers;
  peers.n = ex->n_peer_c;
  for (int i = 0; i < peers.n; ++i) peers.p[i] = ex->peer_c[i];
  peers.mc = ex->mc_c;
  // grid-strided rows / strips: blocks of rows or strips without exceptions only read a flag
  const int64_t cap = int64_t(sms_for_grids()) * 4;
  // row windows x column chunks (each flagged row is fixed by gridDim.y blocks side by side)
  const dim3 ga(unsigned(std::min<int64_t>((M + 31) / 32, cap)),
                unsigned(std::max<int64_t>(1, std::min<int64_t>(8, N / 4096))));
  fix16_a_kernel<<<ga, 256, 0, st>>>(
      A, lda, int(M), int(N), tp->Ah, tp->Al, tp->ldah, tp->ea, tp->Bh, tp->Bl, tp->ldbh, tp->eb,
      tp->xa, tp->wa, tp->sa2, tp->w2a, tp->fa, C, ldc, peers);
  return cudaGetLastError();
}

}  // namespace giga
