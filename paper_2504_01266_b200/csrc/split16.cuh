// split16.cuh -- the 3xFP16 scheme's operand split, shared by the GEMM's
// epilogue (gemm_3xtf32.cu) and the preparation / exception kernels (prep16.cu).
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

namespace giga {

constexpr int kBList = 64;  // B exceptions listed per 32-column strip (compact16_b_kernel)

// TF32 is fp16's 11-bit significand with fp32's exponent range. The scheme keeps the
// significand split of 3xTF32 (x = hi + lo, three products, small terms first) on the fp16
// tensor-core path (K = 16 per instruction: twice kind::tf32's K per MMA time) and moves the
// exponent range into exact power-of-two scales: row i of A is scaled by 2^-ea[i], column j
// of B by 2^-eb[j], so that the row / column maximum lies in [2^15, 65504) (fp16's top binade
// below its largest finite value: the higher the scale, the fewer elements sink to fp16's
// subnormal floor);
// the epilogue multiplies C_ij by 2^(ea[i] + eb[j]). hi = fp16 RN(x'), lo = fp16 RN(x' - hi)
// (x' - hi is exact in fp32). For |x'| >= 2^-3, |x' - hi - lo| <= 2^-22 |x'| (both RN to
// 11 bits, or lo at fp16's subnormal floor: 2^-25 absolute in the scaled units); elements far
// below their row's (column's) maximum lose relative precision to that floor.
// An exponent of a row / column with no finite non-zero maximum is 0 (zeros stay exact,
// Inf / NaN propagate as the contract states).
__device__ __forceinline__ int scale_exp(uint32_t maxbits) {
  if (maxbits == 0u || maxbits >= 0x7f800000u) return 0;
  const float m = __uint_as_float(maxbits);
  const int e = ilogbf(m) - 15;  // max' in [2^15, 2^16) ...
  return ldexpf(m, -e) >= 65504.0f ? e + 1 : e;  // ... below fp16's largest finite value
}
// Returns true when x is an *exception*: its representation 2^e (hi + lo) is off by more than
// 2^-20 |x| (elements more than ~2^20 below their row's / column's maximum, where fp16's
// subnormal floor cuts lo). Exceptions are recorded in a bitmap and their remainders added to
// C by fix16_a_kernel (A) and the GEMM epilogue (B: fix_b_list / fix_b_block), so every
// product keeps a split error <= 2 * 2^-20 + 2^-22 relative. In the scaled domain x' - hi and (x' - hi) - lo are exact in fp32; x' itself
// is exact unless it underflows fp32 (then hi = lo = 0 and x != 0 flags it). NaN / Inf are
// never exceptions (the GEMM propagates them).
__device__ __forceinline__ bool split_f16(float x, int e, uint16_t &h, uint16_t &l) {
  // x 2^-e: one multiplication by the power of two when it is a normal float (ldexpf otherwise)
  const float xs = (e >= -126 && e <= 126) ? x * __int_as_float((127 - e) << 23) : ldexpf(x, -e);
  const __half hh = __float2half_rn(xs);
  const float r = __fsub_rn(xs, __half2float(hh));
  const __half ll = __float2half_rn(r);
  h = __half_as_ushort(hh);
  l = __half_as_ushort(ll);
  // |x'| >= 2^-5 is never an exception: lo is normal (error <= 2^-22 |x'|) or on the subnormal
  // grid (error <= 2^-25 <= 2^-20 |x'|); NaN / Inf fail the comparison below as well. Skips
  // the error test for all but the smallest elements (the pass is partly issue-bound).
  if (!(fabsf(xs) < 0x1p-5f)) return false;
  const float err = fabsf(__fsub_rn(r, __half2float(ll)));
  return err > 0x1p-20f * fabsf(xs) || (xs == 0.0f && x != 0.0f);
}
// Exception bitmaps: bit k of row i of A at word i * wa + k / 32; bit j of row k of B at word
// (j / 32) * K + k (strip-major: compact16_b_kernel and fix_b_block read a strip's words
// contiguously). Their summaries
// (one bit per bitmap word) let the fix kernels skip empty stretches; flag arrays: 1 for a row
// of A / column of B holding any exception.
__device__ __forceinline__ void mark_exception(unsigned *bits, int64_t word, unsigned mask,
                                               unsigned *summ, int64_t sword, int sbit,
                                               int *flag) {
  atomicOr(bits + word, mask);
  atomicOr(summ + sword, 1u << sbit);
  *reinterpret_cast<volatile int *>(flag) = 1;
}

// x 2^e in the GEMM epilogue (e = ea[i] + eb[j], in [-328, 224] by scale_exp's range): two
// multiplications by normal powers of two, 2^e1 with e1 = clamp(e, -126, 127), then 2^(e - e1)
// (clamped). Exact whenever x 2^e is a normal float (then no intermediate leaves the normal
// range) -- the bits ldexpf gives -- and a single rounding, as ldexpf's, whenever e1 = e. Only a
// subnormal result with e < -126 can differ from ldexpf, by the second rounding (1 subnormal
// ulp; outside the contract's normal range, reading R16). Below e = -252 both give 0:
// |x| < K 2^32 < 2^63. ~8 instructions where ldexpf took ~45 (measured: the epilogue's
// scaling was a third of the epilogue warps' samples at K = 1024).
__device__ __forceinline__ float pow2_scale(float x, int e) {
  const int e1 = max(-126, min(127, e));
  const int e2 = max(-126, min(127, e - e1));
  return __fmul_rn(__fmul_rn(x, __int_as_float((e1 + 127) << 23)),
                   __int_as_float((e2 + 127) << 23));
}

__device__ __forceinline__ double rep16(uint16_t h, uint16_t l, int e) {
  return ldexp(double(__half2float(__ushort_as_half(h))) + double(__half2float(__ushort_as_half(l))), e);
}

}  // namespace giga
