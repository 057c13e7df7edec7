// gemm_3xtf32.cu -- the shard GEMM of GigaAPI's row-split matrix multiply, sm_100a.
//
// What it computes (S4.2.7): C[i][j] = sum_k A[i][k] * B[k][j] for the
// rows of one shard, every element assigned once at the end ("the total sum being reported
// and assigned at the end of the loop"). The paper's kernel is one scalar thread per C
// element on sm_75 (16x16 blocks PAPER.md:194); this is a B200 design:
//
//   * fp32 accuracy from TF32 tensor cores (BASELINE.json north_star (3)): x = hi + lo with
//     hi = the tensor core's own TF32 reading of the raw fp32 bits (truncation, measured)
//     and lo = x - hi (exact), computed in shared memory from the raw tile each k-block
//     (transform warps; or, GIGA_LO_PRESPLIT=1, TMA-loaded from arrays split_lo_kernel
//     wrote -- twice the operand traffic, kept for comparison). Per 8-wide k step three
//     tcgen05.mma.kind::tf32 are issued into one TMEM accumulator, small terms first:
//     a_lo*b_hi, a_hi*b_lo, a_hi*b_hi (a_lo*b_lo, ~2^-20 relative, is dropped). hi is never
//     materialised: the MMA is fed the raw fp32 tile and reads only its TF32 part.
//   * terms = 2, TF32 + BF16 (the product scheme for large launches): hi = RN
//     tf32(x); a_hi*b_hi is one kind::tf32 MMA and a_lo*b + a_hi*b_lo ONE K=16 kind::f16 MMA
//     over bf16 operands concatenated along K (2 MMA times per k8 step instead of 3). The
//     operands come prepared from HBM (prep_b_kernel / prep_a_kernel, once per launch) and the
//     MMA waits on the TMA barrier directly ("direct" mode, no transform work); the on-chip
//     variants (xform_tf32_bf16) remain for measurements and the no-scratch case.
//   * Accumulator promotion: the tensor core's fp32 accumulation truncates (measured,
//     tests/test_gpu.py::test_probe_accumulation_rounding), so every `p_kb` k-blocks the
//     MMA issuer switches to the other of two TMEM accumulators and the epilogue warps add
//     the finished partial into an fp32 register sum with round-to-nearest adds.
//   * CTA pairs (CG = 2, cta_group::2): a cluster of two CTAs on one TPC computes a
//     256 x 256 tile; each CTA stages its own 128 rows of A and half (128 columns) of B, the
//     leader issues M=256 UMMAs that read both CTAs' shared memory and write both CTAs'
//     TMEM. Per SM this halves the B operand traffic (smem and L2) of the 1-CTA tile.
//     CG = 1 (128 x 256 per CTA) serves small problems.
//   * Warp specialisation, persistent clusters (one CTA per SM, 1 CTA/SM by smem):
//       warp 0 lane 0  TMA producer: raw A tiles (K-major, 64B swizzle) and B tiles
//                      (N-major, 128B/32B-atom swizzle) into a smem ring (mbarriers `full`)
//       warps 10..11   transform: wait `full`, write lo = x - tf32(x) of both tiles next to
//                      them (same swizzled offsets: the map is elementwise), proxy fence,
//                      arrive on the leader's `lofull`
//       warp 1 lane 0  MMA issuer (leader CTA): waits `lofull`, 3 UMMAs per k8;
//                      tcgen05.commit frees smem stages in both CTAs and publishes finished
//                      accumulators
//       warps 2..9     epilogue: tcgen05.ld TMEM -> registers, RN fp32 promotion adds,
//                      swizzled smem staging -> TMA bulk stores (reduce-add when a K-chunked
//                      pipeline accumulates; load-add-store when the last chunk also writes
//                      the peers' C) into the shard's rows of C and, fused gather, the peers'.
//       warp 0 also allocates / frees the TMEM (see the allocation below).
//     Computing lo on chip halves the L2 -> SM operand traffic and the HBM footprint of the
//     3xTF32 operands (measured: 11% less GEMM time at 32768^3 for the same MMAs). The peer
//     CTA publishes its lo tiles to the leader's MMA with an async-proxy bulk signal
//     (ptx::bulk_signal_leader): a release.cluster arrive per k-block cost 40%.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <list>
#include <mutex>
#include <vector>

#include "kernels.h"
#include "ptx.cuh"
#include "split16.cuh"

namespace giga {

namespace cfg {
constexpr int BM = 128;  // rows of A per CTA (UMMA M per CTA)
constexpr int BN = 256;  // UMMA N: columns of the tile (a CTA pair stages 128 each)
constexpr int BK = 16;   // k-block: two k8 UMMA steps
constexpr int NUM_EPI_WARPS = 8;
constexpr int NUM_XFORM_WARPS = 2;
constexpr int XFORM_WARP0 = 2 + NUM_EPI_WARPS;
constexpr int NUM_THREADS = 64 + NUM_EPI_WARPS * 32 + NUM_XFORM_WARPS * 32;
constexpr uint32_t A_BYTES = BM * BK * 4;        // 8 KiB: 128 rows x 64 B
constexpr uint32_t B_CHUNK_BYTES = BK * 32 * 4;  // 2 KiB: one 32-column chunk of B
constexpr uint32_t ACC_COLS = BN;                // fp32 accumulator: 1 TMEM column per n
constexpr uint32_t TMEM_COLS = 2 * ACC_COLS;     // two accumulators (promotion ping-pong)
constexpr int GROUP_M = 8;                       // L2 raster: default M-tiles per group
constexpr size_t SMEM_RING = 192 * 1024;         // operand ring per CTA
constexpr uint32_t EPI_STAGE_BYTES = 32 * 32 * 4;  // per epilogue warp: 32 rows x 32 fp32
constexpr uint32_t EPI_BYTES = NUM_EPI_WARPS * EPI_STAGE_BYTES;  // 32 KiB C staging
constexpr size_t EPI_SLOT_BYTES = 32 * 128 * 4;  // K-split partial of one epilogue warp
constexpr int SCHED_SLOTS = 8;                   // ring of claimed work units (power of 2)
}  // namespace cfg

template <int CG>
struct Tile {
  static constexpr int TILE_M = cfg::BM * CG;                    // rows per cluster tile
  static constexpr int B_COLS = cfg::BN / CG;                    // B columns this CTA stages
  static constexpr uint32_t B_BYTES = cfg::BK * B_COLS * 4;      // per operand per CTA
  static constexpr uint32_t STAGE_BYTES = 2 * cfg::A_BYTES + 2 * B_BYTES;
  static constexpr int STAGES = int(cfg::SMEM_RING / STAGE_BYTES);  // 4 (CG=1), 6 (CG=2)
  static constexpr size_t SMEM_BYTES =
      size_t(STAGES) * STAGE_BYTES + cfg::EPI_BYTES + 1024 + 512;
};

struct GemmParams {
  int M, N, K, ldc;
  int accumulate; // 1: C += A*B (K-chunked pipelines), 0: C = A*B
  int load_c;     // 1: epilogue adds the block's current C before storing (see GemmExtra)
  int terms;      // 3 = 3xTF32, 2 = TF32 hi*hi + one BF16 correction MMA, 1 = TF32 hi*hi only
  int p_kb;       // k-blocks per TMEM accumulation interval (>= 1)
  int n_kb;       // k-blocks per tile
  int m_tiles, n_tiles, num_tiles;
  // K-split units (deterministic; plan_ksplit): tiles [0, first_split) run whole; each tile
  // t >= first_split runs as `split_s` units over consecutive k-block ranges, combined by
  // split_mode. kSplitWorkspace: a part's epilogue writes its fp32 partial to the workspace
  // slot of (tile, part) and counts itself in; the last part to arrive sums the tile's parts
  // in part order (p0 + p1 + ...: the same bits whichever part arrives last) and stores the
  // tile like a whole one. num_units = first_split + (num_tiles - first_split) * split_s.
  int first_split, split_s, num_units;
  int split_mode;   // kSplitReduce: parts TMA reduce-add into C zeroed before the launch
                    // (s = 2: 0 + a + b is order-independent); kSplitWorkspace: as above
  float *sk_ws;     // (num_tiles - first_split) * split_s * CG * 8 slots of 32 x 128 fp32
  unsigned *sk_cnt; // (num_tiles - first_split) * CG * 8 arrival counters, 0 between launches
  int group_m;    // L2 raster: consecutive tiles walk group_m M-tiles before the next N-tile
  // Dynamic schedule (per-stream counters, zero between launches; the last CTA to finish
  // resets them): sched[0] = next unit to claim, sched[1] = units whose loads a CTA has
  // issued (the producers' wave barrier), sched[2] = CTAs finished. nullptr: static
  // round-robin units, no wave barrier (no counters could be had, e.g. inside a capture).
  unsigned *sched;
  int wave_sync;  // s >= 1: a producer starts unit u's loads once every unit of waves
                  // <= wave(u) - s (wave = u / clusters) has been issued by all its CTAs
                  // (s = 1: every earlier wave); 0: no barrier
  int n_cdst;     // C destinations in CMaps (1 + peers when the gather is fused)
  // how the epilogue writes C: kStoreTma (CMaps), kStoreVec (16-byte st.global to vdst[0..
  // n_cdst)), kStoreMulticast (multimem.st to the team address vdst[0]; n_cdst = 1)
  int st_mode;
  float *vdst[kMaxCDst];
  int lo_smem;    // 1: lo tiles computed in smem from the raw tiles; 0: TMA-loaded (A_lo, B_lo)
  int hi_rn;      // terms == 2: hi = RN tf32(x) written over the raw tile (else hi = trunc)
  int b_pre;      // terms == 2: B_hi and B' precomputed in HBM by prep_b_kernel (TMA-loaded
                  // through tmB / tmBlo); the transform warps handle A only
  int a_pre;      // terms == 2 (with b_pre): A_hi and A' precomputed too (tmA / tmAlo); no
                  // transform work in the kernel
  // terms == 4 (3xFP16): the accumulator holds sum_k a'_ik b'_kj of the scaled operands
  // a' = a 2^-ea[i], b' = b 2^-eb[j]; the epilogue stores ldexp(sum, ea[i] + eb[j])
  const int *ea, *eb;
  // ... and adds sum_k a_ik (b_kj - rep(b_kj)) for the exceptions of B in its columns (fused
  // B-side fix; nullptr xb: none): the original A / B, the fp16 B_hi / B_lo, B's exception
  // bitmap (strip-major), its summary and the per-column flags
  const float *fA, *fB;
  int64_t flda, fldb, fldbh;
  const uint16_t *fBh, *fBl;
  const unsigned *xb, *sb2;
  const int *fb;
  int w2b;
  // per strip of 32 columns: the number of B exceptions and (up to kBList of them) the list
  // (k, column in the strip, b - rep(b) as fp64 halves) in column-then-k order (compact16_b)
  const int *bcnt;
  const int4 *blist;
  uint64_t *cta_ns;  // $GIGA_TRACE: [2 blockIdx.x] = this CTA's start, [+1] = its end (ns)
};

enum { kStoreTma = 0, kStoreVec = 1, kStoreMulticast = 2 };

// C tensor maps: [0] this GPU's C, [1..] the same rows of the peers' C_full buffers.
struct CMaps {
  CUtensorMap m[kMaxCDst];
};

// ---- UMMA descriptors -------------------------------------------------------------------
// Shared-memory matrix descriptor (sm100, "version 1"):
//   [0,14) start address >> 4   [16,30) leading byte offset >> 4   [32,46) stride byte
//   offset >> 4   [46,48) version = 1   [49,52) base offset = 0   [52] lbo mode = 0
//   [61,64) layout: 1 = SWIZZLE_128B_BASE32B, 2 = SWIZZLE_128B, 4 = SWIZZLE_64B
// A (K-major, SW64): rows of 64 B (16 fp32 of K), 8-row atoms of 512 B -> SBO = 512; LBO is
//   unused for swizzled K-major (1). The k8 step j starts 32 B further into the row.
// B (N-major): for 32-bit MN-major operands the only UMMA layout is SWIZZLE_128B_BASE32B
//   (32-byte granules XOR-swizzled inside 128-byte rows with a 4-row period; TMA mode
//   128B_ATOM_32B). Rows of 128 B = 32 n, one row per k; 4-row k-groups 512 B apart -> SBO;
//   32-column chunks 2 KiB apart -> LBO = 2048. The k8 step j starts j * 1024 B further.
//   (Measured on B200 with scripts/debug_umma.py: plain SWIZZLE_128B N-major tf32 yields 0.)
__device__ __forceinline__ uint64_t make_sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                               uint32_t layout) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFF);
  d |= uint64_t((lbo >> 4) & 0x3FFF) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFF) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(layout & 7) << 61;
  return d;
}
// Instruction descriptor, kind::tf32: [4,6) D fmt = 1 (F32); [7,10) A fmt = 2 (TF32);
// [10,13) B fmt = 2 (TF32); [15] A major = 0 (K); [16] B major = 1 (MN); [17,23) N >> 3;
// [24,29) M >> 4.
__host__ __device__ constexpr uint32_t make_idesc(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | (1u << 16) |
         (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}
// Instruction descriptor, kind::f16 with BF16 A and B (format 1), F32 D; A K-major, B
// MN-major (the correction tiles of the TF32 + BF16 scheme, below).
__host__ __device__ constexpr uint32_t make_idesc_bf16(int m, int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (0u << 15) | (1u << 16) |
         (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}

// Instruction descriptor, kind::f16 with FP16 A and B (format 0), F32 D; A K-major, B MN-major
// (the three products of the 3xFP16 scheme).
__host__ __device__ constexpr uint32_t make_idesc_f16(int m, int n) {
  return (1u << 4) | (0u << 7) | (0u << 10) | (0u << 15) | (1u << 16) |
         (uint32_t(n >> 3) << 17) | (uint32_t(m >> 4) << 24);
}

// The B-side exception fix of one 32 x 32 block of C from its strip's exception list (the
// common path): lanes (= rows of C) read the list entries by broadcast, sum a_ik d_kj in fp64
// per column in ascending k (4 entries' A loads in flight at a time) and add each column's sum,
// rounded once, to the staged value.
__device__ __forceinline__ void fix_b_list(const GemmParams &p, float *stg, int row, int strip,
                                           int cnt, int lane) {
  const int4 *Lst = p.blist + int64_t(strip) * kBList;
  const bool live = row < p.M;
  const float *arow = p.fA + int64_t(live ? row : 0) * p.flda;
  int cur = -1;
  double t = 0.0;
  for (int q0 = 0; q0 < cnt; q0 += 4) {
    int4 en[4];
    float av[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) en[u] = q0 + u < cnt ? Lst[q0 + u] : make_int4(0, -1, 0, 0);
#pragma unroll
    for (int u = 0; u < 4; ++u) av[u] = (live && q0 + u < cnt) ? arow[en[u].x] : 0.0f;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (q0 + u >= cnt) break;
      if (en[u].y != cur) {
        if (cur >= 0) {
          float *v = stg + lane * 32 + (((cur >> 2) ^ (lane & 7)) << 2) + (cur & 3);
          *v = float(double(*v) + t);
        }
        cur = en[u].y;
        t = 0.0;
      }
      t = fma(double(av[u]), __hiloint2double(en[u].w, en[u].z), t);
    }
  }
  if (cur >= 0) {
    float *v = stg + lane * 32 + (((cur >> 2) ^ (lane & 7)) << 2) + (cur & 3);
    *v = float(double(*v) + t);
  }
}

// The B-side exception fix of one 32 x 32 block of C in the epilogue's staging tile (3xFP16),
// by scanning the strip's bitmap (strips whose list overflowed kBList: pathological inputs):
// for each column of the block (a strip of B) flagged with exceptions, every lane (= one row
// of C) sums a_ik (b_kj - rep(b_kj)) in fp64 over the column's exceptions in ascending k and
// adds it, rounded once, to its staged value. Columns without exceptions cost one flag read
// per block; the common case (uniform data: ~1e-6 of B's elements) touches nothing else.
__device__ __forceinline__ void fix_b_block(const GemmParams &p, float *stg, int row, int col0,
                                         int lane) {
  const int j = col0 + lane;
  unsigned cols = __ballot_sync(0xffffffffu, j < p.N && p.fb[j] != 0);
  if (!cols) return;
  const int strip = col0 >> 5;
  const unsigned *S = p.sb2 + int64_t(strip) * p.w2b;
  const unsigned *L = p.xb + int64_t(strip) * p.K;
  const bool live = row < p.M;
  while (cols) {
    const int jb = __ffs(cols) - 1;
    cols &= cols - 1;
    const int jj = col0 + jb;
    const int e = p.eb[jj];
    double t = 0.0;
    for (int c0 = 0; c0 < p.w2b; c0 += 32) {
      const unsigned sw = c0 + lane < p.w2b ? S[c0 + lane] : 0u;
      unsigned nz = __ballot_sync(0xffffffffu, sw != 0u);
      while (nz) {
        const int src = __ffs(nz) - 1;
        nz &= nz - 1;
        const unsigned swv = __shfl_sync(0xffffffffu, sw, src);
        const int k = (c0 + src) * 32 + lane;
        const bool hit = ((swv >> lane) & 1u) && k < p.K && ((L[k] >> jb) & 1u);
        unsigned hits = __ballot_sync(0xffffffffu, hit);
        while (hits) {
          const int q = __ffs(hits) - 1;
          hits &= hits - 1;
          const int kk = (c0 + src) * 32 + q;
          const int64_t o = int64_t(kk) * p.fldbh + jj;
          const double rb =
              ldexp(double(__half2float(__ushort_as_half(p.fBh[o]))) +
                        double(__half2float(__ushort_as_half(p.fBl[o]))), e);
          const double d = double(p.fB[int64_t(kk) * p.fldb + jj]) - rb;
          if (live) t = fma(double(p.fA[int64_t(row) * p.flda + kk]), d, t);
        }
      }
    }
    // staging tile: row `lane`, 16-byte chunk (jb / 4) ^ (lane & 7), 128-byte rows
    float *v = stg + lane * 32 + (((jb >> 2) ^ (lane & 7)) << 2) + (jb & 3);
    *v = float(double(*v) + t);
  }
}

// The staged 32 x 32 block (rows row0.., columns col0..) written with 16-byte stores instead of
// the TMA unit (kStoreVec: to C and every peer; kStoreMulticast: once, to the team address,
// which the NVSwitch replicates into every GPU's C_full -- DESIGN.md 7, "Multicast gather").
// Each 8-lane group writes one 128-byte row segment per instruction (4 rows per warp store,
// coalesced), reading the staging tile's swizzled chunks (chunk j of row r at j ^ (r & 7):
// conflict-free). Rows >= M and columns >= N are clipped here (N % 4 == 0: a chunk is all in
// or all out).
__device__ __forceinline__ void vec_store_block(const GemmParams &p, uint32_t stg, int row0,
                                                int col0, int lane) {
  const int col = col0 + 4 * (lane & 7);
#pragma unroll 1
  for (int i = 0; i < 8; ++i) {  // (not unrolled: the epilogue's registers hold the sums)
    const int r = 4 * i + (lane >> 3);
    const float4 v =
        ptx::ld_shared_v4(stg + uint32_t(r) * 128 + uint32_t(((lane & 7) ^ (r & 7)) * 16));
    if (row0 + r < p.M && col < p.N) {
      const int64_t off = int64_t(row0 + r) * p.ldc + col;
      if (p.st_mode == kStoreMulticast) {
        ptx::multimem_st_v4(p.vdst[0] + off, v);
      } else {
        for (int d = 0; d < p.n_cdst; ++d) ptx::st_global_v4(p.vdst[d] + off, v);
      }
    }
  }
}

// ---- split: lo = x - tf32(x) ------------------------------------------------------------
// tf32(x) is what kind::tf32 reads from raw fp32 bits: the top 19 bits (sign, exponent,
// 10 mantissa bits), i.e. truncation toward zero of the low 13 mantissa bits (measured on
// B200 by tests/test_gpu.py::test_probe_tf32_operand_conversion_is_truncation). x - tf32(x)
// is exact in fp32 (same sign, the 13 low bits of x's significand).
__device__ __forceinline__ float tf32_lo(float x) {
  const float hi = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
  return __fsub_rn(x, hi);
}

__host__ __device__ __forceinline__ void tile_coords(int t, const GemmParams &p, int &mb,
                                                    int &nb) {
  const int group_size = p.group_m * p.n_tiles;
  const int g = t / group_size;
  const int first_m = g * p.group_m;
  const int gm = min(p.group_m, p.m_tiles - first_m);
  const int local = t - g * group_size;
  mb = first_m + local % gm;
  nb = local / gm;
}

// Work unit u -> tile t and k-block range [kb0, kb1); part = -1 for a whole tile, else the
// unit's index among its tile's split_s parts (consecutive units: they run side by side).
__host__ __device__ __forceinline__ void unit_coords(int u, const GemmParams &p, int &t,
                                                    int &kb0, int &kb1, int &part) {
  if (u < p.first_split) {
    t = u;
    kb0 = 0;
    kb1 = p.n_kb;
    part = -1;
    return;
  }
  const int v = u - p.first_split;
  t = p.first_split + v / p.split_s;
  part = v % p.split_s;
  kb0 = int(int64_t(p.n_kb) * part / p.split_s);
  kb1 = int(int64_t(p.n_kb) * (part + 1) / p.split_s);
}

// ---- TF32 + BF16 scheme (terms == 2) -------------------------------------------------------
// x = hi + lo with hi = tf32(x) (RN, written over the raw tile when hi_rn, else the MMA's own
// truncation) and lo = x - hi exact. a*b = a_hi*b_hi + a_lo*b + a_hi*b_lo exactly; the first
// product is one kind::tf32 MMA (exact products), the two corrections, each ~2^-11 of a*b,
// are ONE kind::f16 MMA with K = 16 over bf16 operands concatenated along K:
//   A' row  = [bf16(a_lo[k0..k7]) | bf16(a_hi[k0..k7])]           (K-major, SW64, 64 B rows)
//   B' rows = [bf16(b[k0..k7][n]) ; bf16(b_lo[k0..k7][n])]         (MN-major, SW128)
// bf16 keeps 8 significant bits (unit roundoff 2^-8). With RN hi, |lo| <= 2^-11 |x|, and per
// product the four roundings cost at most 2^-8 |a_lo||b| <= 2^-19 |a||b| (b), 2^-20 |a||b|
// (a_lo: its exponent is <= that of a minus 12), 2^-19 (a_hi) and 2^-20 (b_lo): |error| <=
// 3 * 2^-19 |a||b| = 5.7e-6 plus O(2^-27); constructed inputs reach 5.3e-6
// (tests/adversarial.py). Truncated hi (|lo| < 2^-10 |x|) doubles the lo terms: ~3 * 2^-18,
// above the 1e-5 bound, so the product path rounds hi to nearest. A bf16 K16 MMA takes the
// time of a tf32 K8 MMA, so a k8 step costs 2 MMA times instead of 3xTF32's 3.
// Layouts written here (stage = [A raw | A' | B raw | B']):
//   A raw: TMA SW64, 128 rows x 64 B, 16-B chunk c of row r at r*64 + ((c ^ (r>>1 & 3)) << 4).
//     A' has the same geometry: chunk 2h (2h+1) of row r = bf16 lo (hi) of k8 step h.
//   B raw: TMA 128B_ATOM_32B, 32-column chunks of 16 k-rows x 128 B; the 32-B granule g of
//     row k sits at k*128 + ((g ^ (k & 3)) << 5).
//   B': 64-column chunks of 32 rows x 128 B (k8 step j: rows 16j..16j+7 = bf16(b[k]),
//     16j+8.. = bf16(b_lo[k])); 16-B chunk c (8 columns) of row q at q*128 + ((c ^ (q&7)) << 4).
// Thread mapping keeps every 8-lane phase of each 16-B access on distinct bank groups.
// RN (ties away from zero) in two integer ops: add half a TF32 ulp to the magnitude bits, then
// truncate; a carry into the exponent is the correct rounding up to the next binade (cvt.rna
// compiles to a longer sequence on sm_100: 216 -> 233 TFLOP/s in a 4-transform-warp build).
// NaN stays NaN in lo = x - hi.
__device__ __forceinline__ float tf32_hi(float x, int rn) {
  const uint32_t b = __float_as_uint(x);
  return __uint_as_float((rn ? b + 0x1000u : b) & 0xFFFFE000u);
}

template <int CG, bool B_PRE>
__device__ __forceinline__ void xform_tf32_bf16(uint32_t sA, int xt, int rn) {
  using namespace cfg;
  using T = Tile<CG>;
  constexpr int NT = NUM_XFORM_WARPS * 32;
  const uint32_t sAx = sA + A_BYTES, sB = sA + 2 * A_BYTES, sBx = sB + T::B_BYTES;
  // A: units (row r, k8 step h); lanes of a warp take 32 consecutive rows
  constexpr int UA = 2 * BM / NT;  // 4
  float4 xa[UA][2];
#pragma unroll
  for (int i = 0; i < UA; ++i) {
    const int u = i * NT + xt, r = u & (BM - 1), h = u / BM;
    const uint32_t sw = uint32_t(r >> 1) & 3, row = sA + uint32_t(r) * 64;
    xa[i][0] = ptx::ld_shared_v4(row + ((uint32_t(2 * h) ^ sw) << 4));
    xa[i][1] = ptx::ld_shared_v4(row + ((uint32_t(2 * h + 1) ^ sw) << 4));
  }
  // B: units (k-row k, 8-column granule); 8 consecutive lanes cover 64 columns of one row
  constexpr int UB = B_PRE ? 0 : (T::B_COLS / 8) * BK / NT;  // 4 (CG = 2), 8 (CG = 1)
  float4 xb[UB > 0 ? UB : 1][2];
#pragma unroll
  for (int i = 0; i < UB; ++i) {
    const int u = i * NT + xt, g8 = u & 7, k = (u >> 3) & (BK - 1), nch = u >> 7;
    const uint32_t gaddr = sB + uint32_t(2 * nch + (g8 >> 2)) * B_CHUNK_BYTES + uint32_t(k) * 128 +
                           ((uint32_t(g8 & 3) ^ uint32_t(k & 3)) << 5);
    // lanes of the second 32-column chunk read their granule's halves in the other order:
    // the two chunks are 2 KiB apart (same banks)
    const uint32_t q = uint32_t(g8 >> 2) << 4;
    const float4 p0 = ptx::ld_shared_v4(gaddr + q), p1 = ptx::ld_shared_v4(gaddr + (q ^ 16));
    xb[i][0] = q ? p1 : p0;
    xb[i][1] = q ? p0 : p1;
  }
#pragma unroll
  for (int i = 0; i < UA; ++i) {
    const int u = i * NT + xt, r = u & (BM - 1), h = u / BM;
    const uint32_t sw = uint32_t(r >> 1) & 3;
    const uint32_t o0 = uint32_t(r) * 64 + ((uint32_t(2 * h) ^ sw) << 4);
    const uint32_t o1 = uint32_t(r) * 64 + ((uint32_t(2 * h + 1) ^ sw) << 4);
    const float v[8] = {xa[i][0].x, xa[i][0].y, xa[i][0].z, xa[i][0].w,
                        xa[i][1].x, xa[i][1].y, xa[i][1].z, xa[i][1].w};
    float hi[8], lo[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      hi[j] = tf32_hi(v[j], rn);
      lo[j] = __fsub_rn(v[j], hi[j]);
    }
    ptx::st_shared_v4_u32(sAx + o0, ptx::pack_bf16x2(lo[0], lo[1]), ptx::pack_bf16x2(lo[2], lo[3]),
                          ptx::pack_bf16x2(lo[4], lo[5]), ptx::pack_bf16x2(lo[6], lo[7]));
    ptx::st_shared_v4_u32(sAx + o1, ptx::pack_bf16x2(hi[0], hi[1]), ptx::pack_bf16x2(hi[2], hi[3]),
                          ptx::pack_bf16x2(hi[4], hi[5]), ptx::pack_bf16x2(hi[6], hi[7]));
    if (rn) {
      ptx::st_shared_v4(sA + o0, hi[0], hi[1], hi[2], hi[3]);
      ptx::st_shared_v4(sA + o1, hi[4], hi[5], hi[6], hi[7]);
    }
  }
#pragma unroll
  for (int i = 0; i < UB; ++i) {
    const int u = i * NT + xt, g8 = u & 7, k = (u >> 3) & (BK - 1), nch = u >> 7;
    const float v[8] = {xb[i][0].x, xb[i][0].y, xb[i][0].z, xb[i][0].w,
                        xb[i][1].x, xb[i][1].y, xb[i][1].z, xb[i][1].w};
    float hi[8], lo[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      hi[j] = tf32_hi(v[j], rn);
      lo[j] = __fsub_rn(v[j], hi[j]);
    }
    const uint32_t kk = uint32_t(k & 7), chunk = (uint32_t(g8) ^ kk) << 4;
    const uint32_t base = sBx + uint32_t(nch) * 4096 + uint32_t(k >> 3) * 2048;
    ptx::st_shared_v4_u32(base + kk * 128 + chunk, ptx::pack_bf16x2(v[0], v[1]),
                          ptx::pack_bf16x2(v[2], v[3]), ptx::pack_bf16x2(v[4], v[5]),
                          ptx::pack_bf16x2(v[6], v[7]));
    ptx::st_shared_v4_u32(base + (8 + kk) * 128 + chunk, ptx::pack_bf16x2(lo[0], lo[1]),
                          ptx::pack_bf16x2(lo[2], lo[3]), ptx::pack_bf16x2(lo[4], lo[5]),
                          ptx::pack_bf16x2(lo[6], lo[7]));
    if (rn) {
      const uint32_t gaddr = sB + uint32_t(2 * nch + (g8 >> 2)) * B_CHUNK_BYTES +
                             uint32_t(k) * 128 + ((uint32_t(g8 & 3) ^ uint32_t(k & 3)) << 5);
      ptx::st_shared_v4(gaddr, hi[0], hi[1], hi[2], hi[3]);
      ptx::st_shared_v4(gaddr + 16, hi[4], hi[5], hi[6], hi[7]);
    }
  }
}

// Consumer side of the claimed-unit ring: wait for the unit of ring position `it`, read it,
// release the slot on the leader's sched_empty (one arrive per consuming warp: lane 0, after
// the whole warp has read the slot; or a lone thread). Returns the unit, -1 = no more work.
template <int CG>
__device__ __forceinline__ int sched_take(int it, uint64_t *sched_full, uint64_t *sched_empty,
                                          uint32_t sempty_leader, volatile int *ring,
                                          bool whole_warp) {
  const int slot = it & (cfg::SCHED_SLOTS - 1);
  const uint32_t ph = uint32_t(it / cfg::SCHED_SLOTS) & 1;
  if (CG == 2)
    ptx::mbar_wait_cluster(&sched_full[slot], ph);  // the leader published it remotely
  else
    ptx::mbar_wait(&sched_full[slot], ph);
  const int u = ring[slot];
  if (whole_warp) __syncwarp();
  if (!whole_warp || (threadIdx.x & 31) == 0) {
    if (CG == 2)
      ptx::mbar_arrive_cluster(sempty_leader + 8u * uint32_t(slot));
    else
      ptx::mbar_arrive(&sched_empty[slot]);
  }
  return u;
}

template <int CG>
__global__ void __launch_bounds__(cfg::NUM_THREADS, 1)
    gemm_3xtf32_kernel(const __grid_constant__ CUtensorMap tmA,
                       const __grid_constant__ CUtensorMap tmAlo,
                       const __grid_constant__ CUtensorMap tmB,
                       const __grid_constant__ CUtensorMap tmBlo,
                       const __grid_constant__ CMaps cmaps, const GemmParams p) {
  using namespace cfg;
  using T = Tile<CG>;
  constexpr int STAGES = T::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *epi_stage = smem + STAGES * T::STAGE_BYTES;  // C staging for the TMA stores
  uint64_t *full = reinterpret_cast<uint64_t *>(epi_stage + EPI_BYTES);
  uint64_t *empty = full + STAGES;
  uint64_t *tfull = empty + STAGES;
  uint64_t *tempty = tfull + 2;
  uint64_t *lofull = tempty + 2;  // stage ready for the MMA: raw + lo tiles of both CTAs
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(lofull + STAGES);
  uint8_t *sig = reinterpret_cast<uint8_t *>(lofull + STAGES) + 16;  // 16 B aligned, 32 B
  uint64_t *cbar = reinterpret_cast<uint64_t *>(sig + 32);  // per epilogue warp: C block loads
  // claimed-unit ring: the leader's producer claims a unit and publishes it to every consumer
  // warp of both CTAs (sched_full); they release the slot on the leader's sched_empty
  uint64_t *sched_full = cbar + NUM_EPI_WARPS;
  uint64_t *sched_empty = sched_full + SCHED_SLOTS;
  volatile int *sched_ring = reinterpret_cast<volatile int *>(sched_empty + SCHED_SLOTS);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  if (p.cta_ns && threadIdx.x == 0) p.cta_ns[2 * blockIdx.x] = ptx::globaltimer_ns();
  const uint32_t rank = CG == 2 ? ptx::cluster_ctarank() : 0;  // rank in the CTA pair
  const bool leader = rank == 0;
  const int cluster_id = blockIdx.x / CG;
  const int num_clusters = gridDim.x / CG;
  // TF32 + BF16 with both operands prepared in HBM: no transform, the MMA waits on `full`
  // (and the 3xFP16 scheme, whose fp16 hi / lo operands always come prepared)
  const bool direct = (p.terms == 2 && p.a_pre && p.b_pre) || p.terms == 4;

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    if ((p.terms == 3 && !p.lo_smem) || p.terms == 4) {
      ptx::prefetch_tmap(&tmAlo);
      ptx::prefetch_tmap(&tmBlo);
    }
    for (int dst = 0; dst < p.n_cdst; ++dst) ptx::prefetch_tmap(&cmaps.m[dst]);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
      ptx::mbar_init(&lofull[s], NUM_XFORM_WARPS);
    }
    for (int w = 0; w < NUM_EPI_WARPS; ++w) ptx::mbar_init(&cbar[w], 1);
    // consumers of a claimed unit: every epilogue (and, unless direct, transform) warp of both
    // CTAs, the MMA issuer and the peer's producer
    const uint32_t n_cons =
        uint32_t(CG * (NUM_EPI_WARPS + (direct ? 0 : NUM_XFORM_WARPS)) + 1 + (CG == 2 ? 1 : 0));
    for (int q = 0; q < SCHED_SLOTS; ++q) {
      ptx::mbar_init(&sched_full[q], 1);
      ptx::mbar_init(&sched_empty[q], n_cons);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull[b], 1);
      ptx::mbar_init(&tempty[b], NUM_EPI_WARPS * CG);
    }
    ptx::fence_mbar_init();
  }
  // TMEM allocation by warp 0: with cta_group::2 the allocation handshakes with the peer
  // through a barrier in reserved shared memory (0x58) that racecheck sees written by warp 0
  // (lane 31, outside this kernel's code); allocating from another warp ran correctly but was
  // reported as a RAW hazard on that barrier.
  if (warp == 0) {
    __syncwarp();
    if (CG == 2)
      ptx::tmem_alloc_cg2(tmem_slot, TMEM_COLS);
    else
      ptx::tmem_alloc(tmem_slot, TMEM_COLS);
  }
  ptx::tc_fence_before();
  if (CG == 2)
    ptx::cluster_sync();  // peer barriers initialised before any remote arrive / TMA
  else
    __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ======================= TMA producer (both CTAs) =======================
    if (lane == 0) {
      const bool load_lo = p.terms == 3 && !p.lo_smem;
      const bool load_bx = p.terms == 2 && p.b_pre;
      const bool load_ax = (load_bx && p.a_pre) || p.terms == 4;
      const uint32_t tx_cta = (load_lo || load_ax) ? T::STAGE_BYTES
                              : load_bx ? (A_BYTES + 2 * T::B_BYTES)
                                        : (A_BYTES + T::B_BYTES);
      int stage = 0;
      uint32_t phase = 0;
      const uint32_t ring_peer = CG == 2 ? ptx::map_cluster((const void *)sched_ring, 1) : 0;
      const uint32_t sfull_peer = CG == 2 ? ptx::map_cluster(&sched_full[0], 1) : 0;
      const uint32_t sempty_leader = ptx::smem_u32(&sched_empty[0]) & ptx::kPeerBitMask;
      for (int it = 0;; ++it) {
        // Work units are claimed dynamically (an atomic counter, in unit order) by the running
        // clusters, so a cluster that another kernel keeps off the GPU (NCCL's CTAs, a
        // co-running GEMM) takes no units at all instead of owning every num_clusters-th one
        // the others would wait for. The leader's producer claims and publishes the unit to
        // every consumer warp of both CTAs through the ring.
        int u;
        const int slot = it & (SCHED_SLOTS - 1);
        const uint32_t sph = uint32_t(it / SCHED_SLOTS) & 1;
        if (leader) {
          if (it >= SCHED_SLOTS) ptx::mbar_wait_cluster(&sched_empty[slot], sph ^ 1);
          u = p.sched ? int(atomicAdd(&p.sched[0], 1u)) : cluster_id + it * num_clusters;
          if (u >= p.num_units) u = -1;
          sched_ring[slot] = u;
          if (CG == 2) {
            ptx::st_cluster_u32(ring_peer + 4u * uint32_t(slot), uint32_t(u));
            ptx::mbar_arrive_cluster(sfull_peer + 8u * uint32_t(slot));
          }
          ptx::mbar_arrive(&sched_full[slot]);
        } else {
          u = sched_take<CG>(it, sched_full, sched_empty, sempty_leader, sched_ring, false);
        }
        if (u < 0) break;
        const int wave = u / num_clusters;
        if (p.sched && p.wave_sync && wave >= p.wave_sync) {
          // Wave barrier among the producers: start loading unit u only when every unit of
          // the earlier waves has been issued by all its CTAs, so the clusters sharing A / B
          // panels stay within about one tile of each other and hit in L2 (unsynchronised,
          // persistent clusters drift apart and re-fetch panels from HBM: 147 -> 35 GB of
          // DRAM reads at 16384^3). Deadlock-free: units are claimed in increasing order, only
          // by running clusters, and the loads of a claimed unit wait for nothing but earlier
          // units. The 2 ms cap only bounds a locality hint (never needed for correctness).
          const uint32_t target =
              uint32_t(CG) * uint32_t(wave + 1 - p.wave_sync) * uint32_t(num_clusters);
          const uint64_t t_start = ptx::globaltimer_ns();
          while (ptx::ld_acquire_gpu(&p.sched[1]) < target &&
                 ptx::globaltimer_ns() - t_start < 2000000ull)
            __nanosleep(64);
        }
        int t, kb0, kb1, mb, nb, part;
        unit_coords(u, p, t, kb0, kb1, part);
        tile_coords(t, p, mb, nb);
        const int m0 = mb * T::TILE_M + int(rank) * BM;
        const int n0 = nb * BN + int(rank) * T::B_COLS;
        for (int kb = kb0; kb < kb1; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t *sA = smem + stage * T::STAGE_BYTES;
          uint8_t *sAlo = sA + A_BYTES;
          uint8_t *sB = sA + 2 * A_BYTES;
          uint8_t *sBlo = sB + T::B_BYTES;
          const int k0 = kb * BK;
          if (p.terms == 4) {
            // 3xFP16: k-blocks of 32; A_hi / A_lo fp16 K-major boxes {32, 128} (64 B rows,
            // SW64), B_hi / B_lo fp16 N-major boxes {64, 32} (128 B rows, SW128): the same
            // geometry as A' / B' of the TF32 + BF16 scheme
            const int k32 = kb * 32;
            if (CG == 1) {
              ptx::mbar_expect_tx(&full[stage], tx_cta);
              ptx::tma_load_2d(sA, &tmA, &full[stage], k32, m0);
              ptx::tma_load_2d(sAlo, &tmAlo, &full[stage], k32, m0);
#pragma unroll
              for (int c = 0; c < T::B_COLS / 64; ++c) {
                ptx::tma_load_2d(sB + c * 4096, &tmB, &full[stage], n0 + 64 * c, k32);
                ptx::tma_load_2d(sBlo + c * 4096, &tmBlo, &full[stage], n0 + 64 * c, k32);
              }
            } else {
              const uint32_t fb = ptx::smem_u32(&full[stage]) & ptx::kPeerBitMask;
              if (leader) ptx::mbar_expect_tx(&full[stage], 2 * tx_cta);
              ptx::tma_load_2d_cg2(sA, &tmA, fb, k32, m0);
              ptx::tma_load_2d_cg2(sAlo, &tmAlo, fb, k32, m0);
#pragma unroll
              for (int c = 0; c < T::B_COLS / 64; ++c) {
                ptx::tma_load_2d_cg2(sB + c * 4096, &tmB, fb, n0 + 64 * c, k32);
                ptx::tma_load_2d_cg2(sBlo + c * 4096, &tmBlo, fb, n0 + 64 * c, k32);
              }
            }
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
            continue;
          }
          if (direct) {
            // no transform: every tile lands on the leader's `full` barrier, which the MMA
            // issuer waits on (cta_group::2 loads complete on the peer's barrier)
            if (CG == 1) {
              ptx::mbar_expect_tx(&full[stage], tx_cta);
              ptx::tma_load_2d(sA, &tmA, &full[stage], k0, m0);
              ptx::tma_load_2d(sAlo, &tmAlo, &full[stage], 2 * k0, m0);
#pragma unroll
              for (int c = 0; c < T::B_COLS / 32; ++c)
                ptx::tma_load_2d(sB + c * B_CHUNK_BYTES, &tmB, &full[stage], n0 + 32 * c, k0);
#pragma unroll
              for (int c = 0; c < T::B_COLS / 64; ++c)
                ptx::tma_load_2d(sBlo + c * 4096, &tmBlo, &full[stage], n0 + 64 * c, 2 * k0);
            } else {
              const uint32_t fb = ptx::smem_u32(&full[stage]) & ptx::kPeerBitMask;
              if (leader) ptx::mbar_expect_tx(&full[stage], 2 * tx_cta);
              ptx::tma_load_2d_cg2(sA, &tmA, fb, k0, m0);
              ptx::tma_load_2d_cg2(sAlo, &tmAlo, fb, 2 * k0, m0);
#pragma unroll
              for (int c = 0; c < T::B_COLS / 32; ++c)
                ptx::tma_load_2d_cg2(sB + c * B_CHUNK_BYTES, &tmB, fb, n0 + 32 * c, k0);
#pragma unroll
              for (int c = 0; c < T::B_COLS / 64; ++c)
                ptx::tma_load_2d_cg2(sBlo + c * 4096, &tmBlo, fb, n0 + 64 * c, 2 * k0);
            }
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
            continue;
          }
          // every CTA's tiles land on its own `full` barrier (its transform warps wait there)
          ptx::mbar_expect_tx(&full[stage], tx_cta);
          ptx::tma_load_2d(sA, &tmA, &full[stage], k0, m0);
#pragma unroll
          for (int c = 0; c < T::B_COLS / 32; ++c)
            ptx::tma_load_2d(sB + c * B_CHUNK_BYTES, &tmB, &full[stage], n0 + 32 * c, k0);
          if (load_ax) ptx::tma_load_2d(sAlo, &tmAlo, &full[stage], 2 * k0, m0);
          if (load_bx) {
#pragma unroll
            for (int c = 0; c < T::B_COLS / 64; ++c)
              ptx::tma_load_2d(sBlo + c * 4096, &tmBlo, &full[stage], n0 + 64 * c, 2 * k0);
          }
          if (load_lo) {
            ptx::tma_load_2d(sAlo, &tmAlo, &full[stage], k0, m0);
#pragma unroll
            for (int c = 0; c < T::B_COLS / 32; ++c)
              ptx::tma_load_2d(sBlo + c * B_CHUNK_BYTES, &tmBlo, &full[stage], n0 + 32 * c, k0);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (p.sched) atomicAdd(&p.sched[1], 1u);  // this CTA has issued every load of unit u
      }
    }
  } else if (warp == 1) {
    // ======================= MMA issuer (leader CTA) =======================
    if (lane == 0 && leader) {
      constexpr uint32_t idesc = make_idesc(BM * CG, BN);
      constexpr uint32_t idesc2 = make_idesc_bf16(BM * CG, BN);
      constexpr uint32_t idesc4 = make_idesc_f16(BM * CG, BN);
      int stage = 0;
      uint32_t phase = 0;
      uint32_t acc_iter = 0;
      for (int it = 0;; ++it) {
        const int u = sched_take<CG>(it, sched_full, sched_empty,
                                     ptx::smem_u32(&sched_empty[0]), sched_ring, false);
        if (u < 0) break;
        int t, kb, kb1, part;
        unit_coords(u, p, t, kb, kb1, part);
        const int n_int = (kb1 - kb + p.p_kb - 1) / p.p_kb;
        for (int it = 0; it < n_int; ++it, ++acc_iter) {
          const uint32_t buf = acc_iter & 1, use = acc_iter >> 1;
          ptx::mbar_wait(&tempty[buf], (use & 1) ^ 1);
          ptx::tc_fence_after();
          const uint32_t d_tmem = tmem_base + buf * ACC_COLS;
          const int kb_end = min(kb + p.p_kb, kb1);
          uint32_t acc = 0;
          for (; kb < kb_end; ++kb) {
            ptx::mbar_wait(direct ? &full[stage] : &lofull[stage], phase);
            ptx::tc_fence_after();
            const uint32_t sA = ptx::smem_u32(smem + stage * T::STAGE_BYTES);
            const uint32_t sAlo = sA + A_BYTES;
            const uint32_t sB = sA + 2 * A_BYTES;
            const uint32_t sBlo = sB + T::B_BYTES;
            if (p.terms == 4) {
              // 3xFP16, two k16 steps per 32-wide k-block, small terms first:
              // a_lo b_hi, a_hi b_lo, a_hi b_hi (a_lo b_lo, <= 2^-22 relative, is dropped)
#pragma unroll
              for (int j = 0; j < 2; ++j) {
                const uint64_t dAh = make_sdesc(sA + 32 * j, 16, 512, 4);
                const uint64_t dAl = make_sdesc(sAlo + 32 * j, 16, 512, 4);
                const uint64_t dBh = make_sdesc(sB + 2048 * j, 4096, 1024, 2);
                const uint64_t dBl = make_sdesc(sBlo + 2048 * j, 4096, 1024, 2);
                if (CG == 1) {
                  ptx::mma_bf16(d_tmem, dAl, dBh, idesc4, acc);
                  ptx::mma_bf16(d_tmem, dAh, dBl, idesc4, 1u);
                  ptx::mma_bf16(d_tmem, dAh, dBh, idesc4, 1u);
                } else {
                  ptx::mma_bf16_cg2(d_tmem, dAl, dBh, idesc4, acc);
                  ptx::mma_bf16_cg2(d_tmem, dAh, dBl, idesc4, 1u);
                  ptx::mma_bf16_cg2(d_tmem, dAh, dBh, idesc4, 1u);
                }
                acc = 1;
              }
            } else {
#pragma unroll
            for (int k8 = 0; k8 < BK / 8; ++k8) {
              const uint64_t dA = make_sdesc(sA + 32 * k8, 16, 512, 4);
              const uint64_t dB = make_sdesc(sB + 1024 * k8, B_CHUNK_BYTES, 512, 1);
              const uint64_t dAlo = make_sdesc(sAlo + 32 * k8, 16, 512, 4);
              const uint64_t dBlo = make_sdesc(sBlo + 1024 * k8, B_CHUNK_BYTES, 512, 1);
              if (p.terms == 2) {
                // one K=16 bf16 MMA: [a_lo | a_hi] . [b ; b_lo] = a_lo*b + a_hi*b_lo, then hi*hi
                // A' K-major SW64 (the lo tile's geometry); B' MN-major SW128: LBO = 4096
                // between 64-column atoms, SBO = 1024 between 8-row k groups (measured on
                // B200: the swapped reading gives wrong products)
                const uint64_t dAx = make_sdesc(sAlo + 32 * k8, 16, 512, 4);
                const uint64_t dBx = make_sdesc(sBlo + 2048 * k8, 4096, 1024, 2);
                if (CG == 1) {
                  ptx::mma_bf16(d_tmem, dAx, dBx, idesc2, acc);
                  ptx::mma_tf32(d_tmem, dA, dB, idesc, 1u);
                } else {
                  ptx::mma_bf16_cg2(d_tmem, dAx, dBx, idesc2, acc);
                  ptx::mma_tf32_cg2(d_tmem, dA, dB, idesc, 1u);
                }
              } else if (CG == 1) {
                if (p.terms == 3) {
                  ptx::mma_tf32(d_tmem, dAlo, dB, idesc, acc);
                  ptx::mma_tf32(d_tmem, dA, dBlo, idesc, 1u);
                  acc = 1;
                }
                ptx::mma_tf32(d_tmem, dA, dB, idesc, acc);
              } else {
                if (p.terms == 3) {
                  ptx::mma_tf32_cg2(d_tmem, dAlo, dB, idesc, acc);
                  ptx::mma_tf32_cg2(d_tmem, dA, dBlo, idesc, 1u);
                  acc = 1;
                }
                ptx::mma_tf32_cg2(d_tmem, dA, dB, idesc, acc);
              }
              acc = 1;
            }
            }
            if (CG == 1)
              ptx::mma_commit(&empty[stage]);
            else
              ptx::mma_commit_cg2(&empty[stage], 0x3);
            if (++stage == STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
          if (CG == 1)
            ptx::mma_commit(&tfull[buf]);
          else
            ptx::mma_commit_cg2(&tfull[buf], 0x3);
        }
      }
    }
  } else if (warp >= XFORM_WARP0) {
    // ======================= transform (2 warps per CTA) =======================
    // lo = x - tf32(x) of this CTA's raw A and B tiles, written at the same offsets in the lo
    // slots (the swizzle is a permutation of 16-byte chunks and the map is elementwise).
    // 64 threads, consecutive 16-byte chunks per warp instruction: conflict-free.
    const int xt = threadIdx.x - XFORM_WARP0 * 32;
    const bool do_lo = p.terms == 3 && p.lo_smem;
    constexpr int NA = int(A_BYTES / 16) / (NUM_XFORM_WARPS * 32);    // 8
    constexpr int NB = int(T::B_BYTES / 16) / (NUM_XFORM_WARPS * 32); // 8 (CG=2), 16 (CG=1)
    // Pair protocol for `lofull[s]` (leader's): its own two transform warps arrive (the first
    // also expects 16 transaction bytes per peer warp), each peer transform warp completes 16
    // bytes with an async-proxy bulk signal after its proxy fence (ptx::bulk_signal_leader).
    const uint32_t lofull_leader = ptx::smem_u32(&lofull[0]) & ptx::kPeerBitMask;
    const uint32_t sig_leader = ptx::smem_u32(sig) & ptx::kPeerBitMask;
    const int xw = warp - XFORM_WARP0;
    const uint32_t sempty_leader = ptx::smem_u32(&sched_empty[0]) & ptx::kPeerBitMask;
    int stage = 0;
    uint32_t phase = 0;
    for (int it = 0; !direct; ++it) {  // direct: no transform work, not a ring consumer
      const int u = sched_take<CG>(it, sched_full, sched_empty, sempty_leader, sched_ring, true);
      if (u < 0) break;
      int t, kb0, kb1, part;
      unit_coords(u, p, t, kb0, kb1, part);
      for (int kb = kb0; kb < kb1; ++kb) {
        ptx::mbar_wait(&full[stage], phase);
        if (do_lo) {
          const uint32_t sA = ptx::smem_u32(smem + stage * T::STAGE_BYTES);
          const uint32_t sB = sA + 2 * A_BYTES;
          float4 va[NA], vb[NB];
#pragma unroll
          for (int i = 0; i < NA; ++i)
            va[i] = ptx::ld_shared_v4(sA + uint32_t(i * NUM_XFORM_WARPS * 32 + xt) * 16);
#pragma unroll
          for (int i = 0; i < NB; ++i)
            vb[i] = ptx::ld_shared_v4(sB + uint32_t(i * NUM_XFORM_WARPS * 32 + xt) * 16);
#pragma unroll
          for (int i = 0; i < NA; ++i)
            ptx::st_shared_v4(sA + A_BYTES + uint32_t(i * NUM_XFORM_WARPS * 32 + xt) * 16,
                              tf32_lo(va[i].x), tf32_lo(va[i].y), tf32_lo(va[i].z),
                              tf32_lo(va[i].w));
#pragma unroll
          for (int i = 0; i < NB; ++i)
            ptx::st_shared_v4(sB + T::B_BYTES + uint32_t(i * NUM_XFORM_WARPS * 32 + xt) * 16,
                              tf32_lo(vb[i].x), tf32_lo(vb[i].y), tf32_lo(vb[i].z),
                              tf32_lo(vb[i].w));
          ptx::fence_proxy_async_smem();  // generic-proxy writes -> tensor-core reads
        } else if (p.terms == 2 && !p.a_pre) {
          if (p.b_pre)
            xform_tf32_bf16<CG, true>(ptx::smem_u32(smem + stage * T::STAGE_BYTES), xt, p.hi_rn);
          else
            xform_tf32_bf16<CG, false>(ptx::smem_u32(smem + stage * T::STAGE_BYTES), xt, p.hi_rn);
          ptx::fence_proxy_async_smem();
        }
        __syncwarp();
        if (lane == 0) {
          if (CG == 1 || leader) {
            if (CG == 2 && xw == 0)
              ptx::mbar_arrive_expect_tx(&lofull[stage], 16 * NUM_XFORM_WARPS);
            else
              ptx::mbar_arrive(&lofull[stage]);
          } else {
            ptx::bulk_signal_leader(sig_leader, sig + 16, lofull_leader + uint32_t(stage) * 8);
          }
        }
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else {
    // ======================= epilogue (8 warps per CTA) =======================
    const int e = warp - 2;
    const int quad = warp & 3;  // TMEM lane quadrant this warp may access
    const int half = e >> 2;    // column half of the 256-wide tile
    const uint32_t tempty_leader0 = ptx::smem_u32(&tempty[0]) & ptx::kPeerBitMask;
    const uint32_t tempty_leader1 = ptx::smem_u32(&tempty[1]) & ptx::kPeerBitMask;
    const uint32_t sempty_leader = ptx::smem_u32(&sched_empty[0]) & ptx::kPeerBitMask;
    uint32_t acc_iter = 0;
    uint32_t cphase = 0;  // parity of this warp's C-load barrier
    for (int it = 0;; ++it) {
      const int u = sched_take<CG>(it, sched_full, sched_empty, sempty_leader, sched_ring, true);
      if (u < 0) break;
      int t, kb0, kb1, mb, nb, part;
      unit_coords(u, p, t, kb0, kb1, part);
      tile_coords(t, p, mb, nb);
      const int n_int = (kb1 - kb0 + p.p_kb - 1) / p.p_kb;
      float sum[128];  // fp32 running sum of the promoted partials (0 + p == p exactly)
#pragma unroll
      for (int j = 0; j < 128; ++j) sum[j] = 0.0f;
      for (int it = 0; it < n_int; ++it, ++acc_iter) {
        const uint32_t buf = acc_iter & 1, use = acc_iter >> 1;
        ptx::mbar_wait(&tfull[buf], use & 1);
        ptx::tc_fence_after();
        const uint32_t taddr =
            tmem_base + (uint32_t(quad * 32) << 16) + buf * ACC_COLS + half * 128;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          float v[16];
          ptx::tmem_ld16_wait(taddr + c * 16, v);
#pragma unroll
          for (int j = 0; j < 16; ++j) sum[c * 16 + j] = __fadd_rn(sum[c * 16 + j], v[j]);
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (CG == 1)
            ptx::mbar_arrive(&tempty[buf]);
          else
            ptx::mbar_arrive_cluster(buf ? tempty_leader1 : tempty_leader0);
        }
      }
      if (part >= 0 && p.split_mode == kSplitWorkspace) {
        // K-split part: publish this warp's 32 x 128 partial (lane-interleaved float4s: one
        // coalesced 512-byte row of the slot per store), count in; the last of the tile's
        // parts adds all of them in part order and carries on as a whole tile.
        const int st_idx = ((t - p.first_split) * CG + int(rank)) * NUM_EPI_WARPS + e;
        const float4 *slot0 = reinterpret_cast<const float4 *>(p.sk_ws) +
                        size_t(st_idx) * p.split_s * (32 * 32) + lane;  // this lane's column
        float4 *mine = const_cast<float4 *>(slot0) + part * (32 * 32);
#pragma unroll
        for (int j = 0; j < 32; ++j)
          __stcg(mine + j * 32,
                 make_float4(sum[4 * j], sum[4 * j + 1], sum[4 * j + 2], sum[4 * j + 3]));
        __threadfence();
        __syncwarp();
        unsigned arrived = 0;
        if (lane == 0) arrived = atomicAdd(&p.sk_cnt[st_idx], 1u);
        arrived = __shfl_sync(0xffffffffu, arrived, 0);
        if (arrived != unsigned(p.split_s - 1)) continue;  // another part finishes the tile
        if (lane == 0) p.sk_cnt[st_idx] = 0;  // every part has counted in: reset for next launch
        __threadfence();
        // the ordered sum reads every part from memory, own slot included (this thread wrote it)
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          float4 tot = __ldcg(slot0 + j * 32);
          for (int q = 1; q < p.split_s; ++q) {
            const float4 v = __ldcg(slot0 + q * (32 * 32) + j * 32);
            tot.x = __fadd_rn(tot.x, v.x);
            tot.y = __fadd_rn(tot.y, v.y);
            tot.z = __fadd_rn(tot.z, v.z);
            tot.w = __fadd_rn(tot.w, v.w);
          }
          sum[4 * j] = tot.x;
          sum[4 * j + 1] = tot.y;
          sum[4 * j + 2] = tot.z;
          sum[4 * j + 3] = tot.w;
        }
      }
      // C: this warp's 32 rows x 128 columns go out as four 32 x 32 TMA bulk stores through
      // its 4 KiB staging tile (128B-swizzled rows: 16-byte chunk j of row r sits at chunk
      // j ^ (r & 7), so each 8-lane phase of a v4 store covers all 32 banks). The TMA unit
      // writes whole 128-byte row segments and clips rows >= M / columns >= N. Accumulate
      // mode (K-chunked pipelines) uses the TMA reduce-add: C += partial in fp32.
      const bool reduce_store = p.accumulate || (part >= 0 && p.split_mode == kSplitReduce);
      const uint32_t stg = ptx::smem_u32(epi_stage + e * EPI_STAGE_BYTES);
      const int crow0 = mb * T::TILE_M + int(rank) * BM + quad * 32;
      const int ccol0 = nb * BN + half * 128;
      if (p.ea) {
        // 3xFP16: undo the power-of-two operand scales (pow2_scale: exact for every normal
        // result, two multiplications). ea / eb are padded to whole tiles.
        // (lane l holds the exponents of columns 4l..4l+3; the warp shares them by shuffles,
        // which keeps 4 registers live instead of 128 hoisted loads)
        const int ei = p.ea[crow0 + lane];
        const int4 fl = *reinterpret_cast<const int4 *>(p.eb + ccol0 + 4 * lane);
#pragma unroll
        for (int q = 0; q < 32; ++q) {
          sum[4 * q] = pow2_scale(sum[4 * q], ei + __shfl_sync(0xffffffffu, fl.x, q));
          sum[4 * q + 1] = pow2_scale(sum[4 * q + 1], ei + __shfl_sync(0xffffffffu, fl.y, q));
          sum[4 * q + 2] = pow2_scale(sum[4 * q + 2], ei + __shfl_sync(0xffffffffu, fl.z, q));
          sum[4 * q + 3] = pow2_scale(sum[4 * q + 3], ei + __shfl_sync(0xffffffffu, fl.w, q));
        }
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (lane == 0) ptx::bulk_wait_read<0>();  // previous store has left the staging tile
        __syncwarp();
        if (p.load_c) {
          // C += this partial, in registers: TMA-load the block (zero-filled outside C) into
          // the staging tile, then add row `lane` (same swizzle as the store below)
          if (lane == 0) {
            ptx::mbar_expect_tx(&cbar[e], EPI_STAGE_BYTES);
            ptx::tma_load_2d(epi_stage + e * EPI_STAGE_BYTES, &cmaps.m[0], &cbar[e],
                             ccol0 + 32 * c, crow0);
          }
          ptx::mbar_wait(&cbar[e], cphase);
          cphase ^= 1;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 o = ptx::ld_shared_v4(
                stg + uint32_t(lane) * 128 + uint32_t((j ^ (lane & 7)) * 16));
            sum[c * 32 + 4 * j] = __fadd_rn(sum[c * 32 + 4 * j], o.x);
            sum[c * 32 + 4 * j + 1] = __fadd_rn(sum[c * 32 + 4 * j + 1], o.y);
            sum[c * 32 + 4 * j + 2] = __fadd_rn(sum[c * 32 + 4 * j + 2], o.z);
            sum[c * 32 + 4 * j + 3] = __fadd_rn(sum[c * 32 + 4 * j + 3], o.w);
          }
          __syncwarp();  // every lane has read the block before it is overwritten
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const uint32_t off = uint32_t(lane) * 128 + uint32_t((j ^ (lane & 7)) * 16);
          ptx::st_shared_v4(stg + off, sum[c * 32 + 4 * j], sum[c * 32 + 4 * j + 1],
                            sum[c * 32 + 4 * j + 2], sum[c * 32 + 4 * j + 3]);
        }
        // 3xFP16: the B-side exceptions of these 32 columns (once per tile: not in the
        // second half of a reduce-split tile)
        // (blocks right of N -- clipped by the TMA store -- have no strip)
        if (p.xb && ccol0 + 32 * c < p.N && !(part > 0 && p.split_mode == kSplitReduce)) {
          const int strip = (ccol0 + 32 * c) >> 5;
          const int cnt = p.bcnt[strip];
          float *stgf = reinterpret_cast<float *>(epi_stage + e * EPI_STAGE_BYTES);
          if (cnt > kBList)
            fix_b_block(p, stgf, crow0 + lane, ccol0 + 32 * c, lane);
          else if (cnt > 0)
            fix_b_list(p, stgf, crow0 + lane, strip, cnt, lane);
        }
        if (p.st_mode != kStoreTma) {
          __syncwarp();  // every lane's staged row (and the B-side fix) is in place
          vec_store_block(p, stg, crow0, ccol0 + 32 * c, lane);
          __syncwarp();  // all reads done before the block is overwritten (or TMA-loaded into)
          ptx::fence_proxy_async_smem();
          continue;
        }
        ptx::fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          // every destination C buffer (this GPU's, then the peers' when the gather is fused
          // into the epilogue: the same rows land in every GPU's C_full over NVLink)
          for (int dst = 0; dst < p.n_cdst; ++dst) {
            if (reduce_store)
              ptx::tma_store_add_2d(&cmaps.m[dst], epi_stage + e * EPI_STAGE_BYTES,
                                    ccol0 + 32 * c, crow0);
            else
              ptx::tma_store_2d(&cmaps.m[dst], epi_stage + e * EPI_STAGE_BYTES, ccol0 + 32 * c,
                                crow0);
          }
          ptx::bulk_commit();
        }
      }
    }
    if (lane == 0) ptx::bulk_wait<0>();  // all C writes complete before the CTA retires
  }
  __syncwarp();
  ptx::tc_fence_before();
  if (CG == 2)
    ptx::cluster_sync();  // no CTA leaves while its peer may still signal its barriers
  else
    __syncthreads();
  if (warp == 0) {
    ptx::tc_fence_after();
    if (CG == 2)
      ptx::tmem_dealloc_cg2(tmem_base, TMEM_COLS);
    else
      ptx::tmem_dealloc(tmem_base, TMEM_COLS);
  }
  if (p.cta_ns && threadIdx.x == 0) p.cta_ns[2 * blockIdx.x + 1] = ptx::globaltimer_ns();
  if (threadIdx.x == 0 && p.sched) {
    // thread 0 made every claim and issued-count of this CTA; the last CTA of the grid to
    // finish returns the counters to zero for the next launch on this stream
    __threadfence();
    if (atomicAdd(&p.sched[2], 1u) == gridDim.x - 1) {
      p.sched[0] = 0;
      p.sched[1] = 0;
      p.sched[2] = 0;
      __threadfence();
    }
  }
}


__global__ void __launch_bounds__(256) split_lo_kernel(const float *__restrict__ x,
                                                       float *__restrict__ lo, int64_t n) {
  const int64_t n4 = n >> 2;
  const float4 *x4 = reinterpret_cast<const float4 *>(x);
  float4 *lo4 = reinterpret_cast<float4 *>(lo);
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  // 4 independent 16-byte loads in flight per thread
  for (; i + 3 * stride < n4; i += 4 * stride) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldcs(x4 + i + u * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u)
      __stcs(lo4 + i + u * stride,
             make_float4(tf32_lo(v[u].x), tf32_lo(v[u].y), tf32_lo(v[u].z), tf32_lo(v[u].w)));
  }
  for (; i < n4; i += stride) {
    const float4 v = __ldcs(x4 + i);
    __stcs(lo4 + i, make_float4(tf32_lo(v.x), tf32_lo(v.y), tf32_lo(v.z), tf32_lo(v.w)));
  }
  if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
    const int64_t j = (n4 << 2) + threadIdx.x;
    lo[j] = tf32_lo(x[j]);
  }
}

// B operand of the TF32 + BF16 scheme, once per call in HBM (B is read by every M-tile, so the
// transform warps would redo this per tile): B_hi[k][n] = RN tf32(b) (fp32, the tf32 MMA's
// operand) and B'[16 (k / 8) + (k % 8)][n] = bf16(b), B'[16 (k / 8) + 8 + (k % 8)][n] =
// bf16(b - B_hi) (bf16, ldx columns), rows of k >= K zero: the layout one 64 x 32 TMA box
// (128B swizzle) lands as the MN-major SW128 B' chunk the correction MMA reads. HBM-bound:
// 4 B read + 8 B written per element. Thread = 4 columns x one k8 block.
__global__ void __launch_bounds__(256) prep_b_kernel(const float *__restrict__ B, int64_t ldb,
                                                     int K, int N, float *__restrict__ Bhi,
                                                     uint16_t *__restrict__ Bx, int64_t ldx) {
  const int n4 = N >> 2, kb8 = (K + 7) >> 3;
  const int64_t total = int64_t(kb8) * n4;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int kb = int(i / n4), n = int(i - int64_t(kb) * n4) * 4;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int k = kb * 8 + j;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (k < K) v = __ldcs(reinterpret_cast<const float4 *>(B + int64_t(k) * ldb + n));
      const float h0 = tf32_hi(v.x, 1), h1 = tf32_hi(v.y, 1), h2 = tf32_hi(v.z, 1),
                  h3 = tf32_hi(v.w, 1);
      if (k < K)
        __stcs(reinterpret_cast<float4 *>(Bhi + int64_t(k) * N + n), make_float4(h0, h1, h2, h3));
      const uint2 big = make_uint2(ptx::pack_bf16x2(v.x, v.y), ptx::pack_bf16x2(v.z, v.w));
      const uint2 sml = make_uint2(ptx::pack_bf16x2(__fsub_rn(v.x, h0), __fsub_rn(v.y, h1)),
                                   ptx::pack_bf16x2(__fsub_rn(v.z, h2), __fsub_rn(v.w, h3)));
      __stcs(reinterpret_cast<uint2 *>(Bx + int64_t(16 * kb + j) * ldx + n), big);
      __stcs(reinterpret_cast<uint2 *>(Bx + int64_t(16 * kb + 8 + j) * ldx + n), sml);
    }
  }
}

// A operand of the TF32 + BF16 scheme in HBM: A_hi[m][k] = RN tf32(a) (row stride K) and the
// K-major A'[m][16 (k / 8) + (k % 8)] = bf16(a - A_hi), A'[m][16 (k / 8) + 8 + (k % 8)] =
// bf16(A_hi) (row stride ldx = 2 * ceil(K / 8) * 8, k >= K zero): a 32 x 128 TMA box with the
// 64B swizzle lands as the A' tile of a k-block. Thread = one row x one k8 block (32 B out).
__global__ void __launch_bounds__(256) prep_a_kernel(const float *__restrict__ A, int64_t lda,
                                                     int M, int K, float *__restrict__ Ahi,
                                                     uint16_t *__restrict__ Ax, int64_t ldx) {
  const int kb8 = (K + 7) >> 3;
  const int64_t total = int64_t(M) * kb8;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t m = i / kb8;
    const int kb = int(i - m * kb8), k = kb * 8;
    const float *src = A + m * lda + k;
    float v[8];
    if (k + 8 <= K) {
      const float4 a0 = __ldcs(reinterpret_cast<const float4 *>(src));
      const float4 a1 = __ldcs(reinterpret_cast<const float4 *>(src + 4));
      v[0] = a0.x; v[1] = a0.y; v[2] = a0.z; v[3] = a0.w;
      v[4] = a1.x; v[5] = a1.y; v[6] = a1.z; v[7] = a1.w;
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = (k + j < K) ? src[j] : 0.f;
    }
    float h[8], l[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      h[j] = tf32_hi(v[j], 1);
      l[j] = __fsub_rn(v[j], h[j]);
    }
    float *hd = Ahi + m * K + k;
    if (k + 8 <= K) {
      __stcs(reinterpret_cast<float4 *>(hd), make_float4(h[0], h[1], h[2], h[3]));
      __stcs(reinterpret_cast<float4 *>(hd + 4), make_float4(h[4], h[5], h[6], h[7]));
    } else {
      for (int j = 0; j < 8 && k + j < K; ++j) hd[j] = h[j];
    }
    uint4 *xd = reinterpret_cast<uint4 *>(Ax + m * ldx + 16 * kb);
    __stcs(xd, make_uint4(ptx::pack_bf16x2(l[0], l[1]), ptx::pack_bf16x2(l[2], l[3]),
                          ptx::pack_bf16x2(l[4], l[5]), ptx::pack_bf16x2(l[6], l[7])));
    __stcs(xd + 1, make_uint4(ptx::pack_bf16x2(h[0], h[1]), ptx::pack_bf16x2(h[2], h[3]),
                              ptx::pack_bf16x2(h[4], h[5]), ptx::pack_bf16x2(h[6], h[7])));
  }
}

__global__ void stamp_kernel(uint64_t *slot) { *slot = ptx::globaltimer_ns(); }

cudaError_t launch_stamp(uint64_t *slot, cudaStream_t st) {
  stamp_kernel<<<1, 1, 0, st>>>(slot);
  return cudaGetLastError();
}

// ---- host side ----------------------------------------------------------------------------
// Promotion interval: kDefaultPromoteKBlocks, overridable once per process with the
// GIGA_PROMOTE_KBLOCKS environment variable (0 = never promote; tests / sweeps only).
int default_promote_kblocks(int terms) {
  static int v = [] {
    const char *e = getenv("GIGA_PROMOTE_KBLOCKS");
    if (e && *e) {
      const int x = atoi(e);
      if (x >= 0) return x;
    }
    return -1;
  }();
  if (v >= 0) return v;
  static const int v4 = [] {  // $GIGA_PROMOTE_KBLOCKS_T4: the 3xFP16 scheme's alone
    const char *e = getenv("GIGA_PROMOTE_KBLOCKS_T4");
    return (e && *e && atoi(e) > 0) ? atoi(e) : kDefaultPromoteKBlocksT4;
  }();
  return terms == 2 ? kDefaultPromoteKBlocksT2 : terms == 4 ? v4 : kDefaultPromoteKBlocks;
}

static int forced_scheme() {
  static const int forced = [] {
    const char *e = getenv("GIGA_SCHEME");
    if (e && strcmp(e, "3xtf32") == 0) return 3;
    if (e && strcmp(e, "tf32bf16") == 0) return 2;
    if (e && strcmp(e, "3xfp16") == 0) return 4;
    return 0;
  }();
  return forced;
}

bool scheme_forced() { return forced_scheme() != 0; }

int product_terms(const float *A_lo, int64_t M, int64_t N, int64_t K) {
  const int forced = forced_scheme();
  if (A_lo) return 3;
  if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX) return 3;  // the launch rejects these
  if (forced) return forced;
  const double mnk = double(M) * double(N) * double(K);
  // measured crossover, operand preparation and exception fixes included
  // (profiles/r02_scheme_crossover_e.jsonl, scripts/scheme_crossover.py), after the epilogue's
  // scaling became two multiplications (pow2_scale): 3xFP16 wins from 2^35 multiply-adds with
  // K >= 512 -- 4096^3 +28%, 2048 x 4096^2 +10%, 4096^2 x 2048 +16%, 32768 x 1024^2 +3%, the
  // tall 262144 x 1024^2 +23%, 16384 x 32768 x 512 +49%, up to +82% at 16384^3 -- and loses
  // below (2048^3: -21%, 1024^3: -40%, where B's preparation and the per-launch costs are not
  // amortised); at K = 256 the three schemes tie
  if (M >= 2048 && N >= 1024 && K >= 512 && mnk >= 0x1p35) return 4;
  // (TF32 + BF16 is no longer chosen by shape -- 3xFP16 covers its old range; $GIGA_SCHEME
  // forces it)
  return 3;
}

// CTA-group size: 2 (CTA pairs) unless the problem has fewer 256-row tiles than SM pairs,
// or $GIGA_CTA_GROUP forces 1 or 2.
int choose_cta_group(int64_t M, int64_t N, int num_sms) {
  static int forced = [] {
    const char *e = getenv("GIGA_CTA_GROUP");
    return (e && (*e == '1' || *e == '2')) ? (*e - '0') : 0;
  }();
  if (forced) return forced;
  const int64_t tiles2 = ((M + 255) / 256) * ((N + 255) / 256);
  return tiles2 >= num_sms / 2 ? 2 : 1;
}

static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::once_flag g_encode_once;

int ensure_tma_encoder() {
  std::call_once(g_encode_once, [] {
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode ? 0 : -1;
}

// 2-D fp32 map over a row-major (rows x cols, row stride ld elements) matrix.
static bool make_map(CUtensorMap *m, const float *ptr, uint64_t cols, uint64_t rows,
                     uint64_t ld, uint32_t box_cols, uint32_t box_rows, CUtensorMapSwizzle sw) {
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {ld * sizeof(float)};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  // L2 sector promotion of TMA fills ($GIGA_L2_PROMO: 0 none, 1 64B, 2 128B, 3 256B)
  static const CUtensorMapL2promotion promo = [] {
    const char *e = getenv("GIGA_L2_PROMO");
    const int v = (e && *e) ? atoi(e) : 2;  // 128B: same speed as 256B, ~18% less DRAM
    return v == 0   ? CU_TENSOR_MAP_L2_PROMOTION_NONE
           : v == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
           : v == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                    : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }();
  return g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(ptr), dims,
                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw, promo,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 2-D 16-bit map (bf16: A' / B' of the TF32 + BF16 scheme; fp16: the 3xFP16 operands).
static bool make_map_bf16(CUtensorMap *m, const uint16_t *ptr, uint64_t cols, uint64_t rows,
                          uint64_t ld, uint32_t box_cols, uint32_t box_rows,
                          CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B,
                          CUtensorMapDataType dt = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16) {
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {ld * sizeof(uint16_t)};
  const cuuint32_t box[2] = {box_cols, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  return g_encode(m, dt, 2, const_cast<uint16_t *>(ptr), dims,
                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

static int num_sms_current() {
  int dev = 0, n = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

// ---- K-split plan and workspace ------------------------------------------------------------
// Persistent clusters take units round-robin, so T tiles on `nclu` concurrent clusters last
// ceil(T / nclu) tile times. Two ways to cut tiles into k-parts, both deterministic:
//   * kSplitReduce (s = 2, plain-store launches only): the two halves TMA reduce-add into a
//     C region zeroed before the launch; 0 + a + b == a + b in either order. Used for the
//     last wave of a multi-wave launch when it is at most half full (4096^3: 256 tiles on 74
//     pairs = 3 waves + 34 tiles -> 3.5 wave times, measured -11%), and for s = 2 below.
//   * kSplitWorkspace (any s, any epilogue mode): parts write fp32 partials to a workspace,
//     the last part of a tile to finish adds them in part order. Only for grids that fill
//     less than one wave (tiles < nclu), e.g. 24 tiles of 512 x 1536 x 2048 on 148 SMs:
//     measured -41% with 4 parts. Cost model (k-block times; fitted to scripts/ksplit_sweep.py
//     on B200): ceil(n_kb / s) + 14 + 5 s against n_kb, one part wave (tiles * s <= nclu);
//     the 14 + 5 s is the partial write, the arrival count and the latency-bound ordered read
//     of s partials. Cutting the tail of a multi-wave launch into more than two parts measured
//     slower than whole tiles (the tensor pipe ran 84% busy in part waves against 93%), so it
//     is not planned.
// The workspace is capped at kKSplitMaxSlots 16 KiB slots. $GIGA_KSPLIT_S forces s for
// under-filled grids (experiments).
constexpr int kKSplitMaxS = 32;
constexpr int64_t kKSplitMaxSlots = 8192;  // 128 MiB

KSplitPlan plan_ksplit(int num_tiles, int nclu, int n_kb, int cg, bool plain, int p_kb) {
  KSplitPlan whole{num_tiles, 1, kSplitNone};
  if (num_tiles < 1 || nclu < 1 || n_kb < 2) return whole;
  if (num_tiles >= nclu) {
    const int tail = num_tiles % nclu;
    if (plain && tail > 0 && 2 * tail <= nclu && n_kb >= 2 * p_kb)
      return KSplitPlan{num_tiles - tail, 2, kSplitReduce};
    return whole;
  }
  static const int forced_s = [] {
    const char *e = getenv("GIGA_KSPLIT_S");
    return (e && atoi(e) > 0) ? atoi(e) : 0;
  }();
  KSplitPlan best = whole;
  double best_cost = forced_s ? 1e300 : 0.97 * n_kb;
  for (int s = 2; s <= std::min(n_kb, kKSplitMaxS); ++s) {
    if (int64_t(num_tiles) * s > nclu && !forced_s) break;  // one part wave
    if (int64_t(num_tiles) * s * cg * cfg::NUM_EPI_WARPS > kKSplitMaxSlots) break;
    if (forced_s && s != forced_s) continue;
    const bool reduce = plain && s == 2;
    const double cost = double((n_kb + s - 1) / s) * double((int64_t(num_tiles) * s + nclu - 1) / nclu) +
                        (reduce ? 4.0 : 14.0 + 5.0 * s);
    if (cost < best_cost) {
      best_cost = cost;
      best = KSplitPlan{0, s, reduce ? kSplitReduce : kSplitWorkspace};
    }
  }
  return best;
}

// One workspace per (device, stream): launches on one stream are ordered, so they can share
// it; launches on different streams (virtual GPUs sharing a device, concurrent callers) get
// their own. Grow-only; growth waits for the stream's earlier launches (they may still read
// the old slots). The counters start at zero and every launch leaves them at zero.
struct KSplitWs {
  float *ws = nullptr;
  unsigned *cnt = nullptr;
  size_t ws_bytes = 0, cnt_n = 0;
  int dev = 0;
};
static std::mutex g_ksplit_mu;
static std::vector<std::pair<cudaStream_t, KSplitWs>> g_ksplit;

// Superseded buffers kept alive for captured graphs (retire_buffer).
static std::mutex g_retire_mu;
static bool g_keep_superseded = false;
static std::vector<std::pair<int, void *>> g_retired;

void keep_superseded_buffers() {
  std::lock_guard<std::mutex> lk(g_retire_mu);
  g_keep_superseded = true;
}

void retire_buffer(void *p) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_retire_mu);
  if (!g_keep_superseded) {
    cudaFree(p);
    return;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  g_retired.push_back({dev, p});
}

bool ksplit_workspace(cudaStream_t st, size_t ws_bytes, size_t cnt_n, float **ws,
                      unsigned **cnt) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  std::lock_guard<std::mutex> lk(g_ksplit_mu);
  KSplitWs *w = nullptr;
  for (auto &e : g_ksplit)
    if (e.first == st && e.second.dev == dev) w = &e.second;
  if (!w || w->ws_bytes < ws_bytes || w->cnt_n < cnt_n) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
      return false;
    if (cudaStreamSynchronize(st) != cudaSuccess) return false;
    KSplitWs fresh;
    fresh.dev = dev;
    fresh.ws_bytes = std::max(ws_bytes, w ? w->ws_bytes : 0);
    fresh.cnt_n = std::max(cnt_n, w ? w->cnt_n : 0);
    if (cudaMalloc(&fresh.ws, fresh.ws_bytes) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    if (cudaMalloc(&fresh.cnt, fresh.cnt_n * sizeof(unsigned)) != cudaSuccess ||
        cudaMemsetAsync(fresh.cnt, 0, fresh.cnt_n * sizeof(unsigned), st) != cudaSuccess) {
      cudaGetLastError();
      cudaFree(fresh.ws);
      if (fresh.cnt) cudaFree(fresh.cnt);
      return false;
    }
    if (w) {
      retire_buffer(w->ws);
      retire_buffer(w->cnt);
      *w = fresh;
    } else {
      g_ksplit.push_back({st, fresh});
      w = &g_ksplit.back().second;
    }
  }
  *ws = w->ws;
  *cnt = w->cnt;
  return true;
}

// Dynamic-schedule counters of the GEMM (GemmParams::sched): 3 words per (device, stream),
// zeroed once at creation (stream-ordered), returned to zero by the last CTA of every launch.
struct SchedCnt {
  cudaStream_t st;
  int dev;
  unsigned *p;
};
static std::vector<SchedCnt> g_sched;

unsigned *sched_counters(cudaStream_t st) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lk(g_ksplit_mu);
  for (auto &c : g_sched)
    if (c.st == st && c.dev == dev) return c.p;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
    return nullptr;
  void *q = nullptr;
  if (cudaMalloc(&q, 64) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  if (cudaMemsetAsync(q, 0, 64, st) != cudaSuccess) {
    cudaGetLastError();
    cudaFree(q);
    return nullptr;
  }
  g_sched.push_back({st, dev, static_cast<unsigned *>(q)});
  return g_sched.back().p;
}

// Per-(device, stream) scratch of the TF32 + BF16 scheme's B_hi / B' (grow-only, like the
// K-split workspace; growth waits for the stream's earlier launches).
// The B part comes first in the buffer and remembers what it holds (key: B, ldb, K, N of the
// last preparation), so row chunks of one product can skip re-preparing B.
struct ScratchBuf {
  cudaStream_t st;
  int dev;
  void *p;
  size_t bytes;
  const float *key_b;
  int64_t key_ldb, key_k, key_n;
  int key_scheme;
};
static std::list<ScratchBuf> g_bpre;

static ScratchBuf *bpre_scratch(cudaStream_t st, size_t bytes) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lk(g_ksplit_mu);
  for (auto &b : g_bpre)
    if (b.st == st && b.dev == dev && b.bytes >= bytes) return &b;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
    return nullptr;
  if (cudaStreamSynchronize(st) != cudaSuccess) return nullptr;
  for (auto it = g_bpre.begin(); it != g_bpre.end(); ++it)
    if (it->st == st && it->dev == dev) {
      retire_buffer(it->p);
      g_bpre.erase(it);
      break;
    }
  void *p = nullptr;
  if (cudaMalloc(&p, bytes) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  g_bpre.push_back({st, dev, p, bytes, nullptr, 0, 0, 0, 0});
  return &g_bpre.back();
}

void release_gemm_caches() {
  std::lock_guard<std::mutex> lk(g_ksplit_mu);
  for (auto &b : g_bpre) {
    cudaSetDevice(b.dev);
    cudaDeviceSynchronize();
    cudaFree(b.p);
  }
  g_bpre.clear();
  for (auto &e : g_ksplit) {
    cudaSetDevice(e.second.dev);
    cudaDeviceSynchronize();
    cudaFree(e.second.ws);
    cudaFree(e.second.cnt);
  }
  g_ksplit.clear();
  for (auto &c : g_sched) {
    cudaSetDevice(c.dev);
    cudaDeviceSynchronize();
    cudaFree(c.p);
  }
  g_sched.clear();
  std::lock_guard<std::mutex> lr(g_retire_mu);
  for (auto &r : g_retired) {
    cudaSetDevice(r.first);
    cudaDeviceSynchronize();
    cudaFree(r.second);
  }
  g_retired.clear();
  g_keep_superseded = false;
}

GemmSchedule gemm_schedule(int64_t M, int64_t N, int64_t K, int num_sms, int cta_group,
                           bool plain, int p_kb, int bk) {
  GemmSchedule s;
  s.cg = (cta_group == 1 || cta_group == 2) ? cta_group : choose_cta_group(M, N, num_sms);
  const int tile_m = cfg::BM * s.cg;
  s.m_tiles = int((M + tile_m - 1) / tile_m);
  s.n_tiles = int((N + cfg::BN - 1) / cfg::BN);
  s.num_tiles = s.m_tiles * s.n_tiles;
  s.nclu = s.cg == 2 ? num_sms / 2 : num_sms;
  s.n_kb = int((K + bk - 1) / bk);
  if (p_kb <= 0 || p_kb > s.n_kb) p_kb = s.n_kb;
  // $GIGA_TAIL_SPLIT=0 disables the k-split
  static const bool split_env = [] {
    const char *e = getenv("GIGA_TAIL_SPLIT");
    return !(e && *e == '0');
  }();
  const KSplitPlan kp = split_env ? plan_ksplit(s.num_tiles, s.nclu, s.n_kb, s.cg, plain, p_kb)
                                  : KSplitPlan{s.num_tiles, 1, kSplitNone};
  s.first_split = kp.first_split;
  s.s = kp.s;
  s.mode = kp.mode;
  s.num_units = s.first_split + (s.num_tiles - s.first_split) * s.s;
  return s;
}

cudaError_t launch_split_lo(const float *x, float *lo, int64_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  const int64_t n4 = (n + 3) / 4;
  int64_t blocks = (n4 + 255) / 256;
  const int64_t cap = int64_t(num_sms_current()) * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  split_lo_kernel<<<unsigned(blocks), 256, 0, st>>>(x, lo, n);
  return cudaGetLastError();
}

// The same split over a rows x cols block with row stride ld (elements); cols % 4 == 0,
// ld % 4 == 0 and 16-byte aligned bases (a K-chunk of a row-major A shard).
__global__ void __launch_bounds__(256) split_lo_2d_kernel(const float *__restrict__ x,
                                                          float *__restrict__ lo, int64_t rows,
                                                          int64_t cols, int64_t ld) {
  const int64_t c4 = cols >> 2, total = rows * c4;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total; i += stride) {
    const int64_t r = i / c4, c = (i - r * c4) << 2;
    const float4 v = __ldcs(reinterpret_cast<const float4 *>(x + r * ld + c));
    __stcs(reinterpret_cast<float4 *>(lo + r * ld + c),
           make_float4(tf32_lo(v.x), tf32_lo(v.y), tf32_lo(v.z), tf32_lo(v.w)));
  }
}

cudaError_t launch_split_lo_2d(const float *x, float *lo, int64_t rows, int64_t cols,
                               int64_t ld, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  if ((cols & 3) || (ld & 3)) return cudaErrorInvalidValue;
  int64_t blocks = (rows * (cols / 4) + 255) / 256;
  const int64_t cap = int64_t(num_sms_current()) * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  split_lo_2d_kernel<<<unsigned(blocks), 256, 0, st>>>(x, lo, rows, cols, ld);
  return cudaGetLastError();
}

// the smem opt-in is a per-device function attribute
template <int CG>
static cudaError_t ensure_smem_attr() {
  static std::mutex mu;
  static uint64_t done = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if (done >> (dev & 63) & 1) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(gemm_3xtf32_kernel<CG>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       int(Tile<CG>::SMEM_BYTES));
  if (e == cudaSuccess) done |= uint64_t(1) << (dev & 63);
  return e;
}

// ---- TF32 + BF16 operand preparation (terms = 2) ---------------------------------------------
cudaError_t terms_prep_alloc(int64_t M, int64_t N, int64_t K, cudaStream_t st, TermsPrep *tp,
                             int terms) {
  *tp = TermsPrep();
  if (ensure_tma_encoder() != 0) return cudaErrorNotSupported;
  auto up = [](size_t b) { return (b + 255) / 256 * 256; };
  if (terms == 4) {
    // 3xFP16: [B_hi | B_lo | eb | bmax | A_hi | A_lo | ea]; exponent arrays padded to whole
    // 256-row / 256-column tiles (the epilogue reads them unguarded)
    const int64_t ldah = (K + 7) / 8 * 8, ldbh = (N + 7) / 8 * 8;
    const int64_t n_pad = (N + 255) / 256 * 256, m_pad = (M + 255) / 256 * 256;
    const int64_t wa = (K + 31) / 32, wb = (N + 31) / 32;
    const size_t bh = up(size_t(K) * ldbh * 2), ebb = up(size_t(n_pad) * 4);
    const size_t ah = up(size_t(M) * ldah * 2), eab = up(size_t(m_pad) * 4);
    // exception bitmaps + summaries + flags: [xb | sb2 | fb] belongs to B (kept with B for
    // b_prep_reuse), [xa | sa2 | fa] to A
    const int64_t w2a = (wa + 31) / 32, w2b = (K + 31) / 32;
    const size_t xbb = up(size_t(K) * wb * 4 + size_t(wb) * w2b * 4 + size_t(n_pad) * 4);
    const size_t blb = up(size_t(wb) * 4) + up(size_t(wb) * kBList * 16);  // bcnt + blist
    const size_t xab = up(size_t(M) * wa * 4 + size_t(M) * w2a * 4 + size_t(m_pad) * 4);
    const size_t b_part = 2 * bh + 2 * ebb + xbb + blb;
    ScratchBuf *sb = bpre_scratch(st, b_part + 2 * ah + eab + xab);
    if (!sb) return cudaSuccess;
    uint8_t *scr = static_cast<uint8_t *>(sb->p);
    tp->wa = int(wa);
    tp->wb = int(wb);
    tp->w2a = int(w2a);
    tp->w2b = int(w2b);
    tp->xb = reinterpret_cast<unsigned *>(scr + 2 * bh + 2 * ebb);
    tp->sb2 = tp->xb + size_t(K) * wb;
    tp->fb = reinterpret_cast<int *>(tp->sb2 + size_t(wb) * w2b);
    tp->bcnt = reinterpret_cast<int *>(scr + 2 * bh + 2 * ebb + xbb);
    tp->blist = reinterpret_cast<int4 *>(scr + 2 * bh + 2 * ebb + xbb + up(size_t(wb) * 4));
    tp->xa = reinterpret_cast<unsigned *>(scr + b_part + 2 * ah + eab);
    tp->sa2 = tp->xa + size_t(M) * wa;
    tp->fa = reinterpret_cast<int *>(tp->sa2 + size_t(M) * w2a);
    tp->scheme = 4;
    tp->owner = sb;
    tp->ldah = ldah;
    tp->ldbh = ldbh;
    tp->Bh = reinterpret_cast<uint16_t *>(scr);
    tp->Bl = reinterpret_cast<uint16_t *>(scr + bh);
    tp->eb = reinterpret_cast<int *>(scr + 2 * bh);
    tp->bmax = reinterpret_cast<unsigned *>(scr + 2 * bh + ebb);
    tp->Ah = reinterpret_cast<uint16_t *>(scr + b_part);
    tp->Al = reinterpret_cast<uint16_t *>(scr + b_part + ah);
    tp->ea = reinterpret_cast<int *>(scr + b_part + 2 * ah);
    tp->key_b = sb->key_scheme == 4 ? sb->key_b : nullptr;
    tp->key_ldb = sb->key_ldb;
    tp->key_k = sb->key_k;
    tp->key_n = sb->key_n;
    return cudaSuccess;
  }
  // $GIGA_B_PRE=0: the transform warps build B' per tile (and A' too); $GIGA_A_PRE=0: A' only
  static const bool b_pre_env = [] {
    const char *e = getenv("GIGA_B_PRE");
    return !(e && *e == '0');
  }();
  static const bool a_pre_env = [] {
    const char *e = getenv("GIGA_A_PRE");
    return !(e && *e == '0');
  }();
  if (!b_pre_env) return cudaSuccess;
  const int64_t k8 = (K + 7) / 8 * 8, ldx = (N + 7) / 8 * 8;
  const size_t hi_b = up(size_t(K) * size_t(N) * 4), bx_b = up(size_t(2 * k8) * ldx * 2);
  const size_t hi_a = up(size_t(M) * size_t(K) * 4), ax_b = up(size_t(M) * size_t(2 * k8) * 2);
  ScratchBuf *sb = bpre_scratch(st, hi_b + bx_b + (a_pre_env ? hi_a + ax_b : 0));
  if (!sb) return cudaSuccess;  // no scratch (capture, OOM): operands built on chip
  uint8_t *scr = static_cast<uint8_t *>(sb->p);
  tp->owner = sb;
  tp->k8 = k8;
  tp->ldbx = ldx;
  tp->Bhi = reinterpret_cast<float *>(scr);
  tp->Bx = reinterpret_cast<uint16_t *>(scr + hi_b);
  if (a_pre_env) {
    tp->Ahi = reinterpret_cast<float *>(scr + hi_b + bx_b);
    tp->Ax = reinterpret_cast<uint16_t *>(scr + hi_b + bx_b + hi_a);
  }
  tp->key_b = sb->key_scheme == 2 ? sb->key_b : nullptr;
  tp->key_ldb = sb->key_ldb;
  tp->key_k = sb->key_k;
  tp->key_n = sb->key_n;
  return cudaSuccess;
}

bool TermsPrep::b_matches(const float *B, int64_t ldb, int64_t N, int64_t K) const {
  return (Bhi || Bh) && key_b == B && key_ldb == ldb && key_k == K && key_n == N;
}

cudaError_t launch_prep16_b(const float *B, int64_t ldb, int64_t N, int64_t K, TermsPrep *tp,
                            cudaStream_t st) {
  ScratchBuf *sb = static_cast<ScratchBuf *>(tp->owner);
  sb->key_b = nullptr;
  cudaError_t e = prep16_b_kernels(B, ldb, N, K, tp, st);
  if (e != cudaSuccess) return e;
  sb->key_b = tp->key_b = B;
  sb->key_ldb = tp->key_ldb = ldb;
  sb->key_k = tp->key_k = K;
  sb->key_n = tp->key_n = N;
  sb->key_scheme = 4;
  return cudaSuccess;
}



cudaError_t launch_prep_b(const float *B, int64_t ldb, int64_t N, int64_t K, TermsPrep *tp,
                          cudaStream_t st) {
  ScratchBuf *sb = static_cast<ScratchBuf *>(tp->owner);
  const int64_t units = (tp->k8 / 8) * (N / 4);
  const int64_t blocks = std::min<int64_t>((units + 255) / 256, int64_t(num_sms_current()) * 8);
  sb->key_b = nullptr;
  prep_b_kernel<<<unsigned(std::max<int64_t>(blocks, 1)), 256, 0, st>>>(
      B, ldb, int(K), int(N), const_cast<float *>(tp->Bhi), const_cast<uint16_t *>(tp->Bx),
      tp->ldbx);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  sb->key_b = tp->key_b = B;
  sb->key_ldb = tp->key_ldb = ldb;
  sb->key_k = tp->key_k = K;
  sb->key_n = tp->key_n = N;
  sb->key_scheme = 2;
  return cudaSuccess;
}

cudaError_t launch_prep_a(const float *A, int64_t lda, int64_t M, int64_t K, TermsPrep *tp,
                          cudaStream_t st) {
  const int64_t units = M * (tp->k8 / 8);
  const int64_t blocks = std::min<int64_t>((units + 255) / 256, int64_t(num_sms_current()) * 8);
  prep_a_kernel<<<unsigned(std::max<int64_t>(blocks, 1)), 256, 0, st>>>(
      A, lda, int(M), int(K), const_cast<float *>(tp->Ahi), const_cast<uint16_t *>(tp->Ax),
      2 * tp->k8);
  return cudaGetLastError();
}

cudaError_t launch_gemm_3xtf32(const float *A, const float *A_lo, const float *B,
                               const float *B_lo, float *C, int64_t M, int64_t N, int64_t K,
                               int64_t ldc, int terms, int promote_kblocks, cudaStream_t st,
                               int cta_group, const GemmExtra *ex) {
  using namespace cfg;
  GemmExtra dflt;
  if (!ex) ex = &dflt;
  const int64_t lda = ex->lda ? ex->lda : K, ldb = ex->ldb ? ex->ldb : N;
  if (M < 1 || N < 1 || K < 1 || (lda & 3) || (ldb & 3) || (ldc & 3) || ldc < N || lda < K ||
      ldb < N)
    return cudaErrorInvalidValue;
  if (M > INT32_MAX || N > INT32_MAX || K > INT32_MAX || ldc > INT32_MAX)
    return cudaErrorInvalidValue;
  if (terms < 1 || terms > 4) return cudaErrorInvalidValue;
  if (terms == 3 && (!A_lo) != (!B_lo)) return cudaErrorInvalidValue;  // both or neither
  if ((terms == 2 || terms == 4) && (A_lo || B_lo)) return cudaErrorInvalidValue;
  const bool lo_smem = terms == 3 && !A_lo;
  if (ensure_tma_encoder() != 0) return cudaErrorNotSupported;

  int num_sms = num_sms_current();
  if (ex->max_ctas > 0 && ex->max_ctas < num_sms) num_sms = ex->max_ctas & ~1;
  if (num_sms < 2) num_sms = 2;
  const int cg = (cta_group == 1 || cta_group == 2) ? cta_group : choose_cta_group(M, N, num_sms);
  CUtensorMap tA, tAlo, tB, tBlo;
  CMaps tC;
  if (ex->n_peer_c < 0 || ex->n_peer_c > kMaxCDst - 1) return cudaErrorInvalidValue;
  if (!make_map(&tA, A, K, M, lda, BK, BM, CU_TENSOR_MAP_SWIZZLE_64B) ||
      !make_map(&tB, B, N, K, ldb, 32, BK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) ||
      !make_map(&tC.m[0], C, N, M, ldc, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B))
    return cudaErrorInvalidValue;
  for (int i = 0; i < ex->n_peer_c; ++i)
    if (!make_map(&tC.m[1 + i], ex->peer_c[i], N, M, ldc, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B))
      return cudaErrorInvalidValue;
  if (terms == 3 && !lo_smem) {
    if (!make_map(&tAlo, A_lo, K, M, lda, BK, BM, CU_TENSOR_MAP_SWIZZLE_64B) ||
        !make_map(&tBlo, B_lo, N, K, ldb, 32, BK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B))
      return cudaErrorInvalidValue;
  } else {
    tAlo = tA;
    tBlo = tB;
  }

  GemmParams p;
  p.M = int(M);
  p.N = int(N);
  p.K = int(K);
  p.ldc = int(ldc);
  p.accumulate = ex->accumulate ? 1 : 0;
  p.load_c = ex->load_c ? 1 : 0;
  if (p.accumulate && p.load_c) return cudaErrorInvalidValue;
  p.terms = terms;
  p.lo_smem = lo_smem ? 1 : 0;
  static const int hi_rn_env = [] {  // terms == 2: $GIGA_HI_RN=0 keeps the truncated hi
    const char *e = getenv("GIGA_HI_RN");
    return (e && *e == '0') ? 0 : 1;
  }();
  p.hi_rn = hi_rn_env;
  p.b_pre = 0;
  p.a_pre = 0;
  p.ea = nullptr;
  p.eb = nullptr;
  p.fA = p.fB = nullptr;
  p.flda = p.fldb = p.fldbh = 0;
  p.fBh = p.fBl = nullptr;
  p.xb = p.sb2 = nullptr;
  p.fb = nullptr;
  p.w2b = 0;
  p.bcnt = nullptr;
  p.blist = nullptr;
  p.cta_ns = ex->cta_ns;
  // k-block width in elements of K: 16 (tf32 schemes), 32 (3xFP16)
  const int bk = terms == 4 ? 32 : BK;
  TermsPrep local4;
  const TermsPrep *tp4 = nullptr;
  if (terms == 4) {
    // scaled fp16 hi / lo operands (the caller's TermsPrep, else prepared here)
    TermsPrep &local = local4;
    const TermsPrep *tp = ex->prep;
    if (!tp || tp->scheme != 4) {
      cudaError_t e = terms_prep_alloc(M, N, K, st, &local, 4);
      if (e == cudaSuccess && !local.Bh) e = cudaErrorMemoryAllocation;
      if (e == cudaSuccess && !(ex->b_prep_reuse && local.b_matches(B, ldb, N, K)))
        e = launch_prep16_b(B, ldb, N, K, &local, st);
      if (e == cudaSuccess) e = launch_prep16_a(A, lda, M, K, &local, st);
      if (e != cudaSuccess) return e;
      tp = &local;
    }
    if (!make_map_bf16(&tA, tp->Ah, K, M, tp->ldah, 32, BM, CU_TENSOR_MAP_SWIZZLE_64B,
                       CU_TENSOR_MAP_DATA_TYPE_FLOAT16) ||
        !make_map_bf16(&tAlo, tp->Al, K, M, tp->ldah, 32, BM, CU_TENSOR_MAP_SWIZZLE_64B,
                       CU_TENSOR_MAP_DATA_TYPE_FLOAT16) ||
        !make_map_bf16(&tB, tp->Bh, N, K, tp->ldbh, 64, 32, CU_TENSOR_MAP_SWIZZLE_128B,
                       CU_TENSOR_MAP_DATA_TYPE_FLOAT16) ||
        !make_map_bf16(&tBlo, tp->Bl, N, K, tp->ldbh, 64, 32, CU_TENSOR_MAP_SWIZZLE_128B,
                       CU_TENSOR_MAP_DATA_TYPE_FLOAT16))
      return cudaErrorInvalidValue;
    p.ea = tp->ea;
    p.eb = tp->eb;
    // the B-side exception fix runs in the epilogue (fix_b_list / fix_b_block)
    p.fA = A;
    p.flda = lda;
    p.fB = B;
    p.fldb = ldb;
    p.fBh = tp->Bh;
    p.fBl = tp->Bl;
    p.fldbh = tp->ldbh;
    p.xb = tp->xb;
    p.sb2 = tp->sb2;
    p.fb = tp->fb;
    p.w2b = tp->w2b;
    p.bcnt = tp->bcnt;
    p.blist = tp->blist;
    tp4 = tp;
  }
  if (terms == 2) {
    // operands prepared in HBM (the caller's TermsPrep, else here, untimed)
    TermsPrep local;
    const TermsPrep *tp = ex->prep;
    if (!tp) {
      cudaError_t e = terms_prep_alloc(M, N, K, st, &local);
      if (e == cudaSuccess && local.Bhi && !(ex->b_prep_reuse && local.b_matches(B, ldb, N, K)))
        e = launch_prep_b(B, ldb, N, K, &local, st);
      if (e == cudaSuccess && local.Ahi) e = launch_prep_a(A, lda, M, K, &local, st);
      if (e != cudaSuccess) return e;
      tp = &local;
    }
    if (tp->Ahi && tp->Bhi) {
      if (!make_map(&tA, tp->Ahi, K, M, K, BK, BM, CU_TENSOR_MAP_SWIZZLE_64B) ||
          !make_map_bf16(&tAlo, tp->Ax, 2 * tp->k8, M, 2 * tp->k8, 32, BM,
                         CU_TENSOR_MAP_SWIZZLE_64B))
        return cudaErrorInvalidValue;
      p.a_pre = 1;
    }
    if (tp->Bhi) {
      if (!make_map(&tB, tp->Bhi, N, K, N, 32, BK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B) ||
          !make_map_bf16(&tBlo, tp->Bx, N, 2 * tp->k8, tp->ldbx, 64, 32))
        return cudaErrorInvalidValue;
      p.b_pre = 1;
    }
  }
  p.n_kb = int((K + bk - 1) / bk);
  int pk = promote_kblocks < 0 ? default_promote_kblocks(terms) : promote_kblocks;
  p.p_kb = (pk == 0 || pk > p.n_kb) ? p.n_kb : pk;
  // C's store mode: TMA, or 16-byte stores (unicast / one multicast store per piece)
  p.st_mode = ex->mc_c ? kStoreMulticast : ex->vec_store ? kStoreVec : kStoreTma;
  for (int i = 0; i < kMaxCDst; ++i) p.vdst[i] = nullptr;
  if (p.st_mode != kStoreTma) {
    if (p.accumulate || (N & 3) || (ldc & 3) || (reinterpret_cast<uintptr_t>(C) & 15) ||
        (ex->mc_c && (ex->n_peer_c || (reinterpret_cast<uintptr_t>(ex->mc_c) & 15))))
      return cudaErrorInvalidValue;
    p.vdst[0] = ex->mc_c ? ex->mc_c : C;
    for (int i = 0; i < ex->n_peer_c; ++i) {
      if (reinterpret_cast<uintptr_t>(ex->peer_c[i]) & 15) return cudaErrorInvalidValue;
      p.vdst[1 + i] = ex->peer_c[i];
    }
  }
  // (vector / multicast stores have no reduce-add: never the kSplitReduce K-split)
  const bool plain =
      !p.accumulate && !p.load_c && ex->n_peer_c == 0 && p.st_mode == kStoreTma;
  const GemmSchedule sch = gemm_schedule(M, N, K, num_sms, cg, plain, p.p_kb, bk);
  p.m_tiles = sch.m_tiles;
  p.n_tiles = sch.n_tiles;
  p.num_tiles = sch.num_tiles;
  static int group_env = [] {
    const char *e = getenv("GIGA_GROUP_M");
    return (e && atoi(e) > 0) ? atoi(e) : 0;
  }();
  p.group_m = group_env ? group_env : GROUP_M;
  p.sched = nullptr;
  p.wave_sync = 0;
  p.n_cdst = 1 + ex->n_peer_c;
  const int nclu = sch.nclu;
  // K-split (gemm_schedule): kSplitReduce halves reduce-add into C zeroed here; kSplitWorkspace
  // partials go through a workspace owned by this stream (ksplit_workspace).
  p.first_split = sch.first_split;
  p.split_s = sch.s;
  p.split_mode = sch.mode;
  p.sk_ws = nullptr;
  p.sk_cnt = nullptr;
  if (sch.mode == kSplitWorkspace) {
    const size_t slots = size_t(p.num_tiles - sch.first_split) * cg * NUM_EPI_WARPS;
    if (!ksplit_workspace(st, slots * sch.s * EPI_SLOT_BYTES, slots, &p.sk_ws, &p.sk_cnt)) {
      p.first_split = p.num_tiles;  // no workspace (capture, OOM): whole tiles
      p.split_s = 1;
      p.split_mode = kSplitNone;
    }
  } else if (sch.mode == kSplitReduce) {
    // zero the split tiles' bounding rectangle of C (tiles inside it that are not split are
    // stored over later in the same launch)
    int mlo = INT32_MAX, mhi = -1, nlo = INT32_MAX, nhi = -1;
    for (int t = p.first_split; t < p.num_tiles; ++t) {
      int mb, nb;
      tile_coords(t, p, mb, nb);
      mlo = std::min(mlo, mb);
      mhi = std::max(mhi, mb);
      nlo = std::min(nlo, nb);
      nhi = std::max(nhi, nb);
    }
    const int tile_m = BM * cg;
    const int64_t r0 = int64_t(mlo) * tile_m;
    const int64_t r1 = std::min<int64_t>(M, int64_t(mhi + 1) * tile_m);
    const int64_t c0 = int64_t(nlo) * BN, c1 = std::min<int64_t>(N, int64_t(nhi + 1) * BN);
    cudaError_t e = cudaMemset2DAsync(C + r0 * ldc + c0, size_t(ldc) * 4, 0,
                                      size_t(c1 - c0) * 4, size_t(r1 - r0), st);
    if (e != cudaSuccess) return e;
  }
  p.num_units = p.first_split + (p.num_tiles - p.first_split) * p.split_s;
  // producers' per-wave barrier: $GIGA_WAVE_SYNC=0 disables it, s >= 1 lets a producer run
  // s - 1 waves ahead of the slowest cluster [1]
  static const int wave_env = [] {
    const char *e = getenv("GIGA_WAVE_SYNC");
    return (e && *e >= '0' && *e <= '9') ? atoi(e) : 1;
  }();
  static const bool dyn_env = [] {  // $GIGA_DYNAMIC_SCHED=0: static round-robin units
    const char *e = getenv("GIGA_DYNAMIC_SCHED");
    return !(e && *e == '0');
  }();
  // the launch's dynamic-schedule counters (per device and stream: concurrent launches on
  // other streams have their own); none inside a capture that has not seen this stream yet
  if (dyn_env) p.sched = sched_counters(st);
  p.wave_sync = p.num_units > nclu ? wave_env : 0;
  cudaError_t e = cudaSuccess;

  if (cg == 1) {
    e = ensure_smem_attr<1>();
    if (e != cudaSuccess) return e;
    const int grid = p.num_units < num_sms ? p.num_units : num_sms;
    gemm_3xtf32_kernel<1><<<grid, NUM_THREADS, Tile<1>::SMEM_BYTES, st>>>(tA, tAlo, tB, tBlo,
                                                                          tC, p);
    e = cudaGetLastError();
    if (e == cudaSuccess && tp4 && !ex->defer_fix)
      e = launch_fix16(A, lda, B, ldb, M, N, K, tp4, C, ldc, ex, st);
    return e;
  }
  e = ensure_smem_attr<2>();
  if (e != cudaSuccess) return e;
  const int pairs = num_sms / 2;
  const int clusters = p.num_units < pairs ? p.num_units : pairs;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(unsigned(2 * clusters));
  lc.blockDim = dim3(NUM_THREADS);
  lc.dynamicSmemBytes = Tile<2>::SMEM_BYTES;
  lc.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  e = cudaLaunchKernelEx(&lc, gemm_3xtf32_kernel<2>, tA, tAlo, tB, tBlo, tC, p);
  if (e == cudaSuccess && tp4 && !ex->defer_fix)
    e = launch_fix16(A, lda, B, ldb, M, N, K, tp4, C, ldc, ex, st);
  return e;
}

}  // namespace giga

// Bring-up probe (libgiga_debug.so only calls it): how many clusters of `cluster_size` CTAs
// with this kernel's resources (384 threads, Tile<2>::SMEM_BYTES) fit on the device at once.
extern "C" int giga_dbg_max_active_clusters(int cluster_size) {
  using namespace giga;
  if (ensure_smem_attr<2>() != cudaSuccess) return -1;
  if (cluster_size > 8)
    cudaFuncSetAttribute(gemm_3xtf32_kernel<2>, cudaFuncAttributeNonPortableClusterSizeAllowed,
                         1);
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(unsigned(cluster_size * 64));
  lc.blockDim = dim3(cfg::NUM_THREADS);
  lc.dynamicSmemBytes = Tile<2>::SMEM_BYTES;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = unsigned(cluster_size);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  lc.attrs = attr;
  lc.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, gemm_3xtf32_kernel<2>, &lc) != cudaSuccess) return -2;
  return n;
}
