// kernels.h -- host-side launchers of the sm_100a kernels (internal to libgiga).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace giga {

// Default number of 16-wide k-blocks accumulated in TMEM before promotion into the fp32
// register sum. 8 k-blocks = K 128 = 16 k8 steps.
// The TF32 + BF16 scheme adds 2 MMAs per k8 step into TMEM instead of 3; 16 k-blocks would be
// 2% faster but raise its adversarial coherent-error case from 5.0e-6 to 7.3e-6 of the 1e-5
// bound, so it keeps 8 too.
constexpr int kDefaultPromoteKBlocks = 8;
constexpr int kDefaultPromoteKBlocksT2 = 8;
// The 3xFP16 scheme (terms = 4) runs 32-wide k-blocks: 8 of them = K 256 per TMEM partial
// (24 truncating adds per K 128 instead of 3xTF32's 48: the same count per partial as 3xTF32 at
// K 128; measured +8% at 32768^3, worst long-K all-positive error 2.2e-6 vs 1.5e-6 at 4).
constexpr int kDefaultPromoteKBlocksT4 = 8;

// The promotion interval in effect for `terms` (the defaults above or $GIGA_PROMOTE_KBLOCKS).
int default_promote_kblocks(int terms = 3);

// The product path's fp32-accurate scheme for an M x N x K launch:
// 4 = 3xFP16 (the 3xTF32 split on fp16 operands of power-of-two scaled rows / columns, three
// K=16 kind::f16 MMAs per k16 step, operands prepared once per launch in HBM, exceptions fixed)
// where the preparation is amortised: M >= 2048, M N K >= 2^37 and either K, N >= 2048 or
// K >= 1024 with N >= 8192;
// else 2 = TF32 + BF16 (hi*hi as kind::tf32, both corrections as one K=16 kind::f16 MMA) for
// M >= 4096, N >= 8192, K >= 512, M N K >= 2^38; else 3 = 3xTF32 (three kind::tf32 MMAs per
// k8 step, no preparation). Measured crossovers. $GIGA_SCHEME = "3xtf32" / "tf32bf16" /
// "3xfp16" forces one. With pre-split lo operands (A_lo != nullptr) the scheme is always 3.
int product_terms(const float *A_lo, int64_t M, int64_t N, int64_t K);
// true when $GIGA_SCHEME forces the scheme (measurements keep it even without scratch)
bool scheme_forced();

// lo = x - tf32(x) over n elements (HBM-bound elementwise split).
cudaError_t launch_split_lo(const float *x, float *lo, int64_t n, cudaStream_t st);
// The same over a rows x cols block of a row-major matrix with row stride ld (cols, ld % 4 == 0).
cudaError_t launch_split_lo_2d(const float *x, float *lo, int64_t rows, int64_t cols,
                               int64_t ld, cudaStream_t st);

// C[M x N, row stride ldc] = A[M x K] * B[K x N] by 3xTF32 (terms = 3) or 1xTF32 (terms = 1)
// on the tcgen05 tensor cores. Requires K % 4 == 0, N % 4 == 0, ldc % 4 == 0, 16B-aligned
// pointers. promote_kblocks: 0 = never, -1 = default. cta_group: 1 (128x256 tile per CTA),
// 2 (256x256 tile per CTA pair), 0 = chosen by shape. Returns cudaErrorInvalidValue for bad
// shapes, or the launch error.
// Extra operand/launch options: lda / ldb = row strides of A and B in elements (0 = K and
// N, i.e. dense; K-chunked pipelines pass A + k0 with lda = the full K); accumulate = 1 adds
// into C (C += A*B, fp32 RN) instead of overwriting; max_ctas caps the persistent grid (SMs
// left free for concurrent communication kernels; 0 = all SMs); peer_c[0..n_peer_c) are
// further C buffers (same shape and ldc, e.g. the peers' C_full rows over NVLink) that receive
// the same tiles from the epilogue: the gather fused into the GEMM. load_c = 1 (with
// accumulate = 0): the epilogue first reads each block of C and adds it (fp32 RN, the same
// bits as accumulate's reduce-add), then stores the sum to C and every peer -- the last chunk
// of a K-chunked series, so that only final values cross NVLink.
constexpr int kMaxCDst = 8;
// Operands of the TF32 + BF16 scheme prepared in HBM (per-stream scratch, library-owned):
// B_hi = RN tf32(B), B' = bf16 [b ; b_lo] per k8 block (ldbx columns), A_hi = RN tf32(A),
// A' = bf16 [a_lo | a_hi] per k8 block (2 * k8 columns). Null pointers: that operand is built
// by the GEMM's transform warps. key_*: what the B part holds now.
struct TermsPrep {
  const float *Ahi = nullptr, *Bhi = nullptr;
  const uint16_t *Ax = nullptr, *Bx = nullptr;
  int64_t k8 = 0, ldbx = 0;
  // 3xFP16 scheme (terms = 4): fp16 hi / lo of the power-of-two scaled operands, row-major
  // (A: M x K, row stride ldah; B: K x N, row stride ldbh), and the scale exponents: row i
  // of A was scaled by 2^-ea[i], column j of B by 2^-eb[j]
  const uint16_t *Ah = nullptr, *Al = nullptr, *Bh = nullptr, *Bl = nullptr;
  const int *ea = nullptr, *eb = nullptr;
  unsigned *bmax = nullptr;  // per-column max |b| bits (preparation scratch)
  int64_t ldah = 0, ldbh = 0;
  // exceptions (elements the fp16 split cannot carry to 2^-20): bitmaps (A: M rows of wa
  // words, B: K rows of wb words) and per-row / per-column flags
  unsigned *xa = nullptr, *xb = nullptr;
  int *fa = nullptr, *fb = nullptr;
  int wa = 0, wb = 0;
  // summaries of the bitmaps (bit w % 32 of word w / 32 set iff bitmap word w is non-zero):
  // A per row (w2a words), B per 32-column strip (w2b words over its K words)
  unsigned *sa2 = nullptr, *sb2 = nullptr;
  int w2a = 0, w2b = 0;
  // per strip of 32 columns of B: its exception count and list (compact16_b_kernel)
  int *bcnt = nullptr;
  int4 *blist = nullptr;
  int scheme = 2;
  void *owner = nullptr;
  const float *key_b = nullptr;
  int64_t key_ldb = 0, key_k = 0, key_n = 0;
  bool b_matches(const float *B, int64_t ldb, int64_t N, int64_t K) const;
};
// Reserve the scratch for an M x N x K product on `st` (pointers stay null when it cannot be
// had: stream capture, OOM, $GIGA_B_PRE=0), then prepare B and A into it (stream-ordered).
cudaError_t terms_prep_alloc(int64_t M, int64_t N, int64_t K, cudaStream_t st, TermsPrep *tp,
                             int terms = 2);
cudaError_t launch_prep_b(const float *B, int64_t ldb, int64_t N, int64_t K, TermsPrep *tp,
                          cudaStream_t st);
cudaError_t launch_prep_a(const float *A, int64_t lda, int64_t M, int64_t K, TermsPrep *tp,
                          cudaStream_t st);
// Operand preparation of the 3xFP16 scheme (terms = 4): per-row exponents of A / per-column
// exponents of B and the fp16 hi / lo arrays of the scaled operands (stream-ordered).
cudaError_t launch_prep16_b(const float *B, int64_t ldb, int64_t N, int64_t K, TermsPrep *tp,
                            cudaStream_t st);
cudaError_t launch_prep16_a(const float *A, int64_t lda, int64_t M, int64_t K, TermsPrep *tp,
                            cudaStream_t st);
struct GemmExtra {
  int64_t lda = 0, ldb = 0;
  int accumulate = 0;
  int max_ctas = 0;
  float *const *peer_c = nullptr;
  int n_peer_c = 0;
  int load_c = 0;
  // TF32 + BF16 scheme: 1 = B (same pointer, ldb, K, N) is unchanged since the previous launch
  // on this stream (row chunks of one product), so its prepared B_hi / B' are reused
  int b_prep_reuse = 0;
  // rows that share this B (row blocks / row chunks of one product): the scheme choice
  // amortises B's preparation over them (0 = this launch's M)
  int64_t rows_hint = 0;
  const TermsPrep *prep = nullptr;  // terms = 2: operands already prepared by the caller
  // terms = 4: 1 = the caller launches the exception fixes itself (launch_fix16, after the GEMM
  // on the same stream; run_gemm does, to time them apart from the GEMM)
  int defer_fix = 0;
  // $GIGA_TRACE: 2 x (grid size) slots; each CTA writes %globaltimer at its start and its end
  uint64_t *cta_ns = nullptr;
  // How the epilogue writes the staged C blocks ("Multicast
  // gather"):
  //   mc_c != nullptr: the NVLink multicast address of the same rows as C (C and every peer's
  //     C_full bound into one cuMulticastCreate team): each 16-byte piece is written ONCE with
  //     multimem.st and the switch replicates it into every member, C included (peer_c must
  //     be empty). Needs N % 4 == 0 and 16-byte aligned C; no accumulate.
  //   vec_store = 1: C and peer_c written with 16-byte st.global stores from the staging tile
  //     (the same addressing as the multicast mode, unicast; no accumulate) instead of TMA.
  float *mc_c = nullptr;
  int vec_store = 0;
};
// One thread writes %globaltimer (ns) to *slot when `st` reaches it (trace stamps).
cudaError_t launch_stamp(uint64_t *slot, cudaStream_t st);
// The 3xFP16 A-side exception fix of a launch whose GEMM ran with defer_fix (same arguments;
// the B-side fix runs inside the GEMM's epilogue).
cudaError_t launch_fix16(const float *A, int64_t lda, const float *B, int64_t ldb, int64_t M,
                         int64_t N, int64_t K, const TermsPrep *tp, float *C, int64_t ldc,
                         const GemmExtra *ex, cudaStream_t st);
// B's preparation kernels alone (prep16.cu; launch_prep16_b adds the reuse bookkeeping).
cudaError_t prep16_b_kernels(const float *B, int64_t ldb, int64_t N, int64_t K,
                             const TermsPrep *tp, cudaStream_t st);
// Kernels launch_prep16_b / launch_prep16_a / launch_fix16 issue (bench.py's launch count).
constexpr int kPrep16BLaunches = 4, kPrep16ALaunches = 1, kFix16Launches = 1;
cudaError_t launch_gemm_3xtf32(const float *A, const float *A_lo, const float *B,
                               const float *B_lo, float *C, int64_t M, int64_t N, int64_t K,
                               int64_t ldc, int terms, int promote_kblocks, cudaStream_t st,
                               int cta_group = 0, const GemmExtra *ex = nullptr);

// out[0] = sum_i x[i]*y[i] over n elements, fp64 accumulation (vecops.cu). `partials` must
// hold kDotMaxBlocks doubles and `ticket` must be zero before the first launch (the kernel
// resets it). Deterministic for a given device.
constexpr int kDotMaxBlocks = 2048;
cudaError_t launch_dot(const float *x, const float *y, int64_t n, double *partials,
                       unsigned *ticket, double *out, cudaStream_t st);

// K-split plan of a launch (gemm_3xtf32.cu): tiles [0, first_split) run whole, the rest as s
// k-parts each, combined deterministically: kSplitReduce = two halves TMA reduce-add into a
// zeroed C (plain-store launches), kSplitWorkspace = partials summed in part order by the
// last part to finish.
enum { kSplitNone = 0, kSplitReduce = 1, kSplitWorkspace = 2 };
struct KSplitPlan {
  int first_split, s, mode;
};
KSplitPlan plan_ksplit(int num_tiles, int nclu, int n_kb, int cg, bool plain, int p_kb);
// The launch's tiling and unit schedule for an M x N x K product on num_sms SMs (cta_group 0:
// chosen from the shape; plain: C = A*B stored, no accumulate / load_c / peers; p_kb: the
// promotion interval in k-blocks), as launch_gemm_3xtf32 computes it.
struct GemmSchedule {
  int cg, m_tiles, n_tiles, num_tiles, nclu, n_kb, first_split, s, mode, num_units;
};
GemmSchedule gemm_schedule(int64_t M, int64_t N, int64_t K, int num_sms, int cta_group,
                           bool plain, int p_kb, int bk = 16);
// Workspace of the K-split partials for launches on `st` (current device); false when it
// cannot be had (stream capture, out of memory): the launch then runs whole tiles.
bool ksplit_workspace(cudaStream_t st, size_t ws_bytes, size_t cnt_n, float **ws,
                      unsigned **cnt);
// The GEMM's dynamic-schedule counters for launches on `st` (current device): created zeroed
// on first use (outside a capture; nullptr otherwise: the launch then runs static
// round-robin units without the wave barrier).
unsigned *sched_counters(cudaStream_t st);
// Frees the K-split workspaces of every device (giga_finalize).
void release_gemm_caches();
// A library buffer superseded by a larger one (workspace growth): freed at once, unless a
// CUDA graph has captured library work (keep_superseded_buffers()), in which case it stays
// allocated until giga_finalize -- an earlier graph may still reference it.
void retire_buffer(void *p);
void keep_superseded_buffers();

// Resolves cuTensorMapEncodeTiled through the runtime (no libcuda link). 0 on success.
int ensure_tma_encoder();

// CTA-group size the GEMM launch will use for an M x N shard (1 or 2; $GIGA_CTA_GROUP).
int choose_cta_group(int64_t M, int64_t N, int num_sms);

}  // namespace giga
