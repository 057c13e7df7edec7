/*
 * giga.h -- C ABI of the B200-native GigaAPI matrix multiply (arXiv 2504.01266).
 *
 * The operation (S4.2.7 "Matrix Multiplication"):
 *     C[i][j] = sum_k A[i][k] * B[k][j]
 * "each element in C[i,j] is calculated by taking a dot product of the i-th row of the
 *  matrix A and the j-th column of matrix B", the sum "reported and assigned at the end"
 * (PAPER.md:291): C is fully OVERWRITTEN, its prior contents never matter (the paper's
 * dirty-memory bug, cannot happen).
 *
 * Distribution ("we effectively half them ... half the multiplications are
 * carried out on one GPU ... copy over half the matrices"; generalised to g GPUs per
 * PAPER.md:311): the rows of A (and C) are split into contiguous blocks, one per GPU; every
 * GPU receives a full copy of B; the C row blocks are gathered. giga_partition() states the
 * split rule.
 *
 * Layout: every matrix is dense row-major fp32 (SPEC.md:234-236 MatrixF32); A is M x K
 * (row stride K), B is K x N (row stride N), C is M x N (row stride N). No transposes, no
 * alpha/beta.
 *
 * Precision: fp32 in, fp32 out, fp32-accurate: internally each product is formed from
 * hi / lo parts with 11-bit significands on the tcgen05 tensor cores (a_lo*b_hi + a_hi*b_lo +
 * a_hi*b_hi) -- 3xTF32, or for large launches 3xFP16 (the same split on fp16 operands of
 * power-of-two scaled rows of A / columns of B; the few elements fp16 cannot carry are fixed
 * in fp64) or TF32 + BF16 (a_hi*b_hi in TF32, a_lo*b + a_hi*b_lo in one BF16 MMA);
 * giga_product_scheme -- with partial sums promoted into fp32 registers, so that per
 * element
 *     |C - C_exact| <= 1e-5 * sum_k |A_ik| |B_kj|          (BASELINE.json north_star)
 * and integer-valued inputs whose partial sums stay below 2^24 give bit-exact results.
 * Non-finite inputs: NaN propagates; Inf may turn into NaN (Inf - Inf in the split; a row of
 * A / column of B holding Inf or NaN gives Inf or NaN in its row / column of C under 3xFP16).
 *
 * Errors: every function returns GIGA_OK (0) or a negative giga_status; the message of the
 * last failure on the calling thread is in giga_last_error(). After a failed call the
 * device memory in use equals its value before the call (no leaks; the workspace cache is
 * only grown by successful calls and is released by giga_finalize).
 *
 * Ownership: the caller owns every pointer passed in; the library never keeps a caller
 * pointer after returning. The library owns its streams, events, communicators and
 * workspace (padded copies, host-path staging buffers, the TF32 + BF16 and 3xFP16 prepared
 * operands, scales and exception bitmaps, the pre-split low parts in that comparison mode),
 * freed in giga_finalize().
 *
 * Threading: calls are serialised by an internal mutex (one call at a time per process).
 *
 * Determinism: for a given shape, device count and environment every call returns the same
 * bits (fixed reduction orders everywhere; no atomics decide an order of additions).
 *
 * Environment (read at call time unless noted; defaults in brackets):
 *   GIGA_TRANSPORT       nccl | p2p: the N > 1 exchange (NCCL collectives, or copy engines for
 *                        B and the gather fused into the GEMM epilogue) [nccl]
 *   GIGA_P2P_STORE       tma | vec: how the p2p fused gather writes the peers' C_full from the
 *                        epilogue -- TMA stores, or 16-byte st.global stores (the code path
 *                        of the multicast gather, giga_mc_alloc, one store per peer) [tma]
 *   GIGA_BCAST_CHUNKS, GIGA_GATHER_CHUNKS  chunk counts of the N > 1 plans [6 / 16 p2p, 4]
 *   GIGA_COMM_SMS, GIGA_NCCL_MAX_CTAS      SMs left to NCCL beside the GEMM [8, = COMM_SMS]
 *   GIGA_NCCL_CTA_GBPS   per-CTA NCCL rate of the N > 1 plan's transfer model [50]
 *   GIGA_FORCE_COMM      1: run the NCCL pipeline even at one GPU (testing) [0]
 *   GIGA_TRACE           1: print a JSON timeline of each pipelined call on stderr (CUDA-event
 *                        times, transfer GB/s, p2p: %globaltimer copy / GEMM-CTA intervals) [0]
 *   GIGA_HOST_H2D_GBS, GIGA_HOST_D2H_GBS, GIGA_HOST_GEMM_TFLOPS, GIGA_HOST_GEMM4_TFLOPS
 *                        rates of the host-path schedule model [50, 50, 250, 440 (3xFP16)]
 *   GIGA_HOST_PLAN       "Me,P,Q": force that host-path schedule (measurements) [planned]
 *   GIGA_SCHEME          3xtf32 | tf32bf16 | 3xfp16: force the product scheme (once) [by shape]
 *   GIGA_HI_RN, GIGA_A_PRE, GIGA_B_PRE  TF32 + BF16: 0 = truncated hi / A' / B' built on chip
 *                        instead of RN hi / prepared in HBM (measurements; once) [1, 1, 1]
 *   GIGA_LO_PRESPLIT     1: 3xTF32 low parts split in HBM (comparison mode; once) [0]
 *   GIGA_PROMOTE_KBLOCKS TMEM accumulation interval in k-blocks, 16 deep (32 for 3xFP16)
 *                        (once) [8]
 *   GIGA_CTA_GROUP       1 | 2: force the GEMM tile variant (once) [by shape]
 *   GIGA_WAVE_SYNC, GIGA_TAIL_SPLIT  0 disables the GEMM's wave barrier / tail split (once) [1]
 *   GIGA_GROUP_M, GIGA_L2_PROMO      raster group, TMA L2 promotion (once) [8, 2 = 128 B]
 *   GIGA_NCCL_PATH       libnccl.so.2 to dlopen if the default lookup fails
 */
#ifndef GIGA_H_
#define GIGA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum giga_status {
  GIGA_OK = 0,
  GIGA_ERR_INVALID_ARG = -1,         /* M, N or K < 1; ngpus out of range; NULL pointer;
                                        C overlapping A or B; misaligned device pointer */
  GIGA_ERR_NOT_INITIALIZED = -2,     /* call before giga_init / giga_rank_init */
  GIGA_ERR_ALREADY_INITIALIZED = -3, /* init twice without giga_finalize */
  GIGA_ERR_NO_DEVICE = -4,           /* no sm_100 GPU, or fewer than requested */
  GIGA_ERR_OOM = -5,                 /* device (or pinned host) allocation failed */
  GIGA_ERR_CUDA = -6,                /* any other CUDA runtime/driver failure */
  GIGA_ERR_COMM = -7,                /* NCCL / peer-transport failure */
  GIGA_ERR_UNSUPPORTED = -8          /* valid request this build cannot serve */
};
/* SURVEY.md 8(b)'s name for the communication failure (it also covers the p2p transport). */
#define GIGA_ERR_NCCL GIGA_ERR_COMM

/* ------------------------------------------------------------------------------------ */
/* Single-process API: one process drives g GPUs (the paper's GigaGPU object). */

/* Initialise the library on GPUs 0..n-1, n = ngpus_max (ngpus_max <= 0: all visible GPUs).
 * Creates per-GPU compute and copy streams, events, enables peer access between the GPUs
 * and resolves the TMA descriptor encoder. Errors: ALREADY_INITIALIZED, NO_DEVICE
 * (fewer than n sm_100 GPUs), CUDA. */
int giga_init(int ngpus_max);

/* As giga_init on an explicit list of CUDA ordinals: library GPU g runs on devices[g].
 * Ordinals may repeat: several "virtual GPUs" then share one device, each with its own
 * streams and workspace, and the multi-GPU schedules run unchanged with device-local copies
 * (how the N > 1 paths are exercised on a one-GPU machine). NCCL refuses repeated devices,
 * so with repeats only $GIGA_TRANSPORT=p2p serves ngpus > 1. Errors: as giga_init,
 * INVALID_ARG (NULL / n < 1). */
int giga_init_devices(const int *devices, int n);

/* Number of GPUs the library was initialised with (0 if not initialised). */
int giga_num_devices(void);

/* Release everything giga_init / giga_rank_init created (streams, events, communicators,
 * workspace). Safe to call when not initialised (returns GIGA_OK). */
int giga_finalize(void);

/* The row-block rule (PAPER.md:287 halving generalised; "last device takes
 * remainder"): rows_g = floor(M / ngpus) for g < ngpus-1, the last GPU takes
 * M - (ngpus-1)*floor(M/ngpus); row0_g = g*floor(M/ngpus). Shards may be empty when
 * M < ngpus. Pure host arithmetic; needs no initialisation. Errors: INVALID_ARG. */
int giga_partition(int64_t M, int ngpus, int g, int64_t *row0, int64_t *rows);

/* C = A * B on GPUs 0..ngpus-1.
 * A, B, C: either all HOST pointers (pageable or pinned) -- the paper's semantics: the
 * library copies each A row block and B to the GPUs, computes, and copies each GPU's C row
 * block straight back into C -- or all DEVICE pointers on GPU 0 (A, B, C as M x K, K x N,
 * M x N buffers); the result then lands in C on GPU 0. Blocking: returns after C holds the
 * result. Errors: NOT_INITIALIZED, INVALID_ARG (M,N,K < 1; ngpus not in
 * [1, giga_num_devices()]; NULL; C overlapping A or B; mixed host/device pointers),
 * OOM, CUDA, COMM. */
int giga_matmul(const float *A, const float *B, float *C, int64_t M, int64_t N, int64_t K,
                int ngpus);

/* Device-resident, pre-sharded hot path (what bench.py times). Transport for ngpus > 1
 * ($GIGA_TRANSPORT): "nccl" (default) = NCCL broadcast of B in K-chunks overlapped with
 * accumulating GEMMs + row-chunked NCCL gather of C; "p2p" = copy-engine chain broadcast of B
 * (no SMs) + the gather fused into the GEMM epilogue (TMA stores of every C tile into every
 * GPU's C_full over NVLink).
 * A_shard[g]: device pointer on GPU g to the rows_g x K block of A (giga_partition rule).
 * B_buf[0]:   device pointer on GPU 0 holding B (K x N). B_buf[g>0]: K x N receive buffers
 *             on GPU g, overwritten with B.
 * C_full[g]:  device pointer on GPU g to an M x N buffer; on return EVERY GPU holds the full
 *             C (the row blocks are gathered).
 * Errors: as giga_matmul. */
int giga_matmul_sharded(const float *const *A_shard, float *const *B_buf,
                        float *const *C_full, int64_t M, int64_t N, int64_t K, int ngpus);

/* Message describing the last failure on this thread ("" if none). */
const char *giga_last_error(void);

/* ------------------------------------------------------------------------------------ */
/* Multi-process API: one process per GPU (torchrun), a communicator across the processes.
 * Rank 0 calls giga_comm_unique_id and ships the 128 bytes to the others (any channel,
 * e.g. torch.distributed); then every rank calls giga_rank_init. */

int giga_comm_unique_id(uint8_t id[128]);

/* rank in [0, world), device = the CUDA ordinal this process drives. Errors:
 * ALREADY_INITIALIZED, INVALID_ARG, NO_DEVICE, COMM. */
int giga_rank_init(int rank, int world, int device, const uint8_t id[128]);

/* This rank's share of C = A * B, device pointers on this rank's GPU:
 * A_shard: rows_r x K block (giga_partition(M, world, rank)); B: K x N (source on rank 0,
 * receive buffer elsewhere); C_full: M x N, holds the full C on return on every rank.
 * Work is enqueued on `stream` (a cudaStream_t, NULL = the library's stream) and the call
 * returns without synchronising the host (stream-ordered). The call can be captured into a
 * CUDA graph on `stream` after one eager call with the same shapes (which sizes the
 * library's per-stream workspaces); inside a capture it does not order itself against
 * earlier eager calls -- the graph's stream does. Errors: NOT_INITIALIZED, INVALID_ARG,
 * CUDA, COMM. */
int giga_matmul_rank(const float *A_shard, float *B, float *C_full, int64_t M, int64_t N,
                     int64_t K, void *stream);

/* ------------------------------------------------------------------------------------ */
/* Vector operations, the paper's second data-parallel workload (S4.2.8;
 * SPEC.md:284-301): the index range [0, n) is split with giga_partition's rule ("halving,
 * with remainder going on one"), every GPU reduces its range, the partials are summed.
 * Each product of two fp32 values is formed exactly in fp64 and summed in fp64, so
 * |result - exact| <= 2 n 2^-53 sum_i |x_i y_i|; integer-valued inputs give the exact sum.
 * Deterministic for a given device and n. */

/* *result = sum_i x[i] * y[i] on GPUs 0..ngpus-1. x, y: both HOST pointers (copied per GPU)
 * or both DEVICE pointers on GPU 0 (ranges copied to the other GPUs over NVLink). The host
 * sums the per-GPU partials in device order. Blocking. Errors: NOT_INITIALIZED,
 * INVALID_ARG (NULL, n < 1, ngpus out of range, mixed pointer kinds), OOM, CUDA. */
int giga_dot(const float *x, const float *y, int64_t n, int ngpus, double *result);

/* *result = sqrt(giga_dot(x, x)): the square root once, on the host, at the end. */
int giga_l2norm(const float *x, int64_t n, int ngpus, double *result);

/* Rank API: this rank's range of x and y (device pointers, giga_partition(n, world, rank)
 * elements); the partials are all-reduced (NCCL, fp64 sum) so every rank's *result (host)
 * holds the full dot. Enqueued on `stream`, then synchronised. Errors as giga_matmul_rank. */
int giga_dot_rank(const float *x_shard, const float *y_shard, int64_t n, double *result,
                  void *stream);

/* The N > 1 pipeline's chunk plan (pure host arithmetic, identical on every rank; the
 * orchestration of giga_matmul_sharded / giga_matmul_rank uses exactly these functions).
 * B is broadcast from rank 0 in *kchunks K-row chunks [kbounds[c], kbounds[c+1]) (kbounds
 * needs room for 17 entries), growing geometrically so the GEMM starts after a small first
 * chunk; the shard GEMM accumulates chunk by chunk, and the C row blocks are gathered in
 * *rchunks rounds; in round q owner o broadcasts the rows returned by
 * giga_plan_block(M, world, rchunks, o, q) (largest first). The counts (at most 6 K-chunks
 * with NCCL, 16 with $GIGA_TRANSPORT=p2p; at most 4 row chunks) minimise a model of the
 * exposed first transfer and last gather plus ~20 us per extra GEMM launch ($GIGA_LAUNCH_US);
 * $GIGA_BCAST_CHUNKS and $GIGA_GATHER_CHUNKS force them.
 * Errors: INVALID_ARG. */
int giga_pipeline_plan(int64_t M, int64_t N, int64_t K, int world, int *kchunks,
                       int64_t *kbounds, int *rchunks);
int giga_plan_block(int64_t M, int world, int rchunks, int owner, int q, int64_t *row0,
                    int64_t *rows);

/* The schedule giga_matmul uses for HOST buffers on one GPU (inputs built
 * on the host, results copied back; PCIe both ways overlapped with the GEMM):
 *   phase 1: rows [0, *Me): K-chunk c = [kb[c], kb[c+1]) of A's columns and B's rows is
 *            copied host->device, then its GEMM accumulates into C[0:Me];
 *   phase 2: row blocks [rb[q], rb[q+1]) (rb[0] = *Me, rb[*Q] = M) over the full K; each block's
 *            C rows are copied back while the next computes (the early rows after phase 1).
 * Chosen by a three-engine (H2D, GEMM, D2H) model over a few thousand candidates; *t_model is
 * its makespan in seconds. kb and rb need room for 17 entries each. num_sms <= 0 means 148.
 * Model rates: $GIGA_HOST_H2D_GBS, $GIGA_HOST_D2H_GBS (50), $GIGA_HOST_GEMM_TFLOPS (255).
 * No GPU needed. Errors: INVALID_ARG. */
int giga_host_plan(int64_t M, int64_t N, int64_t K, int num_sms, int64_t *Me, int *P,
                   int64_t *kb, int *Q, int64_t *rb, double *t_model);

/* Peer-to-peer transport for the rank API ($GIGA_TRANSPORT=p2p, set before giga_rank_init;
 * no NCCL communicator is created then, and several ranks may share one device). Each rank
 * registers the B and C_full buffers it will pass to giga_matmul_rank:
 *   giga_rank_p2p_export fills GIGA_P2P_BLOB_BYTES bytes (CUDA IPC handles of B, C_full and a
 *   library flag page); the caller all-gathers the blobs (any channel, e.g.
 *   torch.distributed) into world * GIGA_P2P_BLOB_BYTES bytes ordered by rank and passes them
 *   to giga_rank_p2p_import on every rank.
 * giga_matmul_rank then pulls B down a rank chain in K-chunks with copy engines and writes
 * each rank's C rows straight into every rank's C_full from the GEMM epilogue, ordered across
 * processes by device-side flags (no host synchronisation); giga_dot_rank all-reduces through
 * the flag pages. Errors: NOT_INITIALIZED, INVALID_ARG (not device allocations / wrong
 * world), UNSUPPORTED, CUDA. */
#define GIGA_P2P_BLOB_BYTES 256
int giga_rank_p2p_export(const float *B, float *C_full, uint8_t *blob);
int giga_rank_p2p_import(const uint8_t *blobs, int world);

/* ------------------------------------------------------------------------------------ */
/* NVLink multicast C_full buffers: the fused gather with ONE store per piece of C (SURVEY.md
 * 8(f) N4). The gather is a concatenation of the GPUs' row blocks (S4.2.3;
 * PAPER.md:291, S4.2.7). When the C_full buffers the p2p transport is given were allocated
 * here, they are bound into one cuMulticastCreate team: the last K-chunk's GEMM epilogue (and
 * the 3xFP16 A-side fix) writes each 16-byte piece of its rows once, with multimem.st to the
 * team's multicast address, and the NVSwitch replicates it into every GPU's C_full -- NVLink
 * egress 1 x the GPU's rows instead of (g - 1) x with the unicast stores to every peer. With
 * ordinary buffers the transport keeps the unicast gather. Requires N % 4 == 0 (as the p2p
 * transport does). The buffers are zero-filled device memory owned by the library, valid
 * until freed / giga_finalize. NOT RUN on hardware yet: the 1-GPU pool this was built on
 * refuses cuMulticastCreate ("Multicast gather").
 * Errors: UNSUPPORTED (the driver refuses multicast: no NVSwitch / fabric manager, device
 * attribute MULTICAST_SUPPORTED = 0, pidfd_getfd not permitted), NOT_INITIALIZED,
 * INVALID_ARG, OOM, CUDA. */

/* Single process (giga_init over distinct devices): C_full[g] (out) = GPU g's buffer of
 * `bytes` (rounded up to the multicast granularity) for g < ngpus. Pass them as the C_full
 * of giga_matmul_sharded with $GIGA_TRANSPORT=p2p. Repeated devices: INVALID_ARG. */
int giga_mc_alloc(int ngpus, size_t bytes, float **C_full);
/* Releases the team whose GPU-0 buffer is C_full0 (after its work finished). */
int giga_mc_free(float *C_full0);

/* Rank API ($GIGA_TRANSPORT=p2p): three collective phases, each on every rank, with a host
 * barrier (e.g. torch.distributed) between them:
 *   1. rank 0: giga_rank_mc_create(bytes, blob) -- makes the team object for `world`
 *      devices and fills GIGA_MC_BLOB_BYTES bytes (its pid and POSIX descriptor); the caller
 *      broadcasts the blob;
 *   2. every rank: giga_rank_mc_join(blob) -- imports the object (pidfd_getfd; rank 0 uses
 *      its own) and adds this rank's device;  barrier;
 *   3. every rank: giga_rank_mc_bind(&C_full) -- binds this rank's buffer and maps the
 *      multicast address; barrier.
 * Then register C_full with giga_rank_p2p_export (every rank must use its team buffer) and
 * call giga_matmul_rank with it. One team per process; released by giga_finalize. */
#define GIGA_MC_BLOB_BYTES 64
int giga_rank_mc_create(size_t bytes, uint8_t *blob);
int giga_rank_mc_join(const uint8_t *blob);
int giga_rank_mc_bind(float **C_full);

/* ------------------------------------------------------------------------------------ */
/* Single-device building blocks (device pointers on the current CUDA device; work is
 * enqueued on `stream`, a cudaStream_t, 0 = legacy default stream; no host sync). They do
 * not need giga_init. */

/* lo[i] = x[i] - tf32(x[i]) for i < n, where tf32() is the operand conversion the
 * tcgen05 kind::tf32 tensor core applies to raw fp32 bits (truncation of the low 13
 * mantissa bits; measured). The difference is exact in fp32. x and lo
 * 16-byte aligned. Errors: INVALID_ARG, CUDA. */
int giga_split_lo(const float *x, float *lo, int64_t n, void *stream);

/* C[i*ldc + j] = sum_k A[i*K+k] B[k*N+j] for i < M, j < N. A_lo / B_lo: either both NULL
 * (the kernel computes lo = x - tf32(x) of each staged tile in shared memory; the product
 * path's mode) or both the low parts produced by giga_split_lo (TMA-loaded from HBM).
 * Requirements: K % 4 == 0, N % 4 == 0, ldc % 4 == 0, ldc >= N, all pointers 16-byte
 * aligned (TMA). Errors: INVALID_ARG (incl. exactly one of A_lo / B_lo NULL), CUDA. */
int giga_gemm_3xtf32(const float *A, const float *A_lo, const float *B, const float *B_lo,
                     float *C, int64_t M, int64_t N, int64_t K, int64_t ldc, void *stream);

/* As giga_gemm_3xtf32 with the numerics and tiling knobs exposed (tests and probes):
 * terms = 3 (3xTF32), 2 (TF32 + BF16: a_hi*b_hi as one TF32 MMA, a_lo*b + a_hi*b_lo as one
 * K=16 BF16 MMA per k8 step, split error <= 3 * 2^-19 |a||b| (5.7e-6) per product with the
 * default RN hi (5.3e-6 reached by constructed inputs, tests/adversarial.py); $GIGA_HI_RN=0
 * truncates hi, a measurement mode whose split error reaches ~3 * 2^-18 = 1.1e-5 and can
 * exceed the bound; A_lo and B_lo must be NULL), 4 (3xFP16: row i of A scaled by 2^-ea_i and
 * column j of B by 2^-eb_j (exact) so their maxima lie in [2^15, 65504), x' = hi + lo in fp16
 * (RN), three K=16 kind::f16 MMAs per k16 step (a_lo b_hi, a_hi b_lo, a_hi b_hi), the
 * epilogue multiplies by 2^(ea_i + eb_j); elements whose fp16 split is off by more than
 * 2^-20 of themselves (far below their row's / column's maximum) are exceptions whose
 * remainders two fix kernels add in fp64 (deterministic); split error <= 2 * 2^-20 + 2^-22
 * per product; operands prepared once per launch in library-owned HBM scratch; A_lo and B_lo
 * must be NULL) or 1 (plain TF32: a_hi*b_hi only; A_lo/B_lo ignored). The product path
 * picks 4, 3 or 2 per launch (giga_product_scheme);
 * promote_kblocks = number of k-blocks (16 deep; 32 for terms = 4) accumulated in TMEM before
 * the partial sum is added into the fp32 register sum; 0 = never promote (one TMEM
 * accumulation over K); -1 = the library default (8);
 * cta_group = 1 (one CTA per 128 x 256 tile), 2 (a CTA pair per 256 x 256 tile, UMMA
 * cta_group::2), 0 = chosen from the shape. */
int giga_gemm_3xtf32_ex(const float *A, const float *A_lo, const float *B, const float *B_lo,
                        float *C, int64_t M, int64_t N, int64_t K, int64_t ldc, int terms,
                        int promote_kblocks, int cta_group, void *stream);

/* The shard GEMM with its fused-gather epilogue exposed (tests / probes; current device):
 * C = A * B (ldc row stride) written by the epilogue to C and to peer_c[0..n_peer) (same
 * shape and ldc; any device memory this device can store to: NVLink peers, or buffers of the
 * same device as the tests use) with store_mode 0 = TMA bulk stores (the p2p transport's
 * default), 1 = 16-byte st.global stores ($GIGA_P2P_STORE=vec), 2 = 16-byte multimem.st to
 * C as the multicast address (n_peer = 0). Mode 2 is the multicast gather's store path:
 * given a giga_mc_alloc / giga_rank_mc_bind team address it writes every member; given an
 * ordinary address (what a pool without multicast allows) the same SASS store (STG.E.128:
 * multimem.st and st.global assemble alike on sm_100a -- the multicast is in the address)
 * writes that buffer alone, which is how tests check its addressing -- outside the PTX
 * contract, a test hook. terms = 0: the product path's scheme choice (and, for 3xFP16,
 * its exception fixes mirrored to the peers / multicast); 1-4 as giga_gemm_3xtf32_ex.
 * Needs K % 4 == N % 4 == ldc % 4 == 0 and 16-byte aligned pointers. Errors: INVALID_ARG,
 * UNSUPPORTED ($GIGA_LO_PRESPLIT=1), CUDA. */
int giga_gemm_gather_ex(const float *A, const float *B, float *C, float *const *peer_c,
                        int n_peer, int64_t M, int64_t N, int64_t K, int64_t ldc, int terms,
                        int store_mode, void *stream);

/* Measurement tool for the N > 1 pipeline on a single GPU: enqueues on `stream` (current
 * device) exactly the GEMM launches rank `rank` of `world` issues in giga_matmul_rank /
 * giga_matmul_sharded over NCCL -- the K-chunks of giga_pipeline_plan accumulating into the
 * rank's rows of C_full, the last K-chunk in its row chunks, on all SMs but $GIGA_COMM_SMS --
 * with no communication: B is read as if it had arrived. world = 1 is the single-GPU GEMM.
 * With $GIGA_TRANSPORT=p2p: that transport's GEMMs instead -- all SMs, one launch per K-chunk
 * of its plan, the last one load-C (run_p2p_rank's launches without the peer stores).
 * Timing it bounds the per-GPU compute time of the N-GPU step from below
 * (scripts/project_scaling.py). A_shard: the rank's giga_partition rows x K; B: K x N; C_full: M x N (the
 * rank's rows are written). K % 4 == N % 4 == 0, 16-byte aligned pointers. Does not need
 * giga_init. Errors: INVALID_ARG, UNSUPPORTED (GIGA_LO_PRESPLIT=1), CUDA. */
int giga_rank_compute_only(const float *A_shard, const float *B, float *C_full, int64_t M,
                           int64_t N, int64_t K, int world, int rank, void *stream);

/* The work schedule of one giga_gemm_3xtf32 launch (C stored, default promotion interval)
 * over an M x N x K product on `num_sms` SMs (<= 0: 148), computed on the host exactly as
 * the launch computes it (no GPU needed). out must hold 8 values:
 * out[0] = CTA-group size (1: 128 x 256 tiles, 2: 256 x 256 tiles on CTA pairs),
 * out[1] = tiles, out[2] = concurrent tiles (clusters), out[3] = k-blocks per tile (16 deep;
 * 32 when the launch runs 3xFP16),
 * out[4] = first_split: tiles [0, first_split) run whole, out[5] = s: every later tile runs
 * as s units over consecutive k-block ranges [n_kb*q/s, n_kb*(q+1)/s), out[6] = work units,
 * out[7] = how the parts combine, both deterministic (the same bits on every launch of the
 * shape): 0 no split, 1 two halves TMA reduce-add into a C region zeroed before the launch
 * (0 + a + b is order-independent), 2 the parts' fp32 partials are added in the order
 * q = 0, 1, ..., s-1 by the part that finishes last (grids under one wave only).
 * $GIGA_TAIL_SPLIT=0 disables the k-split (s = 1). Errors: INVALID_ARG. */
int giga_gemm_schedule(int64_t M, int64_t N, int64_t K, int num_sms, int64_t *out);

/* The fp32-accurate scheme the product path uses for one M x N x K GEMM launch (host-only,
 * DESIGN.md 6.7, 6.8): *terms = 4 (3xFP16, see giga_gemm_3xtf32_ex: per-product split error
 * <= 2 * 2^-20 + 2^-22 |a||b|; 4 preparation kernels and 2 exception-fix kernels per launch)
 * when M >= 2048, N >= 1024, K >= 512 and M N K >= 2^35; else 3 (3xTF32: three kind::tf32
 * MMAs per k8 step, no preparation). 2 (TF32 + BF16: a_hi*b_hi as one kind::tf32 MMA plus
 * a_lo*b + a_hi*b_lo as one K=16 kind::f16 MMA, hi = RN tf32(x), operands prepared once per
 * launch; split error <= 3 * 2^-19 |a||b|) is no longer chosen by shape (3xFP16 wins its old
 * range since the round-2 epilogue fix). The thresholds are measured crossovers (preparation
 * included, profiles/r02_scheme_crossover_e.jsonl);
 * $GIGA_SCHEME = 3xtf32 | tf32bf16 | 3xfp16 forces one. Errors: INVALID_ARG. */
int giga_product_scheme(int64_t M, int64_t N, int64_t K, int *terms);

/* ------------------------------------------------------------------------------------ */
/* Kernel timing (bench.py's roofline): when enabled, CUDA events bracket every GEMM and
 * split launch on the stream it is launched on; giga_timing_read synchronises on the
 * recorded events and returns the summed device milliseconds and launch counts since the
 * last reset. */
int giga_timing_enable(int on);
int giga_timing_reset(void);
int giga_timing_read(double *gemm_ms, int64_t *gemm_launches, double *split_ms,
                     int64_t *split_launches);

#ifdef __cplusplus
}
#endif
#endif /* GIGA_H_ */
