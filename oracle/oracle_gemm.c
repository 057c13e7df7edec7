/*
 * oracle_gemm.c -- TEST INFRASTRUCTURE ONLY.
 *
 * The independent CPU oracle for GigaAPI's matrix multiply (arXiv 2504.01266).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load this library. The product path (paper_2504_01266_b200/) never links,
 * imports or calls it, and it shares no code, header or constant with that path.
 *
 * What it computes -- the plain definition, nothing more:
 *
 *   C[i][j] = sum_{k=0}^{K-1} A[i][k] * B[k][j]                      (S4.2.7:
 *            "each element in C[i,j] is calculated by taking a dot product of the i-th row of
 *             the matrix A and the j-th column of matrix B"; "the total sum being
 *             reported and assigned at the end of the loop")
 *
 *   S[i][j] = sum_k |A[i][k]| * |B[k][j]|    (the scale of the acceptance bound
 *            |C_gpu - C| <= 1e-5 * S stated in BASELINE.json north_star)
 *
 * Inputs are row-major fp32 (SPEC.md:234-236 MatrixF32), A is MxK, B is KxN. All
 * arithmetic is fp64; each product of two fp32 values is exact in fp64 (24+24 <= 53
 * bits), and every element sums its K products in ascending k. The loop order is i-k-j,
 * which keeps the per-element order ascending in k, so the result is bit-identical to the
 * naive i-j-k loop. Rows are independent ("elements are computed
 * independently"), so rows may be split across threads without changing any bit.
 *
 * Compile: gcc -O2 -fno-fast-math -ffp-contract=off -shared -fPIC -pthread
 * (-ffp-contract=off is belt and braces: an fma of an exact product changes nothing.)
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* One row of the definition: acc[j] = sum_k A[i,k] B[k,j], sabs[j] = sum_k |A[i,k]||B[k,j]|. */
static void oracle_row(const float *A, const float *B, int64_t i, int64_t N, int64_t K,
                       double *acc, double *sabs) {
  for (int64_t j = 0; j < N; ++j) {
    acc[j] = 0.0;
    sabs[j] = 0.0;
  }
  const float *a_row = A + i * K;
  for (int64_t k = 0; k < K; ++k) {
    const double a = (double)a_row[k];
    const double a_abs = fabs(a);
    const float *b_row = B + k * N;
    for (int64_t j = 0; j < N; ++j) {
      const double b = (double)b_row[j];
      acc[j] += a * b;
      sabs[j] += a_abs * fabs(b);
    }
  }
}

typedef struct {
  const float *A, *B;
  const int64_t *rows; /* NULL: rows r0..r1 of A; else rows[r0..r1) index A */
  int64_t r0, r1, N, K;
  double *C, *S; /* output row r (local index) at C + r*N */
} work_t;

static void *worker(void *p) {
  work_t *w = (work_t *)p;
  for (int64_t r = w->r0; r < w->r1; ++r) {
    const int64_t i = w->rows ? w->rows[r] : r;
    oracle_row(w->A, w->B, i, w->N, w->K, w->C + r * w->N, w->S ? w->S + r * w->N : NULL);
  }
  return NULL;
}

/* sabs may not be NULL inside oracle_row; give threads a scratch row when S is unwanted. */
static void *worker_noS(void *p) {
  work_t *w = (work_t *)p;
  double *scratch = (double *)malloc(sizeof(double) * (size_t)(w->N > 0 ? w->N : 1));
  if (!scratch) return (void *)1;
  for (int64_t r = w->r0; r < w->r1; ++r) {
    const int64_t i = w->rows ? w->rows[r] : r;
    oracle_row(w->A, w->B, i, w->N, w->K, w->C + r * w->N, scratch);
  }
  free(scratch);
  return NULL;
}

/*
 * oracle_gemm_rows_f64: rows `rows[0..nrows)` of C = A*B (and of S), written densely into
 * C_out / S_out (nrows x N, row-major fp64). rows == NULL means rows 0..nrows-1.
 * S_out may be NULL. nthreads <= 0 means 1. Returns 0 on success, -1 on bad arguments,
 * -2 if a thread could not be started or allocated.
 */
int oracle_gemm_rows_f64(const float *A, const float *B, const int64_t *rows, int64_t nrows,
                         int64_t N, int64_t K, double *C_out, double *S_out, int nthreads) {
  if (!A || !B || !C_out || nrows < 0 || N < 1 || K < 1) return -1;
  if (nthreads <= 0) nthreads = 1;
  if (nthreads > nrows) nthreads = nrows > 0 ? (int)nrows : 1;
  pthread_t *th = (pthread_t *)calloc((size_t)nthreads, sizeof(pthread_t));
  work_t *ws = (work_t *)calloc((size_t)nthreads, sizeof(work_t));
  if (!th || !ws) {
    free(th);
    free(ws);
    return -2;
  }
  int rc = 0, started = 0;
  for (int t = 0; t < nthreads; ++t) {
    ws[t].A = A;
    ws[t].B = B;
    ws[t].rows = rows;
    ws[t].r0 = nrows * t / nthreads;
    ws[t].r1 = nrows * (t + 1) / nthreads;
    ws[t].N = N;
    ws[t].K = K;
    ws[t].C = C_out;
    ws[t].S = S_out;
    if (pthread_create(&th[t], NULL, S_out ? worker : worker_noS, &ws[t]) != 0) {
      rc = -2;
      break;
    }
    ++started;
  }
  for (int t = 0; t < started; ++t) {
    void *ret = NULL;
    pthread_join(th[t], &ret);
    if (ret) rc = -2;
  }
  free(th);
  free(ws);
  return rc;
}

/* oracle_gemm_f64: the full C (M x N) and S, fp64. */
int oracle_gemm_f64(const float *A, const float *B, int64_t M, int64_t N, int64_t K,
                    double *C_out, double *S_out, int nthreads) {
  if (M < 1) return -1;
  return oracle_gemm_rows_f64(A, B, NULL, M, N, K, C_out, S_out, nthreads);
}
