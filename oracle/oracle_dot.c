/*
 * oracle_dot.c -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py for who may load it).
 *
 * The independent CPU oracle for GigaAPI's vector operations (arXiv 2504.01266 S4.2.8,
 * PAPER.md:294-303): "we essentially calculate a running sum to accumulate the partial dot
 * product"; "the L2 Norm is almost entirely the same: it just deals with one vector,
 * however, and then square roots the final result".
 *
 *   dot(x, y) = sum_{i=0}^{n-1} x[i] * y[i]       accumulated in fp64, ascending i
 *   sabs      = sum_i |x[i] * y[i]|              (scale for the error bound)
 *   l2(x)     = sqrt(dot(x, x))                  (one square root, at the end)
 *
 * Each product of two fp32 values is exact in fp64; only the additions round.
 */
#include <math.h>
#include <stdint.h>

int oracle_dot_f64(const float *x, const float *y, int64_t n, double *dot, double *sabs) {
  if (!x || !y || !dot || n < 0) return -1;
  double acc = 0.0, s = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double p = (double)x[i] * (double)y[i];
    acc += p;
    s += fabs(p);
  }
  *dot = acc;
  if (sabs) *sabs = s;
  return 0;
}

int oracle_l2norm_f64(const float *x, int64_t n, double *norm) {
  if (!x || !norm || n < 0) return -1;
  double d = 0.0;
  if (oracle_dot_f64(x, x, n, &d, 0) != 0) return -1;
  *norm = sqrt(d);
  return 0;
}
