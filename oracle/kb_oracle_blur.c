/*
 * kb_oracle_blur.c -- TEST INFRASTRUCTURE ONLY. blur_direct of the reference (psf.py:170-193)
 * restated bit for bit; compiled with -ffp-contract=off (oracle/Makefile) so every product and
 * every sum is rounded separately, as numpy's `Y += P[a0, b0] * Xp[...]` does.
 */
#include <stdlib.h>

static inline long src_index(long t, long M, int reflective) {
  if (t >= 0 && t < M) return t;
  if (!reflective) return -1;
  if (t < 0) t = -1 - t;
  else t = 2 * M - 1 - t;
  return (t >= 0 && t < M) ? t : -1;
}

/* blur_direct (psf.py:170-193), bit-identical to numpy: P [rows][cols] with 1-based centre
 * (l, q), X [m][n] -> Y [m][n]; bc 0 zero ("constant" pad), 1 numpy "symmetric" pad. */
void kbo_blur_direct(const double* P, int rows, int cols, int l, int q, const double* X, int m, int n, int bc,
                     double* Y) {
  int nnz = 0;
  for (int k = 0; k < rows * cols; ++k) nnz += P[k] != 0.0;
  int* ra = (int*)malloc(sizeof(int) * (nnz + 1));
  int* cb = (int*)malloc(sizeof(int) * (nnz + 1));
  double* pv = (double*)malloc(sizeof(double) * (nnz + 1));
  int t = 0;
  for (int a = 0; a < rows; ++a)
    for (int b = 0; b < cols; ++b)
      if (P[a * cols + b] != 0.0) {
        ra[t] = a;
        cb[t] = b;
        pv[t] = P[a * cols + b];
        ++t;
      }
#pragma omp parallel for schedule(dynamic, 4)
  for (long i = 0; i < m; ++i) {
    double* y = Y + i * n;
    for (long j = 0; j < n; ++j) y[j] = 0.0;
    for (int e = 0; e < nnz; ++e) {
      /* Y += v * Xp[r0+i, c0+j], r0 = rows-1-a: X row i + l - 1 - a, col j + q - 1 - b */
      const long si = src_index(i + l - 1 - ra[e], m, bc);
      const double v = pv[e];
      const long off = q - 1 - cb[e];
      if (si < 0) {
        for (long j = 0; j < n; ++j) y[j] = y[j] + v * 0.0;
        continue;
      }
      const double* x = X + si * n;
      const long jlo = off < 0 ? -off : 0, jhi = n - (off > 0 ? off : 0);
      for (long j = 0; j < jlo && j < n; ++j) {
        const long sj = src_index(j + off, n, bc);
        y[j] = y[j] + v * (sj >= 0 ? x[sj] : 0.0);
      }
      for (long j = jlo; j < jhi; ++j) y[j] = y[j] + v * x[j + off];
      for (long j = jhi > jlo ? jhi : jlo; j < n; ++j) {
        const long sj = src_index(j + off, n, bc);
        y[j] = y[j] + v * (sj >= 0 ? x[sj] : 0.0);
      }
    }
  }
  free(ra);
  free(cb);
  free(pv);
}

