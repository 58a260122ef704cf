/*
 * kb_oracle.c -- TEST INFRASTRUCTURE ONLY (never linked or loaded by the product package).
 *
 * A second, independent CPU restatement of the reference hot path (kronblur, pure Python), in
 * plain C with OpenMP, fp64 throughout. It exists because the numpy oracle port
 * (oracle/kronblur_port.py, the reference's own FFT path) needs ~65 min per iteration at
 * BASELINE cfg5 (16384^2) and ~76 s at cfg4; this direct banded form runs the
 * same arithmetic in seconds per iteration, so full-size parity can be checked (GPU tests) and
 * full-length fixtures generated offline (tests/golden/make_fullsize.py).
 *
 * What it restates (file:line under /root/reference/pkg/src/kronblur/):
 *  - factor rules structured.py:111-123 in stencil form: along an axis of length M a factor F(c)
 *    with anchor j acts as y[s] = sum_d c_d x~(s-d), c_d = c[j+d]; x~ is the zero extension
 *    (Toeplitz, zero BC) or the half-sample reflection x~(-1-t) = x(t), x~(M+t) = x(M-1-t)
 *    (Toeplitz+Hankel, reflective BC). The adjoint is F^T = T^T + H (H symmetric):
 *    correlation over in-domain sources plus the forward fold terms.
 *  - kron_apply / kron_apply_adjoint kron.py:218-235: Y = sum_i H_i X K_i^T, terms summed in
 *    order i = 0..r-1 (kron.py:222-224).
 *  - the _engine loop solvers.py:168-176 with the x >= 0 projection the BASELINE configs add
 *    (np.maximum semantics, NaN kept): R = A y - b, g = A^T R,
 *    x = (L*y - g)/(L + lam^2), x = max(x, 0), y = x + beta_k (x - x_prev).
 *  - estimate_lipschitz solvers.py:115-130 (matrix form): rho_k = <v, A^T A v>, v = w/||w||.
 *  - blur_direct psf.py:170-193, bit for bit: per pixel the products P[a][b] * Xp[...] over the
 *    nonzero PSF entries in row-major order, each product and each sum rounded separately.
 *
 * Bands: the caller passes each axis' band as (dlo, w, taps[r][w]) -- the generator entries
 * c_dlo .. c_{dlo+w-1}; entries outside are zero (zero BC exactly; reflective generators carry
 * ~1e-16 leakage there, which the caller trims; < 1e-13 relative effect).
 *
 * Build: oracle/Makefile. This file is compiled with FMA contraction (the operator is checked to
 * tolerance); blur_direct lives in kb_oracle_blur.c, compiled with
 * -ffp-contract=off so it reproduces numpy's separately rounded products and sums.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
  int m, n, r;
  int bc_a, bc_b; /* 0 zero (Toeplitz), 1 reflective (Toeplitz+Hankel) */
  int a_dlo, a_w;
  const double* a_taps; /* [r][a_w]: H_i (axis 0) */
  int b_dlo, b_w;
  const double* b_taps; /* [r][b_w]: K_i (axis 1) */
} kbo_op;

/* source index of x~(t) on an axis of length M, or -1 when it reads zero */
static inline long src_index(long t, long M, int reflective) {
  if (t >= 0 && t < M) return t;
  if (!reflective) return -1;
  if (t < 0) t = -1 - t;
  else t = 2 * M - 1 - t;
  return (t >= 0 && t < M) ? t : -1; /* bands wider than the axis: beyond one fold reads zero */
}

/* GCC vector extension (portable C; unaligned loads through memcpy) */
typedef double v4d __attribute__((vector_size(32)));
static inline v4d ld4(const double* p) {
  v4d v;
  memcpy(&v, p, sizeof(v));
  return v;
}
static inline void st4(double* p, v4d v) { memcpy(p, &v, sizeof(v)); }

/* one output of factor_vec's rule (edges) */
static double factor_one(const double* in, long M, long s, const double* c, int dlo, int w, int reflective,
                         int adjoint) {
  double acc = 0.0;
  for (int t = 0; t < w; ++t) {
    const long d = dlo + t;
    const double cd = c[t];
    if (cd == 0.0) continue;
    if (!adjoint) {
      const long k = src_index(s - d, M, reflective);
      if (k >= 0) acc += cd * in[k];
    } else {
      const long k = s + d;
      if (k >= 0 && k < M) acc += cd * in[k];
      if (reflective) {
        const long u = s - d;
        if (u < 0 || u >= M) {
          const long kk = src_index(u, M, 1);
          if (kk >= 0) acc += cd * in[kk];
        }
      }
    }
  }
  return acc;
}

static void axis1_rows(const double* in, double* out, long rows, long n, const double* c, int dlo, int w,
                       int reflective, int adjoint) {
  long lo = dlo + w - 1, hi = n - 1 + dlo;
  if (adjoint) {
    const long alo = -dlo, ahi = n - w - dlo;
    if (alo > lo) lo = alo;
    if (ahi < hi) hi = ahi;
  }
  if (lo < 0) lo = 0;
  if (hi > n - 1) hi = n - 1;
  for (long i = 0; i < rows; ++i) {
    const double* x = in + i * n;
    double* y = out + i * n;
    if (hi < lo) {
      for (long s = 0; s < n; ++s) y[s] = factor_one(x, n, s, c, dlo, w, reflective, adjoint);
      continue;
    }
    for (long s = 0; s < lo; ++s) y[s] = factor_one(x, n, s, c, dlo, w, reflective, adjoint);
    long s = lo;
    for (; s + 8 <= hi + 1; s += 8) {
      v4d a0 = {0, 0, 0, 0}, a1 = {0, 0, 0, 0};
      for (int t = 0; t < w; ++t) {
        const long d = dlo + t;
        const double* xp = adjoint ? x + s + d : x + s - d;
        const v4d cv = {c[t], c[t], c[t], c[t]};
        a0 += cv * ld4(xp);
        a1 += cv * ld4(xp + 4);
      }
      st4(y + s, a0);
      st4(y + s + 4, a1);
    }
    for (; s <= hi; ++s) {
      double acc = 0.0;
      for (int t = 0; t < w; ++t) acc += c[t] * x[adjoint ? s + dlo + t : s - dlo - t];
      y[s] = acc;
    }
    for (s = hi + 1; s < n; ++s) y[s] = factor_one(x, n, s, c, dlo, w, reflective, adjoint);
  }
}

/* Axis-0 pass producing output rows [i0, i1) of an (M x n) plane: out[i-i0][:]. Each output
 * row is a weighted sum of source rows (the stencil's, folded / correlated per the rule),
 * vectorised over columns in column blocks. Interior rows (every source in the domain, no fold
 * term) go four at a time so each loaded source vector feeds four outputs. */
#define KBO_MAXP 4096
#define KBO_RB 4
static void axis0_generic_row(const double* in, long M, long n, long s, long jb, long je, double* o,
                              const double* c, int dlo, int w, int reflective, int adjoint) {
  const double* src[KBO_MAXP];
  double cf[KBO_MAXP];
  int np = 0;
  for (int t = 0; t < w && np + 2 <= KBO_MAXP; ++t) {
    const long d = dlo + t;
    const double cd = c[t];
    if (cd == 0.0) continue;
    if (!adjoint) {
      const long k = src_index(s - d, M, reflective);
      if (k >= 0) { src[np] = in + k * n; cf[np++] = cd; }
    } else {
      if (s + d >= 0 && s + d < M) { src[np] = in + (s + d) * n; cf[np++] = cd; }
      if (reflective && (s - d < 0 || s - d >= M)) {
        const long kk = src_index(s - d, M, 1);
        if (kk >= 0) { src[np] = in + kk * n; cf[np++] = cd; }
      }
    }
  }
  long j = jb;
  for (; j + 8 <= je; j += 8) {
    v4d a0 = {0, 0, 0, 0}, a1 = {0, 0, 0, 0};
    for (int p = 0; p < np; ++p) {
      const v4d cv = {cf[p], cf[p], cf[p], cf[p]};
      a0 += cv * ld4(src[p] + j);
      a1 += cv * ld4(src[p] + j + 4);
    }
    st4(o + j, a0);
    st4(o + j + 4, a1);
  }
  for (; j < je; ++j) {
    double acc = 0.0;
    for (int p = 0; p < np; ++p) acc += cf[p] * src[p][j];
    o[j] = acc;
  }
}

static void axis0_rows(const double* in, long M, long n, long i0, long i1, double* out, const double* c, int dlo,
                       int w, int reflective, int adjoint) {
  const long dhi = dlo + w - 1;
  long lo = dhi, hi = M - 1 + dlo; /* forward / fold-free rows */
  if (adjoint) {
    if (-dlo > lo) lo = -dlo;
    if (M - 1 - dhi < hi) hi = M - 1 - dhi;
  }
  /* taps zero-padded by KBO_RB on both sides: cz[t + KBO_RB] = c[t] */
  double cz[KBO_MAXP + 2 * KBO_RB];
  for (int t = 0; t < w + 2 * KBO_RB && t < KBO_MAXP + 2 * KBO_RB; ++t) {
    const int u = t - KBO_RB;
    cz[t] = (u >= 0 && u < w) ? c[u] : 0.0;
  }
  const long JB = 256;
  for (long jb = 0; jb < n; jb += JB) {
    const long je = jb + JB < n ? jb + JB : n;
    long s = i0;
    while (s < i1) {
      if (s >= lo && s + KBO_RB - 1 <= hi && s + KBO_RB <= i1 && w + 2 * KBO_RB <= KBO_MAXP) {
        /* four interior rows s..s+3 */
        double* o = out + (s - i0) * n;
        const long k0 = adjoint ? s + dlo : s - dhi, k1 = adjoint ? s + KBO_RB - 1 + dhi : s + KBO_RB - 1 - dlo;
        long j = jb;
        for (; j + 8 <= je; j += 8) {
          v4d a[KBO_RB][2];
          for (int r = 0; r < KBO_RB; ++r) a[r][0] = a[r][1] = (v4d){0, 0, 0, 0};
          for (long k = k0; k <= k1; ++k) {
            const double* x = in + k * n + j;
            const v4d x0 = ld4(x), x1 = ld4(x + 4);
            for (int r = 0; r < KBO_RB; ++r) {
              /* forward: d = s + r - k; adjoint (correlation): d = k - s - r */
              const long d = adjoint ? k - s - r : s + r - k;
              const double cv = cz[d - dlo + KBO_RB];
              const v4d cc = {cv, cv, cv, cv};
              a[r][0] += cc * x0;
              a[r][1] += cc * x1;
            }
          }
          for (int r = 0; r < KBO_RB; ++r) {
            st4(o + r * n + j, a[r][0]);
            st4(o + r * n + j + 4, a[r][1]);
          }
        }
        for (; j < je; ++j)
          for (int r = 0; r < KBO_RB; ++r) {
            double acc = 0.0;
            for (long k = k0; k <= k1; ++k) {
              const long d = adjoint ? k - s - r : s + r - k;
              acc += cz[d - dlo + KBO_RB] * in[k * n + j];
            }
            o[r * n + j] = acc;
          }
        s += KBO_RB;
      } else {
        axis0_generic_row(in, M, n, s, jb, je, out + (s - i0) * n, c, dlo, w, reflective, adjoint);
        s += 1;
      }
    }
  }
}

/* Y = sum_i H_i X K_i^T (adjoint: sum_i H_i^T X K_i), row strips in parallel. */
void kbo_apply(const kbo_op* op, int adjoint, const double* X, double* Y) {
  const long m = op->m, n = op->n;
  const long S = 8;
#pragma omp parallel
  {
    double* z = (double*)malloc(sizeof(double) * S * n);
    double* t = (double*)malloc(sizeof(double) * S * n);
#pragma omp for schedule(dynamic, 1)
    for (long i0 = 0; i0 < m; i0 += S) {
      const long i1 = i0 + S < m ? i0 + S : m, rows = i1 - i0;
      double* y = Y + i0 * n;
      memset(y, 0, sizeof(double) * rows * n);
      for (int i = 0; i < op->r; ++i) {
        axis0_rows(X, m, n, i0, i1, z, op->a_taps + (long)i * op->a_w, op->a_dlo, op->a_w, op->bc_a, adjoint);
        axis1_rows(z, t, rows, n, op->b_taps + (long)i * op->b_w, op->b_dlo, op->b_w, op->bc_b, adjoint);
        for (long k = 0; k < rows * n; ++k) y[k] += t[k];
      }
    }
    free(z);
    free(t);
  }
}

static double dot(const double* a, const double* b, long count) {
  double s = 0.0;
#pragma omp parallel for reduction(+ : s) schedule(static)
  for (long k = 0; k < count; ++k) s += a[k] * b[k];
  return s;
}

/* Projected sFISTA, iterations k = 1..iters from x_0 = X (in/out), y_1 = X. beta[k-1] =
 * (t_k - 1)/t_{k+1}. Returns the first k with a non-finite x_k, or 0. work: 3 planes. */
int kbo_sfista(const kbo_op* op, const double* B, double* X, double L, double lam, int iters,
               const double* beta, int project, double* work) {
  const long N = (long)op->m * op->n;
  double* y = work;
  double* r = work + N;
  double* g = work + 2 * N;
  const double denom = L + lam * lam;
  memcpy(y, X, sizeof(double) * N);
  for (int k = 1; k <= iters; ++k) {
    kbo_apply(op, 0, y, r);
#pragma omp parallel for schedule(static)
    for (long e = 0; e < N; ++e) r[e] = r[e] - B[e];
    kbo_apply(op, 1, r, g);
    const double bk = beta[k - 1];
    int bad = 0;
#pragma omp parallel for schedule(static) reduction(| : bad)
    for (long e = 0; e < N; ++e) {
      double x = (L * y[e] - g[e]) / denom;
      if (project && !(x > 0.0) && !isnan(x)) x = 0.0;
      if (!isfinite(x)) bad = 1;
      const double xp = X[e];
      X[e] = x;
      y[e] = x + bk * (x - xp);
    }
    if (bad) return k;
  }
  return 0;
}

/* Power iteration on A^T A from the normalised v (overwritten); rho[k] = <v_k, w_k>, nw2[k] =
 * ||w_k||^2 for k < iters. work: 2 planes. */
void kbo_power(const kbo_op* op, double* v, int iters, double* rho, double* nw2, double* work) {
  const long N = (long)op->m * op->n;
  double* u = work;
  double* w = work + N;
  for (int k = 0; k < iters; ++k) {
    kbo_apply(op, 0, v, u);
    kbo_apply(op, 1, u, w);
    rho[k] = dot(v, w, N);
    nw2[k] = dot(w, w, N);
    const double nw = sqrt(nw2[k]);
    if (nw == 0.0) return;
#pragma omp parallel for schedule(static)
    for (long e = 0; e < N; ++e) v[e] = w[e] / nw;
  }
}

int kbo_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
