// kb_persist.cuh — whole-solve persistent kernel for small fp64 images (BASELINE cfg1: 256^2).
//
// At 256^2 one iteration of the four pass kernels is ~65 K pixels of work per launch: the
// passes are launch- and ramp-bound (profiles/README.md: ~8 us per kernel, 3 us of it before the
// first MMA). Here ONE cooperative launch runs all iterations. Each CTA owns a band of RB image
// rows and fuses the two passes of an operator application with halo recompute, so a whole
// iteration needs only two grid-wide barriers:
//   phase 1 (forward + residual, kronblur kron.py:218-225 and solvers.py:170):
//     stage Y rows [r0-Ha, r1+Ha) in shared memory, Z_i = H_i Y on the CTA's rows (axis 0),
//     R = sum_i K_i-filter(Z_i) - B on the same rows (axis 1), R -> global (L2-resident)
//   grid barrier (R rows of the neighbours are the adjoint's halo)
//   phase 2 (adjoint + fused FISTA update, kron.py:228-235 and solvers.py:170-173 + F2/F3):
//     stage R rows with halo, Z_i = H_i^T R (correlation + fold), G = sum_i K_i^T-filter(Z_i),
//     x = (L y - g)/(L + lam^2) [projection], y = x + beta_k (x - x_prev) on the CTA's rows
//   grid barrier (Y rows of the neighbours are the next forward's halo)
// Arithmetic is fp64 FMA (the FP64 pipe and the DMMA path have the same nominal rate on B200,
// SURVEY F8); the factor rules are the stencil form of structured.py:111-123 with the zero /
// half-sample-reflective extension, applied by index mapping (no fill tricks).
#pragma once
#include <cooperative_groups.h>

namespace kb {

constexpr int kPsThreads = 256;

struct PsArgs {
  const double* B;
  double* X;
  double* Y;
  double* R;
  const double* ha;   // [r][Wpa] axis-0 conv taps: ha[k] = c_{Ha-k}
  const double* kbt;  // [r][Wpb] axis-1 conv taps
  const double* beta; // [iters] momentum coefficients beta_{k0+1 ..}
  int* nonfinite;
  double L, denom;
  int m, n, r, Ha, Hb, Wpa, Wpb, refl_a, refl_b;
  int RB;  // rows per CTA
  int k0, iters, project;
};

// index of x~(u) on an axis of length M (zero extension: -1; reflective: one half-sample fold)
__device__ __forceinline__ int ps_src(int u, int M, int refl) {
  if (u >= 0 && u < M) return u;
  if (!refl) return -1;
  u = u < 0 ? -1 - u : 2 * M - 1 - u;
  return (u >= 0 && u < M) ? u : -1;
}

// shared memory of a CTA: rows [RB + 2 Ha][n] of the staged input, [r][RB][n] of Z, the taps
__host__ __device__ inline size_t ps_smem_bytes(int RB, int Ha, int n, int r, int Wpa, int Wpb) {
  return sizeof(double) * ((size_t)(RB + 2 * Ha) * n + (size_t)r * RB * n + (size_t)r * (Wpa + Wpb));
}

__global__ void __launch_bounds__(kPsThreads) kb_solve_persistent(PsArgs a) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double ps_smem[];
  const int n = a.n, m = a.m, Ha = a.Ha, Hb = a.Hb, r = a.r;
  const int rows_in = a.RB + 2 * Ha;
  double* Ys = ps_smem;                          // staged input rows g = r0 - Ha + t
  double* Zs = Ys + (size_t)rows_in * n;         // [r][RB][n]
  double* th = Zs + (size_t)r * a.RB * n;        // [r][Wpa]
  double* tk = th + (size_t)r * a.Wpa;           // [r][Wpb]
  const int tid = threadIdx.x;
  for (int i = tid; i < r * a.Wpa; i += kPsThreads) th[i] = a.ha[i];
  for (int i = tid; i < r * a.Wpb; i += kPsThreads) tk[i] = a.kbt[i];
  const int r0 = blockIdx.x * a.RB;
  const int r1 = min(m, r0 + a.RB), nr = max(0, r1 - r0);

  // stage rows [r0 - Ha, r1 + Ha) of `src` (out-of-domain rows read as zero; the rules map):
  // every pair of elements is an independent 16-byte cp.async, so all of a thread's loads are in
  // flight at once (a load -> store loop serialises ~30 L2 round trips per phase). `.cg` reads
  // through to L2: the rows were written by other CTAs since this SM last read them, and L1 is
  // not coherent across SMs (n is even: persist_plan requires it).
  auto stage = [&](const double* src) {
    const int rows = nr + 2 * Ha, half = n >> 1;
    for (int idx = tid; idx < rows * half; idx += kPsThreads) {
      const int t = idx / half, c = 2 * (idx - t * half);
      const int g = r0 - Ha + t;
      double* dst = Ys + (size_t)t * n + c;
      if (g >= 0 && g < m) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)),
                     "l"(src + (size_t)g * n + c)
                     : "memory");
      } else {
        dst[0] = 0.0;
        dst[1] = 0.0;
      }
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
  };
  // axis-0 pass on the staged rows: Z_i[t][c] for the CTA's rows
  auto axis0 = [&](bool adjoint) {
    for (int t = 0; t < nr; ++t) {
      const int s = r0 + t;
      for (int c = tid; c < n; c += kPsThreads)
        for (int i = 0; i < r; ++i) {
          const double* h = th + (size_t)i * a.Wpa;
          double acc = 0.0;
          for (int k = 0; k <= 2 * Ha; ++k) {
            const int d = Ha - k;  // h[k] = c_d
            const double cd = h[k];
            if (!adjoint) {
              const int g = ps_src(s - d, m, a.refl_a);
              if (g >= 0) acc = fma(cd, Ys[(size_t)(g - r0 + Ha) * n + c], acc);
            } else {
              const int g = s + d;  // correlation over in-domain sources
              if (g >= 0 && g < m) acc = fma(cd, Ys[(size_t)(g - r0 + Ha) * n + c], acc);
              if (a.refl_a && (s - d < 0 || s - d >= m)) {  // + the forward fold (H is symmetric)
                const int f = ps_src(s - d, m, 1);
                if (f >= 0) acc = fma(cd, Ys[(size_t)(f - r0 + Ha) * n + c], acc);
              }
            }
          }
          Zs[((size_t)i * a.RB + t) * n + c] = acc;
        }
    }
  };
  // axis-1 pass of one output element from the CTA's Z rows
  auto axis1 = [&](int t, int c, bool adjoint) {
    double acc = 0.0;
    for (int i = 0; i < r; ++i) {
      const double* kk = tk + (size_t)i * a.Wpb;
      const double* z = Zs + ((size_t)i * a.RB + t) * n;
      for (int k = 0; k <= 2 * Hb; ++k) {
        const int d = Hb - k;
        const double cd = kk[k];
        if (!adjoint) {
          const int q = ps_src(c - d, n, a.refl_b);
          if (q >= 0) acc = fma(cd, z[q], acc);
        } else {
          const int q = c + d;
          if (q >= 0 && q < n) acc = fma(cd, z[q], acc);
          if (a.refl_b && (c - d < 0 || c - d >= n)) {
            const int f = ps_src(c - d, n, 1);
            if (f >= 0) acc = fma(cd, z[f], acc);
          }
        }
      }
    }
    return acc;
  };

  __syncthreads();
  for (int it = 0; it < a.iters; ++it) {
    const int k = a.k0 + it + 1;
    // ---- phase 1: R = A Y - B on rows [r0, r1)
    if (nr > 0) {
      stage(a.Y);
      __syncthreads();
      axis0(false);
      __syncthreads();
      for (int t = 0; t < nr; ++t)
        for (int c = tid; c < n; c += kPsThreads) {
          const size_t e = (size_t)(r0 + t) * n + c;
          a.R[e] = __dsub_rn(axis1(t, c, false), a.B[e]);
        }
    }
    grid.sync();
    // ---- phase 2: G = A^T R, x = (L y - g)/(L + lam^2), projection, momentum
    if (nr > 0) {
      stage(a.R);
      __syncthreads();
      axis0(true);
      __syncthreads();
      const double bk = a.beta[it];
      bool bad = false;
      for (int t = 0; t < nr; ++t)
        for (int c = tid; c < n; c += kPsThreads) {
          const size_t e = (size_t)(r0 + t) * n + c;
          const double g = axis1(t, c, true);
          double x = __ddiv_rn(__dsub_rn(__dmul_rn(a.L, a.Y[e]), g), a.denom);
          if (a.project && !(x > 0.0) && !isnan(x)) x = 0.0;  // np.maximum(x, 0): NaN kept (F3)
          bad |= !isfinite(x);
          const double xp = a.X[e];
          a.X[e] = x;
          a.Y[e] = __dadd_rn(x, __dmul_rn(bk, __dsub_rn(x, xp)));
        }
      if (bad) atomicMin(a.nonfinite, k);
    }
    grid.sync();
  }
}

}  // namespace kb
