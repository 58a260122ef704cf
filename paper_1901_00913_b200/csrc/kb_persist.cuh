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
  int* flags;  // [gridDim.x] phase epochs (neighbour synchronisation), zeroed before the launch;
               // nullptr: grid-wide barriers instead
};

// index of x~(u) on an axis of length M (zero extension: -1; reflective: one half-sample fold)
__device__ __forceinline__ int ps_src(int u, int M, int refl) {
  if (u >= 0 && u < M) return u;
  if (!refl) return -1;
  u = u < 0 ? -1 - u : 2 * M - 1 - u;
  return (u >= 0 && u < M) ? u : -1;
}

// shared memory of a CTA: rows [RB + 2 Ha][n] of the staged input, [r][RB][n + 2 Hb] of Z (Hb
// halo columns each side), the taps [r][2Ha+1] and [r][2Hb+1]
__host__ __device__ inline size_t ps_smem_bytes(int RB, int Ha, int Hb, int n, int r) {
  return sizeof(double) * ((size_t)(RB + 2 * Ha) * n + (size_t)r * RB * (n + 2 * Hb) +
                           (size_t)r * (2 * Ha + 1 + 2 * Hb + 1));
}

// Interiors are branch-free: the staged rows and the Z halo columns hold exactly what the rule
// reads there (forward reflective: the reflected data; otherwise zeros), so every tap is one
// shared load and one FMA. The adjoint's fold terms (reflective only) touch the first / last H
// outputs of an axis and run as separate corrections there.
__global__ void __launch_bounds__(kPsThreads) kb_solve_persistent(PsArgs a) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double ps_smem[];
  const int n = a.n, m = a.m, Ha = a.Ha, Hb = a.Hb, r = a.r, RB = a.RB;
  const int wa = 2 * Ha + 1, wb = 2 * Hb + 1, np = n + 2 * Hb;
  double* Ys = ps_smem;                      // staged rows g = r0 - Ha + t, t < RB + 2 Ha
  double* Zs = Ys + (size_t)(RB + 2 * Ha) * n;  // [r][RB][np], column c at Hb + c
  double* th = Zs + (size_t)r * RB * np;     // [r][wa]: th[i][k] = c_{Ha-k}
  double* tk = th + (size_t)r * wa;          // [r][wb]
  const int tid = threadIdx.x;
  for (int i = tid; i < r * wa; i += kPsThreads) th[i] = a.ha[(i / wa) * a.Wpa + i % wa];
  for (int i = tid; i < r * wb; i += kPsThreads) tk[i] = a.kbt[(i / wb) * a.Wpb + i % wb];
  const int r0 = blockIdx.x * RB;
  const int r1 = min(m, r0 + RB), nr = max(0, r1 - r0);
  const bool edge_rows = r0 < Ha || r1 > m - Ha;

  // stage rows [r0 - Ha, r1 + Ha) of src: in-domain rows by 16-byte cp.async.cg (all in flight
  // at once; .cg reads through to L2 -- other CTAs wrote them since this SM last looked, and L1
  // is not coherent across SMs); out-of-domain rows reflected (refl) or zero
  auto stage = [&](const double* src, int refl) {
    const int rows = nr + 2 * Ha, half = n >> 1;
    // one flat loop over (row, column pair): every thread busy (a row-by-row loop left half the
    // threads idle at n = 256 and doubled the staging iterations: 3.65k -> 3.05k Mpix*it/s)
    for (int idx = tid; idx < rows * half; idx += kPsThreads) {
      const int t = idx / half, c = 2 * (idx - t * half);
      const int g = ps_src(r0 - Ha + t, m, refl);
      double* dst = Ys + (size_t)t * n + c;
      if (g >= 0) {
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
  // axis 0 (rows): forward Z[t][c] = sum_k th[k] Ys[t + k][c] (x~(s - d), d = Ha - k);
  // adjoint correlation Z[t][c] = sum_k th[k] Ys[t + 2Ha - k][c] (x(s + d), zero outside).
  // (Sharing each staged value across the terms measured slower at cfg1: 3.25k vs 3.65k.)
  auto axis0 = [&](bool adjoint) {
    for (int t = 0; t < nr; ++t)
      for (int c = tid; c < n; c += kPsThreads)
        for (int i = 0; i < r; ++i) {
          const double* h = th + i * wa;
          const double* y = Ys + (size_t)t * n + c;
          double acc = 0.0;
          if (!adjoint) {
#pragma unroll 4
            for (int k = 0; k < wa; ++k) acc = fma(h[k], y[(size_t)k * n], acc);
          } else {
#pragma unroll 4
            for (int k = 0; k < wa; ++k) acc = fma(h[k], y[(size_t)(2 * Ha - k) * n], acc);
          }
          Zs[((size_t)i * RB + t) * np + Hb + c] = acc;
        }
    if (!(adjoint && a.refl_a && edge_rows)) return;
    // + the adjoint's forward-fold terms on the edge rows: sources s - d outside [0, m)
    for (int t = 0; t < nr; ++t) {
      const int s = r0 + t;
      if (s >= Ha && s < m - Ha) continue;
      for (int c = tid; c < n; c += kPsThreads)
        for (int i = 0; i < r; ++i) {
          const double* h = th + i * wa;
          double acc = Zs[((size_t)i * RB + t) * np + Hb + c];
          for (int k = 0; k < wa; ++k) {
            const int u = s - (Ha - k);
            if (u >= 0 && u < m) continue;
            const int f = ps_src(u, m, 1);
            if (f >= 0) acc = fma(h[k], Ys[(size_t)(f - r0 + Ha) * n + c], acc);
          }
          Zs[((size_t)i * RB + t) * np + Hb + c] = acc;
        }
    }
  };
  // Z halo columns: reflected values (forward reflective) or zeros
  auto zhalo = [&](int refl) {
    for (int idx = tid; idx < r * nr * 2 * Hb; idx += kPsThreads) {
      const int j = idx % (2 * Hb), row = idx / (2 * Hb);  // row = i * nr + t
      const int i = row / nr, t = row - i * nr;
      double* z = Zs + ((size_t)i * RB + t) * np;
      const int col = j < Hb ? j : Hb + n + (j - Hb);  // storage column
      const int q = ps_src(col - Hb, n, refl);
      z[col] = q >= 0 ? z[Hb + q] : 0.0;
    }
  };
  // axis 1 (columns) of one output: forward sum_k tk[k] z[c + k]; adjoint sum_k tk[k] z[c + 2Hb - k]
  auto axis1 = [&](int t, int c, bool adjoint) {
    double acc = 0.0;
    for (int i = 0; i < r; ++i) {
      const double* kk = tk + i * wb;
      const double* z = Zs + ((size_t)i * RB + t) * np + c;
      if (!adjoint) {
#pragma unroll 4
        for (int k = 0; k < wb; ++k) acc = fma(kk[k], z[k], acc);
      } else {
#pragma unroll 4
        for (int k = 0; k < wb; ++k) acc = fma(kk[k], z[2 * Hb - k], acc);
        if (a.refl_b && (c < Hb || c >= n - Hb)) {  // + the forward fold at the column edges
          for (int k = 0; k < wb; ++k) {
            const int u = c - (Hb - k);
            if (u >= 0 && u < n) continue;
            const int f = ps_src(u, n, 1);
            if (f >= 0) acc = fma(kk[k], z[f - c + Hb], acc);
          }
        }
      }
    }
    return acc;
  };

  // the epilogue operands of a thread's outputs are loaded before the passes run, so their L2
  // round trip overlaps the staging and the two axis passes (up to kPsPre outputs per thread)
  constexpr int kPsPre = 4;
  const int nout = nr * ((n - tid + kPsThreads - 1) / kPsThreads);  // this thread's outputs
  const bool pre = nout <= kPsPre;
  auto out_index = [&](int j) {  // j-th output of this thread: (row t, column c)
    const int per = (n - tid + kPsThreads - 1) / kPsThreads;
    return make_int2(j / per, tid + (j % per) * kPsThreads);
  };
  double p0[kPsPre], p1[kPsPre];

  // Between phases a CTA needs only the rows of the CTAs within Ha rows of its own (the halo of
  // the next axis-0 pass), so by default it waits for those CTAs' phase epochs (release/acquire
  // flags) instead of a grid-wide barrier. Before writing R (resp. Y) it has seen its neighbours
  // finish the phase that read them, so there is no write-after-read hazard either.
  const int b_lo = max(0, (r0 - Ha) / RB), b_hi = min((int)gridDim.x - 1, (r1 - 1 + Ha) / RB);
  auto signal = [&](int epoch) {
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(a.flags + blockIdx.x), "r"(epoch) : "memory");
    }
  };
  auto wait_for = [&](int epoch) {
    for (int b = b_lo + tid; b <= b_hi; b += kPsThreads) {
      int v;
      while (true) {
        asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(a.flags + b) : "memory");
        if (v >= epoch) break;
        __nanosleep(20);
      }
    }
    __syncthreads();
  };
  auto phase_end = [&](int epoch) {
    if (a.flags) signal(epoch);
    else grid.sync();
  };

  __syncthreads();
  for (int it = 0; it < a.iters; ++it) {
    const int k = a.k0 + it + 1;
    // ---- phase 1: R = A Y - B on rows [r0, r1)
    if (nr > 0) {
      if (pre)
#pragma unroll
        for (int j = 0; j < kPsPre; ++j)
          if (j < nout) {
            const int2 tc = out_index(j);
            p0[j] = a.B[(size_t)(r0 + tc.x) * n + tc.y];
          }
      if (a.flags && it > 0) wait_for(2 * it);  // neighbours' y_k rows written
      stage(a.Y, a.refl_a);
      __syncthreads();
      axis0(false);
      __syncthreads();
      zhalo(a.refl_b);
      __syncthreads();
      if (pre) {
#pragma unroll
        for (int j = 0; j < kPsPre; ++j)
          if (j < nout) {
            const int2 tc = out_index(j);
            a.R[(size_t)(r0 + tc.x) * n + tc.y] = __dsub_rn(axis1(tc.x, tc.y, false), p0[j]);
          }
      } else {
        for (int t = 0; t < nr; ++t)
          for (int c = tid; c < n; c += kPsThreads) {
            const size_t e = (size_t)(r0 + t) * n + c;
            a.R[e] = __dsub_rn(axis1(t, c, false), a.B[e]);
          }
      }
    }
    phase_end(2 * it + 1);
    // ---- phase 2: G = A^T R, x = (L y - g)/(L + lam^2), projection, momentum
    if (nr > 0) {
      if (pre)
#pragma unroll
        for (int j = 0; j < kPsPre; ++j)
          if (j < nout) {
            const int2 tc = out_index(j);
            const size_t e = (size_t)(r0 + tc.x) * n + tc.y;
            p0[j] = a.Y[e];
            p1[j] = a.X[e];
          }
      if (a.flags) wait_for(2 * it + 1);  // neighbours' R rows written
      stage(a.R, 0);
      __syncthreads();
      axis0(true);
      __syncthreads();
      zhalo(0);
      __syncthreads();
      const double bk = a.beta[it];
      bool bad = false;
      auto upd = [&](int t, int c, double yv, double xp) {
        const size_t e = (size_t)(r0 + t) * n + c;
        const double g = axis1(t, c, true);
        double x = __ddiv_rn(__dsub_rn(__dmul_rn(a.L, yv), g), a.denom);
        if (a.project && !(x > 0.0) && !isnan(x)) x = 0.0;  // np.maximum(x, 0): NaN kept (F3)
        bad |= !isfinite(x);
        a.X[e] = x;
        a.Y[e] = __dadd_rn(x, __dmul_rn(bk, __dsub_rn(x, xp)));
      };
      if (pre) {
#pragma unroll
        for (int j = 0; j < kPsPre; ++j)
          if (j < nout) {
            const int2 tc = out_index(j);
            upd(tc.x, tc.y, p0[j], p1[j]);
          }
      } else {
        for (int t = 0; t < nr; ++t)
          for (int c = tid; c < n; c += kPsThreads) {
            const size_t e = (size_t)(r0 + t) * n + c;
            upd(t, c, a.Y[e], a.X[e]);
          }
      }
      if (bad) atomicMin(a.nonfinite, k);
    }
    phase_end(2 * it + 2);
  }
}

}  // namespace kb
