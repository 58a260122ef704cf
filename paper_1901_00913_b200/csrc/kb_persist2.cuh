// kb_persist2.cuh — whole-solve persistent kernel, second form: zero-BC fp64 images with narrow
// bands (BASELINE cfg1: 256^2, w = 31, r = 3), one cooperative launch for the whole solve.
//
// Same phase structure as kb_solve_persistent (kb_persist.cuh): per iteration two grid barriers,
//   phase 1: R = A Y - B   (kronblur kron.py:218-225, solvers.py:170)
//   phase 2: G = A^T R, x = (L y - g)/(L + lam^2) [x >= 0], y = x + beta_k (x - x_prev)
//            (solvers.py:170-173)
// but with the per-phase critical path cut where the profile of the first form put it
// (profiles/r02_ncu_persist_cfg1.txt: a third of the stalls in the two axis loops, each FMA
// paired with two shared-memory loads, and 7% in the staging index arithmetic):
//   * staging is a few bulk copies (cp.async.bulk, 8 rows and one mbarrier each) of the
//     contiguous rows [r0 - 15, r1 + 15) clipped to the image, so axis 0 starts on the first rows
//     while the rest arrive; out-of-image rows are zero (zero BC) and stay zero because the
//     copies never touch them;
//   * the taps are compile-time indexed kernel parameters (constant bank operands of DFMA), the
//     band is centred in a fixed 31-tap window (half width 15; narrower bands are zero-padded),
//     and every staged value feeds all r terms' accumulators (r templated: registers);
//   * axis 1 runs on the FP64 tensor cores: for one image row, out[8a + b] =
//     sum_j zpad[8a + j] * tb[j - b] is an (n/8 x 40) . (40 x 8) product whose A operand is read
//     straight from the zero-padded Z row (Hankel view, no copy) and whose B operand (the
//     Toeplitz slice of the taps) is a per-lane table built once per launch; the r terms
//     accumulate in the same DMMA accumulators (m8n8k4, 10 K-steps per term and 64 outputs);
//   * the CTA's own x and y stay in registers for the whole launch (each lane updates the same
//     two outputs per 64-output block every iteration); only y (the neighbours' halo) and R are
//     written each phase, x once at the end; B is loaded once.
// Arithmetic: the update is the reference expression with explicit roundings (__dmul_rn etc.),
// projection np.maximum(x, 0) with NaN kept (F3). Sums run in a different order than the FFT
// path (fp64 tolerance 1e-10); integer data stay exact (bit-exact tests).
#pragma once
#include <cooperative_groups.h>

#include <type_traits>

namespace kb {

constexpr int kP2H = 15;             // window half width (taps centred, zero-padded)
constexpr int kP2W = 2 * kP2H + 1;   // 31 taps
constexpr int kP2KS = 10;            // axis-1 DMMA K-steps per term: W + 7 = 38 -> 40
constexpr int kP2Threads = 256;
constexpr int kP2MaxR = 4;

struct P2Args {
  const double* B;
  double* X;
  double* Y;
  double* R;
  const double* beta;  // [iters] momentum coefficients beta_{k0+1 ..}
  int* nonfinite;
  long long* trace;  // KB_P2_TRACE builds: clock64 stamps [CTA][16] of the middle iteration
  int* flags;  // [gridDim.x] phase epochs, zeroed before the launch; nullptr = grid-wide barriers
  int sync_mode;  // 0: cooperative-groups grid.sync, 1: neighbour flags, 2: one arrival counter (flags[0])
  double L, denom;
  int m, n, k0, iters, project;
  // centred taps: forward axis 0 Z[s] = sum_k fa[i][k] Y[s - 15 + k]; aa = the adjoint's
  // correlation taps; fb / ab the same for axis 1
  double fa[kP2MaxR][kP2W], aa[kP2MaxR][kP2W], fb[kP2MaxR][kP2W], ab[kP2MaxR][kP2W];
};

// Z rows: logical index j (column c at j = 15 + c; 15 zero columns in front, 17 behind) stored at
// j + 4 (j / 16). The axis-1 A fragment of a warp reads j = J0 + 8 (lane / 4) + lane % 4: without
// the gap, lane groups 16 apart hit the same banks (4 wavefronts per load); with it, 2.
#ifndef KB_P2_ZPAD
#define KB_P2_ZPAD 1
#endif
__host__ __device__ __forceinline__ int p2_zidx(int j) { return KB_P2_ZPAD ? j + 4 * (j >> 4) : j; }
__host__ __device__ inline int p2_zrow(int n) { return p2_zidx(n + 32); }
// dynamic shared memory: staged rows [RB + 30][n], Z rows [r][RB][p2_zrow(n)], axis-1 B
// fragments [2][r][10][32]
__host__ __device__ inline size_t p2_smem_bytes(int RB, int n, int r) {
  return sizeof(double) *
         ((size_t)(RB + 2 * kP2H) * n + (size_t)r * RB * p2_zrow(n) + (size_t)2 * r * kP2KS * 32);
}
#ifndef KB_P2_PIECE
#define KB_P2_PIECE 8
#endif
constexpr int kP2Piece = KB_P2_PIECE;  // staged rows per bulk copy / mbarrier (axis 0 starts on the first)
#ifndef KB_P2_FSTRIDE
#define KB_P2_FSTRIDE 32
#endif
#ifndef KB_P2_POLL_NS
#define KB_P2_POLL_NS 0
#endif
constexpr int kP2FlagStride = KB_P2_FSTRIDE;  // ints between two CTAs' phase flags (32: a 128-byte line each)
#ifndef KB_P2_DIRECT
#define KB_P2_DIRECT 0  // 1: axis 0 reads its source rows from L2 straight into registers (measured slower)
#endif
#ifndef KB_P2_BREG
#define KB_P2_BREG 1
#endif
#ifndef KB_P2_CHAINS
#define KB_P2_CHAINS 2
#endif

__device__ __forceinline__ void p2_dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// BREG: the lane's axis-1 B fragments stay in registers for the whole solve (~200 registers: one
// CTA per SM); without it the kernel fits two CTAs per SM (images of up to 2 x 148 x RB rows)
template <int R, int RB, bool BREG = (KB_P2_BREG != 0)>
__global__ void __launch_bounds__(kP2Threads) kb_solve_persistent2(const __grid_constant__ P2Args a) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) double p2_smem[];
  constexpr int NP = (RB + 2 * kP2H + kP2Piece - 1) / kP2Piece;
  __shared__ __align__(8) unsigned long long bar[NP];
  const int n = a.n, m = a.m, NZ = p2_zrow(n);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* Ys = p2_smem;                        // slot t <-> global row r0 - 15 + t
  double* Zs = Ys + (size_t)(RB + 2 * kP2H) * n;  // [R][RB][NZ], column c at p2_zidx(15 + c)
  double* Bf = Zs + (size_t)R * RB * NZ;       // [2][R][kP2KS][32]
  const int r0 = blockIdx.x * RB, nr = min(RB, m - r0);
  const int g_lo = max(0, r0 - kP2H), g_hi = min(m, r0 + RB + kP2H);

  // zero fill (out-of-image staged rows and the Z pads keep it for the whole solve), then the
  // per-lane B fragments: lane l, K-step s holds B[j = 4s + (l & 3)][b = l >> 2] = taps[j - b]
  for (int i = tid; i < (RB + 2 * kP2H) * n + R * RB * NZ; i += kP2Threads) p2_smem[i] = 0.0;
  for (int i = tid; i < 2 * R * kP2KS * 32; i += kP2Threads) {
    const int l = i & 31, s = (i >> 5) % kP2KS, ti = (i / (32 * kP2KS)) % R, adj = i / (32 * kP2KS * R);
    const int d = 4 * s + (l & 3) - (l >> 2);
    const double* tp = adj ? a.ab[ti] : a.fb[ti];
    Bf[i] = (d >= 0 && d < kP2W) ? tp[d] : 0.0;
  }
  if (tid == 0) {
    for (int p = 0; p < NP; ++p) mbar_init(&bar[p], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // the zero fill (generic proxy) precedes the bulk copies (async proxy) into the same rows
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  unsigned parity = 0;
  // staging: slot t <-> row r0 - 15 + t, in pieces of 8 slots, one bulk copy (rows are
  // contiguous) and one mbarrier each, so axis 0 starts on the first rows while the rest arrive;
  // pieces wholly outside the image only arrive
  auto stage = [&](const double* src) {
    // lane p of warp 0 issues piece p (the pieces' issue latencies overlap)
    if (!KB_P2_DIRECT && warp == 0 && lane < NP) {
      // rows written by other CTAs before the barrier (generic proxy) -> bulk copy (async proxy)
      asm volatile("fence.proxy.async.global;" ::: "memory");
      const int p = lane;
      const int lo = max(g_lo, r0 - kP2H + kP2Piece * p);
      const int hi = min(g_hi, r0 - kP2H + min(kP2Piece * (p + 1), RB + 2 * kP2H));
      if (hi > lo) {
        const unsigned bytes = (unsigned)((hi - lo) * n * sizeof(double));
        mbar_arrive_expect_tx(&bar[p], bytes);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(Ys + (size_t)(lo - (r0 - kP2H)) * n)),
            "l"(src + (size_t)lo * n), "r"(bytes), "r"(smem_u32(&bar[p]))
            : "memory");
      } else {
        mbar_arrive(&bar[p]);
      }
    }
  };
  // axis 0 on the staged rows: Z_i[t][c] = sum_k taps[i][k] Ys[t + k][c]; every staged value
  // feeds the R x RB accumulators of its column (taps: compile-time parameter offsets)
  auto axis0 = [&](const double (&tp)[kP2MaxR][kP2W], const double* __restrict__ src) {
    for (int c = tid; c < n; c += kP2Threads) {
      double acc[R][RB];
#pragma unroll
      for (int i = 0; i < R; ++i)
#pragma unroll
        for (int t = 0; t < RB; ++t) acc[i][t] = 0.0;
#if KB_P2_DIRECT
      // the column's RB + 30 source values straight from L2 into registers (ld.global.cg: other
      // SMs wrote them; a warp reads 256 contiguous bytes per row), all in flight at once
      double yv[RB + 2 * kP2H];
#pragma unroll
      for (int k2 = 0; k2 < RB + 2 * kP2H; ++k2) {
        const int gr = r0 - kP2H + k2;
        yv[k2] = (gr >= 0 && gr < m) ? __ldcg(src + (size_t)gr * n + c) : 0.0;
      }
#endif
#pragma unroll
      for (int k2 = 0; k2 < RB + 2 * kP2H; ++k2) {
#if KB_P2_DIRECT
        const double y = yv[k2];
#else
        if (k2 % kP2Piece == 0) mbar_wait(&bar[k2 / kP2Piece], parity);
        const double y = Ys[(size_t)k2 * n + c];
#endif
#pragma unroll
        for (int t = 0; t < RB; ++t) {
          const int k = k2 - t;
          if (k >= 0 && k < kP2W)
#pragma unroll
            for (int i = 0; i < R; ++i) acc[i][t] = fma(tp[i][k], y, acc[i][t]);
        }
      }
#pragma unroll
      for (int i = 0; i < R; ++i)
#pragma unroll
        for (int t = 0; t < RB; ++t) Zs[((size_t)i * RB + t) * NZ + p2_zidx(kP2H + c)] = acc[i][t];
    }
    parity ^= 1;
  };
  // 64-output blocks of axis 1: block mb = row mb / nmb, columns 64 (mb % nmb) + [0, 64);
  // warp w takes blocks w, w + 8 (<= RB per warp at n <= 512)
  const int nmb = n >> 6, nblk = nr * nmb;
  // lane's outputs in its block: column 64 mbc + 8 (lane >> 2) + 2 (lane & 3) + {0, 1}
  // KB_P2_CHAINS independent accumulator chains per term (K-steps dealt round robin), the terms
  // interleaved: a warp has one or two blocks per phase, so one chain of 10 r dependent DMMAs
  // would run at the instruction's latency. KB_P2_BREG: the lane's B fragments (both directions,
  // 20 r doubles) stay in registers for the whole solve instead of being re-read from shared
  // memory for every block (half of axis 1's shared-memory traffic).
  double bfr[BREG ? 2 : 1][BREG ? R : 1][BREG ? kP2KS : 1];
  if constexpr (BREG) {
#pragma unroll
    for (int adj = 0; adj < 2; ++adj)
#pragma unroll
      for (int i = 0; i < R; ++i)
#pragma unroll
        for (int s = 0; s < kP2KS; ++s) bfr[adj][i][s] = Bf[((size_t)(adj * R + i) * kP2KS + s) * 32 + lane];
  }
  auto axis1 = [&](int mb, auto adj_c, double (&d)[2]) {
    constexpr int adj = decltype(adj_c)::value;
    const int t = mb / nmb, mbc = mb - t * nmb;
    const int j0 = 64 * mbc + 8 * (lane >> 2) + (lane & 3);
    double acc[R][KB_P2_CHAINS][2];
#pragma unroll
    for (int i = 0; i < R; ++i)
#pragma unroll
      for (int h = 0; h < KB_P2_CHAINS; ++h) acc[i][h][0] = acc[i][h][1] = 0.0;
#pragma unroll
    for (int s = 0; s < kP2KS; ++s)
#pragma unroll
      for (int i = 0; i < R; ++i) {
        double b;
        if constexpr (BREG) b = bfr[adj][i][s];
        else b = Bf[((size_t)(adj * R + i) * kP2KS + s) * 32 + lane];
        p2_dmma(acc[i][s % KB_P2_CHAINS], Zs[((size_t)i * RB + t) * NZ + p2_zidx(j0 + 4 * s)], b);
      }
    d[0] = d[1] = 0.0;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      double t0 = acc[i][0][0], t1 = acc[i][0][1];
#pragma unroll
      for (int h = 1; h < KB_P2_CHAINS; ++h) {
        t0 = __dadd_rn(t0, acc[i][h][0]);
        t1 = __dadd_rn(t1, acc[i][h][1]);
      }
      d[0] = __dadd_rn(d[0], t0);
      d[1] = __dadd_rn(d[1], t1);
    }
  };
  auto out_col = [&](int mb) { return 64 * (mb % nmb) + 8 * (lane >> 2) + 2 * (lane & 3); };

  // Between phases a CTA needs only the rows of the CTAs within 15 rows of its own (the halo of
  // its next axis-0 pass), so with a.flags it waits for those CTAs' phase epochs -- warp 0, one
  // lane per neighbour, acquire loads -- instead of a grid-wide barrier; lane 0 then issues the
  // bulk copies. The same epochs order the writes: before writing R (resp. Y) a CTA has seen its
  // neighbours finish the phase that read the previous R (resp. Y).
  const int b_lo = max(0, (r0 - kP2H) / RB), b_hi = min((int)gridDim.x - 1, (r0 + RB - 1 + kP2H) / RB);
  auto wait_neighbours = [&](int epoch) {  // b_hi - b_lo < 32: one lane of warp 0 per neighbour
    if (epoch > 0 && a.sync_mode == 1) {
      if (warp == 0) {
        if (b_lo + lane <= b_hi) {
          int v;
          do {
            asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];"
                         : "=r"(v)
                         : "l"(a.flags + (size_t)(b_lo + lane) * kP2FlagStride)
                         : "memory");
            if (KB_P2_POLL_NS > 0 && v < epoch) __nanosleep(KB_P2_POLL_NS);
          } while (v < epoch);
          asm volatile("fence.acq_rel.gpu;" ::: "memory");
        }
        __syncwarp();
      }
      if (KB_P2_DIRECT) __syncthreads();  // every thread loads the neighbours' rows
    }
  };
  auto phase_end = [&](int epoch) {
    if (a.sync_mode == 1) {
      __syncthreads();  // the CTA's stores happen before thread 0's release (cumulative)
      if (tid == 0)
        asm volatile("st.release.gpu.global.s32 [%0], %1;" ::"l"(a.flags + (size_t)blockIdx.x * kP2FlagStride), "r"(epoch) : "memory");
    } else if (a.sync_mode == 2) {
      // grid barrier on one monotonic counter: release-add, relaxed polls, one acquire fence
      __syncthreads();
      if (tid == 0) {
        const int target = epoch * (int)gridDim.x;
        int v;
        asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(a.flags) : "memory");
        do {
          asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(a.flags) : "memory");
        } while (v < target);
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
      __syncthreads();
    } else {
      grid.sync();
    }
  };

  // register-resident state of the lane's outputs
  double xs[RB][2], ys[RB][2], bs[RB][2];
#pragma unroll
  for (int j = 0; j < RB; ++j) {
    const int mb = warp + 8 * j;
    if (mb < nblk) {
      const size_t e = (size_t)(r0 + mb / nmb) * n + out_col(mb);
      const double2 xv = *reinterpret_cast<const double2*>(a.X + e);
      const double2 yv = *reinterpret_cast<const double2*>(a.Y + e);
      const double2 bv = *reinterpret_cast<const double2*>(a.B + e);
      xs[j][0] = xv.x; xs[j][1] = xv.y;
      ys[j][0] = yv.x; ys[j][1] = yv.y;
      bs[j][0] = bv.x; bs[j][1] = bv.y;
    }
  }

#ifdef KB_P2_TRACE
  const bool tracing = a.trace && tid == 0;  // every CTA: [blockIdx.x][16] stamps of the middle iteration
  int tn = 0;
#define P2_STAMP() do { if (tracing && it == a.iters / 2) a.trace[16 * blockIdx.x + tn++] = clock64(); } while (0)
#else
#define P2_STAMP() do { } while (0)
#endif
  for (int it = 0; it < a.iters; ++it) {
    const int k = a.k0 + it + 1;
    // ---- phase 1: R = A Y - B on this CTA's rows
    if (nr > 0) {
      P2_STAMP();
      if (a.sync_mode == 1) wait_neighbours(2 * it);
      P2_STAMP();
      stage(a.Y);
      P2_STAMP();
      axis0(a.fa, a.Y);
      P2_STAMP();
      __syncthreads();
      P2_STAMP();
#pragma unroll
      for (int j = 0; j < RB; ++j) {
        const int mb = warp + 8 * j;
        if (mb < nblk) {
          double d[2];
          axis1(mb, std::integral_constant<int, 0>{}, d);
          const size_t e = (size_t)(r0 + mb / nmb) * n + out_col(mb);
          *reinterpret_cast<double2*>(a.R + e) = make_double2(__dsub_rn(d[0], bs[j][0]), __dsub_rn(d[1], bs[j][1]));
        }
      }
    }
    P2_STAMP();
    phase_end(2 * it + 1);
    P2_STAMP();
    // ---- phase 2: G = A^T R, FISTA update with projection and momentum
    if (nr > 0) {
      if (a.sync_mode == 1) wait_neighbours(2 * it + 1);
      P2_STAMP();
      stage(a.R);
      P2_STAMP();
      axis0(a.aa, a.R);
      P2_STAMP();
      __syncthreads();
      P2_STAMP();
      const double bk = a.beta[it];
      const double rdenom = 1.0 / a.denom;
      bool bad = false;
#pragma unroll
      for (int j = 0; j < RB; ++j) {
        const int mb = warp + 8 * j;
        if (mb < nblk) {
          double g[2];
          axis1(mb, std::integral_constant<int, 1>{}, g);
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            double x = kb_quot(__dsub_rn(__dmul_rn(a.L, ys[j][q]), g[q]), a.denom, rdenom);  // correctly rounded (kb_dmma.cuh)
            if (a.project && !(x > 0.0) && !isnan(x)) x = 0.0;  // np.maximum(x, 0): NaN kept (F3)
            bad |= !isfinite(x);
            ys[j][q] = __dadd_rn(x, __dmul_rn(bk, __dsub_rn(x, xs[j][q])));
            xs[j][q] = x;
          }
          const size_t e = (size_t)(r0 + mb / nmb) * n + out_col(mb);
          *reinterpret_cast<double2*>(a.Y + e) = make_double2(ys[j][0], ys[j][1]);
        }
      }
      if (bad) atomicMin(a.nonfinite, k);
    }
    P2_STAMP();
    phase_end(2 * it + 2);
    P2_STAMP();
  }
#pragma unroll
  for (int j = 0; j < RB; ++j) {
    const int mb = warp + 8 * j;
    if (mb < nblk) {
      const size_t e = (size_t)(r0 + mb / nmb) * n + out_col(mb);
      *reinterpret_cast<double2*>(a.X + e) = make_double2(xs[j][0], xs[j][1]);
    }
  }
}

}  // namespace kb
