// kb_kernels.cuh — sm_100a kernels for the sFISTA hot path (Kronecker-sum blur operator).
//
// The operator A_s X = sum_i H_i X K_i^T (kronblur kron.py:218-225) is evaluated as two
// separable one-dimensional "passes". Both passes read a row-major plane [S][L], filter along
// its slow axis S (each thread walks S in registers, the 32 lanes of a warp cover 32
// consecutive L), and write their result TRANSPOSED, [L][S], through a shared-memory stage —
// so every global access is a coalesced row segment and the second pass sees its filter axis
// as the slow axis again:
//
//   pass A "split" (S = m, L = n):  Z_i^T = (F(a_i) X)^T   for a group of G terms at once, so
//           one shared-memory read of X feeds G*R FMAs per thread; r planes [n][m] out.
//   pass B "sum"   (S = n, L = m):  Y = sum_i (F(b_i) Z_i^T)^T, summed in registers over all r
//           terms (double-buffered tiles), written as [m][n] with a fused epilogue:
//             PLAIN  Y                                 (kron_apply / kron_apply_adjoint)
//             RESID  R = Y - B                         (forward half of an sFISTA step)
//             UPDATE x = max0((L y - G)/(L + lam^2)); y' = x + beta (x - x_prev)
//                                                      (solvers.py:170-173, + projection)
//             POWER  w = Y; <v,w>, ||w||^2 partials    (solvers.py:122-129)
//
// A one-dimensional factor F(c) is the banded Toeplitz (zero BC) or Toeplitz+Hankel
// (reflective BC) matrix of structured.py:111-123. With stencil taps c_d = c[j+d] it is
//     y[s] = sum_d c_d * xt(s - d),
// xt = x inside the domain, x[refl(t)] outside it for the reflective kind (single fold,
// refl(t) = -1-t below 0 and 2M-1-t above M-1, dropped if the fold leaves the domain), 0
// for the zero kind. Written over source offsets e = t - s the forward uses the
// coefficient c_{-e} for every source ("conv" table): its main loop runs over a reflect-filled
// shared-memory tile, so the boundary costs nothing. The transpose F^T (structured.py:191,195)
// uses c_{+e} for in-domain sources ("corr" table) and c_{-e} for folded out-of-domain sources
// (SURVEY F4): its main loop runs over a zero-filled tile with the corr table, and the folded
// part (at most H-s taps for an output s within H of an edge) is added by the small, balanced
// kb_fold_rows / kb_fold_cols kernels, so no warp of the main kernels carries edge work.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace kb {

constexpr int kUB = 16;  // tap tables are padded to a multiple of 16 (>= both passes' R)
constexpr int kNW = 8;   // warps per CTA

enum EpiMode { EPI_PLAIN = 0, EPI_RESID = 1, EPI_UPDATE = 2, EPI_POWER = 3 };

// Geometry of a pass over an input plane [S][L] (row stride L). Local S index 0 is global
// index g0; the plane has `len` local rows and `halo_lo`/`halo_hi` extra readable rows on
// either side (row-block sharding); the domain (for zero-fill / reflection) is [0, Mg).
struct AxisGeom {
  int len;      // local extent along S (rows of the input plane, columns of the output plane)
  int other;    // extent along L (columns of the input plane, rows of the output plane)
  int H;        // half width of the (symmetric, zero padded) tap window
  int Wp;       // padded tap count (multiple of kUB, >= 2H+1): row stride of the tap tables
  int Kw;       // taps the tensor-core passes cover: 2H+1 rounded up to a multiple of 4
  int fill;     // 1 = reflect-fill out-of-domain tile entries (forward, reflective kind)
  int g0;       // global index of local 0
  int Mg;       // global extent of the domain
  int halo_lo;  // readable entries before local 0
  int halo_hi;  // readable entries after local len-1
  int dbg;      // profiling switch (KB_DEBUG_MODE): bit0 skip MMAs, bit1 skip result stores,
                //   bit2 skip tile loads (persistent kernels)
};

template <typename T>
struct Epi {
  int mode;
  T* out;              // PLAIN/RESID/POWER output plane
  const T* bsub;       // RESID: data B
  T* x;                // UPDATE: x_{k-1} in, x_k out
  T* y;                // UPDATE: y_k in, y_{k+1} out
  const double* L;     // UPDATE: per-image Lipschitz constant
  const double* denom; // UPDATE: per-image L + lam^2
  double beta;         // UPDATE: (t_k - 1) / t_{k+1}
  int project;         // UPDATE: clamp x at 0 (NaN preserving)
  int k;               // UPDATE: iteration number (1-based) for the non-finite flag
  int* nonfinite;      // UPDATE: atomicMin target (first k with a non-finite x)
  const T* vin;        // POWER: previous (unnormalised) w, v = vin / sqrt(*vnw2)
  const double* vnw2;  // POWER: per-image ||w_prev||^2 (nullptr: vin already normalised)
  double* partials;    // POWER/UPDATE-with-norms: [batch][gridblocks][4]
  int want_norms;      // UPDATE: accumulate ||x-xp||^2, ||xp||^2, ||x||^2
  long long bstride;   // elements between images for out/bsub/x/y/vin
  const T* fold;       // adjoint, exact fold on axis 1: [batch][m][2*foldH] edge corrections
  int foldH;           // half width of axis 1 (0: no fold corrections)
};

__device__ __forceinline__ double kb_fma(double a, double b, double c) { return fma(a, b, c); }
__device__ __forceinline__ float kb_fma(float a, float b, float c) { return fmaf(a, b, c); }

template <typename T> __device__ __forceinline__ T rn_mul(T a, T b);
template <typename T> __device__ __forceinline__ T rn_add(T a, T b);
template <typename T> __device__ __forceinline__ T rn_sub(T a, T b);
template <typename T> __device__ __forceinline__ T rn_div(T a, T b);
template <> __device__ __forceinline__ double rn_mul<double>(double a, double b) { return __dmul_rn(a, b); }
template <> __device__ __forceinline__ double rn_add<double>(double a, double b) { return __dadd_rn(a, b); }
template <> __device__ __forceinline__ double rn_sub<double>(double a, double b) { return __dsub_rn(a, b); }
template <> __device__ __forceinline__ double rn_div<double>(double a, double b) { return __ddiv_rn(a, b); }
template <> __device__ __forceinline__ float rn_mul<float>(float a, float b) { return __fmul_rn(a, b); }
template <> __device__ __forceinline__ float rn_add<float>(float a, float b) { return __fadd_rn(a, b); }
template <> __device__ __forceinline__ float rn_sub<float>(float a, float b) { return __fsub_rn(a, b); }
template <> __device__ __forceinline__ float rn_div<float>(float a, float b) { return __fdiv_rn(a, b); }

// reflected partner of an out-of-domain global index, or -1 when the single fold leaves the
// domain (structured.py:118-123: the Hankel part only carries one reflection per edge)
__device__ __forceinline__ int kb_fold(int t, int M) {
  int u = (t < 0) ? (-1 - t) : (2 * M - 1 - t);
  return (u >= 0 && u < M) ? u : -1;
}

__device__ __forceinline__ void cp_async_4(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_8(void* smem, const void* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
template <typename T> __device__ __forceinline__ void cp_async_elem(T* smem, const T* gmem);
template <> __device__ __forceinline__ void cp_async_elem<double>(double* s, const double* g) { cp_async_8(s, g); }
template <> __device__ __forceinline__ void cp_async_elem<float>(float* s, const float* g) { cp_async_4(s, g); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> __device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// ------------------------------------------------------------------------------------------
// Register-blocked banded dot products along the serial axis of one thread.
//   acc[g][j] += sum_k c_g[k] * x[(j + k) * 32],   j < R, k < Wp   (Wp a multiple of R)
// x is a column of a [rows][32] shared-memory tile. The window slides R taps at a time through
// two register arrays whose roles alternate, so each tap costs one new load and the loads of
// the next block overlap the FMAs of the current one.
// ------------------------------------------------------------------------------------------
template <typename T, int G, int R>
__device__ __forceinline__ void kb_taps(T (&acc)[G][R], const T* __restrict__ x,
                                        const T* __restrict__ coef, int cstride, int Wp) {
  T A[R], B[R];
#pragma unroll
  for (int j = 0; j < R; ++j) A[j] = x[j * 32];
  for (int k0 = 0; k0 < Wp; k0 += 2 * R) {
#pragma unroll
    for (int j = 0; j < R; ++j) B[j] = x[(k0 + R + j) * 32];
#pragma unroll
    for (int kk = 0; kk < R; ++kk) {
#pragma unroll
      for (int gg = 0; gg < G; ++gg) {
        const T c = coef[gg * cstride + k0 + kk];
#pragma unroll
        for (int j = 0; j < R; ++j) acc[gg][j] = kb_fma(c, (j + kk < R) ? A[j + kk] : B[j + kk - R], acc[gg][j]);
      }
    }
    if (k0 + R >= Wp) break;
#pragma unroll
    for (int j = 0; j < R; ++j) A[j] = x[(k0 + 2 * R + j) * 32];
#pragma unroll
    for (int kk = 0; kk < R; ++kk) {
#pragma unroll
      for (int gg = 0; gg < G; ++gg) {
        const T c = coef[gg * cstride + k0 + R + kk];
#pragma unroll
        for (int j = 0; j < R; ++j) acc[gg][j] = kb_fma(c, (j + kk < R) ? B[j + kk] : A[j + kk - R], acc[gg][j]);
      }
    }
  }
}

// Fill rows [0, rows) of a [rows][32] tile with input rows S = row_lo + rr (global), lanes
// over L = l0 + lane. In-domain rows stream in with cp.async; out-of-domain rows are folded
// (times `sign`) when g.fill, else zero.
template <typename T, int XS = 32>
__device__ __forceinline__ void kb_fill_tile(T* __restrict__ xs, const T* __restrict__ in,
                                             const AxisGeom& g, int row_lo, int rows, int l,
                                             int warp, int lane, int sign) {
  for (int rr = warp; rr < rows; rr += kNW) {
    int gr = row_lo + rr;
    const bool outside = gr < 0 || gr >= g.Mg;
    if (g.fill && outside) gr = kb_fold(gr, g.Mg);
    const int lr = gr - g.g0;
    T* d = xs + rr * XS + lane;
    const bool ok = l < g.other && gr >= 0 && gr < g.Mg && lr >= -g.halo_lo && lr < g.len + g.halo_hi;
    if (ok && !outside) cp_async_elem<T>(d, in + (long long)lr * g.other + l);
    else *d = ok ? (sign < 0 ? -in[(long long)lr * g.other + l] : in[(long long)lr * g.other + l]) : T(0);
  }
}

// ------------------------------------------------------------------------------------------
// pass A (split): Z_i^T[l][s] = sum_k c_i[k] X[s - H + k][l] for every term of a group.
//   CTA = 32 lanes (L) x kNW warps; each warp owns R consecutive outputs along S, so the CTA
//   tile is TS = kNW*R along S by 32 along L; the input tile holds TS + Wp rows.
// in   : input plane [S][L] (local rows may extend to -halo_lo .. len+halo_hi-1)
// z    : r output planes [L][S] (z_ps per plane, z_bs per image)
// tin  : taps [batch][r][Wp], index k = e + H for source offset e
// grp  : term groups; with g.fill the out-of-domain tile rows hold sign * x[refl(row)] with the
//        group's sign (adjoint of (anti)symmetric generators: see kb_capi.cu)
// nw2  : optional per-image ||in||^2; outputs are divided by sqrt(nw2) (power iteration)
// ------------------------------------------------------------------------------------------
#ifndef KB_MAX_GROUPS
#define KB_MAX_GROUPS 160
#endif
constexpr int kMaxGroups = KB_MAX_GROUPS;  // up to 318 (fp64) / 636 (fp32) terms: full-rank restore() operators
struct Groups {
  int n;
  int start[kMaxGroups];
  int count[kMaxGroups];
  int sign[kMaxGroups];
};

template <typename T, int G, int R>
__device__ __forceinline__ void kb_split_group(const T* __restrict__ xs, const T* __restrict__ cin,
                                               T* __restrict__ ot, const AxisGeom& g, int s_off,
                                               int lane, int warp, T* __restrict__ z,
                                               long long z_ps, int gstart, int s0, int l0,
                                               T oscale) {
  constexpr int TS = kNW * R;
  T acc[G][R];
#pragma unroll
  for (int gg = 0; gg < G; ++gg)
#pragma unroll
    for (int j = 0; j < R; ++j) acc[gg][j] = T(0);
  kb_taps<T, G, R>(acc, xs + s_off * 32 + lane, cin, g.Wp, g.Wp);
#pragma unroll
  for (int gg = 0; gg < G; ++gg) {
#pragma unroll
    for (int j = 0; j < R; ++j) ot[lane * (TS + 1) + s_off + j] = acc[gg][j] * oscale;
    __syncthreads();
    T* zp = z + (long long)(gstart + gg) * z_ps;
    for (int l = warp; l < 32; l += kNW) {
      if (l0 + l >= g.other) break;
      T* zrow = zp + (long long)(l0 + l) * g.len + s0;
#pragma unroll
      for (int s = lane; s < TS; s += 32)
        if (s0 + s < g.len) zrow[s] = ot[l * (TS + 1) + s];
    }
    __syncthreads();
  }
}

template <typename T, int GMAX, int R>
__global__ void __launch_bounds__(32 * kNW, 2)
kb_pass_split(const T* __restrict__ in, long long in_bs, T* __restrict__ z, long long z_ps,
              long long z_bs, const T* __restrict__ tin, long long t_bs, AxisGeom g, Groups grp,
              const double* __restrict__ nw2) {
  extern __shared__ __align__(16) unsigned char kb_smem_a[];
  constexpr int TS = kNW * R;
  const int rows_tile = TS + g.Wp;               // window reads reach s_off + Wp + R - 1
  T* xs = reinterpret_cast<T*>(kb_smem_a);       // [rows_tile][32]
  T* cin = xs + rows_tile * 32;                  // [GMAX][Wp]
  T* ot = cin + GMAX * g.Wp;                     // [32][TS + 1] transpose stage
  const int lane = threadIdx.x, warp = threadIdx.y;
  const int tid = warp * 32 + lane;
  const int b = blockIdx.z;
  const int s0 = blockIdx.y * TS;
  const int l0 = blockIdx.x * 32;
  in += b * in_bs;
  z += b * z_bs;
  tin += b * t_bs;
  const int row_lo = g.g0 + s0 - g.H;            // global S index of tile row 0
  const bool has_out = g.fill && (row_lo < 0 || row_lo + rows_tile > g.Mg);
  int cur_sign = grp.sign[0];
  kb_fill_tile<T>(xs, in, g, row_lo, rows_tile, l0 + lane, warp, lane, cur_sign);
  cp_async_commit();
  const T oscale = nw2 ? (T)(1.0 / sqrt(nw2[b])) : T(1);
  cp_async_wait<0>();

  const int s_off = warp * R;
  for (int gi = 0; gi < grp.n; ++gi) {
    const int gstart = grp.start[gi], gcount = grp.count[gi];
    __syncthreads();
    if (has_out && grp.sign[gi] != cur_sign) {  // flip the folded rows for this group's sign
      for (int rr = warp; rr < rows_tile; rr += kNW) {
        const int gr = row_lo + rr;
        if (gr < 0 || gr >= g.Mg) xs[rr * 32 + lane] = -xs[rr * 32 + lane];
      }
    }
    cur_sign = grp.sign[gi];
    for (int idx = tid; idx < gcount * g.Wp; idx += 32 * kNW) cin[idx] = tin[(long long)gstart * g.Wp + idx];
    __syncthreads();
#define KB_GROUP(C)                                                                           \
  case C:                                                                                     \
    if constexpr (C <= GMAX)                                                                  \
      kb_split_group<T, C, R>(xs, cin, ot, g, s_off, lane, warp, z, z_ps, gstart, s0, l0, oscale); \
    break;
    switch (gcount) {
      KB_GROUP(1)
      KB_GROUP(2)
      KB_GROUP(3)
      KB_GROUP(4)
      KB_GROUP(5)
      KB_GROUP(6)
      KB_GROUP(7)
      KB_GROUP(8)
      default: break;
    }
#undef KB_GROUP
  }
}

// ------------------------------------------------------------------------------------------
// Exact adjoint fold corrections (used when the generators are not (anti)symmetric, so the
// sign-reflected tile fill does not apply). For an output index s within H of a reflective
// domain edge, the transpose adds  sum_{t out of domain} c_{s-t} x[refl(t)]  (conv table,
// k = t-s+H):   left/top edge:  u = -1-t in [0, min(H-s, M)),  k = H-s-1-u
//               right/bottom:   t in [max(M, s-H), s+H],  u = 2M-1-t,  k = t-s+H
// ------------------------------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T kb_fold_sum(const T* __restrict__ tc, const T* __restrict__ src,
                                         long long stride, int s, int H, int M) {
  T acc = T(0);
  const int top = min(H - s, M);
#pragma unroll 4
  for (int u = 0; u < top; ++u) acc = kb_fma(tc[H - s - 1 - u], src[(long long)u * stride], acc);
  for (int t = max(M, s - H); t <= s + H; ++t) {
    const int u = 2 * M - 1 - t;
    if (u >= 0) acc = kb_fma(tc[t - s + H], src[(long long)u * stride], acc);
  }
  return acc;
}

// split-pass fold: Z_i^T[l][s] += fold over S of in[:, l], for edge S positions s. One thread
// per (L index, edge slot, term); slot < H is S = slot, slot >= H is S = Mg-2H+slot.
template <typename T>
__global__ void __launch_bounds__(128)
kb_fold_split(const T* __restrict__ in, long long in_bs, T* __restrict__ z, long long z_ps,
              long long z_bs, int r, const T* __restrict__ tconv, long long t_bs, AxisGeom g,
              int mirror_h, const T* __restrict__ msign) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  const int slot = blockIdx.y % (2 * g.H);
  const int i = blockIdx.y / (2 * g.H);
  const int b = blockIdx.z;
  if (l >= g.other || i >= r) return;
  const int H = g.H, M = g.Mg;
  const int s = slot < H ? slot : M - 2 * H + slot;  // global S index
  if (s < 0 || s >= M || (slot >= H && s < H)) return;
  const int ls = s - g.g0;
  if (ls < 0 || ls >= g.len) return;  // not on this row block
  const T* tc = tconv + b * t_bs + (long long)i * g.Wp;
  const T* src = in + b * in_bs + l - (long long)g.g0 * g.other;  // src[u*other] = global row u
  const T acc = kb_fold_sum<T>(tc, src, g.other, s, H, M);
  T* zp = z + b * z_bs + (long long)i * z_ps + ls;
  zp[(long long)l * g.len] += acc;
  if (mirror_h > 0) {  // keep the reflected halo rows of Z^T (see the persistent split) in step
    const T sg = msign ? msign[(long long)b * r + i] : T(1);
    if (l < mirror_h) zp[(long long)(-1 - l) * g.len] += sg * acc;
    if (l >= g.other - mirror_h) zp[(long long)(2 * g.other - 1 - l) * g.len] += sg * acc;
  }
}

// sum-pass fold: fold[b][l][slot] = sum_i fold over S of Z_i^T[:, l] for edge S positions
// (slot < H: S = slot; slot >= H: S = n-2H+slot), added by the sum pass epilogue. One thread
// per (L index, slot); lanes run along L so every source row is read coalesced.
template <typename T>
__global__ void __launch_bounds__(128)
kb_fold_sum_pass(const T* __restrict__ z, long long z_ps, long long z_bs, int r,
                 const T* __restrict__ tconv, long long t_bs, AxisGeom g, T* __restrict__ fold) {
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  const int slot = blockIdx.y;
  const int b = blockIdx.z;
  const int n = g.len, H = g.H;
  if (l >= g.other) return;
  const int s = slot < H ? slot : n - 2 * H + slot;
  T acc = T(0);
  if (s >= 0 && s < n && !(slot >= H && s < H)) {
    const T* zl = z + b * z_bs + l;
    const T* tcb = tconv + b * t_bs;
    for (int i = 0; i < r; ++i)
      acc += kb_fold_sum<T>(tcb + (long long)i * g.Wp, zl + (long long)i * z_ps, g.other, s, H, n);
  }
  fold[((long long)b * g.other + l) * (2 * H) + slot] = acc;
}

// block reduction of NQ doubles into partials[b][block][0..NQ-1] (deterministic order)
template <int NQ>
__device__ __forceinline__ void kb_block_partials(double (&v)[NQ], double* partials, int b,
                                                  int nblk, int blk) {
  __shared__ double red[kNW][4];
  const int lane = threadIdx.x, warp = threadIdx.y;
#pragma unroll
  for (int qq = 0; qq < NQ; ++qq) {
    double s = v[qq];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) red[warp][qq] = s;
  }
  __syncthreads();
  if (warp == 0 && lane < NQ) {
    double s = 0.0;
    for (int w = 0; w < kNW; ++w) s += red[w][lane];
    partials[((long long)b * nblk + blk) * 4 + lane] = s;
  }
}

// Fused epilogue of the sum pass: ot[l*(TS+1) + s] holds the block's [32 L][TS S] results.
// Outputs with S index in [s0, s_end) are written; per-thread norm partials and the
// non-finite flag accumulate in nrm / bad (reduced by kb_sum_finish).
template <typename T, int MODE, int TS>
__device__ __forceinline__ void kb_sum_epilogue(const T* __restrict__ ot, const AxisGeom& g,
                                                const Epi<T>& e, int b, int s0, int s_end, int l0,
                                                int warp, int lane, double (&nrm)[3], bool& bad) {
  // warp w handles output rows l = w, w+kNW, ..; lanes walk the row's TS outputs.
  constexpr int NS = TS / 32;  // outputs per lane per row
  const double vs = (MODE == EPI_POWER && e.vnw2) ? sqrt(e.vnw2[b]) : 1.0;
  const int n = s_end;
  for (int l = warp; l < 32; l += kNW) {
    const int p = l0 + l;
    if (p >= g.other) break;
    const long long base = (long long)b * e.bstride + (long long)p * g.len + s0;
    T v[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      const int s = lane + 32 * k;
      v[k] = ot[l * (TS + 1) + s];
      if (e.foldH > 0) {  // exact-fold corrections near the left / right edges
        const int q = s0 + s, FH = e.foldH, N = g.len;
        const T* fr = e.fold + ((long long)b * g.other + p) * (2 * FH);
        if (q < FH) v[k] += fr[q];
        else if (q >= N - FH && q < N) v[k] += fr[q - (N - 2 * FH)];
      }
    }
    if constexpr (MODE == EPI_PLAIN || MODE == EPI_RESID) {
      T bv[NS];
#pragma unroll
      for (int k = 0; k < NS; ++k) {
        const int s = lane + 32 * k;
        bv[k] = (MODE == EPI_RESID && s0 + s < n) ? e.bsub[base + s] : T(0);
      }
#pragma unroll
      for (int k = 0; k < NS; ++k) {
        const int s = lane + 32 * k;
        if (s0 + s < n) e.out[base + s] = (MODE == EPI_RESID) ? rn_sub<T>(v[k], bv[k]) : v[k];
      }
    } else if constexpr (MODE == EPI_UPDATE) {
      const T Lt = (T)e.L[b], dt = (T)e.denom[b], bt = (T)e.beta;
      T yv[NS], xp[NS];
#pragma unroll
      for (int k = 0; k < NS; ++k) {
        const int s = lane + 32 * k;
        const bool ok = s0 + s < n;
        yv[k] = ok ? e.y[base + s] : T(0);
        xp[k] = ok ? e.x[base + s] : T(0);
      }
#pragma unroll
      for (int k = 0; k < NS; ++k) {
        const int s = lane + 32 * k;
        if (s0 + s < n) {
          T xv = rn_div<T>(rn_sub<T>(rn_mul<T>(Lt, yv[k]), v[k]), dt);
          if (e.project) xv = (xv > T(0) || xv != xv) ? xv : T(0);
          const T d = rn_sub<T>(xv, xp[k]);
          e.x[base + s] = xv;
          e.y[base + s] = rn_add<T>(xv, rn_mul<T>(bt, d));
          bad |= !isfinite((double)xv);
          if (e.want_norms) {
            nrm[0] += (double)d * (double)d;
            nrm[1] += (double)xp[k] * (double)xp[k];
            nrm[2] += (double)xv * (double)xv;
          }
        }
      }
    } else {  // EPI_POWER
      T vi[NS];
#pragma unroll
      for (int k = 0; k < NS; ++k) {
        const int s = lane + 32 * k;
        vi[k] = (s0 + s < n) ? e.vin[base + s] : T(0);
      }
#pragma unroll
      for (int k = 0; k < NS; ++k) {
        const int s = lane + 32 * k;
        if (s0 + s < n) {
          const T w = v[k];
          T vv = vi[k];
          if (e.vnw2) vv = (T)((double)vv / vs);
          e.out[base + s] = w;
          nrm[0] += (double)vv * (double)w;
          nrm[1] += (double)w * (double)w;
        }
      }
    }
  }
}

// Block-level end of the sum pass: non-finite flag and deterministic norm partials.
template <typename T, int MODE>
__device__ __forceinline__ void kb_sum_finish(const Epi<T>& e, double (&nrm)[3], bool bad, int b,
                                              int nblk, int blk, int lane) {
  if constexpr (MODE == EPI_UPDATE) {
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicMin(e.nonfinite, e.k);
    if (e.want_norms) kb_block_partials<3>(nrm, e.partials, b, nblk, blk);
  } else if constexpr (MODE == EPI_POWER) {
    double v2[2] = {nrm[0], nrm[1]};
    kb_block_partials<2>(v2, e.partials, b, nblk, blk);
  }
}

// ------------------------------------------------------------------------------------------
// pass B (sum): Y[l][s] = sum_i sum_k c_i[k] Z_i^T[s - H + k][l], with the fused epilogue.
//   Same CTA geometry as the split pass (TS = kNW*R along S, 32 along L); term tiles are double
//   buffered with cp.async; the result is transposed through shared memory so the epilogue
//   reads and writes [L][S] = [m][n] rows coalesced.
// ------------------------------------------------------------------------------------------
template <typename T, int R, int MODE>
__global__ void __launch_bounds__(32 * kNW, 2)
kb_pass_sum(const T* __restrict__ z, long long z_ps, long long z_bs, int r,
            const T* __restrict__ tin, long long t_bs, AxisGeom g, const T* __restrict__ tsign,
            Epi<T> e) {
  extern __shared__ __align__(16) unsigned char kb_smem_b[];
  constexpr int TS = kNW * R;
  const int rows_tile = TS + g.Wp;
  T* xs = reinterpret_cast<T*>(kb_smem_b);   // [2][rows_tile][32]; reused as [32][TS+1] at the end
  T* cin = xs + 2 * rows_tile * 32;          // [2][Wp]
  const int lane = threadIdx.x, warp = threadIdx.y;
  const int tid = warp * 32 + lane;
  const int b = blockIdx.z;
  const int s0 = blockIdx.y * TS;
  const int l0 = blockIdx.x * 32;
  z += b * z_bs;
  tin += b * t_bs;
  const int row_lo = g.g0 + s0 - g.H;

  auto load_term = [&](int i, int stage) {
    const int sgn = tsign ? (tsign[(long long)b * r + i] < T(0) ? -1 : 1) : 1;
    kb_fill_tile<T>(xs + stage * rows_tile * 32, z + (long long)i * z_ps, g, row_lo, rows_tile,
                    l0 + lane, warp, lane, sgn);
    for (int k = tid; k < g.Wp; k += 32 * kNW) cin[stage * g.Wp + k] = tin[(long long)i * g.Wp + k];
    cp_async_commit();
  };

  T acc[1][R];
#pragma unroll
  for (int j = 0; j < R; ++j) acc[0][j] = T(0);
  const int s_off = warp * R;

  load_term(0, 0);
  for (int i = 0; i < r; ++i) {
    const int st = i & 1;
    if (i + 1 < r) {
      load_term(i + 1, st ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    kb_taps<T, 1, R>(acc, xs + st * rows_tile * 32 + s_off * 32 + lane, cin + st * g.Wp, 0, g.Wp);
    __syncthreads();
  }

  // transpose stage: ot[l][s]
  T* ot = xs;
#pragma unroll
  for (int j = 0; j < R; ++j) ot[lane * (TS + 1) + s_off + j] = acc[0][j];
  __syncthreads();

  // ---------------------------------- epilogue ----------------------------------
  double nrm[3] = {0.0, 0.0, 0.0};
  bool bad = false;
  kb_sum_epilogue<T, MODE, TS>(ot, g, e, b, s0, g.len, l0, warp, lane, nrm, bad);
  kb_sum_finish<T, MODE>(e, nrm, bad, b, gridDim.x * gridDim.y, blockIdx.y * gridDim.x + blockIdx.x, lane);
}

// final deterministic reduction: out[q*qstride + b*bstride] = sum_blk partials[b][blk][q]
__global__ void kb_reduce_partials(const double* __restrict__ partials, int nblk, int nq,
                                   double* __restrict__ out, int qstride, int bstride) {
  const int b = blockIdx.x;
  __shared__ double sh[256][4];
  double s[4] = {0, 0, 0, 0};
  for (int i = threadIdx.x; i < nblk; i += blockDim.x)
    for (int qq = 0; qq < nq; ++qq) s[qq] += partials[((long long)b * nblk + i) * 4 + qq];
  for (int qq = 0; qq < 4; ++qq) sh[threadIdx.x][qq] = s[qq];
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w)
      for (int qq = 0; qq < 4; ++qq) sh[threadIdx.x][qq] += sh[threadIdx.x + w][qq];
    __syncthreads();
  }
  if ((int)threadIdx.x < nq) out[(long long)threadIdx.x * qstride + (long long)b * bstride] = sh[0][threadIdx.x];
}

}  // namespace kb
