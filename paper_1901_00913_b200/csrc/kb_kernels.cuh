// kb_kernels.cuh — sm_100a kernels for the sFISTA hot path (Kronecker-sum blur operator).
//
// The operator A_s X = sum_i H_i X K_i^T (kronblur kron.py:218-225) is evaluated as two
// separable one-dimensional "passes" over row-major (m, n) planes in HBM:
//
//   pass A  (filter along axis 0, lanes along axis 1):  Z_i = F(a_i) X      for a group of
//           G terms at once, so one shared-memory read of X feeds G*R FMAs per thread.
//   pass B  (filter along axis 1, lanes along axis 0):  Y = sum_i Z_i F(b_i)^T, summed in
//           registers over all r terms, followed by a fused epilogue:
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

constexpr int kU = 8;    // taps per unrolled chunk in pass A
constexpr int kUB = 16;  // taps per unrolled chunk in pass B (tables padded to a multiple of 16)
constexpr int kNW = 8;   // warps per CTA

enum EpiMode { EPI_PLAIN = 0, EPI_RESID = 1, EPI_UPDATE = 2, EPI_POWER = 3 };

// Geometry of the filtered axis. Local index 0 of the plane is global index g0; the plane
// has `len` local entries along the axis and `halo_lo`/`halo_hi` extra readable entries on
// either side (row-block sharding); the domain (for zero-fill / reflection) is [0, Mg).
struct AxisGeom {
  int len;      // local extent along the filtered axis
  int other;    // extent of the other axis
  int H;        // half width of the (symmetric, zero padded) tap window
  int Wp;       // padded tap count (multiple of kUB, >= 2H+1)
  int fill;     // 1 = reflect-fill out-of-domain tile entries (forward, reflective kind)
  int g0;       // global index of local 0
  int Mg;       // global extent of the domain
  int halo_lo;  // readable entries before local 0
  int halo_hi;  // readable entries after local len-1
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
  const T* fold;       // adjoint, reflective axis 1: [batch][rows][2*foldH] edge corrections
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
// pass A: filter along axis 0 (rows), terms processed in groups of up to GMAX.
//   CTA = 32 lanes (32 columns) x kNW warps; each warp owns R consecutive output rows, so the
//   CTA tile is (kNW*R) x 32 and the shared tile holds (kNW*R + Wp - 1) input rows.
// in  : plane (local rows may extend to -halo_lo .. len+halo_hi-1), batch stride in_bs
// z   : r output planes, plane stride z_ps, batch stride z_bs (same local row indexing as in)
// tin : taps [batch][r][Wp] (t_bs per image), index k = e + H for source offset e
// grp : term groups; with g.fill the out-of-domain tile rows hold sign * x[refl(row)], the sign
//       being the group's (adjoint of (anti)symmetric generators: see kb_capi.cu, sign_fill)
// nw2 : optional per-image ||in||^2; outputs are divided by sqrt(nw2) (power iteration)
// ------------------------------------------------------------------------------------------
constexpr int kMaxGroups = 16;
struct Groups {
  int n;
  int start[kMaxGroups];
  int count[kMaxGroups];
  int sign[kMaxGroups];
};

template <typename T, int G, int R>
__device__ __forceinline__ void kb_pass_a_group(const T* __restrict__ xs, const T* __restrict__ cin,
                                                int Wp, int s_off, int lane, T* __restrict__ z,
                                                long long z_ps, int gstart, int p0, int len,
                                                int ncol, int q, bool scaled, T oscale) {
  T acc[G][R];
#pragma unroll
  for (int gg = 0; gg < G; ++gg)
#pragma unroll
    for (int j = 0; j < R; ++j) acc[gg][j] = T(0);

  const T* xcol = xs + s_off * 32 + lane;
  for (int k0 = 0; k0 < Wp; k0 += kU) {
    T xw[R + kU - 1];
#pragma unroll
    for (int i = 0; i < R + kU - 1; ++i) xw[i] = xcol[(k0 + i) * 32];
#pragma unroll
    for (int kk = 0; kk < kU; ++kk) {
#pragma unroll
      for (int gg = 0; gg < G; ++gg) {
        const T c = cin[gg * Wp + k0 + kk];
#pragma unroll
        for (int j = 0; j < R; ++j) acc[gg][j] = kb_fma(c, xw[j + kk], acc[gg][j]);
      }
    }
  }
  if (q < ncol) {
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
      T* zp = z + (long long)(gstart + gg) * z_ps;
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const int lr = p0 + s_off + j;
        if (lr < len) zp[(long long)lr * ncol + q] = scaled ? acc[gg][j] * oscale : acc[gg][j];
      }
    }
  }
}

template <typename T, int GMAX, int R>
__global__ void __launch_bounds__(32 * kNW, 2)
kb_pass_a(const T* __restrict__ in, long long in_bs, T* __restrict__ z, long long z_ps,
          long long z_bs, const T* __restrict__ tin, long long t_bs, AxisGeom g, Groups grp,
          const double* __restrict__ nw2) {
  extern __shared__ __align__(16) unsigned char kb_smem_a[];
  constexpr int TP = kNW * R;
  const int rows_tile = TP + g.Wp - 1;
  T* xs = reinterpret_cast<T*>(kb_smem_a);   // [rows_tile][32]
  T* cin = xs + rows_tile * 32;              // [GMAX][Wp]
  const int lane = threadIdx.x, warp = threadIdx.y;
  const int tid = warp * 32 + lane;
  const int b = blockIdx.z;
  const int p0 = blockIdx.y * TP;
  const int q = blockIdx.x * 32 + lane;
  const int ncol = g.other;
  in += b * in_bs;
  z += b * z_bs;
  tin += b * t_bs;
  // Tile fill: rows [p0-H, p0+TP+Wp-1-H) of the input (folded when g.fill), one warp per row,
  // 8-byte cp.async per lane so every row load is in flight at once.
  const int row_lo = g.g0 + p0 - g.H;               // global row of tile row 0
  const bool has_out = g.fill && (row_lo < 0 || row_lo + rows_tile > g.Mg);
  int cur_sign = grp.sign[0];
  for (int rr = warp; rr < rows_tile; rr += kNW) {
    int gr = row_lo + rr;
    const bool outside = gr < 0 || gr >= g.Mg;
    if (g.fill && outside) gr = kb_fold(gr, g.Mg);
    const int lr = gr - g.g0;
    T* d = xs + rr * 32 + lane;
    const bool ok = q < ncol && gr >= 0 && gr < g.Mg && lr >= -g.halo_lo && lr < g.len + g.halo_hi;
    if (ok && !outside) cp_async_elem<T>(d, in + (long long)lr * ncol + q);
    else *d = ok ? (cur_sign < 0 ? -in[(long long)lr * ncol + q] : in[(long long)lr * ncol + q]) : T(0);
  }
  cp_async_commit();
  const bool scaled = nw2 != nullptr;
  const T oscale = scaled ? (T)(1.0 / sqrt(nw2[b])) : T(1);
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
    for (int idx = tid; idx < gcount * g.Wp; idx += 32 * kNW) {
      const int gg = idx / g.Wp, k = idx - gg * g.Wp;
      cin[idx] = tin[(long long)(gstart + gg) * g.Wp + k];
    }
    __syncthreads();
#define KB_GROUP(C)                                                                         \
  case C:                                                                                   \
    if constexpr (C <= GMAX)                                                                \
      kb_pass_a_group<T, C, R>(xs, cin, g.Wp, s_off, lane, z, z_ps, gstart, p0, g.len, ncol, \
                               q, scaled, oscale);                                          \
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

// axis 0: Z_i[s][q] += fold(R[:, q]) for edge rows s. One thread per (edge-row slot, column,
// term); slot < H is row `slot`, slot >= H is row Mg-2H+slot.
template <typename T>
__global__ void __launch_bounds__(128)
kb_fold_rows(const T* __restrict__ in, long long in_bs, T* __restrict__ z, long long z_ps,
             long long z_bs, int r, const T* __restrict__ tconv, long long t_bs, AxisGeom g) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  const int slot = blockIdx.y % (2 * g.H);
  const int i = blockIdx.y / (2 * g.H);
  const int b = blockIdx.z;
  if (q >= g.other || i >= r) return;
  const int H = g.H, M = g.Mg;
  const int s = slot < H ? slot : M - 2 * H + slot;  // global output row
  if (s < 0 || s >= M || (slot >= H && s < H)) return;
  const int ls = s - g.g0;
  if (ls < 0 || ls >= g.len) return;  // not on this row block
  const T* tc = tconv + b * t_bs + (long long)i * g.Wp;
  const T* src = in + b * in_bs + q - (long long)g.g0 * g.other;  // src[u*other] = global row u
  const T acc = kb_fold_sum<T>(tc, src, g.other, s, H, M);
  T* zp = z + b * z_bs + (long long)i * z_ps + (long long)ls * g.other + q;
  *zp = *zp + acc;
}

// axis 1: fold[b][p][slot] = sum_i fold(Z_i[p, :]) for edge columns (slot < H: column slot;
// slot >= H: column n-2H+slot); pass B's epilogue adds them. One thread per (row, slot).
template <typename T>
__global__ void __launch_bounds__(128)
kb_fold_cols(const T* __restrict__ z, long long z_ps, long long z_bs, int r,
             const T* __restrict__ tconv, long long t_bs, AxisGeom g, T* __restrict__ fold) {
  const int slot = blockIdx.x * blockDim.x + threadIdx.x;
  const int p = blockIdx.y;
  const int b = blockIdx.z;
  const int n = g.len, H = g.H;
  if (slot >= 2 * H) return;
  const int s = slot < H ? slot : n - 2 * H + slot;
  T acc = T(0);
  if (s >= 0 && s < n && !(slot >= H && s < H)) {
    const T* zr = z + b * z_bs + (long long)p * n;
    const T* tcb = tconv + b * t_bs;
    for (int i = 0; i < r; ++i)
      acc += kb_fold_sum<T>(tcb + (long long)i * g.Wp, zr + (long long)i * z_ps, 1, s, H, n);
  }
  fold[((long long)b * g.other + p) * (2 * H) + slot] = acc;
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

// ------------------------------------------------------------------------------------------
// pass B: filter along axis 1 (columns), summing all r terms in registers, fused epilogue.
//   CTA = 32 lanes (32 rows) x kNW warps; each warp owns R consecutive output columns, so the
//   CTA tile is 32 x (kNW*R). Term tiles are double buffered in shared memory with cp.async;
//   the tile row stride S is odd so the column-wise register windows are bank-conflict free.
// ------------------------------------------------------------------------------------------
template <typename T, int R, int MODE>
__global__ void __launch_bounds__(32 * kNW, 2)
kb_pass_b(const T* __restrict__ z, long long z_ps, long long z_bs, int r,
          const T* __restrict__ tin, long long t_bs, AxisGeom g, const T* __restrict__ tsign,
          Epi<T> e) {
  extern __shared__ __align__(16) unsigned char kb_smem_b[];
  constexpr int TQ = kNW * R;
  const int cols_tile = TQ + g.Wp - 1;
  const int S = cols_tile | 1;  // odd stride
  T* zs = reinterpret_cast<T*>(kb_smem_b);  // [2][32][S]
  T* cin = zs + 2 * 32 * S;                   // [2][Wp]
  const int lane = threadIdx.x, warp = threadIdx.y;
  const int tid = warp * 32 + lane;
  const int b = blockIdx.z;
  const int nrow = g.other;                   // rows of the plane (axis 0 extent)
  const int q0 = blockIdx.x * TQ;
  const int prow0 = blockIdx.y * 32;
  const int p = prow0 + lane;
  z += b * z_bs;
  tin += b * t_bs;

  // One warp per tile row, lanes across columns. With g.fill the out-of-domain columns hold
  // sign_i * Z_i[p][refl(q)] (sign_i = +1 for the forward; tsign[b][i] for the sign-filled
  // adjoint), loaded synchronously; in-domain columns go through cp.async.
  auto load_term = [&](int i, int stage) {
    const T* zp = z + (long long)i * z_ps;
    const T sgn = tsign ? tsign[(long long)b * r + i] : T(1);
    T* dst = zs + stage * 32 * S;
    for (int rr = warp; rr < 32; rr += kNW) {
      const int gp = prow0 + rr;
      const T* src = zp + (long long)gp * g.len;
      T* drow = dst + rr * S;
      for (int cc = lane; cc < cols_tile; cc += 32) {
        int gq = q0 - g.H + cc;
        const bool outside = gq < 0 || gq >= g.len;
        if (g.fill && outside) gq = kb_fold(gq, g.len);
        const bool ok = gp < nrow && gq >= 0 && gq < g.len;
        if (ok && !outside) cp_async_elem<T>(drow + cc, src + gq);
        else drow[cc] = ok ? sgn * src[gq] : T(0);
      }
    }
    for (int k = tid; k < g.Wp; k += 32 * kNW) cin[stage * g.Wp + k] = tin[(long long)i * g.Wp + k];
    cp_async_commit();
  };

  T acc[R];
#pragma unroll
  for (int j = 0; j < R; ++j) acc[j] = T(0);

  const int c_off = warp * R;
  const int s_first = q0 + c_off;  // first output column of this warp (columns are global)

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
    const T* zrow = zs + st * 32 * S + lane * S + c_off;
    const T* ci = cin + st * g.Wp;
    for (int k0 = 0; k0 < g.Wp; k0 += kUB) {
      T xw[R + kUB - 1];
#pragma unroll
      for (int t = 0; t < R + kUB - 1; ++t) xw[t] = zrow[k0 + t];
#pragma unroll
      for (int kk = 0; kk < kUB; ++kk) {
        const T c = ci[k0 + kk];
#pragma unroll
        for (int j = 0; j < R; ++j) acc[j] = kb_fma(c, xw[j + kk], acc[j]);
      }
    }
    __syncthreads();
  }

  // ---------------------------------- epilogue ----------------------------------
  const long long base = (long long)b * e.bstride + (long long)p * g.len;
  const bool prow_ok = p < nrow;
  if (e.foldH > 0 && prow_ok) {  // adjoint fold corrections near the left / right edges
    const int FH = e.foldH;
    const int right0 = g.len - 2 * FH;  // column of slot 0 in the right-edge numbering
    const T* fr = e.fold + ((long long)b * nrow + p) * (2 * FH);
#pragma unroll
    for (int j = 0; j < R; ++j) {
      const int qq = s_first + j;
      if (qq < FH) acc[j] += fr[qq];
      else if (qq - right0 >= FH && qq < g.len) acc[j] += fr[qq - right0];
    }
  }
  if constexpr (MODE == EPI_PLAIN || MODE == EPI_RESID) {
    if constexpr (MODE == EPI_RESID) {
      T bv[R];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const int qq = s_first + j;
        bv[j] = (prow_ok && qq < g.len) ? e.bsub[base + qq] : T(0);
      }
#pragma unroll
      for (int j = 0; j < R; ++j) acc[j] = rn_sub<T>(acc[j], bv[j]);
    }
    if (prow_ok) {
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const int qq = s_first + j;
        if (qq < g.len) e.out[base + qq] = acc[j];
      }
    }
  } else if constexpr (MODE == EPI_UPDATE) {
    const T Lt = (T)e.L[b];
    const T dt = (T)e.denom[b];
    const T bt = (T)e.beta;
    bool bad = false;
    double nrm[3] = {0.0, 0.0, 0.0};
    T yv_[R], xp_[R];
#pragma unroll
    for (int j = 0; j < R; ++j) {  // issue every operand load before the first use
      const int qq = s_first + j;
      const bool ok = prow_ok && qq < g.len;
      yv_[j] = ok ? e.y[base + qq] : T(0);
      xp_[j] = ok ? e.x[base + qq] : T(0);
    }
    if (prow_ok) {
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const int qq = s_first + j;
        if (qq < g.len) {
          const T yv = yv_[j];
          const T xp = xp_[j];
          T xv = rn_div<T>(rn_sub<T>(rn_mul<T>(Lt, yv), acc[j]), dt);
          if (e.project) xv = (xv > T(0) || xv != xv) ? xv : T(0);
          const T d = rn_sub<T>(xv, xp);
          const T yn = rn_add<T>(xv, rn_mul<T>(bt, d));
          e.x[base + qq] = xv;
          e.y[base + qq] = yn;
          bad |= !isfinite((double)xv);
          if (e.want_norms) {
            nrm[0] += (double)d * (double)d;
            nrm[1] += (double)xp * (double)xp;
            nrm[2] += (double)xv * (double)xv;
          }
        }
      }
    }
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicMin(e.nonfinite, e.k);
    if (e.want_norms) {
      const int nblk = gridDim.x * gridDim.y;
      kb_block_partials<3>(nrm, e.partials, b, nblk, blockIdx.y * gridDim.x + blockIdx.x);
    }
  } else {  // EPI_POWER
    const double vs = e.vnw2 ? sqrt(e.vnw2[b]) : 1.0;
    double pr[2] = {0.0, 0.0};
    if (prow_ok) {
#pragma unroll
      for (int j = 0; j < R; ++j) {
        const int qq = s_first + j;
        if (qq < g.len) {
          const T w = acc[j];
          T v = e.vin[base + qq];
          if (e.vnw2) v = (T)((double)v / vs);
          e.out[base + qq] = w;
          pr[0] += (double)v * (double)w;
          pr[1] += (double)w * (double)w;
        }
      }
    }
    const int nblk = gridDim.x * gridDim.y;
    kb_block_partials<2>(pr, e.partials, b, nblk, blockIdx.y * gridDim.x + blockIdx.x);
  }
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
