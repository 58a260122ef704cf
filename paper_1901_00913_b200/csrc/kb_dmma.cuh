// kb_dmma.cuh — fp64 pass kernels on the FP64 tensor cores (mma.sync m8n8k4 DMMA).
//
// sm_100a has no f64 kind of tcgen05.mma; its FP64 tensor path is the warp-level
// DMMA, measured at 37 TF/s on the box (DFMA: 34 TF/s, tools/microbench.cu). One DMMA is 256
// FMAs and its operands are single registers, so the issue and register budget that limit the
// DFMA loops (kb_taps) mostly disappear.
//
// A banded pass out[s] = sum_k c[k] x[s + k] over an 8-row output block is the product
//     Out(8 x 8 cols) = T(8 x (Wp+7)) * X((Wp+7) x 8 cols),   T[s][t] = c[t - s],
// cut into K-chunks of 4: the A fragment of chunk t0 is the Toeplitz slice c[t0 + col - row]
// (read from a zero-guarded copy of the taps), the B fragment is 4 input rows of the tile.
// The structural overhead is (Wp+7)/Wp (11% at Wp = 64). Fragment layouts (m8n8k4.f64):
//   A: lane holds A[lane/4][lane%4];  B: B[lane%4][lane/4];  C: C[lane/4][2*(lane%4) + i].
#pragma once
#include "kb_kernels.cuh"

namespace kb {

constexpr int kXS = 36;    // tile row stride (doubles): the 16 B-fragment addresses of a
                           // half-warp, rows r0..r0+3 x cols c0..c0+3, hit 16 distinct bank pairs
constexpr int kCG = 8;     // zero guard on each side of the tap copies

__device__ __forceinline__ void dmma_884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// K-chunk count covering t in [0, Wp + 7) for one 8-row output block
__host__ __device__ __forceinline__ int dmma_chunks(int Wp) { return (Wp + 7 + 3) / 4; }

// rows of the input tile the DMMA kernels read for TS outputs
__host__ __device__ __forceinline__ int dmma_rows(int TS, int Wp) { return TS - 8 + 4 * dmma_chunks(Wp); }
// zero-guarded tap copies: every A-fragment index of the chunk loops stays inside
__host__ __device__ __forceinline__ int dmma_cstride_split(int Wp) { return 4 * dmma_chunks(Wp) + 2 * kCG; }
__host__ __device__ __forceinline__ int dmma_cstride_sum(int Wp) { return 4 * dmma_chunks(Wp) + 32; }

// ------------------------------------------------------------------------------------------
// split pass (fp64, DMMA): like kb_pass_split; warp w owns S rows [8w, 8w+8) x 32 L (4 n-tiles)
// and G terms, i.e. 4G accumulator tiles (8G registers).
// ------------------------------------------------------------------------------------------
template <int G>
__device__ __forceinline__ void kb_split_group_dmma(const double* __restrict__ xs,
                                                    const double* __restrict__ cpad, int cstride,
                                                    double* __restrict__ ot, const AxisGeom& g,
                                                    int s_off, int lane, int warp,
                                                    double* __restrict__ z, long long z_ps,
                                                    int gstart, int s0, int l0, double oscale) {
  constexpr int TS = kNW * 8;
  const int ar = lane >> 2, ac = lane & 3;
  double D[G][4][2];
#pragma unroll
  for (int gg = 0; gg < G; ++gg)
#pragma unroll
    for (int j = 0; j < 4; ++j) D[gg][j][0] = D[gg][j][1] = 0.0;
  const int nch = dmma_chunks(g.Wp);
  const double* xb = xs + (s_off + ac) * kXS + ar;
  const double* cb = cpad + kCG + ac - ar;
#pragma unroll 2
  for (int c = 0; c < nch; ++c) {
    double A[G], B[4];
#pragma unroll
    for (int gg = 0; gg < G; ++gg) A[gg] = cb[gg * cstride + 4 * c];
#pragma unroll
    for (int j = 0; j < 4; ++j) B[j] = xb[4 * c * kXS + 8 * j];
#pragma unroll
    for (int gg = 0; gg < G; ++gg)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma_884(D[gg][j][0], D[gg][j][1], A[gg], B[j]);
  }
#pragma unroll
  for (int gg = 0; gg < G; ++gg) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int i = 0; i < 2; ++i) ot[(8 * j + 2 * ac + i) * (TS + 1) + s_off + ar] = D[gg][j][i] * oscale;
    __syncthreads();
    double* zp = z + (long long)(gstart + gg) * z_ps;
    for (int l = warp; l < 32; l += kNW) {
      if (l0 + l >= g.other) break;
      double* zrow = zp + (long long)(l0 + l) * g.len + s0;
#pragma unroll
      for (int s = lane; s < TS; s += 32)
        if (s0 + s < g.len) zrow[s] = ot[l * (TS + 1) + s];
    }
    __syncthreads();
  }
}

template <int GMAX>
__global__ void __launch_bounds__(32 * kNW, 2)
kb_pass_split_dmma(const double* __restrict__ in, long long in_bs, double* __restrict__ z,
                   long long z_ps, long long z_bs, const double* __restrict__ tin, long long t_bs,
                   AxisGeom g, Groups grp, const double* __restrict__ nw2) {
  extern __shared__ __align__(16) unsigned char kb_smem_d[];
  constexpr int TS = kNW * 8;
  const int rows_tile = dmma_rows(TS, g.Wp);
  const int cstride = dmma_cstride_split(g.Wp);
  double* xs = reinterpret_cast<double*>(kb_smem_d);  // [rows_tile][kXS]
  double* cpad = xs + rows_tile * kXS;                 // [GMAX][cstride], taps at offset kCG
  double* ot = cpad + GMAX * cstride;                  // [32][TS + 1]
  const int lane = threadIdx.x, warp = threadIdx.y;
  const int tid = warp * 32 + lane;
  const int b = blockIdx.z;
  const int s0 = blockIdx.y * TS;
  const int l0 = blockIdx.x * 32;
  in += b * in_bs;
  z += b * z_bs;
  tin += b * t_bs;
  const int row_lo = g.g0 + s0 - g.H;
  const bool has_out = g.fill && (row_lo < 0 || row_lo + rows_tile > g.Mg);
  int cur_sign = grp.sign[0];
  kb_fill_tile<double, kXS>(xs, in, g, row_lo, rows_tile, l0 + lane, warp, lane, cur_sign);
  cp_async_commit();
  const double oscale = nw2 ? 1.0 / sqrt(nw2[b]) : 1.0;
  cp_async_wait<0>();

  const int s_off = warp * 8;
  for (int gi = 0; gi < grp.n; ++gi) {
    const int gstart = grp.start[gi], gcount = grp.count[gi];
    __syncthreads();
    if (has_out && grp.sign[gi] != cur_sign) {
      for (int rr = warp; rr < rows_tile; rr += kNW) {
        const int gr = row_lo + rr;
        if (gr < 0 || gr >= g.Mg) xs[rr * kXS + lane] = -xs[rr * kXS + lane];
      }
    }
    cur_sign = grp.sign[gi];
    for (int idx = tid; idx < gcount * cstride; idx += 32 * kNW) {
      const int gg = idx / cstride, k = idx - gg * cstride - kCG;
      cpad[idx] = (k >= 0 && k < g.Wp) ? tin[(long long)(gstart + gg) * g.Wp + k] : 0.0;
    }
    __syncthreads();
#define KB_DGROUP(C)                                                                            \
  case C:                                                                                       \
    if constexpr (C <= GMAX)                                                                    \
      kb_split_group_dmma<C>(xs, cpad, cstride, ot, g, s_off, lane, warp, z, z_ps, gstart, s0, l0, \
                             oscale);                                                           \
    break;
    switch (gcount) {
      KB_DGROUP(1)
      KB_DGROUP(2)
      KB_DGROUP(3)
      KB_DGROUP(4)
      KB_DGROUP(5)
      KB_DGROUP(6)
      default: break;
    }
#undef KB_DGROUP
  }
}

// ------------------------------------------------------------------------------------------
// sum pass (fp64, DMMA): warp w owns S rows [16w, 16w+16) (two m-tiles) x 32 L; term tiles are
// double buffered; m-tile 1 reuses the B fragment of chunk t0 with the A fragment of t0 - 8.
// ------------------------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(32 * kNW, 2)
kb_pass_sum_dmma(const double* __restrict__ z, long long z_ps, long long z_bs, int r,
                 const double* __restrict__ tin, long long t_bs, AxisGeom g,
                 const double* __restrict__ tsign, Epi<double> e) {
  extern __shared__ __align__(16) unsigned char kb_smem_d[];
  constexpr int TS = kNW * 16;
  const int rows_tile = dmma_rows(TS, g.Wp);
  const int cstride = dmma_cstride_sum(g.Wp);  // taps at offset kCG + 8 (m-tile 1 reads t0 - 8)
  double* xs = reinterpret_cast<double*>(kb_smem_d);  // [2][rows_tile][kXS]
  double* cpad = xs + 2 * rows_tile * kXS;             // [2][cstride]
  const int lane = threadIdx.x, warp = threadIdx.y;
  const int tid = warp * 32 + lane;
  const int b = blockIdx.z;
  const int s0 = blockIdx.y * TS;
  const int l0 = blockIdx.x * 32;
  z += b * z_bs;
  tin += b * t_bs;
  const int row_lo = g.g0 + s0 - g.H;

  auto load_term = [&](int i, int stage) {
    const int sgn = tsign ? (tsign[(long long)b * r + i] < 0.0 ? -1 : 1) : 1;
    kb_fill_tile<double, kXS>(xs + stage * rows_tile * kXS, z + (long long)i * z_ps, g, row_lo,
                              rows_tile, l0 + lane, warp, lane, sgn);
    for (int idx = tid; idx < cstride; idx += 32 * kNW) {
      const int k = idx - kCG - 8;
      cpad[stage * cstride + idx] = (k >= 0 && k < g.Wp) ? tin[(long long)i * g.Wp + k] : 0.0;
    }
    cp_async_commit();
  };

  const int ar = lane >> 2, ac = lane & 3;
  double D[2][4][2];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int j = 0; j < 4; ++j) D[mt][j][0] = D[mt][j][1] = 0.0;
  const int s_off = warp * 16;
  const int nch = dmma_chunks(g.Wp);  // per m-tile

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
    const double* xb = xs + st * rows_tile * kXS + (s_off + ac) * kXS + ar;
    const double* cb = cpad + st * cstride + kCG + 8 + ac - ar;
    // chunk c covers tile rows s_off + 4c .. +3: m-tile 0 uses taps 4c + ac - ar, m-tile 1
    // (outputs 8 further down) the taps 8 earlier; both read the same B fragment
#pragma unroll 2
    for (int c = 0; c < nch + 2; ++c) {
      double B[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) B[j] = xb[4 * c * kXS + 8 * j];
      const double a0 = cb[4 * c];       // zero beyond the band
      const double a1 = cb[4 * c - 8];   // zero for c < 2 (guard)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        dmma_884(D[0][j][0], D[0][j][1], a0, B[j]);
        dmma_884(D[1][j][0], D[1][j][1], a1, B[j]);
      }
    }
    __syncthreads();
  }

  // transpose stage: ot[l][s]
  double* ot = xs;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int ii = 0; ii < 2; ++ii) ot[(8 * j + 2 * ac + ii) * (TS + 1) + s_off + 8 * mt + ar] = D[mt][j][ii];
  __syncthreads();
  kb_sum_epilogue<double, MODE, TS>(ot, g, e, b, s0, l0, warp, lane);
}

}  // namespace kb
