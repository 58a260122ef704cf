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
// Persistent work split. The units of a pass are (image b, L-tile lt, S row s), linearised as
// u = (b*LT + lt)*S + s. Block k of NB owns [k*U/NB, (k+1)*U/NB) and walks it in chunks of at
// most TS rows that never cross an (image, L-tile) boundary, so every SM gets the same number
// of output rows (+- one chunk remainder) whatever the image size, and the next chunk's input
// tile streams in (cp.async, double buffered) while the current one is multiplied.
// ------------------------------------------------------------------------------------------
struct Chunk {
  int b, lt, s0, cnt;
};

struct ChunkWalk {
  // work items: (image, L-tile, S-part) with `parts` equal S ranges per L-tile; block k owns
  // items [k*I/NB, (k+1)*I/NB) and walks each item's S range in chunks of <= TS rows
  long long it, it_end;
  int S, LT, parts;
  int b = 0, lt = 0, s = 0, s_end = 0;
  __device__ ChunkWalk(int S_, int LT_, int parts_, int batch) : S(S_), LT(LT_), parts(parts_) {
    const long long I = (long long)batch * LT * parts;
    it = I * blockIdx.x / gridDim.x;
    it_end = I * (blockIdx.x + 1) / gridDim.x;
    load();
  }
  __device__ void load() {
    if (it >= it_end) return;
    const long long q = it / parts;
    const int part = (int)(it - q * parts);
    b = (int)(q / LT);
    lt = (int)(q - (long long)b * LT);
    s = (int)((long long)part * S / parts);
    s_end = (int)((long long)(part + 1) * S / parts);
  }
  __device__ bool next(Chunk& c, int TS) {
    while (it < it_end) {
      if (s < s_end) {
        c.b = b;
        c.lt = lt;
        c.s0 = s;
        c.cnt = min(TS, s_end - s);
        s += c.cnt;
        return true;
      }
      ++it;
      load();
    }
    return false;
  }
};

// Host side: items per L-tile and grid size for a persistent pass over S rows x LT L-tiles
// (x batch). Minimises (waves of items) x (rows per item, rounded to m-tiles, + fill overhead).
inline void plan_items(int S, int LT, int batch, int max_blocks, int& parts, int& nb) {
  long long best = -1;
  parts = 1;
  for (int p = 1; p <= S; ++p) {
    const int rows = (S + p - 1) / p;
    if (p > 1 && rows < 16) break;
    const long long items = (long long)batch * LT * p;
    const long long waves = (items + max_blocks - 1) / max_blocks;
    const long long cost = waves * (((rows + 7) / 8) * 8 + 24);
    if (best < 0 || cost < best) {
      best = cost;
      parts = p;
    }
  }
  const long long items = (long long)batch * LT * parts;
  nb = (int)(items < max_blocks ? items : max_blocks);
}

// ------------------------------------------------------------------------------------------
// split pass (fp64, DMMA, persistent): warp w owns S rows [8w, 8w+8) of a chunk x 32 L (four
// n-tiles) for the G terms of a group: 4G accumulator tiles (8G registers).
// ------------------------------------------------------------------------------------------
template <int G>
__device__ __forceinline__ void kb_split_group_dmma(const double* __restrict__ xs,
                                                    const double* __restrict__ cb, int cstride,
                                                    double* __restrict__ ot, const AxisGeom& g,
                                                    int s_off, int lane, int warp,
                                                    double* __restrict__ z, long long z_ps,
                                                    int gstart, const Chunk& ch, double oscale) {
  constexpr int TS = kNW * 8;
  const int ar = lane >> 2, ac = lane & 3;
  double D[G][4][2];
#pragma unroll
  for (int gg = 0; gg < G; ++gg)
#pragma unroll
    for (int j = 0; j < 4; ++j) D[gg][j][0] = D[gg][j][1] = 0.0;
  if (s_off < ch.cnt) {  // warp-uniform: warps past the chunk's rows idle
    const int nch = dmma_chunks(g.Wp);
    const double* xb = xs + (s_off + ac) * kXS + ar;
    const double* ca = cb + kCG + ac - ar;
#pragma unroll 2
    for (int c = 0; c < nch; ++c) {
      double A[G], B[4];
#pragma unroll
      for (int gg = 0; gg < G; ++gg) A[gg] = ca[gg * cstride + 4 * c];
#pragma unroll
      for (int j = 0; j < 4; ++j) B[j] = xb[4 * c * kXS + 8 * j];
#pragma unroll
      for (int gg = 0; gg < G; ++gg)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_884(D[gg][j][0], D[gg][j][1], A[gg], B[j]);
    }
  }
  // one term at a time through the [32][TS+1] transpose stage, then coalesced row stores
  const int l0 = ch.lt * 32;
#pragma unroll
  for (int gg = 0; gg < G; ++gg) {
    if (s_off < ch.cnt) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int i = 0; i < 2; ++i)
          ot[(8 * j + 2 * ac + i) * (TS + 1) + s_off + ar] = D[gg][j][i] * oscale;
    }
    __syncthreads();
    double* zp = z + (long long)(gstart + gg) * z_ps;
    for (int l = warp; l < 32; l += kNW) {
      if (l0 + l >= g.other) break;
      double* zrow = zp + (long long)(l0 + l) * g.len + ch.s0;
      const double* orow = ot + l * (TS + 1);
#pragma unroll
      for (int s = lane; s < TS; s += 32)
        if (s < ch.cnt) zrow[s] = orow[s];
    }
    __syncthreads();
  }
}

template <int GMAX>
__global__ void __launch_bounds__(32 * kNW, 2)
kb_pass_split_dmma(const double* __restrict__ in, long long in_bs, double* __restrict__ z,
                   long long z_ps, long long z_bs, const double* __restrict__ tin, long long t_bs,
                   AxisGeom g, Groups grp, const double* __restrict__ nw2, int r, int batch,
                   int parts) {
  extern __shared__ __align__(16) unsigned char kb_smem_d[];
  constexpr int TS = kNW * 8;
  const int rows_tile = dmma_rows(TS, g.Wp);
  const int cstride = dmma_cstride_split(g.Wp);
  double* xs = reinterpret_cast<double*>(kb_smem_d);  // [2][rows_tile][kXS]
  double* cpad = xs + 2 * rows_tile * kXS;             // [r][cstride], taps at offset kCG
  double* ot = cpad + r * cstride;                     // [32][TS + 1]
  const int lane = threadIdx.x, warp = threadIdx.y;
  const int tid = warp * 32 + lane;
  const int LT = (g.other + 31) / 32;
  ChunkWalk walk(g.len, LT, parts, batch);

  auto fill = [&](const Chunk& c, int buf) {
    kb_fill_tile<double, kXS>(xs + buf * rows_tile * kXS, in + c.b * in_bs, g, g.g0 + c.s0 - g.H,
                              rows_tile, c.lt * 32 + lane, warp, lane, grp.sign[0]);
    cp_async_commit();
  };

  Chunk cur, nxt;
  if (!walk.next(cur, TS)) return;
  fill(cur, 0);
  // batch-uniform taps: all images of a batched operator share the term layout; per-image taps
  // are reloaded when a chunk starts a new image
  int taps_b = -1;
  int buf = 0;
  bool more = true;
  while (more) {
    more = walk.next(nxt, TS);
    if (more) {
      fill(nxt, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    if (cur.b != taps_b) {
      __syncthreads();
      const double* tb = tin + cur.b * t_bs;
      for (int idx = tid; idx < r * cstride; idx += 32 * kNW) {
        const int i = idx / cstride, k = idx - i * cstride - kCG;
        cpad[idx] = (k >= 0 && k < g.Wp) ? tb[(long long)i * g.Wp + k] : 0.0;
      }
      taps_b = cur.b;
    }
    __syncthreads();
    double* xt = xs + buf * rows_tile * kXS;
    const int row_lo = g.g0 + cur.s0 - g.H;
    const bool has_out = g.fill && (row_lo < 0 || row_lo + rows_tile > g.Mg);
    const double oscale = nw2 ? 1.0 / sqrt(nw2[cur.b]) : 1.0;
    double* zb = z + cur.b * z_bs;
    int cur_sign = grp.sign[0];
    for (int gi = 0; gi < grp.n; ++gi) {
      const int gstart = grp.start[gi], gcount = grp.count[gi];
      if (has_out && grp.sign[gi] != cur_sign) {  // flip the folded rows for this group's sign
        for (int rr = warp; rr < rows_tile; rr += kNW) {
          const int gr = row_lo + rr;
          if (gr < 0 || gr >= g.Mg) xt[rr * kXS + lane] = -xt[rr * kXS + lane];
        }
        __syncthreads();
      }
      cur_sign = grp.sign[gi];
      const double* cb = cpad + gstart * cstride;
#define KB_DGROUP(C)                                                                                 \
  case C:                                                                                            \
    if constexpr (C <= GMAX)                                                                         \
      kb_split_group_dmma<C>(xt, cb, cstride, ot, g, warp * 8, lane, warp, zb, z_ps, gstart, cur, oscale); \
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
    cur = nxt;
    buf ^= 1;
  }
}

// ------------------------------------------------------------------------------------------
// sum pass (fp64, DMMA, persistent): warp w owns S rows [16w, 16w+16) (two m-tiles) x 32 L;
// the (chunk, term) tiles stream through two buffers; m-tile 1 reuses the B fragment of chunk
// t0 with the A fragment of t0 - 8. After a chunk's last term the result is transposed through
// the buffer just consumed and the fused epilogue runs on coalesced [m][n] rows.
// ------------------------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(32 * kNW, 2)
kb_pass_sum_dmma(const double* __restrict__ z, long long z_ps, long long z_bs, int r,
                 const double* __restrict__ tin, long long t_bs, AxisGeom g,
                 const double* __restrict__ tsign, Epi<double> e, int batch, int parts) {
  extern __shared__ __align__(16) unsigned char kb_smem_d[];
  constexpr int TS = kNW * 16;
  const int rows_tile = dmma_rows(TS, g.Wp);
  const int cstride = dmma_cstride_sum(g.Wp);  // taps at offset kCG + 8 (m-tile 1 reads t0 - 8)
  double* xs = reinterpret_cast<double*>(kb_smem_d);  // [2][rows_tile][kXS]
  double* cpad = xs + 2 * rows_tile * kXS;             // [2][cstride] (taps of each buffered tile)
  const int lane = threadIdx.x, warp = threadIdx.y;
  const int tid = warp * 32 + lane;
  const int LT = (g.other + 31) / 32;
  ChunkWalk walk(g.len, LT, parts, batch);
  const int ar = lane >> 2, ac = lane & 3;
  const int s_off = warp * 16;
  const int nch = dmma_chunks(g.Wp);

  auto fill = [&](const Chunk& c, int term, int buf) {
    const int sgn = tsign ? (tsign[(long long)c.b * r + term] < 0.0 ? -1 : 1) : 1;
    kb_fill_tile<double, kXS>(xs + buf * rows_tile * kXS, z + c.b * z_bs + (long long)term * z_ps,
                              g, g.g0 + c.s0 - g.H, rows_tile, c.lt * 32 + lane, warp, lane, sgn);
    const double* tb = tin + c.b * t_bs + (long long)term * g.Wp;
    for (int idx = tid; idx < cstride; idx += 32 * kNW) {
      const int k = idx - kCG - 8;
      cpad[buf * cstride + idx] = (k >= 0 && k < g.Wp) ? tb[k] : 0.0;
    }
    cp_async_commit();
  };

  double nrm[3] = {0.0, 0.0, 0.0};
  bool bad = false;
  const int nblk = gridDim.x, blk = blockIdx.x;

  Chunk cur, nxt;
  if (!walk.next(cur, TS)) {
    if (MODE == EPI_UPDATE || MODE == EPI_POWER) kb_sum_finish<double, MODE>(e, nrm, bad, 0, nblk, blk, lane);
    return;
  }
  bool have_next = walk.next(nxt, TS);
  fill(cur, 0, 0);
  int buf = 0, term = 0, norm_b = cur.b;
  double D[2][4][2];
  while (true) {
    __syncthreads();  // the buffer about to be refilled has been consumed by every warp
    // prefetch the next (chunk, term) tile
    const bool last_term = term + 1 == r;
    const bool prefetch = !last_term || have_next;
    if (prefetch) {
      if (!last_term) fill(cur, term + 1, buf ^ 1);
      else fill(nxt, 0, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    if (term == 0) {
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int j = 0; j < 4; ++j) D[mt][j][0] = D[mt][j][1] = 0.0;
    }
    if (s_off < cur.cnt) {  // warp-uniform
      const double* xb = xs + buf * rows_tile * kXS + (s_off + ac) * kXS + ar;
      const double* cb = cpad + buf * cstride + kCG + 8 + ac - ar;
      const bool two = s_off + 8 < cur.cnt;
#pragma unroll 2
      for (int c = 0; c < nch + 2; ++c) {
        double B[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) B[j] = xb[4 * c * kXS + 8 * j];
        const double a0 = cb[4 * c];      // zero beyond the band
        const double a1 = cb[4 * c - 8];  // zero for c < 2 (guard)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          dmma_884(D[0][j][0], D[0][j][1], a0, B[j]);
          if (two) dmma_884(D[1][j][0], D[1][j][1], a1, B[j]);
        }
      }
    }
    if (last_term) {
      __syncthreads();  // everyone is done reading this buffer: reuse it as the transpose stage
      double* ot = xs + buf * rows_tile * kXS;
#pragma unroll
      for (int mt = 0; mt < 2; ++mt)
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int ii = 0; ii < 2; ++ii)
            ot[(8 * j + 2 * ac + ii) * (TS + 1) + s_off + 8 * mt + ar] = D[mt][j][ii];
      __syncthreads();
      if (MODE == EPI_UPDATE || MODE == EPI_POWER) {
        if (cur.b != norm_b) {  // this block's partials of the previous image are complete
          kb_sum_finish<double, MODE>(e, nrm, bad, norm_b, nblk, blk, lane);
          nrm[0] = nrm[1] = nrm[2] = 0.0;
          bad = false;
          norm_b = cur.b;
        }
      }
      kb_sum_epilogue<double, MODE, TS>(ot, g, e, cur.b, cur.s0, min(g.len, cur.s0 + cur.cnt),
                                        cur.lt * 32, warp, lane, nrm, bad);
      __syncthreads();
      if (!have_next) break;
      cur = nxt;
      have_next = walk.next(nxt, TS);
      term = 0;
    } else {
      ++term;
    }
    buf ^= 1;
  }
  if (MODE == EPI_UPDATE || MODE == EPI_POWER) kb_sum_finish<double, MODE>(e, nrm, bad, norm_b, nblk, blk, lane);
}

}  // namespace kb
