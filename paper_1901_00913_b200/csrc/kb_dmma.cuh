// kb_dmma.cuh — fp64 pass kernels on the FP64 tensor cores (mma.sync m8n8k4 DMMA).
//
// sm_100a has no f64 kind of tcgen05.mma; its FP64 tensor path is the warp-level
// DMMA, measured at 37 TF/s on the box (DFMA: 34 TF/s, tools/microbench.cu). One DMMA is 256
// FMAs and its operands are single registers.
//
// A banded pass out[s] = sum_k c[k] x[s + k] over an 8-row output block is the product
//     Out(8 x 8 cols) = T(8 x (Wp+7)) * X((Wp+7) x 8 cols),   T[s][t] = c[t - s],
// cut into K-chunks of 4: the A fragment of chunk t0 is the Toeplitz slice c[t0 + col - row]
// (read from a zero-guarded copy of the taps), the B fragment is 4 input rows of the tile.
// The structural overhead is (Wp+7)/Wp (11% at Wp = 64). Fragment layouts (m8n8k4.f64):
//   A: lane holds A[lane/4][lane%4];  B: B[lane%4][lane/4];  C: C[lane/4][2*(lane%4) + i].
//
// Both kernels are persistent (balanced (image, L-tile, S-part) work items, one block per
// SM slot) and stream their input tiles through a shared-memory ring synchronised with
// mbarriers, not block barriers: every thread issues its share of a tile as cp.async and arms
// the stage's "full" barrier with cp.async.mbarrier.arrive; every warp releases a stage on its
// "empty" barrier once its MMAs have read it. Warps therefore drift within the ring, and one
// warp's epilogue (straight from its accumulators to global memory) overlaps the other warps'
// MMAs. Out-of-domain tile rows are cp.async'd from their folded source row (or zero-filled);
// the (anti)symmetric adjoint's fill sign is applied to the A fragment of those rows, so tiles
// are never rewritten in shared memory.
#pragma once
#include <cuda.h>  // CUtensorMap

#include "kb_kernels.cuh"

namespace kb {

constexpr int kXS = 36;    // tile row stride (doubles): the 16 B-fragment addresses of a
                           // half-warp, rows r0..r0+3 x cols c0..c0+3, hit 16 distinct bank pairs
constexpr int kCG = 8;     // zero guard on each side of the tap copies
constexpr int kStages = 2; // tile ring depth

__device__ __forceinline__ void dmma_884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// ---- mbarrier / cp.async helpers ---------------------------------------------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("{\n.reg .b64 st;\nmbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// arrive on `bar` once every cp.async this thread issued so far has landed
__device__ __forceinline__ void cp_async_arrive(unsigned long long* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// 8-byte cp.async; src_bytes = 0 zero-fills the destination
__device__ __forceinline__ void cp_async_8z(void* smem, const void* gmem, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem)), "l"(gmem),
               "r"(src_bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// TMA: 3-D box of `map` at (c0 = column, c1 = row, c2 = plane) -> shared memory, completion
// counted in bytes on `bar`; out-of-range coordinates are zero-filled by the hardware
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int c0, int c1, int c2,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];\n" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

// TMA tile geometry: a tile of `rows` rows is fetched as nbox boxes of box_rows (<= 256) rows;
// each stage buffer is padded to a 128-byte multiple.
struct TileBoxes {
  int nbox, box_rows, stage_elems;
};
__host__ __device__ __forceinline__ TileBoxes tile_boxes(int rows) {
  TileBoxes t;
  t.nbox = (rows + 255) / 256;
  t.box_rows = (rows + t.nbox - 1) / t.nbox;
  t.stage_elems = ((t.nbox * t.box_rows * 36 + 15) / 16) * 16;
  return t;
}

// Tile row whose data stands in for tile row tr of a reflect-filled pass: rows outside the
// domain read their folded partner inside the tile scaled by `sign` (at a domain edge the TMA
// box contains every partner an in-chunk output needs). A fold leaving the domain or the tile
// keeps the (zero-filled, out-of-range) row itself with weight 0: DMMA multiplies every B row by
// the whole A column, so even zero-weighted rows must hold finite values.
__device__ __forceinline__ int kb_src_row(int tr, int row_lo, int Mg, int rows, int sign, double& mul) {
  const int gr = row_lo + tr;
  mul = 1.0;
  if (gr >= 0 && gr < Mg) return tr;
  const int f = kb_fold(gr, Mg);
  const int u = f - row_lo;
  if (f < 0 || u < 0 || u >= rows) {
    mul = 0.0;
    return tr;
  }
  mul = (double)sign;
  return u;
}

// K-chunk count covering t in [0, Wp + 7) for one 8-row output block
__host__ __device__ __forceinline__ int dmma_chunks(int Wp) { return (Wp + 7 + 3) / 4; }
// rows of the input tile the DMMA kernels read for TS outputs
__host__ __device__ __forceinline__ int dmma_rows(int TS, int Wp) { return TS - 8 + 4 * dmma_chunks(Wp); }
// zero-guarded tap copies: every A-fragment index of the chunk loops stays inside
__host__ __device__ __forceinline__ int dmma_cstride_split(int Wp) { return 4 * dmma_chunks(Wp) + 2 * kCG; }
__host__ __device__ __forceinline__ int dmma_cstride_sum(int Wp) { return 4 * dmma_chunks(Wp) + 32; }

// ------------------------------------------------------------------------------------------
// Persistent work split. Work items are (image b, L-tile lt, S-part) with `parts` equal S
// ranges per L-tile; block k of NB owns items [k*I/NB, (k+1)*I/NB) and walks each item's S
// range in chunks of at most TS rows.
// ------------------------------------------------------------------------------------------
struct Chunk {
  int b, lt, s0, cnt;
};

struct ChunkWalk {
  long long it, it_end;
  int S, LT, parts;
  int b = 0, lt = 0, s = 0, s_end = 0;
  int align;  // part boundaries rounded down to multiples of `align` rows (vector stores)
  __device__ ChunkWalk(int S_, int LT_, int parts_, int batch, int align_ = 1)
      : S(S_), LT(LT_), parts(parts_), align(align_) {
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
    s = (int)((long long)part * S / parts) / align * align;
    s_end = part + 1 == parts ? S : (int)((long long)(part + 1) * S / parts) / align * align;
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
// split pass (fp64, DMMA): warp w owns S rows [8w, 8w+8) of a chunk x 32 L (four n-tiles)
// for the G terms of a group: 4G accumulator tiles (8G registers). Results go straight from the
// accumulators to Z_i^T (8 consecutive S values = 64 B per output row and store).
// ------------------------------------------------------------------------------------------
// MMA loop of one group: EDGE tiles (reflect-filled pass at a domain edge) read folded rows.
template <int G, bool EDGE>
__device__ __forceinline__ void kb_split_mma(double (&D)[G][4][2], const double* __restrict__ xs,
                                             const double* __restrict__ ca, int cstride, int nch,
                                             int s_off, int ar, int ac, int row_lo, int Mg,
                                             int rows, int sign) {
  const double* xb = xs + (s_off + ac) * kXS + ar;
#pragma unroll 2
  for (int c = 0; c < nch; ++c) {
    double A[G], B[4];
    double mul = 1.0;
    const double* xr = xb + 4 * c * kXS;
    if constexpr (EDGE) xr = xs + kb_src_row(s_off + 4 * c + ac, row_lo, Mg, rows, sign, mul) * kXS + ar;
#pragma unroll
    for (int gg = 0; gg < G; ++gg) A[gg] = EDGE ? ca[gg * cstride + 4 * c] * mul : ca[gg * cstride + 4 * c];
#pragma unroll
    for (int j = 0; j < 4; ++j) B[j] = xr[8 * j];
#pragma unroll
    for (int gg = 0; gg < G; ++gg)
#pragma unroll
      for (int j = 0; j < 4; ++j) dmma_884(D[gg][j][0], D[gg][j][1], A[gg], B[j]);
  }
}

template <int G>
__device__ __forceinline__ void kb_split_group_dmma(const double* __restrict__ xs,
                                                    const double* __restrict__ cb, int cstride,
                                                    const AxisGeom& g, int s_off, int lane,
                                                    double* __restrict__ z, long long z_ps,
                                                    int gstart, const Chunk& ch, double oscale,
                                                    bool scaled, int row_lo, bool edge, int sign) {
  const int ar = lane >> 2, ac = lane & 3;
  double D[G][4][2];
#pragma unroll
  for (int gg = 0; gg < G; ++gg)
#pragma unroll
    for (int j = 0; j < 4; ++j) D[gg][j][0] = D[gg][j][1] = 0.0;
  const int nch = (g.dbg & 1) ? 0 : dmma_chunks(g.Wp);
  const double* ca = cb + kCG + ac - ar;
  const int rows = dmma_rows(kNW * 8, g.Wp);
  if (edge) kb_split_mma<G, true>(D, xs, ca, cstride, nch, s_off, ar, ac, row_lo, g.Mg, rows, sign);
  else kb_split_mma<G, false>(D, xs, ca, cstride, nch, s_off, ar, ac, row_lo, g.Mg, rows, sign);
  const int s = s_off + ar;
  if (s >= ch.cnt || (g.dbg & 2)) return;
  const int l0 = ch.lt * 32;
#pragma unroll
  for (int gg = 0; gg < G; ++gg) {
    double* zp = z + (long long)(gstart + gg) * z_ps + ch.s0 + s;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int l = l0 + 8 * j + 2 * ac + i;
        if (l < g.other) zp[(long long)l * g.len] = scaled ? D[gg][j][i] * oscale : D[gg][j][i];
      }
  }
}

template <int GMAX>
__global__ void __launch_bounds__(32 * kNW, 2)
kb_pass_split_dmma(const __grid_constant__ CUtensorMap tmap, double* __restrict__ z,
                   long long z_ps, long long z_bs, const double* __restrict__ tin, long long t_bs,
                   AxisGeom g, Groups grp, const double* __restrict__ nw2, int r, int batch,
                   int parts) {
  extern __shared__ __align__(128) unsigned char kb_smem_d[];
  __shared__ unsigned long long full[kStages], empty[kStages];
  constexpr int TS = kNW * 8;
  const int rows_tile = dmma_rows(TS, g.Wp);
  const TileBoxes tb = tile_boxes(rows_tile);
  const int cstride = dmma_cstride_split(g.Wp);
  double* xs = reinterpret_cast<double*>(kb_smem_d);  // [kStages][stage_elems]
  double* cpad = xs + kStages * tb.stage_elems;        // [r][cstride], taps at offset kCG
  const int lane = threadIdx.x, warp = threadIdx.y;
  const int tid = warp * 32 + lane;
  const int LT = (g.other + 31) / 32;
  const int s_off = warp * 8;

  if (tid == 0) {
    for (int st = 0; st < kStages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kNW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // thread 0 walks this block's chunk list ahead of the consumers and issues one TMA box per
  // (<= 256-row) part of each tile; the map covers the local plane including its halo rows
  ChunkWalk fill_walk(g.len, LT, parts, batch), use_walk(g.len, LT, parts, batch);
  Chunk fc, ch;
  int nfill = 0;
  auto issue = [&]() {
    if (tid != 0 || !fill_walk.next(fc, TS)) return;
    const int st = nfill % kStages;
    if (nfill >= kStages) mbar_wait(&empty[st], ((nfill / kStages) - 1) & 1);
    mbar_arrive_expect_tx(&full[st], (unsigned)(tb.nbox * tb.box_rows * 36 * sizeof(double)));
    const int row0 = fc.s0 - g.H + g.halo_lo;  // map row of tile row 0
    for (int k = 0; k < tb.nbox; ++k)
      tma_load_3d(xs + st * tb.stage_elems + k * tb.box_rows * kXS, &tmap, fc.lt * 32,
                  row0 + k * tb.box_rows, fc.b, &full[st]);
    ++nfill;
  };
  for (int k = 0; k < kStages - 1; ++k) issue();

  int taps_b = -1;
  for (int t = 0; use_walk.next(ch, TS); ++t) {
    if (ch.b != taps_b) {  // per-image taps (uniform across the block: block-level reload)
      __syncthreads();
      const double* tbp = tin + ch.b * t_bs;
      for (int idx = tid; idx < r * cstride; idx += 32 * kNW) {
        const int i = idx / cstride, k = idx - i * cstride - kCG;
        cpad[idx] = (k >= 0 && k < g.Wp) ? tbp[(long long)i * g.Wp + k] : 0.0;
      }
      __syncthreads();
      taps_b = ch.b;
    }
    issue();  // keep kStages-1 tiles in flight ahead of the one consumed now
    const int st = t % kStages;
    mbar_wait(&full[st], (t / kStages) & 1);
    const double* xt = xs + st * tb.stage_elems;
    const int row_lo = g.g0 + ch.s0 - g.H;
    const bool edge = g.fill && (row_lo < 0 || row_lo + rows_tile > g.Mg);
    const double oscale = nw2 ? 1.0 / sqrt(nw2[ch.b]) : 1.0;
    double* zb = z + ch.b * z_bs;
    if (s_off < ch.cnt) {  // warp-uniform: warps past the chunk's rows idle
      for (int gi = 0; gi < grp.n; ++gi) {
        const int gstart = grp.start[gi];
        const double* cb = cpad + gstart * cstride;
#define KB_DGROUP(C)                                                                                  \
  case C:                                                                                             \
    if constexpr (C <= GMAX)                                                                          \
      kb_split_group_dmma<C>(xt, cb, cstride, g, s_off, lane, zb, z_ps, gstart, ch, oscale,           \
                             nw2 != nullptr, row_lo, edge, grp.sign[gi]);                             \
    break;
        switch (grp.count[gi]) {
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
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
}

// ------------------------------------------------------------------------------------------
// Fused epilogue straight from the sum pass accumulators: lane (ar, ac) of warp s_off holds
// output S = s0+s_off+8mt+ar (n index) for L = l0+8j+2ac+i (m index), i.e. per store 8
// consecutive n values (64 B) of 4 image rows. One m-tile at a time, operand loads first.
// ------------------------------------------------------------------------------------------
template <int MODE>
__device__ __forceinline__ void kb_sum_epilogue_regs(const double (&D)[2][4][2], const AxisGeom& g,
                                                     const Epi<double>& e, const Chunk& ch,
                                                     int s_off, int ar, int ac, double (&nrm)[3],
                                                     bool& bad) {
  const int n = g.len;
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
    const int sl = s_off + 8 * mt + ar;  // row within the chunk
    const int q = ch.s0 + sl;            // n index
    if (sl >= ch.cnt || q >= n) continue;
    const long long rowbase = (long long)ch.b * e.bstride + q;
    double u[4][2], w[4][2];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int p = ch.lt * 32 + 8 * j + 2 * ac + i;
        const long long at = rowbase + (long long)p * n;
        const bool ok = p < g.other;
        if constexpr (MODE == EPI_RESID) u[j][i] = ok ? e.bsub[at] : 0.0;
        if constexpr (MODE == EPI_UPDATE) {
          u[j][i] = ok ? e.y[at] : 0.0;
          w[j][i] = ok ? e.x[at] : 0.0;
        }
        if constexpr (MODE == EPI_POWER) u[j][i] = ok ? e.vin[at] : 0.0;
      }
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int p = ch.lt * 32 + 8 * j + 2 * ac + i;
        if (p >= g.other) continue;
        const long long at = rowbase + (long long)p * n;
        double val = D[mt][j][i];
        if (e.foldH > 0) {
          const int FH = e.foldH;
          const double* f = e.fold + ((long long)ch.b * g.other + p) * (2 * FH);
          if (q < FH) val += f[q];
          else if (q >= n - FH) val += f[q - (n - 2 * FH)];
        }
        if constexpr (MODE == EPI_PLAIN) {
          e.out[at] = val;
        } else if constexpr (MODE == EPI_RESID) {
          e.out[at] = __dsub_rn(val, u[j][i]);
        } else if constexpr (MODE == EPI_UPDATE) {
          double xv = __ddiv_rn(__dsub_rn(__dmul_rn(e.L[ch.b], u[j][i]), val), e.denom[ch.b]);
          if (e.project) xv = (xv > 0.0 || xv != xv) ? xv : 0.0;
          const double d = __dsub_rn(xv, w[j][i]);
          e.x[at] = xv;
          e.y[at] = __dadd_rn(xv, __dmul_rn(e.beta, d));
          bad |= !isfinite(xv);
          if (e.want_norms) {
            nrm[0] += d * d;
            nrm[1] += w[j][i] * w[j][i];
            nrm[2] += xv * xv;
          }
        } else {  // EPI_POWER
          const double vv = e.vnw2 ? u[j][i] / sqrt(e.vnw2[ch.b]) : u[j][i];
          e.out[at] = val;
          nrm[0] += vv * val;
          nrm[1] += val * val;
        }
      }
  }
}

// per-warp end of an image's epilogues: non-finite flag and this warp's norm partials
template <int MODE>
__device__ __forceinline__ void kb_warp_finish(const Epi<double>& e, double (&nrm)[3], bool bad,
                                               int b, int nslots, int slot, int lane) {
  if constexpr (MODE == EPI_UPDATE) {
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicMin(e.nonfinite, e.k);
  }
  if constexpr (MODE == EPI_UPDATE || MODE == EPI_POWER) {
    if (MODE == EPI_POWER || e.want_norms) {
#pragma unroll
      for (int qq = 0; qq < 3; ++qq) {
        double v = nrm[qq];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) e.partials[((long long)b * nslots + slot) * 4 + qq] = v;
      }
    }
  }
}

// MMA loop of one (chunk, term) tile of the sum pass (two m-tiles sharing the B fragment).
template <bool EDGE>
__device__ __forceinline__ void kb_sum_mma(double (&D)[2][4][2], const double* __restrict__ xs,
                                           const double* __restrict__ cb, int nchr, int s_off,
                                           int ar, int ac, int row_lo, int Mg, int rows, int sign,
                                           bool two) {
  const double* xb = xs + (s_off + ac) * kXS + ar;
#pragma unroll 2
  for (int c = 0; c < nchr; ++c) {
    double mul = 1.0;
    const double* xr = xb + 4 * c * kXS;
    if constexpr (EDGE) xr = xs + kb_src_row(s_off + 4 * c + ac, row_lo, Mg, rows, sign, mul) * kXS + ar;
    double B[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) B[j] = xr[8 * j];
    double a0 = cb[4 * c];      // zero beyond the band
    double a1 = cb[4 * c - 8];  // zero for c < 2 (guard)
    if constexpr (EDGE) {
      a0 *= mul;
      a1 *= mul;
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      dmma_884(D[0][j][0], D[0][j][1], a0, B[j]);
      if (two) dmma_884(D[1][j][0], D[1][j][1], a1, B[j]);
    }
  }
}

// ------------------------------------------------------------------------------------------
// sum pass (fp64, DMMA): warp w owns S rows [16w, 16w+16) (two m-tiles) x 32 L of a chunk;
// the (chunk, term) tiles stream through the mbarrier ring; m-tile 1 reuses the B fragment of
// chunk t0 with the A fragment of t0 - 8. After a chunk's last term each warp runs the fused
// epilogue from its registers. Norm partials are per warp: partials[b][block*kNW + warp].
// ------------------------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(32 * kNW, 2)
kb_pass_sum_dmma(const __grid_constant__ CUtensorMap tmap, int r, const double* __restrict__ tin,
                 long long t_bs, AxisGeom g, const double* __restrict__ tsign, Epi<double> e,
                 int batch, int parts) {
  extern __shared__ __align__(128) unsigned char kb_smem_d[];
  __shared__ unsigned long long full[kStages], empty[kStages];
  constexpr int TS = kNW * 16;
  const int rows_tile = dmma_rows(TS, g.Wp);
  const TileBoxes tb = tile_boxes(rows_tile);
  const int cstride = dmma_cstride_sum(g.Wp);  // taps at offset kCG + 8 (m-tile 1 reads t0 - 8)
  double* xs = reinterpret_cast<double*>(kb_smem_d);  // [kStages][stage_elems]
  double* cpad = xs + kStages * tb.stage_elems;        // [r][cstride]
  const int lane = threadIdx.x, warp = threadIdx.y;
  const int tid = warp * 32 + lane;
  const int LT = (g.other + 31) / 32;
  const int ar = lane >> 2, ac = lane & 3;
  const int s_off = warp * 16;
  const int nch = dmma_chunks(g.Wp);
  const int nslots = gridDim.x * kNW, slot = blockIdx.x * kNW + warp;

  if (tid == 0) {
    for (int st = 0; st < kStages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kNW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  // tile sequence: (chunk, term) for every chunk of this block; thread 0 issues the TMA boxes
  ChunkWalk fill_walk(g.len, LT, parts, batch), use_walk(g.len, LT, parts, batch);
  Chunk fc;
  int fterm = r;  // forces fetching the first chunk
  bool fmore = true;
  int nfill = 0;
  auto issue = [&]() {
    if (tid != 0 || !fmore) return;
    if (fterm == r) {
      if (!fill_walk.next(fc, TS)) {
        fmore = false;
        return;
      }
      fterm = 0;
    }
    const int st = nfill % kStages;
    if (nfill >= kStages) mbar_wait(&empty[st], ((nfill / kStages) - 1) & 1);
    mbar_arrive_expect_tx(&full[st], (unsigned)(tb.nbox * tb.box_rows * 36 * sizeof(double)));
    const int row0 = fc.s0 - g.H;  // Z^T planes are not row sharded
    for (int k = 0; k < tb.nbox; ++k)
      tma_load_3d(xs + st * tb.stage_elems + k * tb.box_rows * kXS, &tmap, fc.lt * 32,
                  row0 + k * tb.box_rows, fc.b * r + fterm, &full[st]);
    ++fterm;
    ++nfill;
  };
  for (int k = 0; k < kStages - 1; ++k) issue();

  double nrm[3] = {0.0, 0.0, 0.0};
  bool bad = false;
  int norm_b = -1, taps_b = -1;
  double D[2][4][2];
  Chunk ch;
  int t = 0;
  while (use_walk.next(ch, TS)) {
    if (ch.b != taps_b) {  // per-image taps (uniform across the block)
      __syncthreads();
      const double* tb = tin + ch.b * t_bs;
      for (int idx = tid; idx < r * cstride; idx += 32 * kNW) {
        const int i = idx / cstride, k = idx - i * cstride - kCG - 8;
        cpad[idx] = (k >= 0 && k < g.Wp) ? tb[(long long)i * g.Wp + k] : 0.0;
      }
      __syncthreads();
      taps_b = ch.b;
    }
    if (ch.b != norm_b) {
      if (norm_b >= 0) kb_warp_finish<MODE>(e, nrm, bad, norm_b, nslots, slot, lane);
      nrm[0] = nrm[1] = nrm[2] = 0.0;
      bad = false;
      norm_b = ch.b;
    }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int j = 0; j < 4; ++j) D[mt][j][0] = D[mt][j][1] = 0.0;
    const int row_lo = g.g0 + ch.s0 - g.H;
    const bool edge = g.fill && (row_lo < 0 || row_lo + rows_tile > g.Mg);
    const bool active = s_off < ch.cnt;  // warp-uniform
    const bool two = s_off + 8 < ch.cnt;
    for (int term = 0; term < r; ++term, ++t) {
      issue();
      const int st = t % kStages;
      mbar_wait(&full[st], (t / kStages) & 1);
      if (active) {
        const double* xt = xs + st * tb.stage_elems;
        const double* cb = cpad + term * cstride + kCG + 8 + ac - ar;
        const int sgn = (tsign && tsign[(long long)ch.b * r + term] < 0.0) ? -1 : 1;
        const int nchr = (g.dbg & 1) ? 0 : nch + 2;
        if (edge) kb_sum_mma<true>(D, xt, cb, nchr, s_off, ar, ac, row_lo, g.Mg, rows_tile, sgn, two);
        else kb_sum_mma<false>(D, xt, cb, nchr, s_off, ar, ac, row_lo, g.Mg, rows_tile, sgn, two);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    if (active && !(g.dbg & 2)) kb_sum_epilogue_regs<MODE>(D, g, e, ch, s_off, ar, ac, nrm, bad);
  }
  if (norm_b >= 0) kb_warp_finish<MODE>(e, nrm, bad, norm_b, nslots, slot, lane);
}

}  // namespace kb
