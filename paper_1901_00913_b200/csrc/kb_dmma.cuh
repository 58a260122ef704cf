// kb_dmma.cuh — fp64 pass kernels on the FP64 tensor cores (mma.sync m8n8k4 DMMA).
//
// sm_100a has no f64 kind of tcgen05.mma; its FP64 tensor path is the warp-level
// DMMA, measured at 37 TF/s on the box (DFMA: 34 TF/s, tools/microbench.cu). One DMMA is 256
// FMAs and its operands are single registers.
//
// A banded pass out[s] = sum_k c[k] x[s + k] for 8 consecutive outputs s and 8 columns l is
//     Out^T(8 l x 8 s) = X^T(8 l x (Wp+7)) * T((Wp+7) x 8 s),   T[t][s] = c[t - s],
// cut into K-chunks of 4: the A fragment is 4 input rows of the shared-memory tile read
// transposed, the B fragment the Toeplitz slice c[t0 + row - col] of a zero-guarded tap copy.
// The accumulator then holds, per lane, two consecutive outputs s of one column l, which is
// the layout of the transposed outputs (Z_i^T[l][s], Y[m][n]): results leave as 16-byte
// vectors. Structural overhead (Wp+7)/Wp (11% at Wp = 64). Fragment layouts (m8n8k4.f64):
//   A: lane holds A[lane/4][lane%4];  B: B[lane%4][lane/4];  C: C[lane/4][2*(lane%4) + i].
//
// Both kernels are persistent (balanced (image, L-tile, S-part) work items, one block per
// SM slot). Thread 0 streams the input tiles by TMA (cp.async.bulk.tensor) into a ring of
// shared-memory stages guarded by mbarriers ("full": transaction bytes landed, "empty": every
// warp has read the stage). Warps synchronise only through the ring. For a reflect-filled pass
// the out-of-domain rows of a tile at a domain edge are rewritten in shared memory from their
// folded partner row (times the (anti)symmetric adjoint's sign) before the MMAs; edge tiles
// are block-uniform and rare, interior tiles are used exactly as TMA delivered them.
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
// Profiling timeline (KB_DEBUG_MODE bit 7 in a -DKB_TRACE=1 build): thread 0 of block b stamps
// %globaltimer into kb_trace[kind][b][slot] (kind 0 split, 1 sum; read back with kb_debug_trace).
#ifndef KB_DMMA_EARLY_SCALARS
#define KB_DMMA_EARLY_SCALARS 1
#endif
#ifndef KB_TRACE
#define KB_TRACE 0
#endif
constexpr int kTraceBlocks = 1024;
__device__ unsigned long long kb_trace[2][kTraceBlocks][8];
__device__ __forceinline__ void kb_stamp(const AxisGeom& g, int kind, int slot) {
  if (KB_TRACE && (g.dbg & 128) && threadIdx.x == 0 && threadIdx.y == 0 && blockIdx.x < kTraceBlocks) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    kb_trace[kind][blockIdx.x][slot] = t;
    if (slot == 0) {
      unsigned smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      kb_trace[kind][blockIdx.x][7] = smid;
    }
  }
}
// Programmatic dependent launch (no-ops without the launch attribute): let the next kernel of
// the stream start its prologue on SMs this grid frees; wait until the previous kernel's results
// are visible before touching anything it wrote.
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
// order this thread's generic-proxy shared-memory writes before later async-proxy (TMA) access
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
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
  int it, it_end;  // 32-bit: item counts and S * parts stay far below 2^31 for any plane
  int S, LT, parts, eparts, align;
  int b = 0, lt = 0, s = 0, s_end = 0;
  // eparts: S-parts of the two edge L-tiles (0 and LT-1), which may carry extra work
  __device__ ChunkWalk(int S_, int LT_, int parts_, int batch, int align_ = 1, int eparts_ = 0)
      : S(S_), LT(LT_), parts(parts_), eparts(eparts_ > 0 ? eparts_ : parts_), align(align_) {
    const unsigned I = (unsigned)(batch * per_image());
    it = (int)(I * blockIdx.x / gridDim.x);
    it_end = (int)(I * (blockIdx.x + 1) / gridDim.x);
    load();
  }
  __device__ int per_image() const { return LT >= 2 ? (LT - 2) * parts + 2 * eparts : eparts; }
  __device__ void load() {
    if (it >= it_end) return;
    const int pi = per_image();
    b = it / pi;
    int i = it - b * pi, np;
    if (i < eparts) {
      lt = 0;
      np = eparts;
    } else if (LT >= 2 && i >= eparts + (LT - 2) * parts) {
      lt = LT - 1;
      i -= eparts + (LT - 2) * parts;
      np = eparts;
    } else {
      i -= eparts;
      lt = 1 + i / parts;
      i -= (lt - 1) * parts;
      np = parts;
    }
    s = (int)((unsigned)i * (unsigned)S / (unsigned)np) / align * align;
    s_end = i + 1 == np ? S : (int)((unsigned)(i + 1) * (unsigned)S / (unsigned)np) / align * align;
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
inline void plan_items(int S, int LT, int batch, int max_blocks, int& parts, int& nb, int* eparts = nullptr) {
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
  long long items = (long long)batch * LT * parts;
  if (eparts) {  // one more S-part on each edge L-tile when that still fits the same wave
    *eparts = parts;
    const long long more = (long long)batch * (LT >= 2 ? 2 : 1);
    const long long waves = (items + max_blocks - 1) / max_blocks;
    if (parts < S / 16 && items + more <= waves * max_blocks) {
      *eparts = parts + 1;
      items += more;
    }
  }
  nb = (int)(items < max_blocks ? items : max_blocks);
}

// Rewrite the out-of-domain rows of a landed [rows][kXS] tile: sign * folded partner row, or
// zero when the single fold leaves the domain or the tile (block-level, edge tiles only). Only
// the out-of-domain rows are visited, all threads at once, four independent elements per
// thread in flight (partner rows are in-domain, so reads never see this pass's writes).
__device__ __forceinline__ void kb_fold_tile_d(double* __restrict__ xs, int rows, int row_lo, int Mg,
                                               int sign, int tid) {
  const int top = min(max(-row_lo, 0), rows);        // tile rows [0, top) precede the domain
  const int bot = max(min(Mg - row_lo, rows), top);  // tile rows [bot, rows) follow it
  const int nel = (top + rows - bot) * 32;
  for (int i0 = 0; i0 < nel; i0 += 4 * 32 * kNW) {
    double v[4];
    int dst[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int idx = i0 + k * 32 * kNW + tid;
      dst[k] = -1;
      v[k] = 0.0;
      if (idx < nel) {
        const int q = idx >> 5, col = idx & 31;
        const int rr = q < top ? q : bot + (q - top);
        const int f = kb_fold(row_lo + rr, Mg);
        const int u = f - row_lo;
        if (f >= 0 && u >= 0 && u < rows) v[k] = xs[u * kXS + col];
        dst[k] = rr * kXS + col;
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (dst[k] >= 0) xs[dst[k]] = sign < 0 ? -v[k] : v[k];
  }
}
__device__ __forceinline__ void kb_flip_tile_d(double* __restrict__ xs, int rows, int row_lo, int Mg,
                                               int tid) {
  const int top = min(max(-row_lo, 0), rows);
  const int bot = max(min(Mg - row_lo, rows), top);
  const int nel = (top + rows - bot) * 32;
  for (int idx = tid; idx < nel; idx += 32 * kNW) {
    const int q = idx >> 5, col = idx & 31;
    const int rr = q < top ? q : bot + (q - top);
    xs[rr * kXS + col] = -xs[rr * kXS + col];
  }
}

// a / d correctly rounded for normal results, given rd = RN(1/d): q = RN(a*rd) is within an ulp
// and one exact-remainder correction RN(q + (a - d*q)*rd) rounds correctly (Markstein). Three
// FP64 operations instead of a full division per element, whose dependent Newton chain stalls
// behind the DMMAs of the other warps on the shared FP64 pipe.
__device__ __forceinline__ double kb_quot(double a, double d, double rd) {
  const double q = __dmul_rn(a, rd);
  const double rem = fma(-d, q, a);
  return fma(rem, rd, q);
}

// Per-image taps (global [r][Wp], Wp a multiple of 16) -> shared [r][cstride]: the first Kw taps
// of each row after `guard` zeros, zeros after them. The taps move as 16-byte vectors, all loads
// of a thread issued before any store: one memory round trip at kernel start.
__device__ __forceinline__ void kb_load_taps_d(double* __restrict__ cpad, const double* __restrict__ tb, int r,
                                               int Wp, int Kw, int cstride, int guard, int tid) {
  const int n2 = r * Wp / 2, nw = Wp / 2;
  constexpr int kV = 4;
  for (int j0 = 0; j0 < n2; j0 += kV * 32 * kNW) {
    double2 v[kV];
#pragma unroll
    for (int u = 0; u < kV; ++u) {
      const int j = j0 + u * 32 * kNW + tid;
      if (j < n2) v[u] = reinterpret_cast<const double2*>(tb)[j];
    }
#pragma unroll
    for (int u = 0; u < kV; ++u) {
      const int j = j0 + u * 32 * kNW + tid;
      if (j < n2) {
        const int i = j / nw, k = 2 * (j - i * nw);
        if (k < Kw) cpad[i * cstride + guard + k] = v[u].x;
        if (k + 1 < Kw) cpad[i * cstride + guard + k + 1] = v[u].y;
      }
    }
  }
  const int ng = cstride - Kw;  // guard entries per row
  for (int idx = tid; idx < r * ng; idx += 32 * kNW) {
    const int i = idx / ng, k = idx - i * ng;
    cpad[i * cstride + (k < guard ? k : Kw + k)] = 0.0;
  }
}

__device__ __forceinline__ void st_pair(double* p, double a, double b, bool both) {
  if (both) *reinterpret_cast<double2*>(p) = make_double2(a, b);
  else *p = a;
}

// ------------------------------------------------------------------------------------------
// split pass (fp64, DMMA): warp w owns S rows [8w, 8w+8) of a chunk x 32 L (four 8-column
// M-tiles) for the G terms of a group: 4G accumulator tiles. Lane (ar, ac) of M-tile j ends
// with Z^T[l0 + 8j + ar][s0 + 8w + 2ac + {0,1}]: one 16-byte store per term and M-tile.
// ------------------------------------------------------------------------------------------
// MMA loop of one group over K-chunks [c0, c1): S-tile 0 when T0, S-tile 1 (outputs +8: taps at
// t0 - 8, sharing the A fragment) when T1
template <int G, int NS, bool T0, bool T1>
__device__ __forceinline__ void kb_split_mma(double (&D)[G][NS][4][2], const double* __restrict__ xb,
                                             const double* __restrict__ cbl, int cstride, int c0, int c1) {
#pragma unroll 2
  for (int c = c0; c < c1; ++c) {
    double A[4], B0[G], B1[G];
#pragma unroll
    for (int j = 0; j < 4; ++j) A[j] = xb[4 * c * kXS + 8 * j];
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
      B0[gg] = T0 ? cbl[gg * cstride + 4 * c] : 0.0;
      B1[gg] = T1 ? cbl[gg * cstride + 4 * c - 8] : 0.0;
    }
#pragma unroll
    for (int gg = 0; gg < G; ++gg)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (T0) dmma_884(D[gg][0][j][0], D[gg][0][j][1], A[j], B0[gg]);
        if constexpr (NS == 2)
          if (T1) dmma_884(D[gg][NS - 1][j][0], D[gg][NS - 1][j][1], A[j], B1[gg]);
      }
  }
}

// ------------------------------------------------------------------------------------------
// split pass (fp64, DMMA): warp w owns NS S-tiles of 8 rows ([8 NS w, 8 NS (w+1)) of a chunk) x
// 32 L (four 8-column M-tiles) for the G terms of a group; with NS = 2 the two S-tiles share
// every A fragment (the sum pass's trick). Lane (ar, ac) of M-tile j ends with
// Z^T[l0 + 8j + ar][s0 + s_off + 8mt + 2ac + {0,1}]: one 16-byte store per term, S-tile and
// M-tile (plus the reflected halo rows at an L edge).
// ------------------------------------------------------------------------------------------
template <int G, int NS>
__device__ __forceinline__ void kb_split_group_dmma(const double* __restrict__ xs,
                                                    const double* __restrict__ cb, int cstride,
                                                    const AxisGeom& g, int s_off, int lane,
                                                    double* __restrict__ z, long long z_ps,
                                                    int gstart, const Chunk& ch, double oscale,
                                                    bool scaled, int mirror_h,
                                                    const double* __restrict__ msign) {
  const int ar = lane >> 2, ac = lane & 3;
  double D[G][NS][4][2];
#pragma unroll
  for (int gg = 0; gg < G; ++gg)
#pragma unroll
    for (int mt = 0; mt < NS; ++mt)
#pragma unroll
      for (int j = 0; j < 4; ++j) D[gg][mt][j][0] = D[gg][mt][j][1] = 0.0;
  const int nch = (g.dbg & 1) ? 0 : dmma_chunks(g.Kw);
  const double* cbl = cb + (NS == 2 ? kCG + 8 : kCG) + ac - ar;
  const double* xb = xs + (s_off + ac) * kXS + ar;
  if constexpr (NS == 1) {
    kb_split_mma<G, NS, true, false>(D, xb, cbl, cstride, 0, nch);
  } else if (s_off + 8 < ch.cnt) {
    kb_split_mma<G, NS, true, false>(D, xb, cbl, cstride, 0, 2);
    kb_split_mma<G, NS, true, true>(D, xb, cbl, cstride, 2, nch);
    kb_split_mma<G, NS, false, true>(D, xb, cbl, cstride, nch, nch + 2);
  } else {
    kb_split_mma<G, NS, true, false>(D, xb, cbl, cstride, 0, nch);
  }
  if (g.dbg & 2) return;
  const int l0 = ch.lt * 32 + ar;
#pragma unroll
  for (int mt = 0; mt < NS; ++mt) {
    const int s = s_off + 8 * mt + 2 * ac;
    if (s >= ch.cnt) continue;
    const bool both = s + 1 < ch.cnt;
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
      double* zp = z + (long long)(gstart + gg) * z_ps + ch.s0 + s;
      const double sg = msign ? msign[gstart + gg] : 1.0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int l = l0 + 8 * j;
        if (l >= g.other) continue;
        const double v0 = scaled ? D[gg][mt][j][0] * oscale : D[gg][mt][j][0];
        const double v1 = scaled ? D[gg][mt][j][1] * oscale : D[gg][mt][j][1];
        st_pair(zp + (long long)l * g.len, v0, v1, both);
        if (mirror_h > 0 && !(g.dbg & 32)) {  // reflected halo rows of Z^T for the reflect-filled sum pass
          if (l < mirror_h) st_pair(zp + (long long)(-1 - l) * g.len, sg * v0, sg * v1, both);
          if (l >= g.other - mirror_h)
            st_pair(zp + (long long)(2 * g.other - 1 - l) * g.len, sg * v0, sg * v1, both);
        }
      }
    }
  }
}

template <int GMAX, int NS>
__global__ void __launch_bounds__(32 * kNW, 2)
kb_pass_split_dmma(const __grid_constant__ CUtensorMap tmap, double* __restrict__ z,
                   long long z_ps, long long z_bs, const double* __restrict__ tin, long long t_bs,
                   AxisGeom g, Groups grp, const double* __restrict__ nw2, int r, int batch, int parts,
                   int eparts, int mirror_h, const double* __restrict__ msign) {
  extern __shared__ __align__(128) unsigned char kb_smem_d[];
  kb_stamp(g, 0, 0);
  __shared__ unsigned long long full[kStages], empty[kStages];
  constexpr int TS = kNW * 8 * NS;
  const int rows_tile = dmma_rows(TS, g.Kw);
  const TileBoxes tb = tile_boxes(rows_tile);
  const int cstride = NS == 2 ? dmma_cstride_sum(g.Kw) : dmma_cstride_split(g.Kw);
  const int tguard = NS == 2 ? kCG + 8 : kCG;         // S-tile 1 reads taps at t0 - 8
  double* xs = reinterpret_cast<double*>(kb_smem_d);  // [kStages][stage_elems]
  double* cpad = xs + kStages * tb.stage_elems;        // [r][cstride], taps at offset tguard
  const int lane = threadIdx.x, warp = threadIdx.y;
  const int tid = warp * 32 + lane;
  const int LT = (g.other + 31) / 32;
  const int s_off = warp * 8 * NS;

  if (tid == 0) {
    for (int st = 0; st < kStages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kNW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  kb_stamp(g, 0, 1);

  // thread 0 walks this block's chunk list ahead of the consumers and issues one TMA box per
  // (<= 256-row) part of each tile; the map covers the local plane including its halo rows.
  // Chunks start on even S so the 16-byte result stores stay aligned.
  ChunkWalk fill_walk(g.len, LT, parts, batch, 2, eparts), use_walk(g.len, LT, parts, batch, 2, eparts);
  Chunk fc, ch;
  int nfill = 0;
  auto issue = [&]() {
    if (tid != 0 || !fill_walk.next(fc, TS)) return;
    const int st = nfill % kStages;
    if (nfill >= kStages) mbar_wait(&empty[st], ((nfill / kStages) - 1) & 1);
    if (g.dbg & 4) {  // profiling: no tile traffic
      mbar_arrive(&full[st]);
      ++nfill;
      return;
    }
    mbar_arrive_expect_tx(&full[st], (unsigned)(tb.nbox * tb.box_rows * 36 * sizeof(double)));
    const int row0 = fc.s0 - g.H + g.halo_lo;  // map row of tile row 0
    for (int k = 0; k < tb.nbox; ++k)
      tma_load_3d(xs + st * tb.stage_elems + k * tb.box_rows * kXS, &tmap, fc.lt * 32,
                  row0 + k * tb.box_rows, fc.b, &full[st]);
    ++nfill;
  };
  // the first image's taps do not depend on the previous kernel: load them, then wait for it
  // (programmatic dependent launch) and start the tile ring
  pdl_launch_dependents();
  kb_load_taps_d(cpad, tin + use_walk.b * t_bs, r, g.Wp, g.Kw, cstride, tguard, tid);
  __syncthreads();
  int taps_b = use_walk.b;
  kb_stamp(g, 0, 2);
  pdl_wait();
  for (int k = 0; k < kStages - 1; ++k) issue();

  for (int t = 0; use_walk.next(ch, TS); ++t) {
    if (ch.b != taps_b) {  // per-image taps (uniform across the block: block-level reload)
      __syncthreads();
      kb_load_taps_d(cpad, tin + ch.b * t_bs, r, g.Wp, g.Kw, cstride, tguard, tid);
      __syncthreads();
      taps_b = ch.b;
    }
    issue();  // keep kStages-1 tiles in flight ahead of the one consumed now
    const int st = t % kStages;
    mbar_wait(&full[st], (t / kStages) & 1);
    if (t == 0) kb_stamp(g, 0, 3);
    double* xt = xs + st * tb.stage_elems;
    const int row_lo = g.g0 + ch.s0 - g.H;
    const bool edge = g.fill && (row_lo < 0 || row_lo + rows_tile > g.Mg);  // block-uniform
    if (edge && !(g.dbg & 64)) {
      __syncthreads();
      kb_fold_tile_d(xt, rows_tile, row_lo, g.Mg, grp.sign[0], tid);
      fence_proxy_async();  // generic writes before the stage's next TMA fill
      __syncthreads();
    }
    const double oscale = nw2 ? 1.0 / sqrt(nw2[ch.b]) : 1.0;
    double* zb = z + ch.b * z_bs;
    for (int gi = 0; gi < grp.n; ++gi) {
      if (edge && gi > 0 && grp.sign[gi] != grp.sign[gi - 1]) {
        __syncthreads();
        kb_flip_tile_d(xt, rows_tile, row_lo, g.Mg, tid);
        fence_proxy_async();
        __syncthreads();
      }
      if (s_off < ch.cnt) {  // warp-uniform: warps past the chunk's rows idle
        const int gstart = grp.start[gi];
        const double* cb = cpad + gstart * cstride;
#define KB_DGROUP(C)                                                                                  \
  case C:                                                                                             \
    if constexpr (C <= GMAX)                                                                          \
      kb_split_group_dmma<C, NS>(xt, cb, cstride, g, s_off, lane, zb, z_ps, gstart, ch, oscale, nw2 != nullptr, \
                             mirror_h, msign ? msign + (long long)ch.b * r : nullptr);                \
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
    if (t < 2) kb_stamp(g, 0, 4 + t);
  }
  kb_stamp(g, 0, 6);
}

// ------------------------------------------------------------------------------------------
// Fused epilogue straight from the sum pass accumulators: lane (ar, ac) holds, for an S-tile at
// row offset so and M-tile j, Y[p = l0 + 8j + ar][q = s0 + so + 2ac + {0,1}] (p: m index, q: n
// index), so every operand load and result store is a 16-byte pair. kb_epi_load issues an
// S-tile's operand loads (they can be in flight during MMAs), kb_epi_apply does the arithmetic
// and the stores.
// ------------------------------------------------------------------------------------------
struct EpiScalars {
  double Lb = 0.0, db = 1.0, rd = 1.0, vs = 1.0;
};
template <int MODE>
__device__ __forceinline__ EpiScalars kb_epi_scalars(const Epi<double>& e, int b) {
  EpiScalars c;  // per-image scalars, loaded once (result stores may alias them for the compiler)
  if constexpr (MODE == EPI_UPDATE) {
    c.Lb = e.L[b];
    c.db = e.denom[b];
    c.rd = 1.0 / c.db;  // correctly rounded reciprocal: quotients via Markstein's correction
  }
  if constexpr (MODE == EPI_POWER) c.vs = e.vnw2 ? sqrt(e.vnw2[b]) : 1.0;
  return c;
}

template <int MODE>
__device__ __forceinline__ void kb_epi_load(const AxisGeom& g, const Epi<double>& e, const Chunk& ch, int so,
                                            int ar, int ac, double (&u)[4][2], double (&w)[4][2]) {
  const int sl = so + 2 * ac;
#pragma unroll
  for (int j = 0; j < 4; ++j) u[j][0] = u[j][1] = w[j][0] = w[j][1] = 0.0;
  if constexpr (MODE == EPI_PLAIN) return;
  if (sl >= ch.cnt) return;
  const bool both = sl + 1 < ch.cnt;
  const long long rowbase = (long long)ch.b * e.bstride + ch.s0 + sl;
  auto ld2 = [&](const double* a, long long at, double (&v)[2]) {
    if (both) {
      const double2 t = *reinterpret_cast<const double2*>(a + at);
      v[0] = t.x;
      v[1] = t.y;
    } else {
      v[0] = a[at];
    }
  };
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int p = ch.lt * 32 + 8 * j + ar;
    if (p >= g.other) continue;
    const long long at = rowbase + (long long)p * g.len;
    if constexpr (MODE == EPI_RESID) ld2(e.bsub, at, u[j]);
    if constexpr (MODE == EPI_UPDATE) {
      ld2(e.y, at, u[j]);
      ld2(e.x, at, w[j]);
    }
    if constexpr (MODE == EPI_POWER) ld2(e.vin, at, u[j]);
  }
}

template <int MODE, bool NORMS = true>
__device__ __forceinline__ void kb_epi_apply(const double (&D)[4][2], const AxisGeom& g, const Epi<double>& e,
                                             const EpiScalars& sc, const Chunk& ch, int so, int ar, int ac,
                                             const double (&u)[4][2], const double (&w)[4][2], double (&nrm)[3],
                                             bool& bad) {
  const int n = g.len;
  const int sl = so + 2 * ac;  // first of the lane's two S rows in the chunk
  if (sl >= ch.cnt) return;
  const bool both = sl + 1 < ch.cnt;
  const int q = ch.s0 + sl;
  const long long rowbase = (long long)ch.b * e.bstride + q;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int p = ch.lt * 32 + 8 * j + ar;
    if (p >= g.other) continue;
    const long long at = rowbase + (long long)p * n;
    double val[2] = {D[j][0], D[j][1]};
    if (e.foldH > 0) {
      const int FH = e.foldH;
      const double* f = e.fold + ((long long)ch.b * g.other + p) * (2 * FH);
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int qi = q + i;
        if (qi < FH) val[i] += f[qi];
        else if (qi >= n - FH && qi < n) val[i] += f[qi - (n - 2 * FH)];
      }
    }
    if constexpr (MODE == EPI_PLAIN) {
      st_pair(e.out + at, val[0], val[1], both);
    } else if constexpr (MODE == EPI_RESID) {
      st_pair(e.out + at, __dsub_rn(val[0], u[j][0]), __dsub_rn(val[1], u[j][1]), both);
    } else if constexpr (MODE == EPI_UPDATE) {
      double xv[2], yv[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        xv[i] = kb_quot(__dsub_rn(__dmul_rn(sc.Lb, u[j][i]), val[i]), sc.db, sc.rd);
        if (e.project) xv[i] = (xv[i] > 0.0 || xv[i] != xv[i]) ? xv[i] : 0.0;
        const double d = __dsub_rn(xv[i], w[j][i]);
        yv[i] = __dadd_rn(xv[i], __dmul_rn(e.beta, d));
        if (i == 0 || both) {
          bad |= !isfinite(xv[i]);
          if (NORMS && e.want_norms) {
            nrm[0] += d * d;
            nrm[1] += w[j][i] * w[j][i];
            nrm[2] += xv[i] * xv[i];
          }
        }
      }
      st_pair(e.x + at, xv[0], xv[1], both);
      st_pair(e.y + at, yv[0], yv[1], both);
    } else {  // EPI_POWER
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        if (i == 0 || both) {
          const double vv = e.vnw2 ? u[j][i] / sc.vs : u[j][i];
          nrm[0] += vv * val[i];
          nrm[1] += val[i] * val[i];
        }
      }
      st_pair(e.out + at, val[0], val[1], both);
    }
  }
}

// two S-tiles (the 16-row warps of kb_pass_sum_dmma): loads of a tile before its arithmetic
template <int MODE, bool NORMS = true>
__device__ __forceinline__ void kb_sum_epilogue_regs(const double (&D)[2][4][2], const AxisGeom& g,
                                                     const Epi<double>& e, const Chunk& ch,
                                                     int s_off, int ar, int ac, double (&nrm)[3],
                                                     bool& bad, const EpiScalars& sc) {
#pragma unroll
  for (int mt = 0; mt < 2; ++mt) {
    double u[4][2], w[4][2];
    kb_epi_load<MODE>(g, e, ch, s_off + 8 * mt, ar, ac, u, w);
    kb_epi_apply<MODE, NORMS>(D[mt], g, e, sc, ch, s_off + 8 * mt, ar, ac, u, w, nrm, bad);
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

// MMA loop of one (chunk, term) tile of the sum pass over K-chunks [c0, c1): S-tile 0 (B = taps
// at t0) when M0, S-tile 1 (rows +8: taps at t0 - 8, sharing the A fragment) when M1.
template <bool M0, bool M1>
__device__ __forceinline__ void kb_sum_mma_range(double (&D)[2][4][2], const double* __restrict__ xb,
                                                 const double* __restrict__ cb, int c0, int c1) {
#pragma unroll 2
  for (int c = c0; c < c1; ++c) {
    double A[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) A[j] = xb[4 * c * kXS + 8 * j];
    const double b0 = M0 ? cb[4 * c] : 0.0;
    const double b1 = M1 ? cb[4 * c - 8] : 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (M0) dmma_884(D[0][j][0], D[0][j][1], A[j], b0);
      if (M1) dmma_884(D[1][j][0], D[1][j][1], A[j], b1);
    }
  }
}

// Whole tile: S-tile 0 needs K-chunks [0, nch), S-tile 1 [2, nch + 2); the shared middle range
// runs both, the ends only the S-tile whose band they touch.
__device__ __forceinline__ void kb_sum_mma(double (&D)[2][4][2], const double* __restrict__ xb,
                                           const double* __restrict__ cb, int nch, bool two) {
  if (!two) {
    kb_sum_mma_range<true, false>(D, xb, cb, 0, nch);
    return;
  }
  kb_sum_mma_range<true, false>(D, xb, cb, 0, 2);
  kb_sum_mma_range<true, true>(D, xb, cb, 2, nch);
  kb_sum_mma_range<false, true>(D, xb, cb, nch, nch + 2);
}

// ------------------------------------------------------------------------------------------
// sum pass (fp64, DMMA): warp w owns S rows [16w, 16w+16) (two S-tiles) x 32 L of a chunk;
// the (chunk, term) tiles stream through the mbarrier ring. After a chunk's last term each warp
// runs the fused epilogue from its registers. Norm partials are per warp:
// partials[b][block*kNW + warp].
// ------------------------------------------------------------------------------------------
// NORMS = false: the update epilogue without the history norm partials (fewer registers: the
// norms' accumulators made the update kernel spill)
template <int MODE, bool NORMS = true>
__global__ void __launch_bounds__(32 * kNW, 2)
kb_pass_sum_dmma(const __grid_constant__ CUtensorMap tmap, int r, const double* __restrict__ tin,
                 long long t_bs, AxisGeom g, Epi<double> e, int batch, int parts) {
  extern __shared__ __align__(128) unsigned char kb_smem_d[];
  kb_stamp(g, 1, 0);
  __shared__ unsigned long long full[kStages], empty[kStages];
  constexpr int TS = kNW * 16;
  const int rows_tile = dmma_rows(TS, g.Kw);
  const TileBoxes tb = tile_boxes(rows_tile);
  const int cstride = dmma_cstride_sum(g.Kw);  // taps at offset kCG + 8 (S-tile 1 reads t0 - 8)
  double* xs = reinterpret_cast<double*>(kb_smem_d);  // [kStages][stage_elems]
  double* cpad = xs + kStages * tb.stage_elems;        // [r][cstride]
  const int lane = threadIdx.x, warp = threadIdx.y;
  const int tid = warp * 32 + lane;
  const int LT = (g.other + 31) / 32;
  const int ar = lane >> 2, ac = lane & 3;
  const int s_off = warp * 16;
  const int nch = dmma_chunks(g.Kw);
  const int nslots = gridDim.x * kNW, slot = blockIdx.x * kNW + warp;

  if (tid == 0) {
    for (int st = 0; st < kStages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kNW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  kb_stamp(g, 1, 1);

  // tile sequence: (chunk, term) for every chunk of this block; thread 0 issues the TMA boxes
  ChunkWalk fill_walk(g.len, LT, parts, batch, 2), use_walk(g.len, LT, parts, batch, 2);
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
    if (g.dbg & 4) {  // profiling: no tile traffic
      mbar_arrive(&full[st]);
      ++fterm;
      ++nfill;
      return;
    }
    mbar_arrive_expect_tx(&full[st], (unsigned)(tb.nbox * tb.box_rows * 36 * sizeof(double)));
    const int row0 = fc.s0 - g.H + g.halo_lo;  // halo_lo: reflected rows stored by the split pass
    for (int k = 0; k < tb.nbox; ++k)
      tma_load_3d(xs + st * tb.stage_elems + k * tb.box_rows * kXS, &tmap, fc.lt * 32,
                  row0 + k * tb.box_rows, fc.b * r + fterm, &full[st]);
    ++fterm;
    ++nfill;
  };
  pdl_launch_dependents();
  kb_load_taps_d(cpad, tin + use_walk.b * t_bs, r, g.Wp, g.Kw, cstride, kCG + 8, tid);
  __syncthreads();
  int taps_b = use_walk.b;
  kb_stamp(g, 1, 2);
  pdl_wait();
  for (int k = 0; k < kStages - 1; ++k) issue();

  double nrm[3] = {0.0, 0.0, 0.0};
  bool bad = false;
  int norm_b = -1;
  double D[2][4][2];
  Chunk ch;
  int t = 0;
  while (use_walk.next(ch, TS)) {
    if (ch.b != taps_b) {  // per-image taps (uniform across the block)
      __syncthreads();
      kb_load_taps_d(cpad, tin + ch.b * t_bs, r, g.Wp, g.Kw, cstride, kCG + 8, tid);
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
    const bool active = s_off < ch.cnt;  // warp-uniform
    const bool two = s_off + 8 < ch.cnt;
#if KB_DMMA_EARLY_SCALARS
    // the image's epilogue scalars (and the reciprocal's division) now, off the chunk's tail
    const EpiScalars sc = kb_epi_scalars<MODE>(e, ch.b);
#endif
    for (int term = 0; term < r; ++term, ++t) {
      issue();
      const int st = t % kStages;
      mbar_wait(&full[st], (t / kStages) & 1);
      if (t == 0) kb_stamp(g, 1, 3);
      const double* xt = xs + st * tb.stage_elems;
      if (active && !(g.dbg & 1))
        kb_sum_mma(D, xt + (s_off + ac) * kXS + ar, cpad + term * cstride + kCG + 8 + ac - ar, nch, two);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    if (t == r) kb_stamp(g, 1, 4);
#if !KB_DMMA_EARLY_SCALARS
    const EpiScalars sc = kb_epi_scalars<MODE>(e, ch.b);
#endif
    if (active && !(g.dbg & 2)) kb_sum_epilogue_regs<MODE, NORMS>(D, g, e, ch, s_off, ar, ac, nrm, bad, sc);
    if (t == r) kb_stamp(g, 1, 5);
  }
  if (norm_b >= 0) kb_warp_finish<MODE>(e, nrm, bad, norm_b, nslots, slot, lane);
  kb_stamp(g, 1, 6);
}

}  // namespace kb
