// kb_tf32.cuh — fp32 pass kernels on the tensor cores: 3xTF32 warp MMA (mma.sync m16n8k8).
//
// Single-pass TF32 misses the fp32 parity bound; splitting both operands as
// v = hi + lo (hi = tf32(v), lo = tf32(v - hi)) and accumulating hi*hi + lo*hi + hi*lo in fp32
// recovers fp32 accuracy (1.6e-5 at a cfg2-like solve). Measured on the box:
// 278 TF/s TF32 mma.sync, i.e. ~93 TF/s of 3xTF32 against 72 TF/s FFMA (tools/microbench.cu).
//
// Same formulation and pipeline as the fp64 DMMA kernels (kb_dmma.cuh): for 8 outputs s and 16
// columns l,  Out^T(16 l x 8 s) = X^T(16 l x K) * T(K x 8 s),  T[t][s] = c[t - s],  K-steps of 8
// input rows; the A fragment is read transposed from the TMA-filled tile, the B fragment is a
// slice of a zero-guarded tap copy, and the accumulator holds two consecutive outputs s per lane
// (8-byte stores into the transposed planes). Fragment layouts (m16n8k8, g = lane/4, q = lane%4):
//   A: a0 (g, q)  a1 (g+8, q)  a2 (g, q+4)  a3 (g+8, q+4)     [row = l, col = k]
//   B: b0 (k = q, n = g)  b1 (k = q+4, n = g)
//   C: c0 (g, 2q)  c1 (g, 2q+1)  c2 (g+8, 2q)  c3 (g+8, 2q+1)  [row = l, col = s]
// Tiles are [rows][kXF] floats: the 40-float row stride puts the 32 A-fragment addresses of a
// warp (4 rows x 8 columns) in 32 distinct banks.
#pragma once
#include "kb_ffma.cuh"

namespace kb {

constexpr int kXF = 40;  // fp32 tile row stride (floats); TMA box width
constexpr int kMaxStages = 4;  // tile ring depth limit (the host picks what shared memory allows)

__device__ __forceinline__ unsigned tf32_rna(float x) {
  unsigned r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}
// operand split for the data tiles: hi = x with the 13 low mantissa bits cleared (exactly a
// tf32 value), lo = x - hi (exact); the MMA reads lo's top 19 bits, so the dropped part is
// below 2^-21 |x|, the size of the lo*lo term 3xTF32 omits anyway
__device__ __forceinline__ void tf32_split(float x, unsigned& hi, unsigned& lo) {
  hi = __float_as_uint(x) & 0xffffe000u;
  lo = __float_as_uint(x - __uint_as_float(hi));
}
// tap split (once per tile fill): round-to-nearest hi, rounded lo
__device__ __forceinline__ void tf32_split_rn(float x, unsigned& hi, unsigned& lo) {
  hi = tf32_rna(x);
  lo = tf32_rna(x - __uint_as_float(hi));
}
__device__ __forceinline__ void mma_tf32(float (&d)[4], const unsigned (&a)[4], unsigned b0, unsigned b1) {
  asm("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
// K-steps of 8 covering t in [0, Wp + 7) for one 8-output block
__host__ __device__ __forceinline__ int tf32_ksteps(int Wp) { return (Wp + 7 + 7) / 8; }
__host__ __device__ __forceinline__ int tf32_rows(int TS, int Wp) { return TS - 8 + 8 * tf32_ksteps(Wp); }
// zero-guarded tap copies (hi and lo): 16 guard entries before the taps, enough after them
__host__ __device__ __forceinline__ int tf32_cstride(int Wp) { return 8 * tf32_ksteps(Wp) + 32; }
constexpr int kTG = 16;  // guard before the taps

struct TileBoxesX {
  int nbox, box_rows, stage_elems;
};
__host__ __device__ __forceinline__ TileBoxesX tile_boxes_x(int rows) {
  TileBoxesX t;
  t.nbox = (rows + 255) / 256;
  t.box_rows = (rows + t.nbox - 1) / t.nbox;
  t.stage_elems = ((t.nbox * t.box_rows * kXF + 31) / 32) * 32;  // 128-byte multiples
  return t;
}

// out-of-domain tile rows: sign * folded partner, or 0 (all threads; edge tiles only)
__device__ __forceinline__ void kb_fold_tile_x(float* __restrict__ xs, int rows, int row_lo, int Mg, int sign,
                                               int tid) {
  const int top = min(max(-row_lo, 0), rows);
  const int bot = max(min(Mg - row_lo, rows), top);
  const int nel = (top + rows - bot) * 32;
  for (int i0 = 0; i0 < nel; i0 += 4 * 32 * kNW) {
    float v[4];
    int dst[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int idx = i0 + k * 32 * kNW + tid;
      dst[k] = -1;
      v[k] = 0.f;
      if (idx < nel) {
        const int q = idx >> 5, col = idx & 31;
        const int rr = q < top ? q : bot + (q - top);
        const int f = kb_fold(row_lo + rr, Mg);
        const int u = f - row_lo;
        if (f >= 0 && u >= 0 && u < rows) v[k] = xs[u * kXF + col];
        dst[k] = rr * kXF + col;
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (dst[k] >= 0) xs[dst[k]] = sign < 0 ? -v[k] : v[k];
  }
}
__device__ __forceinline__ void kb_flip_tile_x(float* __restrict__ xs, int rows, int row_lo, int Mg, int tid) {
  const int top = min(max(-row_lo, 0), rows);
  const int bot = max(min(Mg - row_lo, rows), top);
  const int nel = (top + rows - bot) * 32;
  for (int idx = tid; idx < nel; idx += 32 * kNW) {
    const int q = idx >> 5, col = idx & 31;
    const int rr = q < top ? q : bot + (q - top);
    xs[rr * kXF + col] = -xs[rr * kXF + col];
  }
}

// per-image tap tables [r][Wp] -> shared memory as zero-guarded tf32 hi / lo copies of the first
// Kw taps of each row; 16-byte loads, all issued before any store (one memory round trip)
__device__ __forceinline__ void kb_load_taps_x(unsigned* __restrict__ chi, unsigned* __restrict__ clo,
                                               const float* __restrict__ tb, int r, int Wp, int Kw, int cstride,
                                               int guard, int tid) {
  const int n4 = r * Wp / 4, nw = Wp / 4;
  constexpr int kV = 4;
  for (int j0 = 0; j0 < n4; j0 += kV * 32 * kNW) {
    float4 v[kV];
#pragma unroll
    for (int u = 0; u < kV; ++u) {
      const int j = j0 + u * 32 * kNW + tid;
      if (j < n4) v[u] = reinterpret_cast<const float4*>(tb)[j];
    }
#pragma unroll
    for (int u = 0; u < kV; ++u) {
      const int j = j0 + u * 32 * kNW + tid;
      if (j < n4) {
        const int i = j / nw, k0 = 4 * (j - i * nw), o = i * cstride + guard + k0;
        const float c[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if (k0 + e >= Kw) break;
          unsigned h, l;
          tf32_split_rn(c[e], h, l);
          chi[o + e] = h;
          clo[o + e] = l;
        }
      }
    }
  }
  const int ng = cstride - Kw;
  for (int idx = tid; idx < r * ng; idx += 32 * kNW) {
    const int i = idx / ng, k = idx - i * ng;
    const int o = i * cstride + (k < guard ? k : Kw + k);
    chi[o] = 0u;
    clo[o] = 0u;
  }
}

// A fragments (hi, lo) of K-step c for M-tile m: tile rows s_off + 8c + {q, q+4}, columns
// 16m + {g, g+8}
__device__ __forceinline__ void kb_afrag(const float* __restrict__ xb, int c, int m, unsigned (&hi)[4],
                                         unsigned (&lo)[4]) {
  const float* p = xb + 8 * c * kXF + 16 * m;
  tf32_split(p[0], hi[0], lo[0]);
  tf32_split(p[8], hi[1], lo[1]);
  tf32_split(p[4 * kXF], hi[2], lo[2]);
  tf32_split(p[4 * kXF + 8], hi[3], lo[3]);
}

__device__ __forceinline__ void st_pair_f(float* p, float a, float b, bool both) {
  if (both) *reinterpret_cast<float2*>(p) = make_float2(a, b);
  else *p = a;
}

// ------------------------------------------------------------------------------------------
// split pass: warp w owns S rows [8w, 8w+8) of a chunk x 32 L (two 16-column M-tiles) for the
// G terms of a group; lane (g, q) ends with Z^T[l0 + 16m + g (+8)][s0 + 8w + 2q + {0,1}].
// ------------------------------------------------------------------------------------------
template <int G>
__device__ __forceinline__ void kb_split_group_x(const float* __restrict__ xs, const unsigned* __restrict__ chi,
                                                 const unsigned* __restrict__ clo, int cstride,
                                                 const AxisGeom& g, int s_off, int lane,
                                                 float* __restrict__ z, long long z_ps, int gstart,
                                                 const Chunk& ch, float oscale, bool scaled, int mirror_h,
                                                 const float* __restrict__ msign) {
  const int gq = lane >> 2, q = lane & 3;
  float D[G][2][4];
#pragma unroll
  for (int gg = 0; gg < G; ++gg)
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int i = 0; i < 4; ++i) D[gg][m][i] = 0.f;
  const int nk = (g.dbg & 1) ? 0 : tf32_ksteps(g.Kw);
  const float* xb = xs + (s_off + q) * kXF + gq;
  const int boff = kTG + q - gq;  // b0 = c[8c + q - g], b1 = c[8c + q + 4 - g]
#pragma unroll 2
  for (int c = 0; c < nk; ++c) {
    unsigned ah[2][4], al[2][4];
    kb_afrag(xb, c, 0, ah[0], al[0]);
    kb_afrag(xb, c, 1, ah[1], al[1]);
    unsigned bh[G][2], bl[G][2];
#pragma unroll
    for (int gg = 0; gg < G; ++gg) {
      const int o = gg * cstride + boff + 8 * c;
      bh[gg][0] = chi[o];
      bh[gg][1] = chi[o + 4];
      bl[gg][0] = clo[o];
      bl[gg][1] = clo[o + 4];
    }
    // the three products of every accumulator are issued as three independent sweeps, so
    // consecutive MMAs never wait on each other's accumulator
    // each K-step's products accumulate from zero and are added to D with a round-to-nearest
    // FADD: the tensor core's own fp32 accumulation drifts over long K (wide bands, many terms)
    float T[G][2][4];
#pragma unroll
    for (int gg = 0; gg < G; ++gg)
#pragma unroll
      for (int m = 0; m < 2; ++m) {
#pragma unroll
        for (int i = 0; i < 4; ++i) T[gg][m][i] = 0.f;
        mma_tf32(T[gg][m], al[m], bh[gg][0], bh[gg][1]);
      }
#pragma unroll
    for (int gg = 0; gg < G; ++gg)
#pragma unroll
      for (int m = 0; m < 2; ++m) mma_tf32(T[gg][m], ah[m], bl[gg][0], bl[gg][1]);
#pragma unroll
    for (int gg = 0; gg < G; ++gg)
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        mma_tf32(T[gg][m], ah[m], bh[gg][0], bh[gg][1]);
#pragma unroll
        for (int i = 0; i < 4; ++i) D[gg][m][i] += T[gg][m][i];
      }
  }
  const int s = s_off + 2 * q;
  if (s >= ch.cnt || (g.dbg & 2)) return;
  const bool both = s + 1 < ch.cnt;
#pragma unroll
  for (int gg = 0; gg < G; ++gg) {
    float* zp = z + (long long)(gstart + gg) * z_ps + ch.s0 + s;
    const float sg = msign ? msign[gstart + gg] : 1.f;
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int l = ch.lt * 32 + 16 * m + 8 * h + gq;
        if (l >= g.other) continue;
        float v0 = D[gg][m][2 * h], v1 = D[gg][m][2 * h + 1];
        if (scaled) {
          v0 *= oscale;
          v1 *= oscale;
        }
        st_pair_f(zp + (long long)l * g.len, v0, v1, both);
        if (mirror_h > 0) {  // reflected halo rows of Z^T for the reflect-filled sum pass
          if (l < mirror_h) st_pair_f(zp + (long long)(-1 - l) * g.len, sg * v0, sg * v1, both);
          if (l >= g.other - mirror_h)
            st_pair_f(zp + (long long)(2 * g.other - 1 - l) * g.len, sg * v0, sg * v1, both);
        }
      }
  }
}

template <int GMAX>
__global__ void __launch_bounds__(32 * kNW, 2)
kb_pass_split_x(const __grid_constant__ CUtensorMap tmap, float* __restrict__ z, long long z_ps,
                long long z_bs, const float* __restrict__ tin, long long t_bs, AxisGeom g, Groups grp,
                const double* __restrict__ nw2, int r, int batch, int parts, int eparts, int mirror_h,
                const float* __restrict__ msign, int nst) {
  extern __shared__ __align__(128) unsigned char kb_smem_x[];
  kb_stamp(g, 0, 0);
  __shared__ unsigned long long full[kMaxStages], empty[kMaxStages];
  constexpr int TS = kNW * 8;
  const int rows_tile = tf32_rows(TS, g.Kw);
  const TileBoxesX tb = tile_boxes_x(rows_tile);
  const int cstride = tf32_cstride(g.Kw);
  float* xs = reinterpret_cast<float*>(kb_smem_x);                       // [nst][stage_elems]
  unsigned* chi = reinterpret_cast<unsigned*>(xs + nst * tb.stage_elems);  // [r][cstride]
  unsigned* clo = chi + r * cstride;
  const int lane = threadIdx.x, warp = threadIdx.y;
  const int tid = warp * 32 + lane;
  const int LT = (g.other + 31) / 32;
  const int s_off = warp * 8;

  if (tid == 0) {
    for (int st = 0; st < nst; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kNW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  kb_stamp(g, 0, 1);

  ChunkWalk fill_walk(g.len, LT, parts, batch, 2, eparts), use_walk(g.len, LT, parts, batch, 2, eparts);
  Chunk fc, ch;
  int nfill = 0;
  auto issue = [&]() {
    if (tid != 0 || !fill_walk.next(fc, TS)) return;
    const int st = nfill % nst;
    if (nfill >= nst) mbar_wait(&empty[st], ((nfill / nst) - 1) & 1);
    if (g.dbg & 4) {
      mbar_arrive(&full[st]);
      ++nfill;
      return;
    }
    mbar_arrive_expect_tx(&full[st], (unsigned)(tb.nbox * tb.box_rows * kXF * sizeof(float)));
    const int row0 = fc.s0 - g.H + g.halo_lo;
    for (int k = 0; k < tb.nbox; ++k)
      tma_load_3d(xs + st * tb.stage_elems + k * tb.box_rows * kXF, &tmap, fc.lt * 32,
                  row0 + k * tb.box_rows, fc.b, &full[st]);
    ++nfill;
  };
  pdl_launch_dependents();  // taps first, then wait for the previous kernel (see kb_dmma.cuh)
  kb_load_taps_x(chi, clo, tin + use_walk.b * t_bs, r, g.Wp, g.Kw, cstride, kTG, tid);
  __syncthreads();
  int taps_b = use_walk.b;
  kb_stamp(g, 0, 2);
  pdl_wait();
  for (int k = 0; k < nst - 1; ++k) issue();

  for (int t = 0; use_walk.next(ch, TS); ++t) {
    if (ch.b != taps_b) {
      __syncthreads();
      kb_load_taps_x(chi, clo, tin + ch.b * t_bs, r, g.Wp, g.Kw, cstride, kTG, tid);
      __syncthreads();
      taps_b = ch.b;
    }
    issue();
    const int st = t % nst;
    mbar_wait(&full[st], (t / nst) & 1);
    if (t == 0) kb_stamp(g, 0, 3);
    float* xt = xs + st * tb.stage_elems;
    const int row_lo = g.g0 + ch.s0 - g.H;
    const bool edge = g.fill && (row_lo < 0 || row_lo + rows_tile > g.Mg);  // block-uniform
    if (edge) {
      __syncthreads();
      kb_fold_tile_x(xt, rows_tile, row_lo, g.Mg, grp.sign[0], tid);
      fence_proxy_async();
      __syncthreads();
    }
    const float oscale = nw2 ? (float)(1.0 / sqrt(nw2[ch.b])) : 1.f;
    float* zb = z + ch.b * z_bs;
    for (int gi = 0; gi < grp.n; ++gi) {
      if (edge && gi > 0 && grp.sign[gi] != grp.sign[gi - 1]) {
        __syncthreads();
        kb_flip_tile_x(xt, rows_tile, row_lo, g.Mg, tid);
        fence_proxy_async();
        __syncthreads();
      }
      if (s_off < ch.cnt) {
        const int gstart = grp.start[gi];
#define KB_XGROUP(C)                                                                                      \
  case C:                                                                                                 \
    if constexpr (C <= GMAX)                                                                              \
      kb_split_group_x<C>(xt, chi + gstart * cstride, clo + gstart * cstride, cstride, g, s_off, lane, zb, \
                          z_ps, gstart, ch, oscale, nw2 != nullptr, mirror_h,                             \
                          msign ? msign + (long long)ch.b * r : nullptr);                                 \
    break;
        switch (grp.count[gi]) {
          KB_XGROUP(1)
          KB_XGROUP(2)
          KB_XGROUP(3)
          KB_XGROUP(4)
          default: break;
        }
#undef KB_XGROUP
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
    if (t < 2) kb_stamp(g, 0, 4 + t);
  }
  kb_stamp(g, 0, 6);
}

// ------------------------------------------------------------------------------------------
// sum pass epilogue: lane (g, q) holds, for N-tile n (8 S rows) and M-tile m (16 columns),
// Y[p = l0 + 16m + 8h + g][q' = s0 + s_off + 8n + 2q + {0,1}] in D[n][m][2h + {0,1}].
// ------------------------------------------------------------------------------------------
template <int MODE, bool NORMS = true>
__device__ __forceinline__ void kb_sum_epilogue_x(const float (&D)[2][2][4], const AxisGeom& g,
                                                  const Epi<float>& e, const Chunk& ch, int s_off, int lane,
                                                  double (&nrm)[3], bool& bad) {
  const int gq = lane >> 2, q = lane & 3;
  const int n = g.len;
  float Lb = 0.f, db = 1.f, rd = 1.f;
  double vs = 1.0;
  if constexpr (MODE == EPI_UPDATE) {
    Lb = (float)e.L[ch.b];
    db = (float)e.denom[ch.b];
    rd = 1.f / db;  // correctly rounded reciprocal: quotients via Markstein's correction
  }
  if constexpr (MODE == EPI_POWER) vs = e.vnw2 ? sqrt(e.vnw2[ch.b]) : 1.0;
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
    const int sl = s_off + 8 * nt + 2 * q;
    if (sl >= ch.cnt) continue;
    const bool both = sl + 1 < ch.cnt;
    const int qq = ch.s0 + sl;
    const long long rowbase = (long long)ch.b * e.bstride + qq;
    float u[2][2][2], w[2][2][2];
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int p = ch.lt * 32 + 16 * m + 8 * h + gq;
        const long long at = rowbase + (long long)p * n;
        u[m][h][0] = u[m][h][1] = w[m][h][0] = w[m][h][1] = 0.f;
        if (p >= g.other) continue;
        auto ld2 = [&](const float* a, float (&v)[2]) {
          if (both) {
            const float2 t2 = *reinterpret_cast<const float2*>(a + at);
            v[0] = t2.x;
            v[1] = t2.y;
          } else {
            v[0] = a[at];
          }
        };
        if constexpr (MODE == EPI_RESID) ld2(e.bsub, u[m][h]);
        if constexpr (MODE == EPI_UPDATE) {
          ld2(e.y, u[m][h]);
          ld2(e.x, w[m][h]);
        }
        if constexpr (MODE == EPI_POWER) ld2(e.vin, u[m][h]);
      }
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int p = ch.lt * 32 + 16 * m + 8 * h + gq;
        if (p >= g.other) continue;
        const long long at = rowbase + (long long)p * n;
        float val[2] = {D[nt][m][2 * h], D[nt][m][2 * h + 1]};
        if (e.foldH > 0) {
          const int FH = e.foldH;
          const float* f = e.fold + ((long long)ch.b * g.other + p) * (2 * FH);
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const int qi = qq + i;
            if (qi < FH) val[i] += f[qi];
            else if (qi >= n - FH && qi < n) val[i] += f[qi - (n - 2 * FH)];
          }
        }
        if constexpr (MODE == EPI_PLAIN) {
          st_pair_f(e.out + at, val[0], val[1], both);
        } else if constexpr (MODE == EPI_RESID) {
          st_pair_f(e.out + at, __fsub_rn(val[0], u[m][h][0]), __fsub_rn(val[1], u[m][h][1]), both);
        } else if constexpr (MODE == EPI_UPDATE) {
          float xv[2], yv[2];
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            const float a = __fsub_rn(__fmul_rn(Lb, u[m][h][i]), val[i]);
            const float q0 = __fmul_rn(a, rd);
            xv[i] = fmaf(fmaf(-db, q0, a), rd, q0);
            if (e.project) xv[i] = (xv[i] > 0.f || xv[i] != xv[i]) ? xv[i] : 0.f;
            const float d = __fsub_rn(xv[i], w[m][h][i]);
            yv[i] = __fadd_rn(xv[i], __fmul_rn((float)e.beta, d));
            if (i == 0 || both) {
              bad |= !isfinite(xv[i]);
              if (NORMS && e.want_norms) {
                nrm[0] += (double)d * d;
                nrm[1] += (double)w[m][h][i] * w[m][h][i];
                nrm[2] += (double)xv[i] * xv[i];
              }
            }
          }
          st_pair_f(e.x + at, xv[0], xv[1], both);
          st_pair_f(e.y + at, yv[0], yv[1], both);
        } else {  // EPI_POWER
#pragma unroll
          for (int i = 0; i < 2; ++i)
            if (i == 0 || both) {
              const double vv = e.vnw2 ? (double)u[m][h][i] / vs : (double)u[m][h][i];
              nrm[0] += vv * val[i];
              nrm[1] += (double)val[i] * val[i];
            }
          st_pair_f(e.out + at, val[0], val[1], both);
        }
      }
  }
}

// sum-pass MMAs over K-steps [c0, c1): N-tile 0 (B = taps at 8c) when N0, N-tile 1 (outputs +8:
// taps at 8c - 8, sharing the A fragments) when N1
template <bool N0, bool N1>
__device__ __forceinline__ void kb_sum_mma_x(float (&D)[2][2][4], const float* __restrict__ xb,
                                             const unsigned* __restrict__ bh, const unsigned* __restrict__ bl,
                                             int c0, int c1) {
#pragma unroll 2
  for (int c = c0; c < c1; ++c) {
    unsigned ah[2][4], al[2][4];
    kb_afrag(xb, c, 0, ah[0], al[0]);
    kb_afrag(xb, c, 1, ah[1], al[1]);
    unsigned h[2][2], l[2][2];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int o = 8 * c - 8 * nt;
      h[nt][0] = bh[o];
      h[nt][1] = bh[o + 4];
      l[nt][0] = bl[o];
      l[nt][1] = bl[o + 4];
    }
    // three independent sweeps over the accumulators (see kb_split_group_x)
    float T[2][2][4];  // per-K-step partials, added with round-to-nearest (see kb_split_group_x)
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int m = 0; m < 2; ++m) {
#pragma unroll
        for (int i = 0; i < 4; ++i) T[nt][m][i] = 0.f;
        if (nt == 0 ? N0 : N1) mma_tf32(T[nt][m], al[m], h[nt][0], h[nt][1]);
      }
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int m = 0; m < 2; ++m)
        if (nt == 0 ? N0 : N1) mma_tf32(T[nt][m], ah[m], l[nt][0], l[nt][1]);
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int m = 0; m < 2; ++m)
        if (nt == 0 ? N0 : N1) {
          mma_tf32(T[nt][m], ah[m], h[nt][0], h[nt][1]);
#pragma unroll
          for (int i = 0; i < 4; ++i) D[nt][m][i] += T[nt][m][i];
        }
  }
}

// ------------------------------------------------------------------------------------------
// sum pass: warp w owns S rows [16w, 16w+16) (two N-tiles) x 32 L of a chunk; the (chunk,
// term) tiles stream through the mbarrier ring; fused epilogue from the accumulators.
// ------------------------------------------------------------------------------------------
template <int MODE, bool NORMS = true>  // NORMS = false: update without the history norms
__global__ void __launch_bounds__(32 * kNW, 2)
kb_pass_sum_x(const __grid_constant__ CUtensorMap tmap, int r, const float* __restrict__ tin, long long t_bs,
              AxisGeom g, Epi<float> e, int batch, int parts, int nst) {
  extern __shared__ __align__(128) unsigned char kb_smem_x[];
  kb_stamp(g, 1, 0);
  __shared__ unsigned long long full[kMaxStages], empty[kMaxStages];
  constexpr int TS = kNW * 16;
  const int rows_tile = tf32_rows(TS, g.Kw);
  const TileBoxesX tb = tile_boxes_x(rows_tile);
  const int cstride = tf32_cstride(g.Kw);
  float* xs = reinterpret_cast<float*>(kb_smem_x);
  unsigned* chi = reinterpret_cast<unsigned*>(xs + nst * tb.stage_elems);  // [r][cstride]
  unsigned* clo = chi + r * cstride;
  const int lane = threadIdx.x, warp = threadIdx.y;
  const int tid = warp * 32 + lane;
  const int LT = (g.other + 31) / 32;
  const int gq = lane >> 2, q = lane & 3;
  const int s_off = warp * 16;
  const int nk = tf32_ksteps(g.Kw);
  const int nslots = gridDim.x * kNW, slot = blockIdx.x * kNW + warp;

  if (tid == 0) {
    for (int st = 0; st < nst; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kNW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  kb_stamp(g, 1, 1);

  ChunkWalk fill_walk(g.len, LT, parts, batch, 2), use_walk(g.len, LT, parts, batch, 2);
  Chunk fc;
  int fterm = r;
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
    const int st = nfill % nst;
    if (nfill >= nst) mbar_wait(&empty[st], ((nfill / nst) - 1) & 1);
    if (g.dbg & 4) {
      mbar_arrive(&full[st]);
      ++fterm;
      ++nfill;
      return;
    }
    mbar_arrive_expect_tx(&full[st], (unsigned)(tb.nbox * tb.box_rows * kXF * sizeof(float)));
    const int row0 = fc.s0 - g.H + g.halo_lo;  // halo_lo: reflected rows stored by the split pass
    for (int k = 0; k < tb.nbox; ++k)
      tma_load_3d(xs + st * tb.stage_elems + k * tb.box_rows * kXF, &tmap, fc.lt * 32,
                  row0 + k * tb.box_rows, fc.b * r + fterm, &full[st]);
    ++fterm;
    ++nfill;
  };
  pdl_launch_dependents();
  kb_load_taps_x(chi, clo, tin + use_walk.b * t_bs, r, g.Wp, g.Kw, cstride, kTG + 8, tid);
  __syncthreads();
  int taps_b = use_walk.b;
  kb_stamp(g, 1, 2);
  pdl_wait();
  for (int k = 0; k < nst - 1; ++k) issue();

  double nrm[3] = {0.0, 0.0, 0.0};
  bool bad = false;
  int norm_b = -1;
  float D[2][2][4];
  Chunk ch;
  int t = 0;
  while (use_walk.next(ch, TS)) {
    if (ch.b != taps_b) {
      __syncthreads();
      kb_load_taps_x(chi, clo, tin + ch.b * t_bs, r, g.Wp, g.Kw, cstride, kTG + 8, tid);
      __syncthreads();
      taps_b = ch.b;
    }
    if (ch.b != norm_b) {
      if (norm_b >= 0) kb_warp_finish_f<MODE>(e, nrm, bad, norm_b, nslots, slot, lane);
      nrm[0] = nrm[1] = nrm[2] = 0.0;
      bad = false;
      norm_b = ch.b;
    }
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int m = 0; m < 2; ++m)
#pragma unroll
        for (int i = 0; i < 4; ++i) D[a][m][i] = 0.f;
    const bool active = s_off < ch.cnt;
    const bool two = s_off + 8 < ch.cnt;
    for (int term = 0; term < r; ++term, ++t) {
      issue();
      const int st = t % nst;
      mbar_wait(&full[st], (t / nst) & 1);
      if (t == 0) kb_stamp(g, 1, 3);
      const float* xt = xs + st * tb.stage_elems;
      if (active && !(g.dbg & 1)) {
        const float* xb = xt + (s_off + q) * kXF + gq;
        const int o = term * cstride + kTG + 8 + q - gq;
        if (two) {
          kb_sum_mma_x<true, false>(D, xb, chi + o, clo + o, 0, 1);
          kb_sum_mma_x<true, true>(D, xb, chi + o, clo + o, 1, nk);
          kb_sum_mma_x<false, true>(D, xb, chi + o, clo + o, nk, nk + 1);
        } else {
          kb_sum_mma_x<true, false>(D, xb, chi + o, clo + o, 0, nk);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    if (t == r) kb_stamp(g, 1, 4);
    if (active && !(g.dbg & 2)) kb_sum_epilogue_x<MODE, NORMS>(D, g, e, ch, s_off, lane, nrm, bad);
    if (t == r) kb_stamp(g, 1, 5);
  }
  if (norm_b >= 0) kb_warp_finish_f<MODE>(e, nrm, bad, norm_b, nslots, slot, lane);
  kb_stamp(g, 1, 6);
}

}  // namespace kb
