// kb_ffma.cuh — fp32 pass kernels: persistent, TMA-fed, FFMA register windows.
//
// Same pipeline as the fp64 DMMA kernels (kb_dmma.cuh): balanced persistent work items, input
// tiles streamed by TMA boxes into a shared-memory ring guarded by mbarriers, results written
// straight from registers. The arithmetic is FP32 FMA with the sliding register windows of
// kb_taps (the fp32 tensor path — 3xTF32 on tcgen05 — is the planned K2 kernel).
//
// Thread mapping: lane = L column, warp = R consecutive S rows; tiles are [rows][32] floats
// (128-byte rows, conflict-free column reads). For a reflect-filled pass at a domain edge the
// out-of-domain rows of a landed split-pass tile are rewritten in shared memory from their folded
// partner (times the term group's sign); the split pass also stores the reflected halo rows of
// Z^T, so the sum pass reads its edge tiles as plain TMA boxes.
#pragma once
#include "kb_dmma.cuh"

namespace kb {

struct TileBoxesF {
  int nbox, box_rows, stage_elems;
};
__host__ __device__ __forceinline__ TileBoxesF tile_boxes_f(int rows) {
  TileBoxesF t;
  t.nbox = (rows + 255) / 256;
  t.box_rows = (rows + t.nbox - 1) / t.nbox;
  t.stage_elems = t.nbox * t.box_rows * 32;  // 128-byte rows
  return t;
}

// rewrite the out-of-domain rows of a landed [rows][32] tile: sign * folded partner, or 0
// (all threads, only the out-of-domain rows, four independent elements per thread in flight)
__device__ __forceinline__ void kb_fold_tile_f(float* __restrict__ xs, int rows, int row_lo, int Mg,
                                               int sign, int tid) {
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
        if (f >= 0 && u >= 0 && u < rows) v[k] = xs[u * 32 + col];
        dst[k] = rr * 32 + col;
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (dst[k] >= 0) xs[dst[k]] = sign < 0 ? -v[k] : v[k];
  }
}

// flip the out-of-domain rows (group sign change on an already folded tile)
__device__ __forceinline__ void kb_flip_tile_f(float* __restrict__ xs, int rows, int row_lo, int Mg, int tid) {
  const int top = min(max(-row_lo, 0), rows);
  const int bot = max(min(Mg - row_lo, rows), top);
  const int nel = (top + rows - bot) * 32;
  for (int idx = tid; idx < nel; idx += 32 * kNW) {
    const int q = idx >> 5, col = idx & 31;
    const int rr = q < top ? q : bot + (q - top);
    xs[rr * 32 + col] = -xs[rr * 32 + col];
  }
}

// ------------------------------------------------------------------------------------------
// split pass (fp32): warp w owns S rows [8w, 8w+8) of a chunk, lane l one L column; G terms
// per group in registers (kb_taps). Each thread stores its 8 consecutive S outputs (32 B) of
// Z_i^T[l][.] as two 16-byte vectors.
// ------------------------------------------------------------------------------------------
template <int G>
__device__ __forceinline__ void kb_split_group_f(const float* __restrict__ xs, const float* __restrict__ cin,
                                                 int Wp, const AxisGeom& g, int s_off, int lane,
                                                 float* __restrict__ z, long long z_ps, int gstart,
                                                 const Chunk& ch, float oscale, bool scaled, int mirror_h,
                                                 const float* __restrict__ msign) {
  float acc[G][8];
#pragma unroll
  for (int gg = 0; gg < G; ++gg)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[gg][j] = 0.f;
  if (!(g.dbg & 1)) kb_taps<float, G, 8>(acc, xs + s_off * 32 + lane, cin, Wp, Wp);
  const int l = ch.lt * 32 + lane;
  if (l >= g.other || (g.dbg & 2)) return;
  const bool full = s_off + 8 <= ch.cnt;
  auto put = [&](float* zp, const float (&v)[8], float sg) {
    if (full) {
      reinterpret_cast<float4*>(zp)[0] = make_float4(sg * v[0], sg * v[1], sg * v[2], sg * v[3]);
      reinterpret_cast<float4*>(zp)[1] = make_float4(sg * v[4], sg * v[5], sg * v[6], sg * v[7]);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (s_off + j < ch.cnt) zp[j] = sg * v[j];
    }
  };
#pragma unroll
  for (int gg = 0; gg < G; ++gg) {
    float* zp = z + (long long)(gstart + gg) * z_ps + ch.s0 + s_off;
    if (scaled) {
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[gg][j] *= oscale;
    }
    put(zp + (long long)l * g.len, acc[gg], 1.f);
    if (mirror_h > 0) {  // reflected halo rows of Z^T for the reflect-filled sum pass
      const float sg = msign ? msign[gstart + gg] : 1.f;
      if (l < mirror_h) put(zp + (long long)(-1 - l) * g.len, acc[gg], sg);
      if (l >= g.other - mirror_h) put(zp + (long long)(2 * g.other - 1 - l) * g.len, acc[gg], sg);
    }
  }
}

template <int GMAX>
__global__ void __launch_bounds__(32 * kNW, 2)
kb_pass_split_f(const __grid_constant__ CUtensorMap tmap, float* __restrict__ z, long long z_ps,
                long long z_bs, const float* __restrict__ tin, long long t_bs, AxisGeom g, Groups grp,
                const double* __restrict__ nw2, int r, int batch, int parts, int eparts, int mirror_h,
                const float* __restrict__ msign) {
  extern __shared__ __align__(128) unsigned char kb_smem_f[];
  __shared__ unsigned long long full[kStages], empty[kStages];
  constexpr int TS = kNW * 8;
  const int rows_tile = TS + g.Wp;  // kb_taps reads rows s_off .. s_off + Wp + 7
  const TileBoxesF tb = tile_boxes_f(rows_tile);
  float* xs = reinterpret_cast<float*>(kb_smem_f);  // [kStages][stage_elems]
  float* cpad = xs + kStages * tb.stage_elems;       // [r][Wp]
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
  pdl_wait();  // launched with programmatic serialization: the previous kernel's outputs are read below

  ChunkWalk fill_walk(g.len, LT, parts, batch, 4, eparts), use_walk(g.len, LT, parts, batch, 4, eparts);
  Chunk fc, ch;
  int nfill = 0;
  auto issue = [&]() {
    if (tid != 0 || !fill_walk.next(fc, TS)) return;
    const int st = nfill % kStages;
    if (nfill >= kStages) mbar_wait(&empty[st], ((nfill / kStages) - 1) & 1);
    mbar_arrive_expect_tx(&full[st], (unsigned)(tb.stage_elems * sizeof(float)));
    const int row0 = fc.s0 - g.H + g.halo_lo;
    for (int k = 0; k < tb.nbox; ++k)
      tma_load_3d(xs + st * tb.stage_elems + k * tb.box_rows * 32, &tmap, fc.lt * 32,
                  row0 + k * tb.box_rows, fc.b, &full[st]);
    ++nfill;
  };
  for (int k = 0; k < kStages - 1; ++k) issue();

  int taps_b = -1;
  for (int t = 0; use_walk.next(ch, TS); ++t) {
    if (ch.b != taps_b) {
      __syncthreads();
      const float* tbp = tin + ch.b * t_bs;
      for (int idx = tid; idx < r * g.Wp; idx += 32 * kNW) cpad[idx] = tbp[idx];
      __syncthreads();
      taps_b = ch.b;
    }
    issue();
    const int st = t % kStages;
    mbar_wait(&full[st], (t / kStages) & 1);
    float* xt = xs + st * tb.stage_elems;
    const int row_lo = g.g0 + ch.s0 - g.H;
    const bool edge = g.fill && (row_lo < 0 || row_lo + rows_tile > g.Mg);
    if (edge) {  // block-uniform
      __syncthreads();
      kb_fold_tile_f(xt, rows_tile, row_lo, g.Mg, grp.sign[0], tid);
      fence_proxy_async();
      __syncthreads();
    }
    const float oscale = nw2 ? (float)(1.0 / sqrt(nw2[ch.b])) : 1.f;
    float* zb = z + ch.b * z_bs;
    for (int gi = 0; gi < grp.n; ++gi) {
      if (edge && gi > 0 && grp.sign[gi] != grp.sign[gi - 1]) {
        __syncthreads();
        kb_flip_tile_f(xt, rows_tile, row_lo, g.Mg, tid);
        fence_proxy_async();
        __syncthreads();
      }
      if (s_off < ch.cnt) {
        const int gstart = grp.start[gi];
        const float* cb = cpad + gstart * g.Wp;
#define KB_FGROUP(C)                                                                                  \
  case C:                                                                                             \
    if constexpr (C <= GMAX)                                                                          \
      kb_split_group_f<C>(xt, cb, g.Wp, g, s_off, lane, zb, z_ps, gstart, ch, oscale, nw2 != nullptr, \
                          mirror_h, msign ? msign + (long long)ch.b * r : nullptr);                 \
    break;
        switch (grp.count[gi]) {
          KB_FGROUP(1)
          KB_FGROUP(2)
          KB_FGROUP(3)
          KB_FGROUP(4)
          KB_FGROUP(5)
          KB_FGROUP(6)
          KB_FGROUP(7)
          KB_FGROUP(8)
          default: break;
        }
#undef KB_FGROUP
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
}

// ------------------------------------------------------------------------------------------
// sum pass (fp32): warp w owns S rows [16w, 16w+16) of a chunk, lane l one L column; all terms
// accumulate in 16 registers; the epilogue works on each thread's 16 consecutive outputs of
// image row l (64 B) with 16-byte vector loads and stores.
// ------------------------------------------------------------------------------------------
template <int MODE>
__device__ __forceinline__ void kb_sum_epilogue_f(float (&acc)[16], const AxisGeom& g, const Epi<float>& e,
                                                  const Chunk& ch, int s_off, int lane, double (&nrm)[3],
                                                  bool& bad) {
  const int p = ch.lt * 32 + lane;  // image row (m index)
  if (p >= g.other) return;
  const int n = g.len;
  const int q0 = ch.s0 + s_off;    // first n index
  const int cnt = min(16, ch.cnt - s_off);
  if (cnt <= 0) return;
  const long long base = (long long)ch.b * e.bstride + (long long)p * n + q0;
  if (e.foldH > 0) {
    const int FH = e.foldH;
    const float* fr = e.fold + ((long long)ch.b * g.other + p) * (2 * FH);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int q = q0 + j;
      if (j < cnt) {
        if (q < FH) acc[j] += fr[q];
        else if (q >= n - FH) acc[j] += fr[q - (n - 2 * FH)];
      }
    }
  }
  const bool vec = cnt == 16;  // q0 is a multiple of 8, rows are 16-byte aligned (n % 4 == 0)
  auto ld = [&](const float* a, float (&v)[16]) {
    if (vec) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float4 t = reinterpret_cast<const float4*>(a + base)[k];
        v[4 * k] = t.x; v[4 * k + 1] = t.y; v[4 * k + 2] = t.z; v[4 * k + 3] = t.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = j < cnt ? a[base + j] : 0.f;
    }
  };
  auto st = [&](float* a, const float (&v)[16]) {
    if (vec) {
#pragma unroll
      for (int k = 0; k < 4; ++k)
        reinterpret_cast<float4*>(a + base)[k] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < cnt) a[base + j] = v[j];
    }
  };
  if constexpr (MODE == EPI_PLAIN) {
    st(e.out, acc);
  } else if constexpr (MODE == EPI_RESID) {
    float bv[16];
    ld(e.bsub, bv);
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = __fsub_rn(acc[j], bv[j]);
    st(e.out, acc);
  } else if constexpr (MODE == EPI_UPDATE) {
    float yv[16], xp[16];
    ld(e.y, yv);
    ld(e.x, xp);
    const float Lt = (float)e.L[ch.b], dt = (float)e.denom[ch.b], bt = (float)e.beta;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      float xv = __fdiv_rn(__fsub_rn(__fmul_rn(Lt, yv[j]), acc[j]), dt);
      if (e.project) xv = (xv > 0.f || xv != xv) ? xv : 0.f;
      const float d = __fsub_rn(xv, xp[j]);
      if (j < cnt) {
        bad |= !isfinite(xv);
        if (e.want_norms) {
          nrm[0] += (double)d * d;
          nrm[1] += (double)xp[j] * xp[j];
          nrm[2] += (double)xv * xv;
        }
      }
      yv[j] = __fadd_rn(xv, __fmul_rn(bt, d));
      xp[j] = xv;
    }
    st(e.x, xp);
    st(e.y, yv);
  } else {  // EPI_POWER
    float vi[16];
    ld(e.vin, vi);
    const double vs = e.vnw2 ? sqrt(e.vnw2[ch.b]) : 1.0;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      if (j < cnt) {
        const double vv = e.vnw2 ? (double)vi[j] / vs : (double)vi[j];
        nrm[0] += vv * acc[j];
        nrm[1] += (double)acc[j] * acc[j];
      }
    }
    st(e.out, acc);
  }
}

template <int MODE>
__device__ __forceinline__ void kb_warp_finish_f(const Epi<float>& e, double (&nrm)[3], bool bad, int b,
                                                 int nslots, int slot, int lane) {
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

template <int MODE>
__global__ void __launch_bounds__(32 * kNW, 2)
kb_pass_sum_f(const __grid_constant__ CUtensorMap tmap, int r, const float* __restrict__ tin, long long t_bs,
              AxisGeom g, Epi<float> e, int batch, int parts) {
  extern __shared__ __align__(128) unsigned char kb_smem_f[];
  __shared__ unsigned long long full[kStages], empty[kStages];
  constexpr int TS = kNW * 16;
  const int rows_tile = TS + g.Wp;
  const TileBoxesF tb = tile_boxes_f(rows_tile);
  float* xs = reinterpret_cast<float*>(kb_smem_f);  // [kStages][stage_elems]
  float* cpad = xs + kStages * tb.stage_elems;       // [r][Wp]
  const int lane = threadIdx.x, warp = threadIdx.y;
  const int tid = warp * 32 + lane;
  const int LT = (g.other + 31) / 32;
  const int s_off = warp * 16;
  const int nslots = gridDim.x * kNW, slot = blockIdx.x * kNW + warp;

  if (tid == 0) {
    for (int st = 0; st < kStages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], kNW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  pdl_wait();  // launched with programmatic serialization: the previous kernel's outputs are read below

  ChunkWalk fill_walk(g.len, LT, parts, batch, 4), use_walk(g.len, LT, parts, batch, 4);
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
    const int st = nfill % kStages;
    if (nfill >= kStages) mbar_wait(&empty[st], ((nfill / kStages) - 1) & 1);
    mbar_arrive_expect_tx(&full[st], (unsigned)(tb.stage_elems * sizeof(float)));
    const int row0 = fc.s0 - g.H + g.halo_lo;  // halo_lo: reflected rows stored by the split pass
    for (int k = 0; k < tb.nbox; ++k)
      tma_load_3d(xs + st * tb.stage_elems + k * tb.box_rows * 32, &tmap, fc.lt * 32,
                  row0 + k * tb.box_rows, fc.b * r + fterm, &full[st]);
    ++fterm;
    ++nfill;
  };
  for (int k = 0; k < kStages - 1; ++k) issue();

  double nrm[3] = {0.0, 0.0, 0.0};
  bool bad = false;
  int norm_b = -1, taps_b = -1;
  Chunk ch;
  int t = 0;
  while (use_walk.next(ch, TS)) {
    if (ch.b != taps_b) {
      __syncthreads();
      const float* tbp = tin + ch.b * t_bs;
      for (int idx = tid; idx < r * g.Wp; idx += 32 * kNW) cpad[idx] = tbp[idx];
      __syncthreads();
      taps_b = ch.b;
    }
    if (ch.b != norm_b) {
      if (norm_b >= 0) kb_warp_finish_f<MODE>(e, nrm, bad, norm_b, nslots, slot, lane);
      nrm[0] = nrm[1] = nrm[2] = 0.0;
      bad = false;
      norm_b = ch.b;
    }
    float acc[1][16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[0][j] = 0.f;
    for (int term = 0; term < r; ++term, ++t) {
      issue();
      const int st = t % kStages;
      mbar_wait(&full[st], (t / kStages) & 1);
      const float* xt = xs + st * tb.stage_elems;
      if (s_off < ch.cnt && !(g.dbg & 1))
        kb_taps<float, 1, 16>(acc, xt + s_off * 32 + lane, cpad + term * g.Wp, 0, g.Wp);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
    if (s_off < ch.cnt && !(g.dbg & 2)) kb_sum_epilogue_f<MODE>(acc[0], g, e, ch, s_off, lane, nrm, bad);
  }
  if (norm_b >= 0) kb_warp_finish_f<MODE>(e, nrm, bad, norm_b, nslots, slot, lane);
}

}  // namespace kb
