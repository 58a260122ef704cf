// kb_fused.cuh — one-sweep operator application on the tcgen05 tensor cores (fp32, 3xTF32).
//
// The two-sweep passes (kb_tc.cuh) write the r intermediate planes Z_i^T = (H_i X)^T to HBM in
// pass A and read them back in pass B: at cfg5 that round trip is ~45 GB of DRAM traffic per
// iteration against ~9 GB compulsory. This kernel runs both passes of one application
// (kron.py:218-225 forward, :228-235 adjoint) per output tile with the intermediate tile kept on
// chip:
//
//   output tile  = 128 rows [l0, l0+128) x C columns [c0, c0+C)   (C = 16 * nblk <= 96)
//   pass A (axis 0, lanes = columns): Z_i[l][t] for the tile's rows and the C + 2Hb columns
//       t in [c0-Hb, c0-Hb+128) that pass B reads -- the same MMA as kb_pass_split_tc
//       (M = 128 columns, N = 16 rows per N-block, 8 N-blocks, K = 8 input rows, A = the X tile
//       transposed in tensor memory by the converter warps, B = Toeplitz bricks), accumulated in
//       a double-buffered 128 x 128 tensor-memory accumulator;
//   hand-off: four drain warps move the accumulator (lane = column t) into a [t][l] shared tile
//       (16-byte chunks XOR-swizzled by t & 7, conflict-free both ways), then read it back with
//       lane = row l, split into tf32 hi + lo and store pass B's A stages to tensor memory;
//   pass B (axis 1, lanes = rows): Y[l][s] += sum_t Z_i[l][t] d_i[t - s] into one 128 x C
//       accumulator that collects all r terms;
//   epilogue: the sum pass' fused epilogues (PLAIN / RESID / UPDATE / POWER, tc_sum_epi8).
//
// The X tile (128 + 2Ha rows x 128 columns, <= 6 TMA stages of 32 rows) stays resident in shared
// memory for all r terms of a tile; only the bricks change per term. Reflective axes fill the
// out-of-domain rows / columns of the tile from the folded source (times the term's fill sign
// for the symmetric adjoint), so Z's halo columns come out reflected exactly as the two-sweep
// split pass stores them. Exact (non-symmetric) adjoint folds are not handled here (host
// selection falls back to the two-sweep passes).
//
// Warp roles (20 warps): 0 TMA producer (X stages, bricks); 1-2 pass-A MMA issuers (N-blocks
// 0-3 / 4-7); 3 pass-B MMA issuer; 4-7 X converters (lane quarters); 8-11 drain + Z converters;
// 12-19 epilogue (lane quarter x column half).
#pragma once
#include "kb_tc.cuh"

namespace kb {

constexpr int kFuL = 128;        // output rows per tile (pass-A outputs, pass-B lanes)
#ifndef KB_FU_SA
#define KB_FU_SA 3
#endif
#ifndef KB_FU_SB
#define KB_FU_SB 2
#endif
constexpr int kFuSA = KB_FU_SA;  // pass-A A stages (tensor memory, 2 K-steps each)
constexpr int kFuSB = KB_FU_SB;  // pass-B A stages
constexpr int kFuXStMax = 6;     // resident 32-row X stages per tile
constexpr int kFuNbMax = 6;      // pass-B N-blocks per tile (96 output columns)
constexpr int kFuAccA = 0;       // tensor-memory columns: pass-A accumulators (2 x 128)
constexpr int kFuAccB = 256;     //   pass-B accumulator (<= 96)
constexpr int kFuStA = 352;      //   pass-A A stages (3 x 32)
constexpr int kFuStB = 448;      //   pass-B A stages (2 x 32)
constexpr int kFuWIssA = 1, kFuWIssB = 3, kFuWConvX = 4, kFuWDrain = 8, kFuWEpi = 12;
constexpr int kFuEpi = 8;
constexpr int kFuThreads = 32 * (kFuWEpi + kFuEpi);
constexpr unsigned kFuZsBytes = 128u * 128u * 4u;  // the [t][l] hand-off tile

struct FuGeom {
  int len;          // local rows of the block (axis 0)
  int n;            // columns (axis 1)
  int Ha, Hb;
  int nbr_a, nbr_b;  // bricks per term
  int qmax_a, qmax_b;
  int na_a;          // pass-A A stages per term
  int nxs;           // 32-row X stages per tile
  int nblk;          // pass-B N-blocks of a full chunk
  int nchunks, LT;   // column chunks per row tile, row tiles
  int fill_a, fill_b;
  int g0, Mg, halo_lo, halo_hi;  // axis-0 block geometry (single image: 0, len, 0, 0)
  unsigned sa_neg;   // bit i: term i's axis-0 fill sign is -1 (symmetric adjoint)
  int dbg;
};

struct FuTile {
  int b, l0, c0, nblk, cnt;
};

// Tiles dealt round-robin over the CTAs, column chunk fastest: the CTAs running together hold
// neighbouring chunks of one row band, so the X halo columns / rows one CTA loads were just
// fetched into L2 by its neighbours. Chunks split the N-blocks of a row evenly.
struct FuWalk {
  int k, total;
  __device__ FuWalk(const FuGeom& f, int batch) : k(blockIdx.x), total(batch * f.LT * f.nchunks) {}
  __device__ bool next(FuTile& t, const FuGeom& f) {
    if (k >= total) return false;
    const int cj = k % f.nchunks, rest = k / f.nchunks;
    t.l0 = (rest % f.LT) * kFuL;
    t.b = rest / f.LT;
    const int NB = (f.n + 15) >> 4;
    const int lo = (int)((long long)NB * cj / f.nchunks), hi = (int)((long long)NB * (cj + 1) / f.nchunks);
    t.c0 = 16 * lo;
    t.nblk = hi - lo;
    t.cnt = min(16 * t.nblk, f.n - t.c0);
    k += gridDim.x;
    return true;
  }
};

__device__ __forceinline__ int fu_nab(const FuGeom& f, int nblk) {  // pass-B A stages of a tile
  return (2 * (nblk - 1) + f.qmax_b + 2) >> 1;
}

// out-of-domain entry of the X tile on a reflective axis: the folded source times the fill
// signs (zero where the fold leaves the domain or the axis has zero boundary conditions)
__device__ __forceinline__ float fu_edge(const float* __restrict__ in, long long img, int lr, int col,
                                         const FuGeom& f, float sa, float sb, float tile_v) {
  const int gr = f.g0 + lr;
  const bool rin = gr >= 0 && gr < f.Mg, cin = col >= 0 && col < f.n;
  if (rin && cin) return tile_v;
  float s = 1.f;
  int rr = gr, cc = col;
  if (!rin) {
    if (!f.fill_a) return 0.f;
    rr = kb_fold(gr, f.Mg);
    s = sa;
  }
  if (!cin) {
    if (!f.fill_b) return 0.f;
    cc = kb_fold(col, f.n);
    s *= sb;
  }
  const int lrr = rr - f.g0;
  if (rr < 0 || cc < 0 || lrr < -f.halo_lo || lrr >= f.len + f.halo_hi) return 0.f;
  return s * in[img + (long long)lrr * f.n + cc];
}

__device__ __forceinline__ void tc_ld32(unsigned addr, float (&v)[32]) {
  unsigned u[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]),
        "=r"(u[8]), "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]), "=r"(u[14]), "=r"(u[15]),
        "=r"(u[16]), "=r"(u[17]), "=r"(u[18]), "=r"(u[19]), "=r"(u[20]), "=r"(u[21]), "=r"(u[22]), "=r"(u[23]),
        "=r"(u[24]), "=r"(u[25]), "=r"(u[26]), "=r"(u[27]), "=r"(u[28]), "=r"(u[29]), "=r"(u[30]), "=r"(u[31])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(u[i]);
}

__device__ __forceinline__ void fu_named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <int MODE, bool NORMS = true>
__global__ void __launch_bounds__(kFuThreads, 1)
kb_fused_tc(const __grid_constant__ CUtensorMap xmap, const float* __restrict__ in, long long in_bs,
            const unsigned* __restrict__ btab_a, const unsigned* __restrict__ btab_b, FuGeom f,
            const float* __restrict__ sb_tab, const double* __restrict__ nw2, Epi<float> e, int r, int batch) {
  extern __shared__ __align__(16) unsigned char kb_smem_fu[];
  __shared__ unsigned long long xfull[kFuXStMax], xfree[kFuXStMax], a_ready[kFuSA], a_free[kFuSA],
      b_ready[kFuSB], b_free[kFuSB], accA_full[2], accA_empty[2], accB_full, accB_empty, bready[2], bfree[2];
  __shared__ unsigned tmem_base;
  unsigned char* base = kb_smem_fu + ((1024 - (smem_u32(kb_smem_fu) & 1023)) & 1023);
  float* xs = reinterpret_cast<float*>(base);                                  // [nxs][32][128]
  float* zs = reinterpret_cast<float*>(base + (size_t)f.nxs * kTcStageBytes);  // [128 t][128 l]
  unsigned* bricks = reinterpret_cast<unsigned*>(base + (size_t)f.nxs * kTcStageBytes + kFuZsBytes);
  const unsigned bterm = (unsigned)(f.nbr_a + f.nbr_b) * 1024;  // one term's bricks: [A bricks][B bricks]
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;

  if (tid == 0) {
    for (int j = 0; j < f.nxs; ++j) {
      mbar_init(&xfull[j], 1);
      mbar_init(&xfree[j], 4);
    }
    for (int s = 0; s < kFuSA; ++s) {
      mbar_init(&a_ready[s], 4);
      mbar_init(&a_free[s], 2);
    }
    for (int s = 0; s < kFuSB; ++s) {
      mbar_init(&b_ready[s], 4);
      mbar_init(&b_free[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&accA_full[i], 2);
      mbar_init(&accA_empty[i], 4);
      mbar_init(&bready[i], 1);
      mbar_init(&bfree[i], 3);
    }
    mbar_init(&accB_full, 1);
    mbar_init(&accB_empty, kFuEpi);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kFuWIssA) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned tmem = __shfl_sync(0xffffffffu, tmem_base, 0);
  pdl_launch_dependents();
  pdl_wait();

  if (warp == 0) {
    // ---------------- producer: per tile the resident X stages, per term the bricks ----------------
    if (lane == 0) {
      FuWalk walk(f, batch);
      FuTile t;
      int T = 0, u = 0;
      auto load_bricks = [&](const FuTile& tt, int term) {
        const int bb = u & 1;
        if (u >= 2) mbar_wait_idle(&bfree[bb], ((u >> 1) - 1) & 1, kTcSpinNs);
        mbar_arrive_expect_tx(&bready[bb], bterm);
        unsigned char* dst = reinterpret_cast<unsigned char*>(bricks) + bb * bterm;
        const long long bt = (long long)tt.b * r + term;
        bulk_g2s(dst, btab_a + bt * f.nbr_a * 256, (unsigned)f.nbr_a * 1024, &bready[bb]);
        bulk_g2s(dst + (size_t)f.nbr_a * 1024, btab_b + bt * f.nbr_b * 256, (unsigned)f.nbr_b * 1024, &bready[bb]);
        ++u;
      };
      while (walk.next(t, f)) {
        load_bricks(t, 0);
        for (int j = 0; j < f.nxs; ++j) {
          if (T >= 1) mbar_wait_idle(&xfree[j], (T - 1) & 1, kTcSpinNs);
          mbar_arrive_expect_tx(&xfull[j], kTcStageBytes);
          tma_load_3d(xs + j * (kTcStageBytes / 4), &xmap, t.c0 - f.Hb, t.l0 - f.Ha + f.halo_lo + 32 * j, t.b,
                      &xfull[j]);
        }
        for (int term = 1; term < r; ++term) load_bricks(t, term);
        ++T;
      }
    }
  } else if (warp < kFuWIssB) {
    // ---------------- pass-A MMA issuers: N-blocks 4w .. 4w+3 of the 128 tile rows ----------------
    const int w = warp - kFuWIssA;
    const unsigned long long b0 = tc_desc(smem_u32(bricks), 128, 256, 0);
    const bool live = !(f.dbg & 1);
    FuWalk walk(f, batch);
    FuTile t;
    RingPos a;
    int u = 0;
    while (walk.next(t, f)) {
      for (int term = 0; term < r; ++term, ++u) {
        const int ab = u & 1, bb = u & 1;
        if (u >= 2) mbar_wait(&accA_empty[ab], ((u >> 1) - 1) & 1);  // drained two terms ago
        mbar_wait(&bready[bb], (u >> 1) & 1);
        __syncwarp();
        tc_fence_after();
        const unsigned dcol = tmem + kFuAccA + ab * 128;
        const unsigned long long bbase = b0 + ((unsigned)bb * bterm >> 4);
        for (int ia = 0; ia < f.na_a; ++ia, a.advance(kFuSA)) {
          mbar_wait(&a_ready[a.i], a.phase);
          __syncwarp();
          tc_fence_after();
          const unsigned ahi = tmem + kFuStA + a.i * 32;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int k = 2 * ia + h;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int nb = 4 * w + j, q = k - 2 * nb;
              if (live && q >= 0 && q <= f.qmax_a) {
                const unsigned long long bh = bbase + ((unsigned)q * 1024 >> 4);
                tc_mma3(dcol + 16 * nb, ahi + 8 * h, ahi + 16 + 8 * h, bh, bh + (512 >> 4), q != 0);
              }
            }
          }
          tc_commit_elect(&a_free[a.i]);
        }
        tc_commit_elect(&accA_full[ab]);
        tc_commit_elect(&bfree[bb]);
      }
    }
  } else if (warp == kFuWIssB) {
    // ---------------- pass-B MMA issuer: one accumulator over all r terms ----------------
    const unsigned long long b0 = tc_desc(smem_u32(bricks), 128, 256, 0);
    const bool live = !(f.dbg & 1);
    FuWalk walk(f, batch);
    FuTile t;
    RingPos s;
    int u = 0, T = 0;
    while (walk.next(t, f)) {
      const int nab = fu_nab(f, t.nblk);
      for (int term = 0; term < r; ++term, ++u) {
        const int bb = u & 1;
        if (term == 0 && T >= 1) mbar_wait(&accB_empty, (T - 1) & 1);  // epilogue read the previous tile
        mbar_wait(&bready[bb], (u >> 1) & 1);
        __syncwarp();
        tc_fence_after();
        const unsigned long long bbase = b0 + ((unsigned)(bb * bterm + f.nbr_a * 1024) >> 4);
        for (int ib = 0; ib < nab; ++ib, s.advance(kFuSB)) {
          mbar_wait(&b_ready[s.i], s.phase);
          __syncwarp();
          tc_fence_after();
          const unsigned ahi = tmem + kFuStB + s.i * 32;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int k = 2 * ib + h;
            for (int nb = 0; nb < t.nblk; ++nb) {
              const int q = k - 2 * nb;
              if (live && q >= 0 && q <= f.qmax_b) {
                const unsigned long long bh = bbase + ((unsigned)q * 1024 >> 4);
                tc_mma3(tmem + kFuAccB + 16 * nb, ahi + 8 * h, ahi + 16 + 8 * h, bh, bh + (512 >> 4),
                        (term > 0 || q != 0) ? 1u : 0u);
              }
            }
          }
          tc_commit_elect(&b_free[s.i]);
        }
        tc_commit_elect(&bfree[bb]);
        if (term == r - 1) tc_commit_elect(&accB_full);
      }
      ++T;
    }
  } else if (warp < kFuWDrain) {
    // ---------------- X converters: resident X stages -> pass-A A stages (lane = column) ----------------
    const int q = warp & 3, tcol = 32 * q + lane;
    const unsigned lane_base = tmem + ((unsigned)(32 * q) << 16);
    FuWalk walk(f, batch);
    FuTile t;
    RingPos a;
    int T = 0;
    while (walk.next(t, f)) {
      const int col = t.c0 - f.Hb + tcol;
      const bool cedge = f.fill_b && (t.c0 - f.Hb < 0 || t.c0 - f.Hb + 128 > f.n);
      const long long img = (long long)t.b * in_bs;
      for (int term = 0; term < r; ++term) {
        const float sa = (f.sa_neg >> term) & 1 ? -1.f : 1.f;
        const float sb = sb_tab ? sb_tab[(long long)t.b * r + term] : 1.f;
        int ia = 0;
        for (int j = 0; j < f.nxs && ia < f.na_a; ++j) {
          if (term == 0) mbar_wait(&xfull[j], T & 1);
          const float* tile = xs + j * (kTcStageBytes / 4) + tcol;
          int st0 = -1, st1 = -1;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (ia >= f.na_a) break;
            (h == 0 ? st0 : st1) = a.i;
            mbar_wait(&a_free[a.i], a.phase ^ 1);
            __syncwarp();  // reconverge before the .sync.aligned tensor-memory stores
            const int lr0 = t.l0 - f.Ha + 32 * j + 16 * h;  // local row of the half's first row
            const bool redge = f.fill_a && (f.g0 + lr0 < 0 || f.g0 + lr0 + 16 > f.Mg);
            float xv[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) xv[i] = tile[(16 * h + i) * 128];
            if (redge || cedge) {
#pragma unroll
              for (int i = 0; i < 16; ++i) xv[i] = fu_edge(in, img, lr0 + i, col, f, sa, sb, xv[i]);
            }
            unsigned hi[16], lo[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              hi[i] = __float_as_uint(xv[i]) & 0xffffe000u;
              lo[i] = __float_as_uint(xv[i] - __uint_as_float(hi[i]));
            }
            const unsigned ahi = lane_base + kFuStA + a.i * 32;
            if (!(f.dbg & 4)) {
              tc_st16(ahi, hi);
              tc_st16(ahi + 16, lo);
            }
            a.advance(kFuSA);
            ++ia;
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(&a_ready[st0]);
            if (st1 >= 0) mbar_arrive(&a_ready[st1]);
            if (term == r - 1) mbar_arrive(&xfree[j]);  // the stage's last reader this tile
          }
        }
      }
      ++T;
    }
  } else if (warp < kFuWEpi) {
    // ---------------- drain (lane = column t) + Z converters (lane = row l) ----------------
    const int q = warp & 3, tt = 32 * q + lane, l = tt;
    const unsigned lane_base = tmem + ((unsigned)(32 * q) << 16);
    FuWalk walk(f, batch);
    FuTile t;
    RingPos s;
    int u = 0;
    float4* zrow = reinterpret_cast<float4*>(zs + tt * 128);
    while (walk.next(t, f)) {
      const int nab = fu_nab(f, t.nblk);
      const float oscale = nw2 ? (float)(1.0 / sqrt(nw2[t.b])) : 1.f;
      for (int term = 0; term < r; ++term, ++u) {
        const int ab = u & 1;
        mbar_wait(&accA_full[ab], (u >> 1) & 1);
        __syncwarp();
        tc_fence_after();
        fu_named_sync(1, 128);  // every Z converter of the previous term has read zs
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float v[32];
          if (!(f.dbg & 8)) {
            tc_ld32(lane_base + kFuAccA + ab * 128 + 32 * j, v);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0.f;
          }
#pragma unroll
          for (int c = 0; c < 8; ++c)
            zrow[(8 * j + c) ^ (tt & 7)] =
                make_float4(v[4 * c] * oscale, v[4 * c + 1] * oscale, v[4 * c + 2] * oscale, v[4 * c + 3] * oscale);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&accA_empty[ab]);
        fu_named_sync(1, 128);  // zs complete
        __syncwarp();
        for (int ib = 0; ib < nab; ++ib, s.advance(kFuSB)) {
          mbar_wait(&b_free[s.i], s.phase ^ 1);
          __syncwarp();
          unsigned hi[16], lo[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int tr = 16 * ib + i;
            const float z = zs[tr * 128 + (((l >> 2) ^ (tr & 7)) << 2) + (l & 3)];
            hi[i] = __float_as_uint(z) & 0xffffe000u;
            lo[i] = __float_as_uint(z - __uint_as_float(hi[i]));
          }
          const unsigned ahi = lane_base + kFuStB + s.i * 32;
          if (!(f.dbg & 16)) {
            tc_st16(ahi, hi);
            tc_st16(ahi + 16, lo);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&b_ready[s.i]);
        }
      }
    }
  } else {
    // ---------------- epilogue: the tile's accumulated sum -> fused update of the output rows ----------------
    const int ew = warp - kFuWEpi, q = warp & 3, hh = ew >> 2;  // lane quarter, 48-column half
    const unsigned lane_base = tmem + ((unsigned)(32 * q) << 16);
    const int nslots = gridDim.x * kFuEpi, slot = blockIdx.x * kFuEpi + ew;
    const int n = f.n;
    double nrm[3] = {0.0, 0.0, 0.0};
    bool bad = false;
    int norm_b = -1, T = 0;
    FuWalk walk(f, batch);
    FuTile t;
    while (walk.next(t, f)) {
      if (t.b != norm_b) {
        if (norm_b >= 0) kb_warp_finish_f<MODE>(e, nrm, bad, norm_b, nslots, slot, lane);
        nrm[0] = nrm[1] = nrm[2] = 0.0;
        bad = false;
        norm_b = t.b;
      }
      const int l = t.l0 + 32 * q + lane;
      const int cbeg = 48 * hh, cend = min(cbeg + 48, 16 * t.nblk);
      double sc_L = 0.0, sc_d = 1.0;
      if constexpr (MODE == EPI_UPDATE) {
        sc_L = e.L[t.b];
        sc_d = e.denom[t.b];
      }
      if constexpr (MODE == EPI_POWER) sc_L = e.vnw2 ? e.vnw2[t.b] : 1.0;
      const long long row = (long long)t.b * e.bstride + (long long)l * n + t.c0;
      {  // operand rows to L2 while the tile's r terms accumulate
        if (cbeg < t.cnt && l < f.len) {
          const long long at = row + cbeg;
          if constexpr (MODE == EPI_RESID) prefetch_l2(e.bsub + at);
          if constexpr (MODE == EPI_UPDATE) {
            prefetch_l2(e.y + at);
            prefetch_l2(e.x + at);
          }
          if constexpr (MODE == EPI_POWER) prefetch_l2(e.vin + at);
        }
      }
      mbar_wait_idle(&accB_full, T & 1, 2000);
      __syncwarp();
      tc_fence_after();
      float v[48];
#pragma unroll
      for (int p = 0; p < 3; ++p) {
        if (cbeg + 16 * p < cend && !(f.dbg & 32)) {
          float w[16];
          tc_ld16(lane_base + kFuAccB + cbeg + 16 * p, w);
#pragma unroll
          for (int i = 0; i < 16; ++i) v[16 * p + i] = w[i];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&accB_empty);
      if (l < f.len && !(f.dbg & 2)) {
        const float Lb = (float)sc_L, db = (float)sc_d, rd = 1.f / db;
        const double vs = MODE == EPI_POWER && e.vnw2 ? sqrt(sc_L) : 1.0;
#pragma unroll
        for (int j = 0; j < 6; ++j) {
          const int c = min(cend, t.cnt) - cbeg - 8 * j;
          if (c <= 0) break;
          float v8[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) v8[i] = v[8 * j + i];
          tc_sum_epi8<MODE, NORMS>(v8, e, row + cbeg + 8 * j, min(8, c), Lb, db, rd, vs, nrm, bad);
        }
      }
      ++T;
    }
    if (norm_b >= 0) kb_warp_finish_f<MODE>(e, nrm, bad, norm_b, nslots, slot, lane);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kFuWIssA) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

}  // namespace kb
