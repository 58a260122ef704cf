// kb_tc1.cuh — tcgen05 sum pass with 128-output chunks and one tensor-memory accumulator per
// chunk across all r terms (fp32, 3xTF32).
//
// kb_pass_sum_tc (kb_tc.cuh) gives every (64-output chunk, term) its own accumulator slot and the
// epilogue warps add the r slots in fp32 registers: per term and output that is one tcgen05.ld
// (TMEM reads run at 64 B/clk per SM -- at cfg5 the slot reads of a chunk-term take ~500 cycles
// against ~580 of MMA work) and (64 + 2H)/64 converted input rows. Here a chunk is 128 outputs
// (8 N-blocks), the r terms accumulate in one 128-column accumulator (double-buffered across
// chunks: 2 x 128 columns + 8 A stages x 32 = 512), the epilogue reads it once, and a term
// converts (128 + 2H)/128 rows per output. The tensor core's own accumulation then spans all r
// terms: at cfg5 8.5e-6 of the full-length fixture. Wider bands chain more products per output
// (cfg4: 6.4e-5 with one accumulator, 4.9e-5 with SLOTS = 2, 3.4e-5 with kb_tc.cuh's per-term
// slots; tolerance 1e-4) and stay on the slot kernel unless KB_TC_SUM1=2.
//
// Warp roles: 0 TMA producer (term bricks + Z^T tiles); 1-4 MMA issuers (N-blocks w, w + 4);
// 5-12 two converter sets (alternate 32-row tiles); 13-20 epilogue (lane quarter x 64-output half).
#pragma once
#include "kb_tc.cuh"

namespace kb {

constexpr int kT1TS = 128;                       // outputs per chunk: 8 N-blocks of 16
constexpr int kT1Epi = 8;
constexpr int kT1EpiW = kTcConv + 8;             // first epilogue warp (after 2 converter sets)
constexpr int kT1Threads = 32 * (kT1EpiW + kT1Epi);
constexpr int kT1Stages = 8;                     // tensor-memory A stages at column 256

__host__ __device__ __forceinline__ int t1_ksteps(int Kw) { return (Kw + 126) / 8 + 1; }

// TMA-staged epilogue operands (TMAE): every epilogue warp owns 32 rows x 64 outputs of a chunk
// as two 32 x 32 boxes per operand plane (128-byte swizzled, 4 KB each), loaded by TMA while the
// chunk's r terms accumulate and stored back by TMA: the update's y / x (or the residual's B, the
// power step's v) no longer wait on global-load latency after the accumulator is ready.
// Planes per warp: UPDATE 2 (y, x: read and rewritten), RESID / POWER 1 (B / v, rewritten in place
// with R / w), PLAIN 1 (staging for the output).
template <int MODE>
__host__ __device__ constexpr int t1_planes() { return MODE == EPI_UPDATE ? 2 : 1; }
constexpr unsigned kT1Box = 32 * 32 * 4;
template <int MODE>
__host__ __device__ constexpr unsigned t1_ebuf_bytes() { return kT1Epi * t1_planes<MODE>() * 2 * kT1Box; }

// SLOTS = 1: one accumulator per chunk, double-buffered across chunks. SLOTS = 2 (wide bands,
// cfg4): two accumulators per chunk, terms [0, ceil(r/2)) and the rest, added in fp32 by the
// epilogue -- half the chained tensor-core accumulations per output -- single-buffered (the next
// chunk's first term waits for the epilogue to read both)
template <int MODE, bool NORMS = true, int SLOTS = 1, bool TMAE = false>
__global__ void __launch_bounds__(kT1Threads, 1)
kb_pass_sum_tc1(const __grid_constant__ CUtensorMap tmap, int r, const unsigned* __restrict__ btab, AxisGeom g,
                Epi<float> e, int batch, int nst, const __grid_constant__ CUtensorMap emap0,
                const __grid_constant__ CUtensorMap emap1) {
  extern __shared__ __align__(16) unsigned char kb_smem_tc[];
  __shared__ unsigned long long full[kTcRingMax], sfree[kTcRingMax], a_ready[kT1Stages], a_free[kT1Stages],
      acc_full[2], acc_empty[2], bready[2], bfree[2], eful[kT1Epi];
  __shared__ unsigned tmem_base;
  unsigned char* base = kb_smem_tc + ((1024 - (smem_u32(kb_smem_tc) & 1023)) & 1023);
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;
  const int LT = (g.other + 127) / 128;
  const int nk = t1_ksteps(g.Kw), nrb = (nk + 3) / 4, na = (nk + 1) / 2, nbr = tc_bricks(g.Kw);
  const int qmax = (g.Kw + 14) >> 3;
  const int acol = 256;  // A stages above the two accumulators
  float* stages = reinterpret_cast<float*>(base);                                  // [nst][32][128]
  unsigned* bricks = reinterpret_cast<unsigned*>(base + nst * kTcStageBytes);       // [2][nbr][256]
  // epilogue boxes (TMAE), 1 KB aligned for the 128-byte swizzle
  unsigned char* ebuf = base + (((size_t)nst * kTcStageBytes + 2 * (size_t)nbr * 1024 + 1023) & ~(size_t)1023);

  if (tid == 0) {
    for (int st = 0; st < nst; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&sfree[st], 4);
    }
    for (int st = 0; st < kT1Stages; ++st) {
      mbar_init(&a_ready[st], 4);
      mbar_init(&a_free[st], kTcIssuers);
    }
    for (int w = 0; w < kT1Epi; ++w) mbar_init(&eful[w], 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], kTcIssuers);
      mbar_init(&acc_empty[b], kT1Epi);
      mbar_init(&bready[b], 1);
      mbar_init(&bfree[b], kTcIssuers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
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
    // ---------------- TMA producer: per chunk and term the term's bricks and Z^T tiles ----------------
    if (lane == 0) {
      RingPos t;
      int tb = 0;
      const unsigned bbytes = (unsigned)nbr * 1024;
      StrideWalk walk(g.len, LT, batch, kT1TS);
      Chunk ch;
      while (walk.next(ch, kT1TS)) {
        for (int term = 0; term < r; ++term, ++tb) {
          const int bb = tb & 1;
          if (tb >= 2) mbar_wait_idle(&bfree[bb], ((tb >> 1) - 1) & 1, kTcSpinNs);
          mbar_arrive_expect_tx(&bready[bb], bbytes);
          bulk_g2s(bricks + bb * nbr * 256, btab + ((long long)ch.b * r + term) * nbr * 256, bbytes, &bready[bb]);
          for (int rb = 0; rb < nrb; ++rb, t.advance(nst)) {
            mbar_wait_idle(&sfree[t.i], t.phase ^ 1, kTcSpinNs);
            mbar_arrive_expect_tx(&full[t.i], kTcStageBytes);
            const int row0 = ch.s0 - g.H + g.halo_lo + kTcRB * rb;
            tma_load_3d(stages + t.i * (kTcStageBytes / 4), &tmap, ch.lt * 128, row0, ch.b * r + term, &full[t.i]);
          }
        }
      }
    }
  } else if (warp < kTcConv) {
    // ---------------- MMA issuers: N-blocks nb = w and w + 4 ----------------
    const int w = warp - 1;
    RingPos a;
    int tb = 0, chunk = 0;
    const unsigned long long b0 = tc_desc(smem_u32(bricks), 128, 256, 0);
    StrideWalk walk(g.len, LT, batch, kT1TS);
    Chunk ch;
    const int rh = (r + 1) / 2;
    while (walk.next(ch, kT1TS)) {
      const int ab = SLOTS == 1 ? chunk & 1 : 0;
      if (SLOTS == 1 && chunk >= 2) mbar_wait_lazy(&acc_empty[ab], ((chunk >> 1) - 1) & 1, kTcSpinNs);  // drained
      if (SLOTS == 2 && chunk >= 1) mbar_wait_lazy(&acc_empty[0], (chunk - 1) & 1, kTcSpinNs);
      for (int term = 0; term < r; ++term, ++tb) {
        const int slot = SLOTS == 1 ? ab : (term >= rh ? 1 : 0);
        const bool fresh = SLOTS == 1 ? term == 0 : (term == 0 || term == rh);
        const int bb = tb & 1;
        mbar_wait_lazy(&bready[bb], (tb >> 1) & 1, kTcSpinNs);
        __syncwarp();
        tc_fence_after();
        const unsigned long long bbase = b0 + ((unsigned)(bb * nbr) * 1024 >> 4);
        for (int ia = 0; ia < na; ++ia, a.advance(kT1Stages)) {
          mbar_wait_lazy(&a_ready[a.i], a.phase, kTcSpinNs);
          __syncwarp();
          tc_fence_after();
          const unsigned ahi = tmem + acol + a.i * 32;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int k = 2 * ia + h;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const int nb = w + 4 * j, q = k - 2 * nb;
              if (!(g.dbg & 1) && k < nk && q >= 0 && q <= qmax) {
                const unsigned long long bh = bbase + ((unsigned)q * 1024 >> 4);
                tc_mma3(tmem + slot * 128 + 16 * nb, ahi + 8 * h, ahi + 16 + 8 * h, bh, bh + (512 >> 4),
                        (!fresh || q != 0) ? 1u : 0u);
              }
            }
          }
          tc_commit_elect(&a_free[a.i]);
        }
        tc_commit_elect(&bfree[bb]);  // the brick buffer may be refilled
      }
      tc_commit_elect(&acc_full[ab]);  // the chunk's r terms are accumulated
      ++chunk;
    }
  } else if (warp < kT1EpiW) {
    // ---------------- converters: A stages (two sets, alternate tiles) ----------------
    const int wt = tid - 32 * kTcConv;  // 0..255
    const int cs = wt >> 7;
    const int q = warp & 3;
    const unsigned lane_base = tmem + ((unsigned)(32 * q) << 16);
    RingPos a, t;
    int tg = 0;
    StrideWalk walk(g.len, LT, batch, kT1TS);
    Chunk ch;
    while (walk.next(ch, kT1TS)) {
      for (int term = 0; term < r; ++term) {
        for (int rb = 0; rb < nrb; ++rb, ++tg, t.advance(nst)) {
          const int nat = min(2, na - 2 * rb);
          if ((tg & 1) != cs) {
            a.advance(kT1Stages);
            if (nat == 2) a.advance(kT1Stages);
            continue;
          }
          mbar_wait_lazy(&full[t.i], t.phase, kTcSpinNs);
          tc_fence_after();
          const float* tile = stages + t.i * (kTcStageBytes / 4) + 32 * q + lane;
          int st0 = a.i, st1 = -1;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (h == nat) break;
            if (h == 1) st1 = a.i;
            mbar_wait_lazy(&a_free[a.i], a.phase ^ 1, kTcSpinNs);
            __syncwarp();
            unsigned hi[16], lo[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float x = tile[(16 * h + i) * 128];
              hi[i] = __float_as_uint(x) & 0xffffe000u;
              lo[i] = __float_as_uint(x - __uint_as_float(hi[i]));
            }
            const unsigned ahi = lane_base + acol + a.i * 32;
            tc_st16(ahi, hi);
            tc_st16(ahi + 16, lo);
            a.advance(kT1Stages);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(&a_ready[st0]);
            if (st1 >= 0) mbar_arrive(&a_ready[st1]);
            mbar_arrive(&sfree[t.i]);
          }
        }
      }
    }
  } else if (!TMAE) {
    // ---------------- epilogue: the chunk's accumulated sum -> fused update of the output rows ----------------
    const int ew = warp - kT1EpiW, q = warp & 3, hh = ew >> 2;  // lane quarter, 64-output half
    const unsigned lane_base = tmem + ((unsigned)(32 * q) << 16);
    const int nslots = gridDim.x * kT1Epi, slot = blockIdx.x * kT1Epi + ew;
    const int n = g.len;
    double nrm[3] = {0.0, 0.0, 0.0};
    bool bad = false;
    int norm_b = -1, chunk = 0;
    StrideWalk walk(g.len, LT, batch, kT1TS);
    Chunk ch;
    while (walk.next(ch, kT1TS)) {
      if (ch.b != norm_b) {
        if (norm_b >= 0) kb_warp_finish_f<MODE>(e, nrm, bad, norm_b, nslots, slot, lane);
        nrm[0] = nrm[1] = nrm[2] = 0.0;
        bad = false;
        norm_b = ch.b;
      }
      const int ab = SLOTS == 1 ? chunk & 1 : 0;
      const int l = ch.lt * 128 + 32 * q + lane;
      const bool live = 64 * hh < ch.cnt && l < g.other;
      double sc_L = 0.0, sc_d = 1.0;
      if constexpr (MODE == EPI_UPDATE) {
        sc_L = e.L[ch.b];
        sc_d = e.denom[ch.b];
      }
      if constexpr (MODE == EPI_POWER) sc_L = e.vnw2 ? e.vnw2[ch.b] : 1.0;
      const long long row = (long long)ch.b * e.bstride + (long long)l * n + ch.s0 + 64 * hh;
      if (live) {  // operand rows to L2 while the chunk's r terms accumulate
#pragma unroll
        for (int c = 0; c < 64; c += 32) {
          if (64 * hh + c >= ch.cnt) break;
          if constexpr (MODE == EPI_RESID) prefetch_l2(e.bsub + row + c);
          if constexpr (MODE == EPI_UPDATE) {
            prefetch_l2(e.y + row + c);
            prefetch_l2(e.x + row + c);
          }
          if constexpr (MODE == EPI_POWER) prefetch_l2(e.vin + row + c);
        }
      }
      mbar_wait_lazy(&acc_full[ab], (SLOTS == 1 ? chunk >> 1 : chunk) & 1, 2000);
      __syncwarp();
      tc_fence_after();
      const float Lb = (float)sc_L, db = (float)sc_d, rd = 1.f / db;
      const double vs = MODE == EPI_POWER && e.vnw2 ? sqrt(sc_L) : 1.0;
      const bool fold_edge = e.foldH > 0 && (ch.s0 < e.foldH || ch.s0 + kT1TS > n - e.foldH);
#pragma unroll 1
      for (int p = 0; p < 4; ++p) {  // 16-output pieces of this warp's 64-output half
        const int o0 = 64 * hh + 16 * p;
        if (o0 >= ch.cnt) break;  // warp-uniform
        float v[16];
        tc_ld16(lane_base + ab * 128 + o0, v);
        if (SLOTS == 2 && r > (r + 1) / 2) {  // the second half of the terms, added in fp32
          float v1[16];
          tc_ld16(lane_base + 128 + o0, v1);
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = __fadd_rn(v[i], v1[i]);
        }
        if (live && !(g.dbg & 2)) {
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const int c = ch.cnt - o0 - 8 * j;
            if (c <= 0) break;
            float v8[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) v8[i] = v[8 * j + i];
            if (fold_edge) {  // exact adjoint fold corrections of the reflective axis (edge chunks)
              const int FH = e.foldH;
              const float* fz = e.fold + ((long long)ch.b * g.other + l) * (2 * FH);
#pragma unroll
              for (int i = 0; i < 8; ++i) {
                const int qi = ch.s0 + o0 + 8 * j + i;
                if (qi < FH) v8[i] += fz[qi];
                else if (qi >= n - FH && qi < n) v8[i] += fz[qi - (n - 2 * FH)];
              }
            }
            tc_sum_epi8<MODE, NORMS>(v8, e, row + 16 * p + 8 * j, min(8, c), Lb, db, rd, vs, nrm, bad);
          }
        }
        __syncwarp();  // reconverge before the next .sync.aligned tensor-memory load
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[ab]);
      ++chunk;
    }
    if (norm_b >= 0) kb_warp_finish_f<MODE>(e, nrm, bad, norm_b, nslots, slot, lane);
  } else {
    // ---------------- epilogue with TMA-staged operands (see t1_planes) ----------------
    constexpr int NPL = t1_planes<MODE>();
    const int ew = warp - kT1EpiW, q = warp & 3, hh = ew >> 2;  // lane quarter, 64-output half
    const unsigned lane_base = tmem + ((unsigned)(32 * q) << 16);
    const int nslots = gridDim.x * kT1Epi, slot = blockIdx.x * kT1Epi + ew;
    const int n = g.len;
    unsigned char* mybox = ebuf + (size_t)ew * NPL * 2 * kT1Box;  // [plane][box b]
    // the tensor maps by address in parameter space (a lambda capturing the __grid_constant__
    // parameters by reference could copy them to the stack, where TMA cannot read them)
    const CUtensorMap* pm0 = &emap0;
    const CUtensorMap* pm1 = &emap1;
    double nrm[3] = {0.0, 0.0, 0.0};
    bool bad = false;
    int norm_b = -1, chunk = 0;
    StrideWalk walk(g.len, LT, batch, kT1TS);
    // operand boxes of a chunk: rows lt*128 + 32q, columns s0 + 64hh + 32b, image plane b
    auto load_boxes = [&](const Chunk& c2) {
      if (MODE == EPI_PLAIN) return;
      if (lane == 0) {
        mbar_arrive_expect_tx(&eful[ew], NPL * 2 * kT1Box);
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          const int c0 = c2.s0 + 64 * hh + 32 * b, r0 = c2.lt * 128 + 32 * q;
          tma_load_3d(mybox + b * kT1Box, pm0, c0, r0, c2.b, &eful[ew]);
          if (NPL == 2) tma_load_3d(mybox + (2 + b) * kT1Box, pm1, c0, r0, c2.b, &eful[ew]);
        }
      }
    };
    {
      StrideWalk peek = walk;
      Chunk c2;
      if (peek.next(c2, kT1TS)) load_boxes(c2);
    }
    Chunk ch;
    while (walk.next(ch, kT1TS)) {
      if (ch.b != norm_b) {
        if (norm_b >= 0) kb_warp_finish_f<MODE>(e, nrm, bad, norm_b, nslots, slot, lane);
        nrm[0] = nrm[1] = nrm[2] = 0.0;
        bad = false;
        norm_b = ch.b;
      }
      const int ab = SLOTS == 1 ? chunk & 1 : 0;
      const int l = ch.lt * 128 + 32 * q + lane;
      const bool row_ok = l < g.other;
      double sc_L = 0.0, sc_d = 1.0;
      if constexpr (MODE == EPI_UPDATE) {
        sc_L = e.L[ch.b];
        sc_d = e.denom[ch.b];
      }
      if constexpr (MODE == EPI_POWER) sc_L = e.vnw2 ? e.vnw2[ch.b] : 1.0;
      if (MODE != EPI_PLAIN) mbar_wait_lazy(&eful[ew], chunk & 1, 2000);
      mbar_wait_lazy(&acc_full[ab], (SLOTS == 1 ? chunk >> 1 : chunk) & 1, 2000);
      __syncwarp();
      tc_fence_after();
      const float Lb = (float)sc_L, db = (float)sc_d, rd = 1.f / db;
      const double vs = MODE == EPI_POWER && e.vnw2 ? sqrt(sc_L) : 1.0;
      const float beta = (float)e.beta;
      const bool fold_edge = e.foldH > 0 && (ch.s0 < e.foldH || ch.s0 + kT1TS > n - e.foldH);
#pragma unroll 1
      for (int pc = 0; pc < 4; ++pc) {  // 16-output pieces: box b = pc >> 1, chunks 4 (pc & 1) ..
        const int o0 = 64 * hh + 16 * pc;
        if (o0 >= ch.cnt) break;  // warp-uniform
        float v[16];
        tc_ld16(lane_base + ab * 128 + o0, v);
        if (SLOTS == 2 && r > (r + 1) / 2) {
          float v1[16];
          tc_ld16(lane_base + 128 + o0, v1);
#pragma unroll
          for (int i = 0; i < 16; ++i) v[i] = __fadd_rn(v[i], v1[i]);
        }
        if (fold_edge && row_ok) {  // exact adjoint fold corrections of the reflective axis (edge chunks)
          const int FH = e.foldH;
          const float* fz = e.fold + ((long long)ch.b * g.other + l) * (2 * FH);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int qi = ch.s0 + o0 + i;
            if (qi < FH) v[i] += fz[qi];
            else if (qi >= n - FH && qi < n) v[i] += fz[qi - (n - 2 * FH)];
          }
        }
        if (!(g.dbg & 2)) {
          const int b = pc >> 1;
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {
            const int c16 = 4 * (pc & 1) + cc;  // 16-byte chunk of the box row
            const unsigned off = (unsigned)lane * 128 + (unsigned)((c16 ^ (lane & 7)) * 16);
            float4* p0 = reinterpret_cast<float4*>(mybox + b * kT1Box + off);
            const float* vv = v + 4 * cc;
            float4 a0 = *p0;
            float* u = reinterpret_cast<float*>(&a0);
            const int col0 = o0 + 4 * cc;
            if constexpr (MODE == EPI_PLAIN) {
              *p0 = make_float4(vv[0], vv[1], vv[2], vv[3]);
            } else if constexpr (MODE == EPI_RESID) {
              *p0 = make_float4(__fsub_rn(vv[0], u[0]), __fsub_rn(vv[1], u[1]), __fsub_rn(vv[2], u[2]),
                                __fsub_rn(vv[3], u[3]));
            } else if constexpr (MODE == EPI_UPDATE) {
              float4* p1 = reinterpret_cast<float4*>(mybox + (2 + b) * kT1Box + off);
              float4 a1 = *p1;
              float* w = reinterpret_cast<float*>(&a1);
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float a = __fsub_rn(__fmul_rn(Lb, u[i]), vv[i]);
                const float q0 = __fmul_rn(a, rd);
                float x = fmaf(fmaf(-db, q0, a), rd, q0);
                if (e.project) x = (x > 0.f || x != x) ? x : 0.f;
                const float d = __fsub_rn(x, w[i]);
                if (row_ok && col0 + i < ch.cnt) {
                  bad |= !isfinite(x);
                  if (NORMS && e.want_norms) {
                    nrm[0] += (double)d * d;
                    nrm[1] += (double)w[i] * w[i];
                    nrm[2] += (double)x * x;
                  }
                }
                u[i] = __fadd_rn(x, __fmul_rn(beta, d));  // y_{k+1} into the y box
                w[i] = x;                                  // x_k into the x box
              }
              *p0 = a0;
              *p1 = a1;
            } else {  // EPI_POWER: w (the application) into the v box, <v, w> and ||w||^2
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                if (row_ok && col0 + i < ch.cnt) {
                  const double vvv = e.vnw2 ? (double)u[i] / vs : (double)u[i];
                  nrm[0] += vvv * vv[i];
                  nrm[1] += (double)vv[i] * vv[i];
                }
              }
              *p0 = make_float4(vv[0], vv[1], vv[2], vv[3]);
            }
          }
        }
        __syncwarp();  // reconverge before the next .sync.aligned tensor-memory load
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[ab]);  // tensor memory read: the next chunk may accumulate
      // results back to global memory from the boxes (rows / columns past the plane are clipped)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0 && !(g.dbg & 2)) {
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          const int c0 = ch.s0 + 64 * hh + 32 * b, r0 = ch.lt * 128 + 32 * q;
          if (64 * hh + 32 * b >= ch.cnt) break;
          if constexpr (MODE == EPI_UPDATE) {
            tma_store_3d(pm0, mybox + b * kT1Box, c0, r0, ch.b);        // y
            tma_store_3d(pm1, mybox + (2 + b) * kT1Box, c0, r0, ch.b);  // x
          } else if constexpr (MODE == EPI_PLAIN) {
            tma_store_3d(pm0, mybox + b * kT1Box, c0, r0, ch.b);
          } else {
            tma_store_3d(pm1, mybox + b * kT1Box, c0, r0, ch.b);
          }
        }
        bulk_commit();
        bulk_wait_read<0>();  // the boxes may be refilled
      }
      __syncwarp();
      {
        StrideWalk peek = walk;
        Chunk c2;
        if (peek.next(c2, kT1TS)) load_boxes(c2);
      }
      ++chunk;
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores complete
    if (norm_b >= 0) kb_warp_finish_f<MODE>(e, nrm, bad, norm_b, nslots, slot, lane);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

}  // namespace kb
