// kb_tc.cuh — fp32 split pass on the 5th-generation tensor cores (tcgen05.mma kind::tf32, 3xTF32).
//
// The same banded GEMM as the other split passes, Z_i^T[l][s] = sum_t X[t][l] c_i[t - s] for a
// 128-column L-tile (M = 128) and 16-output N-blocks, accumulated in tensor memory:
//   A = X^T from tensor memory: the natural [rows][cols] input tile is streamed by TMA in 32-row
//       blocks; worker warps (lane = column) split each value into tf32 hi + lo and store them to an
//       A stage in tensor memory (lane = column, column = K). With A read from shared memory the
//       operand traffic of 16-wide MMAs bounds the tensor core at ~1/4 of its rate (ncu: 57% of the
//       shared-memory bandwidth at 9% tensor activity).
//   B = Toeplitz bricks: for N-block nb and K-step k the 16 x 8 operand B[n][kk] = taps[8k + kk -
//       16nb - n] depends only on o = 8k - 16nb, so each term keeps (Kw+14)/8 + 1 bricks (hi and lo,
//       K-major INTERLEAVE core matrices) in shared memory.
//   D = tensor memory: one 16-column accumulator per (term, N-block) of the chunk; every term
//       accumulates only its own K-range (the 3xTF32 products of one output stay in one accumulator,
//       33-35 K-steps at the widest BASELINE band).
// Warp roles: warp 0 streams the tile (TMA); warps 1-12 each issue the MMAs of one (term, N-block)
// accumulator (one thread each: a single issuing thread serialises its MMAs, ~120 cycles each on
// the box, so twelve streams feed the tensor core; warp 1 owns the tensor memory); warps 13-16
// (converters) split the tiles into A stages and rebuild the bricks when the image or term group
// changes; warps 17-20 run the epilogue (tcgen05.ld -> swizzled staging -> TMA store of Z^T) on
// the other of two accumulator sets while the next chunk's MMAs run. Zero boundary conditions
// only (no edge folds); the reflect-filled split takes the mma.sync kernels.
#pragma once
#include "kb_tf32.cuh"

namespace kb {

constexpr int kTcTS = 64;        // outputs (S rows) per chunk: 4 N-blocks of 16
constexpr int kTcRB = 32;        // input rows per ring stage (4 K-steps)
constexpr int kTcStagesMax = 8;  // tensor-memory A stages (2 K-steps: hi 16 + lo 16 columns each)
constexpr int kTcRingMax = 8;    // shared-memory tile ring depth (runtime nst <= this)
constexpr int kTcG = 3;          // terms per group (two accumulator sets of kTcG x 64 columns)
constexpr int kTcIssuers = 4;    // one MMA-issuing warp per N-block
constexpr int kTcConv = 1 + kTcIssuers, kTcEpi = kTcConv + 8;  // first converter / epilogue warp
constexpr int kTcThreads = 32 * (kTcEpi + 4);  // TMA warp, issuers, 2 x 4 converters, 4 epilogue warps
constexpr unsigned kTcStageBytes = kTcRB * 128 * 4;  // one [32 rows][128 cols] fp32 tile
// tensor memory: two accumulator sets of G x 64 columns, then the A stages
__host__ __device__ __forceinline__ int tc_astages(int G) { return min(kTcStagesMax, (512 - 128 * G) / 32); }
constexpr unsigned kTcStoreBytes = 4 * 2 * 4096;  // epilogue staging: 4 warps x 2 buffers x [32 L][32 S]
// dynamic shared memory: [staging][tile ring][bricks][tap scratch] (1 KB alignment slack in front)
__host__ __device__ __forceinline__ unsigned tc_tap_bytes(int G, int Kw) { return (G * Kw * 4 + 1023) & ~1023u; }

__host__ __device__ __forceinline__ int tc_ksteps(int Kw) { return (Kw + 62) / 8 + 1; }
__host__ __device__ __forceinline__ int tc_bricks(int Kw) { return (Kw + 14) / 8 + 1; }

__device__ __forceinline__ unsigned long long tc_desc(unsigned addr, unsigned lbo, unsigned sbo, unsigned layout) {
  unsigned long long d = (unsigned long long)((addr >> 4) & 0x3FFF);
  d |= (unsigned long long)((lbo >> 4) & 0x3FFF) << 16;
  d |= (unsigned long long)((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;  // descriptor version (sm_100)
  d |= (unsigned long long)(layout & 7) << 61;
  return d;
}
// kind::tf32, D f32, A from tensor memory, B K-major, M = 128, N = 16
constexpr unsigned kTcIdesc = (1u << 4) | (2u << 7) | (2u << 10) | (2u << 17) | (8u << 24);

// Profiling (KB_DEBUG_MODE bit 7): per-role stall cycles into kb_trace[0][block][slot]:
// 0 producer waiting for free tiles, 1/2 converters waiting for A stages / tiles, 3 epilogue
// waiting for the accumulators, 4 epilogue busy, 5/6 issuer 0 waiting for drained accumulators /
// A stages, 7 converter-0 kernel cycles.
struct TcProf {
  bool on;
  unsigned long long acc = 0, t0 = 0;
  __device__ TcProf(const AxisGeom& g, bool me) : on((g.dbg & 128) && me && blockIdx.x < kTraceBlocks) {}
  __device__ __forceinline__ void start() { if (on) t0 = clock64(); }
  __device__ __forceinline__ void stop() { if (on) acc += clock64() - t0; }
  __device__ __forceinline__ void put(int slot) { if (on) kb_trace[0][blockIdx.x][slot] = acc; }
};

// ring position: slot index and the parity of the current lap. Waiting on a consumer-release
// barrier with parity (phase ^ 1) passes at once on the first lap (fresh barrier).
struct RingPos {
  int i = 0;
  unsigned phase = 0;
  __device__ __forceinline__ void advance(int n) {
    if (++i == n) {
      i = 0;
      phase ^= 1;
    }
  }
};

// one 3xTF32 K-step, issued by one elected lane of a converged warp: D (+)= lo*hi + hi*lo + hi*hi
__device__ __forceinline__ void tc_mma3(unsigned d, unsigned ahi, unsigned alo, unsigned long long bh,
                                        unsigned long long bl, unsigned acc) {
  asm volatile(
      "{\n.reg .pred p, q;\nsetp.ne.b32 q, %6, 0;\nelect.sync _|p, 0xffffffff;\n"
      "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%2], %3, %5, q;\n"
      "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %4, %5, 1;\n"
      "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %3, %5, 1;\n}" ::"r"(d),
      "r"(ahi), "r"(alo), "l"(bh), "l"(bl), "r"(kTcIdesc), "r"(acc));
}
// the same K-step for three terms (accumulators d, d + 64, d + 128; bricks bh + j * bstep)
__device__ __forceinline__ void tc_mma3x3(unsigned d, unsigned ahi, unsigned alo, unsigned long long bh,
                                          unsigned long long bstep, unsigned acc) {
  const unsigned long long bh1 = bh + bstep, bh2 = bh1 + bstep, lo = 512 >> 4;
  asm volatile(
      "{\n.reg .pred p, q;\nsetp.ne.b32 q, %9, 0;\nelect.sync _|p, 0xffffffff;\n"
      "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%4], %5, %11, q;\n"
      "@p tcgen05.mma.cta_group::1.kind::tf32 [%1], [%4], %6, %11, q;\n"
      "@p tcgen05.mma.cta_group::1.kind::tf32 [%2], [%4], %7, %11, q;\n"
      "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%3], %8, %11, 1;\n"
      "@p tcgen05.mma.cta_group::1.kind::tf32 [%1], [%3], %10, %11, 1;\n"
      "@p tcgen05.mma.cta_group::1.kind::tf32 [%2], [%3], %12, %11, 1;\n"
      "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%3], %5, %11, 1;\n"
      "@p tcgen05.mma.cta_group::1.kind::tf32 [%1], [%3], %6, %11, 1;\n"
      "@p tcgen05.mma.cta_group::1.kind::tf32 [%2], [%3], %7, %11, 1;\n}" ::"r"(d),
      "r"(d + 64), "r"(d + 128), "r"(ahi), "r"(alo), "l"(bh), "l"(bh1), "l"(bh2), "l"(bh + lo), "r"(acc),
      "l"(bh1 + lo), "r"(kTcIdesc), "l"(bh2 + lo));
}
__device__ __forceinline__ void tc_commit_elect(unsigned long long* bar) {
  asm volatile(
      "{\n.reg .pred p;\nelect.sync _|p, 0xffffffff;\n"
      "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(smem_u32(bar))
      : "memory");
}
// TMA store of a shared-memory box to `map` at (c0, c1, c2); completion tracked by bulk groups
__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(map),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_ld16(unsigned addr, float (&v)[16]) {
  unsigned u[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7]), "=r"(u[8]),
        "=r"(u[9]), "=r"(u[10]), "=r"(u[11]), "=r"(u[12]), "=r"(u[13]), "=r"(u[14]), "=r"(u[15])
      : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(u[i]);
}
__device__ __forceinline__ void tc_st16(unsigned addr, const unsigned (&u)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          addr),
      "r"(u[0]), "r"(u[1]), "r"(u[2]), "r"(u[3]), "r"(u[4]), "r"(u[5]), "r"(u[6]), "r"(u[7]), "r"(u[8]), "r"(u[9]),
      "r"(u[10]), "r"(u[11]), "r"(u[12]), "r"(u[13]), "r"(u[14]), "r"(u[15]));
}

// Tensor-core split pass. Work: (image b, 128-column L-tile, S-part) items walked in 64-output
// chunks, once per group of G terms (bricks of a group stay resident; the tile is re-streamed per
// group). Stage flow: TMA -> shared tile [32 rows][128 cols] -> workers (lane = column) split each
// value into tf32 hi + lo and store them to a tensor-memory A stage (lane = column, 32 + 32
// columns = K) -> MMAs (A from tensor memory, so the only shared-memory operand traffic is the 512-B
// bricks). bricks: [G][nbr][hi 512 B | lo 512 B]. Results leave
// through a 128-byte-swizzled [32 L][32 S] staging box per worker warp and a TMA store (zmap:
// Z^T planes b * r + term), so every global write is a full line; ragged chunk ends store directly.
__global__ void __launch_bounds__(kTcThreads, 1)
kb_pass_split_tc(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap zmap,
                 float* __restrict__ z, long long z_ps, long long z_bs,
                 const float* __restrict__ tin, long long t_bs, AxisGeom g, const double* __restrict__ nw2, int r,
                 int batch, int parts, int G, int nst) {
  extern __shared__ __align__(1024) unsigned char kb_smem_tc[];
  __shared__ unsigned long long full[kTcRingMax], sfree[kTcRingMax], a_ready[kTcStagesMax],
      a_free[kTcStagesMax], acc_full[2], acc_empty[2];
  __shared__ unsigned tmem_base;
  __shared__ long long stamp_issue[kTcStagesMax], stamp_ready[kTcStagesMax];  // KB_DEBUG_MODE bit 9
  const bool lat = (g.dbg & 512) && blockIdx.x < kTraceBlocks;
  unsigned char* base = kb_smem_tc + ((1024 - (smem_u32(kb_smem_tc) & 1023)) & 1023);
  float* staging = reinterpret_cast<float*>(base);  // [4 warps][2][32][32], 128-byte swizzled rows
  float* stages = reinterpret_cast<float*>(base + kTcStoreBytes);  // [nst][32][128]
  unsigned* bricks = reinterpret_cast<unsigned*>(base + kTcStoreBytes + nst * kTcStageBytes);
  // warp index and tensor-memory base through a lane-0 shuffle: provably warp-uniform, so the MMA
  // operands are computed in uniform registers (no per-MMA register-to-uniform moves)
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;
  const int LT = (g.other + 127) / 128;
  const int nk = tc_ksteps(g.Kw), nrb = (nk + 3) / 4, na = (nk + 1) / 2, nbr = tc_bricks(g.Kw);
  const int ngroups = (r + G - 1) / G;
  const int nas = tc_astages(G), acol = 128 * G;  // A stages at columns acol + 32 st
  float* taps_s = reinterpret_cast<float*>(bricks + G * nbr * 256);  // [G][Kw]

  if (tid == 0) {
    for (int st = 0; st < nst; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&sfree[st], 8);
    }
    for (int st = 0; st < nas; ++st) {
      mbar_init(&a_ready[st], 4);
      mbar_init(&a_free[st], kTcIssuers);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], kTcIssuers);
      mbar_init(&acc_empty[b], 4);
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
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      TcProf pw(g, true);
      RingPos t;
      for (int gr = 0; gr < ngroups; ++gr) {
        ChunkWalk walk(g.len, LT, parts, batch, 4);
        Chunk ch;
        while (walk.next(ch, kTcTS)) {
          for (int rb = 0; rb < nrb; ++rb, t.advance(nst)) {
            pw.start();
            mbar_wait(&sfree[t.i], t.phase ^ 1);
            pw.stop();
            mbar_arrive_expect_tx(&full[t.i], kTcStageBytes);
            const int row0 = ch.s0 - g.H + g.halo_lo + kTcRB * rb;
            tma_load_3d(stages + t.i * (kTcStageBytes / 4), &tmap, ch.lt * 128, row0, ch.b, &full[t.i]);
          }
        }
      }
    }
  } else if (warp < kTcConv) {
    // ---------------- MMA issuers: one warp per (term, N-block) accumulator ----------------
    // the whole warp walks the loop (warp-uniform operands); one elected lane issues
    const int nb = warp - 1;
    TcProf pe(g, warp == 1 && lane == 0), pa(g, warp == 1 && lane == 0);
    RingPos a;
    int chunk = 0;
    long long lat_wake = 0, lat_n = 0;
    // brick descriptors advance by adding (bytes >> 4) to the start-address field
    const unsigned long long b0 = tc_desc(smem_u32(bricks), 128, 256, 0);
    const int qmax = (g.Kw + 14) >> 3;
    for (int gr = 0; gr < ngroups; ++gr) {
      const int g0 = gr * G, gc = min(G, r - g0);
      const bool live = !(g.dbg & 1);
      ChunkWalk walk(g.len, LT, parts, batch, 4);
      Chunk ch;
      while (walk.next(ch, kTcTS)) {
        const int ab = chunk & 1;
        pe.start();
        if (chunk >= 2) mbar_wait(&acc_empty[ab], ((chunk >> 1) - 1) & 1);  // epilogue drained this set
        __syncwarp();
        pe.stop();
        tc_fence_after();
        const unsigned dcol = tmem + ab * 64 * G + nb * 16;
        for (int ia = 0; ia < na; ++ia, a.advance(nas)) {
          const int st = a.i;
          pa.start();
          mbar_wait(&a_ready[st], a.phase);  // A stage (and, at a group change, bricks) ready
          __syncwarp();  // reconverge: elect.sync below must see the whole warp
          pa.stop();
          if (lat && warp == 1 && lane == 0) {
            lat_wake += clock64() - stamp_ready[st];
            ++lat_n;
          }
          if (!(g.dbg & 8)) tc_fence_after();
          const unsigned ahi = tmem + acol + st * 32;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int k = 2 * ia + h, q = k - 2 * nb;  // brick index o / 8 with o = 8k - 16nb
            if (live && k < nk && q >= 0 && q <= qmax) {
              if (gc == 3) {
                const unsigned long long bh = b0 + ((unsigned)q * 1024 >> 4);
                tc_mma3x3(dcol, ahi + 8 * h, ahi + 16 + 8 * h, bh, (unsigned)nbr * 1024 >> 4, q != 0);
                continue;
              }
#pragma unroll
              for (int gi = 0; gi < kTcG; ++gi) {
                if (gi >= gc) break;
                const unsigned long long bh = b0 + ((unsigned)(gi * nbr + q) * 1024 >> 4);
                tc_mma3(dcol + gi * kTcTS, ahi + 8 * h, ahi + 16 + 8 * h, bh, bh + (512 >> 4), q != 0);
              }
            }
          }
          tc_commit_elect(&a_free[st]);  // the A stage can be refilled once these MMAs have read it
          if (lat && warp == 1 && lane == 0) stamp_issue[st] = clock64();
        }
        tc_commit_elect(&acc_full[ab]);
        ++chunk;
      }
    }
    if (!(g.dbg & 256)) pa.put(6);
    if (lat && warp == 1 && lane == 0) {
      kb_trace[0][blockIdx.x][4] = lat_wake;
      kb_trace[0][blockIdx.x][6] = lat_n;
    }
  } else if (warp < kTcEpi) {
    // ---------------- converters: bricks and A stages ----------------
    // two sets of four warps (one per tensor-memory lane quarter) take alternate A stages
    const int wt = tid - 32 * kTcConv;  // 0..255
    const int cs = wt >> 7;
    const int q = warp & 3;             // tensor-memory lane quarter this warp may access
    const unsigned lane_base = tmem + ((unsigned)(32 * q) << 16);
    TcProf p1(g, wt == 0), p2(g, wt == 0), pt(g, wt == 0), pc(g, wt == 0), ps(g, wt == 0), pb(g, wt == 0), pm(g, wt == 0), pr(g, wt == 0);
    pt.start();
    RingPos a, t;
    int chunk = 0, bricks_key = -1;
    long long lat_mma = 0;
    for (int gr = 0; gr < ngroups; ++gr) {
      const int g0 = gr * G, gc = min(G, r - g0);
      ChunkWalk walk(g.len, LT, parts, batch, 4);
      Chunk ch;
      while (walk.next(ch, kTcTS)) {
        const int key = ch.b * ngroups + gr;
        if (key != bricks_key) {
          pb.start();
          // the previous chunk's MMAs (the last readers of the old bricks) must have completed
          if (chunk > 0) mbar_wait(&acc_full[(chunk - 1) & 1], ((chunk - 1) >> 1) & 1);
          // taps -> shared scratch (independent loads), then bricks from the scratch
          const float* tb = tin + ch.b * t_bs + (long long)g0 * g.Wp;
#pragma unroll 4
          for (int idx = wt; idx < gc * g.Kw; idx += 256) {
            const int gg = idx / g.Kw;
            taps_s[idx] = tb[(long long)gg * g.Wp + (idx - gg * g.Kw)];
          }
          asm volatile("bar.sync 1, 256;" ::: "memory");
          for (int idx = wt; idx < gc * nbr * 128; idx += 256) {
            const int gg = idx / (nbr * 128), rem = idx - gg * nbr * 128, qb = rem >> 7, e = rem & 127;
            const int nn = e >> 3, kk = e & 7;  // B[n][kk]
            const int ti = 8 * qb + kk - nn;
            const float c = (ti >= 0 && ti < g.Kw) ? taps_s[gg * g.Kw + ti] : 0.f;
            unsigned h, l;
            tf32_split_rn(c, h, l);
            // K-major INTERLEAVE: core (n/8, kk/4) at (n/8)*256 + (kk/4)*128, row n%8 at 16 B
            const int off = ((nn >> 3) * 64 + (kk >> 2) * 32 + (nn & 7) * 4 + (kk & 3));
            unsigned* bp = bricks + (gg * nbr + qb) * 256;
            bp[off] = h;
            bp[128 + off] = l;
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          asm volatile("bar.sync 1, 256;" ::: "memory");  // all bricks written before any a_ready
          bricks_key = key;
          pb.stop();
        }
        // A stages (16 tile rows each): column 32q + lane of each row -> tensor-memory lane, K -> column.
        // Set cs converts the stages with n % 2 == cs; both sets release every tile once.
        for (int ia = 0; ia < na; ++ia, a.advance(nas)) {
          const int ts = t.i;
          pm.start();
          if ((a.i & 1) == cs) {  // nas is even: stage parity alternates with the global stage count
            const int st = a.i;
            p1.start();
            mbar_wait(&a_free[st], a.phase ^ 1);
            p1.stop();
            if (lat && wt == 0 && a.phase) lat_mma += clock64() - stamp_issue[st];
            p2.start();
            mbar_wait(&full[ts], t.phase);
            p2.stop();
            if (!(g.dbg & 8)) tc_fence_after();
            const float* tile = stages + ts * (kTcStageBytes / 4) + (ia & 1) * 16 * 128 + 32 * q + lane;
            const unsigned ahi = lane_base + acol + st * 32;
            pc.start();
            if (!(g.dbg & 4)) {
              unsigned hi[16], lo[16];
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                const float x = tile[i * 128];
                hi[i] = __float_as_uint(x) & 0xffffe000u;
                lo[i] = __float_as_uint(x - __uint_as_float(hi[i]));
              }
              tc_st16(ahi, hi);
              tc_st16(ahi + 16, lo);
            }
            pc.stop();
            ps.start();
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            ps.stop();
            if (!(g.dbg & 8)) tc_fence_before();
            if (!(g.dbg & 16)) __syncwarp();
            if (lat && (wt & 127) == 0) stamp_ready[st] = clock64();
            if (lane == 0) mbar_arrive(&a_ready[st]);
          }
          pm.stop();
          pr.start();
          if ((ia & 1) || ia == na - 1) {  // this set is done with the tile: TMA may refill it
            __syncwarp();
            if (lane == 0) mbar_arrive(&sfree[ts]);
            t.advance(nst);
          }
          pr.stop();
        }
        ++chunk;
      }
    }
    pt.stop();
    p1.put(1);
    p2.put(2);
    pc.put(0);
    ps.put(5);
    pb.put(3);
    if (lat && wt == 0) kb_trace[0][blockIdx.x][3] = lat_mma;
    if (g.dbg & 256) {
      pm.put(4);
      pr.put(6);
    }
    pt.put(7);
  } else {
    // ---------------- epilogue: accumulators -> Z^T rows ----------------
    const int q = warp & 3;
    const unsigned lane_base = tmem + ((unsigned)(32 * q) << 16);
    TcProf p3(g, warp == kTcEpi && lane == 0), p4(g, warp == kTcEpi && lane == 0);
    int chunk = 0, nstore = 0;
    for (int gr = 0; gr < ngroups; ++gr) {
      const int g0 = gr * G, gc = min(G, r - g0);
      ChunkWalk walk(g.len, LT, parts, batch, 4);
      Chunk ch;
      while (walk.next(ch, kTcTS)) {
        const int ab = chunk & 1;
        p3.start();
        mbar_wait(&acc_full[ab], (chunk >> 1) & 1);
        p3.stop();
        p4.start();
        tc_fence_after();
        const int l0 = ch.lt * 128 + 32 * q, l = l0 + lane;
        const float oscale = nw2 ? (float)(1.0 / sqrt(nw2[ch.b])) : 1.f;
        for (int gg = 0; gg < gc; ++gg) {
          float* zp = z + ch.b * z_bs + (long long)(g0 + gg) * z_ps + (long long)l * g.len + ch.s0;
          for (int h = 0; h < kTcTS / 32; ++h) {
            const int s = 32 * h;
            if (s >= ch.cnt) break;
            float va[16], vb[16];
            const unsigned col = lane_base + ab * 64 * G + gg * kTcTS + 32 * h;
            if (!(g.dbg & 32)) {
              tc_ld16(col, va);
              tc_ld16(col + 16, vb);
            } else {
#pragma unroll
              for (int i = 0; i < 16; ++i) va[i] = vb[i] = 0.f;
            }
            if (g.dbg & 2) continue;
            float v[32];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              v[i] = va[i] * oscale;
              v[16 + i] = vb[i] * oscale;
            }
            if (s + 32 <= ch.cnt) {
              // swizzled staging row `lane`: 16-byte chunk c at position c ^ (lane & 7)
              if (nstore >= 2 && lane == 0) bulk_wait_read<1>();
              __syncwarp();
              float* sb = staging + (2 * q + (nstore & 1)) * 1024;
#pragma unroll
              for (int c = 0; c < 8; ++c)
                reinterpret_cast<float4*>(sb + lane * 32)[c ^ (lane & 7)] =
                    make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              __syncwarp();
              if (lane == 0) {
                tma_store_3d(&zmap, sb, ch.s0 + s, l0, ch.b * r + g0 + gg);
                bulk_commit();
              }
              ++nstore;
            } else if (l < g.other) {
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (s + i < ch.cnt) zp[s + i] = v[i];
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[ab]);
        p4.stop();
        ++chunk;
      }
    }
    if (lane == 0) bulk_wait_read<0>();  // staging must outlive the TMA stores' reads
    if (!(g.dbg & 768)) p4.put(4);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

}  // namespace kb
