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
//       (rows padded to 132 floats, conflict-free both ways), then read it back with
//       lane = row l, split into tf32 hi + lo and store pass B's A stages to tensor memory -- into
//       a 4-slot ring inside the accumulator buffer they just drained, so pass A's next-but-one
//       term reuses the buffer once pass B has consumed those stages;
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
// Warp roles (27 warps): 0 TMA producer (X stages, bricks); 1-4 pass-A MMA issuers (two N-blocks
// each); 5-6 pass-B MMA issuers (alternate N-blocks); 7-14 X converters (two sets of four lane
// quarters, one per 16-row half of an X stage); 15-22 drain + Z converters (two sets: half the
// drained columns and alternate pass-B stages each); 23-26 epilogue (one per lane quarter). Tensor memory: 2 x 128 pass-A accumulator columns (pass-B stages once drained), 96
// pass-B accumulator columns, 5 x 32 pass-A stage columns.
#pragma once
#include "kb_tc.cuh"

namespace kb {

constexpr int kFuL = 128;        // output rows per tile (pass-A outputs, pass-B lanes)
#ifndef KB_FU_SA
#define KB_FU_SA 5
#endif
#ifndef KB_FU_SB
#define KB_FU_SB 4
#endif
constexpr int kFuSA = KB_FU_SA;  // pass-A A stages (tensor memory, 2 K-steps each)
constexpr int kFuSB = KB_FU_SB;  // pass-B A-stage slots inside a drained pass-A accumulator buffer
constexpr int kFuXStMax = 6;     // resident 32-row X stages per tile
constexpr int kFuNbMax = 6;      // pass-B N-blocks per tile (96 output columns)
#ifndef KB_FU_ACCA
#define KB_FU_ACCA 0
#define KB_FU_ACCB 256
#endif
constexpr int kFuAccA = KB_FU_ACCA;  // tensor-memory columns: pass-A accumulators (2 x 128; once a buffer
                                 //   is drained, its columns hold that term's pass-B A stages)
constexpr int kFuAccB = KB_FU_ACCB;  // pass-B accumulator (<= 96)
constexpr int kFuStA = 352;      //   pass-A A stages (5 x 32)
static_assert(kFuStA + 32 * kFuSA <= 512 && 32 * kFuSB <= 128, "tensor-memory budget");
constexpr int kFuXSets = 2;      // X converter sets
// MMA issuers: one warp issues a kind::tf32 MMA every ~27 cycles at best (tools/tc_rate.cu,
// three MMAs per elect), the N = 16 MMA takes 8 -- so pass A gets four issuing warps (two
// N-blocks each) and pass B two (alternate N-blocks)
#ifndef KB_FU_ISSB
#define KB_FU_ISSB 2
#endif
constexpr int kFuIssA = 4, kFuIssB = KB_FU_ISSB;
constexpr int kFuDSets = 2;      // drain / Z converter sets (64 drain columns and alternate stages each)
constexpr int kFuWIssA = 1, kFuWIssB = kFuWIssA + kFuIssA, kFuWConvX = kFuWIssB + kFuIssB,
              kFuWDrain = kFuWConvX + 4 * kFuXSets, kFuWEpi = kFuWDrain + 4 * kFuDSets;
constexpr int kFuEpi = 4;        // epilogue warps (one per lane quarter, 32 columns per round)
constexpr int kFuThreads = 32 * (kFuWEpi + kFuEpi);
// the [t][l] hand-off tile: rows padded to 132 floats (528 B = 33 x 16 B), so the drain's float4
// stores (lane = row t: 8 lanes per phase land on 8 distinct 16-byte bank groups) and the Z
// converters' loads (lane = column l, consecutive words) are both conflict-free without index math
constexpr int kFuZsStride = 132;
constexpr unsigned kFuZsBytes = 128u * kFuZsStride * 4u;

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

// Per-role wait / busy cycles of block < kTraceBlocks into kb_trace[slot >> 3][block][slot & 7]
// (compiled in with -DKB_FU_PROF=1; tools/fu_profile.py reads them back):
//  0 pass-A issuer a_ready wait   1 pass-A issuer acc/brick wait   2 pass-B issuer b_ready wait
//  3 pass-B issuer acc/brick wait 4 X converter a_free wait        5 X converter xfull wait
//  6 drain accA_full wait         7 Z converter b_free wait        8 drain tcgen05.ld + st.shared
//  9 drain named-barrier waits    10 epilogue accB_full wait       11 X converter total
//  12 X converter busy            13 Z converter busy              14 epilogue busy
//  15 producer waits
#ifndef KB_FU_PROF
#define KB_FU_PROF 0
#endif
#ifndef KB_FU_NOLDS
#define KB_FU_NOLDS 0  // profiling: X converters skip their shared-memory loads
#endif
struct FuProf {
  unsigned long long acc = 0, t0 = 0;
  bool on;
  __device__ explicit FuProf(bool me) : on(KB_FU_PROF && me && blockIdx.x < kTraceBlocks) {}
  __device__ __forceinline__ void start() { if (KB_FU_PROF && on) t0 = clock64(); }
  __device__ __forceinline__ void stop() { if (KB_FU_PROF && on) acc += clock64() - t0; }
  __device__ __forceinline__ void put(int slot) { if (KB_FU_PROF && on) kb_trace[slot >> 3][blockIdx.x][slot & 7] = acc; }
};

// one kind::tf32 MMA (A from tensor memory, B K-major bricks) issued by one elected lane
__device__ __forceinline__ void tc_mma1(unsigned d, unsigned a, unsigned long long b, unsigned acc) {
  asm volatile(
      "{\n.reg .pred p, q;\nsetp.ne.b32 q, %4, 0;\nelect.sync _|p, 0xffffffff;\n"
      "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, q;\n}" ::"r"(d),
      "r"(a), "l"(b), "r"(kTcIdesc), "r"(acc));
}

// Event timeline of block 0 (-DKB_FU_TRACE=1): clock64 of event `ev` of term u < 1024 into the
// flat kb_trace array at ev * 1024 + u (tools/fu_timeline.py). Events: 0 pass-A issuer 0 starts
// a term, 1 it committed the term, 2 drain has the accumulator, 3 drain done, 4 Z converter set 0
// done, 5 pass-B issuer 0 has the first stage, 6 pass-B issuer 0 committed the term, 7 X converter
// set 0 first stage of the term converted, 8 its last stage converted.
#ifndef KB_FU_TRACE
#define KB_FU_TRACE 0
#endif
__device__ __forceinline__ void fu_ev(int ev, int u, bool me) {
  if (KB_FU_TRACE && me && blockIdx.x == 0 && u < 1024)
    (&kb_trace[0][0][0])[ev * 1024 + u] = clock64();
}
// per-stage events (terms u < 32, stage < 16) at 9216 + ev * 512 + 16 u + stage: 0 X stage
// stored, 1 pass-A issuer 0 has it, 2 issuer 0 committed it, 3 Z stage stored, 4 pass-B issuer 0
// has it, 5 it committed it, 6 its first MMA issued, 7 its last MMA issued
__device__ __forceinline__ void fu_sev(int ev, int u, int st, bool me) {
  if (KB_FU_TRACE && me && blockIdx.x == 0 && u < 32 && st < 16)
    (&kb_trace[0][0][0])[9216 + ev * 512 + 16 * u + st] = clock64();
}

// the fused kernel's barrier waits: a suspend-time hint (KB_FU_WAIT_NS, 0 = plain spin) lets a
// waiting warp leave its issue slots to the working warps of its SM sub-partition
#ifndef KB_FU_WAIT_NS
#define KB_FU_WAIT_NS 0
#endif
__device__ __forceinline__ void fu_wait(unsigned long long* bar, unsigned parity) {
  if (KB_FU_WAIT_NS > 0) mbar_wait_lazy(bar, parity, KB_FU_WAIT_NS);
  else mbar_wait(bar, parity);
}
// waits off the critical path (producer, epilogue): suspended in try_wait (KB_FU_IDLE_NS hint)
// rather than polling, so they leave the issue slots to the working warps
#ifndef KB_FU_IDLE_NS
#define KB_FU_IDLE_NS 20000
#endif
__device__ __forceinline__ void fu_wait_idle(unsigned long long* bar, unsigned parity) {
  mbar_wait_lazy(bar, parity, KB_FU_IDLE_NS);
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
      b_ready[2][kFuSB], b_free[2][kFuSB], accA_full[2], accA_empty[2], accB_full, accB_empty, bready[2], bfree[2];
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
      mbar_init(&xfree[j], 4 * kFuXSets);
    }
    for (int s = 0; s < kFuSA; ++s) {
      mbar_init(&a_ready[s], 4);
      mbar_init(&a_free[s], kFuIssA);
    }
    for (int i = 0; i < 2; ++i) {
      for (int s = 0; s < kFuSB; ++s) {
        mbar_init(&b_ready[i][s], 4);
        mbar_init(&b_free[i][s], kFuIssB);
      }
      mbar_init(&accA_full[i], kFuIssA);
      mbar_init(&accA_empty[i], kFuIssB);
      mbar_init(&bready[i], 1);
      mbar_init(&bfree[i], kFuIssA + kFuIssB);
    }
    mbar_init(&accB_full, kFuIssB);
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
      FuProf p15(true);
      int T = 0, u = 0;
      auto load_bricks = [&](const FuTile& tt, int term) {
        const int bb = u & 1;
        p15.start();
        if (u >= 2) fu_wait_idle(&bfree[bb], ((u >> 1) - 1) & 1);
        p15.stop();
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
          p15.start();
          if (T >= 1) fu_wait_idle(&xfree[j], (T - 1) & 1);
          p15.stop();
          mbar_arrive_expect_tx(&xfull[j], kTcStageBytes);
          tma_load_3d(xs + j * (kTcStageBytes / 4), &xmap, t.c0 - f.Hb, t.l0 - f.Ha + f.halo_lo + 32 * j, t.b,
                      &xfull[j]);
        }
        for (int term = 1; term < r; ++term) load_bricks(t, term);
        ++T;
      }
      p15.put(15);
    }
  } else if (warp < kFuWIssB) {
    // ---------------- pass-A MMA issuers: N-blocks 2w, 2w+1 of the 128 tile rows ----------------
    const int w = warp - kFuWIssA;
    const unsigned long long b0 = tc_desc(smem_u32(bricks), 128, 256, 0);
    const bool live = !(f.dbg & 1) && !(f.dbg & 64);  // bit 6: pass-A MMAs off (profiling)
    FuWalk walk(f, batch);
    FuTile t;
    RingPos a;
    FuProf p0(w == 0 && lane == 0), p1(w == 0 && lane == 0), m0(w == 0 && lane == 0), m1(w == 0 && lane == 0);
    int u = 0;
    while (walk.next(t, f)) {
      for (int term = 0; term < r; ++term, ++u) {
        const int ab = u & 1, bb = u & 1;
        p1.start();
        // buffer ab was last used by term u - 2: drained, and its pass-B stages consumed
        if (u >= 2) fu_wait(&accA_empty[ab], ((u >> 1) - 1) & 1);
        fu_wait(&bready[bb], (u >> 1) & 1);
        p1.stop();
        fu_ev(0, u, w == 0 && lane == 0);
        __syncwarp();
        tc_fence_after();
        const unsigned dcol = tmem + kFuAccA + ab * 128;
        const unsigned long long bbase = b0 + ((unsigned)bb * bterm >> 4);
        for (int ia = 0; ia < f.na_a; ++ia, a.advance(kFuSA)) {
          p0.start();
          fu_wait(&a_ready[a.i], a.phase);
          p0.stop();
          fu_sev(1, u, ia, w == 0 && lane == 0);
          __syncwarp();
          tc_fence_after();
          const unsigned ahi = tmem + kFuStA + a.i * 32;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int k = 2 * ia + h;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const int nb = 2 * w + j, q = k - 2 * nb;
              if (live && q >= 0 && q <= f.qmax_a) {
                const unsigned long long bh = bbase + ((unsigned)q * 1024 >> 4);
                if (KB_FU_PROF == 3) m0.start();
                tc_mma3(dcol + 16 * nb, ahi + 8 * h, ahi + 16 + 8 * h, bh, bh + (512 >> 4), q != 0);
                if (KB_FU_PROF == 3) {
                  m0.stop();
                  ++m1.acc;
                }
              }
            }
          }
          tc_commit_elect(&a_free[a.i]);
          fu_sev(2, u, ia, w == 0 && lane == 0);
        }
        tc_commit_elect(&accA_full[ab]);
        fu_ev(1, u, w == 0 && lane == 0);
        tc_commit_elect(&bfree[bb]);
      }
    }
    if (KB_FU_PROF == 3) {
      m0.put(0);
      m1.put(1);
    } else {
      p0.put(0);
      p1.put(1);
    }
  } else if (warp < kFuWConvX) {
    // ---------------- pass-B MMA issuers: one accumulator over all r terms; warp w2 takes the
    // N-blocks nb = w2 (mod 2) ----------------
    // A stages: a ring of kFuSB 32-column slots inside term u's drained pass-A buffer (u & 1)
    const unsigned long long b0 = tc_desc(smem_u32(bricks), 128, 256, 0);
    const bool live = !(f.dbg & 1) && !(f.dbg & 512);  // bit 9: pass-B MMAs off (profiling)
    FuWalk walk(f, batch);
    FuTile t;
    RingPos sb0, sb1;  // per-buffer ring positions (scalars: a runtime-indexed array would live in local memory)
    const int w2 = warp - kFuWIssB;
    FuProf p2(w2 == 0 && lane == 0), p3(w2 == 0 && lane == 0), m2(w2 == 0 && lane == 0), m3(w2 == 0 && lane == 0);
    int u = 0, T = 0;
    while (walk.next(t, f)) {
      const int nab = fu_nab(f, t.nblk);
      for (int term = 0; term < r; ++term, ++u) {
        const int ab = u & 1, bb = u & 1;
        RingPos s = ab ? sb1 : sb0;
        p3.start();
        if (term == 0 && T >= 1) fu_wait(&accB_empty, (T - 1) & 1);  // epilogue read the previous tile
        fu_wait(&bready[bb], (u >> 1) & 1);
        p3.stop();
        __syncwarp();
        tc_fence_after();
        const unsigned long long bbase = b0 + ((unsigned)(bb * bterm + f.nbr_a * 1024) >> 4);
        for (int ib = 0; ib < nab; ++ib, s.advance(kFuSB)) {
          p2.start();
          fu_wait(&b_ready[ab][s.i], s.phase);
          p2.stop();
          if (ib == 0) fu_ev(5, u, w2 == 0 && lane == 0);
          fu_sev(4, u, ib, w2 == 0 && lane == 0);
          __syncwarp();
          tc_fence_after();
          const unsigned ahi = tmem + kFuAccA + ab * 128 + s.i * 32;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int k = 2 * ib + h;
            // N-blocks nb = w2 + kFuIssB j of this issuer, fully unrolled like the pass-A issuers so
            // the MMA operands stay in uniform registers
#pragma unroll
            for (int j = 0; j < (kFuNbMax + kFuIssB - 1) / kFuIssB; ++j) {
              const int nb = w2 + kFuIssB * j, q = k - 2 * nb;
              if (live && nb < t.nblk && q >= 0 && q <= f.qmax_b) {
                const unsigned long long bh = bbase + ((unsigned)q * 1024 >> 4);
                if (KB_FU_PROF == 3) m2.start();
                tc_mma3(tmem + kFuAccB + 16 * nb, ahi + 8 * h, ahi + 16 + 8 * h, bh, bh + (512 >> 4),
                        (term > 0 || q != 0) ? 1u : 0u);
                if (h == 0 && j == 0) fu_sev(6, u, ib, w2 == 0 && lane == 0);
                fu_sev(7, u, ib, w2 == 0 && lane == 0);
                if (KB_FU_PROF == 3) {
                  m2.stop();
                  ++m3.acc;
                }
              }
            }
          }
          tc_commit_elect(&b_free[ab][s.i]);
          fu_sev(5, u, ib, w2 == 0 && lane == 0);
        }
        tc_commit_elect(&accA_empty[ab]);  // the buffer's pass-B stages are read: pass A may reuse it
        fu_ev(6, u, w2 == 0 && lane == 0);
        if (ab) sb1 = s;
        else sb0 = s;
        tc_commit_elect(&bfree[bb]);
        if (term == r - 1) tc_commit_elect(&accB_full);
      }
      ++T;
    }
    if (KB_FU_PROF == 3) {
      m2.put(2);
      m3.put(3);
    } else {
      p2.put(2);
      p3.put(3);
    }
  } else if (warp < kFuWDrain) {
    // ---------------- X converters: resident X stages -> pass-A A stages (lane = column) ----------------
    // two sets of four warps (one per lane quarter); set cs converts the half h == cs of every
    // 32-row X stage (A stage 2j + cs)
    const int q = warp & 3, tcol = 32 * q + lane, cs = (warp - kFuWConvX) >> 2;
    const unsigned lane_base = tmem + ((unsigned)(32 * q) << 16);
    FuWalk walk(f, batch);
    FuTile t;
    RingPos a;
    const bool me = tid == 32 * kFuWConvX;
    FuProf p4(me), p5(me), p11(me), p12(me), q13(me), q14(me);
    p11.start();
    int T = 0;
    while (walk.next(t, f)) {
      const int col = t.c0 - f.Hb + tcol;
      const bool cedge = f.fill_b && (t.c0 - f.Hb < 0 || t.c0 - f.Hb + 128 > f.n);
      // edge tiles: this lane's column source in the resident tile (identity inside the domain,
      // the fold source outside it; -1: zero -- the fold leaves the domain or the source lies
      // outside the tile, which only columns no output of the tile reads can hit)
      int csrc = tcol;
      bool cflip = false;
      if (col < 0 || col >= f.n) {
        const int cc = f.fill_b ? kb_fold(col, f.n) : -1;
        csrc = cc < 0 ? -1 : cc - (t.c0 - f.Hb);
        if (csrc >= 128) csrc = -1;
        cflip = true;
      }
      // a tile with reflected rows or columns reads fold sources from any of its X stages
      const bool edge_tile = cedge || (f.fill_a && (f.g0 + t.l0 - f.Ha < 0 || f.g0 + t.l0 + kFuL + f.Ha > f.Mg));
      for (int term = 0; term < r; ++term) {
        const int uu = T * r + term;
        const float sa = (f.sa_neg >> term) & 1 ? -1.f : 1.f;
        const float sb = sb_tab ? sb_tab[(long long)t.b * r + term] : 1.f;
        for (int j = 0; j < f.nxs; ++j) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int ia = 2 * j + h;
            if (ia >= f.na_a) break;
            if (h == cs) {
              p5.start();
              if (term == 0) {
                if (!edge_tile) {
                  fu_wait(&xfull[j], T & 1);
                } else if (j == 0) {
                  for (int jj = 0; jj < f.nxs; ++jj) fu_wait(&xfull[jj], T & 1);
                }
              }
              p5.stop();
              p4.start();
              fu_wait(&a_free[a.i], a.phase ^ 1);
              p4.stop();
              __syncwarp();  // reconverge before the .sync.aligned tensor-memory stores
              p12.start();
              const float* tile = xs + j * (kTcStageBytes / 4) + (16 * h) * 128 + tcol;
              const int lr0 = t.l0 - f.Ha + 32 * j + 16 * h;  // local row of the half's first row
              const bool redge = f.fill_a && (f.g0 + lr0 < 0 || f.g0 + lr0 + 16 > f.Mg);
              float xv[16];
#pragma unroll
              for (int i = 0; i < 16; ++i) xv[i] = KB_FU_NOLDS ? __int_as_float(0x3f800000 + i + tcol) : tile[i * 128];
              if (redge || cedge) {
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                  // row source (warp-uniform): the row itself, its fold source, or none
                  const int gr = f.g0 + lr0 + i;
                  int ti = 32 * j + 16 * h + i;
                  bool ok = csrc >= 0;
                  float sg = cflip ? sb : 1.f;
                  if (gr < 0 || gr >= f.Mg) {
                    const int rr = f.fill_a ? kb_fold(gr, f.Mg) : -1;
                    ok = ok && rr >= 0;
                    ti = rr - f.g0 - (t.l0 - f.Ha);
                    sg *= sa;
                  }
                  xv[i] = (ok && ti >= 0 && ti < 32 * f.nxs) ? sg * xs[ti * 128 + csrc] : 0.f;
                }
              }
              unsigned hi[16], lo[16];
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                hi[i] = __float_as_uint(xv[i]) & 0xffffe000u;
                lo[i] = __float_as_uint(xv[i] - __uint_as_float(hi[i]));
              }
              const unsigned ahi = lane_base + kFuStA + a.i * 32;
              if (KB_FU_PROF == 2) {
                p12.stop();
                q13.start();
              }
              if (!(f.dbg & 4)) {
                tc_st16(ahi, hi);
                tc_st16(ahi + 16, lo);
              }
              asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
              if (KB_FU_PROF == 2) {
                q13.stop();
                q14.start();
              }
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&a_ready[a.i]);
              if (KB_FU_PROF == 2) q14.stop();
              else p12.stop();
              if (ia == cs) fu_ev(7, uu, me);
              fu_sev(0, uu, ia, q == 0 && lane == 0);
              if (ia + 2 >= f.na_a) fu_ev(8, uu, me);
            }
            a.advance(kFuSA);
          }
          if (term == r - 1) {  // the stage's last reader this tile (both sets arrive)
            __syncwarp();
            if (lane == 0) mbar_arrive(&xfree[j]);
          }
        }
      }
      ++T;
    }
    p11.stop();
    p4.put(4);
    p5.put(5);
    p11.put(11);
    p12.put(12);
    if (KB_FU_PROF == 2) {  // X converter sub-steps instead of the Z converter / epilogue slots
      q13.put(13);
      q14.put(14);
    }
  } else if (warp < kFuWEpi) {
    // ---------------- drain (lane = column t) + Z converters (lane = row l) ----------------
    // two sets of four warps: set ds drains accumulator columns [64 ds, 64 ds + 64) of its lane
    // quarter, then converts the pass-B stages ib = ds (mod 2)
    const int q = warp & 3, tt = 32 * q + lane, l = tt, ds = (warp - kFuWDrain) >> 2;
    const unsigned lane_base = tmem + ((unsigned)(32 * q) << 16);
    FuWalk walk(f, batch);
    FuTile t;
    RingPos sb0, sb1;  // per-buffer ring positions (scalars: a runtime-indexed array would live in local memory)
    int u = 0;
    float4* zrow = reinterpret_cast<float4*>(zs + tt * kFuZsStride);
    const bool me = tid == 32 * kFuWDrain;
    FuProf p6(me), p7(me), p8(me), p9(me), p13(me);
    while (walk.next(t, f)) {
      const int nab = fu_nab(f, t.nblk);
      const float oscale = nw2 ? (float)(1.0 / sqrt(nw2[t.b])) : 1.f;
      for (int term = 0; term < r; ++term, ++u) {
        const int ab = u & 1;
        RingPos s = ab ? sb1 : sb0;
        p6.start();
        fu_wait(&accA_full[ab], (u >> 1) & 1);
        p6.stop();
        fu_ev(2, u, me);
        __syncwarp();
        tc_fence_after();
        p9.start();
        fu_named_sync(1, 128 * kFuDSets);  // every Z converter of the previous term has read zs
        p9.stop();
        __syncwarp();
        p8.start();
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int jj = 2 * ds + j;  // 32-column group of the drain
          float v[32];
          if (!(f.dbg & 8)) {
            tc_ld32(lane_base + kFuAccA + ab * 128 + 32 * jj, v);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = 0.f;
          }
#pragma unroll
          for (int c = 0; c < 8; ++c)
            zrow[8 * jj + c] =
                make_float4(v[4 * c] * oscale, v[4 * c + 1] * oscale, v[4 * c + 2] * oscale, v[4 * c + 3] * oscale);
        }
        p8.stop();
        fu_ev(3, u, me);
        p9.start();
        fu_named_sync(1, 128 * kFuDSets);  // zs complete
        p9.stop();
        __syncwarp();
        // pass-B A stages into the drained buffer's slots (every drain warp's tensor-memory reads
        // of this buffer completed before the barrier above)
        for (int ib = 0; ib < nab; ++ib, s.advance(kFuSB)) {
          if ((ib & 1) != ds) continue;
          p7.start();
          fu_wait(&b_free[ab][s.i], s.phase ^ 1);
          p7.stop();
          __syncwarp();
          p13.start();
          tc_fence_after();
          unsigned hi[16], lo[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int tr = 16 * ib + i;
            const float z = zs[tr * kFuZsStride + l];
            hi[i] = __float_as_uint(z) & 0xffffe000u;
            lo[i] = __float_as_uint(z - __uint_as_float(hi[i]));
          }
          const unsigned ahi = lane_base + kFuAccA + ab * 128 + s.i * 32;
          if (!(f.dbg & 16)) {
            tc_st16(ahi, hi);
            tc_st16(ahi + 16, lo);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&b_ready[ab][s.i]);
          p13.stop();
          fu_sev(3, u, ib, q == 0 && lane == 0);
        }
        fu_ev(4, u, me);
        if (ab) sb1 = s;
        else sb0 = s;
      }
    }
    p6.put(6);
    p7.put(7);
    p8.put(8);
    p9.put(9);
    if (KB_FU_PROF != 2) p13.put(13);
  } else {
    // ---------------- epilogue: the tile's accumulated sum -> fused update of the output rows ----------------
    const int ew = warp - kFuWEpi, q = warp & 3;  // lane quarter
    const unsigned lane_base = tmem + ((unsigned)(32 * q) << 16);
    const int nslots = gridDim.x * kFuEpi, slot = blockIdx.x * kFuEpi + ew;
    const int n = f.n;
    double nrm[3] = {0.0, 0.0, 0.0};
    bool bad = false;
    int norm_b = -1, T = 0;
    FuWalk walk(f, batch);
    FuTile t;
    FuProf p10(tid == 32 * kFuWEpi), p14(tid == 32 * kFuWEpi);
    while (walk.next(t, f)) {
      if (t.b != norm_b) {
        if (norm_b >= 0) kb_warp_finish_f<MODE>(e, nrm, bad, norm_b, nslots, slot, lane);
        nrm[0] = nrm[1] = nrm[2] = 0.0;
        bad = false;
        norm_b = t.b;
      }
      const int l = t.l0 + 32 * q + lane;
      const int ncols = 16 * t.nblk;
      double sc_L = 0.0, sc_d = 1.0;
      if constexpr (MODE == EPI_UPDATE) {
        sc_L = e.L[t.b];
        sc_d = e.denom[t.b];
      }
      if constexpr (MODE == EPI_POWER) sc_L = e.vnw2 ? e.vnw2[t.b] : 1.0;
      const long long row = (long long)t.b * e.bstride + (long long)l * n + t.c0;
      if (l < f.len) {  // operand rows to L2 while the tile's r terms accumulate
#pragma unroll
        for (int c = 0; c < 96; c += 32) {
          if (c >= t.cnt) break;
          if constexpr (MODE == EPI_RESID) prefetch_l2(e.bsub + row + c);
          if constexpr (MODE == EPI_UPDATE) {
            prefetch_l2(e.y + row + c);
            prefetch_l2(e.x + row + c);
          }
          if constexpr (MODE == EPI_POWER) prefetch_l2(e.vin + row + c);
        }
      }
      p10.start();
      fu_wait_idle(&accB_full, T & 1);
      p10.stop();
      __syncwarp();
      p14.start();
      tc_fence_after();
      const float Lb = (float)sc_L, db = (float)sc_d, rd = 1.f / db;
      const double vs = MODE == EPI_POWER && e.vnw2 ? sqrt(sc_L) : 1.0;
      // rounds of 32 columns: the accumulator is released once the last round is loaded
#pragma unroll 1
      for (int cbeg = 0; cbeg < ncols; cbeg += 32) {
        float v[32];
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          if (cbeg + 16 * p < ncols && !(f.dbg & 32)) {
            float w[16];
            tc_ld16(lane_base + kFuAccB + cbeg + 16 * p, w);
#pragma unroll
            for (int i = 0; i < 16; ++i) v[16 * p + i] = w[i];
          }
        }
        if (cbeg + 32 >= ncols) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&accB_empty);
        }
        if (l < f.len && !(f.dbg & 2)) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int c = t.cnt - cbeg - 8 * j;
            if (c <= 0) break;
            float v8[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) v8[i] = v[8 * j + i];
            tc_sum_epi8<MODE, NORMS>(v8, e, row + cbeg + 8 * j, min(8, c), Lb, db, rd, vs, nrm, bad);
          }
        }
      }
      p14.stop();
      ++T;
    }
    p10.put(10);
    if (KB_FU_PROF != 2) p14.put(14);
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
