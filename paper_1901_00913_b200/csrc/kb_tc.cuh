// kb_tc.cuh — fp32 passes on the 5th-generation tensor cores (tcgen05.mma kind::tf32, 3xTF32).
//
// The same banded GEMM as the other passes, Z_i^T[l][s] = sum_t X[t][l] c_i[t - s] for a
// 128-column L-tile (M = 128) and 16-output N-blocks, accumulated in tensor memory:
//   A = X^T from tensor memory: the natural [rows][cols] input tile is streamed by TMA in 32-row
//       blocks; converter warps (lane = column) split each value into tf32 hi + lo and store them
//       to an A stage in tensor memory (lane = column, column = K; 2 K-steps per stage). With A
//       read from shared memory the operand traffic of 16-wide MMAs bounds the tensor core at ~1/4
//       of its rate (ncu: 57% of the shared-memory bandwidth at 9% tensor activity).
//   B = Toeplitz bricks: for N-block nb and K-step k the 16 x 8 operand B[n][kk] = taps[8k + kk -
//       16nb - n] depends only on o = 8k - 16nb, so each term needs (Kw+14)/8 + 1 bricks (hi and
//       lo, K-major INTERLEAVE core matrices), built once per operator (kb_build_bricks) and
//       bulk-copied into shared memory.
//   D = tensor memory: 16-column accumulators per (term, N-block); each term accumulates only
//       its own K-range (the 3xTF32 products of one output stay in one accumulator, 33-35 K-steps
//       at the widest BASELINE band).
// Warp roles: warp 0 streams tiles (TMA) [and, in the sum pass, bricks]; warps 1-4 issue the MMAs
// of one N-block each (a converged warp issues from uniform registers; warp 1 owns the tensor
// memory); two sets of four converter warps own alternate tiles and fill the A stages; the last
// warps run the epilogue on one accumulator set while the MMAs fill the other.
#pragma once
#ifndef KB_TC_SPIN_NS
#define KB_TC_SPIN_NS 1000
#endif
#include "kb_ffma.cuh"
#include "kb_tf32.cuh"

namespace kb {

constexpr int kTcTS = 64;        // outputs (S rows) per chunk: 4 N-blocks of 16
constexpr int kTcRB = 32;        // input rows per ring stage (4 K-steps)
constexpr int kTcStagesMax = 8;  // tensor-memory A stages (2 K-steps: hi 16 + lo 16 columns each)
#ifndef KB_TC_RING_MAX
#define KB_TC_RING_MAX 8
#endif
constexpr int kTcRingMax = KB_TC_RING_MAX;  // shared-memory tile ring depth (runtime nst <= this)
constexpr int kTcG = 3;          // terms per group (two accumulator sets of kTcG x 64 columns)
constexpr int kTcIssuers = 4;    // one MMA-issuing warp per N-block
constexpr int kTcConv = 1 + kTcIssuers, kTcEpi = kTcConv + 8;  // first converter / epilogue warp
// The split pass is instantiated with 4 epilogue warps (one per tensor-memory lane quarter) or 8
// (two per quarter, each storing one 32-output half of a chunk: at cfg5 the split is bound by its
// Z^T stores, 3.3 -> 3.1 ms). 8 needs 32 KB more staging, so the host picks it only when a
// >= 4-stage tile ring still fits beside the bricks.
__host__ __device__ constexpr int tc_split_threads(int epi) { return 32 * (kTcEpi + epi); }
constexpr unsigned kTcStageBytes = kTcRB * 128 * 4;  // one [32 rows][128 cols] fp32 tile
// tensor memory: two accumulator sets of G x 64 columns, then the A stages
__host__ __device__ __forceinline__ int tc_astages(int G) { return min(kTcStagesMax, (512 - 128 * G) / 32); }
#ifndef KB_TC_STORE_BUFS
#define KB_TC_STORE_BUFS 2
#endif
constexpr int kTcStoreBufs = KB_TC_STORE_BUFS;  // TMA-store staging buffers per epilogue warp
// epilogue staging: warps x buffers x [32 L][32 S]
__host__ __device__ constexpr unsigned tc_store_bytes(int epi) { return epi * kTcStoreBufs * 4096; }
// dynamic shared memory: [staging][tile ring][bricks] (1 KB alignment slack in front)

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
// Compiled in only with -DKB_TC_PROF=1 (tools/tc_profile.py builds that variant): the runtime
// checks alone cost ~8% of the sum pass' issued instructions.
#ifndef KB_TC_PROF
#define KB_TC_PROF 0
#endif
struct TcProf {
  bool on;
  unsigned long long acc = 0, t0 = 0;
  __device__ TcProf(const AxisGeom& g, bool me) : on(KB_TC_PROF && (g.dbg & 128) && me && blockIdx.x < kTraceBlocks) {}
  __device__ __forceinline__ void start() { if (on) t0 = clock64(); }
  __device__ __forceinline__ void stop() { if (on) acc += clock64() - t0; }
  __device__ __forceinline__ void put(int slot, int kind = 0) { if (on) kb_trace[kind][blockIdx.x][slot] = acc; }
};

// mbarrier wait for threads off the critical path (epilogue warps): each unsuccessful probe
// suspends the thread for up to `ns` nanoseconds instead of re-polling at once, so the waiting
// warps leave the issue slots to the converter and MMA warps that share their SM sub-partition
__device__ __forceinline__ void mbar_wait_lazy(unsigned long long* bar, unsigned parity, unsigned ns) {
  asm volatile(
      "{\n.reg .pred p;\nWAITL_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
      "@!p bra WAITL_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(ns)
      : "memory");
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
// mbarrier wait that sleeps between probes: for the roles that are never on the critical path
// (the TMA producer waiting for a free ring stage, the epilogue waiting for a finished term),
// so their polling does not take issue slots from the converter and MMA warps of the same SM
// sub-partition
#ifndef KB_TC_SLEEP_NS
#define KB_TC_SLEEP_NS 256
#endif
__device__ __forceinline__ bool mbar_test(unsigned long long* bar, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_idle(unsigned long long* bar, unsigned parity, unsigned lazy_ns) {
  if (KB_TC_SLEEP_NS > 0) {
    while (!mbar_test(bar, parity)) __nanosleep(KB_TC_SLEEP_NS);
  } else {
    mbar_wait_lazy(bar, parity, lazy_ns);
  }
}

// suspend-time hint of the tcgen05 kernels' barrier waits (KB_TC_SPIN_NS experiments)
constexpr unsigned kTcSpinNs = KB_TC_SPIN_NS;

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

// reflect fill of 16 consecutive tile rows starting at global row r0 (edge tiles of a reflective
// axis only; the interior tiles load all 16 rows before this branch):
// out-of-domain rows take sign * X[fold(row)] from global memory
__device__ __forceinline__ void tc_reflect_fill(float* xv, int r0, const AxisGeom& g, const float* __restrict__ in,
                                             long long img, int col, float fsign) {
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int gr = r0 + i;
    if (gr < 0 || gr >= g.Mg) {
      const int f = kb_fold(gr, g.Mg);
      xv[i] = (f >= 0 && col < g.other) ? fsign * in[img + (long long)(f - g.g0) * g.other + col] : 0.f;
    }
  }
}

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
__device__ __forceinline__ void tc_ld8(unsigned addr, float (&v)[8]) {
  unsigned u[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7])
               : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(u[i]);
}
__device__ __forceinline__ void tc_st16(unsigned addr, const unsigned (&u)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          addr),
      "r"(u[0]), "r"(u[1]), "r"(u[2]), "r"(u[3]), "r"(u[4]), "r"(u[5]), "r"(u[6]), "r"(u[7]), "r"(u[8]), "r"(u[9]),
      "r"(u[10]), "r"(u[11]), "r"(u[12]), "r"(u[13]), "r"(u[14]), "r"(u[15]));
}

// 1-D bulk copy global -> shared, completion counted in bytes on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Brick table of one tap table [batch][r][Wp] (built once per operator at creation): per
// (image, term) the nbr bricks of kb_pass_split_tc / kb_pass_sum_tc in their shared-memory
// layout, [batch][r][nbr][hi 128 | lo 128 words], so a pass loads a term's bricks with one bulk
// copy instead of rebuilding them on its threads.
// `shift` > 0 builds the bricks of the same taps for a window widened by `shift` on each side
// (half width H + shift; the fused kernel's TMA-aligned tile origin, kb_fused.cuh)
__global__ void kb_build_bricks(const float* __restrict__ tin, int Wp, int Kw, int nbr, long long bt_total,
                                unsigned* __restrict__ out, int shift = 0) {
  const long long total = bt_total * nbr * 128;
  for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
       idx += (long long)gridDim.x * blockDim.x) {
    const long long bt = idx / (nbr * 128);
    const int rem = (int)(idx - bt * nbr * 128), qb = rem >> 7, e = rem & 127, nn = e >> 3, kk = e & 7;
    const int ti = 8 * qb + kk - nn - shift;
    const float c = (ti >= 0 && ti < Kw) ? tin[bt * Wp + ti] : 0.f;
    unsigned h, l;
    tf32_split_rn(c, h, l);
    const int off = (nn >> 3) * 64 + (kk >> 2) * 32 + (nn & 7) * 4 + (kk & 3);
    unsigned* bp = out + (bt * nbr + qb) * 256;
    bp[off] = h;
    bp[128 + off] = l;
  }
}

// Tensor-core split pass. Work: (image b, 128-column L-tile, S-part) items walked in 64-output
// chunks, once per group of G terms (bricks of a group stay resident; the tile is re-streamed per
// group). Stage flow: TMA -> shared tile [32 rows][128 cols] -> workers (lane = column) split each
// value into tf32 hi + lo and store them to a tensor-memory A stage (lane = column, 32 + 32
// columns = K) -> MMAs (A from tensor memory, so the only shared-memory operand traffic is the 512-B
// bricks). bricks: [G][nbr][hi 512 B | lo 512 B]. Results leave
// through a 128-byte-swizzled [32 L][32 S] staging box per worker warp and a TMA store (zmap:
// Z^T planes b * r + term), so every global write is a full line; ragged chunk ends store directly.
// (chunk, term group) pairs of the split pass, in one of two orders: group-major (each group
// streams the whole plane, holding one group's bricks) or chunk-major (all groups of a chunk back
// to back, every term's bricks resident: the chunk's input tiles are re-read from L2 rather than
// DRAM -- at cfg5, r = 10 in 4 groups, that is 3 of the 4 reads of X)
struct PairWalk {
  ChunkWalk w0, walk;
  Chunk ch;
  int gr = 0, ngroups;
  bool chunk_major, fresh = true;
  __device__ PairWalk(const ChunkWalk& w, int ng, bool cm) : w0(w), walk(w), ngroups(ng), chunk_major(cm) {}
  __device__ bool next(Chunk& c, int& g) {
    if (chunk_major) {
      if (fresh || ++gr == ngroups) {
        if (!walk.next(ch, kTcTS)) return false;
        gr = 0;
        fresh = false;
      }
    } else {
      while (!walk.next(ch, kTcTS)) {
        if (++gr >= ngroups) return false;
        walk = w0;
      }
    }
    c = ch;
    g = gr;
    return true;
  }
};

// the split pass' barrier waits: plain polling, or (KB_TC_SPLIT_LAZY=1 at build time) try_wait
// with a suspend-time hint so waiting warps leave their issue slots (and power) to the others
// (A/B at cfg5: 21.13k either way, the clock stays at the 1.5 GHz power cap)
#ifndef KB_TC_SPLIT_LAZY
#define KB_TC_SPLIT_LAZY 0
#endif
#define KB_TCS_WAIT(bar, par) \
  (KB_TC_SPLIT_LAZY ? mbar_wait_lazy((bar), (par), kTcSpinNs) : mbar_wait((bar), (par)))
template <int EPI>
__global__ void __launch_bounds__(tc_split_threads(EPI), 1)
kb_pass_split_tc(const __grid_constant__ CUtensorMap tmap, const __grid_constant__ CUtensorMap zmap,
                 float* __restrict__ z, long long z_ps, long long z_bs, const unsigned* __restrict__ btab,
                 AxisGeom g, const double* __restrict__ nw2, int r, int batch, int parts, Groups grp, int G,
                 int nst, const float* __restrict__ in, long long in_bs, int mirror_h,
                 const float* __restrict__ msign, int chunk_major) {
  extern __shared__ __align__(16) unsigned char kb_smem_tc[];
  __shared__ unsigned long long full[kTcRingMax], sfree[kTcRingMax], a_ready[kTcStagesMax],
      a_free[kTcStagesMax], acc_full[2], acc_empty[2], bready;
  __shared__ unsigned tmem_base;
  unsigned char* base = kb_smem_tc + ((1024 - (smem_u32(kb_smem_tc) & 1023)) & 1023);
  float* staging = reinterpret_cast<float*>(base);  // [4 warps][2][32][32], 128-byte swizzled rows
  constexpr unsigned kStore = tc_store_bytes(EPI);
  float* stages = reinterpret_cast<float*>(base + kStore);  // [nst][32][128]
  unsigned* bricks = reinterpret_cast<unsigned*>(base + kStore + nst * kTcStageBytes);
  // warp index and tensor-memory base through a lane-0 shuffle: provably warp-uniform, so the MMA
  // operands are computed in uniform registers (no per-MMA register-to-uniform moves)
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;
  const int LT = (g.other + 127) / 128;
  const int nk = tc_ksteps(g.Kw), nrb = (nk + 3) / 4, na = (nk + 1) / 2, nbr = tc_bricks(g.Kw);
  const int ngroups = grp.n;  // sign-uniform term groups of <= G terms
  const int nas = tc_astages(G), acol = 128 * G;  // A stages at columns acol + 32 st

  if (tid == 0) {
    for (int st = 0; st < nst; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&sfree[st], 4);  // the owning converter set
    }
    for (int st = 0; st < nas; ++st) {
      mbar_init(&a_ready[st], 4);
      mbar_init(&a_free[st], kTcIssuers);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], kTcIssuers);
      mbar_init(&acc_empty[b], EPI);
    }
    mbar_init(&bready, 1);
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
      PairWalk pairs(ChunkWalk(g.len, LT, parts, batch, 4), ngroups, chunk_major);
      Chunk ch;
      int gr;
      while (pairs.next(ch, gr)) {
        {
          for (int rb = 0; rb < nrb; ++rb, t.advance(nst)) {
            pw.start();
#if KB_TC_SPLIT_PRODUCER_SPIN
            mbar_wait(&sfree[t.i], t.phase ^ 1);
#else
            mbar_wait_idle(&sfree[t.i], t.phase ^ 1, kTcSpinNs);
#endif
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
    // brick descriptors advance by adding (bytes >> 4) to the start-address field
    const unsigned long long b0 = tc_desc(smem_u32(bricks), 128, 256, 0);
    const int qmax = (g.Kw + 14) >> 3;
    const bool live = !(g.dbg & 1);
    PairWalk pairs(ChunkWalk(g.len, LT, parts, batch, 4), ngroups, chunk_major);
    Chunk ch;
    int gr;
    while (pairs.next(ch, gr)) {
      const int gc = grp.count[gr];
      const unsigned boff = chunk_major ? (unsigned)grp.start[gr] * nbr : 0u;  // resident bricks
      {
        const int ab = chunk & 1;
        pe.start();
        if (chunk >= 2) KB_TCS_WAIT(&acc_empty[ab], ((chunk >> 1) - 1) & 1);  // epilogue drained this set
        __syncwarp();
        pe.stop();
        tc_fence_after();
        const unsigned dcol = tmem + ab * 64 * G + nb * 16;
        for (int ia = 0; ia < na; ++ia, a.advance(nas)) {
          const int st = a.i;
          pa.start();
          KB_TCS_WAIT(&a_ready[st], a.phase);  // A stage (and, at a group change, bricks) ready
          __syncwarp();  // reconverge: elect.sync below must see the whole warp
          pa.stop();
          if (!(g.dbg & 8)) tc_fence_after();
          const unsigned ahi = tmem + acol + st * 32;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int k = 2 * ia + h, q = k - 2 * nb;  // brick index o / 8 with o = 8k - 16nb
            if (live && k < nk && q >= 0 && q <= qmax) {
              if (gc == 3) {
                const unsigned long long bh = b0 + ((boff + (unsigned)q) * 1024 >> 4);
                tc_mma3x3(dcol, ahi + 8 * h, ahi + 16 + 8 * h, bh, (unsigned)nbr * 1024 >> 4, q != 0);
                continue;
              }
#pragma unroll
              for (int gi = 0; gi < kTcG; ++gi) {
                if (gi >= gc) break;
                const unsigned long long bh = b0 + ((boff + (unsigned)(gi * nbr + q)) * 1024 >> 4);
                tc_mma3(dcol + gi * kTcTS, ahi + 8 * h, ahi + 16 + 8 * h, bh, bh + (512 >> 4), q != 0);
              }
            }
          }
          tc_commit_elect(&a_free[st]);  // the A stage can be refilled once these MMAs have read it
        }
        tc_commit_elect(&acc_full[ab]);
        ++chunk;
      }
    }
    if (!(g.dbg & 256)) pa.put(6);
  } else if (warp < kTcEpi) {
    // ---------------- converters: bricks and A stages ----------------
    // two sets of four warps (one per tensor-memory lane quarter); set cs owns the tiles with
    // global tile index parity cs and converts both of their A stages
    const int wt = tid - 32 * kTcConv;  // 0..255
    const int cs = wt >> 7;
    const int q = warp & 3;             // tensor-memory lane quarter this warp may access
    const unsigned lane_base = tmem + ((unsigned)(32 * q) << 16);
    TcProf p1(g, wt == 0), p2(g, wt == 0), pt(g, wt == 0), pc(g, wt == 0), ps(g, wt == 0), pb(g, wt == 0);
    pt.start();
    RingPos a, t;
    int chunk = 0, bricks_key = -1, nbl = 0, tg = 0;
    PairWalk pairs(ChunkWalk(g.len, LT, parts, batch, 4), ngroups, chunk_major);
    Chunk ch;
    int gr;
    while (pairs.next(ch, gr)) {
      const int g0 = grp.start[gr], gc = grp.count[gr];
      const float fsign = grp.sign[gr] < 0 ? -1.f : 1.f;
      {
        const int key = chunk_major ? ch.b : ch.b * ngroups + gr;
        if (key != bricks_key) {
          // the group's bricks (chunk-major: every term's) in one bulk copy from the brick table,
          // once the previous chunk's MMAs (the last readers of the old bricks) completed
          pb.start();
          if (wt == 0) {
            if (chunk > 0) KB_TCS_WAIT(&acc_full[(chunk - 1) & 1], ((chunk - 1) >> 1) & 1);
            const int t0 = chunk_major ? 0 : g0, tn = chunk_major ? r : gc;
            const unsigned bytes = (unsigned)(tn * nbr) * 1024;
            mbar_arrive_expect_tx(&bready, bytes);
            bulk_g2s(bricks, btab + ((long long)ch.b * r + t0) * nbr * 256, bytes, &bready);
          }
          KB_TCS_WAIT(&bready, nbl & 1);  // before any A stage of this chunk is announced
          ++nbl;
          bricks_key = key;
          pb.stop();
        }
        for (int rb = 0; rb < nrb; ++rb, ++tg, t.advance(nst)) {
          const int nat = min(2, na - 2 * rb);  // A stages of this tile
          if ((tg & 1) != cs) {
            a.advance(nas);
            if (nat == 2) a.advance(nas);
            continue;
          }
          p2.start();
          KB_TCS_WAIT(&full[t.i], t.phase);
          p2.stop();
          tc_fence_after();
          const float* tile = stages + t.i * (kTcStageBytes / 4) + 32 * q + lane;
          const int row_lo = g.g0 + ch.s0 - g.H + kTcRB * rb;  // global row of tile row 0
          const bool edge = g.fill && (row_lo < 0 || row_lo + kTcRB > g.Mg);
          int st0 = a.i, st1 = -1;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (h == nat) break;
            if (h == 1) st1 = a.i;
            p1.start();
            KB_TCS_WAIT(&a_free[a.i], a.phase ^ 1);
            p1.stop();
            pc.start();
            if (!(g.dbg & 4)) {
              unsigned hi[16], lo[16];
              float xv[16];
#pragma unroll
              for (int i = 0; i < 16; ++i) xv[i] = tile[(16 * h + i) * 128];
              if (edge) tc_reflect_fill(xv, row_lo + 16 * h, g, in, ch.b * in_bs, ch.lt * 128 + 32 * q + lane, fsign);
#pragma unroll
              for (int i = 0; i < 16; ++i) {
                hi[i] = __float_as_uint(xv[i]) & 0xffffe000u;
                lo[i] = __float_as_uint(xv[i] - __uint_as_float(hi[i]));
              }
              const unsigned ahi = lane_base + acol + a.i * 32;
              tc_st16(ahi, hi);
              tc_st16(ahi + 16, lo);
            }
            pc.stop();
            a.advance(nas);
          }
          ps.start();
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          ps.stop();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(&a_ready[st0]);
            if (st1 >= 0) mbar_arrive(&a_ready[st1]);
            mbar_arrive(&sfree[t.i]);  // shared tile read: TMA may refill it
          }
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
    pt.put(7);
  } else {
    // ---------------- epilogue: accumulators -> Z^T rows ----------------
    const int q = warp & 3, ew = warp - kTcEpi, hsel = ew >> 2;  // lane quarter, output half (8 warps)
    const unsigned lane_base = tmem + ((unsigned)(32 * q) << 16);
    TcProf p3(g, warp == kTcEpi && lane == 0), p4(g, warp == kTcEpi && lane == 0);
    int chunk = 0, nstore = 0;
    PairWalk pairs(ChunkWalk(g.len, LT, parts, batch, 4), ngroups, chunk_major);
    Chunk ch;
    int gr;
    while (pairs.next(ch, gr)) {
      const int g0 = grp.start[gr], gc = grp.count[gr];
      {
        const int ab = chunk & 1;
        p3.start();
        KB_TCS_WAIT(&acc_full[ab], (chunk >> 1) & 1);
        p3.stop();
        p4.start();
        tc_fence_after();
        const int l0 = ch.lt * 128 + 32 * q, l = l0 + lane;
        const float oscale = nw2 ? (float)(1.0 / sqrt(nw2[ch.b])) : 1.f;
        for (int gg = 0; gg < gc; ++gg) {
          float* zp = z + ch.b * z_bs + (long long)(g0 + gg) * z_ps + (long long)l * g.len + ch.s0;
          for (int h = EPI == 8 ? hsel : 0; h < kTcTS / 32; h += EPI / 4) {
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
              if (nstore >= kTcStoreBufs && lane == 0) bulk_wait_read<kTcStoreBufs - 1>();
              __syncwarp();
              float* sb = staging + (kTcStoreBufs * ew + (nstore % kTcStoreBufs)) * 1024;
#pragma unroll
              for (int c = 0; c < 8; ++c)
                reinterpret_cast<float4*>(sb + lane * 32)[c ^ (lane & 7)] =
                    make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
              __syncwarp();
              if (lane == 0 && l0 < g.other) {  // boxes wholly past the last row carry no data
                tma_store_3d(&zmap, sb, ch.s0 + s, l0, ch.b * r + g0 + gg);
                bulk_commit();
              }
              ++nstore;
            } else if (l < g.other) {
#pragma unroll
              for (int i = 0; i < 32; ++i)
                if (s + i < ch.cnt) zp[s + i] = v[i];
            }
            // reflected halo rows of Z^T for a reflect-filled sum pass (edge L-tiles only):
            // row -1 - l and / or row 2 * other - 1 - l (both when the halo spans the plane),
            // times the term's mirror sign
            if (mirror_h > 0 && l < g.other && (l < mirror_h || l >= g.other - mirror_h)) {
              const float sg = msign ? msign[(long long)ch.b * r + g0 + gg] : 1.f;
#pragma unroll
              for (int side = 0; side < 2; ++side) {
                if (side == 0 ? l >= mirror_h : l < g.other - mirror_h) continue;
                float* zm = zp + (long long)((side == 0 ? -1 - l : 2 * g.other - 1 - l) - l) * g.len;
                if (s + 32 <= ch.cnt) {
#pragma unroll
                  for (int c = 0; c < 8; ++c)
                    reinterpret_cast<float4*>(zm + s)[c] =
                        make_float4(sg * v[4 * c], sg * v[4 * c + 1], sg * v[4 * c + 2], sg * v[4 * c + 3]);
                } else {
#pragma unroll
                  for (int i = 0; i < 32; ++i)
                    if (s + i < ch.cnt) zm[s + i] = sg * v[i];
                }
              }
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

// Chunks of the tensor-core sum pass, dealt round-robin: block i takes global chunk indices i,
// i + gridDim.x, ... with the S-chunk index fastest (then L-tile, then image). The blocks that run
// at the same time then hold adjacent chunks of the same planes, so the 2H halo rows one block
// re-reads were fetched moments earlier by its neighbour (L2 hits): with one block walking its
// own chunk range instead, r term planes pass between its reuses and the halo rows come from
// HBM again (5x the compulsory plane traffic at cfg4).
struct StrideWalk {
  int k, nsc, LT, S, total;
  __device__ StrideWalk(int S_, int LT_, int batch, int TS) : nsc((S_ + TS - 1) / TS), LT(LT_), S(S_) {
    k = blockIdx.x;
    total = nsc * LT * batch;
  }
  __device__ bool next(Chunk& c, int TS) {
    if (k >= total) return false;
    const int sc = k % nsc, rest = k / nsc;
    c.lt = rest % LT;
    c.b = rest / LT;
    c.s0 = sc * TS;
    c.cnt = min(TS, S - c.s0);
    k += gridDim.x;
    return true;
  }
};

// ------------------------------------------------------------------------------------------
// Tensor-core sum pass: Y[l][s] = sum_i sum_t Z_i^T[t][l] d_i[t - s] for a 128-column L-tile and
// 64-output chunks. Every (chunk, term) accumulates in its own 64-column tensor-memory slot (a
// ring of four), and eight epilogue warps (lane quarter x 32-output half) add the slots into
// fp32 registers in term order and run the fused epilogue after the last term: the tensor
// core's own accumulation stays as long as one split-pass term (one accumulator across all r
// terms drifts past the fp32 parity bound at the widest BASELINE band). Same producer /
// issuer / converter pipeline as kb_pass_split_tc; the bricks of consecutive terms alternate
// between two shared-memory buffers: the producer bulk-copies term t's bricks from the
// operator's brick table (kb_build_bricks) once the MMAs of term t - 2 completed (bfree), and
// the issuers wait for them (bready). Reflective axes read the reflected halo rows the split
// pass stored (TMA boxes over the padded planes) and add the adjoint's fold corrections in the
// epilogue; epilogue operands move as 16-byte vectors per lane row.
// ------------------------------------------------------------------------------------------
#ifndef KB_TC_V8
#define KB_TC_V8 1  // 256-bit epilogue loads / stores (sm_100: LDG/STG.256)
#endif
constexpr int kTcSumSlots = 4;                       // per-term accumulator slots (64 columns each)
constexpr int kTcSumEpi = 8;                         // epilogue warps
// converter sets of the sum pass (4 warps each, alternate tiles): the sum pass is converter-bound
// (per-role timeline at cfg5: the issuers wait 39% of the time for A stages)
#ifndef KB_TC_SUM_SETS
#define KB_TC_SUM_SETS 2
#endif
constexpr int kTcSumSets = KB_TC_SUM_SETS;
constexpr int kTcSumEpiW = kTcConv + 4 * kTcSumSets;  // first epilogue warp of the sum pass
constexpr int kTcSumThreads = 32 * (kTcSumEpiW + kTcSumEpi);
template <int MODE, bool NORMS = true>
__device__ __forceinline__ void tc_sum_epi8(const float (&v)[8], const Epi<float>& e, long long at, int cnt,
                                            float Lb, float db, float rd, double vs, double (&nrm)[3],
                                            bool& bad) {
  // 8 consecutive outputs of one row: elements [at, at + cnt), cnt <= 8, at % 4 == 0 when cnt == 8
  float u[8], w[8];
  const bool full8 = cnt == 8;
  auto ld8 = [&](const float* a, float (&o)[8]) {
    if (full8 && KB_TC_V8 && !(reinterpret_cast<unsigned long long>(a + at) & 31)) {  // one 32-byte sector
      asm volatile("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=f"(o[0]), "=f"(o[1]), "=f"(o[2]), "=f"(o[3]), "=f"(o[4]), "=f"(o[5]), "=f"(o[6]), "=f"(o[7])
                   : "l"(a + at));
    } else if (full8) {
      const float4 p0 = *reinterpret_cast<const float4*>(a + at), p1 = *reinterpret_cast<const float4*>(a + at + 4);
      o[0] = p0.x, o[1] = p0.y, o[2] = p0.z, o[3] = p0.w, o[4] = p1.x, o[5] = p1.y, o[6] = p1.z, o[7] = p1.w;
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = i < cnt ? a[at + i] : 0.f;
    }
  };
  auto st8 = [&](float* a, const float (&o)[8]) {
    if (full8 && KB_TC_V8 && !(reinterpret_cast<unsigned long long>(a + at) & 31)) {
      asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(a + at), "f"(o[0]), "f"(o[1]), "f"(o[2]),
                   "f"(o[3]), "f"(o[4]), "f"(o[5]), "f"(o[6]), "f"(o[7])
                   : "memory");
    } else if (full8) {
      *reinterpret_cast<float4*>(a + at) = make_float4(o[0], o[1], o[2], o[3]);
      *reinterpret_cast<float4*>(a + at + 4) = make_float4(o[4], o[5], o[6], o[7]);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (i < cnt) a[at + i] = o[i];
    }
  };
  if constexpr (MODE == EPI_PLAIN) {
    st8(e.out, v);
  } else if constexpr (MODE == EPI_RESID) {
    ld8(e.bsub, u);
#pragma unroll
    for (int i = 0; i < 8; ++i) u[i] = __fsub_rn(v[i], u[i]);
    st8(e.out, u);
  } else if constexpr (MODE == EPI_UPDATE) {
    // in place (u: y_k -> x_k, w: x_{k-1} -> y_{k+1}): the epilogue warps share the kernel's
    // register budget with the sum[32] accumulators
    ld8(e.y, u);
    ld8(e.x, w);
    const float beta = (float)e.beta;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float a = __fsub_rn(__fmul_rn(Lb, u[i]), v[i]);
      const float q0 = __fmul_rn(a, rd);
      float x = fmaf(fmaf(-db, q0, a), rd, q0);
      if (e.project) x = (x > 0.f || x != x) ? x : 0.f;
      const float d = __fsub_rn(x, w[i]);
      if (i < cnt) {
        bad |= !isfinite(x);
        if (NORMS && e.want_norms) {
          nrm[0] += (double)d * d;
          nrm[1] += (double)w[i] * w[i];
          nrm[2] += (double)x * x;
        }
      }
      u[i] = x;
      w[i] = __fadd_rn(x, __fmul_rn(beta, d));
    }
    st8(e.x, u);
    st8(e.y, w);
  } else {  // EPI_POWER
    ld8(e.vin, u);
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i < cnt) {
        const double vv = e.vnw2 ? (double)u[i] / vs : (double)u[i];
        nrm[0] += vv * v[i];
        nrm[1] += (double)v[i] * v[i];
      }
    st8(e.out, v);
  }
}

// TMAE: the epilogue operands staged by TMA (one 32 x 32 128-byte-swizzled box per epilogue warp
// and operand plane, loaded during the chunk's terms, results stored by TMA; see kb_tc1.cuh)
template <int MODE>
__host__ __device__ constexpr unsigned tc_ebuf_bytes() { return kTcSumEpi * (MODE == EPI_UPDATE ? 2 : 1) * 4096u; }
template <int MODE, bool NORMS = true, bool TMAE = false>  // NORMS = false: update without the history norms
__global__ void __launch_bounds__(kTcSumThreads, 1)
kb_pass_sum_tc(const __grid_constant__ CUtensorMap tmap, int r, const unsigned* __restrict__ btab, AxisGeom g,
               Epi<float> e, int batch, int nst, const __grid_constant__ CUtensorMap emap0,
               const __grid_constant__ CUtensorMap emap1) {
  extern __shared__ __align__(16) unsigned char kb_smem_tc[];
  __shared__ unsigned long long full[kTcRingMax], sfree[kTcRingMax], a_ready[kTcStagesMax],
      a_free[kTcStagesMax], slot_full[kTcSumSlots], slot_empty[kTcSumSlots], bready[2], bfree[2], eful[kTcSumEpi];
  __shared__ unsigned tmem_base;
  unsigned char* base = kb_smem_tc + ((1024 - (smem_u32(kb_smem_tc) & 1023)) & 1023);
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), lane = tid & 31;
  const int LT = (g.other + 127) / 128;
  const int nk = tc_ksteps(g.Kw), nrb = (nk + 3) / 4, na = (nk + 1) / 2, nbr = tc_bricks(g.Kw);
  const int nas = kTcStagesMax, acol = 64 * kTcSumSlots;  // term slots at 64 j, A stages above
  float* stages = reinterpret_cast<float*>(base);  // [nst][32][128]
  unsigned* bricks = reinterpret_cast<unsigned*>(base + nst * kTcStageBytes);  // [2][nbr][256]
  unsigned char* ebuf = base + (((size_t)nst * kTcStageBytes + 2 * (size_t)nbr * 1024 + 1023) & ~(size_t)1023);

  if (tid == 0) {
    for (int st = 0; st < nst; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&sfree[st], 4);
    }
    for (int st = 0; st < nas; ++st) {
      mbar_init(&a_ready[st], 4);
      mbar_init(&a_free[st], kTcIssuers);
    }
    for (int j = 0; j < kTcSumSlots; ++j) {
      mbar_init(&slot_full[j], kTcIssuers);
      mbar_init(&slot_empty[j], kTcSumEpi);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bready[b], 1);
      mbar_init(&bfree[b], kTcIssuers);
    }
    for (int w = 0; w < kTcSumEpi; ++w) mbar_init(&eful[w], 1);
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
    // ---------------- TMA producer: per chunk and term, the term's bricks (bulk copy into the
    // buffer the MMAs of term - 2 released) and its plane's tiles ----------------
    if (lane == 0) {
      RingPos t;
      int tb = 0;
      const unsigned bbytes = (unsigned)nbr * 1024;
      StrideWalk walk(g.len, LT, batch, kTcTS);
      Chunk ch;
      while (walk.next(ch, kTcTS)) {
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
    // ---------------- MMA issuers: one warp per N-block ----------------
    const int nb = warp - 1;
    RingPos a, sl;
    int tb = 0;
    TcProf pa(g, warp == 1 && lane == 0), pb(g, warp == 1 && lane == 0);
    const unsigned long long b0 = tc_desc(smem_u32(bricks), 128, 256, 0);
    const int qmax = (g.Kw + 14) >> 3;
    StrideWalk walk(g.len, LT, batch, kTcTS);
    Chunk ch;
    while (walk.next(ch, kTcTS)) {
      for (int term = 0; term < r; ++term, ++tb, sl.advance(kTcSumSlots)) {
        const int bb = tb & 1;
        pb.start();
        mbar_wait_lazy(&slot_empty[sl.i], sl.phase ^ 1, kTcSpinNs);  // the epilogue added this slot's previous term
        mbar_wait_lazy(&bready[bb], (tb >> 1) & 1, kTcSpinNs);        // this term's bricks are built
        pb.stop();
        __syncwarp();
        tc_fence_after();
        const unsigned dcol = tmem + sl.i * 64 + nb * 16;
        bool first = true;
        for (int ia = 0; ia < na; ++ia, a.advance(nas)) {
          pa.start();
          mbar_wait_lazy(&a_ready[a.i], a.phase, kTcSpinNs);
          pa.stop();
          __syncwarp();
          tc_fence_after();
          const unsigned ahi = tmem + acol + a.i * 32;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int k = 2 * ia + h, q = k - 2 * nb;
            if (!(g.dbg & 1) && k < nk && q >= 0 && q <= qmax) {
              const unsigned long long bh = b0 + ((unsigned)(bb * nbr + q) * 1024 >> 4);
              tc_mma3(dcol, ahi + 8 * h, ahi + 16 + 8 * h, bh, bh + (512 >> 4), first ? 0u : 1u);
              first = false;
            }
          }
          tc_commit_elect(&a_free[a.i]);
        }
        tc_commit_elect(&bfree[bb]);       // the brick buffer may be rebuilt
        tc_commit_elect(&slot_full[sl.i]);  // this term's accumulator is complete
      }
    }
    pa.put(4, 1);
    pb.put(5, 1);
  } else if (warp < kTcSumEpiW) {
    // ---------------- converters: A stages ----------------
    // set cs owns the tiles with global tile index parity cs and converts both of a tile's A
    // stages (16 rows each: column 32q + lane of each row -> tensor-memory lane, K -> column)
    const int wt = tid - 32 * kTcConv;  // 0 .. 128 * kTcSumSets - 1
    const int cs = wt >> 7;
    const int q = warp & 3;
    const unsigned lane_base = tmem + ((unsigned)(32 * q) << 16);
    RingPos a, t;
    int tg = 0;
    TcProf p0(g, wt == 0), p1(g, wt == 0), p2(g, wt == 0), p3(g, wt == 0), p6(g, wt == 0), p7(g, wt == 0);
    p7.start();
    StrideWalk walk(g.len, LT, batch, kTcTS);
    Chunk ch;
    while (walk.next(ch, kTcTS)) {
      for (int term = 0; term < r; ++term) {
        for (int rb = 0; rb < nrb; ++rb, ++tg, t.advance(nst)) {
          const int nat = min(2, na - 2 * rb);  // A stages of this tile
          if (tg % kTcSumSets != cs) {
            a.advance(nas);
            if (nat == 2) a.advance(nas);
            continue;
          }
          p2.start();
          mbar_wait_lazy(&full[t.i], t.phase, kTcSpinNs);
          p2.stop();
          tc_fence_after();
          const float* tile = stages + t.i * (kTcStageBytes / 4) + 32 * q + lane;
          int st0 = a.i, st1 = -1;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (h == nat) break;
            if (h == 1) st1 = a.i;
            p1.start();
            mbar_wait_lazy(&a_free[a.i], a.phase ^ 1, kTcSpinNs);
            p1.stop();
            p0.start();
            if (!(g.dbg & 4)) {
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
            }
            p0.stop();
            a.advance(nas);
          }
          p6.start();
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          p6.stop();
          p3.start();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(&a_ready[st0]);
            if (st1 >= 0) mbar_arrive(&a_ready[st1]);
            mbar_arrive(&sfree[t.i]);  // shared tile read: TMA may refill it
          }
          p3.stop();
        }
      }
    }
    p7.stop();
    p0.put(0, 1);
    p1.put(1, 1);
    p2.put(2, 1);
    p3.put(3, 1);
    p6.put(6, 1);
    p7.put(7, 1);
  } else if (!TMAE) {
    // ---------------- epilogue: term slots -> fp32 sums -> fused update of the output rows ----------------
    const int ew = warp - kTcSumEpiW, q = warp & 3, hh = ew >> 2;  // lane quarter, 32-output half
    const unsigned lane_base = tmem + ((unsigned)(32 * q) << 16);
    const int nslots = gridDim.x * kTcSumEpi, slot = blockIdx.x * kTcSumEpi + ew;
    const int n = g.len;
    double nrm[3] = {0.0, 0.0, 0.0};
    bool bad = false;
    int norm_b = -1;
    RingPos sl;
    StrideWalk walk(g.len, LT, batch, kTcTS);
    Chunk ch;
    while (walk.next(ch, kTcTS)) {
      if (ch.b != norm_b) {
        if (norm_b >= 0) kb_warp_finish_f<MODE>(e, nrm, bad, norm_b, nslots, slot, lane);
        nrm[0] = nrm[1] = nrm[2] = 0.0;
        bad = false;
        norm_b = ch.b;
      }
      const bool live = 32 * hh < ch.cnt;
      // the image's scalars, loaded now so their latency hides behind the term accumulation
      double sc_L = 0.0, sc_d = 1.0;
      if constexpr (MODE == EPI_UPDATE) {
        sc_L = e.L[ch.b];
        sc_d = e.denom[ch.b];
      }
      if constexpr (MODE == EPI_POWER) sc_L = e.vnw2 ? e.vnw2[ch.b] : 1.0;
#if !KB_TC_NO_PREFETCH
      {  // this chunk's epilogue operand rows go to L2 now, while its r terms accumulate: the
         // epilogue's own loads then wait for L2, not DRAM (short-band batches are bound by them)
        const int lp = ch.lt * 128 + 32 * q + lane;
        if (live && lp < g.other) {
          const long long at = (long long)ch.b * e.bstride + (long long)lp * n + ch.s0 + 32 * hh;
          if constexpr (MODE == EPI_RESID) prefetch_l2(e.bsub + at);
          if constexpr (MODE == EPI_UPDATE) {
            prefetch_l2(e.y + at);
            prefetch_l2(e.x + at);
          }
          if constexpr (MODE == EPI_POWER) prefetch_l2(e.vin + at);
        }
      }
#endif
      float sum[32];
      for (int term = 0; term < r; ++term, sl.advance(kTcSumSlots)) {
        mbar_wait_idle(&slot_full[sl.i], sl.phase, 2000);
        __syncwarp();
        tc_fence_after();
        if (live) {
          const unsigned col = lane_base + sl.i * 64 + 32 * hh;
          float v[16];
#pragma unroll
          for (int p2 = 0; p2 < 2; ++p2) {
            tc_ld16(col + 16 * p2, v);
#pragma unroll
            for (int i = 0; i < 16; ++i) sum[16 * p2 + i] = term ? __fadd_rn(sum[16 * p2 + i], v[i]) : v[i];
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&slot_empty[sl.i]);
      }
      const int l = ch.lt * 128 + 32 * q + lane;
      if (live && l < g.other && !(g.dbg & 2)) {
        const float Lb = (float)sc_L, db = (float)sc_d, rd = 1.f / db;
        const double vs = MODE == EPI_POWER && e.vnw2 ? sqrt(sc_L) : 1.0;
        const long long row = (long long)ch.b * e.bstride + (long long)l * n + ch.s0 + 32 * hh;
        const bool fold_edge = e.foldH > 0 && (ch.s0 < e.foldH || ch.s0 + kTcTS > n - e.foldH);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c = ch.cnt - 32 * hh - 8 * j;
          if (c <= 0) break;
          float v8[8] = {sum[8 * j], sum[8 * j + 1], sum[8 * j + 2], sum[8 * j + 3],
                         sum[8 * j + 4], sum[8 * j + 5], sum[8 * j + 6], sum[8 * j + 7]};
          if (fold_edge) {  // exact adjoint fold corrections of the reflective axis (edge chunks)
            const int FH = e.foldH;
            const float* f = e.fold + ((long long)ch.b * g.other + l) * (2 * FH);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int qi = ch.s0 + 32 * hh + 8 * j + i;
              if (qi < FH) v8[i] += f[qi];
              else if (qi >= n - FH && qi < n) v8[i] += f[qi - (n - 2 * FH)];
            }
          }
          tc_sum_epi8<MODE, NORMS>(v8, e, row + 8 * j, min(8, c), Lb, db, rd, vs, nrm, bad);
        }
      }
    }
    if (norm_b >= 0) kb_warp_finish_f<MODE>(e, nrm, bad, norm_b, nslots, slot, lane);
  } else {
    // ---------------- epilogue with TMA-staged operands: term slots -> fp32 sums -> boxes ----------------
    constexpr int NPL = MODE == EPI_UPDATE ? 2 : 1;
    const int ew = warp - kTcSumEpiW, q = warp & 3, hh = ew >> 2;  // lane quarter, 32-output half
    const unsigned lane_base = tmem + ((unsigned)(32 * q) << 16);
    const int nslots = gridDim.x * kTcSumEpi, slot = blockIdx.x * kTcSumEpi + ew;
    const int n = g.len;
    unsigned char* mybox = ebuf + (size_t)ew * NPL * 4096;
    const CUtensorMap* pm0 = &emap0;  // parameter-space addresses (see kb_tc1.cuh)
    const CUtensorMap* pm1 = &emap1;
    double nrm[3] = {0.0, 0.0, 0.0};
    bool bad = false;
    int norm_b = -1, chunk = 0;
    RingPos sl;
    StrideWalk walk(g.len, LT, batch, kTcTS);
    auto load_boxes = [&](const Chunk& c2) {
      if (MODE == EPI_PLAIN) return;
      if (lane == 0) {
        mbar_arrive_expect_tx(&eful[ew], NPL * 4096);
        const int c0 = c2.s0 + 32 * hh, r0 = c2.lt * 128 + 32 * q;
        tma_load_3d(mybox, pm0, c0, r0, c2.b, &eful[ew]);
        if (NPL == 2) tma_load_3d(mybox + 4096, pm1, c0, r0, c2.b, &eful[ew]);
      }
    };
    {
      StrideWalk peek = walk;
      Chunk c2;
      if (peek.next(c2, kTcTS)) load_boxes(c2);
    }
    Chunk ch;
    while (walk.next(ch, kTcTS)) {
      if (ch.b != norm_b) {
        if (norm_b >= 0) kb_warp_finish_f<MODE>(e, nrm, bad, norm_b, nslots, slot, lane);
        nrm[0] = nrm[1] = nrm[2] = 0.0;
        bad = false;
        norm_b = ch.b;
      }
      const bool live = 32 * hh < ch.cnt;
      double sc_L = 0.0, sc_d = 1.0;
      if constexpr (MODE == EPI_UPDATE) {
        sc_L = e.L[ch.b];
        sc_d = e.denom[ch.b];
      }
      if constexpr (MODE == EPI_POWER) sc_L = e.vnw2 ? e.vnw2[ch.b] : 1.0;
      float sum[32];
      for (int term = 0; term < r; ++term, sl.advance(kTcSumSlots)) {
        mbar_wait_idle(&slot_full[sl.i], sl.phase, 2000);
        __syncwarp();
        tc_fence_after();
        if (live) {
          const unsigned col = lane_base + sl.i * 64 + 32 * hh;
          float v[16];
#pragma unroll
          for (int p2 = 0; p2 < 2; ++p2) {
            tc_ld16(col + 16 * p2, v);
#pragma unroll
            for (int i = 0; i < 16; ++i) sum[16 * p2 + i] = term ? __fadd_rn(sum[16 * p2 + i], v[i]) : v[i];
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&slot_empty[sl.i]);
      }
      const int l = ch.lt * 128 + 32 * q + lane;
      const bool row_ok = l < g.other;
      if (MODE != EPI_PLAIN) mbar_wait_lazy(&eful[ew], chunk & 1, 2000);
      if (live && !(g.dbg & 2)) {
        const float Lb = (float)sc_L, db = (float)sc_d, rd = 1.f / db;
        const double vs = MODE == EPI_POWER && e.vnw2 ? sqrt(sc_L) : 1.0;
        const float beta = (float)e.beta;
        const bool fold_edge = e.foldH > 0 && (ch.s0 < e.foldH || ch.s0 + kTcTS > n - e.foldH);
        if (fold_edge && row_ok) {  // exact adjoint fold corrections of the reflective axis (edge chunks)
          const int FH = e.foldH;
          const float* fz = e.fold + ((long long)ch.b * g.other + l) * (2 * FH);
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int qi = ch.s0 + 32 * hh + i;
            if (qi < FH) sum[i] += fz[qi];
            else if (qi >= n - FH && qi < n) sum[i] += fz[qi - (n - 2 * FH)];
          }
        }
#pragma unroll
        for (int c16 = 0; c16 < 8; ++c16) {
          const unsigned off = (unsigned)lane * 128 + (unsigned)((c16 ^ (lane & 7)) * 16);
          float4* p0 = reinterpret_cast<float4*>(mybox + off);
          const float* vv = sum + 4 * c16;
          const int col0 = 32 * hh + 4 * c16;
          float4 a0 = *p0;
          float* u = reinterpret_cast<float*>(&a0);
          if constexpr (MODE == EPI_PLAIN) {
            *p0 = make_float4(vv[0], vv[1], vv[2], vv[3]);
          } else if constexpr (MODE == EPI_RESID) {
            *p0 = make_float4(__fsub_rn(vv[0], u[0]), __fsub_rn(vv[1], u[1]), __fsub_rn(vv[2], u[2]),
                              __fsub_rn(vv[3], u[3]));
          } else if constexpr (MODE == EPI_UPDATE) {
            float4* p1 = reinterpret_cast<float4*>(mybox + 4096 + off);
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
              u[i] = __fadd_rn(x, __fmul_rn(beta, d));
              w[i] = x;
            }
            *p0 = a0;
            *p1 = a1;
          } else {  // EPI_POWER
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
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0 && live && !(g.dbg & 2)) {
        const int c0 = ch.s0 + 32 * hh, r0 = ch.lt * 128 + 32 * q;
        if constexpr (MODE == EPI_UPDATE) {
          tma_store_3d(pm0, mybox, c0, r0, ch.b);
          tma_store_3d(pm1, mybox + 4096, c0, r0, ch.b);
        } else if constexpr (MODE == EPI_PLAIN) {
          tma_store_3d(pm0, mybox, c0, r0, ch.b);
        } else {
          tma_store_3d(pm1, mybox, c0, r0, ch.b);
        }
        bulk_commit();
      }
      if (lane == 0) bulk_wait_read<0>();  // the box may be refilled
      __syncwarp();
      {
        StrideWalk peek = walk;
        Chunk c2;
        if (peek.next(c2, kTcTS)) load_boxes(c2);
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

// ------------------------------------------------------------------------------------------
// Roofline denominator for the tcgen05 passes (kb_fma_peak, KB_PEAK_TC_TF32): two warps per CTA
// each issue `iters` kind::tf32 MMAs of M = 128, N = 256, K = 8 (A and B from shared memory,
// K-major INTERLEAVE) into their own 256-column accumulator; one CTA per SM.
// ------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(128, 1) kb_tc_burn(int iters, float* out) {
  __shared__ __align__(1024) float ops[3 * 1024];  // A: 4 KB, B: 8 KB
  __shared__ unsigned long long done;
  __shared__ unsigned tmem_base;
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  for (int i = tid; i < 3 * 1024; i += 128) ops[i] = 1.f + 1e-3f * (float)((i * 37) & 255);
  if (tid == 0) {
    mbar_init(&done, 2);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const unsigned tmem = __shfl_sync(0xffffffffu, tmem_base, 0);
  if (warp < 2) {
    const unsigned long long ad = tc_desc(smem_u32(ops), 128, 256, 0), bd = tc_desc(smem_u32(ops + 1024), 128, 256, 0);
    constexpr unsigned idesc = (1u << 4) | (2u << 7) | (2u << 10) | (32u << 17) | (8u << 24);
    const unsigned d = tmem + 256 * warp;
    for (int i = 0; i < iters; ++i)
      asm volatile(
          "{\n.reg .pred p, q;\nsetp.ne.b32 q, %4, 0;\nelect.sync _|p, 0xffffffff;\n"
          "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, q;\n}" ::"r"(d),
          "l"(ad), "l"(bd), "r"(idesc), "r"(i));
    tc_commit_elect(&done);
  }
  mbar_wait(&done, 0);
  tc_fence_after();
  if (warp == 0) {
    float v[16];
    tc_ld16(tmem, v);  // keep the result observable
    if (tid == 0 && blockIdx.x == 0) out[0] = v[0];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

}  // namespace kb
