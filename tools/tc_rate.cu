// tcgen05 kind::tf32 issue-rate probe (not shipped): `streams` warps per CTA each issue `iters`
// MMAs (M = 128, N = 16/32, K = 8, A from tensor memory) into their own accumulator, with three
// issue styles (lane-0 loop, whole-warp elect per MMA, three MMAs per elect).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned long long make_desc(unsigned addr, unsigned lbo, unsigned sbo, unsigned layout) {
  unsigned long long d = (unsigned long long)((addr >> 4) & 0x3FFF);
  d |= (unsigned long long)((lbo >> 4) & 0x3FFF) << 16;
  d |= (unsigned long long)((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;
  d |= (unsigned long long)(layout & 7) << 61;
  return d;
}

__global__ void rate(int iters, unsigned idesc, int amode, int streams, long long* cycles, int naccum, int ncols) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ unsigned long long bar;
  __shared__ unsigned tmem_base;
  __shared__ unsigned long long dummy[32];
  if (threadIdx.x < 32)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&dummy[threadIdx.x])), "r"(1 << 20));
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 1e-3f * (i & 63);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(streams));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tmem = tmem_base;
  long long t0 = clock64();
  if (warp < streams) {
    const unsigned long long bd = make_desc(smem_u32(smem), 128, 256, 0);
    const unsigned d = tmem + warp * ncols, a = tmem + 504;
    if (amode == 0) {  // lane 0 alone walks the loop (as kb_pass_split_tc's issuers)
      if ((tid & 31) == 0)
        for (int i = 0; i < iters; ++i)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(d),
                       "r"(a), "l"(bd + (i & 3) * 64), "r"(idesc), "r"(i));
    } else if (amode == 1) {  // whole warp, elect per MMA
      for (int i = 0; i < iters; ++i) {
        asm volatile("{\n.reg .pred p, q;\nsetp.ne.b32 q, %4, 0;\nelect.sync _|p, 0xffffffff;\n"
                     "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, q;\n}" ::"r"(d),
                     "r"(a), "l"(bd + (i & 3) * 64), "r"(idesc), "r"(i));
      }
    } else if (amode >= 3) {  // kb_pass_split_tc's pattern: 3 terms x 3xTF32 per elect
      // accumulators d, d + 64, d + 128 (mode 3: lo A at column 496, hi at 504; mode 4: one A column)
      const unsigned dd = tmem + warp * 16, ahi = tmem + 504, alo = amode == 3 ? tmem + 496 : ahi;
      for (int i = 0; i < iters; i += 9) {
        const unsigned long long bh = bd + ((i / 9) & 3) * 64, bh1 = bh + 256, bh2 = bh1 + 256, lo = 32;
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
            "@p tcgen05.mma.cta_group::1.kind::tf32 [%2], [%3], %7, %11, 1;\n}" ::"r"(dd),
            "r"(dd + 64), "r"(dd + 128), "r"(ahi), "r"(alo), "l"(bh), "l"(bh1), "l"(bh2), "l"(bh + lo), "r"(i),
            "l"(bh1 + lo), "r"(idesc), "l"(bh2 + lo));
        if (amode == 5 && (i / 9) % 2 == 1)  // commit per two K-steps (kb_pass_split_tc's a_free)
          asm volatile("{\n.reg .pred p;\nelect.sync _|p, 0xffffffff;\n"
                       "@p tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(
                           smem_u32(&dummy[warp]))
                       : "memory");
      }
    } else {  // whole warp, three MMAs per asm block (one 3xTF32 K-step)
      for (int i = 0; i < iters; i += 3) {
        asm volatile("{\n.reg .pred p, q;\nsetp.ne.b32 q, %4, 0;\nelect.sync _|p, 0xffffffff;\n"
                     "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, q;\n"
                     "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %5, %3, 1;\n"
                     "@p tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %6, %3, 1;\n}" ::"r"(d),
                     "r"(a), "l"(bd + (i & 3) * 64), "r"(idesc), "r"(i), "l"(bd + 32), "l"(bd + 96));
      }
    }
    if ((tid & 31) == 0)
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
  }
  if (tid == 0) {
    asm volatile("{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(smem_u32(&bar)) : "memory");
    cycles[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

int main(int argc, char** argv) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* dc;
  cudaMalloc(&dc, sms * sizeof(long long));
  cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int amode : {0, 1, 2, 3}) {
    for (int N : {16, 32, 64}) {
      for (int streams : {1, 4, 8}) {
        if (streams * N > 496 || (amode >= 3 && streams > 4)) continue;
        const int iters = 3078;
        unsigned idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((unsigned)(N >> 3) << 17) | (8u << 24);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        rate<<<sms, 800, 100 * 1024>>>(63, idesc, amode, streams, dc, 1, N);
        cudaEventRecord(e0);
        rate<<<sms, 800, 100 * 1024>>>(iters, idesc, amode, streams, dc, 1, N);
        cudaEventRecord(e1);
        cudaError_t err = cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        long long c0;
        cudaMemcpy(&c0, dc, 8, cudaMemcpyDeviceToHost);
        const double flop = 2.0 * 128 * N * 8 * (double)iters * streams * sms;
        printf("mode %d N %2d streams %2d: %7.1f TFLOP/s  %6.1f clk/MMA/stream  %5.1f clk/MMA/SM (%s)\n", amode, N,
               streams, flop / ms / 1e9, (double)c0 / iters, (double)c0 / iters / streams, cudaGetErrorString(err));
      }
    }
  }
  return 0;
}
