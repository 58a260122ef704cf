// tcgen05 kind::tf32 probe (not shipped): validates the shared-memory descriptor encodings used by
// the tensor-core pass kernels against a CPU GEMM.
//   D[m][n] = sum_k A[m][k] * B[n][k],  M = 128, N = 16, K = 64 (8 MMAs of K = 8)
//   A: global [K][M] fp32 (M contiguous) -> TMA SWIZZLE_128B boxes {32 cols, 64 rows} -> MN-major
//      canonical SW128 (LBO = 8 KB between 32-column blocks, SBO = 1 KB between 8-row groups)
//   B: built by threads as K-major INTERLEAVE core matrices (8 n x 4 k, 128 B), LBO 128 B (k),
//      SBO 256 B (n) per 8-deep K-step brick of 512 B
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_));       \
      exit(1);                                                                       \
    }                                                                                \
  } while (0)

constexpr int M = 128, N = 16, K = 64;

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ unsigned long long make_desc(unsigned addr, unsigned lbo, unsigned sbo, unsigned layout) {
  unsigned long long d = 0;
  d |= (unsigned long long)((addr >> 4) & 0x3FFF);
  d |= (unsigned long long)((lbo >> 4) & 0x3FFF) << 16;
  d |= (unsigned long long)((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;  // version 1 (Blackwell)
  d |= (unsigned long long)(layout & 7) << 61;
  return d;
}

__global__ void probe(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap kmap,
                      const __grid_constant__ CUtensorMap amap32, const float* __restrict__ Bg, float* __restrict__ Dg,
                      unsigned idesc, int* status, int dbg, const float* __restrict__ Ag, int amode,
                      unsigned getenv_lbo, unsigned getenv_sbo, int bmode) {
  extern __shared__ __align__(1024) unsigned char smem[];
  __shared__ unsigned long long bar_a, bar_mma;
  __shared__ unsigned tmem_base;
  // 1024-byte aligned base (the dynamic window follows the static shared variables)
  unsigned char* base = smem + ((1024 - (smem_u32(smem) & 1023)) & 1023);
  float* sa = reinterpret_cast<float*>(base);               // 4 blocks x [64 rows][32] = 32 KB
  float* sb = reinterpret_cast<float*>(base + 32768);       // 8 bricks x 512 B
  if (threadIdx.x == 0 && dbg) printf("smem base mod 1024 = %u\n", smem_u32(smem) & 1023);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar_a)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar_mma)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // B bricks: brick kk holds B[n][8kk + k]: core (nb, kc) at nb*256 + kc*128, row i at 16 B
  for (int idx = tid; idx < N * K; idx += blockDim.x) {
    const int n = idx / K, k = idx % K;
    const int kk = k / 8, kin = k % 8, kc = kin / 4, ke = kin % 4, nb = n / 8, ni = n % 8;
    if (bmode == 0) sb[kk * 128 + nb * 64 + kc * 32 + ni * 4 + ke] = Bg[n * K + k];
    // MN-major INTERLEAVE: core (nb4 = n/4) = 8 k-rows x 4 n (128 B), cores along n at 128 B
    else sb[kk * 128 + (n / 4) * 32 + kin * 4 + (n % 4)] = Bg[n * K + k];
  }
  float* sak = reinterpret_cast<float*>(base + 40960);  // K-major A: 8 bricks x (128 m x 8 k) = 8 x 4 KB
  if (amode == 1) {  // brick kk: core (mb, kc) at mb*256 + kc*128 B? no: 16 m-blocks x 2 k-chunks
    for (int idx = tid; idx < M * K; idx += blockDim.x) {
      const int m = idx % M, k = idx / M;
      const int kk = k / 8, kin = k % 8, kc = kin / 4, ke = kin % 4, mb = m / 8, mi = m % 8;
      // core (mb, kc) at mb*SBO(256 B) + kc*LBO(128 B); 16 m-blocks -> 4 KB per brick
      sak[kk * 1024 + mb * 64 + kc * 32 + mi * 4 + ke] = Ag[k * M + m];
    }
  }
  if (amode == 2) {  // MN-major INTERLEAVE: core (mb) = 8 k-rows x 4 m (128 B), cores along m at 128 B
    for (int idx = tid; idx < M * K; idx += blockDim.x) {
      const int m = idx % M, k = idx / M;
      const int kk = k / 8, kin = k % 8, mb = m / 4, me = m % 4;
      sak[kk * 1024 + mb * 32 + kin * 4 + me] = Ag[k * M + m];
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const unsigned tmem = tmem_base;
  if (warp < 4 && dbg) {  // debug: seed D with known values and accumulate onto them
    unsigned v[16];
    for (int n = 0; n < 16; ++n) v[n] = __float_as_uint(1000.f * n + 32 * warp + lane);
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
            tmem + ((unsigned)(32 * warp) << 16)),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  if (amode == 5 && warp < 4) {  // A[m][k] -> TMEM lane m, column 32 + k
    const int m = 32 * warp + lane;
    for (int k0 = 0; k0 < K; k0 += 16) {
      unsigned v[16];
      for (int i = 0; i < 16; ++i) v[i] = __float_as_uint(Ag[(k0 + i) * M + m]);
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
              tmem + ((unsigned)(32 * warp) << 16) + 32 + k0),
          "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
          "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0 && amode == 5) {
    for (int kk = 0; kk < K / 8; ++kk) {
      const unsigned long long bd = make_desc(smem_u32(sb) + kk * 512, 128, 256, 0);
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}" ::"r"(tmem),
          "r"(tmem + 32 + 8 * kk), "l"(bd), "r"(idesc), "r"(dbg ? 1 : kk));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar_mma))
                 : "memory");
  } else if (tid == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar_a)), "r"(32768u) : "memory");
    if (amode == 3) {  // two boxes {32 K, 128 M} of the K-contiguous A^T copy
      for (int j = 0; j < 2; ++j)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                smem_u32(sa + j * 4096)),
            "l"(&kmap), "r"(32 * j), "r"(0), "r"(smem_u32(&bar_a))
            : "memory");
    } else {
      for (int j = 0; j < 4; ++j)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                smem_u32(sa + j * 2048)),
            "l"(amode == 4 ? &amap32 : &amap), "r"(32 * j), "r"(0), "r"(smem_u32(&bar_a))
            : "memory");
    }
    asm volatile(
        "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}" ::"r"(smem_u32(&bar_a))
        : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    for (int kk = 0; kk < K / 8; ++kk) {
      const unsigned lbo = getenv_lbo, sbo = getenv_sbo;
      const unsigned long long ad = amode == 4 ? make_desc(smem_u32(sa) + kk * 1024, lbo ? lbo : 8192, sbo ? sbo : 512, 1)
                                  : amode == 3 ? make_desc(smem_u32(sa) + (kk / 4) * 16384 + (kk % 4) * 32, lbo ? lbo : 16, sbo ? sbo : 1024, 2)
                                  : amode == 1 ? make_desc(smem_u32(sak) + kk * 4096, 128, 256, 0)
                                  : amode == 2 ? make_desc(smem_u32(sak) + kk * 4096, lbo ? lbo : 4096, sbo ? sbo : 128, 0)
                                               : make_desc(smem_u32(sa) + kk * 1024, lbo ? lbo : 8192, sbo ? sbo : 1024, 2);
      const unsigned long long bd = bmode == 0 ? make_desc(smem_u32(sb) + kk * 512, 128, 256, 0 /*SWIZZLE_NONE*/)
                                               : make_desc(smem_u32(sb) + kk * 512, 512, 128, 0);
      asm volatile(
          "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
          "l"(ad), "l"(bd), "r"(idesc), "r"(dbg ? 1 : kk));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar_mma))
                 : "memory");
  }
  __syncwarp();
  // all threads wait for the MMAs (bounded spin: report a hang instead of hanging the GPU)
  {
    unsigned done = 0;
    for (long it = 0; it < (1l << 26) && !done; ++it)
      asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\nselp.u32 %0, 1, 0, p;\n}"
                   : "=r"(done)
                   : "r"(smem_u32(&bar_mma))
                   : "memory");
    if (!done) {
      if (tid == 0) *status = 1;
      return;
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp < 4) {
    unsigned v[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(tmem + ((unsigned)(32 * warp) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int m = 32 * warp + lane;
    for (int n = 0; n < N; ++n) Dg[m * N + n] = __uint_as_float(v[n]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

int main() {
  std::vector<float> A(K * M), B(N * K), D(M * N);
  srand(3);
  auto rnd = [] { return (float)((rand() % 2001) - 1000) / 512.0f; };  // exact in tf32
  for (auto& x : A) x = rnd();
  for (auto& x : B) x = rnd();
  float *dA, *dB, *dD;
  int* dS;
  CK(cudaMalloc(&dA, A.size() * 4));
  CK(cudaMalloc(&dB, B.size() * 4));
  CK(cudaMalloc(&dD, D.size() * 4));
  CK(cudaMalloc(&dS, 4));
  CK(cudaMemset(dS, 0, 4));
  CK(cudaMemset(dD, 0, D.size() * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
  CUtensorMap amap;
  const cuuint64_t dims[2] = {M, K};
  const cuuint64_t strides[1] = {M * 4};
  const cuuint32_t box[2] = {32, K};
  const cuuint32_t es[2] = {1, 1};
  if (enc(&amap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dA, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("tensor map encode failed\n");
    return 1;
  }
  // K-contiguous copy of A ([M][K]) and its map for the K-major SW128 mode
  std::vector<float> AT(M * K);
  for (int m = 0; m < M; ++m)
    for (int k = 0; k < K; ++k) AT[m * K + k] = A[k * M + m];
  float* dAT;
  CK(cudaMalloc(&dAT, AT.size() * 4));
  CK(cudaMemcpy(dAT, AT.data(), AT.size() * 4, cudaMemcpyHostToDevice));
  CUtensorMap kmap;
  {
    const cuuint64_t kd[2] = {K, M};
    const cuuint64_t ks[1] = {K * 4};
    const cuuint32_t kb[2] = {32, M};
    if (enc(&kmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dAT, kd, ks, kb, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
      printf("kmap encode failed\n");
      return 1;
    }
  }
  CUtensorMap amap32;
  if (enc(&amap32, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dA, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS) {
    printf("amap32 encode failed\n");
    return 1;
  }
  unsigned idesc = 0;
  idesc |= 1u << 4;           // D format F32
  idesc |= 2u << 7;           // A TF32
  idesc |= 2u << 10;          // B TF32
  idesc |= 1u << 15;          // A MN-major
  idesc |= 0u << 16;          // B K-major
  idesc |= (unsigned)(N >> 3) << 17;
  idesc |= (unsigned)(M >> 4) << 24;
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 81 * 1024));
  const int dbg = getenv("DBG") ? 1 : 0;
  const int amode = getenv("AMODE") ? atoi(getenv("AMODE")) : 0;
  if (amode == 1 || amode == 3 || amode == 5) idesc &= ~(1u << 15);  // A K-major (TMEM A: no major bit)
  const unsigned lbo = getenv("LBO") ? atoi(getenv("LBO")) : 0, sbo = getenv("SBO") ? atoi(getenv("SBO")) : 0;
  const int bmode = getenv("BMODE") ? atoi(getenv("BMODE")) : 0;
  if (bmode == 1) idesc |= 1u << 16;  // B MN-major
  probe<<<1, 128, 81 * 1024>>>(amap, kmap, amap32, dB, dD, idesc, dS, dbg, dA, amode, lbo, sbo, bmode);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  int st = 0;
  CK(cudaMemcpy(&st, dS, 4, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
  double maxerr = 0, maxref = 0;
  int bad = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = getenv("DBG") ? 1000.0 * n + m : 0.0;
      for (int k = 0; k < K; ++k) ref += (double)A[k * M + m] * B[n * K + k];
      const double err = fabs(ref - D[m * N + n]);
      if (err > 1e-3 * (1 + fabs(ref)) && bad++ < 5) printf("m %d n %d got %f want %f\n", m, n, D[m * N + n], ref);
      maxerr = fmax(maxerr, err);
      maxref = fmax(maxref, fabs(ref));
    }
  printf("status %d  max err %.3e (max |D| %.3e)  bad %d / %d  -> %s\n", st, maxerr, maxref, bad, M * N,
         (st == 0 && bad == 0) ? "PASS" : "FAIL");
  return 0;
}
