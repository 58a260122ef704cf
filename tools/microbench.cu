// Throughput microbenchmarks used to pick the fp64 / fp32 inner-loop instruction (not shipped).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_k(double* out, int iters, double a, double b) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(x[i], a, b);
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == -1.2345) out[0] = s;
}

__global__ void ffma_k(float* out, int iters, float a, float b) {
  float x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fmaf(x[i], a, b);
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == -1.2345f) out[0] = s;
}

// FFMA with a distinct multiplicand per chain (3 distinct registers per instruction)
__global__ void ffma3_k(float* out, int iters, float a) {
  float x[8], y[8];
  for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x + i; y[i] = a + i * 1e-3f; }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fmaf(y[i], x[(i + 1) & 7], x[i]);
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == -1.2345f) out[0] = s;
}

// DMMA m8n8k4: 4 independent accumulators per warp
__global__ void dmma_k(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = threadIdx.x * 2e-3;
  double c[4][2];
  for (int i = 0; i < 4; ++i) c[i][0] = c[i][1] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  if (s == -1.2345) out[0] = s;
}

// DMMA with distinct A/B registers per MMA (8 accumulators, 4 A x 2 B operands)
__global__ void dmma2_k(double* out, int iters) {
  double a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int i = 0; i < 2; ++i) b[i] = threadIdx.x * 2e-3 - i;
  double c[8][2];
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a[i & 3]), "d"(b[i >> 2]));
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == -1.2345) out[0] = s;
}

// DMMA fed from shared memory every iteration (the banded-pass pattern)
__global__ void dmma_smem_k(double* out, int iters) {
  __shared__ double sm[64 * 36];
  for (int i = threadIdx.x; i < 64 * 36; i += blockDim.x) sm[i] = i * 1e-4;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double c[16][2];
  for (int i = 0; i < 16; ++i) c[i][0] = c[i][1] = 0;
  for (int it = 0; it < iters; ++it) {
    const int base = (it & 7) * 4;
    double A[4], B[4];
#pragma unroll
    for (int g = 0; g < 4; ++g) A[g] = sm[(base + g) * 36 + (lane & 3)];
#pragma unroll
    for (int j = 0; j < 4; ++j) B[j] = sm[(base + (lane & 3)) * 36 + 8 * j + (lane >> 2)];
#pragma unroll
    for (int g = 0; g < 4; ++g)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[g * 4 + j][0]), "+d"(c[g * 4 + j][1]) : "d"(A[g]), "d"(B[j]));
  }
  double s = 0;
  for (int i = 0; i < 16; ++i) s += c[i][0] + c[i][1];
  if (s == -1.2345) out[0] = s;
}

// DFMA with 3 distinct registers and changing multiplicands
__global__ void dfma3_k(double* out, int iters, double a) {
  double x[8], y[8];
  for (int i = 0; i < 8; ++i) { x[i] = threadIdx.x + i; y[i] = a + i * 1e-3; }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fma(y[i], x[(i + 1) & 7], x[i]);
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == -1.2345) out[0] = s;
}

// the split-pass inner loop alone: tile [128][36] in smem, G terms x 4 n-tiles, 18 chunks
template <int G>
__global__ void __launch_bounds__(256, 2) dmma_split_k(double* out, int reps) {
  __shared__ double xs[136 * 36];
  __shared__ double cp[4 * 96];
  for (int i = threadIdx.x; i < 136 * 36; i += 256) xs[i] = i * 1e-5;
  for (int i = threadIdx.x; i < 4 * 96; i += 256) cp[i] = i * 1e-3;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ar = lane >> 2, ac = lane & 3;
  double D[G][4][2] = {};
  const double* xb = xs + (warp * 8 + ac) * 36 + ar;
  const double* cb = cp + 8 + ac - ar;
  for (int rep = 0; rep < reps; ++rep) {
#pragma unroll 2
    for (int c = 0; c < 18; ++c) {
      double A[G], B[4];
#pragma unroll
      for (int g = 0; g < G; ++g) A[g] = cb[g * 96 + 4 * c];
#pragma unroll
      for (int j = 0; j < 4; ++j) B[j] = xb[4 * c * 36 + 8 * j];
#pragma unroll
      for (int g = 0; g < G; ++g)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                       : "+d"(D[g][j][0]), "+d"(D[g][j][1]) : "d"(B[j]), "d"(A[g]));
    }
  }
  double s = 0;
  for (int g = 0; g < G; ++g)
    for (int j = 0; j < 4; ++j) s += D[g][j][0] + D[g][j][1];
  if (s == -1.2345) out[0] = s;
}

// legacy warp-level TF32 MMA (m16n8k8): 8 independent accumulators per warp
__global__ void tf32_k(float* out, int iters) {
  unsigned a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(threadIdx.x * 1e-3f + i);
  for (int i = 0; i < 2; ++i) b[i] = __float_as_uint(threadIdx.x * 2e-3f - i);
  float c[8][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == -1.2345f) out[0] = s;
}

// legacy warp-level BF16 MMA (m16n8k16)
__global__ void bf16_k(float* out, int iters) {
  unsigned a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = 0x3f803f80u + threadIdx.x + i;
  for (int i = 0; i < 2; ++i) b[i] = 0x3f803f80u + threadIdx.x - i;
  float c[8][4] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (s == -1.2345f) out[0] = s;
}

// DMMA with NACC independent accumulators per warp, operands in registers only
template <int NACC>
__global__ void dmma_ilp_k(double* out, int iters) {
  double a[4], b[4];
  for (int i = 0; i < 4; ++i) { a[i] = threadIdx.x * 1e-3 + i; b[i] = threadIdx.x * 2e-3 - i; }
  double c[NACC][2];
  for (int i = 0; i < NACC; ++i) c[i][0] = c[i][1] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < NACC; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a[i & 3]), "d"(b[(i >> 2) & 3]));
  }
  double s = 0;
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == -1.2345) out[0] = s;
}

// half the warps DMMA, half DFMA: do the two FP64 paths share one pipe?
__global__ void mixed_k(double* out, int iters) {
  const int warp = threadIdx.x >> 5;
  double s = 0;
  if (warp & 1) {
    double a = threadIdx.x * 1e-3, b = threadIdx.x * 2e-3;
    double c[8][2];
    for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    }
    for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  } else {
    double x[8];
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x + i;
    // 64 DFMA per thread per DMMA-iteration keeps the flop count per warp equal (8 DMMA = 2048 FMA)
    for (int it = 0; it < iters * 8; ++it)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = fma(x[i], 0.999999, 1e-7);
    for (int i = 0; i < 8; ++i) s += x[i];
  }
  if (s == -1.2345) out[0] = s;
}

template <typename K, typename... A>
float timeit(K k, int blocks, int threads, A... a) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<<<blocks, threads>>>(a...);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<<<blocks, threads>>>(a...);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms / 5;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* dout;
  float* fout;
  cudaMalloc(&dout, 8);
  cudaMalloc(&fout, 8);
  for (int tpb : {128, 256, 512}) {
    const int blocks = sms * 8, it = 4096;
    float ms = timeit(dfma_k, blocks, tpb, dout, it, 0.999999, 1e-7);
    printf("DFMA  tpb=%d  %.2f TFLOP/s\n", tpb, 2.0 * 8 * it * (double)blocks * tpb / ms / 1e9);
    ms = timeit(ffma_k, blocks, tpb, fout, it * 4, 0.999999f, 1e-7f);
    printf("FFMA  tpb=%d  %.2f TFLOP/s\n", tpb, 2.0 * 8 * it * 4 * (double)blocks * tpb / ms / 1e9);
    ms = timeit(ffma3_k, blocks, tpb, fout, it * 4, 0.999999f);
    printf("FFMA3 tpb=%d  %.2f TFLOP/s\n", tpb, 2.0 * 8 * it * 4 * (double)blocks * tpb / ms / 1e9);
    ms = timeit(dmma_k, blocks, tpb, dout, it / 4);
    // per warp per mma: 8*8*4 = 256 FMA
    printf("DMMA  tpb=%d  %.2f TFLOP/s\n", tpb, 2.0 * 256 * 4 * (it / 4) * (double)blocks * (tpb / 32) / ms / 1e9);
    ms = timeit(dmma2_k, blocks, tpb, dout, it / 8);
    printf("DMMA2 tpb=%d  %.2f TFLOP/s\n", tpb, 2.0 * 256 * 8 * (it / 8) * (double)blocks * (tpb / 32) / ms / 1e9);
    ms = timeit(dmma_smem_k, blocks, tpb, dout, it / 16);
    printf("DMMAs tpb=%d  %.2f TFLOP/s\n", tpb, 2.0 * 256 * 16 * (it / 16) * (double)blocks * (tpb / 32) / ms / 1e9);
    ms = timeit(dfma3_k, blocks, tpb, dout, it, 0.999);
    printf("DFMA3 tpb=%d  %.2f TFLOP/s\n", tpb, 2.0 * 8 * it * (double)blocks * tpb / ms / 1e9);
  }
  {
    const int it = 256;
    // per warp pair: DMMA warp 8*it DMMAs (8*256*it FMA... 2048*it flop*?), DFMA warp 32*64*it FMA
    float ms = timeit(mixed_k, sms * 2, 512, dout, it);
    const double fl_dmma = 2.0 * 256 * 8 * it * (double)sms * 2 * 8;      // 8 DMMA warps per block
    const double fl_dfma = 2.0 * 32 * 8 * 8 * it * (double)sms * 2 * 8;   // 8 DFMA warps per block
    printf("MIXED DMMA+DFMA  %.1f TFLOP/s total (dmma share %.1f, dfma share %.1f)\n", (fl_dmma + fl_dfma) / ms / 1e9,
           fl_dmma / ms / 1e9, fl_dfma / ms / 1e9);
  }
  for (int wps : {4, 8, 16, 32}) {  // warps per SM (one block per SM)
    const int it = 512;
    float ms = timeit(dmma_ilp_k<8>, sms, 32 * wps, dout, it);
    printf("DMMA ilp8  %2d warps/SM  %.1f TFLOP/s\n", wps, 2.0 * 256 * 8 * it * (double)sms * wps / ms / 1e9);
    ms = timeit(dmma_ilp_k<16>, sms, 32 * wps, dout, it);
    printf("DMMA ilp16 %2d warps/SM  %.1f TFLOP/s\n", wps, 2.0 * 256 * 16 * it * (double)sms * wps / ms / 1e9);
    ms = timeit(dmma_ilp_k<32>, sms, 32 * wps, dout, it / 2);
    printf("DMMA ilp32 %2d warps/SM  %.1f TFLOP/s\n", wps, 2.0 * 256 * 32 * (it / 2) * (double)sms * wps / ms / 1e9);
  }
  for (int tpb : {128, 256, 512}) {
    const int blocks = sms * 4, it = 2048;
    float ms = timeit(tf32_k, blocks, tpb, fout, it);
    printf("TF32 mma.sync m16n8k8 tpb=%d  %.1f TFLOP/s\n", tpb, 2.0 * 16 * 8 * 8 * 8 * it * (double)blocks * (tpb / 32) / ms / 1e9);
    ms = timeit(bf16_k, blocks, tpb, fout, it);
    printf("BF16 mma.sync m16n8k16 tpb=%d  %.1f TFLOP/s\n", tpb, 2.0 * 16 * 8 * 16 * 8 * it * (double)blocks * (tpb / 32) / ms / 1e9);
  }
  {
    const int reps = 200;
    for (int bps : {1, 2}) {
      float ms = timeit(dmma_split_k<4>, sms * bps, 256, dout, reps);
      printf("DMMA split-loop G=4 %d warps/SM  %.2f TFLOP/s\n", 8 * bps, 2.0 * 256 * 16 * 18 * reps * (double)sms * bps * 8 / ms / 1e9);
      ms = timeit(dmma_split_k<3>, sms * bps, 256, dout, reps);
      printf("DMMA split-loop G=3 %d warps/SM  %.2f TFLOP/s\n", 8 * bps, 2.0 * 256 * 12 * 18 * reps * (double)sms * bps * 8 / ms / 1e9);
      ms = timeit(dmma_split_k<2>, sms * bps, 256, dout, reps);
      printf("DMMA split-loop G=2 %d warps/SM  %.2f TFLOP/s\n", 8 * bps, 2.0 * 256 * 8 * 18 * reps * (double)sms * bps * 8 / ms / 1e9);
      ms = timeit(dmma_split_k<1>, sms * bps, 256, dout, reps);
      printf("DMMA split-loop G=1 %d warps/SM  %.2f TFLOP/s\n", 8 * bps, 2.0 * 256 * 4 * 18 * reps * (double)sms * bps * 8 / ms / 1e9);
    }
  }
  return 0;
}
