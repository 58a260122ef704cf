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
  }
  return 0;
}
