// Cost of a persistent-pass skeleton inside a CUDA graph (not shipped): empty kernels with the
// pass kernels' launch shape, with and without dynamic shared memory and a taps prologue.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void empty_k(double* out) {
  extern __shared__ double sm[];
  if (threadIdx.x == 1234567) out[0] = sm[0];
}
__global__ void taps_k(const double* taps, double* out, int n) {
  extern __shared__ double sm[];
  const int tid = threadIdx.y * 32 + threadIdx.x;
  for (int i = tid; i < n; i += 256) sm[i] = taps[i];
  __syncthreads();
  if (sm[tid] == -1.2345) out[0] = sm[tid];
}

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
      return -1.f;                                                             \
    }                                                                          \
  } while (0)

template <typename F>
float graph_us(F launch, int reps) {
  static cudaStream_t s = nullptr;
  if (!s) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  cudaGraph_t g;
  cudaGraphExec_t ge;
  CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
  for (int r = 0; r < reps; ++r) launch(s);
  CK(cudaStreamEndCapture(s, &g));
  CK(cudaGraphInstantiate(&ge, g, 0));
  CK(cudaGraphLaunch(ge, s));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, s));
  CK(cudaGraphLaunch(ge, s));
  CK(cudaEventRecord(e1, s));
  CK(cudaEventSynchronize(e1));
  float ms;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return ms * 1000.f / reps;
}

int main() {
  double *out, *taps;
  cudaMalloc(&out, 8);
  cudaMalloc(&taps, 8 * 4096);
  cudaMemset(taps, 0, 8 * 4096);
  printf("attr %s\n", cudaGetErrorString(cudaFuncSetAttribute(empty_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024)));
  printf("attr %s\n", cudaGetErrorString(cudaFuncSetAttribute(taps_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024)));
  for (int grid : {148, 290, 296, 592}) {
    for (int smem : {0, 48 * 1024, 80 * 1024, 112 * 1024}) {
      if (grid > 296 && smem > 100 * 1024) continue;
      float us = graph_us([&](cudaStream_t s) { empty_k<<<grid, dim3(32, 8), smem, s>>>(out); }, 50);
      float us2 = graph_us([&](cudaStream_t s) { taps_k<<<grid, dim3(32, 8), smem + 4096, s>>>(taps, out, 440); }, 50);
      printf("grid %4d smem %6d  empty %.2f us  taps %.2f us\n", grid, smem, us, us2);
    }
  }
  return 0;
}
