// kb_norms.cuh — history reductions of the sFISTA loop (solvers.py:133-141 objective, :181 eta).
//
// With record_history the reference evaluates, per iteration, Phi(x) = 1/2 ||A x - b||^2 +
// lam^2/2 ||x||^2 and eta = ||x - truth|| / ||truth||. The update epilogue already reduces
// ||x_k||^2; this kernel adds ||A x - b||^2 and ||x - truth||^2 in one pass over A x, b, x and
// truth (fp64 accumulation for both dtypes), so a history iteration costs one extra forward
// application plus this pass and a 16-byte read-back instead of two image downloads.
// Deterministic: a fixed grid-stride assignment, fixed-order block reductions, and one block
// summing the per-block partials in block order.
#pragma once

namespace kb {

constexpr int kNormBlocks = 296, kNormThreads = 256;

template <typename T>
__global__ void __launch_bounds__(kNormThreads)
kb_resid_norms_k(const T* __restrict__ ax, const T* __restrict__ b, const T* __restrict__ x,
                 const T* __restrict__ truth, long long count, double* __restrict__ partial) {
  double s0 = 0.0, s1 = 0.0;
  for (long long i = (long long)blockIdx.x * kNormThreads + threadIdx.x; i < count;
       i += (long long)gridDim.x * kNormThreads) {
    const double r = (double)ax[i] - (double)b[i];
    s0 += r * r;
    if (truth) {
      const double e = (double)x[i] - (double)truth[i];
      s1 += e * e;
    }
  }
  __shared__ double red[kNormThreads / 32][2];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5][0] = s0;
    red[threadIdx.x >> 5][1] = s1;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double s = 0.0;
    for (int w = 0; w < kNormThreads / 32; ++w) s += red[w][threadIdx.x];
    partial[2 * blockIdx.x + threadIdx.x] = s;
  }
}

__global__ void kb_resid_norms_finish(const double* __restrict__ partial, int nblocks, double* __restrict__ out) {
  if (threadIdx.x < 2) {
    double s = 0.0;
    for (int k = 0; k < nblocks; ++k) s += partial[2 * k + threadIdx.x];
    out[threadIdx.x] = s;
  }
}

// <a, b> and ||b||^2 over `count` elements, fp64 accumulation, deterministic (the sharded power
// iteration's local reductions, solvers.py:124-125, all-reduced across ranks by the caller).
template <typename T>
__global__ void __launch_bounds__(kNormThreads)
kb_inner2_k(const T* __restrict__ a, const T* __restrict__ b, long long count, double* __restrict__ partial) {
  double s0 = 0.0, s1 = 0.0;
  for (long long i = (long long)blockIdx.x * kNormThreads + threadIdx.x; i < count;
       i += (long long)gridDim.x * kNormThreads) {
    const double bv = (double)b[i];
    s0 += (double)a[i] * bv;
    s1 += bv * bv;
  }
  __shared__ double red[kNormThreads / 32][2];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5][0] = s0;
    red[threadIdx.x >> 5][1] = s1;
  }
  __syncthreads();
  if (threadIdx.x < 2) {
    double s = 0.0;
    for (int w = 0; w < kNormThreads / 32; ++w) s += red[w][threadIdx.x];
    partial[2 * blockIdx.x + threadIdx.x] = s;
  }
}

}  // namespace kb
