// kb_blur.cuh — exact 2-D blur on the GPU: kronblur's blur_direct (psf.py:170-193).
//
// The reference pads X by ((rows - l, l - 1), (cols - q, q - 1)) with zeros (zero BC) or numpy's
// "symmetric" mode (reflective BC: edge sample repeated, a single fold since the PSF is no larger
// than the image), then for every NONZERO PSF entry (a, b) in row-major order (np.nonzero) adds
//     Y += P[a, b] * Xpad[rows-1-a : rows-1-a+m, cols-1-b : cols-1-b+n],
// i.e. per pixel  Y[i][j] = (...((0 + P[a0,b0]*X~[i+l-1-a0][j+q-1-b0]) + P[a1,b1]*X~[...]) ...)
// with the product and the sum rounded separately (numpy evaluates the product array first).
// The kernel performs exactly that sequence per pixel (__dmul_rn / __dadd_rn, no contraction,
// zero entries skipped), so its output is bit-identical to the reference for any input.
//
// Layout: block = 16 output rows x 64 output columns of one image; thread = 4 consecutive
// columns of one row. For each PSF row a (outer loop, reference order) the block stages the
// 16 x (64 + cols - 1) input window X~[i0+l-1-a .. +16)[j0+q-cols .. +64+cols-1) and the PSF row
// in shared memory (extension applied while staging; rows wider than kBlCW go in column chunks,
// in order), then every thread walks the PSF row b = 0..cols-1 with a 4-value sliding register
// window (one shared load per 4 products).
// Work is nnz(P)·m·n multiply-adds (FP64 pipe, the same O(nnz·m·n) as the reference, but on
// 148 SMs): setup / data generation only, never inside the timed solve.
#pragma once

namespace kb {

constexpr int kBlTH = 16, kBlTW = 64, kBlThreads = 256;

__device__ __forceinline__ int kb_blur_ext(int t, int M, bool reflect) {
  if (t >= 0 && t < M) return t;
  if (!reflect) return -1;
  t = t < 0 ? -1 - t : 2 * M - 1 - t;  // numpy "symmetric": edge sample repeated
  return (t >= 0 && t < M) ? t : -1;   // only rows / columns of discarded outputs get here
}

// PSF columns are taken in chunks of at most kBlCW (in order), so any PSF width fits the
// staged window; the host crops all-zero PSF borders first (they add nothing).
constexpr int kBlCW = 512;
__host__ __device__ inline size_t kb_blur_smem(int cols) {
  const int cw = cols < kBlCW ? cols : kBlCW;
  return sizeof(double) * ((size_t)kBlTH * (kBlTW + cw - 1) + cw);
}

__global__ void __launch_bounds__(kBlThreads)
kb_blur_direct_k(const double* __restrict__ psf, long long psf_bs, int rows, int cols, int l, int q,
                 const double* __restrict__ X, double* __restrict__ Y, int m, int n, int reflect) {
  extern __shared__ double kb_smem_bl[];
  const int cwmax = cols < kBlCW ? cols : kBlCW;
  double* slab = kb_smem_bl;                     // [kBlTH][kBlTW + cw - 1]
  double* prow = slab + kBlTH * (kBlTW + cwmax - 1);  // [cw]
  const int b = blockIdx.z, i0 = blockIdx.y * kBlTH, j0 = blockIdx.x * kBlTW;
  const double* P = psf + b * psf_bs;
  const double* Xb = X + (long long)b * m * n;
  const int tr = threadIdx.x >> 4, tc = (threadIdx.x & 15) * 4;
  double y0 = 0.0, y1 = 0.0, y2 = 0.0, y3 = 0.0;
  for (int a = 0; a < rows; ++a) {
    const int rbase = i0 + l - 1 - a;  // input row of window row 0
    for (int c0 = 0; c0 < cols; c0 += kBlCW) {
      const int cw = min(kBlCW, cols - c0), W = kBlTW + cw - 1;
      const int cbase = j0 + q - c0 - cw;  // input column of window column 0
      int nz = 0;
      for (int t = threadIdx.x; t < cw; t += kBlThreads) {
        const double p = P[(long long)a * cols + c0 + t];
        prow[t] = p;
        nz |= p != 0.0;
      }
      if (!__syncthreads_or(nz)) continue;  // all-zero PSF entries add nothing (np.nonzero)
      for (int idx = threadIdx.x; idx < kBlTH * W; idx += kBlThreads) {
        const int rr = idx / W, cc = idx - rr * W;
        const int gi = kb_blur_ext(rbase + rr, m, reflect), gj = kb_blur_ext(cbase + cc, n, reflect);
        slab[idx] = (gi >= 0 && gj >= 0) ? Xb[(long long)gi * n + gj] : 0.0;
      }
      __syncthreads();
      // output column j0 + tc + k with PSF column c0 + c reads window column tc + k + cw - 1 - c
      const double* s = slab + tr * W + tc;
      double w0 = s[cw - 1], w1 = s[cw], w2 = s[cw + 1], w3 = s[cw + 2];
      for (int c = 0; c < cw; ++c) {
        const double p = prow[c];
        if (p != 0.0) {  // block-uniform
          y0 = __dadd_rn(y0, __dmul_rn(p, w0));
          y1 = __dadd_rn(y1, __dmul_rn(p, w1));
          y2 = __dadd_rn(y2, __dmul_rn(p, w2));
          y3 = __dadd_rn(y3, __dmul_rn(p, w3));
        }
        w3 = w2;
        w2 = w1;
        w1 = w0;
        if (c + 1 < cw) w0 = s[cw - 2 - c];
      }
      __syncthreads();
    }
  }
  const int i = i0 + tr;
  if (i >= m) return;
  double* yr = Y + ((long long)b * m + i) * n + j0 + tc;
  const double v[4] = {y0, y1, y2, y3};
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (j0 + tc + k < n) yr[k] = v[k];
}

}  // namespace kb
