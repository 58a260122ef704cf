/*
 * kronblur_b200.h — C ABI of the B200 (sm_100a) sFISTA hot path.
 *
 * The reference package (kronblur, pure Python) has no native interface of its own; this header is
 * what its solver layer would bind through ctypes. Each entry point names the
 * reference function it replaces. All array pointers are DEVICE pointers to contiguous row-major
 * (batch, m, n) planes of the operator's dtype (float64 or float32); `stream` is a cudaStream_t
 * (pass torch.cuda.current_stream().cuda_stream). Every call is stream ordered and returns a
 * KB_* status; kb_last_error() gives the message of the last failing call on this thread.
 *
 * Band convention: along an axis the factor F(c) (kronblur structured.py:111-123) acts as the
 * stencil y[s] = sum_d c_d * x~(s - d) with c_d = c[j + d] (c the length-n generator, j its
 * 1-based anchor). A band is given as its first offset `dlo` and its `w` taps c_dlo..c_{dlo+w-1}
 * for every term (zero outside). bc = KB_BC_ZERO means Toeplitz factors (zero extension),
 * KB_BC_REFLECTIVE means Toeplitz+Hankel factors (single half-sample fold at each edge).
 */
#ifndef KRONBLUR_B200_H
#define KRONBLUR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KB_OK 0
#define KB_ERR_ARGUMENT 2 /* kronblur.errors.ArgumentError (CLI exit code 2, cli.py:34) */
#define KB_ERR_CUDA 3     /* CUDA runtime failure */
#define KB_ERR_NUMERIC 4  /* kronblur.errors.NumericError */

#define KB_F64 0
#define KB_F32 1
#define KB_PEAK_TC_TF32 2 /* kb_fma_peak only: the tcgen05 kind::tf32 rate */

/* pass engines reported by kb_last_engines */
#define KB_ENGINE_GENERIC 0  /* generic tiled kernels (odd shapes, misaligned buffers) */
#define KB_ENGINE_FFMA 1     /* persistent FFMA register-window kernels (fp32) */
#define KB_ENGINE_DMMA 2     /* persistent FP64 tensor-core DMMA kernels */
#define KB_ENGINE_MMA_TF32 3 /* persistent 3xTF32 mma.sync kernels */
#define KB_ENGINE_TC_TF32 4  /* tcgen05 3xTF32 kernels (tensor-memory accumulators) */
#define KB_ENGINE_PERSIST_F64 5 /* whole-solve persistent fp64 kernel (small images, one launch) */
#define KB_ENGINE_TC_FUSED 6 /* one-sweep tcgen05 3xTF32 kernel: both passes of an application in one launch */

#define KB_BC_ZERO 0
#define KB_BC_REFLECTIVE 1

typedef struct kb_op kb_op; /* immutable device copy of a KronOperator's factor bands */

/* Library version string and the sm target it was built for. */
const char* kb_version(void);
/* Message of the last failing call on the calling thread ("" if none). */
const char* kb_last_error(void);

/*
 * Upload a KronOperator (kron.py:61-86) — or `batch` operators of equal shape and term count —
 * as device tap tables. a_* describe the H_i (axis 0) bands, b_* the K_i (axis 1) bands; the
 * value arrays are [batch][r][w] float64. bc_a / bc_b select Toeplitz or Toeplitz+Hankel per
 * axis (decompose() uses the same kind on both, kron.py:185-195). Replaces the per-factor
 * FFT plans built by structured.py:97-108.
 */
int kb_op_create(kb_op** out, int dtype, int m, int n, int r, int batch, int bc_a, int bc_b,
                 int a_dlo, int a_w, const double* a_taps, int b_dlo, int b_w,
                 const double* b_taps);
int kb_op_destroy(kb_op* op);
/*
 * Layout facts of an operator, info[0..n): {Ha, Wpa, Hb, Wpb, sym_a, sym_b, adjoint pass-A groups,
 * max group, twin}. twin = 1: kb_sfista_run's fast path solves the transposed problem with an
 * axis-swapped copy of the operator (the wider band in pass A; large fp32 images, KB_AXIS_SWAP). sym_* = 1 when every generator on that reflective axis is symmetric or
 * antisymmetric to 1e-11 relative, so the adjoint folds through sign-reflected tile fills
 * instead of the exact fold kernels (set KB_EXACT_FOLD=1 to force the exact path).
 */
int kb_op_info(const kb_op* op, int* info, int n);
/* Device workspace (bytes) the calls below need for this operator. */
size_t kb_workspace_bytes(const kb_op* op);

/* Y = sum_i H_i X K_i^T  — kron.py:218-225 (kron_apply). */
int kb_apply(const kb_op* op, const void* X, void* Y, void* work, void* stream);
/* X = sum_i H_i^T Y K_i  — kron.py:228-235 (kron_apply_adjoint). */
int kb_apply_adjoint(const kb_op* op, const void* Y, void* X, void* work, void* stream);

/*
 * `iters` sFISTA iterations k = k0+1 .. k0+iters of solvers.py:168-174 (the _engine loop body,
 * no history): R = A Y - B; G = A^T R; x = (L y - G)/(L + lam^2) [then x = max(x, 0) keeping NaN
 * when project != 0]; y = x + beta[k-1] (x - x_prev). X holds x_{k0} on entry and x_{k0+iters}
 * on exit, Y holds y_{k0+1} on entry and y_{k0+iters+1} on exit (both in place).
 * beta: host array, beta[k-1] = (t_k - 1)/t_{k+1} from momentum_next (solvers.py:96-101).
 * L: host array [batch] (SolveConfig.lipschitz per image). nonfinite: device int, atomically
 * min-ed with the first k whose x had a non-finite entry (solvers.py:175-176); initialise it
 * to INT_MAX. norms: optional device double[iters][4][batch] receiving per iteration
 * ||x_k - x_{k-1}||^2, ||x_{k-1}||^2, ||x_k||^2 (solvers.py:178-179), or NULL.
 * use_graph != 0 captures the launch sequence in a CUDA graph (same arithmetic).
 */
int kb_sfista_run(const kb_op* op, const void* B, void* X, void* Y, void* work,
                  const double* beta, int k0, int iters, const double* L, double lam,
                  int project, int* nonfinite, double* norms, int use_graph, void* stream);
/* kb_sfista_run with a per-image lam (host array [batch]): the batched lambda probes of
 * select_lambda (solvers.py:294-305), one image per candidate lambda. */
int kb_sfista_run_lams(const kb_op* op, const void* B, void* X, void* Y, void* work,
                       const double* beta, int k0, int iters, const double* L, const double* lam,
                       int project, int* nonfinite, double* norms, int use_graph, void* stream);

/*
 * Power iteration of solvers.py:104-130 on A^T A: v (device, normalised start vector drawn on
 * the host from rand.stream(seed, "lipschitz")) is overwritten; w is a scratch plane of the same
 * size. hist (device double[iters][2][batch]) receives rho_k = <v_k, w_k> and ||w_k||^2 per
 * iteration; the host applies the zero-operator rule and the 1.05 safety factor.
 */
int kb_power_iter(const kb_op* op, void* v, void* w, void* work, int iters, double* hist,
                  void* stream);

/*
 * Row-block sharded operator application (multi-GPU halo exchange): like kb_apply /
 * kb_apply_adjoint on the local rows [g0, g0+m_local) of a global m_global x n image whose
 * plane pointer X addresses local row 0 and whose rows -halo_lo .. m_local+halo_hi-1 are
 * readable (filled by the neighbours). The operator must have been created with m = m_local.
 */
int kb_apply_block(const kb_op* op, int adjoint, const void* X, void* Y, void* work, int g0,
                   int m_global, int halo_lo, int halo_hi, void* stream);
/* sFISTA epilogue pieces for the sharded solver: R = A Y - B and the fused adjoint+update,
 * each on a local row block (same halo contract as kb_apply_block). */
int kb_block_residual(const kb_op* op, const void* Yh, const void* B, void* R, void* work,
                      int g0, int m_global, int halo_lo, int halo_hi, void* stream);
/* norms: optional device double[4] receiving this block's ||x_k - x_{k-1}||^2, ||x_{k-1}||^2,
 * ||x_k||^2 (solvers.py:178-179); the sharded solver all-reduces them across ranks (sum) for
 * history and rel_tol. NULL: no norms (the fast kernels). */
int kb_block_update(const kb_op* op, const void* Rh, void* X, void* Y, void* work, int g0,
                    int m_global, int halo_lo, int halo_hi, double beta, int k, double L,
                    double lam, int project, int* nonfinite, double* norms, void* stream);
/* out2 (device double[2]) = { <a, b>, ||b||^2 } over `count` elements of dtype, fp64
 * accumulation, deterministic; work: KB_RESID_NORMS_WORK bytes. The sharded power iteration's
 * local reductions (solvers.py:124-125), all-reduced across ranks by the caller. */
int kb_inner2(int dtype, const void* a, const void* b, long long count, double* out2, void* work,
              void* stream);

/*
 * Exact blur of `batch` float64 images — psf.py:170-193 (blur_direct), the `exact_apply` of
 * solvers.py:182 / pipeline.py:180,294 and the data generator of pipeline.py:88. Y gets, per
 * pixel, the reference's own sequence: the products P[a][b] * X~[i+l-1-a][j+q-1-b] over the
 * NONZERO PSF entries in row-major order, each product and each sum rounded separately, X~ the
 * zero (bc = KB_BC_ZERO) or numpy-"symmetric" (KB_BC_REFLECTIVE) extension of X. The result is
 * bit-identical to the reference. psf: device [batch or 1][rows][cols] float64 with 1-based
 * centre (l, q); psf_batch_stride = 0 shares one PSF, rows*cols gives one PSF per image.
 * Errors (KB_ERR_ARGUMENT) as the reference: PSF larger than the image; X and Y must not
 * overlap. All-zero PSF borders may be cropped by the caller (they add nothing), so the centre
 * may lie outside the passed block.
 */
int kb_blur_direct(const double* psf, long long psf_batch_stride, int rows, int cols, int l, int q,
                   const double* X, double* Y, int m, int n, int batch, int bc, void* stream);

/*
 * History reductions of one sFISTA iteration with record_history (solvers.py:133-141, :181):
 * out2 (device double[2]) = { ||AX - B||^2, ||X - truth||^2 } over `count` elements of dtype
 * (truth may be NULL: out2[1] = 0). With ||x_k||^2 from kb_sfista_run's norms this gives the
 * objective 1/2 ||A x - b||^2 + lam^2/2 ||x||^2 and eta. work: device scratch of at least
 * KB_RESID_NORMS_WORK bytes. Deterministic (fixed reduction order), fp64 accumulation.
 */
#define KB_RESID_NORMS_WORK (2 * 8 * 296)
int kb_resid_norms(int dtype, const void* AX, const void* B, const void* X, const void* truth,
                   long long count, double* out2, void* work, void* stream);

/*
 * Measurement helpers used by bench.py (no reference counterpart).
 * kb_fma_peak: measured throughput (TFLOP/s) of the arithmetic instruction the pass kernels issue
 * for dtype - FP64 tensor-core DMMA (m8n8k4) for KB_F64, TF32 tensor-core mma.sync (m16n8k8)
 * for KB_F32, tcgen05.mma kind::tf32 (M128 N256 K8, operands in shared memory) for
 * KB_PEAK_TC_TF32; the fp32 3xTF32 passes issue three per product (roofline denominator).
 * kb_time_passes: average device time (ms, CUDA events on `stream`) of each of the four kernels of
 * one sFISTA iteration, `reps` back-to-back launches each: ms4 = {forward pass A, forward pass B
 * (residual epilogue), adjoint pass A, adjoint pass B (update epilogue, beta = 0)}. X/Yio are
 * overwritten.
 */
int kb_fma_peak(int dtype, float* tflops, void* stream);
/* Arithmetic engine (KB_ENGINE_*) of each phase {forward pass A, forward pass B, adjoint pass
 * A, adjoint pass B} of the latest kb_sfista_run / kb_sfista_run_lams / kb_time_passes on `op`,
 * so tests can assert which kernels ran and the roofline of a phase divides by the peak of the
 * instruction it actually issued. */
int kb_last_engines(const kb_op* op, int* engines4);
/* Profiling timeline of the latest fp64 pass kernels launched with KB_DEBUG_MODE bit 7 set:
 * host[kind][block][slot] %globaltimer stamps (kind 0 split, 1 sum; 1024 blocks x 8 slots,
 * slot 7 = SM id); copies min(n, 16384) values. */
int kb_debug_trace(unsigned long long* host, int n);
int kb_time_passes(const kb_op* op, const void* Y, const void* B, void* R, void* X, void* Yio,
                   void* work, int reps, const double* L, double lam, int* nonfinite,
                   float* ms4, void* stream);

/* Maximum half band width supported per axis. */
int kb_max_half_width(void);

#ifdef __cplusplus
}
#endif
#endif /* KRONBLUR_B200_H */
