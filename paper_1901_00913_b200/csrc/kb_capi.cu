// kb_capi.cu — C ABI (include/kronblur_b200.h) over the sm_100a pass kernels.
//
// Owns the device tap tables of an operator, the workspace layout, and the native iteration
// loop of the sFISTA engine (kronblur solvers.py:168-174) including optional CUDA-graph
// capture of the whole launch sequence. No torch types cross this boundary.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/kronblur_b200.h"
#include "kb_kernels.cuh"
#include "kb_dmma.cuh"
#include "kb_ffma.cuh"
#include "kb_tf32.cuh"
#include "kb_tc.cuh"
#include "kb_fused.cuh"
#include "kb_tc1.cuh"
#include "kb_blur.cuh"
#include "kb_norms.cuh"
#include "kb_persist.cuh"
#include "kb_persist2.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define KB_CUDA(call)                                                                   \
  do {                                                                                  \
    cudaError_t _e = (call);                                                            \
    if (_e != cudaSuccess)                                                              \
      return fail(KB_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e));     \
  } while (0)

#define KB_TRY(...)           \
  do {                        \
    int _rc = (__VA_ARGS__);  \
    if (_rc != KB_OK) return _rc; \
  } while (0)

constexpr int kMaxHalf = 1024;
// wide-band (Kw > 64) sum passes on kb_tc1.cuh's two-accumulator variant (SLOTS = 2, opt-in with
// KB_TC_SUM1=2): cfg4 8.96k -> 9.79k Mpix*it/s, but one application drifts to 1.9e-5 of the fp64
// result (per-term slots: < 1e-5) and the full-length solve to 4.9e-5 of the fixture (slots:
// 3.4e-5; tolerance 1e-4), so by default they stay on the per-term slot kernel
constexpr bool kT1WideSlots = false;
constexpr int kGmaxF64 = 2;  // pass A term group (register budget: G*R accumulators)
constexpr int kGmaxF32 = 4;
constexpr double kSymTol = 1e-11;  // (anti)symmetry residual allowed for sign-reflected fills
constexpr int kRA = 8;   // pass A rows per warp
constexpr int kRB = 16;  // pass B columns per warp

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct GraphCache {
  std::mutex mu;
  cudaGraphExec_t exec = nullptr;
  std::vector<unsigned char> key;
  int engines[4] = {-1, -1, -1, -1};  // phase engines of the captured launches
};

}  // namespace

struct kb_op {
  int dtype, m, n, r, batch, bc_a, bc_b;
  int Ha, Wpa, Hb, Wpb;
  int gmax;                  // largest term group of pass A
  int sym_a = 0, sym_b = 0;  // adjoint uses sign-reflected tile fills (no fold kernels)
  kb::Groups grp_fwd, grp_adj;
  void* sign_b = nullptr;    // [batch][r] +-1 fill sign of each term on axis 1 (sym_b only)
  void* ta_conv = nullptr;  // [batch][r][Wpa] taps c_{H-k}
  void* ta_corr = nullptr;  // [batch][r][Wpa] taps c_{k-H}
  void* tb_conv = nullptr;
  void* tb_corr = nullptr;
  // fp32: brick tables of the four tap tables (kb::kb_build_bricks) for the tcgen05 passes,
  // [batch][r][nbr][256]; null where the axis' band is too narrow for them
  unsigned* br_a_conv = nullptr;
  unsigned* br_a_corr = nullptr;
  unsigned* br_b_conv = nullptr;
  unsigned* br_b_corr = nullptr;
  // pass-B bricks of the fused kernel (kb_fused.cuh): half width Hbf = Hb rounded up to a
  // multiple of 4, so its X tiles start on a 16-byte column (TMA); alias br_b_* when Hb % 4 == 0
  int Hbf = 0;
  unsigned* br_bf_conv = nullptr;
  unsigned* br_bf_corr = nullptr;
  GraphCache* graph = nullptr;
  // > 1 for the strip / image-group views of an L2-blocked solve (sfista_blocked): engine
  // selection then counts the chunks of the whole problem, not of one strip
  long long chunk_scale = 1;
  int slots_cap = 0;  // views: norm-partial slots of the parent's workspace (0: sum_blocks(op))
  // the operator of the transposed image (H and K swapped, m and n swapped) when running the
  // wider band first is faster (kb_op_create: axis_swap_wanted); the fast sFISTA path then
  // solves the transposed problem Y^T = sum_i K_i X^T H_i^T in the same workspace
  kb_op* twin = nullptr;
  // fp64: host copies of the four tap tables ([batch][r][Wp], axis a then b) for the launch
  // parameters of the zero-BC whole-solve kernel (kb_persist2.cuh)
  std::vector<double> h_conv[2], h_corr[2];
  // engines of the latest kb_time_passes phases (reporting only; written under g_phase_mu)
  mutable int phase_engine[4] = {0, 0, 0, 0};
};

namespace {

size_t elem(const kb_op* op) { return op->dtype == KB_F64 ? 8 : 4; }
size_t plane_elems(const kb_op* op) { return (size_t)op->m * op->n; }
// Z_i^T planes are [n + 2 Hb][m]: Hb halo rows on each side hold the reflected rows the
// persistent split kernels store for a reflect-filled sum pass (kb_dmma.cuh, kb_ffma.cuh).
long long z_plane(const kb_op* op) { return (long long)(op->n + 2 * op->Hb) * op->m; }
template <typename T>
T* z_row0(const kb_op* op, void* z) { return static_cast<T*>(z) + (long long)op->Hb * op->m; }

// Per-call launch state: what the latest pass launch of THIS call did. It lives in the call's
// Work (never in the shared kb_op), so concurrent calls on one operator from several host
// threads (each with its own workspace) do not see each other's launches.
struct Ctx {
  int mirror = 0;  // the latest split pass stored Z^T's reflected halo rows
  int slots = 0;   // norm partial slots per image written by the latest sum pass
  int engine = 0;  // KB_ENGINE_* of the latest pass launch
  int phase[4] = {-1, -1, -1, -1};  // engines of the call's four phases (split/sum fwd, adj)
};

// workspace: [Z: batch*r planes][R: batch planes][partials][scalars]
struct Work {
  mutable Ctx ctx;
  void* z;
  void* rp;
  void* fold;  // [batch][m][2*Hb] adjoint column-fold corrections
  double* partials;
  double* scal;  // [4][batch]: L, denom
  size_t bytes;
};

// Resident blocks for the persistent fp64 kernels: two per SM.
int persistent_blocks() {
  static const int nb = [] {  // thread-safe one-time init (C++11 magic static)
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return 2 * sms;
  }();
  return nb;
}

// TMA descriptor of a 3-D [planes][rows][cols] array (cols contiguous) with a {box_cols x
// box_rows} box: fp64 tiles are 36 columns wide (padded rows for the DMMA fragments), fp32 tiles
// 32 (128-byte rows). False when TMA's alignment rules rule it out.
bool make_tmap(CUtensorMap* map, const void* base, long long cols, long long rows, long long planes,
               long long row_stride, long long plane_stride, int box_rows, int esize = 8,
               int box_cols = 0, CUtensorMapSwizzle swizzle = CU_TENSOR_MAP_SWIZZLE_NONE) {
  static const PFN_cuTensorMapEncodeTiled_v12000 encode = [] {  // thread-safe one-time lookup
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    return (PFN_cuTensorMapEncodeTiled_v12000) nullptr;
  }();
  if (!encode) return false;
  if (reinterpret_cast<uintptr_t>(base) % 16 || (row_stride * esize) % 16 || (plane_stride * esize) % 16)
    return false;
  if (box_rows < 1 || box_rows > 256) return false;
  const cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, (cuuint64_t)planes};
  const cuuint64_t strides[2] = {(cuuint64_t)row_stride * esize, (cuuint64_t)plane_stride * esize};
  const cuuint32_t box[3] = {box_cols > 0 ? (cuuint32_t)box_cols : (esize == 8 ? 36u : 32u),
                             (cuuint32_t)box_rows, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  return encode(map, esize == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                const_cast<void*>(base), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle,
                CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// fp64 runs on the TMA + DMMA kernels when both image extents are even (16-byte row strides)
bool use_dmma(const kb_op* op) { return op->dtype == KB_F64 && op->m % 2 == 0 && op->n % 2 == 0; }
// fp32 runs on the persistent TMA + FFMA kernels when both extents are multiples of 4 (16-byte
// row strides and vector stores); other shapes take the generic tiled kernels.
bool use_tma_f32(const kb_op* op) { return op->dtype == KB_F32 && op->m % 4 == 0 && op->n % 4 == 0; }
// fp32 zero-BC passes on tcgen05 (kb_tc.cuh). KB_FP32_TC=1 / 0 forces them on / off; by default
// they take the wide bands where they measured faster than the mma.sync kernels on the box
// (tools/time_kernels.py): split from Kw >= 64, sum from Kw >= 128, and only with
// enough 64 x 128 chunks to occupy the SMs (a 256^2 image has 8).
// (KB_FP32_TC=split / sum force one pass only.)
int tc_policy(int pass) {  // pass: 1 split, 2 sum
  static const int p = [] {
    const char* v = std::getenv("KB_FP32_TC");
    if (!v) return -1;
    const std::string s(v);
    return s == "1" ? 3 : s == "split" ? 1 : s == "sum" ? 2 : 0;
  }();
  return p < 0 ? -1 : (p & pass) ? 1 : 0;
}
int sm_count();
bool use_tc(const kb_op* op, const kb::AxisGeom& g, int min_kw) {
  const int pol = tc_policy(min_kw == 64 ? 1 : 2);
  if (!use_tma_f32(op) || pol == 0) return false;
  if (pol == 1) return true;
  const long long chunks =
      (long long)((g.len + kb::kTcTS - 1) / kb::kTcTS) * ((g.other + 127) / 128) * op->batch * op->chunk_scale;
  // wide bands with enough chunks to occupy the SMs, or any band from 32 taps once there are
  // >= 8 chunks per SM (cfg3's 512-image batch, cfg5's 16384^2: 2x the mma.sync passes there);
  // the sum pass from 32 taps with >= 128 chunks (cfg2 fp32: 12.8 / 17.4 us against 19.5 / 24.6
  // on mma.sync, while its split stays faster on mma.sync)
  if (min_kw == 128 && g.Kw >= 32 && chunks >= 128) return true;
  return (g.Kw >= min_kw && chunks >= 128) || (g.Kw >= 32 && chunks >= 8LL * sm_count());
}
// the brick table built from tap table `tin`, or null
const unsigned* brick_table(const kb_op* op, const void* tin) {
  if (tin == op->ta_conv) return op->br_a_conv;
  if (tin == op->ta_corr) return op->br_a_corr;
  if (tin == op->tb_conv) return op->br_b_conv;
  if (tin == op->tb_corr) return op->br_b_corr;
  return nullptr;
}

bool use_tc_split(const kb_op* op, const kb::AxisGeom& g) { return use_tc(op, g, 64); }
// fp32 arithmetic of the persistent kernels: 3xTF32 tensor-core MMA (kb_tf32.cuh, default) or
// FFMA register windows (kb_ffma.cuh; KB_FP32_PATH=ffma)
bool use_tf32(const kb_op* op) {
  static const bool ffma = [] {
    const char* v = std::getenv("KB_FP32_PATH");
    return v && std::string(v) == "ffma";
  }();
  return use_tma_f32(op) && !ffma;
}
bool al16(const void* p) { return reinterpret_cast<uintptr_t>(p) % 16 == 0; }
// the persistent sum kernels move epilogue operands as 16-byte vectors
template <typename T>
bool epi_aligned(const kb::Epi<T>& e) {
  return al16(e.out) && al16(e.bsub) && al16(e.x) && al16(e.y) && al16(e.vin);
}

// Norm partial slots of the sum pass per image: one per warp of the persistent kernels, one
// per block of the generic tiled kernel (used for shapes / pointers the persistent kernels
// do not take). The workspace holds the larger count; each launch records its own.
int persistent_slots(const kb_op* op) {
  int parts, nb;
  kb::plan_items(op->n, (op->m + 31) / 32, op->batch, persistent_blocks(), parts, nb);
  return nb * kb::kNW;
}
int generic_slots(const kb_op* op) {
  const int TS = kb::kNW * kRB;
  return ((op->n + TS - 1) / TS) * ((op->m + 31) / 32);
}
int sum_blocks(const kb_op* op) { return std::max(persistent_slots(op), generic_slots(op)); }
// doubles in the partials region: the norm slots, and at least room for a whole-solve launch's
// beta table plus one 128-byte phase flag per CTA (kb_persist2.cuh)
size_t partials_doubles(const kb_op* op) {
  return std::max<size_t>(4 * (size_t)op->batch * sum_blocks(op), 16384);
}

Work layout(const kb_op* op, void* base) {
  Work w;
  size_t off = 0;
  const size_t pe = plane_elems(op) * elem(op);
  unsigned char* b = static_cast<unsigned char*>(base);
  w.z = b ? b + off : nullptr;
  off = align_up(off + (size_t)z_plane(op) * elem(op) * op->r * op->batch, 256);
  w.rp = b ? b + off : nullptr;
  off = align_up(off + pe * op->batch, 256);
  w.fold = b ? b + off : nullptr;
  off = align_up(off + elem(op) * (size_t)op->batch * op->m * 2 * std::max(op->Hb, 1), 256);
  w.partials = b ? reinterpret_cast<double*>(b + off) : nullptr;
  off = align_up(off + sizeof(double) * partials_doubles(op), 256);
  w.scal = b ? reinterpret_cast<double*>(b + off) : nullptr;
  off = align_up(off + sizeof(double) * 4 * (size_t)op->batch, 256);
  w.bytes = off;
  return w;
}

// With an axis-swapped twin the workspace holds the larger of the two layouts, then the
// transposed B, X and Y planes of the twin's solve.
size_t twin_planes_offset(const kb_op* op) {
  return align_up(std::max(layout(op, nullptr).bytes, layout(op->twin, nullptr).bytes), 256);
}
void* twin_plane(const kb_op* op, void* base, int i) {
  return static_cast<unsigned char*>(base) + twin_planes_offset(op) + i * align_up(plane_elems(op) * elem(op), 256);
}

// out[n][m] = in[m][n] (32 x 32 shared-memory tiles, both sides coalesced)
template <typename T>
__global__ void kb_transpose_k(const T* __restrict__ in, T* __restrict__ out, int m, int n) {
  __shared__ T tile[32][33];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += 8) {
    const int r = r0 + j, c = c0 + threadIdx.x;
    if (r < m && c < n) tile[j][threadIdx.x] = in[(size_t)r * n + c];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += 8) {
    const int c = c0 + j, r = r0 + threadIdx.x;
    if (c < n && r < m) out[(size_t)c * m + r] = tile[threadIdx.x][j];
  }
}
template <typename T>
int transpose_t(const T* in, T* out, int m, int n, cudaStream_t s) {
  dim3 grid((n + 31) / 32, (m + 31) / 32);
  kb_transpose_k<T><<<grid, dim3(32, 8), 0, s>>>(in, out, m, n);
  KB_CUDA(cudaGetLastError());
  return KB_OK;
}

// Split `count` terms starting at `start` into near-equal groups of at most gmax, all with
// the given tile-fill sign.
void add_groups(kb::Groups& g, int start, int count, int gmax, int sign) {
  if (count <= 0) return;
  const int ng = (count + gmax - 1) / gmax;
  for (int k = 0; k < ng; ++k) {
    const int lo = start + (int)((long)count * k / ng), hi = start + (int)((long)count * (k + 1) / ng);
    g.start[g.n] = lo;
    g.count[g.n] = hi - lo;
    g.sign[g.n] = sign;
    ++g.n;
  }
}

// Opt a kernel into the full 227 KB of shared memory (minus its static shared memory). Keyed by
// the kernel's address: instantiations that differ only in a template value share a type.
std::mutex g_smem_mu;
std::mutex g_phase_mu;
std::unordered_map<const void*, int> g_smem_limit;

template <typename K>
int allow_smem(K kernel, size_t dyn_bytes) {
  const void* key = reinterpret_cast<const void*>(kernel);
  int limit;
  {
    std::lock_guard<std::mutex> lock(g_smem_mu);
    auto it = g_smem_limit.find(key);
    if (it == g_smem_limit.end()) {
      cudaFuncAttributes attr;
      KB_CUDA(cudaFuncGetAttributes(&attr, kernel));
      limit = 227 * 1024 - (int)attr.sharedSizeBytes;
      KB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, limit));
      // one carveout (all shared memory) for every pass kernel: consecutive kernels of an
      // iteration then never wait for an SM's L1/shared split to be reconfigured
      KB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                   (int)cudaSharedmemCarveoutMaxShared));
      g_smem_limit[key] = limit;
    } else {
      limit = it->second;
    }
  }
  if (dyn_bytes > (size_t)limit) return fail(KB_ERR_ARGUMENT, "band too wide for the shared-memory tile");
  return KB_OK;
}

// Tile ring depth for a persistent kernel: as many stages (2..kMaxStages) as fit next to the
// taps at `bps` resident blocks per SM. KB_RING_STAGES caps it (profiling).
int ring_stages(size_t stage_bytes, size_t fixed_bytes, int bps) {
  static const int cap = [] {
    const char* v = std::getenv("KB_RING_STAGES");
    return v ? std::max(2, std::min(kb::kMaxStages, std::atoi(v))) : kb::kMaxStages;
  }();
  const size_t budget = (bps >= 2 ? 114 : 228) * 1024 - 1024 - 128;
  int n = 2;
  while (n < cap && fixed_bytes + (n + 1) * stage_bytes <= budget) ++n;
  return n;
}

int split_ns() {
  static const int ns = [] {
    const char* v = std::getenv("KB_SPLIT_NS");
    return (v && v[0] == '1') ? 1 : 2;
  }();
  return ns;
}

// Launch a persistent pass kernel (one block of 32 x kNW threads per work slot) with
// programmatic stream serialization: in a stream or captured graph it may start while the
// previous kernel drains; it loads its taps, then waits in griddepcontrol.wait for that
// kernel's results (kb_dmma.cuh: pdl_wait). KB_PDL=0 turns it off.
bool use_pdl() {
  static const bool on = [] {
    const char* v = std::getenv("KB_PDL");
    return !(v && v[0] == '0');
  }();
  return on;
}
template <typename... KArgs, typename... Args>
cudaError_t launch_persistent(void (*kernel)(KArgs...), int nb, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nb);
  cfg.blockDim = dim3(32, kb::kNW);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = use_pdl() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

template <typename T, int GMAX>
int launch_a_g(const T* in, long long in_bs, T* z, long long z_ps, long long z_bs,
               const T* tin, long long t_bs, const kb::AxisGeom& g, const kb::Groups& grp,
               const double* nw2, int batch, cudaStream_t s) {
  constexpr int TS = kb::kNW * kRA;
  const size_t smem = sizeof(T) * ((size_t)(TS + g.Wp) * 32 + (size_t)GMAX * g.Wp + 32 * (TS + 1));
  auto kern = kb::kb_pass_split<T, GMAX, kRA>;
  KB_TRY(allow_smem(kern, smem));
  dim3 grid((g.other + 31) / 32, (g.len + TS - 1) / TS, batch);
  dim3 block(32, kb::kNW);
  kern<<<grid, block, smem, s>>>(in, in_bs, z, z_ps, z_bs, tin, t_bs, g, grp, nw2);
  KB_CUDA(cudaGetLastError());
  return KB_OK;
}

// Resident blocks per SM of a persistent pass kernel with `smem` bytes of dynamic shared memory:
// 2 when two fit, 1 when only one does (wide bands), 0 when none does (the generic tiled
// kernels then take the pass).
int blocks_per_sm(size_t smem) {
  const size_t per = smem + 1024 + 128;  // per-block reservation and static shared memory
  if (2 * per <= 228 * 1024) return 2;
  if (per <= 228 * 1024) return 1;
  return 0;
}
int sm_count() { return persistent_blocks() / 2; }

// Pass A into the Z^T planes (z: row 0 of image 0, term 0). mirror_h > 0 asks the persistent
// kernels to also store the reflected halo rows (times msign[b][i]) for a reflect-filled pass B;
// c.mirror records whether they did.
template <typename T>
int launch_a(const kb_op* op, Ctx& c, const T* in, T* z, const T* tin, const kb::AxisGeom& g,
             const kb::Groups& grp, const double* nw2, int mirror_h, const T* msign, cudaStream_t s) {
  const long long in_bs = (long long)plane_elems(op);
  const long long z_ps = z_plane(op);
  c.mirror = 0;
  const long long z_bs = z_ps * op->r;
  const long long t_bs = (long long)op->r * g.Wp;
  const T* in_map = in - (long long)g.halo_lo * g.other;
  const long long in_rows = g.len + g.halo_lo + g.halo_hi;
  // common tail of the persistent launches: balanced items on `bps` blocks per SM
  auto plan = [&](int bps, int& parts, int& nb, int& eparts) {
    kb::plan_items(g.len, (g.other + 31) / 32, op->batch, sm_count() * bps, parts, nb,
                   mirror_h > 0 ? &eparts : nullptr);  // edge L-tiles also store the halo rows
    if (mirror_h == 0) eparts = parts;
  };
  if constexpr (sizeof(T) == 8) {
    // NS = 2: 16-row warps whose two S-tiles share the A fragments (KB_SPLIT_NS=1: 8-row warps)
    const int ns = split_ns();
    const kb::TileBoxes tb = kb::tile_boxes(kb::dmma_rows(kb::kNW * 8 * ns, g.Kw));
    const size_t smem = sizeof(double) * ((size_t)kb::kStages * tb.stage_elems +
                                          (size_t)op->r * (ns == 2 ? kb::dmma_cstride_sum(g.Kw)
                                                                   : kb::dmma_cstride_split(g.Kw)));
    const int bps = blocks_per_sm(smem);
    CUtensorMap map;
    if (use_dmma(op) && bps > 0 &&
        make_tmap(&map, in_map, g.other, in_rows, op->batch, g.other, in_bs, tb.box_rows)) {
      auto kern = ns == 2 ? kb::kb_pass_split_dmma<kGmaxF64, 2> : kb::kb_pass_split_dmma<kGmaxF64, 1>;
      KB_TRY(allow_smem(kern, smem));
      int parts, nb, eparts;
      plan(bps, parts, nb, eparts);
      c.engine = sizeof(T) == 8 ? KB_ENGINE_DMMA : KB_ENGINE_FFMA;
      KB_CUDA(launch_persistent(kern, nb, smem, s, map, z, z_ps, z_bs, tin, t_bs, g, grp, nw2, op->r, op->batch,
                                parts, eparts, mirror_h, msign));
      c.mirror = mirror_h > 0;
      return KB_OK;
    }
    c.engine = KB_ENGINE_GENERIC;
    return launch_a_g<T, kGmaxF64>(in, in_bs, z, z_ps, z_bs, tin, t_bs, g, grp, nw2, op->batch, s);
  } else {
    const unsigned* btab = brick_table(op, tin);
    if (btab && use_tc_split(op, g) && z_bs == (long long)op->r * z_ps) {
      const int nbr = kb::tc_bricks(g.Kw);
      // bricks of up to kTcG terms first, then as deep a tile ring as the rest of shared memory
      // holds (at least 4 stages: with 3 the pipeline hangs or faults -- found with
      // -DKB_TC_RING_MAX=3 at cfg4/cfg5 -- so narrower rings fall back to the mma.sync passes)
      const size_t avail = 226 * 1024 - 1024 - kb::tc_store_bytes(4);
      static const int gmax = [] {
        const char* v = std::getenv("KB_TC_G");
        return v ? std::max(1, std::min(kb::kTcG, std::atoi(v))) : kb::kTcG;
      }();
      int G = std::min(op->r, gmax);
      while (G > 1 && (size_t)G * nbr * 1024 + 4 * kb::kTcStageBytes > avail) --G;
      // sign-uniform term groups of <= G terms: the runs of equal fill sign of the pass' groups,
      // each cut into near-equal pieces
      kb::Groups tg{};
      for (int i = 0; i < grp.n;) {
        int j = i + 1, count = grp.count[i];
        while (j < grp.n && grp.sign[j] == grp.sign[i] && grp.start[j] == grp.start[i] + count) count += grp.count[j++];
        add_groups(tg, grp.start[i], count, G, grp.sign[i]);
        i = j;
      }
      G = 0;
      for (int i = 0; i < tg.n; ++i) G = std::max(G, tg.count[i]);
      // chunk-major order with every term's bricks resident (KB_TC_CHUNK_MAJOR=1, when they fit
      // beside a >= 6-stage ring): the groups of a chunk re-read its input tiles from L2 instead
      // of streaming the plane from DRAM once per group. Opt-in: measured no faster at cfg5
      // (16.8k either way) and slower at cfg3 (41.1k -> 38.4k; profiles/r02_ab_chunk_major.txt).
      static const int cm_env = [] {
        const char* v = std::getenv("KB_TC_CHUNK_MAJOR");
        return v ? std::atoi(v) : 0;
      }();
      const int chunk_major = tg.n > 1 && cm_env == 1 &&
                              (size_t)op->r * nbr * 1024 + 6 * kb::kTcStageBytes <= avail;
      const size_t fixed = (size_t)(chunk_major ? op->r : G) * nbr * 1024;
      // 8 epilogue warps when a >= 4-stage ring still fits beside their staging (cfg5: the split
      // is bound by its Z^T stores, 3.3 -> 3.1 ms); KB_TC_SPLIT_EPI=4/8 overrides
      static const int epi_env = [] {
        const char* v = std::getenv("KB_TC_SPLIT_EPI");
        return v ? std::atoi(v) : 0;
      }();
      auto ring = [&](int epi) {
        const size_t av = 226 * 1024 - 1024 - kb::tc_store_bytes(epi);
        return std::min<int>(kb::kTcRingMax, (int)((av - std::min(fixed, av)) / kb::kTcStageBytes));
      };
      const int epi = epi_env == 4 ? 4 : (epi_env == 8 || ring(8) >= 4) ? 8 : 4;
      const int nst = ring(epi);
      const size_t smem = std::max<size_t>(1024 + kb::tc_store_bytes(epi) + (size_t)nst * kb::kTcStageBytes + fixed,
                                           116 * 1024);  // one CTA per SM
      CUtensorMap mapt, mapz;
      if (nst >= 4 && tg.n <= kb::kMaxGroups &&
          make_tmap(&mapt, in_map, g.other, in_rows, op->batch, g.other, in_bs, kb::kTcRB, 4, 128) &&
          make_tmap(&mapz, z, g.len, g.other, (long long)op->batch * op->r, g.len, z_ps, 32, 4, 32,
                    CU_TENSOR_MAP_SWIZZLE_128B)) {
        auto kern = epi == 8 ? kb::kb_pass_split_tc<8> : kb::kb_pass_split_tc<4>;
        KB_TRY(allow_smem(kern, smem));
        int parts, nb;
        kb::plan_items(g.len, (g.other + 127) / 128, op->batch, sm_count(), parts, nb);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(nb);
        cfg.blockDim = dim3(kb::tc_split_threads(epi));
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = use_pdl() ? 1 : 0;
        c.engine = KB_ENGINE_TC_TF32;
        KB_CUDA(cudaLaunchKernelEx(&cfg, kern, mapt, mapz, z, z_ps, z_bs, btab, g, nw2, op->r, op->batch, parts,
                                   tg, G, nst, reinterpret_cast<const float*>(in), in_bs, mirror_h,
                                   reinterpret_cast<const float*>(msign), chunk_major));
        c.mirror = mirror_h > 0;
        return KB_OK;
      }
    }
    if (use_tf32(op)) {
      const kb::TileBoxesX tx = kb::tile_boxes_x(kb::tf32_rows(kb::kNW * 8, g.Kw));
      const size_t fixed = 2 * (size_t)op->r * kb::tf32_cstride(g.Kw) * sizeof(float);
      const int bps = blocks_per_sm(fixed + 2 * tx.stage_elems * sizeof(float));
      const int nst = ring_stages(tx.stage_elems * sizeof(float), fixed, bps);
      const size_t smem = fixed + sizeof(float) * (size_t)nst * tx.stage_elems;
      CUtensorMap mapx;
      if (bps > 0 && make_tmap(&mapx, in_map, g.other, in_rows, op->batch, g.other, in_bs, tx.box_rows, 4, kb::kXF)) {
        auto kern = kb::kb_pass_split_x<kGmaxF32>;
        KB_TRY(allow_smem(kern, smem));
        int parts, nb, eparts;
        plan(bps, parts, nb, eparts);
        c.engine = KB_ENGINE_MMA_TF32;
        KB_CUDA(launch_persistent(kern, nb, smem, s, mapx, z, z_ps, z_bs, tin, t_bs, g, grp, nw2, op->r,
                                  op->batch, parts, eparts, mirror_h, msign, nst));
        c.mirror = mirror_h > 0;
        return KB_OK;
      }
    }
    const kb::TileBoxesF tb = kb::tile_boxes_f(kb::kNW * 8 + g.Wp);
    const size_t smem = sizeof(float) * ((size_t)kb::kStages * tb.stage_elems + (size_t)op->r * g.Wp);
    const int bps = blocks_per_sm(smem);
    CUtensorMap map;
    if (use_tma_f32(op) && bps > 0 &&
        make_tmap(&map, in_map, g.other, in_rows, op->batch, g.other, in_bs, tb.box_rows, 4)) {
      auto kern = kb::kb_pass_split_f<kGmaxF32>;
      KB_TRY(allow_smem(kern, smem));
      int parts, nb, eparts;
      plan(bps, parts, nb, eparts);
      c.engine = sizeof(T) == 8 ? KB_ENGINE_DMMA : KB_ENGINE_FFMA;
      KB_CUDA(launch_persistent(kern, nb, smem, s, map, z, z_ps, z_bs, tin, t_bs, g, grp, nw2, op->r, op->batch,
                                parts, eparts, mirror_h, msign));
      c.mirror = mirror_h > 0;
      return KB_OK;
    }
    c.engine = KB_ENGINE_GENERIC;
    return launch_a_g<T, kGmaxF32>(in, in_bs, z, z_ps, z_bs, tin, t_bs, g, grp, nw2, op->batch, s);
  }
}

// Pass B over the Z^T planes (z: row 0 of image 0, term 0). The persistent kernels read a
// reflect-filled pass's out-of-domain rows from the halo rows the split pass stored (the TMA
// map then spans them: halo_lo = Hb); without them the generic kernel folds at read time.
template <typename T, int MODE>
int launch_b(const kb_op* op, Ctx& c, const T* z, const T* tin, const kb::AxisGeom& g_in, const T* tsign,
             const kb::Epi<T>& e, cudaStream_t s) {
  const long long z_ps = z_plane(op);
  const bool mirrored = g_in.fill && c.mirror;
  kb::AxisGeom g = g_in;
  if (mirrored) g.halo_lo = g.halo_hi = op->Hb;
  const T* zmap = z - (long long)g.halo_lo * g.other;
  const long long zrows = g.len + g.halo_lo + g.halo_hi;
  const bool persistent_ok = (!g_in.fill || mirrored) && epi_aligned(e);
  // common tail of the persistent launches
  auto launch = [&](auto kern, size_t smem, int bps, const CUtensorMap& map, auto... extra) -> int {
    KB_TRY(allow_smem(kern, smem));
    int parts, nb;
    kb::plan_items(g.len, (g.other + 31) / 32, op->batch, sm_count() * bps, parts, nb);
    if (op->batch > 1 && (MODE == kb::EPI_POWER || e.want_norms))  // warps skip untouched images
      KB_CUDA(cudaMemsetAsync(e.partials, 0, sizeof(double) * 4 * (size_t)op->batch * nb * kb::kNW, s));
    c.slots = nb * kb::kNW;
    KB_CUDA(launch_persistent(kern, nb, smem, s, map, op->r, tin, (long long)op->r * g.Wp, g, e, op->batch,
                              parts, extra...));
    return KB_OK;
  };
  if constexpr (sizeof(T) == 8) {
    const kb::TileBoxes tb = kb::tile_boxes(kb::dmma_rows(kb::kNW * 16, g.Kw));
    const size_t smem = sizeof(double) * ((size_t)kb::kStages * tb.stage_elems +
                                          (size_t)op->r * kb::dmma_cstride_sum(g.Kw));
    const int bps = blocks_per_sm(smem);
    CUtensorMap map;
    if (use_dmma(op) && persistent_ok && bps > 0 &&
        make_tmap(&map, zmap, g.other, zrows, (long long)op->batch * op->r, g.other, z_ps, tb.box_rows))
    {
      c.engine = KB_ENGINE_DMMA;
      if (MODE == kb::EPI_UPDATE && !e.want_norms) return launch(kb::kb_pass_sum_dmma<MODE, false>, smem, bps, map);
      return launch(kb::kb_pass_sum_dmma<MODE>, smem, bps, map);
    }
  } else {
    const unsigned* btab = brick_table(op, tin);
    // 128-output chunks with one accumulator across the r terms (kb_tc1.cuh) for bands up to
    // Kw = 64 (KB_TC_SUM1=0 / 1: off / on wherever the tcgen05 sum pass runs)
    static const int sum1_env = [] {
      const char* v = std::getenv("KB_TC_SUM1");
      return v ? std::atoi(v) : -1;
    }();
    const long long nch1 = (long long)((g.len + kb::kT1TS - 1) / kb::kT1TS) * ((g.other + 127) / 128) * op->batch;
    // (KB_TC_SUM1=2: the two-accumulator variant for wider bands, tested at cfg4)
    const int slots1 = sum1_env == 2 || (sum1_env < 0 && g.Kw > 64) ? 2 : 1;
    if (btab && use_tc(op, g, 128) && persistent_ok && sum1_env != 0 &&
        (sum1_env >= 1 || ((g.Kw <= 64 || kT1WideSlots) && nch1 * op->chunk_scale >= 2LL * sm_count()))) {
      const int nbr = kb::tc_bricks(g.Kw);
      // epilogue operands staged by TMA (kb_tc1.cuh TMAE; KB_TC1_TMAE=0 turns it off) when the
      // planes take 128-byte-swizzled 32 x 32 boxes
      static const int tmae_env = [] {
        const char* v = std::getenv("KB_TC1_TMAE");
        return v ? std::atoi(v) : 1;
      }();
      CUtensorMap em0, em1;
      std::memset(&em0, 0, sizeof(em0));
      std::memset(&em1, 0, sizeof(em1));
      auto emap = [&](CUtensorMap* m, const float* p) {
        return p && make_tmap(m, p, g.len, g.other, op->batch, g.len, e.bstride, 32, 4, 32, CU_TENSOR_MAP_SWIZZLE_128B);
      };
      bool tmae = tmae_env != 0;
      if (tmae) {
        if (MODE == kb::EPI_PLAIN) tmae = emap(&em0, e.out);
        else if (MODE == kb::EPI_RESID) tmae = emap(&em0, e.bsub) && emap(&em1, e.out);
        else if (MODE == kb::EPI_UPDATE) tmae = emap(&em0, e.y) && emap(&em1, e.x);
        else tmae = emap(&em0, e.vin) && emap(&em1, e.out);
      }
      const size_t ebytes = tmae ? kb::t1_ebuf_bytes<MODE>() + 1024 : 0;  // + alignment of the boxes
      const size_t fixed = 2 * (size_t)nbr * 1024 + ebytes;
      const size_t avail = 226 * 1024 - 1024;
      static const int nst_cap = [] {  // debugging: ring depth cap (KB_TC1_NST)
        const char* v = std::getenv("KB_TC1_NST");
        return v ? std::max(4, std::atoi(v)) : kb::kTcRingMax;
      }();
      // an even ring depth: with 5 stages the update kernel faulted ("unspecified launch failure",
      // legacy and TMA epilogues alike, while 4, 6 and 8 run clean); not root-caused
      const int nst = (fixed < avail ? std::min<int>(std::min(nst_cap, kb::kTcRingMax), (int)((avail - fixed) / kb::kTcStageBytes)) : 0) & ~1;
      const size_t smem = std::max<size_t>(1024 + (size_t)nst * kb::kTcStageBytes + fixed, 116 * 1024);
      const int nb = (int)std::min<long long>(sm_count(), nch1);
      CUtensorMap mapt;
      if (nst >= 4 && nb * kb::kT1Epi <= (op->slots_cap ? op->slots_cap : sum_blocks(op)) &&
          make_tmap(&mapt, zmap, g.other, zrows, (long long)op->batch * op->r, g.other, z_ps, kb::kTcRB, 4, 128)) {
        const bool nrm = !(MODE == kb::EPI_UPDATE && !e.want_norms);
        auto pick = [&](auto k11, auto k21, auto k12, auto k22, auto t11, auto t21, auto t12, auto t22) {
          using K = decltype(k11);
          K k = tmae ? (slots1 == 2 ? (nrm ? t12 : t22) : (nrm ? t11 : t21))
                     : (slots1 == 2 ? (nrm ? k12 : k22) : (nrm ? k11 : k21));
          return k;
        };
        auto kern = pick(kb::kb_pass_sum_tc1<MODE, true, 1, false>, kb::kb_pass_sum_tc1<MODE, false, 1, false>,
                         kb::kb_pass_sum_tc1<MODE, true, 2, false>, kb::kb_pass_sum_tc1<MODE, false, 2, false>,
                         kb::kb_pass_sum_tc1<MODE, true, 1, true>, kb::kb_pass_sum_tc1<MODE, false, 1, true>,
                         kb::kb_pass_sum_tc1<MODE, true, 2, true>, kb::kb_pass_sum_tc1<MODE, false, 2, true>);
        KB_TRY(allow_smem(kern, smem));
        if (op->batch > 1 && (MODE == kb::EPI_POWER || e.want_norms))  // warps skip untouched images
          KB_CUDA(cudaMemsetAsync(e.partials, 0, sizeof(double) * 4 * (size_t)op->batch * nb * kb::kT1Epi, s));
        c.slots = nb * kb::kT1Epi;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(nb);
        cfg.blockDim = dim3(kb::kT1Threads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = use_pdl() ? 1 : 0;
        c.engine = KB_ENGINE_TC_TF32;
        static const bool trace1 = std::getenv("KB_TC1_TRACE") != nullptr;
        if (trace1)
          std::fprintf(stderr, "[tc1] mode %d len %d other %d batch %d r %d Kw %d H %d nbr %d nst %d smem %zu tmae %d slots %d grid %d\n",
                       MODE, g.len, g.other, op->batch, op->r, g.Kw, g.H, nbr, nst, smem, (int)tmae, slots1, nb);
        KB_CUDA(cudaLaunchKernelEx(&cfg, kern, mapt, op->r, btab, g, e, op->batch, nst, em0, em1));
        return KB_OK;
      }
    }
    if (btab && use_tc(op, g, 128) && persistent_ok) {
      // tcgen05 sum pass (kb_tc.cuh): double-buffered bricks from the brick table, tile ring
      const int nbr = kb::tc_bricks(g.Kw);
      // epilogue operands staged by TMA (KB_TC1_TMAE=0 turns it off here too)
      static const int tmae_env = [] {
        const char* v = std::getenv("KB_TC1_TMAE");
        return v ? std::atoi(v) : 1;
      }();
      CUtensorMap em0, em1;
      std::memset(&em0, 0, sizeof(em0));
      std::memset(&em1, 0, sizeof(em1));
      auto emap = [&](CUtensorMap* m, const float* p) {
        return p && make_tmap(m, p, g.len, g.other, op->batch, g.len, e.bstride, 32, 4, 32, CU_TENSOR_MAP_SWIZZLE_128B);
      };
      bool tmae = tmae_env != 0;
      if (tmae) {
        if (MODE == kb::EPI_PLAIN) tmae = emap(&em0, e.out);
        else if (MODE == kb::EPI_RESID) tmae = emap(&em0, e.bsub) && emap(&em1, e.out);
        else if (MODE == kb::EPI_UPDATE) tmae = emap(&em0, e.y) && emap(&em1, e.x);
        else tmae = emap(&em0, e.vin) && emap(&em1, e.out);
      }
      const size_t fixed = 2 * (size_t)nbr * 1024 + (tmae ? kb::tc_ebuf_bytes<MODE>() + 1024 : 0);
      const size_t avail = 226 * 1024 - 1024;
      const int nst = (fixed < avail ? std::min<int>(kb::kTcRingMax, (int)((avail - fixed) / kb::kTcStageBytes)) : 0) & ~1;
      const size_t smem = std::max<size_t>(1024 + (size_t)nst * kb::kTcStageBytes + fixed, 116 * 1024);
      // chunks are dealt round-robin over one block per SM (kb::StrideWalk)
      const long long nch = (long long)((g.len + kb::kTcTS - 1) / kb::kTcTS) * ((g.other + 127) / 128) * op->batch;
      const int nb = (int)std::min<long long>(sm_count(), nch);
      CUtensorMap mapt;
      if (nst >= 4 && nb * kb::kTcSumEpi <= (op->slots_cap ? op->slots_cap : sum_blocks(op)) &&
          make_tmap(&mapt, zmap, g.other, zrows, (long long)op->batch * op->r, g.other, z_ps, kb::kTcRB, 4, 128)) {
        const bool nrm = !(MODE == kb::EPI_UPDATE && !e.want_norms);
        auto kern = tmae ? (nrm ? kb::kb_pass_sum_tc<MODE, true, true> : kb::kb_pass_sum_tc<MODE, false, true>)
                         : (nrm ? kb::kb_pass_sum_tc<MODE, true, false> : kb::kb_pass_sum_tc<MODE, false, false>);
        KB_TRY(allow_smem(kern, smem));
        if (op->batch > 1 && (MODE == kb::EPI_POWER || e.want_norms))  // warps skip untouched images
          KB_CUDA(cudaMemsetAsync(e.partials, 0, sizeof(double) * 4 * (size_t)op->batch * nb * kb::kTcSumEpi, s));
        c.slots = nb * kb::kTcSumEpi;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(nb);
        cfg.blockDim = dim3(kb::kTcSumThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = use_pdl() ? 1 : 0;
        c.engine = KB_ENGINE_TC_TF32;
        KB_CUDA(cudaLaunchKernelEx(&cfg, kern, mapt, op->r, btab, g, e, op->batch, nst, em0, em1));
        return KB_OK;
      }
    }
    if (use_tf32(op) && persistent_ok) {
      const kb::TileBoxesX tx = kb::tile_boxes_x(kb::tf32_rows(kb::kNW * 16, g.Kw));
      const size_t fixed = 2 * (size_t)op->r * kb::tf32_cstride(g.Kw) * sizeof(float);
      const int bps = blocks_per_sm(fixed + 2 * tx.stage_elems * sizeof(float));
      const int nst = ring_stages(tx.stage_elems * sizeof(float), fixed, bps);
      const size_t smem = fixed + sizeof(float) * (size_t)nst * tx.stage_elems;
      CUtensorMap mapx;
      if (bps > 0 && make_tmap(&mapx, zmap, g.other, zrows, (long long)op->batch * op->r, g.other, z_ps,
                               tx.box_rows, 4, kb::kXF))
      {
        c.engine = KB_ENGINE_MMA_TF32;
        if (MODE == kb::EPI_UPDATE && !e.want_norms) return launch(kb::kb_pass_sum_x<MODE, false>, smem, bps, mapx, nst);
        return launch(kb::kb_pass_sum_x<MODE>, smem, bps, mapx, nst);
      }
    }
    const kb::TileBoxesF tb = kb::tile_boxes_f(kb::kNW * 16 + g.Wp);
    const size_t smem = sizeof(float) * ((size_t)kb::kStages * tb.stage_elems + (size_t)op->r * g.Wp);
    const int bps = blocks_per_sm(smem);
    CUtensorMap map;
    if (use_tma_f32(op) && persistent_ok && bps > 0 &&
        make_tmap(&map, zmap, g.other, zrows, (long long)op->batch * op->r, g.other, z_ps, tb.box_rows, 4))
      return c.engine = KB_ENGINE_FFMA, launch(kb::kb_pass_sum_f<MODE>, smem, bps, map);
  }
  constexpr int TS = kb::kNW * kRB;
  const size_t smem = sizeof(T) * (2 * (size_t)(TS + g.Wp) * 32 + 2 * (size_t)g.Wp);
  auto kern = kb::kb_pass_sum<T, kRB, MODE>;
  KB_TRY(allow_smem(kern, smem));
  g = g_in;
  const long long z_bs = z_ps * op->r;
  const long long t_bs = (long long)op->r * g.Wp;
  dim3 grid((g.other + 31) / 32, (g.len + TS - 1) / TS, op->batch);
  dim3 block(32, kb::kNW);
  c.slots = (int)(grid.x * grid.y);
  c.engine = KB_ENGINE_GENERIC;
  kern<<<grid, block, smem, s>>>(z, z_ps, z_bs, op->r, tin, t_bs, g, tsign, e);
  KB_CUDA(cudaGetLastError());
  return KB_OK;
}

// Local row block of a (possibly sharded) image: rows [g0, g0+m) of m_global, with halo rows.
struct RowBlock {
  int g0, mg, hlo, hhi;
};

int debug_mode() {
  static const int mode = [] {
    const char* v = std::getenv("KB_DEBUG_MODE");
    return v ? std::atoi(v) : 0;
  }();
  return mode;
}

kb::AxisGeom geom_a(const kb_op* op, int adjoint, const RowBlock& rb) {
  kb::AxisGeom g;
  g.dbg = debug_mode();
  g.len = op->m;
  g.other = op->n;
  g.H = op->Ha;
  g.Wp = op->Wpa;
  g.Kw = (2 * op->Ha + 1 + 3) / 4 * 4;
  g.fill = op->bc_a == KB_BC_REFLECTIVE && (!adjoint || op->sym_a);
  g.g0 = rb.g0;
  g.Mg = rb.mg;
  g.halo_lo = rb.hlo;
  g.halo_hi = rb.hhi;
  return g;
}

kb::AxisGeom geom_b(const kb_op* op, int adjoint) {  // sum pass over Z_i^T [n][m]
  kb::AxisGeom g;
  g.dbg = debug_mode();
  g.len = op->n;
  g.other = op->m;
  g.H = op->Hb;
  g.Wp = op->Wpb;
  g.Kw = (2 * op->Hb + 1 + 3) / 4 * 4;
  g.fill = op->bc_b == KB_BC_REFLECTIVE && (!adjoint || op->sym_b);
  g.g0 = 0;
  g.Mg = op->n;
  g.halo_lo = 0;
  g.halo_hi = 0;
  return g;
}

template <typename T>
kb::Epi<T> epi_base(const kb_op* op, int mode) {
  kb::Epi<T> e;
  std::memset(&e, 0, sizeof(e));
  e.mode = mode;
  e.bstride = (long long)plane_elems(op);
  return e;
}

// Stage 0/2: pass A (forward / adjoint) incl. the adjoint's row fold. Stage 1/3 go through
// stage_b below (the column fold is launched just before pass B).
template <typename T>
int stage_a(const kb_op* op, int adjoint, const T* in, const Work& w, const RowBlock& rb,
            const double* nw2, cudaStream_t s) {
  T* z = z_row0<T>(op, w.z);
  const kb::AxisGeom ga = geom_a(op, adjoint, rb);
  // the following pass B reflect-fills axis 1: let the split store Z^T's reflected halo rows
  const int mirror_h = geom_b(op, adjoint).fill ? op->Hb : 0;
  const T* msign = (adjoint && op->sym_b) ? static_cast<const T*>(op->sign_b) : nullptr;
  if (mirror_h > op->n)  // folds leaving the domain: those halo rows must read as zero
    KB_CUDA(cudaMemsetAsync(w.z, 0, (size_t)z_plane(op) * op->r * op->batch * sizeof(T), s));
  KB_TRY(launch_a<T>(op, w.ctx, in, z, static_cast<const T*>(adjoint ? op->ta_corr : op->ta_conv), ga,
                     adjoint ? op->grp_adj : op->grp_fwd, nw2, mirror_h, msign, s));
  w.ctx.phase[adjoint ? 2 : 0] = w.ctx.engine;
  if (adjoint && op->bc_a == KB_BC_REFLECTIVE && !op->sym_a && op->Ha > 0) {
    const long long z_ps = z_plane(op);
    dim3 grid((op->n + 127) / 128, 2 * op->Ha * op->r, op->batch);
    kb::kb_fold_split<T><<<grid, 128, 0, s>>>(in, (long long)plane_elems(op), z, z_ps, z_ps * op->r, op->r,
                                               static_cast<const T*>(op->ta_conv),
                                               (long long)op->r * op->Wpa, ga,
                                               w.ctx.mirror ? mirror_h : 0, msign);
    KB_CUDA(cudaGetLastError());
  }
  return KB_OK;
}

template <typename T, int MODE>
int stage_b(const kb_op* op, int adjoint, kb::Epi<T> e, const Work& w, cudaStream_t s) {
  const T* z = z_row0<T>(op, w.z);
  const kb::AxisGeom gb = geom_b(op, adjoint);
  if (adjoint && op->bc_b == KB_BC_REFLECTIVE && !op->sym_b && op->Hb > 0) {
    dim3 grid((op->m + 127) / 128, 2 * op->Hb, op->batch);
    const long long z_ps = z_plane(op);
    kb::kb_fold_sum_pass<T><<<grid, 128, 0, s>>>(z, z_ps, z_ps * op->r, op->r,
                                                  static_cast<const T*>(op->tb_conv),
                                                  (long long)op->r * op->Wpb, gb,
                                                  static_cast<T*>(w.fold));
    KB_CUDA(cudaGetLastError());
    e.fold = static_cast<const T*>(w.fold);
    e.foldH = op->Hb;
  }
  const T* tsign = (adjoint && op->sym_b) ? static_cast<const T*>(op->sign_b) : nullptr;
  const int rc = launch_b<T, MODE>(op, w.ctx, z, static_cast<const T*>(adjoint ? op->tb_corr : op->tb_conv), gb,
                                   tsign, e, s);
  w.ctx.phase[adjoint ? 3 : 1] = w.ctx.engine;
  return rc;
}

// ---- one-sweep tcgen05 application (kb_fused.cuh) ------------------------------------------
// Both passes of one application in one kernel, the Z_i tiles handed over on chip (no Z^T round
// trip through HBM). Applies to fp32 operators whose pass-A band fits a resident 6-stage X tile
// (Ha <= 31) and whose pass-B band leaves >= 2 N-blocks per 128-column Z tile, without exact
// adjoint folds. OPT-IN (KB_FUSED=1): measured on the B200 it is latency-bound at ~9-12k cycles
// per (tile, term) against ~2.5k of MMA work -- cfg5 9.3 + 10.1 ms per iteration against 14.3 ms
// for the two-sweep passes, cfg3 4.2 against 3.3 ms (profiles/r02_fused_*.txt).
int fused_policy() {
  static const int p = [] {
    const char* v = std::getenv("KB_FUSED");
    return v ? std::atoi(v) : -1;
  }();
  return p;
}

size_t fused_smem(const kb::FuGeom& f) {
  return 1024 + (size_t)f.nxs * kb::kTcStageBytes + kb::kFuZsBytes + 2 * (size_t)(f.nbr_a + f.nbr_b) * 1024;
}

long long fused_tiles(const kb_op* op, const kb::FuGeom& f) { return (long long)f.LT * f.nchunks * op->batch; }

bool fused_plan(const kb_op* op, int adjoint, const RowBlock& rb, kb::FuGeom& f) {
  const int pol = fused_policy();
  if (pol == 0 || tc_policy(3) == 0 || op->dtype != KB_F32 || !use_tma_f32(op) || op->r > 32) return false;
  if (!(adjoint ? op->br_a_corr : op->br_a_conv) || !(adjoint ? op->br_bf_corr : op->br_bf_conv)) return false;
  const bool refl_a = op->bc_a == KB_BC_REFLECTIVE, refl_b = op->bc_b == KB_BC_REFLECTIVE;
  if (adjoint && ((refl_a && !op->sym_a) || (refl_b && !op->sym_b))) return false;  // exact folds
  std::memset(&f, 0, sizeof(f));
  // pass B's window is Hbf = Hb rounded up to 4: the X tile then starts at column c0 - Hbf, a
  // 16-byte boundary, as TMA requires of a box's innermost coordinate
  const int Kwa = (2 * op->Ha + 1 + 3) / 4 * 4, Kwb = (2 * op->Hbf + 1 + 3) / 4 * 4;
  f.qmax_a = (Kwa + 14) >> 3;
  f.qmax_b = (Kwb + 14) >> 3;
  const int nk_a = (15 + f.qmax_a + 1) & ~1;  // 8 N-blocks of 16 rows: K-steps 0 .. 14 + qmax_a
  f.na_a = nk_a / 2;
  f.nxs = (f.na_a + 1) / 2;
  if (f.nxs > kb::kFuXStMax) return false;
  // pass-B N-blocks whose K range (K-steps 0 .. 2(nblk-1) + qmax_b) stays inside the 128-row Z tile
  f.nblk = std::min(kb::kFuNbMax, (15 - f.qmax_b) / 2 + 1);
  if (f.qmax_b > 13 || f.nblk < 2) return false;
  f.nbr_a = kb::tc_bricks(Kwa);
  f.nbr_b = kb::tc_bricks(Kwb);
  f.len = op->m;
  f.n = op->n;
  f.Ha = op->Ha;
  f.Hb = op->Hbf;
  f.nchunks = ((op->n + 15) / 16 + f.nblk - 1) / f.nblk;
  f.LT = (op->m + kb::kFuL - 1) / kb::kFuL;
  f.fill_a = refl_a;
  f.fill_b = refl_b;
  f.g0 = rb.g0;
  f.Mg = rb.mg;
  f.halo_lo = rb.hlo;
  f.halo_hi = rb.hhi;
  f.sa_neg = 0;
  if (adjoint && refl_a)
    for (int i = 0; i < op->grp_adj.n; ++i)
      if (op->grp_adj.sign[i] < 0)
        for (int k = 0; k < op->grp_adj.count[i]; ++k) f.sa_neg |= 1u << (op->grp_adj.start[i] + k);
  f.dbg = debug_mode();
  if (fused_smem(f) > 226 * 1024) return false;
  const long long tiles = fused_tiles(op, f);
  const int nb = (int)std::min<long long>(sm_count(), tiles);
  if (nb * kb::kFuEpi > (op->slots_cap ? op->slots_cap : sum_blocks(op))) return false;
  (void)tiles;
  return pol == 1;
}

template <int MODE>
int launch_fused(const kb_op* op, Ctx& c, int adjoint, const float* in, const kb::FuGeom& f,
                 const kb::Epi<float>& e, const double* nw2, cudaStream_t s) {
  const unsigned* ba = adjoint ? op->br_a_corr : op->br_a_conv;
  const unsigned* bb = adjoint ? op->br_bf_corr : op->br_bf_conv;
  const float* sb = (adjoint && op->sym_b && op->bc_b == KB_BC_REFLECTIVE) ? static_cast<const float*>(op->sign_b)
                                                                          : nullptr;
  const size_t smem = fused_smem(f);
  static const int grid_cap = [] {  // debugging: fewer CTAs (KB_FUSED_GRID)
    const char* v = std::getenv("KB_FUSED_GRID");
    return v ? std::max(1, std::atoi(v)) : 1 << 30;
  }();
  const int nb = (int)std::min<long long>(std::min(sm_count(), grid_cap), fused_tiles(op, f));
  const long long in_bs = (long long)plane_elems(op);
  CUtensorMap map;
  if (!make_tmap(&map, in - (long long)f.halo_lo * op->n, op->n, (long long)op->m + f.halo_lo + f.halo_hi,
                 op->batch, op->n, in_bs, kb::kTcRB, 4, 128))
    return fail(KB_ERR_ARGUMENT, "input not aligned for the fused tcgen05 kernel");
  auto kern = MODE == kb::EPI_UPDATE && !e.want_norms ? kb::kb_fused_tc<MODE, false> : kb::kb_fused_tc<MODE>;
  KB_TRY(allow_smem(kern, smem));
  if (op->batch > 1 && (MODE == kb::EPI_POWER || e.want_norms))  // warps skip untouched images
    KB_CUDA(cudaMemsetAsync(e.partials, 0, sizeof(double) * 4 * (size_t)op->batch * nb * kb::kFuEpi, s));
  c.slots = nb * kb::kFuEpi;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(nb);
  cfg.blockDim = dim3(kb::kFuThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = use_pdl() ? 1 : 0;
  c.engine = KB_ENGINE_TC_FUSED;
  static const bool trace = std::getenv("KB_FUSED_TRACE") != nullptr;
  if (trace)
    std::fprintf(stderr,
                 "[fused] mode %d adj %d m %d n %d batch %d r %d Ha %d Hb %d qa %d qb %d na_a %d nxs %d nblk %d "
                 "nchunks %d LT %d fill %d/%d sa_neg %x grid %d smem %zu\n",
                 MODE, adjoint, op->m, op->n, op->batch, op->r, f.Ha, f.Hb, f.qmax_a, f.qmax_b, f.na_a, f.nxs, f.nblk,
                 f.nchunks, f.LT, f.fill_a, f.fill_b, f.sa_neg, nb, smem);
  KB_CUDA(cudaLaunchKernelEx(&cfg, kern, map, in, in_bs, ba, bb, f, sb, nw2, e, op->r, op->batch));
  return KB_OK;
}

// One application with epilogue MODE: the fused kernel where it applies, else pass A + pass B.
template <typename T, int MODE>
int apply_stage(const kb_op* op, int adjoint, const T* in, kb::Epi<T> e, const Work& w, const RowBlock& rb,
                const double* nw2, cudaStream_t s) {
  if constexpr (sizeof(T) == 4) {
    kb::FuGeom f;
    if (!(debug_mode() & 1024) && epi_aligned(e) && al16(in) && fused_plan(op, adjoint, rb, f)) {
      KB_TRY(launch_fused<MODE>(op, w.ctx, adjoint, in, f, e, nw2, s));
      w.ctx.phase[adjoint ? 2 : 0] = w.ctx.phase[adjoint ? 3 : 1] = KB_ENGINE_TC_FUSED;
      return KB_OK;
    }
  }
  KB_TRY(stage_a<T>(op, adjoint, in, w, rb, nw2, s));
  if (debug_mode() & 1024) return KB_OK;  // profiling / debugging: pass A only (Z^T left in the workspace)
  return stage_b<T, MODE>(op, adjoint, e, w, s);
}

// ---- operator application (one direction) ------------------------------------------------
template <typename T>
int apply_t(const kb_op* op, int adjoint, const T* X, T* Y, const Work& w, const RowBlock& rb,
            cudaStream_t s) {
  kb::Epi<T> e = epi_base<T>(op, kb::EPI_PLAIN);
  e.out = Y;
  return apply_stage<T, kb::EPI_PLAIN>(op, adjoint, X, e, w, rb, nullptr, s);
}

template <typename T>
int residual_t(const kb_op* op, const T* Y, const T* B, T* R, const Work& w, const RowBlock& rb,
               cudaStream_t s) {
  kb::Epi<T> e = epi_base<T>(op, kb::EPI_RESID);
  e.out = R;
  e.bsub = B;
  return apply_stage<T, kb::EPI_RESID>(op, 0, Y, e, w, rb, nullptr, s);
}

template <typename T>
kb::Epi<T> update_epi(const kb_op* op, T* X, T* Y, const Work& w, double beta, int k,
                      const double* Ldev, const double* ddev, int project, int* nonfinite,
                      bool norms) {
  kb::Epi<T> e = epi_base<T>(op, kb::EPI_UPDATE);
  e.x = X;
  e.y = Y;
  e.L = Ldev;
  e.denom = ddev;
  e.beta = beta;
  e.project = project;
  e.k = k;
  e.nonfinite = nonfinite;
  e.partials = w.partials;
  e.want_norms = norms;
  return e;
}

template <typename T>
int update_t(const kb_op* op, const T* R, T* X, T* Y, const Work& w, const RowBlock& rb,
             double beta, int k, const double* Ldev, const double* ddev, int project,
             int* nonfinite, double* norms_out, cudaStream_t s) {
  KB_TRY((apply_stage<T, kb::EPI_UPDATE>(op, 1, R, update_epi<T>(op, X, Y, w, beta, k, Ldev, ddev, project,
                                                                 nonfinite, norms_out != nullptr), w, rb, nullptr, s)));
  if (norms_out) {
    kb::kb_reduce_partials<<<op->batch, 256, 0, s>>>(w.partials, w.ctx.slots, 3, norms_out,
                                                      op->batch, 1);
    KB_CUDA(cudaGetLastError());
  }
  return KB_OK;
}

// ---- L2-blocked schedule of the fast path ------------------------------------------------
// The two-sweep iteration writes r Z_i^T planes in pass A and reads them back in pass B. When
// they do not fit in L2 (cfg3's 512-image batch: 2.2 GB; cfg5's 16384^2: 11 GB) that round trip
// dominates DRAM traffic. The blocked schedule runs the same kernels on L2-sized pieces so each
// piece's Z^T is consumed while it is still in L2:
//  * batches: groups of whole images; per group residual then update (images are independent);
//  * one image: row strips [r0, r0+S) viewed as row blocks (the multi-GPU halo machinery, the
//    neighbouring strips' rows are the halo); strip s's update needs R of strip s+1 (axis-0 halo
//    of the adjoint), so the order is res(0), res(1), upd(0), res(2), upd(1), ..., upd(N-1).
// A piece is a shallow view of the operator (same device tables, offset per image group).
struct BlockPlanC {
  int pieces = 1;  // image groups or row strips
  int size = 0;    // images per group / rows per strip
  bool strips = false;
};

// Rows per strip / images per group: env KB_L2_STRIP / KB_L2_GROUP (0 = off; "auto" = the
// largest piece whose Z^T set fits in the L2 budget, only when the whole set does not). OFF by
// default: measured on the B200 (tools/l2_blocking_exp.py, profiles/README.md) the smaller
// launches lose more to ramp/tail and wave quantisation than the L2 round trip saves
// (cfg5: 14.6 -> 16.2-19.8 ms per iteration; cfg3: 3.14 -> 3.56-6.14 ms).
BlockPlanC blocked_plan(const kb_op* op) {
  BlockPlanC p;
  const size_t zrow = (size_t)op->r * (op->n + 2 * op->Hb) * elem(op);  // Z^T bytes per image row
  const size_t zimg = zrow * op->m;
  static const long long budget = [] {
    const char* v = std::getenv("KB_L2_BUDGET_MB");
    return (v ? std::atoll(v) : 48LL) << 20;
  }();
  const char* es = std::getenv("KB_L2_STRIP");
  const char* eg = std::getenv("KB_L2_GROUP");
  if (op->batch > 1) {
    if (!eg) return p;
    int g = std::atoi(eg);
    if (std::string(eg) == "auto") {
      if (zimg * op->batch <= (size_t)budget * 2) return p;
      g = (int)std::max<long long>(1, budget / (long long)zimg);
    }
    if (g <= 0 || g >= op->batch) return p;
    p.size = g;
    p.pieces = (op->batch + g - 1) / g;
    return p;
  }
  if (!es) return p;
  int S = std::atoi(es);
  if (std::string(es) == "auto") {
    if (zimg <= (size_t)budget * 2) return p;
    S = (int)(budget / (long long)zrow) / 128 * 128;
    if (S < 128) S = 128;
  }
  if (S <= 0 || S >= op->m || S < op->Ha) return p;
  p.size = S;
  p.pieces = (op->m + S - 1) / S;
  p.strips = true;
  return p;
}

// view of images [b0, b0+gb) of a batched operator
kb_op group_view(const kb_op* op, int b0, int gb, long long scale) {
  kb_op v = *op;
  v.graph = nullptr;
  v.slots_cap = sum_blocks(op);
  v.batch = gb;
  v.chunk_scale = scale;
  const size_t e = elem(op);
  auto off = [&](void* p, long long per_image_elems, size_t esz) -> void* {
    return p ? static_cast<unsigned char*>(p) + (size_t)b0 * per_image_elems * esz : nullptr;
  };
  v.ta_conv = off(op->ta_conv, (long long)op->r * op->Wpa, e);
  v.ta_corr = off(op->ta_corr, (long long)op->r * op->Wpa, e);
  v.tb_conv = off(op->tb_conv, (long long)op->r * op->Wpb, e);
  v.tb_corr = off(op->tb_corr, (long long)op->r * op->Wpb, e);
  v.sign_b = off(op->sign_b, op->r, e);
  const long long ka = (2 * op->Ha + 1 + 3) / 4 * 4, kbw = (2 * op->Hb + 1 + 3) / 4 * 4;
  const long long bra = (long long)op->r * kb::tc_bricks((int)ka) * 256;
  const long long brb = (long long)op->r * kb::tc_bricks((int)kbw) * 256;
  v.br_a_conv = static_cast<unsigned*>(off(op->br_a_conv, bra, sizeof(unsigned)));
  v.br_a_corr = static_cast<unsigned*>(off(op->br_a_corr, bra, sizeof(unsigned)));
  v.br_b_conv = static_cast<unsigned*>(off(op->br_b_conv, brb, sizeof(unsigned)));
  v.br_b_corr = static_cast<unsigned*>(off(op->br_b_corr, brb, sizeof(unsigned)));
  const long long brbf = (long long)op->r * kb::tc_bricks((2 * op->Hbf + 1 + 3) / 4 * 4) * 256;
  v.br_bf_conv = static_cast<unsigned*>(off(op->br_bf_conv, brbf, sizeof(unsigned)));
  v.br_bf_corr = static_cast<unsigned*>(off(op->br_bf_corr, brbf, sizeof(unsigned)));
  return v;
}

// view of a row strip of height S of a single-image operator
kb_op strip_view(const kb_op* op, int S, long long scale) {
  kb_op v = *op;
  v.graph = nullptr;
  v.slots_cap = sum_blocks(op);
  v.m = S;
  v.chunk_scale = scale;
  return v;
}

template <typename T>
int sfista_blocked(const kb_op* op, const BlockPlanC& p, const T* B, T* X, T* Y, const Work& w,
                   const double* beta, int k0, int iters, int project, int* nonfinite, cudaStream_t s) {
  T* R = static_cast<T*>(w.rp);
  const long long pe = (long long)plane_elems(op);
  if (!p.strips) {
    for (int it = 0; it < iters; ++it) {
      const int k = k0 + it + 1;
      for (int g = 0; g < p.pieces; ++g) {
        const int b0 = g * p.size, gb = std::min(p.size, op->batch - b0);
        const kb_op v = group_view(op, b0, gb, p.pieces);
        Work wv = w;
        const long long o = (long long)b0 * pe;
        const RowBlock rb{0, op->m, 0, 0};
        KB_TRY(residual_t<T>(&v, Y + o, B + o, R + o, wv, rb, s));
        KB_TRY(update_t<T>(&v, R + o, X + o, Y + o, wv, rb, beta[k - 1], k, w.scal + b0,
                           w.scal + op->batch + b0, project, nonfinite, nullptr, s));
        for (int i = 0; i < 4; ++i) w.ctx.phase[i] = wv.ctx.phase[i];
      }
    }
    return KB_OK;
  }
  const int N = p.pieces, S = p.size;
  auto piece = [&](int i, int& r0, int& rows, RowBlock& rb) {
    r0 = i * S;
    rows = std::min(S, op->m - r0);
    rb = RowBlock{r0, op->m, r0 > 0 ? op->Ha : 0, r0 + rows < op->m ? op->Ha : 0};
  };
  auto res = [&](int i) -> int {
    int r0, rows;
    RowBlock rb;
    piece(i, r0, rows, rb);
    const kb_op v = strip_view(op, rows, N);
    Work wv = w;
    const long long o = (long long)r0 * op->n;
    const int rc = residual_t<T>(&v, Y + o, B + o, R + o, wv, rb, s);
    w.ctx.phase[0] = wv.ctx.phase[0];
    w.ctx.phase[1] = wv.ctx.phase[1];
    return rc;
  };
  auto upd = [&](int i, int k) -> int {
    int r0, rows;
    RowBlock rb;
    piece(i, r0, rows, rb);
    const kb_op v = strip_view(op, rows, N);
    Work wv = w;
    const long long o = (long long)r0 * op->n;
    const int rc = update_t<T>(&v, R + o, X + o, Y + o, wv, rb, beta[k - 1], k, w.scal, w.scal + 1, project,
                               nonfinite, nullptr, s);
    w.ctx.phase[2] = wv.ctx.phase[2];
    w.ctx.phase[3] = wv.ctx.phase[3];
    return rc;
  };
  for (int it = 0; it < iters; ++it) {
    const int k = k0 + it + 1;
    KB_TRY(res(0));
    for (int i = 0; i + 1 < N; ++i) {
      KB_TRY(res(i + 1));
      KB_TRY(upd(i, k));
    }
    KB_TRY(upd(N - 1, k));
  }
  return KB_OK;
}

template <typename T>
int sfista_launches(const kb_op* op, const T* B, T* X, T* Y, const Work& w, const double* beta,
                    int k0, int iters, int project, int* nonfinite, double* norms,
                    cudaStream_t s) {
  T* R = static_cast<T*>(w.rp);
  if (!norms) {
    const BlockPlanC p = blocked_plan(op);
    if (p.pieces > 1) return sfista_blocked<T>(op, p, B, X, Y, w, beta, k0, iters, project, nonfinite, s);
  }
  const RowBlock rb{0, op->m, 0, 0};
  for (int it = 0; it < iters; ++it) {
    const int k = k0 + it + 1;
    KB_TRY(residual_t<T>(op, Y, B, R, w, rb, s));
    KB_TRY(update_t<T>(op, R, X, Y, w, rb, beta[k - 1], k, w.scal, w.scal + op->batch, project,
                       nonfinite, norms ? norms + (size_t)it * 4 * op->batch : nullptr, s));
  }
  return KB_OK;
}

template <typename T>
int power_t(const kb_op* op, T* v, T* wbuf, const Work& w, int iters, double* hist,
            cudaStream_t s) {
  T* u = static_cast<T*>(w.rp);
  const RowBlock rb{0, op->m, 0, 0};
  for (int k = 0; k < iters; ++k) {
    T* cur = (k & 1) ? wbuf : v;   // holds w_{k-1} (unnormalised) or v_0
    T* nxt = (k & 1) ? v : wbuf;
    const double* nw2 = k == 0 ? nullptr : hist + (size_t)(k - 1) * 2 * op->batch + op->batch;
    kb::Epi<T> e1 = epi_base<T>(op, kb::EPI_PLAIN);
    e1.out = u;
    KB_TRY((apply_stage<T, kb::EPI_PLAIN>(op, 0, cur, e1, w, rb, nw2, s)));
    kb::Epi<T> e2 = epi_base<T>(op, kb::EPI_POWER);
    e2.out = nxt;
    e2.vin = cur;
    e2.vnw2 = nw2;
    e2.partials = w.partials;
    KB_TRY((apply_stage<T, kb::EPI_POWER>(op, 1, u, e2, w, rb, nullptr, s)));
    kb::kb_reduce_partials<<<op->batch, 256, 0, s>>>(w.partials, w.ctx.slots, 2,
                                                      hist + (size_t)k * 2 * op->batch,
                                                      op->batch, 1);
    KB_CUDA(cudaGetLastError());
  }
  return KB_OK;
}

int check_op(const kb_op* op) {
  if (!op) return fail(KB_ERR_ARGUMENT, "null operator handle");
  return KB_OK;
}

// table build: conv[k] = c_{H-k}, corr[k] = c_{k-H}, k in [0, 2H], zero elsewhere; row
// (b, i) of the tables holds host term perm[i] of image b
template <typename T>
void build_tables(int dlo, int w, const double* taps, int batch, int r, const std::vector<int>& perm,
                  int H, int Wp, std::vector<T>& conv, std::vector<T>& corr) {
  conv.assign((size_t)batch * r * Wp, T(0));
  corr.assign((size_t)batch * r * Wp, T(0));
  for (int b = 0; b < batch; ++b)
    for (int i = 0; i < r; ++i) {
      const double* src = taps + ((size_t)b * r + perm[i]) * w;
      T* cv = conv.data() + ((size_t)b * r + i) * Wp;
      T* cr = corr.data() + ((size_t)b * r + i) * Wp;
      for (int t = 0; t < w; ++t) {
        const int d = dlo + t;
        cv[H - d] = (T)src[t];
        cr[H + d] = (T)src[t];
      }
    }
}

template <typename T>
int upload_tables(kb_op* op, int dlo, int w, const double* taps, const std::vector<int>& perm, int H,
                  int Wp, void** conv_d, void** corr_d, std::vector<double>* keep_conv = nullptr,
                  std::vector<double>* keep_corr = nullptr) {
  std::vector<T> conv, corr;
  build_tables<T>(dlo, w, taps, op->batch, op->r, perm, H, Wp, conv, corr);
  if constexpr (sizeof(T) == 8) {
    if (keep_conv) *keep_conv = conv;
    if (keep_corr) *keep_corr = corr;
  }
  const size_t bytes = conv.size() * sizeof(T);
  KB_CUDA(cudaMalloc(conv_d, bytes));
  KB_CUDA(cudaMalloc(corr_d, bytes));
  KB_CUDA(cudaMemcpy(*conv_d, conv.data(), bytes, cudaMemcpyHostToDevice));
  KB_CUDA(cudaMemcpy(*corr_d, corr.data(), bytes, cudaMemcpyHostToDevice));
  return KB_OK;
}

// brick tables of an axis' two fp32 tap tables, when its band can take the tcgen05 passes
int build_brick_tables(kb_op* op, int H, int Wp, const void* conv, const void* corr, unsigned** bconv,
                       unsigned** bcorr, int shift = 0) {
  const int Kw = (2 * H + 1 + 3) / 4 * 4;  // every fp32 band: the fused kernel takes narrow ones too
  const int nbr = kb::tc_bricks((2 * (H + shift) + 1 + 3) / 4 * 4);
  const long long bt = (long long)op->batch * op->r;
  const size_t bytes = (size_t)bt * nbr * 1024;
  KB_CUDA(cudaMalloc(bconv, bytes));
  KB_CUDA(cudaMalloc(bcorr, bytes));
  const int blocks = (int)std::min<long long>((bt * nbr * 128 + 255) / 256, 4096);
  kb::kb_build_bricks<<<blocks, 256>>>(static_cast<const float*>(conv), Wp, Kw, nbr, bt, *bconv, shift);
  kb::kb_build_bricks<<<blocks, 256>>>(static_cast<const float*>(corr), Wp, Kw, nbr, bt, *bcorr, shift);
  KB_CUDA(cudaGetLastError());
  KB_CUDA(cudaDeviceSynchronize());
  return KB_OK;
}
template <typename T>
int upload_signs(kb_op* op, const std::vector<int>& sign) {
  std::vector<T> v(sign.begin(), sign.end());
  KB_CUDA(cudaMalloc(&op->sign_b, v.size() * sizeof(T)));
  KB_CUDA(cudaMemcpy(op->sign_b, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return KB_OK;
}

// (Anti)symmetry of a band: sign +1 if c_d ~ c_{-d}, -1 if c_d ~ -c_{-d}; ok when the residual
// is within kSymTol * max|c|. For such generators the adjoint's folded sources equal the
// reflect-filled tile times the sign, so F^T needs no separate fold (see kb_kernels.cuh).
void classify(const double* taps, int dlo, int w, int& sign, bool& ok) {
  const int H = std::max(std::abs(dlo), std::abs(dlo + w - 1));
  std::vector<double> full(2 * H + 1, 0.0);
  for (int t = 0; t < w; ++t) full[dlo + t + H] = taps[t];
  double mx = 0, rs = 0, ra = 0;
  for (int k = 0; k <= 2 * H; ++k) {
    mx = std::max(mx, std::fabs(full[k]));
    rs = std::max(rs, std::fabs(full[k] - full[2 * H - k]));
    ra = std::max(ra, std::fabs(full[k] + full[2 * H - k]));
  }
  sign = rs <= ra ? 1 : -1;
  ok = std::min(rs, ra) <= kSymTol * mx;
}

void free_op(kb_op* op) {
  if (!op) return;
  free_op(op->twin);
  cudaFree(op->sign_b);
  cudaFree(op->ta_conv);
  cudaFree(op->ta_corr);
  cudaFree(op->tb_conv);
  cudaFree(op->tb_corr);
  cudaFree(op->br_a_conv);
  cudaFree(op->br_a_corr);
  cudaFree(op->br_b_conv);
  cudaFree(op->br_b_corr);
  if (op->br_bf_conv != op->br_b_conv) cudaFree(op->br_bf_conv);
  if (op->br_bf_corr != op->br_b_corr) cudaFree(op->br_bf_corr);
  if (op->graph) {
    if (op->graph->exec) cudaGraphExecDestroy(op->graph->exec);
    delete op->graph;
  }
  delete op;
}


// ---- measurement helpers (bench.py) --------------------------------------------------------
template <typename T>
__global__ void kb_fma_burn(T* out, int iters, T a, T b) {
  T x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = T(threadIdx.x + i) * T(1e-3);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = kb::kb_fma(x[i], a, b);
  }
  T s = T(0);
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == T(-12345.678)) out[0] = s;  // never true; keeps the chains alive
}

// FP64 tensor-core burn: 8 independent m8n8k4 DMMA accumulators per warp (256 FMAs each)
__global__ void kb_dmma_burn(double* out, int iters) {
  const double a = threadIdx.x * 1e-3, b = threadIdx.x * 2e-3;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) kb::dmma_884(c[i][0], c[i][1], a, b);
  }
  double sum = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) sum += c[i][0] + c[i][1];
  if (sum == -12345.678) out[0] = sum;
}

// TF32 tensor-core burn: 12 independent m16n8k8 accumulators per warp (1024 FMAs each)
__global__ void kb_tf32_burn(float* out, int iters) {
  unsigned a[4], b[2];
#pragma unroll
  for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(threadIdx.x * 1e-3f + i);
#pragma unroll
  for (int i = 0; i < 2; ++i) b[i] = __float_as_uint(threadIdx.x * 2e-3f - i);
  float c[12][4];
#pragma unroll
  for (int i = 0; i < 12; ++i) c[i][0] = c[i][1] = c[i][2] = c[i][3] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 12; ++i) kb::mma_tf32(c[i], a, b[0], b[1]);
  }
  float sum = 0.f;
#pragma unroll
  for (int i = 0; i < 12; ++i) sum += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  if (sum == -12345.678f) out[0] = sum;
}

// Peak of the arithmetic instruction the pass kernels issue: DMMA for fp64, TF32 mma.sync for
// fp32 (raw TF32 rate; the 3xTF32 passes issue three per product).
template <typename T>
int fma_peak_t(float* tflops, cudaStream_t s) {
  int dev = 0, sms = 0;
  KB_CUDA(cudaGetDevice(&dev));
  KB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  T* out = nullptr;
  KB_CUDA(cudaMalloc(&out, sizeof(T)));
  const int blocks = sms * 8, threads = 256, iters = sizeof(T) == 8 ? 4096 : 16384;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 5;
  auto burn = [&]() {
    if constexpr (sizeof(T) == 8) kb_dmma_burn<<<blocks, threads, 0, s>>>(out, iters / 8);
    else kb_tf32_burn<<<blocks, threads, 0, s>>>(reinterpret_cast<float*>(out), iters / 16);
  };
  burn();  // warm-up
  cudaEventRecord(e0, s);
  for (int r = 0; r < reps; ++r) burn();
  cudaEventRecord(e1, s);
  cudaError_t ce = cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (ce != cudaSuccess) return fail(KB_ERR_CUDA, cudaGetErrorString(ce));
  const double flops = sizeof(T) == 8 ? 2.0 * 256.0 * 8.0 * (double)(iters / 8) * (threads / 32) * blocks * reps
                                      : 2.0 * 1024.0 * 12.0 * (double)(iters / 16) * (threads / 32) * blocks * reps;
  *tflops = (float)(flops / (ms * 1e-3) / 1e12);
  return KB_OK;
}

// tcgen05 kind::tf32 rate (TFLOP/s): kb_tc_burn, one CTA per SM, two MMA streams each
int tc_peak(float* tflops, cudaStream_t s) {
  const int sms = sm_count(), iters = 4096, reps = 5;
  float* out = nullptr;
  KB_CUDA(cudaMalloc(&out, sizeof(float)));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kb::kb_tc_burn<<<sms, 128, 0, s>>>(256, out);  // warm-up
  cudaEventRecord(e0, s);
  for (int r = 0; r < reps; ++r) kb::kb_tc_burn<<<sms, 128, 0, s>>>(iters, out);
  cudaEventRecord(e1, s);
  cudaError_t ce = cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (ce != cudaSuccess) return fail(KB_ERR_CUDA, cudaGetErrorString(ce));
  *tflops = (float)(2.0 * 128 * 256 * 8 * (double)iters * 2 * sms * reps / (ms * 1e-3) / 1e12);
  return KB_OK;
}

// Per-phase GPU time of one iteration's four kernels: each phase's `reps` launches are
// captured into a CUDA graph (as in the solver's fast path, so host launch cost is excluded)
// and the graph is timed with events on a private stream.
template <typename T>
int time_passes_t(const kb_op* op, const T* Y, const T* B, T* R, T* X, T* Yio, const Work& w,
                  int reps, float* ms4, int* nonfinite, cudaStream_t caller) {
  cudaStream_t s;
  KB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  KB_CUDA(cudaStreamSynchronize(caller));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const RowBlock rb{0, op->m, 0, 0};
  kb::Epi<T> er = epi_base<T>(op, kb::EPI_RESID);
  er.out = R;
  er.bsub = B;
  const kb::Epi<T> eu = update_epi<T>(op, X, Yio, w, 0.0, 1, w.scal, w.scal + op->batch, 1,
                                      nonfinite, false);
  int rc = KB_OK;
  // fused directions (kb_fused.cuh): phase 0 / 2 time the one-sweep kernel, phase 1 / 3 are empty
  bool fused[2] = {false, false};
  if constexpr (sizeof(T) == 4) {
    kb::FuGeom f;
    fused[0] = !(debug_mode() & 1024) && epi_aligned(er) && al16(Y) && fused_plan(op, 0, rb, f);
    fused[1] = !(debug_mode() & 1024) && epi_aligned(eu) && al16(R) && fused_plan(op, 1, rb, f);
  }
  for (int phase = 0; phase < 4 && rc == KB_OK; ++phase) {
    if (fused[phase >> 1] && (phase & 1)) {
      ms4[phase] = 0.f;
      std::lock_guard<std::mutex> lock(g_phase_mu);
      op->phase_engine[phase] = KB_ENGINE_TC_FUSED;
      continue;
    }
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      rc = fail(KB_ERR_CUDA, "stream capture failed");
      break;
    }
    for (int rep = 0; rep < reps && rc == KB_OK; ++rep) {
      switch (phase) {
        case 0:
          rc = fused[0] ? apply_stage<T, kb::EPI_RESID>(op, 0, Y, er, w, rb, nullptr, s)
                        : stage_a<T>(op, 0, Y, w, rb, nullptr, s);
          break;
        case 1: rc = stage_b<T, kb::EPI_RESID>(op, 0, er, w, s); break;
        case 2:
          rc = fused[1] ? apply_stage<T, kb::EPI_UPDATE>(op, 1, R, eu, w, rb, nullptr, s)
                        : stage_a<T>(op, 1, R, w, rb, nullptr, s);
          break;
        default: rc = stage_b<T, kb::EPI_UPDATE>(op, 1, eu, w, s); break;
      }
    }
    {
      std::lock_guard<std::mutex> lock(g_phase_mu);
      op->phase_engine[phase] = w.ctx.engine;
    }
    cudaError_t ce = cudaStreamEndCapture(s, &graph);
    if (rc == KB_OK && ce == cudaSuccess) ce = cudaGraphInstantiate(&exec, graph, 0);
    if (rc == KB_OK && ce == cudaSuccess) ce = cudaGraphLaunch(exec, s);  // warm-up
    if (rc == KB_OK && ce == cudaSuccess) {
      cudaEventRecord(e0, s);
      ce = cudaGraphLaunch(exec, s);
      cudaEventRecord(e1, s);
    }
    if (rc == KB_OK && ce == cudaSuccess) ce = cudaEventSynchronize(e1);
    if (rc == KB_OK && ce == cudaSuccess) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      ms4[phase] = ms / reps;
    }
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    if (rc == KB_OK && ce != cudaSuccess) rc = fail(KB_ERR_CUDA, cudaGetErrorString(ce));
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  return rc;
}

}  // namespace

extern "C" {

const char* kb_version(void) { return "kronblur_b200 0.1 sm_100a"; }
const char* kb_last_error(void) { return g_err.c_str(); }
int kb_max_half_width(void) { return kMaxHalf; }

int kb_op_create(kb_op** out, int dtype, int m, int n, int r, int batch, int bc_a, int bc_b,
                 int a_dlo, int a_w, const double* a_taps, int b_dlo, int b_w,
                 const double* b_taps) {
  static thread_local bool creating_twin = false;
  if (!out) return fail(KB_ERR_ARGUMENT, "null output handle");
  *out = nullptr;
  if (dtype != KB_F64 && dtype != KB_F32) return fail(KB_ERR_ARGUMENT, "dtype must be KB_F64 or KB_F32");
  if (m < 1 || n < 1 || r < 1 || batch < 1) return fail(KB_ERR_ARGUMENT, "m, n, r, batch must be >= 1");
  if (a_w < 1 || b_w < 1 || !a_taps || !b_taps) return fail(KB_ERR_ARGUMENT, "empty band");
  if ((bc_a != KB_BC_ZERO && bc_a != KB_BC_REFLECTIVE) || (bc_b != KB_BC_ZERO && bc_b != KB_BC_REFLECTIVE))
    return fail(KB_ERR_ARGUMENT, "bad boundary condition");
  const int Ha = std::max(std::abs(a_dlo), std::abs(a_dlo + a_w - 1));
  const int Hb = std::max(std::abs(b_dlo), std::abs(b_dlo + b_w - 1));
  if (Ha > kMaxHalf || Hb > kMaxHalf) return fail(KB_ERR_ARGUMENT, "band half width exceeds kb_max_half_width()");
  kb_op* op = new kb_op();
  op->dtype = dtype;
  op->m = m;
  op->n = n;
  op->r = r;
  op->batch = batch;
  op->bc_a = bc_a;
  op->bc_b = bc_b;
  op->Ha = Ha;
  op->Hb = Hb;
  op->Wpa = (2 * Ha + 1 + kb::kUB - 1) / kb::kUB * kb::kUB;  // multiple of both passes' R
  op->Wpb = (2 * Hb + 1 + kb::kUB - 1) / kb::kUB * kb::kUB;
  op->gmax = dtype == KB_F64 ? kGmaxF64 : kGmaxF32;
  if ((r + op->gmax - 1) / op->gmax + 1 > kb::kMaxGroups) {
    delete op;
    return fail(KB_ERR_ARGUMENT, "too many terms for the pass A group table");
  }
  op->graph = new GraphCache();

  // Symmetry classes. Axis a: terms are reordered so that the adjoint's pass A groups are
  // homogeneous in fill sign (same order for every image, else the exact fold path is used).
  const char* exact_env = std::getenv("KB_EXACT_FOLD");
  const bool exact = exact_env && exact_env[0] && exact_env[0] != '0';
  std::vector<int> sa((size_t)batch * r), sb((size_t)batch * r);
  bool ok_a = bc_a == KB_BC_REFLECTIVE && !exact, ok_b = bc_b == KB_BC_REFLECTIVE && !exact;
  for (int b = 0; b < batch; ++b)
    for (int i = 0; i < r; ++i) {
      bool oka, okb;
      classify(a_taps + ((size_t)b * r + i) * a_w, a_dlo, a_w, sa[(size_t)b * r + i], oka);
      classify(b_taps + ((size_t)b * r + i) * b_w, b_dlo, b_w, sb[(size_t)b * r + i], okb);
      ok_a = ok_a && oka;
      ok_b = ok_b && okb;
    }
  std::vector<int> perm(r);
  for (int i = 0; i < r; ++i) perm[i] = i;
  if (ok_a) {
    std::stable_sort(perm.begin(), perm.end(), [&](int x, int y) { return sa[x] > sa[y]; });
    for (int b = 1; b < batch && ok_a; ++b)
      for (int i = 0; i < r; ++i)
        if (sa[(size_t)b * r + perm[i]] != sa[perm[i]]) ok_a = false;
    if (!ok_a)
      for (int i = 0; i < r; ++i) perm[i] = i;
  }
  op->sym_a = ok_a;
  op->sym_b = ok_b;
  op->grp_fwd.n = 0;
  add_groups(op->grp_fwd, 0, r, op->gmax, 1);
  op->grp_adj.n = 0;
  if (ok_a) {
    int nsym = 0;
    while (nsym < r && sa[perm[nsym]] > 0) ++nsym;
    add_groups(op->grp_adj, 0, nsym, op->gmax, 1);
    add_groups(op->grp_adj, nsym, r - nsym, op->gmax, -1);
  } else {
    add_groups(op->grp_adj, 0, r, op->gmax, 1);
  }
  std::vector<int> sign_b((size_t)batch * r);
  for (int b = 0; b < batch; ++b)
    for (int i = 0; i < r; ++i) sign_b[(size_t)b * r + i] = sb[(size_t)b * r + perm[i]];

  int rc;
  if (dtype == KB_F64) {
    rc = upload_tables<double>(op, a_dlo, a_w, a_taps, perm, Ha, op->Wpa, &op->ta_conv, &op->ta_corr,
                               &op->h_conv[0], &op->h_corr[0]);
    if (rc == KB_OK)
      rc = upload_tables<double>(op, b_dlo, b_w, b_taps, perm, Hb, op->Wpb, &op->tb_conv, &op->tb_corr,
                                 &op->h_conv[1], &op->h_corr[1]);
    if (rc == KB_OK && ok_b) rc = upload_signs<double>(op, sign_b);
  } else {
    rc = upload_tables<float>(op, a_dlo, a_w, a_taps, perm, Ha, op->Wpa, &op->ta_conv, &op->ta_corr);
    if (rc == KB_OK) rc = upload_tables<float>(op, b_dlo, b_w, b_taps, perm, Hb, op->Wpb, &op->tb_conv, &op->tb_corr);
    if (rc == KB_OK && ok_b) rc = upload_signs<float>(op, sign_b);
    if (rc == KB_OK)
      rc = build_brick_tables(op, Ha, op->Wpa, op->ta_conv, op->ta_corr, &op->br_a_conv, &op->br_a_corr);
    if (rc == KB_OK)
      rc = build_brick_tables(op, Hb, op->Wpb, op->tb_conv, op->tb_corr, &op->br_b_conv, &op->br_b_corr);
    op->Hbf = (Hb + 3) / 4 * 4;
    if (rc == KB_OK && op->Hbf != Hb)
      rc = build_brick_tables(op, Hb, op->Wpb, op->tb_conv, op->tb_corr, &op->br_bf_conv, &op->br_bf_corr,
                              op->Hbf - Hb);
    if (op->Hbf == Hb) {
      op->br_bf_conv = op->br_b_conv;
      op->br_bf_corr = op->br_b_corr;
    }
  }
  if (rc != KB_OK) {
    free_op(op);
    return rc;
  }
  // Axis swap (measured at cfg5, tools/swap_exp.py: 15.2-15.5 -> 14.7 ms per iteration): the
  // two-sweep passes re-read and re-convert (TS + 2H)/TS input rows per output in pass B, so the
  // wider band belongs in pass A. For large fp32 single images with a markedly wider axis-1 band
  // the fast sFISTA path solves the transposed problem with this twin. KB_AXIS_SWAP=0/1 overrides.
  static const int swap_env = [] {
    const char* v = std::getenv("KB_AXIS_SWAP");
    return v ? std::atoi(v) : -1;
  }();
  const bool want = swap_env == 1 || (swap_env < 0 && dtype == KB_F32 && (long long)m * n >= 4096LL * 4096);
  if (!creating_twin && batch == 1 && Hb >= Ha + 8 && want) {
    creating_twin = true;
    kb_op* tw = nullptr;
    rc = kb_op_create(&tw, dtype, n, m, r, batch, bc_b, bc_a, b_dlo, b_w, b_taps, a_dlo, a_w, a_taps);
    creating_twin = false;
    if (rc != KB_OK) {
      free_op(op);
      return rc;
    }
    op->twin = tw;
  }
  *out = op;
  return KB_OK;
}

int kb_op_destroy(kb_op* op) {
  free_op(op);
  return KB_OK;
}

size_t kb_workspace_bytes(const kb_op* op) {
  if (!op) return 0;
  size_t b = layout(op, nullptr).bytes;
  if (op->twin) b = twin_planes_offset(op) + 3 * align_up(plane_elems(op) * elem(op), 256);
  return b;
}

int kb_op_info(const kb_op* op, int* info, int n) {
  KB_TRY(check_op(op));
  const int v[9] = {op->Ha, op->Wpa, op->Hb, op->Wpb, op->sym_a, op->sym_b, op->grp_adj.n, op->gmax,
                    op->twin != nullptr};
  for (int i = 0; i < n && i < 9; ++i) info[i] = v[i];
  return KB_OK;
}

int kb_apply(const kb_op* op, const void* X, void* Y, void* work, void* stream) {
  KB_TRY(check_op(op));
  Work w = layout(op, work);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (op->dtype == KB_F64)
    return apply_t<double>(op, 0, static_cast<const double*>(X), static_cast<double*>(Y), w, RowBlock{0, op->m, 0, 0}, s);
  return apply_t<float>(op, 0, static_cast<const float*>(X), static_cast<float*>(Y), w, RowBlock{0, op->m, 0, 0}, s);
}

int kb_apply_adjoint(const kb_op* op, const void* Y, void* X, void* work, void* stream) {
  KB_TRY(check_op(op));
  Work w = layout(op, work);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (op->dtype == KB_F64)
    return apply_t<double>(op, 1, static_cast<const double*>(Y), static_cast<double*>(X), w, RowBlock{0, op->m, 0, 0}, s);
  return apply_t<float>(op, 1, static_cast<const float*>(Y), static_cast<float*>(X), w, RowBlock{0, op->m, 0, 0}, s);
}

int kb_apply_block(const kb_op* op, int adjoint, const void* X, void* Y, void* work, int g0,
                   int m_global, int halo_lo, int halo_hi, void* stream) {
  KB_TRY(check_op(op));
  if (g0 < 0 || g0 + op->m > m_global || halo_lo < 0 || halo_hi < 0)
    return fail(KB_ERR_ARGUMENT, "bad row block");
  Work w = layout(op, work);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (op->dtype == KB_F64)
    return apply_t<double>(op, adjoint, static_cast<const double*>(X), static_cast<double*>(Y), w, RowBlock{g0, m_global, halo_lo, halo_hi}, s);
  return apply_t<float>(op, adjoint, static_cast<const float*>(X), static_cast<float*>(Y), w, RowBlock{g0, m_global, halo_lo, halo_hi}, s);
}

int kb_block_residual(const kb_op* op, const void* Yh, const void* B, void* R, void* work,
                      int g0, int m_global, int halo_lo, int halo_hi, void* stream) {
  KB_TRY(check_op(op));
  if (g0 < 0 || g0 + op->m > m_global || halo_lo < 0 || halo_hi < 0)
    return fail(KB_ERR_ARGUMENT, "bad row block");
  Work w = layout(op, work);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (op->dtype == KB_F64)
    return residual_t<double>(op, static_cast<const double*>(Yh), static_cast<const double*>(B), static_cast<double*>(R), w, RowBlock{g0, m_global, halo_lo, halo_hi}, s);
  return residual_t<float>(op, static_cast<const float*>(Yh), static_cast<const float*>(B), static_cast<float*>(R), w, RowBlock{g0, m_global, halo_lo, halo_hi}, s);
}

int kb_block_update(const kb_op* op, const void* Rh, void* X, void* Y, void* work, int g0,
                    int m_global, int halo_lo, int halo_hi, double beta, int k, double L,
                    double lam, int project, int* nonfinite, double* norms, void* stream) {
  KB_TRY(check_op(op));
  if (op->batch != 1) return fail(KB_ERR_ARGUMENT, "row-block update needs batch == 1");
  if (g0 < 0 || g0 + op->m > m_global || halo_lo < 0 || halo_hi < 0)
    return fail(KB_ERR_ARGUMENT, "bad row block");
  Work w = layout(op, work);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const double host[2] = {L, L + lam * lam};
  KB_CUDA(cudaMemcpyAsync(w.scal, host, sizeof(host), cudaMemcpyHostToDevice, s));
  if (op->dtype == KB_F64)
    return update_t<double>(op, static_cast<const double*>(Rh), static_cast<double*>(X), static_cast<double*>(Y), w, RowBlock{g0, m_global, halo_lo, halo_hi}, beta, k, w.scal, w.scal + 1, project, nonfinite, norms, s);
  return update_t<float>(op, static_cast<const float*>(Rh), static_cast<float*>(X), static_cast<float*>(Y), w, RowBlock{g0, m_global, halo_lo, halo_hi}, beta, k, w.scal, w.scal + 1, project, nonfinite, norms, s);
}

namespace {
int sfista_run_impl(const kb_op* op, const void* B, void* X, void* Y, void* work, const double* beta, int k0,
                    int iters, const double* L, const double* lam, int lam_per_image, int project,
                    int* nonfinite, double* norms, int use_graph, void* stream);
}  // namespace

int kb_sfista_run(const kb_op* op, const void* B, void* X, void* Y, void* work,
                  const double* beta, int k0, int iters, const double* L, double lam,
                  int project, int* nonfinite, double* norms, int use_graph, void* stream) {
  return sfista_run_impl(op, B, X, Y, work, beta, k0, iters, L, &lam, 0, project, nonfinite, norms, use_graph,
                         stream);
}

int kb_sfista_run_lams(const kb_op* op, const void* B, void* X, void* Y, void* work,
                       const double* beta, int k0, int iters, const double* L, const double* lam,
                       int project, int* nonfinite, double* norms, int use_graph, void* stream) {
  if (!lam) return fail(KB_ERR_ARGUMENT, "null argument");
  return sfista_run_impl(op, B, X, Y, work, beta, k0, iters, L, lam, 1, project, nonfinite, norms, use_graph,
                         stream);
}
}  // extern "C"

namespace {
// Whole-solve persistent kernel (kb_persist.cuh) for small fp64 single images: one cooperative
// launch runs every iteration with two grid barriers each. KB_PERSIST=0 disables it, =1 uses it
// whenever it fits; by default it takes images up to 512^2 (cfg1: launch-bound otherwise).
struct PsPlan {
  int RB = 0, nblk = 0;
  size_t smem = 0;
  int v2 = 0;  // kb_solve_persistent2 (zero BC, narrow bands) instead of kb_solve_persistent
  bool breg = false;  // v2: the register-resident-B-fragment instantiation (one CTA per SM)
};

using Ps2Kernel = void (*)(kb::P2Args);
template <int R>
Ps2Kernel ps2_kernel_r(int RB, bool breg) {
  if (breg) return RB == 1 ? kb::kb_solve_persistent2<R, 1, true> : kb::kb_solve_persistent2<R, 2, true>;
  return RB == 1 ? kb::kb_solve_persistent2<R, 1, false> : kb::kb_solve_persistent2<R, 2, false>;
}
Ps2Kernel ps2_kernel(int r, int RB, bool breg) {
  switch (r) {
    case 1: return ps2_kernel_r<1>(RB, breg);
    case 2: return ps2_kernel_r<2>(RB, breg);
    case 3: return ps2_kernel_r<3>(RB, breg);
    default: return ps2_kernel_r<4>(RB, breg);
  }
}
#ifndef KB_P2_SYNC_DEFAULT
#define KB_P2_SYNC_DEFAULT 0  // KB_PERSIST2_SYNC unset: 0 grid.sync, 1 neighbour flags, 2 arrival counter
#endif
// The second whole-solve form (kb_persist2.cuh): zero BC on both axes, half widths <= 15,
// r <= 4, n a multiple of 64 up to 512. KB_PERSIST2=0 keeps the first form; KB_PERSIST_RB picks
// the rows per CTA (1 or 2).
PsPlan persist2_plan(const kb_op* op) {
  PsPlan p;
  const char* v = std::getenv("KB_PERSIST2");
  if (v && v[0] == '0') return p;
  if (op->bc_a != KB_BC_ZERO || op->bc_b != KB_BC_ZERO || op->Ha > kb::kP2H || op->Hb > kb::kP2H ||
      op->r > kb::kP2MaxR || op->n % 64 || op->n > 512 || op->h_conv[0].empty() || op->h_conv[1].empty())
    return p;
  const char* rbv = std::getenv("KB_PERSIST_RB");
  const int want = rbv ? std::atoi(rbv) : 0;
  const int sms = sm_count();
  // two rows per CTA before one; the register-resident-B instantiation (one CTA per SM) when the
  // CTAs fit that way, else the lean one (two per SM)
  for (int RB = want == 1 || want == 2 ? want : 2; RB >= 1; --RB) {
    for (int breg = 1; breg >= 0; --breg) {
      const Ps2Kernel k = ps2_kernel(op->r, RB, breg != 0);
      const size_t smem = kb::p2_smem_bytes(RB, op->n, op->r);
      int per_sm = 0;
      if (smem <= 200 * 1024 && allow_smem(k, smem) == KB_OK &&
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, kb::kP2Threads, smem) == cudaSuccess &&
          per_sm >= 1 && (op->m + RB - 1) / RB <= per_sm * sms) {
        p.RB = RB;
        p.nblk = (op->m + RB - 1) / RB;
        p.smem = smem;
        p.v2 = 1;
        p.breg = breg != 0;
        return p;
      }
    }
    if (want == 1 || want == 2) break;
  }
  return p;
}
PsPlan persist_plan(const kb_op* op) {
  PsPlan p;
  static const int mode = [] {
    const char* v = std::getenv("KB_PERSIST");
    return v ? std::atoi(v) : -1;
  }();
  if (mode == 0 || op->dtype != KB_F64 || op->batch != 1 || op->n % 2) return p;
  if (mode < 0 && (long long)op->m * op->n > 512LL * 512) return p;
  {
    const PsPlan p2 = persist2_plan(op);
    if (p2.v2) return p2;
  }
  const int sms = sm_count();
  static const int rb_env = [] {
    const char* v = std::getenv("KB_PERSIST_RB");
    return v ? std::atoi(v) : 0;
  }();
  // one row per CTA when the rows fit co-resident (measured fastest at cfg1: 3.5k vs 3.1k Mpix*it/s
  // with two rows), else the fewest rows per CTA that do
  int RB = rb_env > 0 ? rb_env : 1;
  size_t smem = kb::ps_smem_bytes(RB, op->Ha, op->Hb, op->n, op->r);
  if (rb_env <= 0) {
    while (RB < op->m) {
      int ps = 0;
      smem = kb::ps_smem_bytes(RB, op->Ha, op->Hb, op->n, op->r);
      if (smem <= 200 * 1024 && allow_smem(kb::kb_solve_persistent, smem) == KB_OK &&
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, kb::kb_solve_persistent, kb::kPsThreads, smem) ==
              cudaSuccess &&
          ps >= 1 && (op->m + RB - 1) / RB <= ps * sms)
        break;
      ++RB;
    }
    smem = kb::ps_smem_bytes(RB, op->Ha, op->Hb, op->n, op->r);
  }
  if (smem > 200 * 1024) return p;
  if (allow_smem(kb::kb_solve_persistent, smem) != KB_OK) return p;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kb::kb_solve_persistent, kb::kPsThreads, smem) !=
          cudaSuccess ||
      per_sm < 1)
    return p;
  p.RB = RB;
  p.nblk = (op->m + RB - 1) / RB;
  if (p.nblk > per_sm * sms) return PsPlan{};  // a cooperative launch must be co-resident
  p.smem = smem;
  return p;
}

int launch_persist(const kb_op* op, const PsPlan& pp, const double* B, double* X, double* Y, const Work& w,
                   const double* beta, int k0, int iters, double L, double lam, int project, int* nonfinite,
                   cudaStream_t s) {
  // beta_k go to the (unused on this path) norm-partials region of the workspace
  // beta (doubles) then the CTAs' phase flags (ints) in the partials region
  // grid-wide barriers by default: measured faster than the neighbour-flag waits at cfg1
  // (3.65k vs 2.70k Mpix*it/s, tools/cfg1_ab.sh); KB_PERSIST_SYNC=flags selects the latter
  static const bool grid_sync = [] {
    const char* v = std::getenv("KB_PERSIST_SYNC");
    return !(v && std::string(v) == "flags");
  }();
  const int cap = (int)partials_doubles(op) - (pp.nblk + 1) / 2 - 2;
  if (cap < 1) return fail(KB_ERR_ARGUMENT, "workspace too small for the persistent solve");
  int* flags = reinterpret_cast<int*>(w.partials + cap + 1);
  if (pp.v2) {
    kb::P2Args a{};
    a.B = B;
    a.X = X;
    a.Y = Y;
    a.R = static_cast<double*>(w.rp);
    a.beta = w.partials;
    a.nonfinite = nonfinite;
    a.L = L;
    a.denom = L + lam * lam;
    a.m = op->m;
    a.n = op->n;
    a.project = project;
    // KB_PERSIST2_SYNC=grid|flags|counter: cooperative-groups barrier, neighbour phase epochs, or one
    // release/acquire arrival counter: the
    // flags, one 128-byte line per CTA, sit behind the beta table in the partials region
    const int p2_sync = [] {  // read per launch (the tests switch it)
      const char* v = std::getenv("KB_PERSIST2_SYNC");
      const std::string m = v ? v : "";
      return m == "flags" ? 1 : m == "counter" ? 2 : m == "grid" ? 0 : KB_P2_SYNC_DEFAULT;
    }();
    const int fdoubles = (pp.nblk * kb::kP2FlagStride + 1) / 2 + 16;
    const int cap2 = (int)partials_doubles(op) - fdoubles - 2;
    const bool use_flags = p2_sync != 0 && cap2 >= 1;
    const int capv = use_flags ? cap2 : cap;
    a.sync_mode = use_flags ? p2_sync : 0;
    if (use_flags)  // 128-byte aligned
      a.flags = reinterpret_cast<int*>((reinterpret_cast<uintptr_t>(w.partials + capv + 1) + 127) & ~(uintptr_t)127);
    // centred 31-tap windows: window tap k' <-> table tap k' - 15 + H
    auto centre = [&](const std::vector<double>& tab, int H, int Wp, double (*dst)[kb::kP2W]) {
      for (int i = 0; i < op->r; ++i)
        for (int k = 0; k < kb::kP2W; ++k) {
          const int t = k - kb::kP2H + H;
          dst[i][k] = (t >= 0 && t <= 2 * H) ? tab[(size_t)i * Wp + t] : 0.0;
        }
    };
    centre(op->h_conv[0], op->Ha, op->Wpa, a.fa);
    centre(op->h_corr[0], op->Ha, op->Wpa, a.aa);
    centre(op->h_conv[1], op->Hb, op->Wpb, a.fb);
    centre(op->h_corr[1], op->Hb, op->Wpb, a.ab);
    const Ps2Kernel kern = ps2_kernel(op->r, pp.RB, pp.breg);
#ifdef KB_P2_TRACE
    static long long* trace_d = nullptr;
    if (!trace_d) cudaMalloc(&trace_d, 16 * 1024 * sizeof(long long));
    cudaMemsetAsync(trace_d, 0, 16 * 1024 * sizeof(long long), s);
    a.trace = trace_d;
#endif
    for (int done = 0; done < iters;) {
      const int cnt = std::min(iters - done, capv);
      KB_CUDA(cudaMemcpyAsync(w.partials, beta + k0 + done, sizeof(double) * cnt, cudaMemcpyHostToDevice, s));
      if (a.flags) KB_CUDA(cudaMemsetAsync(a.flags, 0, sizeof(int) * pp.nblk * kb::kP2FlagStride, s));
      a.k0 = k0 + done;
      a.iters = cnt;
      void* args[] = {&a};
      KB_CUDA(cudaLaunchCooperativeKernel((const void*)kern, dim3(pp.nblk), dim3(kb::kP2Threads), args, pp.smem, s));
      done += cnt;
    }
#ifdef KB_P2_TRACE
    if (std::getenv("KB_P2_TRACE")) {
      std::vector<long long> h(16 * 1024);
      cudaStreamSynchronize(s);
      cudaMemcpy(h.data(), trace_d, h.size() * sizeof(long long), cudaMemcpyDeviceToHost);
      static const char* names[] = {"p1 start", "p1 waited", "p1 staged(issued)", "p1 axis0", "p1 sync", "p1 axis1+store",
                                    "p1 phase_end", "p2 waited", "p2 staged(issued)", "p2 axis0", "p2 sync",
                                    "p2 axis1+update", "p2 phase_end"};
      // per segment: min / mean / max over the CTAs (cycles of each CTA's own SM clock)
      const int nb = std::min(pp.nblk, 1024);
      std::fprintf(stderr, "[p2 trace] %d CTAs, min/mean/max cycles per segment:", nb);
      for (int i = 1; i < 13; ++i) {
        long long lo = LLONG_MAX, hi = 0, sum = 0;
        for (int b = 0; b < nb; ++b) {
          const long long d = h[16 * b + i] - h[16 * b + i - 1];
          lo = std::min(lo, d);
          hi = std::max(hi, d);
          sum += d;
        }
        std::fprintf(stderr, " %s %lld/%lld/%lld;", names[i], lo, sum / nb, hi);
      }
      long long tl = LLONG_MAX, th = 0;
      for (int b = 0; b < nb; ++b) {
        tl = std::min(tl, h[16 * b + 12] - h[16 * b]);
        th = std::max(th, h[16 * b + 12] - h[16 * b]);
      }
      std::fprintf(stderr, " total %lld..%lld\n", tl, th);
    }
#endif
    for (int i = 0; i < 4; ++i) w.ctx.phase[i] = KB_ENGINE_PERSIST_F64;
    return KB_OK;
  }
  for (int done = 0; done < iters;) {
    const int cnt = std::min(iters - done, cap);
    KB_CUDA(cudaMemcpyAsync(w.partials, beta + k0 + done, sizeof(double) * cnt, cudaMemcpyHostToDevice, s));
    if (!grid_sync) KB_CUDA(cudaMemsetAsync(flags, 0, sizeof(int) * pp.nblk, s));
    kb::PsArgs a;
    a.B = B;
    a.X = X;
    a.Y = Y;
    a.R = static_cast<double*>(w.rp);
    a.ha = static_cast<const double*>(op->ta_conv);
    a.kbt = static_cast<const double*>(op->tb_conv);
    a.beta = w.partials;
    a.nonfinite = nonfinite;
    a.L = L;
    a.denom = L + lam * lam;
    a.m = op->m;
    a.n = op->n;
    a.r = op->r;
    a.Ha = op->Ha;
    a.Hb = op->Hb;
    a.Wpa = op->Wpa;
    a.Wpb = op->Wpb;
    a.refl_a = op->bc_a == KB_BC_REFLECTIVE;
    a.refl_b = op->bc_b == KB_BC_REFLECTIVE;
    a.RB = pp.RB;
    a.k0 = k0 + done;
    a.iters = cnt;
    a.project = project;
    a.flags = grid_sync ? nullptr : flags;
    void* args[] = {&a};
    KB_CUDA(cudaLaunchCooperativeKernel((const void*)kb::kb_solve_persistent, dim3(pp.nblk), dim3(kb::kPsThreads),
                                        args, pp.smem, s));
    done += cnt;
  }
  for (int i = 0; i < 4; ++i) w.ctx.phase[i] = KB_ENGINE_PERSIST_F64;
  return KB_OK;
}

int sfista_run_impl(const kb_op* op, const void* B, void* X, void* Y, void* work, const double* beta, int k0,
                    int iters, const double* L, const double* lam, int lam_per_image, int project,
                    int* nonfinite, double* norms, int use_graph, void* stream) {
  KB_TRY(check_op(op));
  if (!B || !X || !Y || !work || !beta || !L || !nonfinite) return fail(KB_ERR_ARGUMENT, "null argument");
  if (iters < 0 || k0 < 0) return fail(KB_ERR_ARGUMENT, "iters and k0 must be >= 0");
  if (iters == 0) return KB_OK;
  // fast path with an axis-swapped twin: the launches run the twin on transposed planes
  const kb_op* run = (op->twin && !norms && op->batch == 1) ? op->twin : op;
  Work w = layout(run, work);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<double> host(2 * (size_t)op->batch);
  for (int b = 0; b < op->batch; ++b) {
    const double lb = lam[lam_per_image ? b : 0];
    host[b] = L[b];
    host[op->batch + b] = L[b] + lb * lb;
  }
  KB_CUDA(cudaMemcpyAsync(w.scal, host.data(), host.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  // cudaMemcpyAsync from pageable memory returns after staging, so `host` may go out of scope.
  auto body = [&](cudaStream_t cs) -> int {
    if (op->dtype == KB_F64)
      return sfista_launches<double>(op, static_cast<const double*>(B), static_cast<double*>(X),
                                     static_cast<double*>(Y), w, beta, k0, iters, project, nonfinite, norms, cs);
    if (run != op) {  // solve the transposed problem: B^T, X^T, Y^T in, X, Y back
      float* Bt = static_cast<float*>(twin_plane(op, work, 0));
      float* Xt = static_cast<float*>(twin_plane(op, work, 1));
      float* Yt = static_cast<float*>(twin_plane(op, work, 2));
      KB_TRY(transpose_t<float>(static_cast<const float*>(B), Bt, op->m, op->n, cs));
      KB_TRY(transpose_t<float>(static_cast<const float*>(X), Xt, op->m, op->n, cs));
      KB_TRY(transpose_t<float>(static_cast<const float*>(Y), Yt, op->m, op->n, cs));
      KB_TRY(sfista_launches<float>(run, Bt, Xt, Yt, w, beta, k0, iters, project, nonfinite, nullptr, cs));
      KB_TRY(transpose_t<float>(Xt, static_cast<float*>(X), op->n, op->m, cs));
      return transpose_t<float>(Yt, static_cast<float*>(Y), op->n, op->m, cs);
    }
    return sfista_launches<float>(op, static_cast<const float*>(B), static_cast<float*>(X),
                                  static_cast<float*>(Y), w, beta, k0, iters, project, nonfinite, norms, cs);
  };
  auto publish = [&](const int* eng) {
    std::lock_guard<std::mutex> lock(g_phase_mu);
    for (int i = 0; i < 4; ++i)
      if (eng[i] >= 0) op->phase_engine[i] = eng[i];
  };
  if (!norms && al16(B) && al16(X) && al16(Y) && al16(w.rp)) {
    const PsPlan pp = persist_plan(op);
    if (pp.nblk > 0) {  // one launch for the whole solve: no graph needed
      const int rc = launch_persist(op, pp, static_cast<const double*>(B), static_cast<double*>(X),
                                    static_cast<double*>(Y), w, beta, k0, iters, L[0], lam[0], project, nonfinite, s);
      if (rc == KB_OK) publish(w.ctx.phase);
      return rc;
    }
  }
  if (!use_graph) {
    const int rc = body(s);
    if (rc == KB_OK) publish(w.ctx.phase);
    return rc;
  }

  // graph path: key = every pointer and scalar the captured launches bake in
  std::vector<unsigned char> key;
  auto put = [&](const void* p, size_t nb) {
    const unsigned char* c = static_cast<const unsigned char*>(p);
    key.insert(key.end(), c, c + nb);
  };
  put(&B, sizeof(B)); put(&X, sizeof(X)); put(&Y, sizeof(Y)); put(&work, sizeof(work));
  put(&k0, sizeof(k0)); put(&iters, sizeof(iters)); put(&project, sizeof(project));
  put(&nonfinite, sizeof(nonfinite)); put(&norms, sizeof(norms));
  put(beta + k0, sizeof(double) * iters);
  GraphCache* gc = op->graph;
  std::lock_guard<std::mutex> lock(gc->mu);
  if (!gc->exec || gc->key != key) {
    if (gc->exec) {
      cudaGraphExecDestroy(gc->exec);
      gc->exec = nullptr;
    }
    cudaStream_t cs;
    KB_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    cudaGraph_t graph;
    cudaError_t ce = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
    if (ce != cudaSuccess) {
      cudaStreamDestroy(cs);
      return fail(KB_ERR_CUDA, std::string("begin capture: ") + cudaGetErrorString(ce));
    }
    const int rc = body(cs);
    ce = cudaStreamEndCapture(cs, &graph);
    cudaStreamDestroy(cs);
    if (rc != KB_OK) {
      if (ce == cudaSuccess) cudaGraphDestroy(graph);
      return rc;
    }
    if (ce != cudaSuccess) return fail(KB_ERR_CUDA, std::string("end capture: ") + cudaGetErrorString(ce));
    ce = cudaGraphInstantiate(&gc->exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ce != cudaSuccess) {
      gc->exec = nullptr;
      return fail(KB_ERR_CUDA, std::string("instantiate: ") + cudaGetErrorString(ce));
    }
    gc->key = key;
    for (int i = 0; i < 4; ++i) gc->engines[i] = w.ctx.phase[i];
  }
  KB_CUDA(cudaGraphLaunch(gc->exec, s));
  publish(gc->engines);
  return KB_OK;
}
}  // namespace

extern "C" {

int kb_power_iter(const kb_op* op, void* v, void* wb, void* work, int iters, double* hist,
                  void* stream) {
  KB_TRY(check_op(op));
  if (!v || !wb || !work || !hist || iters < 1) return fail(KB_ERR_ARGUMENT, "bad power-iteration arguments");
  Work w = layout(op, work);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (op->dtype == KB_F64)
    return power_t<double>(op, static_cast<double*>(v), static_cast<double*>(wb), w, iters, hist, s);
  return power_t<float>(op, static_cast<float*>(v), static_cast<float*>(wb), w, iters, hist, s);
}

int kb_blur_direct(const double* psf, long long psf_batch_stride, int rows, int cols, int l, int q,
                   const double* X, double* Y, int m, int n, int batch, int bc, void* stream) {
  if (!psf || !X || !Y) return fail(KB_ERR_ARGUMENT, "null pointer");
  if (m < 1 || n < 1 || batch < 1) return fail(KB_ERR_ARGUMENT, "invalid image shape");
  if (rows < 1 || cols < 1) return fail(KB_ERR_ARGUMENT, "PSF must be a nonempty 2-D array");
  if (rows > m || cols > n)
    return fail(KB_ERR_ARGUMENT, "PSF of shape (" + std::to_string(rows) + ", " + std::to_string(cols) +
                                     ") larger than image (" + std::to_string(m) + ", " + std::to_string(n) + ")");
  // (l, q) may lie outside a PSF whose all-zero borders the caller cropped (blur.py); the
  // extension stays a single fold as long as the uncropped PSF fits the image
  if (l < 1 - m || l > rows + m || q < 1 - n || q > cols + n) return fail(KB_ERR_ARGUMENT, "PSF center too far outside the array");
  if (bc != KB_BC_ZERO && bc != KB_BC_REFLECTIVE) return fail(KB_ERR_ARGUMENT, "unknown boundary condition");
  if (psf_batch_stride < 0) return fail(KB_ERR_ARGUMENT, "negative PSF batch stride");
  const size_t img = (size_t)m * n * sizeof(double) * batch;
  const char* xb = reinterpret_cast<const char*>(X);
  const char* yb = reinterpret_cast<const char*>(Y);
  if (xb < yb + img && yb < xb + img) return fail(KB_ERR_ARGUMENT, "X and Y overlap");
  const size_t smem = kb::kb_blur_smem(cols);
  KB_TRY(allow_smem(kb::kb_blur_direct_k, smem));
  dim3 grid((n + kb::kBlTW - 1) / kb::kBlTW, (m + kb::kBlTH - 1) / kb::kBlTH, batch);
  kb::kb_blur_direct_k<<<grid, kb::kBlThreads, smem, static_cast<cudaStream_t>(stream)>>>(
      psf, psf_batch_stride, rows, cols, l, q, X, Y, m, n, bc == KB_BC_REFLECTIVE);
  KB_CUDA(cudaGetLastError());
  return KB_OK;
}

int kb_resid_norms(int dtype, const void* AX, const void* B, const void* X, const void* truth,
                   long long count, double* out2, void* work, void* stream) {
  if (!AX || !B || !out2 || !work || (truth && !X) || count < 0)
    return fail(KB_ERR_ARGUMENT, "bad kb_resid_norms arguments");
  if (dtype != KB_F64 && dtype != KB_F32) return fail(KB_ERR_ARGUMENT, "unknown dtype");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double* partial = static_cast<double*>(work);
  if (dtype == KB_F64)
    kb::kb_resid_norms_k<double><<<kb::kNormBlocks, kb::kNormThreads, 0, s>>>(
        static_cast<const double*>(AX), static_cast<const double*>(B), static_cast<const double*>(X),
        static_cast<const double*>(truth), count, partial);
  else
    kb::kb_resid_norms_k<float><<<kb::kNormBlocks, kb::kNormThreads, 0, s>>>(
        static_cast<const float*>(AX), static_cast<const float*>(B), static_cast<const float*>(X),
        static_cast<const float*>(truth), count, partial);
  kb::kb_resid_norms_finish<<<1, 32, 0, s>>>(partial, kb::kNormBlocks, out2);
  KB_CUDA(cudaGetLastError());
  return KB_OK;
}

int kb_inner2(int dtype, const void* a, const void* b, long long count, double* out2, void* work,
              void* stream) {
  if (!a || !b || !out2 || !work || count < 0) return fail(KB_ERR_ARGUMENT, "bad kb_inner2 arguments");
  if (dtype != KB_F64 && dtype != KB_F32) return fail(KB_ERR_ARGUMENT, "unknown dtype");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double* partial = static_cast<double*>(work);
  if (dtype == KB_F64)
    kb::kb_inner2_k<double><<<kb::kNormBlocks, kb::kNormThreads, 0, s>>>(
        static_cast<const double*>(a), static_cast<const double*>(b), count, partial);
  else
    kb::kb_inner2_k<float><<<kb::kNormBlocks, kb::kNormThreads, 0, s>>>(
        static_cast<const float*>(a), static_cast<const float*>(b), count, partial);
  kb::kb_resid_norms_finish<<<1, 32, 0, s>>>(partial, kb::kNormBlocks, out2);
  KB_CUDA(cudaGetLastError());
  return KB_OK;
}

int kb_fma_peak(int dtype, float* tflops, void* stream) {
  if (!tflops) return fail(KB_ERR_ARGUMENT, "null output");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (dtype == KB_PEAK_TC_TF32) return tc_peak(tflops, s);
  return dtype == KB_F64 ? fma_peak_t<double>(tflops, s) : fma_peak_t<float>(tflops, s);
}

int kb_last_engines(const kb_op* op, int* engines4) {
  KB_TRY(check_op(op));
  if (!engines4) return fail(KB_ERR_ARGUMENT, "null output");
  std::lock_guard<std::mutex> lock(g_phase_mu);
  for (int i = 0; i < 4; ++i) engines4[i] = op->phase_engine[i];
  return KB_OK;
}

int kb_debug_trace(unsigned long long* host, int n) {
  if (!host || n < 0) return fail(KB_ERR_ARGUMENT, "bad kb_debug_trace arguments");
  const size_t all = sizeof(kb::kb_trace);
  KB_CUDA(cudaMemcpyFromSymbol(host, kb::kb_trace, std::min(all, (size_t)n * sizeof(unsigned long long))));
  return KB_OK;
}

int kb_time_passes(const kb_op* op, const void* Y, const void* B, void* R, void* X, void* Yio,
                   void* work, int reps, const double* L, double lam, int* nonfinite,
                   float* ms4, void* stream) {
  KB_TRY(check_op(op));
  if (!Y || !B || !R || !X || !Yio || !work || !L || !nonfinite || !ms4 || reps < 1)
    return fail(KB_ERR_ARGUMENT, "bad kb_time_passes arguments");
  // with an axis-swapped twin the fast path runs the twin's kernels: time those (the planes are
  // only buffers here, of the same element count)
  const kb_op* top = op->twin ? op->twin : op;
  Work w = layout(top, work);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  std::vector<double> host(2 * (size_t)op->batch);
  for (int b = 0; b < op->batch; ++b) {
    host[b] = L[b];
    host[op->batch + b] = L[b] + lam * lam;
  }
  KB_CUDA(cudaMemcpyAsync(w.scal, host.data(), host.size() * sizeof(double), cudaMemcpyHostToDevice, s));
  if (op->twin) {
    const int rc = time_passes_t<float>(top, static_cast<const float*>(Y), static_cast<const float*>(B),
                                        static_cast<float*>(R), static_cast<float*>(X), static_cast<float*>(Yio), w,
                                        reps, ms4, nonfinite, s);
    std::lock_guard<std::mutex> lock(g_phase_mu);
    for (int i = 0; i < 4; ++i) op->phase_engine[i] = top->phase_engine[i];
    return rc;
  }
  if (op->dtype == KB_F64)
    return time_passes_t<double>(op, static_cast<const double*>(Y), static_cast<const double*>(B), static_cast<double*>(R), static_cast<double*>(X), static_cast<double*>(Yio), w, reps, ms4, nonfinite, s);
  return time_passes_t<float>(op, static_cast<const float*>(Y), static_cast<const float*>(B), static_cast<float*>(R), static_cast<float*>(X), static_cast<float*>(Yio), w, reps, ms4, nonfinite, s);
}

}  // extern "C"
