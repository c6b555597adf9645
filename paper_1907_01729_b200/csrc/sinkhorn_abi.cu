// sinkhorn_abi.cu -- host runtime + C ABI of the B200 Sinkhorn loss.
//
// The iteration loop (batch.py:314-324) runs here in C++: it enqueues the
// half-sweep kernels on the caller's stream with programmatic dependent
// launch, keeps every intermediate in the caller-provided workspace, and only
// synchronises when the reference's semantics need a host decision (the
// convergence test every check_interval iterations when tolerance > 0) and once
// at the end to report the status word.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>
#include <cstdlib>

#include "../../include/sinkhorn_b200.h"
#include "aux_kernels.cuh"
#include "common.cuh"
#include "sweep_lane.cuh"
#include "sweep_tiled.cuh"
#include "persistent.cuh"
#include "sweep_small.cuh"
#include "sweep_sep.cuh"
#include "sweep_fused.cuh"
#include "sweep_f64.cuh"
#include "sweep_gemm.cuh"
#include "sweep_umma.cuh"

using namespace skb;

namespace {

thread_local std::string g_last_error;
thread_local unsigned long long g_launches = 0;   // kernels this thread launched
thread_local float g_last_loop_ms = -1.f;         // last timed iteration loop (ms)
// SINKHORN_FLAG_TIME_KERNEL: CUDA events around every launch of the solve's
// dominant kernel (the per-iteration sweep / contraction), for the roofline.
struct KernelTimer {
  bool on = false;
  std::vector<cudaEvent_t> ev;   // begin / end pairs
  float last_ms = -1.f;
  int last_launches = 0;
};
thread_local KernelTimer g_kt;
inline void kt_mark(cudaStream_t st) {
  if (!g_kt.on) return;
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) == cudaSuccess) {
    cudaEventRecord(e, st);
    g_kt.ev.push_back(e);
  }
}
thread_local const char* g_last_path = "none";    // solver path of the last forward
thread_local unsigned long long g_exact_reruns = 0;  // solves redone without estimates
// non-check fused iterations of shared costs as the two-GEMM block pass
// (SKB_FUSED_ROWS=1: the warp-per-row linear pass instead; diagnostics / A-B)
const bool g_use_fgemm = getenv("SKB_FUSED_ROWS") == nullptr;
// Optional cross-rank agreement on the stopping test (batch-sharded solves).
thread_local sinkhorn_residual_reducer_v1 g_reducer = nullptr;
thread_local void* g_reducer_user = nullptr;
// Row-sharded GEMM solves (sinkhorn_forward_rows_device_v1): the caller's
// collective, enqueued on the solve's stream after every partial column
// contraction (T = K_r^T a, summed over the ranks) and after the E0 partials.
thread_local sinkhorn_allreduce_v1 g_allreduce = nullptr;
thread_local void* g_allreduce_user = nullptr;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define CK(expr)                                                                           \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess)                                                                 \
      return fail(SINKHORN_STATUS_CUDA_ERROR,                                              \
                  std::string(#expr) + ": " + cudaGetErrorString(_e));                     \
  } while (0)

// ---- tiled-sweep configuration ---------------------------------------------
constexpr int QC = 32, RB = 4, RP = 4, NSTAGE = 4;
constexpr int PT_MAX = 64;    // output-tile widths: 64 or 56 (picked per sweep, see pick_pt)
constexpr int TILE_PAD = 64;  // buffer extents padded to 64 (>= every tile / TMA box)
constexpr int MAX_OCC = SKB_OCC_SMALL > 2 ? SKB_OCC_SMALL : 2;
constexpr int kEstFromIter = 3;   // first iteration whose sweeps start from the previous lse

template <int BT, int PT, bool kGrid, int kMode>
struct TiledK {
  using S = TiledSweep<BT, PT, QC, RB, RP, NSTAGE, kGrid, kMode>;
  static void* fn() {
    return reinterpret_cast<void*>(&tiled_sweep_kernel<BT, PT, QC, RB, RP, NSTAGE, kGrid, kMode>);
  }
};

// Lane tile: 128 lanes (one 16-warp CTA per SM: no inter-CTA warp-priority
// skew, half as many stream-K pieces per tile) whenever the batch has > 64 lanes.
#ifndef SKB_BT_BIG
#define SKB_BT_BIG 128
#endif
int pick_bt(int64_t B) { return B > 64 ? SKB_BT_BIG : 64; }

// Output-tile width.  Always 64 (8 warps: an even 4 warps per scheduler at 2
// CTAs/SM; 7-warp tiles left the 4 SMSPs 4/4/3/3).  A ragged extent is covered
// by shifting the last tile left (it overlaps its neighbour) so no tile is partial.
int pick_pt(int /*P*/) { return 64; }

struct DeviceInfo {
  int dev = -1;
  int sms = 148;
};

DeviceInfo device_info() {
  static thread_local int cached_dev = -1, cached_sms = 0;
  DeviceInfo di;
  cudaGetDevice(&di.dev);
  if (di.dev != cached_dev) {
    cudaDeviceGetAttribute(&cached_sms, cudaDevAttrMultiProcessorCount, di.dev);
    cached_dev = di.dev;
  }
  di.sms = cached_sms;
  return di;
}

size_t round_up(size_t x, size_t m) { return (x + m - 1) / m * m; }

inline float neg_inf_host() { return -INFINITY; }

// ---- TMA descriptor encoding through the driver entry point ----------------
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D fp32 row-major [rows][cols] tensor, box {box_cols, box_rows}.
bool make_tmap(CUtensorMap* m, const float* base, size_t rows, size_t cols, int box_rows,
               int box_cols) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {cols * sizeof(float)};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// Operand map of the tensor-core contractions: [rows][cols] fp32 with row pitch
// `pitch` elements, box 32 (one 128-byte swizzle row) x box_rows, SWIZZLE_128B;
// elements past `cols` / `rows` read as 0.
bool make_tmap_sw128(CUtensorMap* m, const float* base, size_t rows, size_t cols, size_t pitch,
                     int box_rows) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {pitch * sizeof(float)};
  cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// ---- launch helpers ----------------------------------------------------------
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ++g_launches;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

int grid_for(size_t n) { return (int)std::min<size_t>((n + 255) / 256, 148 * 16); }
// Kernels with one grid row per lane (grid.y = lane) launch at most this many
// lanes at a time (the grid.y limit), with the first lane in their params.
constexpr long long kMaxLanesPerLaunch = 65535;
unsigned lanes_in_launch(long long B, long long b0) {
  return (unsigned)std::min<long long>(kMaxLanesPerLaunch, B - b0);
}

// ---- workspace layout --------------------------------------------------------
struct Carver {
  size_t off = 0;
  size_t take(size_t bytes) {
    size_t o = off;
    off = round_up(off + bytes, 256);
    return o;
  }
};

struct Layout {
  bool tiled = true;
  bool sep = false;               // grid cost, separable sweeps (lane-major buffers)
  int64_t B = 0, d1 = 0, d2 = 0;
  int Bp = 0, D1p = 0, D2p = 0;   // padded extents (tiled) / leading dims (lane)
  long long sb1 = 0, si1 = 0, sb2 = 0, si2 = 0;  // element (b,i) at b*sb + i*si
  size_t a2 = 0, a2t = 0, f2 = 0, g2[2] = {0, 0}, l2mu = 0, l2nu = 0, mu = 0, nu = 0, e0 = 0;
  size_t res = 0, scratch = 0, part = 0, counters = 0, status = 0, badrow = 0, total = 0;
  size_t kmat = 0;                // fused: K = 2^A2 [D1p][D2p]
  size_t sep_ax = 0, sep_ay = 0;   // separable grid: Ax [nx][nblk*32], Ay [ny][sep_ld(ny)]
  bool sep_split = false;          // large grids: the two-kernel separable sweep
  size_t sep_tg = 0, sep_rg = 0;   // its T (and tail R) [B][nblk][ny][32]
  size_t f2T = 0, g2T[2] = {0, 0}; // separable grid: the potentials transposed per lane
  size_t part_bytes = 0, counter_count = 0;
  size_t part_cap = 0;   // bytes actually reserved at `part`
  int lane_nsplit = 1, lane_nj = 1, lane_vec = 4;
  bool fused = false;             // shared cost, one fused row->column pass per iteration
  int fused_nct = 0, fused_maxseg = 0;
  size_t cpad = 0;   // per-sample fused pass, d2 % 4 != 0: zero-padded copy of the costs
  int ldc = 0;       // its row stride (floats)
  bool padded = false;
  int fg_nct = 0, fg_maxseg = 0;  // the two-GEMM block pass (units: 16 lanes x 16 rows)
  bool gemm = false;              // large shared cost: two fp32 GEMMs per iteration
  size_t kc = 0, gx = 0, gs = 0, gt = 0, ga = 0, gvmax = 0, gvmax0 = 0, gfall = 0;
  size_t kmatT = 0, gxh = 0, gxl = 0, gah = 0, gal = 0, um_part = 0;
  int ldk1 = 0, ldk2 = 0;
};

// Fused passes (sweep_fused.cuh): shared stored cost, both padded extents
// within the register-resident row (NQ <= kFusedMaxNQ 64-column chunks).
constexpr int kFusedMaxNQ = kFusedMaxChunks;
// Per-sample costs (sweep_fused.cuh fused_ps_kernel): rows of d2 <= 2048
// floats; the bulk copies move whole 16-byte units, so d2 % 4 != 0 runs on a
// zero-padded copy of the costs made once per solve (Layout::cpad).
// Lanes per group of the per-sample pass: rows above 2048 (4096, 8192) columns
// take two (four, eight) warps per lane (fused_ps_kernel<..., kHalves>, 8 warps).
int ps_group_lanes(int d2p) {
  const int nq = d2p / 64;
  return nq <= kPsMaxChunks ? fused_warps(nq) : nq <= 2 * kPsMaxChunks ? 4
                                             : nq <= 4 * kPsMaxChunks ? 2 : 1;
}
bool fused_eligible(const sinkhorn_problem_v1& pr) {
  if (pr.B < 1) return false;
  if (pr.cost_kind == SINKHORN_COST_PER_SAMPLE)   // d2 % 4 != 0: through a padded copy
    return round_up(pr.d2, TILE_PAD) <= 8 * 64 * kPsMaxChunks;   // > 2048: 2, 4 or 8 warps per lane
  return pr.cost_kind == SINKHORN_COST_SHARED &&
         round_up(pr.d1, TILE_PAD) <= 64 * kFusedMaxNQ && round_up(pr.d2, TILE_PAD) <= 64 * kFusedMaxNQ;
}

#ifndef SKB_SEP_RN
#define SKB_SEP_RN 2
#endif
using SepGridShape = SepShape<32, SKB_SEP_RN, (SKB_SEP_RN == 2) ? 256 : 128>;
// The separable sweep stages a lane's whole nx x ny potential plus both factor
// tables in shared memory; larger grids take the dense on-the-fly sweeps.
constexpr size_t kSepSmemLimit = 227 * 1024;
bool sep_fits(const sinkhorn_problem_v1& pr) {
  return sep_smem_floats<SepGridShape>((int)pr.grid_nx, (int)pr.grid_ny, true) * 4 <=
         kSepSmemLimit;
}
// the two-kernel split (sweep_sep.cuh sep_step1/2_kernel): O(n * 96) floats
bool sep_split_fits(const sinkhorn_problem_v1& pr) {
  return sep_split1_floats<SepGridShape>((int)pr.grid_nx) * 4 <= kSepSmemLimit &&
         sep_split2_floats<SepGridShape>((int)pr.grid_ny, true) * 4 <= kSepSmemLimit;
}

// Grid costs run the separable sweeps on lane-major buffers unless the dense
// on-the-fly tiled sweeps are requested (SINKHORN_FLAG_DENSE_GRID) or the grid
// is too large for the separable sweep's shared memory.
Layout make_layout(const sinkhorn_problem_v1& pr, int sms, bool dense_grid = false,
                   bool fused = false, bool gemm = false) {
  Layout L;
  L.B = pr.B;
  L.d1 = pr.d1;
  L.d2 = pr.d2;
  L.gemm = gemm && pr.cost_kind == SINKHORN_COST_SHARED;
  L.fused = !L.gemm && fused && fused_eligible(pr);
  static const bool force_split = getenv("SKB_SEP_SPLIT") != nullptr;   // diagnostics / tests
  if (pr.cost_kind == SINKHORN_COST_GRID2D && !dense_grid) {
    L.sep_split = force_split || !sep_fits(pr);
    // degenerate aspect (nx*ny/(nx+ny) < 8: the separable saving is below 8x)
    // or too large even for the split kernels: the dense on-the-fly sweeps
    const double gain = (double)pr.grid_nx * pr.grid_ny / (double)(pr.grid_nx + pr.grid_ny);
    if (L.sep_split && (!sep_split_fits(pr) || (!force_split && gain < 8.0))) dense_grid = true;
  }
  L.sep = pr.cost_kind == SINKHORN_COST_GRID2D && !dense_grid;
  if (!L.sep) L.sep_split = false;
  L.tiled = !L.fused && !L.gemm && (pr.cost_kind == SINKHORN_COST_SHARED ||
                                    (pr.cost_kind == SINKHORN_COST_GRID2D && dense_grid));
  Carver c;
  if (L.gemm) {
    // exact extents, lane-major: the GEMMs read K / KC row-major [d1][d2]
    L.Bp = (int)pr.B;
    L.D1p = (int)pr.d1;
    L.D2p = (int)pr.d2;
    L.sb1 = L.D1p;
    L.si1 = 1;
    L.sb2 = L.D2p;
    L.si2 = 1;
    // K and K o C over (d1 rows, d2 reduction), K^T over (d2 rows, d1
    // reduction) -- the column sweep's A operand, so both contractions read
    // K-major tiles -- in the tile-major operand layout of sweep_umma.cuh
    // (extents padded to 128 rows x 32-column chunks)
    L.ldk1 = (int)round_up(pr.d1, 128);   // padded row / reduction extents
    L.ldk2 = (int)round_up(pr.d2, 128);
    L.kmat = c.take((size_t)L.ldk1 * L.ldk2 * 4);
    L.kmatT = c.take((size_t)L.ldk2 * L.ldk1 * 4);
    const size_t n1 = (size_t)L.B * L.D1p * 4, n2 = (size_t)L.B * L.D2p * 4;
    // tf32 hi / lo planes of X (reduction d2) and a (reduction d1): the MMAs'
    // B operands, tiled [B/64][chunks][64][32]
    const size_t bpad = round_up(pr.B, kUmBN);
    L.gxh = c.take(bpad * L.ldk2 * 4);
    L.gxl = c.take(bpad * L.ldk2 * 4);
    L.gah = c.take(bpad * L.ldk1 * 4);
    L.gal = c.take(bpad * L.ldk1 * 4);
    L.um_part = c.take((size_t)sms * 2 * kUmBN * kUmBM * 4);
    L.f2 = c.take(n1);
    L.g2[0] = c.take(n2);
    L.g2[1] = c.take(n2);
    L.l2mu = c.take(n1);
    L.l2nu = c.take(n2);
    L.mu = c.take(n1);
    L.nu = c.take(n2);
    L.gx = c.take(n2);
    L.gt = c.take(n2);
    L.gs = c.take(n1);
    L.ga = c.take(n1);
    L.gvmax = c.take((size_t)L.B * 4);
    L.gvmax0 = c.take((size_t)L.B * 4);
    L.gfall = c.take((size_t)L.B * L.D1p * 4);
    L.e0 = c.take(64);
    L.counter_count = 1;
  } else if (L.fused) {
    // lane-major potentials [B][Dp], Dp = the cost rows' padded length
    L.Bp = (int)pr.B;
    L.D1p = (int)round_up(pr.d1, TILE_PAD);
    L.D2p = (int)round_up(pr.d2, TILE_PAD);
    L.sb1 = L.D1p;
    L.si1 = 1;
    L.sb2 = L.D2p;
    L.si2 = 1;
    if (pr.cost_kind == SINKHORN_COST_SHARED) {
      L.a2 = c.take((size_t)L.D1p * L.D2p * 4);
      L.a2t = c.take((size_t)L.D2p * L.D1p * 4);
      L.kmat = c.take((size_t)L.D1p * L.D2p * 4);
    } else {   // the first column sweep runs lane_col_kernel (one split per column block)
      L.ldc = (int)round_up(pr.d2, 4);
      L.padded = L.ldc != pr.d2;   // rows of whole 16-byte units for the bulk copies
      if (L.padded) L.cpad = c.take((size_t)pr.B * pr.d1 * L.ldc * 4);
      L.lane_vec = (pr.d2 % 4 == 0 && pr.d1 % 4 == 0) ? 4 : 1;
      L.lane_nj = (int)((pr.d2 + 256 * L.lane_vec - 1) / (256 * L.lane_vec));
      L.lane_nsplit = 1;
    }
    const size_t n1 = (size_t)L.B * L.D1p * 4, n2 = (size_t)L.B * L.D2p * 4;
    L.f2 = c.take(n1);
    L.g2[0] = c.take(n2);
    L.g2[1] = c.take(n2);
    L.l2mu = c.take(n1);
    L.l2nu = c.take(n2);
    L.mu = c.take(n1);
    L.nu = c.take(n2);
    L.e0 = c.take(std::max(n1, n2));
    const int nw = pr.cost_kind == SINKHORN_COST_PER_SAMPLE ? ps_group_lanes(L.D2p)
                                                            : fused_warps(L.D2p / 64);
    const long long groups = (pr.B + nw - 1) / nw;
    const long long U = groups * pr.d1;
    const int occ = pr.cost_kind == SINKHORN_COST_PER_SAMPLE ? ps_ctas_per_sm(L.D2p / 64) : 1;
    L.fused_nct = (int)std::max<long long>(
        1, std::min<long long>(std::min<long long>((long long)sms * occ, kFusedMaxCtas), U));
    const long long per = (U + L.fused_nct - 1) / L.fused_nct;
    L.fused_maxseg = (int)((per - 1) / pr.d1 + 2);
    L.part_bytes = (size_t)L.fused_nct * L.fused_maxseg * nw * L.D2p * 4;
    if (pr.cost_kind == SINKHORN_COST_SHARED) {   // fgemm_pass_kernel's pieces
      const long long Ufg = ((pr.B + kFgLanes - 1) / kFgLanes) * (L.D1p / kFgRows);
      L.fg_nct = (int)std::max<long long>(1, std::min<long long>(sms, Ufg));
      const long long pfg = (Ufg + L.fg_nct - 1) / L.fg_nct;
      L.fg_maxseg = (int)((pfg - 1) / (L.D1p / kFgRows) + 2);
      L.part_bytes = std::max(L.part_bytes,
                              (size_t)L.fg_nct * L.fg_maxseg * kFgLanes * L.D2p * 4);
    }
    L.part_cap = L.part_bytes;
    L.part = c.take(L.part_cap);
    L.counter_count = 1;
  } else if (L.tiled) {
    L.Bp = (int)round_up(pr.B, pick_bt(pr.B));
    L.D1p = (int)round_up(pr.d1, TILE_PAD);
    L.D2p = (int)round_up(pr.d2, TILE_PAD);
    L.sb1 = L.sb2 = 1;
    L.si1 = L.si2 = L.Bp;
    if (pr.cost_kind == SINKHORN_COST_SHARED) {
      L.a2 = c.take((size_t)L.D1p * L.D2p * 4);
      L.a2t = c.take((size_t)L.D2p * L.D1p * 4);
    }
    const size_t n1 = (size_t)L.D1p * L.Bp * 4, n2 = (size_t)L.D2p * L.Bp * 4;
    L.f2 = c.take(n1);
    L.g2[0] = c.take(n2);
    L.g2[1] = c.take(n2);
    L.l2mu = c.take(n1);
    L.l2nu = c.take(n2);
    L.mu = c.take(n1);
    L.nu = c.take(n2);
    L.e0 = c.take(n2);
    L.part_bytes = (size_t)sms * MAX_OCC * 2 * 3 * 64 * PT_MAX * 4;   // G*BT is constant
    L.part_cap = L.part_bytes;
    L.part = c.take(L.part_cap);
    L.counter_count = (size_t)(L.Bp / 64) * (std::max(L.D1p, L.D2p) / 32 + 1);
  } else {
    L.lane_vec = (pr.d2 % 4 == 0 && pr.d1 % 4 == 0) ? 4 : 1;
    L.Bp = (int)pr.B;
    L.D1p = (int)round_up(pr.d1, 4);
    L.D2p = (int)round_up(pr.d2, 4);
    L.sb1 = L.D1p;
    L.si1 = 1;
    L.sb2 = L.D2p;
    L.si2 = 1;
    const size_t n1 = (size_t)L.B * L.D1p * 4, n2 = (size_t)L.B * L.D2p * 4;
    L.f2 = c.take(n1);
    L.g2[0] = c.take(n2);
    L.g2[1] = c.take(n2);
    L.l2mu = c.take(n1);
    L.l2nu = c.take(n2);
    L.mu = c.take(n1);
    L.nu = c.take(n2);
    L.e0 = c.take(n2);
    L.lane_nj = (int)((pr.d2 + 256 * L.lane_vec - 1) / (256 * L.lane_vec));
    const long long ctas = (long long)pr.B * L.lane_nj;
    const long long want = 4LL * sms * 8;   // a few waves of resident CTAs
    int ns = (int)std::min<long long>(std::max<long long>(1, want / std::max(1LL, ctas)), 16);
    ns = (int)std::min<long long>(ns, std::max<long long>(1, pr.d1 / 64));
    L.lane_nsplit = ns;
    L.part_bytes = ns > 1 ? (size_t)pr.B * L.lane_nj * ns * 3 * 256 * L.lane_vec * 4 : 256;
    // (also the small solver's per-check CTA maxima, [2][grid], for per-sample costs)
    L.part_cap = std::max<size_t>(L.part_bytes, (size_t)sms * 8 * 2 * 4);
    L.part = c.take(L.part_cap);
    L.counter_count = (size_t)pr.B * L.lane_nj;
  }
  L.res = c.take((size_t)std::max(L.Bp, 1) * 4);
  if (L.sep) {
    L.part_cap = std::max<size_t>(L.part_bytes, (size_t)sms * 8 * 2 * 4);
    L.part = c.take(L.part_cap);
    const size_t nblk = (size_t)(pr.grid_nx + 31) / 32;
    L.sep_ax = c.take((size_t)pr.grid_nx * nblk * 32 * 4);
    L.sep_ay = c.take((size_t)pr.grid_ny * sep_ld((int)pr.grid_ny) * 4);
    L.f2T = c.take((size_t)L.B * L.D1p * 4);
    L.g2T[0] = c.take((size_t)L.B * L.D2p * 4);
    L.g2T[1] = c.take((size_t)L.B * L.D2p * 4);
    if (L.sep_split) {
      const size_t tsz = (size_t)pr.B * nblk * pr.grid_ny * 32 * 4;
      L.sep_tg = c.take(tsz);
      L.sep_rg = c.take(tsz);
    }
  }
  L.scratch = c.take(64);
  L.counters = c.take(std::max<size_t>(L.counter_count, 1) * 4);
  L.status = c.take(4);
  L.badrow = c.take(4);
  L.total = c.off;
  return L;
}

// Workspace bytes for a problem under every option set (grid costs can take
// either the separable or the dense tiled layout).
// ---- point-cloud costs (SINKHORN_COST_POINTS) ---------------------------------
// The cost is materialised once per solve at the front of the workspace --
// the dot products on the tensor cores, then |x|^2 + |y|^2 - 2 x.y -- and the
// solve proceeds as a shared stored cost on the rest of the workspace.
struct PointLayout {
  size_t cost = 0, ya = 0, xh = 0, xl = 0, nrm = 0, part = 0, total = 0;
  long long kch = 0;
};
PointLayout point_layout(const sinkhorn_problem_v1& pr, int sms) {
  PointLayout P;
  Carver c;
  const int D = pr.grid_nx;
  P.kch = (D + kUmBK - 1) / kUmBK;
  P.cost = c.take((size_t)pr.d1 * pr.d2 * 4);
  P.ya = c.take((size_t)round_up(pr.d2, kUmBM) * P.kch * kUmBK * 4);
  P.xh = c.take((size_t)round_up(pr.d1, kUmBN) * P.kch * kUmBK * 4);
  P.xl = c.take((size_t)round_up(pr.d1, kUmBN) * P.kch * kUmBK * 4);
  P.nrm = c.take((size_t)(pr.d1 + pr.d2) * 4);
  P.part = c.take((size_t)sms * 2 * kUmBN * kUmBM * 4);
  P.total = c.take(256);
  return P;
}
sinkhorn_problem_v1 as_shared(const sinkhorn_problem_v1& pr) {
  sinkhorn_problem_v1 q = pr;
  q.cost_kind = SINKHORN_COST_SHARED;
  q.grid_nx = q.grid_ny = 0;
  q.grid_hx = q.grid_hy = 0.f;
  return q;
}

size_t workspace_total(const sinkhorn_problem_v1& pr, int sms) {
  if (pr.cost_kind == SINKHORN_COST_POINTS)
    return point_layout(pr, sms).total + workspace_total(as_shared(pr), sms);
  size_t t = make_layout(pr, sms).total;
  if (fused_eligible(pr)) t = std::max(t, make_layout(pr, sms, false, true).total);
  if (pr.cost_kind == SINKHORN_COST_SHARED) t = std::max(t, make_layout(pr, sms, false, false, true).total);
  if (pr.cost_kind == SINKHORN_COST_GRID2D) t = std::max(t, make_layout(pr, sms, true).total);
  return t;
}

template <typename T>
T* at(void* ws, size_t off) {
  return reinterpret_cast<T*>(static_cast<char*>(ws) + off);
}

// Dynamic shared-memory opt-in for a kernel on the current device.  The
// attribute is per (function, device), so the cache is keyed on both: a thread
// that solves on a second GPU sets it there too.
int set_max_smem(const void* fn, size_t bytes) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<const void*, int>, size_t>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  for (auto& e : done)
    if (e.first.first == fn && e.first.second == dev && e.second >= bytes) return 0;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess)
    return fail(SINKHORN_STATUS_CUDA_ERROR,
                std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
  for (auto& x : done)
    if (x.first.first == fn && x.first.second == dev) { x.second = bytes; return 0; }
  done.push_back({{fn, dev}, bytes});
  return 0;
}

// Resident CTAs per SM for a kernel; the attribute set + occupancy query cost
// tens of microseconds, so they run once per (kernel, device) and are cached.
int occupancy_tiled(void* fn, int threads, size_t smem) {
  static std::mutex mu;
  static std::vector<std::pair<std::pair<void*, int>, int>> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  for (auto& e : cache)
    if (e.first.first == fn && e.first.second == dev) return e.second;
  int occ = 1;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem);
  occ = std::max(1, std::min(occ, MAX_OCC));
  cache.push_back({{fn, dev}, occ});
  return occ;
}

// One tiled half-sweep launch.
struct TiledArgs {
  const CUtensorMap* tg;
  const CUtensorMap* tx;
  int Qv, Pv, Qp, Pp;
  const float* target;
  const float* marg;
  float* out;
  const float* old;
  float* res;
  int res_kind;
  float* e0;
  float* pmax;
  float* psum;
  const float* est_old = nullptr;   // estimate mode: output-side potentials before the sweep
  int use_est = 0;
  int* est_fail = nullptr;
  int use_poly = 0;                 // FMA-pipe exponentials for part of the cells
};

template <int BT, int PT>
TiledSweepParams build_tiled_params(const Layout& L, void* ws, const TiledArgs& a,
                                    const sinkhorn_problem_v1& pr, float lam, int G) {
  TiledSweepParams p = {};
  p.Qv = a.Qv;
  p.Pv = a.Pv;
  p.Bp = L.Bp;
  p.ntile_b = L.Bp / BT;
  p.ntile_p = (a.Pv + PT - 1) / PT;
  p.nq = (a.Qv + QC - 1) / QC;
#ifndef SKB_SEG_ROWS
#define SKB_SEG_ROWS 12
#endif
  p.seg_x = SKB_SEG_ROWS;   // ~3 us of per-segment cost, in rows of a 128x64 tile
  p.W = (long long)p.ntile_b * p.ntile_p * (a.Qv + p.seg_x);   // virtual rows (atom_begin)
  p.G = G;
  p.fast32 = ((unsigned long long)(p.W + 1) * (unsigned long long)(G + 1) < (1ull << 32)) ? 1 : 0;
  p.target = a.target;
  p.marg = a.marg;
  p.out = a.out;
  p.old = a.old;
  p.res = a.res;
  p.res_kind = a.res_kind;
  p.e0 = a.e0;
  p.pmax = a.pmax;
  p.psum = a.psum;
  p.part = at<float>(ws, L.part);
  p.counters = at<int>(ws, L.counters);
  p.cinv = -lam * kLn2;
  p.gk = -kLog2e / lam;
  p.gnx = pr.grid_nx;
  p.ghx2 = pr.grid_hx * pr.grid_hx;
  p.ghy2 = pr.grid_hy * pr.grid_hy;
  p.est_old = a.est_old;
  p.use_est = (a.use_est && a.est_old != nullptr) ? 1 : 0;
  p.est_fail = a.est_fail;
  p.use_poly = a.use_poly;
  p.dbg = nullptr;
  return p;
}

// chunks of the (tile, q) space: every CTA of a sweep must own >= 1 row
template <int BT, int PT>
long long tiled_chunks(const Layout& L, int Pv, int Qv) {
  return (long long)(L.Bp / BT) * ((Pv + PT - 1) / PT) * ((Qv + QC - 1) / QC);
}

template <int BT, int PT, bool kGrid, int kMode>
int launch_tiled_pt(const Layout& L, void* ws, const DeviceInfo& di, const TiledArgs& a,
                    const sinkhorn_problem_v1& pr, float lam, cudaStream_t st) {
  using K = TiledK<BT, PT, kGrid, kMode>;
  const size_t smem = K::S::SMEM_BYTES;
  const int occ = std::min(K::S::OCC, occupancy_tiled(K::fn(), K::S::NT, smem));
  const int G = (int)std::min<long long>(tiled_chunks<BT, PT>(L, a.Pv, a.Qv), (long long)di.sms * occ);
  TiledSweepParams p = build_tiled_params<BT, PT>(L, ws, a, pr, lam, G);
  // diagnostics (SKB_TIMELINE=n): per-CTA globaltimer stamps of the n-th sweep
  static const long long tl_at = getenv("SKB_TIMELINE") ? atoll(getenv("SKB_TIMELINE")) : -1;
  static long long tl_count = 0;
  static unsigned long long* tl_buf = nullptr;
  const bool tl = tl_at >= 0 && tl_count++ == tl_at;
  if (tl) {
    if (!tl_buf) CK(cudaMalloc(&tl_buf, 16384 * 8));
    CK(cudaMemsetAsync(tl_buf, 0, 16384 * 8, st));
    p.dbg = tl_buf;
  }
  auto kern = &tiled_sweep_kernel<BT, PT, QC, RB, RP, NSTAGE, kGrid, kMode>;
  kt_mark(st);
  CK(launch_pdl(kern, dim3(p.G), dim3(K::S::NT), smem, st, *a.tg, *a.tx, p));
  kt_mark(st);
  // merge + epilogue of the tiles the stream-K split cut between CTAs
  const unsigned nfix = (unsigned)(p.ntile_b * p.ntile_p * (K::S::NT * 4 / 256));
  CK(launch_pdl(&tiled_fixup_kernel<BT, PT, QC, RB, RP, kMode>, dim3(nfix), dim3(256), 0, st, p));
  if (tl) {
    std::vector<unsigned long long> h(16384);
    CK(cudaMemcpyAsync(h.data(), tl_buf, 16384 * 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    auto stats = [&](int base, int n, const char* name) {
      unsigned long long s0 = ~0ull, s1 = 0, e0 = ~0ull, e1 = 0;
      for (int i = 0; i < n; ++i) {
        s0 = std::min(s0, h[base + 2 * i]);
        s1 = std::max(s1, h[base + 2 * i]);
        e0 = std::min(e0, h[base + 2 * i + 1]);
        e1 = std::max(e1, h[base + 2 * i + 1]);
      }
      fprintf(stderr, "[skb] %s x%d: start %llu..%llu end %llu..%llu (ns)\n", name, n, s0, s1,
              e0, e1);
    };
    stats(0, p.G, "sweep");
    stats(4096, (int)nfix, "fixup");
    unsigned long long t0 = ~0ull;
    for (int c = 0; c < p.G; ++c) t0 = std::min(t0, h[2 * c]);
    for (int c = 0; c < p.G; ++c) {
      const long long a0 = atom_begin(p, c), a1 = atom_begin(p, c + 1);
      const long long segs = (a1 - 1) / p.Qv - a0 / p.Qv + 1;
      fprintf(stderr, "[skb] cta %d rows %lld segs %lld start %.2f end %.2f us chunks", c, a1 - a0,
              segs, (h[2 * c] - t0) * 1e-3, (h[2 * c + 1] - t0) * 1e-3);
      for (int l = 0; l < 16 && h[8192 + c * 16 + l]; ++l)
        fprintf(stderr, " %.2f", (h[8192 + c * 16 + l] - t0) * 1e-3);
      fprintf(stderr, " | first row %lld | setup %.2f issued %.2f waited %.2f\n", a0,
              (h[12288 + c * 4] - t0) * 1e-3, (h[12288 + c * 4 + 1] - t0) * 1e-3,
              (h[12288 + c * 4 + 2] - t0) * 1e-3);
    }
  }
  return 0;
}

template <bool kGrid, int kMode>
int launch_tiled(const Layout& L, void* ws, const DeviceInfo& di, const TiledArgs& a,
                 const sinkhorn_problem_v1& pr, float lam, cudaStream_t st) {
  return pick_bt(pr.B) == 128 ? launch_tiled_pt<128, 64, kGrid, kMode>(L, ws, di, a, pr, lam, st)
                               : launch_tiled_pt<64, 64, kGrid, kMode>(L, ws, di, a, pr, lam, st);
}

// ---- the solver --------------------------------------------------------------
struct Solve {
  sinkhorn_problem_v1 pr;
  sinkhorn_options_v1 op;
  Layout L;
  DeviceInfo di;
  void* ws;
  cudaStream_t st;
  float lam;
  CUtensorMap tm_a2, tm_a2t, tm_f2, tm_g2[2];
  const float* cost;
  bool est = false;        // estimate mode for the tiled sweeps (set per iteration)
  bool poly = true;        // FMA-pipe polynomial exponentials for part of the cells
  int* est_fail = nullptr;

  float* F(size_t off) const { return at<float>(ws, off); }

  int setup_maps() {
    if (!L.tiled) return 0;
    const float* gsrc_col = pr.cost_kind == SINKHORN_COST_SHARED ? F(L.a2) : F(L.f2);
    const float* gsrc_row = pr.cost_kind == SINKHORN_COST_SHARED ? F(L.a2t) : F(L.f2);
    bool ok = true;
    if (pr.cost_kind == SINKHORN_COST_SHARED) {
      // G boxes are [QC][PT] with PT picked from the sweep's output extent
      ok &= make_tmap(&tm_a2, gsrc_col, L.D1p, L.D2p, QC, pick_pt((int)pr.d2));
      ok &= make_tmap(&tm_a2t, gsrc_row, L.D2p, L.D1p, QC, pick_pt((int)pr.d1));
    }
    const int bt = pick_bt(pr.B);
    ok &= make_tmap(&tm_f2, F(L.f2), L.D1p, L.Bp, QC, bt);
    ok &= make_tmap(&tm_g2[0], F(L.g2[0]), L.D2p, L.Bp, QC, bt);
    ok &= make_tmap(&tm_g2[1], F(L.g2[1]), L.D2p, L.Bp, QC, bt);
    if (pr.cost_kind != SINKHORN_COST_SHARED) {
      tm_a2 = tm_f2;   // unused by the grid kernel; any valid map
      tm_a2t = tm_f2;
    }
    return ok ? 0 : fail(SINKHORN_STATUS_CUDA_ERROR, "cuTensorMapEncodeTiled failed");
  }

  // column half-sweep: g2[dst] = l2nu - LSE_i(A2 + f2)
  // ---- separable grid sweeps (sweep_sep.cuh) --------------------------------
  using SepS = SepGridShape;
  static constexpr int kSepNB = SepS::NB;
  int sep_sweep(int mode, const float* xT, const float* target, const float* marg,
                const float* old, float* out, float* outT, int res_kind,
                const float* est_src = nullptr) {
    SepParams p = {};
    p.nx = (int)pr.grid_nx;
    p.ny = (int)pr.grid_ny;
    p.ax_tab = F(L.sep_ax);
    p.ay_tab = F(L.sep_ay);
    p.cinv = -lam * kLn2;
    p.xT = xT;
    p.outT = outT;
    p.target = target;
    p.marg = marg;
    p.old = old;
    p.out = out;
    p.res = F(L.res);
    p.res_kind = res_kind;
    p.ld = L.D1p;
    p.B = (int)pr.B;
    p.nblk = (p.nx + kSepNB - 1) / kSepNB;
    p.use_poly = poly ? 1 : 0;
    p.est_src = est_src;
    p.redo = at<unsigned int>(ws, L.scratch + 48);
    const bool tail = mode == kModeTail;
    if (L.sep_split) {   // large grid: step 1 -> T in global -> step 2
      p.tg = F(L.sep_tg);
      p.rg = F(L.sep_rg);
      const size_t sm1 = sep_split1_floats<SepS>(p.nx) * 4;
      const size_t sm2 = sep_split2_floats<SepS>(p.ny, tail) * 4;
      auto k1 = tail ? &sep_step1_kernel<SepS, kModeTail> : &sep_step1_kernel<SepS, kModeUpdate>;
      auto k2 = tail ? &sep_step2_kernel<SepS, kModeTail> : &sep_step2_kernel<SepS, kModeUpdate>;
      if (int e = set_max_smem(reinterpret_cast<const void*>(k1), sm1)) return e;
      if (int e = set_max_smem(reinterpret_cast<const void*>(k2), sm2)) return e;
      const unsigned mblk = (unsigned)((p.ny + SepS::MT - 1) / SepS::MT);
      kt_mark(st);
      for (long long b0 = 0; b0 < pr.B; b0 += kMaxLanesPerLaunch) {
        p.b0 = (int)b0;
        const dim3 grid((unsigned)p.nblk, mblk, lanes_in_launch(pr.B, b0));
        CK(launch_pdl(k1, grid, dim3(SepS::NT), sm1, st, p));
        CK(launch_pdl(k2, grid, dim3(SepS::NT), sm2, st, p));
      }
      kt_mark(st);
      return 0;
    }
    const size_t smem = sep_smem_floats<SepS>(p.nx, p.ny, tail) * 4;
    auto kern = tail ? &sep_sweep_kernel<SepS, kModeTail> : &sep_sweep_kernel<SepS, kModeUpdate>;
    if (int e = set_max_smem(reinterpret_cast<const void*>(kern), smem)) return e;
    dim3 grid((unsigned)p.nblk, (unsigned)pr.B);
    // diagnostics (SKB_SEP_TIMELINE=n): per-CTA start / staged / end stamps of the n-th sweep
    static const long long tl_at = getenv("SKB_SEP_TIMELINE") ? atoll(getenv("SKB_SEP_TIMELINE")) : -1;
    static long long tl_count = 0;
    static unsigned long long* tl_buf = nullptr;
    const bool tl = tl_at >= 0 && tl_count++ == tl_at;
    const size_t nct = (size_t)grid.x * grid.y;
    if (tl) {
      if (!tl_buf) CK(cudaMalloc(&tl_buf, 8 * 4096 * 8));
      p.dbg = tl_buf;
    }
    kt_mark(st);
    for (long long b0 = 0; b0 < pr.B; b0 += kMaxLanesPerLaunch) {
      p.b0 = (int)b0;
      grid.y = lanes_in_launch(pr.B, b0);
      CK(launch_pdl(kern, grid, dim3(SepS::NT), smem, st, p));
    }
    kt_mark(st);
    if (tl) {
      std::vector<unsigned long long> h(8 * 4096);
      CK(cudaMemcpyAsync(h.data(), tl_buf, 8 * 4096 * 8, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      unsigned long long t0 = ~0ull;
      for (size_t c = 0; c < nct; ++c) t0 = std::min(t0, h[4 * c]);
      for (size_t c = 0; c < nct; ++c)
        fprintf(stderr, "[skb] sep cta %zu sm %llu start %.2f staged %.2f end %.2f | factors %.2f "
                "waited %.2f loaded %.2f\n", c, h[4 * c + 3],
                (h[4 * c] - t0) * 1e-3, (h[4 * c + 1] - t0) * 1e-3, (h[4 * c + 2] - t0) * 1e-3,
                (h[16384 + 4 * c] - t0) * 1e-3, (h[16384 + 4 * c + 1] - t0) * 1e-3,
                (h[16384 + 4 * c + 2] - t0) * 1e-3);
    }
    return 0;
  }

  int col_sweep(int dst, int src_old, int res_kind) {
    if (L.tiled) {
      TiledArgs a = {&tm_a2, &tm_f2, (int)pr.d1, (int)pr.d2, L.D1p, L.D2p, F(L.l2nu), F(L.nu),
                     F(L.g2[dst]), F(L.g2[src_old]), F(L.res), res_kind, nullptr, nullptr,
                     nullptr, F(L.g2[src_old]), est ? 1 : 0, est_fail, poly ? 1 : 0};
      return pr.cost_kind == SINKHORN_COST_GRID2D
                 ? launch_tiled<true, kModeUpdate>(L, ws, di, a, pr, lam, st)
                 : launch_tiled<false, kModeUpdate>(L, ws, di, a, pr, lam, st);
    }
    if (L.sep)
      return sep_sweep(kModeUpdate, F(L.f2T), F(L.l2nu), F(L.nu), F(L.g2[src_old]), F(L.g2[dst]),
                       F(L.g2T[dst]), res_kind, est ? F(L.g2[src_old]) : nullptr);
    return lane_col(kModeUpdate, F(L.g2[dst]), F(L.g2[src_old]), res_kind);
  }

  // row half-sweep: f2 = l2mu - LSE_j(A2^T + g2[src])
  int row_sweep(int src, int res_kind) {
    if (L.tiled) {
      TiledArgs a = {&tm_a2t, &tm_g2[src], (int)pr.d2, (int)pr.d1, L.D2p, L.D1p, F(L.l2mu),
                     F(L.mu), F(L.f2), nullptr, F(L.res), res_kind, nullptr, nullptr, nullptr,
                     F(L.f2), est ? 1 : 0, est_fail, poly ? 1 : 0};
      return pr.cost_kind == SINKHORN_COST_GRID2D
                 ? launch_tiled<true, kModeUpdate>(L, ws, di, a, pr, lam, st)
                 : launch_tiled<false, kModeUpdate>(L, ws, di, a, pr, lam, st);
    }
    if (L.sep)
      return sep_sweep(kModeUpdate, F(L.g2T[src]), F(L.l2mu), F(L.mu), nullptr, F(L.f2),
                       F(L.f2T), res_kind, est ? F(L.f2) : nullptr);
    LaneSweepParams p = lane_params();
    p.x = F(L.g2[src]);
    p.ldx = L.D2p;
    p.ldo = L.D1p;
    p.target = F(L.l2mu);
    p.marg = F(L.mu);
    p.out = F(L.f2);
    p.res = F(L.res);
    p.res_kind = res_kind;
    const int rows = 32;
    for (long long b0 = 0; b0 < pr.B; b0 += kMaxLanesPerLaunch) {
      p.b0 = (int)b0;
      dim3 grid((unsigned)((pr.d1 + rows - 1) / rows), lanes_in_launch(pr.B, b0));
      if (L.lane_vec == 4)
        CK(launch_pdl(&lane_row_kernel<4>, grid, dim3(256), 0, st, p, rows));
      else
        CK(launch_pdl(&lane_row_kernel<1>, grid, dim3(256), 0, st, p, rows));
    }
    return 0;
  }

  // final column pass: E0 terms + column residual against g2[cur]
  int tail(int cur) {
    if (L.tiled) {
      TiledArgs a = {&tm_a2, &tm_f2, (int)pr.d1, (int)pr.d2, L.D1p, L.D2p, F(L.l2nu), F(L.nu),
                     nullptr, F(L.g2[cur]), F(L.res), kResCol, F(L.e0), nullptr, nullptr,
                     F(L.g2[cur]), est ? 1 : 0, est_fail, poly ? 1 : 0};
      return pr.cost_kind == SINKHORN_COST_GRID2D
                 ? launch_tiled<true, kModeTail>(L, ws, di, a, pr, lam, st)
                 : launch_tiled<false, kModeTail>(L, ws, di, a, pr, lam, st);
    }
    if (L.sep)
      return sep_sweep(kModeTail, F(L.f2T), nullptr, F(L.nu), F(L.g2[cur]), F(L.e0), nullptr,
                       kResCol);
    return lane_col(kModeTail, nullptr, F(L.g2[cur]), kResCol);
  }

  // ---- fused row->column passes (sweep_fused.cuh) ---------------------------
  template <int NQ, bool kRowOnly, bool kTail, bool kLin>
  int launch_fused_t(const FusedParams& fp) {
    auto kern = &fused_pass_kernel<NQ, kRowOnly, kTail, kLin>;
    if (int e = set_max_smem(reinterpret_cast<const void*>(kern), fused_smem_bytes<NQ>())) return e;
    const size_t smem = (size_t)kFusedStages * fp.rowlen * 4 + kFusedStages * 8;
    ++g_launches;
    kt_mark(st);
    CK(launch_pdl(kern, dim3((unsigned)fp.nct), dim3(fused_warps(NQ) * 32), smem, st, fp));
    kt_mark(st);
    return 0;
  }
  template <int NQ, bool kRowOnly>
  int launch_fused_nq(const FusedParams& fp) {
    if constexpr (NQ > kFusedMaxChunks) {
      return fail(SINKHORN_STATUS_BAD_ARGUMENT, "fused pass: row too long");
    } else {
      if (fp.nq != NQ) return launch_fused_nq<NQ + 1, kRowOnly>(fp);
      if constexpr (kRowOnly) return launch_fused_t<NQ, true, false, false>(fp);
      return fp.e0 != nullptr ? launch_fused_t<NQ, false, true, false>(fp)
                              : launch_fused_t<NQ, false, false, true>(fp);
    }
  }
  template <int NQ, bool kTail, int kHalves = 1>
  int launch_fused_ps_t(const FusedParams& fp) {
    auto kern = &fused_ps_kernel<NQ, kTail, fused_warps(NQ), kHalves>;
    const size_t smem = fused_ps_smem_bytes<NQ>();
    if (int e = set_max_smem(reinterpret_cast<const void*>(kern), smem)) return e;
    ++g_launches;
    kt_mark(st);
    const float* rows = L.padded ? F(L.cpad) : cost;
    CK(launch_pdl(kern, dim3((unsigned)fp.nct), dim3(fused_warps(NQ) * 32), smem, st, fp, rows,
                  (int)pr.d2, L.ldc, (float)(-kLog2e / lam)));
    kt_mark(st);
    return 0;
  }
  template <int NQ>
  int launch_fused_ps(const FusedParams& fp) {
    if constexpr (NQ > kPsMaxChunks) {
      return launch_fused_ps2<kPsMaxChunks / 2 + 2>(fp);   // rows above 2048 columns
    } else {
      if (fp.nq != NQ) return launch_fused_ps<NQ + 1>(fp);
      return fp.e0 != nullptr ? launch_fused_ps_t<NQ, true>(fp) : launch_fused_ps_t<NQ, false>(fp);
    }
  }
  // two warps per lane, NQ chunks each (ceil(nq / 2) rounded up to even, 18..32:
  // half the instantiations; the extra columns are zero-filled), then four
  template <int NQ>
  int launch_fused_ps2(const FusedParams& fp) {
    if constexpr (NQ > kPsMaxChunks) {
      return launch_fused_ps4<kPsMaxChunks / 2 + 2>(fp);
    } else {
      if ((((fp.nq + 1) / 2) + 1) / 2 * 2 != NQ) return launch_fused_ps2<NQ + 2>(fp);
      return fp.e0 != nullptr ? launch_fused_ps_t<NQ, true, 2>(fp)
                              : launch_fused_ps_t<NQ, false, 2>(fp);
    }
  }
  template <int NQ>
  int launch_fused_ps4(const FusedParams& fp) {
    if constexpr (NQ > kPsMaxChunks) {
      return launch_fused_ps8<kPsMaxChunks / 2 + 2>(fp);
    } else {
      if ((((fp.nq + 3) / 4) + 1) / 2 * 2 != NQ) return launch_fused_ps4<NQ + 2>(fp);
      return fp.e0 != nullptr ? launch_fused_ps_t<NQ, true, 4>(fp)
                              : launch_fused_ps_t<NQ, false, 4>(fp);
    }
  }
  template <int NQ>
  int launch_fused_ps8(const FusedParams& fp) {
    if constexpr (NQ > kPsMaxChunks) {
      return fail(SINKHORN_STATUS_BAD_ARGUMENT, "fused pass: row too long");
    } else {
      if ((((fp.nq + 7) / 8) + 1) / 2 * 2 != NQ) return launch_fused_ps8<NQ + 2>(fp);
      return fp.e0 != nullptr ? launch_fused_ps_t<NQ, true, 8>(fp)
                              : launch_fused_ps_t<NQ, false, 8>(fp);
    }
  }
  template <int NQ>
  int launch_fgemm(const FusedParams& fp, int nrb) {
    if constexpr (NQ > kFusedMaxChunks) {
      return fail(SINKHORN_STATUS_BAD_ARGUMENT, "fused pass: row too long");
    } else {
      if (fp.nq != NQ) return launch_fgemm<NQ + 1>(fp, nrb);
      const int mode = fp.vmax_out != nullptr ? 2 : fp.e0 != nullptr ? 1 : 0;
      auto kern = mode == 2 ? &fgemm_pass_kernel<NQ, 2>
                  : mode == 1 ? &fgemm_pass_kernel<NQ, 1> : &fgemm_pass_kernel<NQ, 0>;
      const size_t smem = fg_smem_bytes<NQ>();
      if (int e = set_max_smem(reinterpret_cast<const void*>(kern), smem)) return e;
      ++g_launches;
      kt_mark(st);
      CK(launch_pdl(kern, dim3((unsigned)fp.nct), dim3(kFgThreads), smem, st, fp, nrb));
      kt_mark(st);
      return 0;
    }
  }
  template <bool kRowOnly>
  int launch_fused(const FusedParams& fp) {
    return launch_fused_nq<1, kRowOnly>(fp);
  }
  FusedParams fused_common() const {
    FusedParams fp = {};
    fp.B = (int)pr.B;
    fp.status = at<int>(ws, L.status);
    fp.est_fail = est_fail;
    fp.e0_log2scale = std::log2(lam * kLn2);
    return fp;
  }
  // first column sweep (no plan yet): g2[dst] = l2nu - LSE_i(A2^T[j, i] + f2[i])
  int fused_row_only(int dst) {
    FusedParams fp = fused_common();
    const int nw = fused_warps(L.D1p / 64);
    const long long groups = (pr.B + nw - 1) / nw;
    fp.nrows = (int)pr.d2;
    fp.rowlen = L.D1p;
    fp.nq = L.D1p / 64;
    fp.U = groups * pr.d2;
    fp.nct = (int)std::max<long long>(1, std::min<long long>(di.sms, fp.U));
    fp.a2 = F(L.a2t);
    fp.x = F(L.f2);
    fp.target = F(L.l2nu);
    fp.marg = F(L.nu);
    fp.out = F(L.g2[dst]);
    fp.ldo = L.D2p;
    return launch_fused<true>(fp);
  }
  // iteration k: u_k from v_k = g2[cur] (row sweep), then v_{k+1} into
  // g2[cur ^ 1] from the plan's column marginal; residuals / E0 row terms on request
  int fused_iteration(int cur, bool res, bool e0, bool first = false) {
    FusedParams fp = fused_common();
    const int nw = pr.cost_kind == SINKHORN_COST_PER_SAMPLE ? ps_group_lanes(L.D2p)
                                                            : fused_warps(L.D2p / 64);
    const long long groups = (pr.B + nw - 1) / nw;
    fp.nrows = (int)pr.d1;
    fp.rowlen = L.D2p;
    fp.nq = L.D2p / 64;
    fp.U = groups * pr.d1;
    fp.nct = L.fused_nct;
    fp.maxseg = L.fused_maxseg;
    // check / last iterations: log-domain rows (residual and E0 terms);
    // the others: linear rows K_ij * 2^(v_j - vmax) with a log-domain fallback
    fp.a2 = (res || e0) ? F(L.a2) : F(L.kmat);
    fp.a2log = F(L.a2);
    fp.x = F(L.g2[cur]);
    fp.target = F(L.l2mu);
    fp.marg = F(L.mu);
    fp.out = F(L.f2);
    fp.ldo = L.D1p;
    fp.part = F(L.part);
    fp.res = (res || e0) ? F(L.res) : nullptr;   // kTail: residual and E0 together
    fp.e0 = (res || e0) ? F(L.e0) : nullptr;
    // non-check iterations of shared costs: the two-GEMM block pass (units are
    // 16 lanes x 16 rows; the merge walks the same unit space)
    const bool fg = pr.cost_kind == SINKHORN_COST_SHARED && g_use_fgemm;
    int merge_nw = nw, merge_rows = (int)pr.d1;
    if (fg) {
      const int nrb = L.D1p / kFgRows;
      fp.U = ((pr.B + kFgLanes - 1) / kFgLanes) * (long long)nrb;
      fp.nct = L.fg_nct;
      fp.maxseg = L.fg_maxseg;
      fp.a2 = F(L.kmat);   // the block pass streams K (its tail recovers c from K)
      if (first) fp.vmax_out = F(L.g2[cur]);   // v := umax_b, then the merge writes v_1
      merge_nw = kFgLanes;
      merge_rows = nrb;
      if (int e = launch_fgemm<1>(fp, nrb)) return e;
    } else if (pr.cost_kind == SINKHORN_COST_PER_SAMPLE) {
      if (int e = launch_fused_ps<1>(fp)) return e;
    } else {
      if (int e = launch_fused<false>(fp)) return e;
    }
    FusedMergeParams mp = {};
    mp.B = (int)pr.B;
    mp.nrows = merge_rows;
    mp.rowlen = L.D2p;
    mp.nw = merge_nw;
    mp.U = fp.U;
    mp.nct = fp.nct;
    mp.maxseg = fp.maxseg;
    mp.part = F(L.part);
    mp.v_old = F(L.g2[cur]);
    mp.v_new = F(L.g2[cur ^ 1]);
    mp.target = F(L.l2nu);
    mp.marg = F(L.nu);
    mp.res = res ? F(L.res) : nullptr;
    mp.est_fail = est_fail;
    for (long long b0 = 0; b0 < pr.B; b0 += kMaxLanesPerLaunch) {
      mp.b0 = (int)b0;
      CK(launch_pdl(&fused_merge_kernel,
                    dim3((unsigned)((L.D2p + 511) / 512), lanes_in_launch(pr.B, b0)), dim3(256), 0,
                    st, mp));
    }
    return 0;
  }

  // ---- GEMM path (sweep_gemm.cuh, contractions in sweep_umma.cuh) -------------
  // rows: S[b][i] = sum_j K[i][j] X[b][j]  (A = K or K o C, B operand = X)
  // cols: T[b][j] = sum_i K^T[j][i] a[b][i] (A = K^T, B operand = a)
  CUtensorMap tm_k, tm_kt, tm_xh, tm_xl, tm_ah, tm_al;
  int setup_umma_maps() {
    if (!L.gemm) return 0;
    // tiled operands: 2-D [tiles * chunks * sub-blocks * rows][32] maps, pitch 128 B
    const size_t k1 = (size_t)(pr.d1 + kUmBK - 1) / kUmBK * kUmSub;   // 32-wide sub-blocks
    const size_t k2 = (size_t)(pr.d2 + kUmBK - 1) / kUmBK * kUmSub;
    const size_t mt1 = (size_t)L.ldk1 / kUmBM, mt2 = (size_t)L.ldk2 / kUmBM;
    const size_t nt = (size_t)(pr.B + kUmBN - 1) / kUmBN;
    bool ok = make_tmap_sw128(&tm_k, F(L.kmat), mt1 * k2 * kUmBM, 32, 32, kUmBM);
    ok &= make_tmap_sw128(&tm_kt, F(L.kmatT), mt2 * k1 * kUmBM, 32, 32, kUmBM);
    ok &= make_tmap_sw128(&tm_xh, F(L.gxh), nt * k2 * kUmBN, 32, 32, kUmBN);
    ok &= make_tmap_sw128(&tm_xl, F(L.gxl), nt * k2 * kUmBN, 32, 32, kUmBN);
    ok &= make_tmap_sw128(&tm_ah, F(L.gah), nt * k1 * kUmBN, 32, 32, kUmBN);
    ok &= make_tmap_sw128(&tm_al, F(L.gal), nt * k1 * kUmBN, 32, 32, kUmBN);
    return ok ? 0 : fail(SINKHORN_STATUS_CUDA_ERROR, "cuTensorMapEncodeTiled failed (umma)");
  }
  // (x: blocks over a lane's d elements, y: lanes) for the lane-wise epilogues
  dim3 lane_grid(int64_t d) const {
    const int64_t per_lane = std::max<int64_t>(1, (int64_t)di.sms * 8 / std::max<int64_t>(pr.B, 1));
    return dim3((unsigned)std::min<int64_t>((d + 255) / 256, per_lane), (unsigned)pr.B);
  }
  // the lane operand's tf32 planes (tiled) from its lane-major fp32 array
  int umma_split(const float* x, int d, float* hi, float* lo) {
    const long long kch = (d + kUmBK - 1) / kUmBK;
    ++g_launches;
    umma_split_kernel<<<grid_for((size_t)round_up(pr.B, kUmBN) * kch * kUmBK), 256, 0, st>>>(
        x, (int)pr.B, d, kch, hi, lo);
    CK(cudaGetLastError());
    return 0;
  }
  int gemm(bool rows, const CUtensorMap& tA, float* C, bool kc = false) {
    UmmaParams p = {};
    p.M = (int)(rows ? pr.d1 : pr.d2);
    p.K = (int)(rows ? pr.d2 : pr.d1);
    p.N = (int)pr.B;
    p.MT = (p.M + kUmBM - 1) / kUmBM;
    p.NT = (p.N + kUmBN - 1) / kUmBN;
    p.KCH = (p.K + kUmBK - 1) / kUmBK;
    p.units = (long long)p.MT * p.NT * p.KCH;
    p.G = (int)std::min<long long>(di.sms, p.units);
    p.out = C;
    p.ldo = p.M;
    p.part = F(L.um_part);
    p.status = at<int>(ws, L.status);
    p.kc_scale = (float)(lam * kLn2);
    auto kern = kc ? &umma_gemm_kernel<true> : &umma_gemm_kernel<false>;
    if (int e = set_max_smem(reinterpret_cast<const void*>(kern), kUmSmemBytes)) return e;
    kt_mark(st);
    CK(launch_pdl(kern, dim3(p.G), dim3(kUmThreads), kUmSmemBytes, st, tA,
                  rows ? tm_xh : tm_ah, rows ? tm_xl : tm_al, p));
    kt_mark(st);
    CK(launch_pdl(umma_fixup_kernel, dim3((unsigned)p.G), dim3(256), 0, st, p));
    return 0;
  }
  int gemm_col(const float* vmax, const float* v_old, float* v_new, bool res) {
    GemmColParams cp = {};
    cp.B = (int)pr.B;
    cp.d2 = (int)pr.d2;
    cp.T = F(L.gt);
    cp.vmax = vmax;
    cp.v_old = v_old;
    cp.v_new = v_new;
    cp.l2nu = F(L.l2nu);
    cp.nu = F(L.nu);
    cp.res = res ? F(L.res) : nullptr;
    cp.est_fail = est_fail;
    cp.status = at<int>(ws, L.status);
    ++g_launches;
    for (long long b0 = 0; b0 < pr.B; b0 += kMaxLanesPerLaunch) {
      cp.b0 = (int)b0;
      dim3 g = lane_grid(pr.d2);
      g.y = lanes_in_launch(pr.B, b0);
      gemm_col_kernel<<<g, 256, 0, st>>>(cp);
    }
    CK(cudaGetLastError());
    return 0;
  }
  // the first column sweep: v_1 = l2nu - LSE_i(A2 + u_0), u_0 = 0 on the support
  int gemm_first() {
    ++g_launches;
    gemm_first_a_kernel<<<grid_for((size_t)pr.B * pr.d1), 256, 0, st>>>(F(L.mu),
                                                                       (size_t)pr.B * pr.d1, F(L.ga));
    CK(cudaMemsetAsync(F(L.gvmax0), 0, (size_t)pr.B * 4, st));
    if (int e = umma_split(F(L.ga), (int)pr.d1, F(L.gah), F(L.gal))) return e;
    if (int e = gemm(false, tm_kt, F(L.gt))) return e;
    if (int e = sum_over_ranks(F(L.gt), pr.B * pr.d2)) return e;
    return gemm_col(F(L.gvmax0), nullptr, F(L.g2[1]), false);
  }
  // iteration k from v_k = g2[cur]: X, S = K X, u and a, T = K^T a, v_{k+1}
  int gemm_iteration(int cur, bool res) {
    ++g_launches;
    gemm_scale_kernel<<<(unsigned)pr.B, 1024, 0, st>>>(F(L.g2[cur]), (int)pr.d2, F(L.gx),
                                                        F(L.gvmax));
    CK(cudaGetLastError());
    if (int e = umma_split(F(L.gx), (int)pr.d2, F(L.gxh), F(L.gxl))) return e;
    if (int e = gemm(true, tm_k, F(L.gs))) return e;
    int* nfall = at<int>(ws, L.counters);
    CK(cudaMemsetAsync(nfall, 0, 4, st));
    GemmRowParams rp = {};
    rp.B = (int)pr.B;
    rp.d1 = (int)pr.d1;
    rp.d2 = (int)pr.d2;
    rp.S = F(L.gs);
    rp.vmax = F(L.gvmax);
    rp.l2mu = F(L.l2mu);
    rp.mu = F(L.mu);
    rp.u = F(L.f2);
    rp.a = F(L.ga);
    rp.nfall = nfall;
    rp.fall = at<int>(ws, L.gfall);
    rp.res = res ? F(L.res) : nullptr;
    rp.status = at<int>(ws, L.status);
    ++g_launches;
    for (long long b0 = 0; b0 < pr.B; b0 += kMaxLanesPerLaunch) {
      rp.b0 = (int)b0;
      dim3 g = lane_grid(pr.d1);
      g.y = lanes_in_launch(pr.B, b0);
      gemm_row_kernel<<<g, 256, 0, st>>>(rp);
    }
    ++g_launches;
    gemm_row_fallback_kernel<<<(unsigned)di.sms, 256, 0, st>>>(rp, cost, F(L.g2[cur]),
                                                                -kLog2e / lam);
    CK(cudaGetLastError());
    if (int e = umma_split(F(L.ga), (int)pr.d1, F(L.gah), F(L.gal))) return e;
    if (int e = gemm(false, tm_kt, F(L.gt))) return e;
    if (int e = sum_over_ranks(F(L.gt), pr.B * pr.d2)) return e;
    return gemm_col(F(L.gvmax), F(L.g2[cur]), F(L.g2[cur ^ 1]), res);
  }
  // E0 from the last iteration's X and a: sum_i a_i ((K o C) X)_i
  int gemm_e0(float* out_cost) {
    if (int e = gemm(true, tm_k, F(L.gs), true)) return e;   // (K o C) X from K
    ++g_launches;
    gemm_e0_kernel<<<(unsigned)pr.B, 256, 0, st>>>(F(L.ga), F(L.gs), (int)pr.d1, out_cost,
                                                   at<int>(ws, L.status));
    CK(cudaGetLastError());
    return sum_over_ranks(out_cost, pr.B);   // row shards: E0 = sum of the ranks' row partials
  }
  // Row-sharded solves: the column sums of the local rows become the global
  // ones.  In the linear domain every rank's partial carries the same shift
  // (vmax_b: all ranks hold the full v), so the (max, sum-exp) merge of
  // OnlineLseAccumulator.merge (batch.py:116-130) needs no max exchange: it is
  // one sum all-reduce of the partial sums, enqueued on the solve's stream.
  int sum_over_ranks(float* data, int64_t count) {
    if (!g_allreduce) return 0;
    g_allreduce(data, count, SINKHORN_REDUCE_SUM, st, g_allreduce_user);
    CK(cudaGetLastError());
    return 0;
  }

  LaneSweepParams lane_params() {
    LaneSweepParams p = {};
    p.d1 = (int)pr.d1;
    p.d2 = (int)pr.d2;
    p.cost = cost;
    p.kscale = -kLog2e / lam;
    p.part = F(L.part);
    p.counters = at<int>(ws, L.counters);
    p.nsplit = L.lane_nsplit;
    p.status = at<int>(ws, L.status);
    return p;
  }

  bool validate_cost_in_sweep = false;   // per-sample: the first column sweep checks the cost

  int lane_col(int mode, float* out, const float* old, int res_kind) {
    LaneSweepParams p = lane_params();
    const bool validate = validate_cost_in_sweep && mode == kModeUpdate;
    if (validate) {
      validate_cost_in_sweep = false;
      p.vstatus = at<int>(ws, L.status);
      dim3 grid((unsigned)L.lane_nsplit, (unsigned)pr.B, (unsigned)L.lane_nj);
      p.x = F(L.f2);
      p.ldx = L.D1p;
      p.ldo = L.D2p;
      p.target = F(L.l2nu);
      p.marg = F(L.nu);
      p.out = out;
      p.old = old;
      p.res = F(L.res);
      p.res_kind = res_kind;
      p.e0 = F(L.e0);
      for (long long b0 = 0; b0 < pr.B; b0 += kMaxLanesPerLaunch) {
        p.b0 = (int)b0;
        grid.y = lanes_in_launch(pr.B, b0);
        if (L.lane_vec == 4)
          CK(launch_pdl(&lane_col_kernel<4, kModeUpdate, true>, grid, dim3(256), 0, st, p));
        else
          CK(launch_pdl(&lane_col_kernel<1, kModeUpdate, true>, grid, dim3(256), 0, st, p));
      }
      return 0;
    }
    p.x = F(L.f2);
    p.ldx = L.D1p;
    p.ldo = L.D2p;
    p.target = F(L.l2nu);
    p.marg = F(L.nu);
    p.out = out;
    p.old = old;
    p.res = F(L.res);
    p.res_kind = res_kind;
    p.e0 = F(L.e0);
    dim3 grid((unsigned)L.lane_nsplit, (unsigned)pr.B, (unsigned)L.lane_nj);
    for (long long b0 = 0; b0 < pr.B; b0 += kMaxLanesPerLaunch) {
      p.b0 = (int)b0;
      grid.y = lanes_in_launch(pr.B, b0);
      if (mode == kModeTail) {
        if (L.lane_vec == 4) CK(launch_pdl(&lane_col_kernel<4, kModeTail>, grid, dim3(256), 0, st, p));
        else CK(launch_pdl(&lane_col_kernel<1, kModeTail>, grid, dim3(256), 0, st, p));
      } else {
        if (L.lane_vec == 4) CK(launch_pdl(&lane_col_kernel<4, kModeUpdate>, grid, dim3(256), 0, st, p));
        else CK(launch_pdl(&lane_col_kernel<1, kModeUpdate>, grid, dim3(256), 0, st, p));
      }
    }
    return 0;
  }

  int zero_res() {
    CK(cudaMemsetAsync(F(L.res), 0, (size_t)std::max(L.Bp, 1) * 4, st));
    return 0;
  }

  template <int BT, bool kGrid>
  int persistent_loop_bt(const sinkhorn_options_v1& op, bool allow_est, int* iters, int* cur) {
    constexpr int PT = 64;
    using K = TiledK<BT, PT, kGrid, kModeUpdate>;
    auto kern = &persistent_solve_kernel<BT, PT, QC, RB, RP, NSTAGE, kGrid>;
    const size_t smem = K::S::SMEM_BYTES;
    if (int e = set_max_smem(reinterpret_cast<const void*>(kern), smem)) return e;
    // every CTA must own >= 1 row of both sweep orientations
    const long long G = std::min<long long>(
        di.sms, std::min(tiled_chunks<BT, PT>(L, (int)pr.d2, (int)pr.d1),
                         tiled_chunks<BT, PT>(L, (int)pr.d1, (int)pr.d2)));
    PersistMaps maps;
    maps.a2 = tm_a2;
    maps.a2t = tm_a2t;
    maps.f2 = tm_f2;
    maps.g2[0] = tm_g2[0];
    maps.g2[1] = tm_g2[1];
    PersistParams P = {};
    TiledArgs ca = {&tm_a2, &tm_f2, (int)pr.d1, (int)pr.d2, L.D1p, L.D2p, F(L.l2nu), F(L.nu),
                    nullptr, nullptr, F(L.res), kResNone, nullptr, nullptr, nullptr,
                    nullptr, 0, est_fail, poly ? 1 : 0};
    TiledArgs ra = {&tm_a2t, &tm_g2[0], (int)pr.d2, (int)pr.d1, L.D2p, L.D1p, F(L.l2mu),
                    F(L.mu), F(L.f2), nullptr, F(L.res), kResNone, nullptr, nullptr, nullptr,
                    nullptr, 0, est_fail, poly ? 1 : 0};
    P.col = build_tiled_params<BT, PT>(L, ws, ca, pr, lam, (int)G);
    P.row = build_tiled_params<BT, PT>(L, ws, ra, pr, lam, (int)G);
    P.g2[0] = F(L.g2[0]);
    P.g2[1] = F(L.g2[1]);
    P.f2 = F(L.f2);
    P.res = F(L.res);
    P.B = (int)pr.B;
    P.Bp = L.Bp;
    P.max_iters = op.max_iters;
    P.check_interval = op.check_interval;
    P.est_from = allow_est ? kEstFromIter : (op.max_iters + 1);
    P.tol = op.tolerance;
    P.bar = at<unsigned int>(ws, L.scratch + 32);
    P.result = at<int>(ws, L.scratch + 40);
    CK(cudaMemsetAsync(P.bar, 0, 4, st));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)G);
    cfg.blockDim = dim3(K::S::NT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;   // all CTAs co-resident: grid barriers are safe
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    ++g_launches;
    CK(cudaLaunchKernelEx(&cfg, kern, maps, P));
    int h[2] = {0, 0};
    CK(cudaMemcpyAsync(h, P.result, 8, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    *iters = h[0];
    *cur = h[1];
    return 0;
  }

  int persistent_loop(const sinkhorn_options_v1& op, bool allow_est, int* iters, int* cur) {
    const bool grid = pr.cost_kind == SINKHORN_COST_GRID2D;
    if (pick_bt(pr.B) == 128)
      return grid ? persistent_loop_bt<128, true>(op, allow_est, iters, cur)
                  : persistent_loop_bt<128, false>(op, allow_est, iters, cur);
    return grid ? persistent_loop_bt<64, true>(op, allow_est, iters, cur)
                : persistent_loop_bt<64, false>(op, allow_est, iters, cur);
  }

  // ---- small shared / grid costs: the whole solve in one launch -----------
  // (sweep_small.cuh).  Eligible when both cost orientations and the lanes'
  // potentials fit in one CTA's shared memory and each CTA's share of a sweep
  // is small enough that launches, not exponentials, would bound the tiled path.
  static constexpr int kSmallNT = 512;
  static constexpr long long kSmallMaxCells = 1LL << 17;   // per CTA per half-sweep

  static int pick_group(long long units, long long n) {
    int best = 1;
    double bc = 1e300;
    for (int S = 1; S <= 32; S <<= 1) {
      const long long rounds = (units * S + kSmallNT - 1) / kSmallNT;
      const double E = (double)((n + S - 1) / S);
      const double c = (double)rounds * (2.0 * E + 8.0 * std::log2((double)S) + 10.0);
      if (c < bc) {
        bc = c;
        best = S;
      }
    }
    return best;
  }

  // Returns a status (non-zero only on a CUDA error); *ok says whether to use it.
  bool warm = false;   // the solve starts from a caller's log u (f2 holds it)

  int plan_small(SmallParams& sp, int& G, size_t& smem, bool* ok) {
    *ok = false;
    // per-sample costs: the small solver reads each lane's cost once per solve
    // instead of once per iteration, which pays below ~64 x 64 cells per lane
    // (tools/ps_small_bench.py: d = 32 3.3x, 64 1.15x, 128 0.97x the fused pass)
    const bool ps = pr.cost_kind == SINKHORN_COST_PER_SAMPLE && pr.d1 * pr.d2 <= 4096;
    if (pr.cost_kind == SINKHORN_COST_PER_SAMPLE && !ps) return 0;
    if (!(L.tiled || L.sep || ps) || g_reducer != nullptr || (op.flags & SINKHORN_FLAG_TILED_ONLY))
      return 0;
    if (pr.cost_kind != SINKHORN_COST_SHARED && pr.cost_kind != SINKHORN_COST_GRID2D && !ps)
      return 0;
    int smem_optin = 0;
    cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, di.dev);
    const long long d1 = pr.d1, d2 = pr.d2, B = pr.B;
    auto kern = ps ? &small_solve_kernel<kSmallNT, true> : &small_solve_kernel<kSmallNT, false>;
    {
      cudaFuncAttributes fa = {};
      CK(cudaFuncGetAttributes(&fa, kern));
      if (int e = set_max_smem(reinterpret_cast<const void*>(kern),
                               (size_t)(smem_optin - (int)fa.sharedSizeBytes)))
        return e;
      // a function attribute, also per device; cheap enough to set every call
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    }
    for (int occ = 4; occ >= 1; --occ) {
      int Lc = (int)((B + (long long)di.sms * occ - 1) / ((long long)di.sms * occ));
      if (ps) {   // per-sample: each lane stages its own cost; as many lanes as fit (no clusters)
        const int S0c = pick_group((long long)d2, d1), S0r = pick_group((long long)d1, d2);
        const int ldc0 = (int)round_up(d1, 32) + (S0c % 32), ldr0 = (int)round_up(d2, 32) + (S0r % 32);
        Lc = 0;
        while (Lc < 16 && Lc < B &&
               SmallSmem::floats((int)d1, (int)d2, Lc + 1, ldc0, ldr0, 1, true) * 4 <=
                   (size_t)smem_optin / occ - 2048)
          ++Lc;
        if (Lc == 0) continue;
      }
      if ((long long)Lc * d1 * d2 > kSmallMaxCells) continue;
      const int Gl = (int)((B + Lc - 1) / Lc);   // lane groups
      // spread a lane group over a cluster while SMs are left idle and every
      // CTA keeps >= 16 outputs and >= 16k cells per half-sweep: a cluster
      // barrier costs ~0.5 us per half-sweep, and below that size the sweep is
      // bound by its serial chain, not its cell count (config 1, d = 100:
      // C = 1 0.317 ms per loop, C = 4 0.328)
      int Cc = 1;
      while (!ps && Cc < 8 && (long long)Gl * Cc * 2 <= di.sms && std::min(d1, d2) / (Cc * 2) >= 16 &&
             (long long)Lc * d1 * d2 / (Cc * 2) >= 16384)
        Cc *= 2;
      static const int force_c = getenv("SKB_SMALL_C") ? atoi(getenv("SKB_SMALL_C")) : 0;
      if (force_c > 0 && !ps) Cc = force_c;   // diagnostics: cluster size A/B
      int Sc = 1, Sr = 1, ldc = 0, ldr = 0;
      size_t bytes = 0;
      for (;; Cc *= 2) {   // a larger cluster when the cost slices do not fit one CTA
        const long long units_c = (long long)Lc * ((d2 + Cc - 1) / Cc);
        const long long units_r = (long long)Lc * ((d1 + Cc - 1) / Cc);
        Sc = pick_group(units_c, d1);
        Sr = pick_group(units_r, d2);
        ldc = (int)round_up(d1, 32) + (Sc % 32);
        ldr = (int)round_up(d2, 32) + (Sr % 32);
        bytes = SmallSmem::floats((int)d1, (int)d2, Lc, ldc, ldr, Cc, ps) * 4;
        if (bytes <= (size_t)smem_optin / occ - 2048 || force_c > 0 || Cc >= 8 || ps ||
            (long long)Gl * Cc * 2 > di.sms || std::min(d1, d2) / (Cc * 2) < 16)
          break;
      }
      if (bytes > (size_t)smem_optin / occ - 2048) continue;
      int fit = 0;
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&fit, kern, kSmallNT, bytes));
      if (fit < 1) return 0;
      G = Gl * Cc;
      // per-check CTA maxima [2][G] live in the layout's `part` region
      if (op.tolerance > 0 && (size_t)2 * G * 4 > L.part_cap) continue;
      if (op.tolerance > 0) {   // the grid barrier needs every CTA (cluster) co-resident
        if (G > fit * di.sms) continue;
        if (Cc > 1) {
          cudaLaunchConfig_t qc = {};
          qc.gridDim = dim3((unsigned)G);
          qc.blockDim = dim3(kSmallNT);
          qc.dynamicSmemBytes = bytes;
          cudaLaunchAttribute qa[1];
          qa[0].id = cudaLaunchAttributeClusterDimension;
          qa[0].val.clusterDim.x = (unsigned)Cc;
          qa[0].val.clusterDim.y = 1;
          qa[0].val.clusterDim.z = 1;
          qc.attrs = qa;
          qc.numAttrs = 1;
          int nclusters = 0;
          CK(cudaOccupancyMaxActiveClusters(&nclusters, kern, &qc));
          if (nclusters < Gl) continue;
        }
      }
      smem = bytes;
      sp = SmallParams{};
      sp.cps = ps ? cost : nullptr;
      sp.kscale = (float)(-kLog2e / lam);
      sp.a2 = (pr.cost_kind == SINKHORN_COST_SHARED) ? F(L.a2) : nullptr;
      sp.a2t = (pr.cost_kind == SINKHORN_COST_SHARED) ? F(L.a2t) : nullptr;
      sp.D1p = L.D1p;
      sp.D2p = L.D2p;
      sp.grid = pr.cost_kind == SINKHORN_COST_GRID2D;
      sp.gnx = (int)pr.grid_nx;
      sp.gk = (float)(-kLog2e / lam);
      sp.ghx2 = pr.grid_hx * pr.grid_hx;
      sp.ghy2 = pr.grid_hy * pr.grid_hy;
      sp.cinv = -lam * kLn2;
      sp.l2mu = F(L.l2mu);
      sp.l2nu = F(L.l2nu);
      sp.mu = F(L.mu);
      sp.nu = F(L.nu);
      sp.f2_init = warm ? F(L.f2) : nullptr;
      sp.B = (int)B;
      sp.sb1 = L.sb1;
      sp.si1 = L.si1;
      sp.sb2 = L.sb2;
      sp.si2 = L.si2;
      sp.d1 = (int)d1;
      sp.d2 = (int)d2;
      sp.L = Lc;
      sp.C = Cc;
      sp.Sc = Sc;
      sp.Sr = Sr;
      sp.ldc = ldc;
      sp.ldr = ldr;
      sp.max_iters = op.max_iters;
      sp.check_interval = op.check_interval;
      sp.checks = op.tolerance > 0 ? 1 : 0;
      sp.tol = (float)op.tolerance;
      sp.res = F(L.res);
      sp.cta_res = F(L.part);
      sp.bar = at<unsigned int>(ws, L.scratch + 32);
      sp.result = at<int>(ws, L.scratch + 40);
      sp.status = at<int>(ws, L.status);
      *ok = true;
      return 0;
    }
    return 0;
  }

  int small_solve(SmallParams& sp, int G, size_t smem, float* out_cost, float* out_log_u,
                  float* out_log_v, int* iters) {
    sp.out_cost = out_cost;
    sp.out_log_u = out_log_u;
    sp.out_log_v = out_log_v;
    CK(cudaMemsetAsync(sp.bar, 0, 4, st));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)G);
    cfg.blockDim = dim3(kSmallNT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = (unsigned)sp.C;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
    if (sp.checks) {
      attr[na].id = cudaLaunchAttributeCooperative;   // grid barrier at the stopping tests
      attr[na].val.cooperative = 1;
      ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = (unsigned)na;
    static const bool tl = getenv("SKB_SMALL_TIMELINE") != nullptr;   // diagnostics
    static unsigned long long* tl_buf = nullptr;
    if (tl) {
      if (!tl_buf) CK(cudaMalloc(&tl_buf, 64 * 8));
      CK(cudaMemsetAsync(tl_buf, 0, 64 * 8, st));
      sp.dbg = tl_buf;
    }
    ++g_launches;
    kt_mark(st);
    CK(cudaLaunchKernelEx(&cfg, sp.cps != nullptr ? &small_solve_kernel<kSmallNT, true>
                                                 : &small_solve_kernel<kSmallNT, false>,
                          sp));
    kt_mark(st);
    if (tl) {
      unsigned long long h[64];
      CK(cudaMemcpyAsync(h, tl_buf, sizeof(h), cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      for (int k = 1; k <= 8; ++k)
        fprintf(stderr, "[skb] small it %d: col %.2f sync %.2f row %.2f sync %.2f us\n", k,
                (h[4 * k] - (k == 1 ? h[0] : h[4 * k - 1])) * 1e-3, (h[4 * k + 1] - h[4 * k]) * 1e-3,
                (h[4 * k + 2] - h[4 * k + 1]) * 1e-3, (h[4 * k + 3] - h[4 * k + 2]) * 1e-3);
      fprintf(stderr, "[skb] small C %d L %d Sc %d Sr %d grid %d\n", sp.C, sp.L, sp.Sc, sp.Sr,
              (int)cfg.gridDim.x);
    }
    if (sp.checks) {
      CK(cudaMemcpyAsync(iters, sp.result, 4, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
    } else {
      *iters = sp.max_iters;
    }
    return 0;
  }

  int read_status(int* out) {
    CK(cudaMemcpyAsync(out, at<int>(ws, L.status), 4, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return 0;
  }
};

int fill(float* p, size_t n, float v, cudaStream_t st) {
  if (n == 0) return 0;
  ++g_launches;
  fill_kernel<<<grid_for(n), 256, 0, st>>>(p, n, v);
  CK(cudaGetLastError());
  return 0;
}

int check_problem(const sinkhorn_problem_v1* pr) {
  if (!pr) return fail(SINKHORN_STATUS_BAD_ARGUMENT, "null problem");
  if (pr->B < 0 || pr->d1 < 0 || pr->d2 < 0)
    return fail(SINKHORN_STATUS_SHAPE_MISMATCH, "negative extent");
  if (pr->B > INT32_MAX || pr->d1 > INT32_MAX || pr->d2 > INT32_MAX)
    return fail(SINKHORN_STATUS_SHAPE_MISMATCH, "extent exceeds int32");
  if (pr->cost_kind == SINKHORN_COST_GRID2D) {
    if (pr->grid_nx < 1 || pr->grid_ny < 1 || (int64_t)pr->grid_nx * pr->grid_ny != pr->d1 ||
        pr->d1 != pr->d2)
      return fail(SINKHORN_STATUS_SHAPE_MISMATCH, "grid cost needs d1 = d2 = nx*ny");
    if (!(std::isfinite(pr->grid_hx) && std::isfinite(pr->grid_hy) && pr->grid_hx >= 0 &&
          pr->grid_hy >= 0))
      return fail(SINKHORN_STATUS_INVALID_COST, "grid spacing must be finite and >= 0");
  } else if (pr->cost_kind == SINKHORN_COST_POINTS) {
    if (pr->grid_nx < 1 || pr->grid_nx > 4096)
      return fail(SINKHORN_STATUS_SHAPE_MISMATCH, "point dimension (grid_nx) must be in 1..4096");
  } else if (pr->cost_kind != SINKHORN_COST_SHARED && pr->cost_kind != SINKHORN_COST_PER_SAMPLE) {
    return fail(SINKHORN_STATUS_BAD_ARGUMENT, "unknown cost_kind");
  }
  return 0;
}

int check_options(const sinkhorn_options_v1* op) {
  if (!op) return fail(SINKHORN_STATUS_BAD_ARGUMENT, "null options");
  // SinkhornConfig.__post_init__ (core.py:88-96)
  if (!(std::isfinite(op->lambda) && op->lambda > 0))
    return fail(SINKHORN_STATUS_INVALID_CONFIG, "lam must be positive and finite");
  if (op->max_iters < 1) return fail(SINKHORN_STATUS_INVALID_CONFIG, "max_iters must be >= 1");
  if (!(std::isfinite(op->tolerance) && op->tolerance >= 0))
    return fail(SINKHORN_STATUS_INVALID_CONFIG, "tolerance must be >= 0");
  if (op->check_interval < 1)
    return fail(SINKHORN_STATUS_INVALID_CONFIG, "check_interval must be >= 1");
  return 0;
}

// ---- CUDA graphs of the fused iteration loop (tolerance 0) -----------------
struct FusedGraphKey {
  const void* ws;
  const float* cost;
  int64_t B, d1, d2;
  int32_t kind;
  double lambda;
  int32_t max_iters;
  int dev;
  int path;   // 1 fused passes, 2 GEMM iteration (the same problem can take either)
  bool operator==(const FusedGraphKey& o) const {
    return ws == o.ws && cost == o.cost && B == o.B && d1 == o.d1 && d2 == o.d2 && kind == o.kind &&
           lambda == o.lambda && max_iters == o.max_iters && dev == o.dev && path == o.path;
  }
};
struct FusedGraph {
  FusedGraphKey key;
  bool seen = false;
  cudaGraphExec_t exec = nullptr;
  unsigned long long launches = 0;
  int iters = 0, cur = 0;
  unsigned long long used = 0;
};
thread_local std::vector<FusedGraph> g_fused_graphs;   // a few recent problems per thread
thread_local unsigned long long g_fused_graph_clock = 0;
const bool g_no_graph = getenv("SKB_NO_GRAPH") != nullptr;   // diagnostics

FusedGraph* fused_graph_slot(const FusedGraphKey& k) {
  ++g_fused_graph_clock;
  for (auto& g : g_fused_graphs)
    if (g.key == k) {
      g.used = g_fused_graph_clock;
      return &g;
    }
  if (g_fused_graphs.size() >= 8) {   // evict the least recently used
    auto it = std::min_element(g_fused_graphs.begin(), g_fused_graphs.end(),
                               [](const FusedGraph& a, const FusedGraph& b) { return a.used < b.used; });
    if (it->exec) cudaGraphExecDestroy(it->exec);
    g_fused_graphs.erase(it);
  }
  FusedGraph g;
  g.key = k;
  g.used = g_fused_graph_clock;
  g_fused_graphs.push_back(g);
  return &g_fused_graphs.back();
}

int enqueue_async_tail(const sinkhorn_problem_v1& pr, const sinkhorn_options_v1& op,
                       const float* mu, const float* nu, const float* cost, float* out_cost,
                       float* out_log_u, float* out_log_v, float* out_residuals, void* ws,
                       size_t ws_bytes, cudaStream_t st, const float* init_log_u,
                       int32_t* device_status, const int* ws_status, const int* est_fail,
                       bool can_fail);

// capturing: enqueue only (the body of an asynchronous solve's rerun graph);
// device_status != nullptr: asynchronous solve (tolerance 0) -- no host
// synchronisation, the status and the rerun decision stay on the device.
__global__ void fill_int_kernel(int* p, int n, int v) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = v;
}
// Asynchronous solves: the rerun decision on the device (a conditional graph
// node reads est_fail), and the final status copied to the caller's word.
__global__ void async_gate_kernel(cudaGraphConditionalHandle h, const int* est_fail,
                                  const int* status) {
  cudaGraphSetConditional(h, (*est_fail != 0 && *status == 0) ? 1u : 0u);
}
__global__ void async_status_kernel(const int* status, int32_t* out) { *out = *status; }

int forward_impl(const sinkhorn_problem_v1& pr, const sinkhorn_options_v1& op, const float* mu,
                 const float* nu, const float* cost, float* out_cost, float* out_log_u,
                 float* out_log_v, int32_t* out_iterations, float* out_residuals, void* ws,
                 size_t ws_bytes, cudaStream_t st, bool allow_est = true,
                 const float* init_log_u = nullptr, int32_t* device_status = nullptr,
                 bool capturing = false) {
  const bool async_mode = device_status != nullptr;
  const bool force_rerun_diag = (op.flags & SINKHORN_FLAG_FORCE_RERUN) != 0;
  for (cudaEvent_t e : g_kt.ev) cudaEventDestroy(e);
  g_kt.ev.clear();
  g_kt.on = !async_mode && (op.flags & SINKHORN_FLAG_TIME_KERNEL) != 0;
  Solve S;
  S.pr = pr;
  S.op = op;
  S.di = device_info();
  S.L = make_layout(pr, S.di.sms, (op.flags & SINKHORN_FLAG_DENSE_GRID) != 0);
  S.ws = ws;
  S.st = st;
  S.lam = (float)op.lambda;
  S.cost = cost;
  S.poly = (op.flags & SINKHORN_FLAG_MUFU_ONLY) == 0;
  S.warm = init_log_u != nullptr;
  // one fused row->column pass per iteration for shared costs, unless the
  // problem takes the single-launch small solver (or this is the exact rerun)
  const bool cost_aligned = (reinterpret_cast<uintptr_t>(cost) & 15) == 0;
  if (allow_est && !(op.flags & (SINKHORN_FLAG_NO_FUSED | SINKHORN_FLAG_FORCE_GEMM)) &&
      fused_eligible(pr) &&
      (pr.cost_kind != SINKHORN_COST_PER_SAMPLE || cost_aligned)) {
    SmallParams sp0;
    int g0 = 0;
    size_t sm0 = 0;
    bool small0 = false;
    if (int e = S.plan_small(sp0, g0, sm0, &small0)) return e;
    if (!small0) S.L = make_layout(pr, S.di.sms, false, true);
  }
  // large shared costs (and on request any shared cost): two GEMMs per iteration
  if (allow_est && pr.cost_kind == SINKHORN_COST_SHARED && !S.L.fused &&
      !(op.flags & SINKHORN_FLAG_NO_GEMM) &&
      ((op.flags & SINKHORN_FLAG_FORCE_GEMM) || !fused_eligible(pr))) {
    SmallParams sp0;
    int g0 = 0;
    size_t sm0 = 0;
    bool small0 = false;
    if (int e = S.plan_small(sp0, g0, sm0, &small0)) return e;
    if (!small0) S.L = make_layout(pr, S.di.sms, false, false, true);
  }
  const Layout& L = S.L;
  if (ws_bytes < L.total || ws == nullptr)
    return fail(SINKHORN_STATUS_WORKSPACE, "workspace too small");
  int* status = at<int>(ws, L.status);
  int* badrow = at<int>(ws, L.badrow);
  S.est_fail = at<int>(ws, L.scratch + 16);

  // ---- setup (batch.py:279-296) ----
  CK(cudaMemsetAsync(status, 0, 4, st));
  CK(cudaMemsetAsync(S.est_fail, 0, 4, st));
  CK(cudaMemsetAsync(at<int>(ws, L.scratch + 48), 0, 4, st));   // estimate redo count
  CK(cudaMemsetAsync(badrow, 0x7f, 4, st));
  CK(cudaMemsetAsync(at<int>(ws, L.counters), 0, std::max<size_t>(L.counter_count, 1) * 4, st));
  CK(cudaMemsetAsync(S.F(L.res), 0, (size_t)std::max(L.Bp, 1) * 4, st));
  if (!(op.flags & SINKHORN_FLAG_SKIP_VALIDATION)) {
    ++g_launches;
    validate_rows_kernel<float><<<(unsigned)pr.B, 256, 0, st>>>(mu, (int)pr.d1, status, badrow);
    ++g_launches;
    validate_rows_kernel<float><<<(unsigned)pr.B, 256, 0, st>>>(nu, (int)pr.d2, status, badrow);
    CK(cudaGetLastError());
  }
  {
    dim3 g1((unsigned)((L.D1p + 31) / 32), (unsigned)((L.Bp + 31) / 32));
    ++g_launches;
    prep_marginal_kernel<<<g1, 256, 0, st>>>(mu, (int)pr.B, (int)pr.d1, L.Bp, L.D1p, L.sb1,
                                              L.si1, S.F(L.l2mu), S.F(L.mu), S.F(L.f2), 1);
    dim3 g2((unsigned)((L.D2p + 31) / 32), (unsigned)((L.Bp + 31) / 32));
    ++g_launches;
    prep_marginal_kernel<<<g2, 256, 0, st>>>(nu, (int)pr.B, (int)pr.d2, L.Bp, L.D2p, L.sb2,
                                              L.si2, S.F(L.l2nu), S.F(L.nu), S.F(L.g2[0]), 0);
    CK(cudaGetLastError());
    if (int e = fill(S.F(L.g2[1]), (size_t)(L.tiled ? (size_t)L.D2p * L.Bp : (size_t)L.B * L.D2p),
                     neg_inf_host(), st))
      return e;
  }
  if (init_log_u != nullptr) {   // warm start: log u from the caller, -inf off the support
    dim3 gi((unsigned)((L.D1p + 31) / 32), (unsigned)((L.Bp + 31) / 32));
    ++g_launches;
    import_potential_kernel<<<gi, 256, 0, st>>>(init_log_u, (int)pr.B, (int)pr.d1, L.Bp, L.D1p,
                                                L.sb1, L.si1, S.F(L.f2));
    const size_t n1 = L.tiled ? (size_t)L.D1p * L.Bp : (size_t)L.B * L.D1p;
    ++g_launches;
    mask_potential_kernel<<<grid_for(n1), 256, 0, st>>>(S.F(L.f2), S.F(L.mu), n1);
    CK(cudaGetLastError());
  }
  if (L.gemm) {
    ++g_launches;
    if (pr.d2 % 4 == 0 && (reinterpret_cast<uintptr_t>(cost) & 15) == 0) {
      dim3 g((unsigned)(L.ldk2 / 128), (unsigned)(L.ldk1 / 32));
      umma_kernel_matrices_vec4<<<g, 256, 0, st>>>(cost, (int)pr.d1, (int)pr.d2,
                                                   (float)(-kLog2e / op.lambda), S.F(L.kmat),
                                                   S.F(L.kmatT), status);
    } else {
      dim3 g((unsigned)(L.ldk2 / 32), (unsigned)(L.ldk1 / 32));
      umma_kernel_matrices<<<g, 256, 0, st>>>(cost, (int)pr.d1, (int)pr.d2,
                                              (float)(-kLog2e / op.lambda), S.F(L.kmat),
                                              S.F(L.kmatT), status);
    }
    CK(cudaGetLastError());
  } else if (pr.cost_kind == SINKHORN_COST_SHARED) {
    dim3 g((unsigned)((L.D2p + 31) / 32), (unsigned)((L.D1p + 31) / 32));
    ++g_launches;
    prep_cost_kernel<<<g, 256, 0, st>>>(cost, (int)pr.d1, (int)pr.d2, L.D1p, L.D2p,
                                         (float)(-1.4426950408889634 / op.lambda), S.F(L.a2),
                                         S.F(L.a2t), status);
    CK(cudaGetLastError());
    if (L.fused) {
      const size_t nk = (size_t)L.D1p * L.D2p;
      ++g_launches;
      kernel_matrix_kernel<<<grid_for(nk), 256, 0, st>>>(S.F(L.a2), S.F(L.kmat), nk);
      CK(cudaGetLastError());
    }
  } else if (pr.cost_kind == SINKHORN_COST_PER_SAMPLE && !(op.flags & SINKHORN_FLAG_SKIP_VALIDATION)) {
    // checked by the first column sweep, which reads every element once anyway
    // (lane_col_kernel<..., kValidate>): no separate pass over the 4.3 GB
    S.validate_cost_in_sweep = true;
  }
  if (L.padded) {   // fused per-sample pass with d2 % 4 != 0: rows padded to 16-byte units
    ++g_launches;
    pad_rows_kernel<<<grid_for((size_t)pr.B * pr.d1 * 32), 256, 0, st>>>(
        cost, (long long)pr.B * pr.d1, (int)pr.d2, L.ldc, S.F(L.cpad));
    CK(cudaGetLastError());
  }
  if (L.sep) {   // the separable sweeps' factor tables (once per solve), log u transposed
    const int nblk = (int)((pr.grid_nx + 31) / 32);
    ++g_launches;
    sep_transpose_kernel<<<grid_for((size_t)pr.B * pr.d1), 256, 0, st>>>(
        S.F(L.f2), S.F(L.f2T), (int)pr.B, L.D1p, (int)pr.grid_nx, (int)pr.grid_ny);
    ++g_launches;
    sep_tables_kernel<<<64, 256, 0, st>>>(S.F(L.sep_ax), S.F(L.sep_ay), (int)pr.grid_nx,
                                          (int)pr.grid_ny, nblk * 32,
                                          (float)(-kLog2e / op.lambda) * (pr.grid_hx * pr.grid_hx),
                                          (float)(-kLog2e / op.lambda) * (pr.grid_hy * pr.grid_hy));
    CK(cudaGetLastError());
  }
  SmallParams sp;
  int small_grid = 0;
  size_t small_smem = 0;
  bool small = false;
  if (int e = S.plan_small(sp, small_grid, small_smem, &small)) return e;
  if (!small) {
    if (int e = S.setup_maps()) return e;
    if (int e = S.setup_umma_maps()) return e;
  }

  // ---- lockstep iteration (batch.py:314-324) ----
  // Optional: CUDA events on the caller's stream around the iteration loop, so
  // a benchmark can report the sweep kernels' average launch duration.
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  const bool timed = !async_mode && (op.flags & SINKHORN_FLAG_TIME_LOOP) != 0;
  if (timed) {
    CK(cudaEventCreate(&ev0));
    CK(cudaEventCreate(&ev1));
    CK(cudaEventRecord(ev0, st));
  }
  const bool checks = op.tolerance > 0;
  int cur = 0;            // g2[cur] holds log_v_k
  bool have_next = false; // g2[cur] already advanced by a check sweep
  int iters = 0;
  // Opt-in: the whole loop in one cooperative kernel (no launches, device-side
  // stopping test).  Off by default: its grid barriers (~3.5 us each, two per
  // half-sweep) cost more than the launch gaps they remove.
  const bool persist = L.tiled && g_reducer == nullptr &&
                       (op.flags & SINKHORN_FLAG_PERSISTENT) != 0;
  if (small) {
    if (int e = S.small_solve(sp, small_grid, small_smem, out_cost, out_log_u, out_log_v, &iters))
      return e;
  } else if (persist) {
    if (int e = S.persistent_loop(op, allow_est, &iters, &cur)) return e;
  }
  g_last_path = small     ? "small"
                : persist ? "persistent"
                : L.fused ? "fused"
                : L.gemm  ? "gemm"
                : L.tiled ? "tiled"
                : L.sep   ? "separable"
                          : "lane";
  // Without a stopping test the loop has no host decision: a repeated solve
  // (same workspace, cost and shape) replays it as one CUDA graph, so its
  // launches (2 per iteration fused, 8 on the GEMM iteration) cannot stall
  // behind the host.
  auto run_loop = [&](auto&& loop, bool graphable) -> int {
    FusedGraph* fg = nullptr;
    if (graphable && !checks && g_reducer == nullptr && !g_no_graph && !g_kt.on && !capturing)
      fg = fused_graph_slot(FusedGraphKey{ws, cost, pr.B, pr.d1, pr.d2, pr.cost_kind, op.lambda,
                                          op.max_iters, S.di.dev, L.gemm ? 2 : 1});
    if (fg != nullptr && fg->seen && fg->exec == nullptr) {   // second sighting: capture
      // a capture stream per (thread, device): a stream belongs to the device
      // that was current when it was created
      static thread_local cudaStream_t cs_dev[64] = {};
      if (S.di.dev < 0 || S.di.dev >= 64) return fail(SINKHORN_STATUS_CUDA_ERROR, "device ordinal");
      cudaStream_t& cs = cs_dev[S.di.dev];
      if (cs == nullptr) CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
      const unsigned long long l0 = g_launches;
      S.st = cs;
      CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
      const int e = loop();
      cudaGraph_t graph = nullptr;
      const cudaError_t ce = cudaStreamEndCapture(cs, &graph);
      S.st = st;
      if (e) return e;
      CK(ce);
      CK(cudaGraphInstantiate(&fg->exec, graph, 0));
      CK(cudaGraphDestroy(graph));
      fg->launches = g_launches - l0;
      fg->iters = iters;
      fg->cur = cur;
      g_launches = l0;
    }
    if (fg != nullptr && fg->exec != nullptr) {
      CK(cudaGraphLaunch(fg->exec, st));
      g_launches += fg->launches;
      iters = fg->iters;
      cur = fg->cur;
    } else {
      if (fg != nullptr) fg->seen = true;
      if (int e = loop()) return e;
    }
    return 0;
  };
  if (L.fused && !small) {
    // v_1 from u_0, then one fused pass (+ column merge) per iteration
    auto fused_loop = [&]() -> int {
      if (pr.cost_kind == SINKHORN_COST_PER_SAMPLE) {
        if (int e = S.lane_col(kModeUpdate, S.F(L.g2[1]), S.F(L.g2[0]), kResNone)) return e;
      } else if (g_use_fgemm) {   // the block pass from u0 (cur = 0), merged into g2[1]
        if (int e = S.fused_iteration(0, false, false, true)) return e;
      } else {
        if (int e = S.fused_row_only(1)) return e;
      }
      cur = 1;
      for (int k = 1; k <= op.max_iters; ++k) {
        const bool last = (k == op.max_iters);
        const bool check = checks && (k % op.check_interval == 0) && !last;
        if (check || last) {
          if (int e = S.zero_res()) return e;
        }
        if (int e = S.fused_iteration(cur, check || last, check || last)) return e;
        iters = k;
        if (last) break;
        if (check) {
          ++g_launches;
          reduce_max_kernel<<<1, 256, 0, S.st>>>(S.F(L.res), (int)pr.B, S.F(L.scratch));
          CK(cudaGetLastError());
          float hmax = 0.f;
          int hstatus = 0;
          CK(cudaMemcpyAsync(&hmax, S.F(L.scratch), 4, cudaMemcpyDeviceToHost, S.st));
          CK(cudaMemcpyAsync(&hstatus, status, 4, cudaMemcpyDeviceToHost, S.st));
          CK(cudaStreamSynchronize(S.st));
          double gmax = (hstatus != 0) ? NAN : (double)hmax;
          if (g_reducer) gmax = g_reducer(gmax, g_reducer_user);
          if (hstatus != 0) break;
          if (gmax <= op.tolerance) break;   // converged: g2[cur] = log_v_k, f2 = log_u_k
        }
        cur ^= 1;
      }
      return 0;
    };
    if (int e = run_loop(fused_loop, true)) return e;
  }
  if (L.gemm && !small) {
    auto gemm_loop = [&]() -> int {
      if (int e = S.gemm_first()) return e;
      cur = 1;
      for (int k = 1; k <= op.max_iters; ++k) {
        const bool last = (k == op.max_iters);
        const bool check = checks && (k % op.check_interval == 0) && !last;
        if (check || last) {
          if (int e = S.zero_res()) return e;
        }
        if (int e = S.gemm_iteration(cur, check || last)) return e;
        iters = k;
        if (last) break;
        if (check) {
          ++g_launches;
          reduce_max_kernel<<<1, 256, 0, S.st>>>(S.F(L.res), (int)pr.B, S.F(L.scratch));
          CK(cudaGetLastError());
          float hmax = 0.f;
          int hstatus = 0;
          CK(cudaMemcpyAsync(&hmax, S.F(L.scratch), 4, cudaMemcpyDeviceToHost, S.st));
          CK(cudaMemcpyAsync(&hstatus, status, 4, cudaMemcpyDeviceToHost, S.st));
          CK(cudaStreamSynchronize(S.st));
          double gmax = (hstatus != 0) ? NAN : (double)hmax;
          if (g_reducer) gmax = g_reducer(gmax, g_reducer_user);
          if (hstatus != 0) break;
          if (gmax <= op.tolerance) break;   // converged: g2[cur] = log_v_k, X and a of iteration k
        }
        cur ^= 1;
      }
      return 0;
    };
    // (row shards call the all-reduce between contractions: not captured)
    if (int e = run_loop(gemm_loop, g_allreduce == nullptr)) return e;
  }
  for (int k = 1; !persist && !small && !L.fused && !L.gemm && k <= op.max_iters; ++k) {
    // estimate mode once the potentials have settled past the first sweeps
    S.est = allow_est && k >= kEstFromIter;
    if (!have_next) {
      if (int e = S.col_sweep(cur ^ 1, cur, kResNone)) return e;
      cur ^= 1;
    }
    have_next = false;
    const bool last = (k == op.max_iters);
    const bool check = checks && (k % op.check_interval == 0) && !last;
    if (check || last) {
      if (int e = S.zero_res()) return e;
    }
    if (int e = S.row_sweep(cur, (check || last) ? kResRow : kResNone)) return e;
    iters = k;
    if (check) {
      // column sweep k+1 doubles as the column residual of iteration k
      if (int e = S.col_sweep(cur ^ 1, cur, kResCol)) return e;
      ++g_launches;
      reduce_max_kernel<<<1, 256, 0, st>>>(S.F(L.res), (int)pr.B, S.F(L.scratch));
      CK(cudaGetLastError());
      float hmax = 0.f;
      int hstatus = 0;
      CK(cudaMemcpyAsync(&hmax, S.F(L.scratch), 4, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(&hstatus, status, 4, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      double gmax = (hstatus != 0) ? NAN : (double)hmax;
      if (g_reducer) gmax = g_reducer(gmax, g_reducer_user);   // every rank calls it per check
      if (hstatus != 0) break;
      if (gmax <= op.tolerance) {
        // converged: keep g2[cur] = log_v_k; discard the k+1 sweep
        break;
      }
      cur ^= 1;
      have_next = true;
    }
  }
  if (timed) CK(cudaEventRecord(ev1, st));
  // ---- tail: residual + stable E0 in one column pass (batch.py:323-337) ----
  S.est = allow_est && iters >= kEstFromIter;
  if (!small && !L.fused && !L.gemm) {   // the fused / GEMM passes produced the tail terms
    if (int e = S.tail(cur)) return e;
  }
  if (small) {
    if (out_residuals)
      CK(cudaMemcpyAsync(out_residuals, S.F(L.res), (size_t)pr.B * 4, cudaMemcpyDeviceToDevice,
                         st));
  } else {
    const int nb = (int)((pr.B + 31) / 32);
    const long long sb = L.tiled ? 1 : L.D2p, sj = L.tiled ? L.Bp : 1;
    ++g_launches;
    if (L.gemm) {
      if (int e = S.gemm_e0(out_cost)) return e;
    } else if (L.fused)   // per-row E0 terms of the fused passes
      e0_rows_finalize_kernel<<<(unsigned)((pr.B + 7) / 8), 256, 0, st>>>(
          S.F(L.e0), (int)pr.B, (int)pr.d1, L.D1p, out_cost, status);
    else if (sj == 1)   // per-column E0 terms of the tail pass, lane-major
      e0_finalize_rows_kernel<<<(unsigned)((pr.B + 7) / 8), 256, 0, st>>>(
          S.F(L.e0), (int)pr.B, (int)pr.d2, sb, out_cost, status, 0);
    else
      e0_finalize_kernel<<<nb, 256, 0, st>>>(S.F(L.e0), (int)pr.B, (int)pr.d2, sb, sj, out_cost,
                                             status, 0);
    dim3 gu((unsigned)((pr.d1 + 31) / 32), (unsigned)((pr.B + 31) / 32));
    ++g_launches;
    export_potential_kernel<<<gu, 256, 0, st>>>(S.F(L.f2), (int)pr.B, (int)pr.d1, L.sb1, L.si1,
                                                out_log_u, status, kLn2);
    dim3 gv((unsigned)((pr.d2 + 31) / 32), (unsigned)((pr.B + 31) / 32));
    ++g_launches;
    export_potential_kernel<<<gv, 256, 0, st>>>(S.F(L.g2[cur]), (int)pr.B, (int)pr.d2, L.sb2,
                                                L.si2, out_log_v, status, kLn2);
    CK(cudaGetLastError());
    if (out_residuals)
      CK(cudaMemcpyAsync(out_residuals, S.F(L.res), (size_t)pr.B * 4, cudaMemcpyDeviceToDevice,
                         st));
  }
  if (out_iterations) *out_iterations = iters;
  if (force_rerun_diag && allow_est && (L.tiled || L.fused || L.gemm)) {   // diagnostics
    ++g_launches;
    fill_int_kernel<<<1, 32, 0, st>>>(S.est_fail, 1, 1);
    CK(cudaGetLastError());
  }
  if (capturing) {   // the rerun body reports its own status word
    ++g_launches;
    async_status_kernel<<<1, 1, 0, st>>>(at<int>(ws, L.status), device_status);
    CK(cudaGetLastError());
    return 0;
  }
  if (device_status)
    return enqueue_async_tail(pr, op, mu, nu, cost, out_cost, out_log_u, out_log_v,
                              out_residuals, ws, ws_bytes, st, init_log_u, device_status,
                              at<int>(ws, L.status), S.est_fail,
                              allow_est && (L.tiled || L.fused || L.gemm));
  int hstatus = 0;
  if (int e = S.read_status(&hstatus)) return e;
  static const bool no_rerun = getenv("SKB_NO_RERUN") != nullptr;   // diagnostics
  if (allow_est) {
    int hfail = 0;
    if ((L.tiled || L.fused || L.gemm) && !no_rerun)
      CK(cudaMemcpy(&hfail, S.est_fail, 4, cudaMemcpyDeviceToHost));
    // With a reducer installed (batch-sharded solves) the rerun is decided
    // across ranks: every rank's first attempt calls the reducer here once,
    // whatever its path, and all ranks rerun if any rank's estimate failed --
    // the reruns' stopping tests then call the reducer in step on every rank.
    if (g_reducer) hfail = g_reducer(hfail ? 1.0 : 0.0, g_reducer_user) > 0.0 ? 1 : 0;
    if (hfail && g_allreduce) {   // row shards: the caller reruns the exact log-domain shards
      if (timed) {
        cudaEventDestroy(ev0);
        cudaEventDestroy(ev1);
      }
      return fail(SINKHORN_STATUS_EXACT_NEEDED,
                  "row-sharded GEMM solve: a guard fired (sums below 2^-60); rerun exactly");
    }
    if (hfail) {   // an estimate overshot: recompute the whole solve exactly
      ++g_exact_reruns;
      if (timed) {
        cudaEventDestroy(ev0);
        cudaEventDestroy(ev1);
      }
      return forward_impl(pr, op, mu, nu, cost, out_cost, out_log_u, out_log_v, out_iterations,
                          out_residuals, ws, ws_bytes, st, false, init_log_u);
    }
  }
  static const bool stats = getenv("SKB_SEP_STATS") != nullptr;   // diagnostics
  if (stats && L.sep) {
    unsigned int redo = 0;
    cudaMemcpy(&redo, at<unsigned int>(ws, L.scratch + 48), 4, cudaMemcpyDeviceToHost);
    fprintf(stderr, "[skb] separable estimate redos: %u thread tiles\n", redo);
  }
  if (timed) {
    float ms = -1.f;
    cudaEventElapsedTime(&ms, ev0, ev1);
    g_last_loop_ms = ms;
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
  }
  if (g_kt.on) {   // the stream was synchronised by read_status
    float tot = 0.f;
    for (size_t k = 0; k + 1 < g_kt.ev.size(); k += 2) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, g_kt.ev[k], g_kt.ev[k + 1]) == cudaSuccess) tot += ms;
    }
    g_kt.last_ms = tot;
    g_kt.last_launches = (int)(g_kt.ev.size() / 2);
    for (cudaEvent_t e : g_kt.ev) cudaEventDestroy(e);
    g_kt.ev.clear();
    g_kt.on = false;
  }
  if (hstatus == 11) {
    int row = 0;
    cudaMemcpy(&row, badrow, 4, cudaMemcpyDeviceToHost);
    return fail(11, "invalid histogram in row " + std::to_string(row));
  }
  if (hstatus != 0) return fail(hstatus, "device status " + std::to_string(hstatus));
  return 0;
}

// Point clouds -> the materialised (d1, d2) cost at the front of the workspace.
// Returns the cost pointer through *cost_out and the workspace after it.
int materialize_points(const sinkhorn_problem_v1& pr, const float* pts, void* ws, size_t ws_bytes,
                       cudaStream_t st, const float** cost_out, void** ws_rest,
                       size_t* ws_rest_bytes) {
  const DeviceInfo di = device_info();
  const PointLayout P = point_layout(pr, di.sms);
  if (ws == nullptr || ws_bytes < P.total) return fail(SINKHORN_STATUS_WORKSPACE, "workspace too small");
  const int D = pr.grid_nx, d1 = (int)pr.d1, d2 = (int)pr.d2;
  const float* x = pts;
  const float* y = pts + (size_t)d1 * D;
  float* C = at<float>(ws, P.cost);
  float* nrm = at<float>(ws, P.nrm);
  // a non-finite point makes its cost entries NaN, which the shared-cost
  // solve's cost validation reports as status 15 (core.py:53-63)
  ++g_launches;
  points_norms_kernel<<<grid_for((size_t)(d1 + d2)), 256, 0, st>>>(pts, d1 + d2, D, nrm);
  ++g_launches;
  points_tile_a_kernel<<<grid_for((size_t)round_up(d2, kUmBM) * P.kch * kUmBK), 256, 0, st>>>(
      y, d2, D, P.kch, at<float>(ws, P.ya));
  ++g_launches;
  umma_split_kernel<<<grid_for((size_t)round_up(d1, kUmBN) * P.kch * kUmBK), 256, 0, st>>>(
      x, d1, D, P.kch, at<float>(ws, P.xh), at<float>(ws, P.xl));
  CK(cudaGetLastError());
  CUtensorMap ta, tbh, tbl;
  const size_t mt = (size_t)round_up(d2, kUmBM) / kUmBM, nt = (size_t)round_up(d1, kUmBN) / kUmBN;
  const size_t sub = (size_t)P.kch * kUmSub;
  bool ok = make_tmap_sw128(&ta, at<float>(ws, P.ya), mt * sub * kUmBM, 32, 32, kUmBM);
  ok &= make_tmap_sw128(&tbh, at<float>(ws, P.xh), nt * sub * kUmBN, 32, 32, kUmBN);
  ok &= make_tmap_sw128(&tbl, at<float>(ws, P.xl), nt * sub * kUmBN, 32, 32, kUmBN);
  if (!ok) return fail(SINKHORN_STATUS_CUDA_ERROR, "cuTensorMapEncodeTiled failed (points)");
  // dot[i][j] = y_j . x_i: M = d2 (rows of A = y), N = d1 (x as the lane operand),
  // out[n * ldo + m] with ldo = d2 is the row-major (d1, d2) matrix
  UmmaParams p = {};
  p.M = d2;
  p.N = d1;
  p.K = D;
  p.MT = (int)mt;
  p.NT = (int)nt;
  p.KCH = (int)P.kch;
  p.units = (long long)p.MT * p.NT * p.KCH;
  p.G = (int)std::min<long long>(di.sms, p.units);
  p.out = C;
  p.ldo = d2;
  p.part = at<float>(ws, P.part);
  p.status = nullptr;
  if (int e = set_max_smem(reinterpret_cast<const void*>(&umma_gemm_kernel<false>), kUmSmemBytes)) return e;
  g_launches += 2;
  CK(launch_pdl(umma_gemm_kernel<false>, dim3(p.G), dim3(kUmThreads), kUmSmemBytes, st, ta, tbh, tbl, p));
  CK(launch_pdl(umma_fixup_kernel, dim3((unsigned)p.G), dim3(256), 0, st, p));
  ++g_launches;
  points_cost_kernel<<<grid_for((size_t)d1 * d2), 256, 0, st>>>(C, nrm, nrm + d1, d1, d2);
  CK(cudaGetLastError());
  *cost_out = C;
  *ws_rest = at<char>(ws, P.total);
  *ws_rest_bytes = ws_bytes - P.total;
  return 0;
}

// ---- asynchronous solves (SINKHORN_FLAG_ASYNC, tolerance 0) ------------------
// The tail of an asynchronous forward is one graph launch: a gate kernel sets
// a conditional node from the estimate guard (est_fail) and the status word;
// the node's body is the whole exact solve (allow_est = false), captured once
// per (workspace, pointers, problem, options) and replayed; a last kernel
// copies the status word to the caller's device int.  So the rerun decision
// (batch.py semantics are unchanged: the exact solve replaces the estimate
// one) never waits on the host.
struct AsyncGraphKey {   // the slot: workspace + problem + options (pointers may change)
  const void* ws;
  int64_t B, d1, d2;
  int32_t kind, max_iters, flags, dev;
  double lambda;
  size_t ws_bytes;
  bool operator==(const AsyncGraphKey& o) const {
    return ws == o.ws && B == o.B && d1 == o.d1 && d2 == o.d2 && kind == o.kind &&
           max_iters == o.max_iters && flags == o.flags && dev == o.dev && lambda == o.lambda &&
           ws_bytes == o.ws_bytes;
  }
};
struct AsyncGraph {
  AsyncGraphKey key;
  const void* ptrs[9] = {};   // the buffers the captured rerun body reads / writes
  cudaGraphExec_t exec = nullptr;
  unsigned long long used = 0;
};
thread_local std::vector<AsyncGraph> g_async_graphs;
thread_local unsigned long long g_async_clock = 0;

// Parent graph of an asynchronous solve's tail: gate -> status copy ->
// IF(guard fired) { exact solve }.
int build_async_graph(cudaGraph_t* out, const sinkhorn_problem_v1& pr,
                      const sinkhorn_options_v1& op, const float* mu, const float* nu,
                      const float* cost, float* out_cost, float* out_log_u, float* out_log_v,
                      float* out_residuals, void* ws, size_t ws_bytes, const float* init_log_u,
                      int32_t* device_status, const int* ws_status, const int* est_fail,
                      int dev) {
  cudaGraph_t parent = nullptr;
  CK(cudaGraphCreate(&parent, 0));
  cudaGraphConditionalHandle h;
  CK(cudaGraphConditionalHandleCreate(&h, parent, 0, cudaGraphCondAssignDefault));
  cudaGraphNode_t gate, fin, cond;
  {
    void* args[3] = {&h, const_cast<int**>(&est_fail), const_cast<int**>(&ws_status)};
    cudaKernelNodeParams kp = {};
    kp.func = reinterpret_cast<void*>(&async_gate_kernel);
    kp.gridDim = dim3(1);
    kp.blockDim = dim3(1);
    kp.kernelParams = args;
    CK(cudaGraphAddKernelNode(&gate, parent, nullptr, 0, &kp));
  }
  {   // the fast solve's status first; a rerun overwrites it with its own
    void* args[2] = {const_cast<int**>(&ws_status), &device_status};
    cudaKernelNodeParams kp = {};
    kp.func = reinterpret_cast<void*>(&async_status_kernel);
    kp.gridDim = dim3(1);
    kp.blockDim = dim3(1);
    kp.kernelParams = args;
    CK(cudaGraphAddKernelNode(&fin, parent, &gate, 1, &kp));
  }
  cudaGraphNodeParams cp = {};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeIf;
  cp.conditional.size = 1;
  CK(cudaGraphAddNode(&cond, parent, &fin, 1, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  static thread_local cudaStream_t cs_dev[64] = {};
  if (dev < 0 || dev >= 64) return fail(SINKHORN_STATUS_CUDA_ERROR, "device ordinal");
  cudaStream_t& cs = cs_dev[dev];
  if (cs == nullptr) CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
  const unsigned long long l0 = g_launches;
  CK(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  sinkhorn_options_v1 exact = op;
  exact.flags &= ~SINKHORN_FLAG_FORCE_RERUN;
  int32_t it = 0;
  const char* fast_path = g_last_path;   // the capture is not a solve of its own
  const int e = forward_impl(pr, exact, mu, nu, cost, out_cost, out_log_u, out_log_v, &it,
                             out_residuals, ws, ws_bytes, cs, false, init_log_u, device_status,
                             true);
  cudaGraph_t captured = nullptr;
  const cudaError_t ce = cudaStreamEndCapture(cs, &captured);
  g_last_path = fast_path;
  g_launches = l0;
  if (e) return e;
  CK(ce);
  *out = parent;
  return 0;
}

int enqueue_async_tail(const sinkhorn_problem_v1& pr, const sinkhorn_options_v1& op,
                       const float* mu, const float* nu, const float* cost, float* out_cost,
                       float* out_log_u, float* out_log_v, float* out_residuals, void* ws,
                       size_t ws_bytes, cudaStream_t st, const float* init_log_u,
                       int32_t* device_status, const int* ws_status, const int* est_fail,
                       bool can_fail) {
  if (!can_fail) {   // no estimate guard on this path: only the status copy
    ++g_launches;
    async_status_kernel<<<1, 1, 0, st>>>(ws_status, device_status);
    CK(cudaGetLastError());
    return 0;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  const AsyncGraphKey k = {ws, pr.B, pr.d1, pr.d2, pr.cost_kind, op.max_iters,
                           (int32_t)op.flags, dev, op.lambda, ws_bytes};
  const void* ptrs[9] = {mu, nu, cost, out_cost, out_log_u, out_log_v, out_residuals, init_log_u,
                         device_status};
  ++g_async_clock;
  // an exact (problem, buffers) match replays as is
  AsyncGraph* ag = nullptr;
  for (auto& g : g_async_graphs)
    if (g.key == k && std::equal(ptrs, ptrs + 9, g.ptrs)) ag = &g;
  if (ag == nullptr) {
    // same problem, other buffers: update that entry in place (capture + update
    // cost ~1 ms of host time; instantiating costs tens)
    for (auto& g : g_async_graphs)
      if (g.key == k && (ag == nullptr || g.used < ag->used)) ag = &g;
  }
  if (ag == nullptr) {
    if (g_async_graphs.size() >= 8) {   // recycle the least recently used entry
      ag = &*std::min_element(g_async_graphs.begin(), g_async_graphs.end(),
                              [](const AsyncGraph& a, const AsyncGraph& b) { return a.used < b.used; });
      if (ag->exec) {   // a different problem: new topology
        cudaGraphExecDestroy(ag->exec);
        ag->exec = nullptr;
      }
    } else {
      g_async_graphs.push_back(AsyncGraph{});
      ag = &g_async_graphs.back();
    }
  }
  if (!std::equal(ptrs, ptrs + 9, ag->ptrs) || ag->exec == nullptr) {
    ag->key = k;
    // new buffers: capture the tail; update an executable graph of the same
    // problem in place (cheaper than instantiating), else instantiate
    cudaGraph_t parent = nullptr;
    if (int e = build_async_graph(&parent, pr, op, mu, nu, cost, out_cost, out_log_u, out_log_v,
                                  out_residuals, ws, ws_bytes, init_log_u, device_status,
                                  ws_status, est_fail, dev))
      return e;
    bool updated = false;
    if (ag->exec != nullptr) {
      cudaGraphExecUpdateResultInfo info = {};
      updated = cudaGraphExecUpdate(ag->exec, parent, &info) == cudaSuccess;
      if (!updated) {
        cudaGetLastError();
        cudaGraphExecDestroy(ag->exec);
        ag->exec = nullptr;
      }
    }
    if (!updated) CK(cudaGraphInstantiate(&ag->exec, parent, 0));
    CK(cudaGraphDestroy(parent));
    std::copy(ptrs, ptrs + 9, ag->ptrs);
  }
  ag->used = g_async_clock;
  CK(cudaGraphLaunch(ag->exec, st));
  g_launches += 2;   // gate + status copy (the conditional body only runs when a guard fired)
  return 0;
}

}  // namespace

// =============================================================================
// C ABI (the only symbols the library exports; built with -fvisibility=hidden)
// =============================================================================
#pragma GCC visibility push(default)
extern "C" {

const char* sinkhorn_last_error(void) { return g_last_error.c_str(); }

const char* sinkhorn_version(void) { return "paper_1907_01729_b200 0.1.0 sm_100a"; }

unsigned long long sinkhorn_launch_count_v1(void) { return g_launches; }

unsigned long long sinkhorn_exact_reruns_v1(void) { return g_exact_reruns; }

float sinkhorn_last_loop_ms_v1(void) { return g_last_loop_ms; }
float sinkhorn_last_kernel_ms_v1(int32_t* launches) {
  if (launches) *launches = g_kt.last_launches;
  return g_kt.last_ms;
}

const char* sinkhorn_last_path_v1(void) { return g_last_path; }

size_t sinkhorn_workspace_bytes_v1(const sinkhorn_problem_v1* prob) {
  if (check_problem(prob) != 0) return 0;
  return workspace_total(*prob, device_info().sms);
}

int32_t sinkhorn_forward_device_v1(const sinkhorn_problem_v1* prob,
                                   const sinkhorn_options_v1* opt, const float* mu,
                                   const float* nu, const float* cost, float* out_cost,
                                   float* out_log_u, float* out_log_v, int32_t* out_iterations,
                                   float* out_residuals, void* workspace,
                                   size_t workspace_bytes, void* stream) {
  if (int e = check_problem(prob)) return e;
  if (prob->B == 0) {   // ffi.ts:107-109
    if (out_iterations) *out_iterations = 0;
    return 0;
  }
  if (prob->d1 == 0 || prob->d2 == 0)
    return fail(SINKHORN_STATUS_INVALID_HISTOGRAM, "empty histogram cannot sum to 1");
  if (int e = check_options(opt)) return e;
  if (!mu || !nu || !out_cost || !out_log_u || !out_log_v ||
      (prob->cost_kind != SINKHORN_COST_GRID2D && !cost))
    return fail(SINKHORN_STATUS_BAD_ARGUMENT, "null pointer");
  sinkhorn_problem_v1 pr = *prob;
  if (pr.cost_kind == SINKHORN_COST_POINTS) {   // materialise, then a shared stored cost
    if (int e = materialize_points(pr, cost, workspace, workspace_bytes,
                                   static_cast<cudaStream_t>(stream), &cost, &workspace,
                                   &workspace_bytes))
      return e;
    pr = as_shared(pr);
  }
  return forward_impl(pr, *opt, mu, nu, cost, out_cost, out_log_u, out_log_v, out_iterations,
                      out_residuals, workspace, workspace_bytes,
                      static_cast<cudaStream_t>(stream),
                      (opt->flags & SINKHORN_FLAG_EXACT_MAX) == 0);
}

int32_t sinkhorn_forward_async_device_v1(const sinkhorn_problem_v1* prob,
                                         const sinkhorn_options_v1* opt, const float* mu,
                                         const float* nu, const float* cost, float* out_cost,
                                         float* out_log_u, float* out_log_v,
                                         float* out_residuals, int32_t* device_status,
                                         void* workspace, size_t workspace_bytes, void* stream) {
  if (int e = check_problem(prob)) return e;
  if (int e = check_options(opt)) return e;
  if (opt->tolerance != 0.0)
    return fail(SINKHORN_STATUS_INVALID_CONFIG,
                "asynchronous solves need tolerance 0 (a stopping test is a host decision)");
  if (!device_status) return fail(SINKHORN_STATUS_BAD_ARGUMENT, "null device status");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (prob->B == 0) {   // ffi.ts:107-109
    CK(cudaMemsetAsync(device_status, 0, 4, st));
    return 0;
  }
  if (prob->d1 == 0 || prob->d2 == 0)
    return fail(SINKHORN_STATUS_INVALID_HISTOGRAM, "empty histogram cannot sum to 1");
  if (!mu || !nu || !out_cost || !out_log_u || !out_log_v ||
      (prob->cost_kind != SINKHORN_COST_GRID2D && !cost))
    return fail(SINKHORN_STATUS_BAD_ARGUMENT, "null pointer");
  sinkhorn_options_v1 op = *opt;
  op.flags &= ~(SINKHORN_FLAG_TIME_LOOP | SINKHORN_FLAG_TIME_KERNEL | SINKHORN_FLAG_PERSISTENT);
  int32_t iters = 0;
  sinkhorn_problem_v1 pr = *prob;
  if (pr.cost_kind == SINKHORN_COST_POINTS) {
    if (int e = materialize_points(pr, cost, workspace, workspace_bytes, st, &cost, &workspace,
                                   &workspace_bytes))
      return e;
    pr = as_shared(pr);
  }
  return forward_impl(pr, op, mu, nu, cost, out_cost, out_log_u, out_log_v, &iters,
                      out_residuals, workspace, workspace_bytes, st,
                      (op.flags & SINKHORN_FLAG_EXACT_MAX) == 0, nullptr, device_status);
}

int32_t sinkhorn_forward_rows_device_v1(const sinkhorn_problem_v1* prob,
                                        const sinkhorn_options_v1* opt, const float* mu_rows,
                                        const float* nu, const float* cost_rows,
                                        float* out_cost, float* out_log_u_rows, float* out_log_v,
                                        int32_t* out_iterations, float* out_residuals,
                                        sinkhorn_allreduce_v1 allreduce, void* user,
                                        void* workspace, size_t workspace_bytes, void* stream) {
  if (int e = check_problem(prob)) return e;
  if (prob->cost_kind != SINKHORN_COST_SHARED)
    return fail(SINKHORN_STATUS_BAD_ARGUMENT, "row sharding needs a stored shared cost");
  if (prob->B == 0) {
    if (out_iterations) *out_iterations = 0;
    return 0;
  }
  if (prob->d2 == 0) return fail(SINKHORN_STATUS_INVALID_HISTOGRAM, "empty histogram");
  if (int e = check_options(opt)) return e;
  if (!mu_rows || !nu || !cost_rows || !out_cost || !out_log_u_rows || !out_log_v || !allreduce)
    return fail(SINKHORN_STATUS_BAD_ARGUMENT, "null pointer");
  sinkhorn_options_v1 op = *opt;
  // the GEMM iteration, no single-launch solver; the caller validates the
  // histograms globally (a rank's slice of mu does not sum to 1)
  op.flags |= SINKHORN_FLAG_FORCE_GEMM | SINKHORN_FLAG_TILED_ONLY | SINKHORN_FLAG_SKIP_VALIDATION;
  op.flags &= ~(SINKHORN_FLAG_NO_GEMM | SINKHORN_FLAG_EXACT_MAX);
  g_allreduce = allreduce;
  g_allreduce_user = user;
  const int rc = forward_impl(*prob, op, mu_rows, nu, cost_rows, out_cost, out_log_u_rows,
                              out_log_v, out_iterations, out_residuals, workspace, workspace_bytes,
                              static_cast<cudaStream_t>(stream), true);
  g_allreduce = nullptr;
  g_allreduce_user = nullptr;
  return rc;
}

int32_t sinkhorn_forward_warm_device_v1(const sinkhorn_problem_v1* prob,
                                   const sinkhorn_options_v1* opt, const float* mu,
                                   const float* nu, const float* cost, const float* init_log_u,
                                   float* out_cost,
                                   float* out_log_u, float* out_log_v, int32_t* out_iterations,
                                   float* out_residuals, void* workspace,
                                   size_t workspace_bytes, void* stream) {
  if (int e = check_problem(prob)) return e;
  if (prob->B == 0) {   // ffi.ts:107-109
    if (out_iterations) *out_iterations = 0;
    return 0;
  }
  if (prob->d1 == 0 || prob->d2 == 0)
    return fail(SINKHORN_STATUS_INVALID_HISTOGRAM, "empty histogram cannot sum to 1");
  if (int e = check_options(opt)) return e;
  if (!mu || !nu || !out_cost || !out_log_u || !out_log_v ||
      (prob->cost_kind != SINKHORN_COST_GRID2D && !cost))
    return fail(SINKHORN_STATUS_BAD_ARGUMENT, "null pointer");
  sinkhorn_problem_v1 pr = *prob;
  if (pr.cost_kind == SINKHORN_COST_POINTS) {
    if (int e = materialize_points(pr, cost, workspace, workspace_bytes,
                                   static_cast<cudaStream_t>(stream), &cost, &workspace,
                                   &workspace_bytes))
      return e;
    pr = as_shared(pr);
  }
  return forward_impl(pr, *opt, mu, nu, cost, out_cost, out_log_u, out_log_v, out_iterations,
                      out_residuals, workspace, workspace_bytes,
                      static_cast<cudaStream_t>(stream),
                      (opt->flags & SINKHORN_FLAG_EXACT_MAX) == 0, init_log_u);
}


extern "C++" {
namespace {
template <typename T>
int backward_device(int64_t B, int64_t d1, int64_t d2, double lambda, const T* log_u,
                    const T* log_v, const T* upstream, T* out_grad_mu, T* out_grad_nu,
                    int32_t* out_zero_mass_lane, void* workspace, size_t workspace_bytes,
                    void* stream) {
  if (B < 0 || d1 < 0 || d2 < 0) return fail(SINKHORN_STATUS_SHAPE_MISMATCH, "negative extent");
  if (B == 0) return 0;
  if (!log_u || !log_v || !upstream || !out_grad_mu || !out_grad_nu || !workspace)
    return fail(SINKHORN_STATUS_BAD_ARGUMENT, "null pointer");
  if (workspace_bytes < 8) return fail(SINKHORN_STATUS_WORKSPACE, "backward needs 8 bytes");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int* status = static_cast<int*>(workspace);
  int* bad = status + 1;
  CK(cudaMemsetAsync(status, 0, 4, st));
  CK(cudaMemsetAsync(bad, 0x7f, 4, st));
  ++g_launches;
  backward_kernel<T><<<dim3((unsigned)B, 2), 256, 0, st>>>(
      log_u, log_v, (int)d1, (int)d2, lambda, upstream, out_grad_mu, out_grad_nu, status, bad);
  CK(cudaGetLastError());
  int h[2] = {0, 0};
  CK(cudaMemcpyAsync(h, status, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (h[0] == SINKHORN_STATUS_ZERO_MASS_LANE) {
    if (out_zero_mass_lane) *out_zero_mass_lane = h[1];
    return fail(SINKHORN_STATUS_ZERO_MASS_LANE, "zero-mass bin in lane " + std::to_string(h[1]));
  }
  return h[0];
}

// ---- float64 parity mode (sweep_f64.cuh) ----------------------------------
struct F64Layout {
  size_t a = 0, at = 0, lmu = 0, lnu = 0, u = 0, v = 0, rrow = 0, rcol = 0, e0 = 0, res = 0;
  size_t status = 0, total = 0;
};

F64Layout f64_layout(const sinkhorn_problem_v1& pr) {
  F64Layout L;
  Carver c;
  const size_t lanes = pr.cost_kind == SINKHORN_COST_PER_SAMPLE ? (size_t)pr.B : 1;
  const size_t n1 = (size_t)pr.B * pr.d1 * 8, n2 = (size_t)pr.B * pr.d2 * 8;
  L.a = c.take(lanes * pr.d1 * pr.d2 * 8);
  L.at = c.take(lanes * pr.d1 * pr.d2 * 8);
  L.lmu = c.take(n1);
  L.u = c.take(n1);
  L.rrow = c.take(n1);
  L.lnu = c.take(n2);
  L.v = c.take(n2);
  L.rcol = c.take(n2);
  L.e0 = c.take(n2);
  L.res = c.take((size_t)pr.B * 8);
  L.status = c.take(8);
  L.total = c.off;
  return L;
}

int forward_f64_impl(const sinkhorn_problem_v1& pr, const sinkhorn_options_v1& op, const double* mu,
                     const double* nu, const double* cost, double* out_cost, double* out_log_u,
                     double* out_log_v, int32_t* out_iterations, double* out_residuals, void* ws,
                     size_t ws_bytes, cudaStream_t st) {
  const F64Layout L = f64_layout(pr);
  if (ws == nullptr || ws_bytes < L.total) return fail(SINKHORN_STATUS_WORKSPACE, "workspace too small");
  auto D = [&](size_t off) { return at<double>(ws, off); };
  int* status = at<int>(ws, L.status);
  int* badrow = status + 1;
  const int B = (int)pr.B, d1 = (int)pr.d1, d2 = (int)pr.d2;
  const bool per_sample = pr.cost_kind == SINKHORN_COST_PER_SAMPLE;
  g_last_path = "fp64";
  CK(cudaMemsetAsync(status, 0, 4, st));
  CK(cudaMemsetAsync(badrow, 0x7f, 4, st));
  if (!(op.flags & SINKHORN_FLAG_SKIP_VALIDATION)) {
    ++g_launches;
    validate_rows_kernel<double><<<(unsigned)B, 256, 0, st>>>(mu, d1, status, badrow);
    ++g_launches;
    validate_rows_kernel<double><<<(unsigned)B, 256, 0, st>>>(nu, d2, status, badrow);
  }
  ++g_launches;
  f64_prep_kernel<<<grid_for((size_t)B * (d1 + d2)), 256, 0, st>>>(mu, nu, B, d1, d2, D(L.lmu),
                                                                    D(L.lnu), D(L.u), D(L.v));
  {
    dim3 g((unsigned)((d2 + 31) / 32), (unsigned)((d1 + 31) / 32),
           per_sample ? lanes_in_launch(B, 0) : 1u);   // the kernel strides over the rest
    ++g_launches;
    f64_cost_kernel<<<g, 256, 0, st>>>(pr.cost_kind == SINKHORN_COST_GRID2D ? nullptr : cost,
                                       per_sample ? B : 1, d1, d2, op.lambda, (int)pr.grid_nx,
                                       (double)pr.grid_hx * pr.grid_hx,
                                       (double)pr.grid_hy * pr.grid_hy, D(L.a), D(L.at), status);
  }
  CK(cudaGetLastError());
  const long long lane_cells = per_sample ? (long long)d1 * d2 : 0;
  auto sweep = [&](int mode, bool col, double* out, const double* pot, const double* marg) -> int {
    F64SweepParams p = {};
    p.B = B;
    p.P = col ? d2 : d1;
    p.Q = col ? d1 : d2;
    p.G = col ? D(L.at) : D(L.a);
    p.g_lane = lane_cells;
    p.x = col ? D(L.u) : D(L.v);
    p.target = col ? D(L.lnu) : D(L.lmu);
    p.out = out;
    p.pot = pot;
    p.marg = marg;
    p.lam = op.lambda;
    p.status = status;
    for (long long b0 = 0; b0 < B; b0 += kMaxLanesPerLaunch) {
      p.b0 = (int)b0;
      dim3 g((unsigned)((p.P + 7) / 8), lanes_in_launch(B, b0));
      ++g_launches;
      if (mode == kF64Update) f64_sweep_kernel<kF64Update><<<g, 256, 0, st>>>(p);
      else if (mode == kF64Residual) f64_sweep_kernel<kF64Residual><<<g, 256, 0, st>>>(p);
      else f64_sweep_kernel<kF64E0><<<g, 256, 0, st>>>(p);
      CK(cudaGetLastError());
    }
    return 0;
  };
  // lane_residuals (batch.py:303-309): row term with A, column term with A^T
  auto residuals = [&]() -> int {
    if (int e = sweep(kF64Residual, false, D(L.rrow), D(L.u), mu)) return e;
    if (int e = sweep(kF64Residual, true, D(L.rcol), D(L.v), nu)) return e;
    ++g_launches;
    f64_lane_reduce_kernel<<<(unsigned)((B + 7) / 8), 256, 0, st>>>(D(L.rrow), d1, D(L.rcol), d2, B,
                                                                    D(L.res), 0);
    CK(cudaGetLastError());
    return 0;
  };
  // ---- lockstep iteration (batch.py:314-324) ----
  int iters = 0;
  bool have_res = false, converged = false;
  std::vector<double> hres((size_t)B);
  for (int k = 1; k <= op.max_iters; ++k) {
    if (int e = sweep(kF64Update, true, D(L.v), nullptr, nullptr)) return e;    // v first
    if (int e = sweep(kF64Update, false, D(L.u), nullptr, nullptr)) return e;   // then u
    iters = k;
    if (op.tolerance > 0 && k % op.check_interval == 0) {
      if (int e = residuals()) return e;
      have_res = true;
      int hstatus = 0;
      CK(cudaMemcpyAsync(hres.data(), D(L.res), (size_t)B * 8, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(&hstatus, status, 4, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      double gmax = 0.0;
      for (double r : hres) gmax = (r != r || gmax != gmax) ? NAN : std::max(gmax, r);
      if (hstatus != 0) gmax = NAN;
      if (g_reducer) gmax = g_reducer(gmax, g_reducer_user);
      if (hstatus != 0) break;
      if (gmax <= op.tolerance) {
        converged = true;
        break;
      }
    }
  }
  if (!have_res || !converged) {
    if (int e = residuals()) return e;
  }
  ++g_launches;
  f64_nan_kernel<<<grid_for((size_t)B * (d1 + d2)), 256, 0, st>>>(D(L.u), (size_t)B * d1, D(L.v),
                                                                  (size_t)B * d2, status);
  // stable E0 (batch.py:329-337)
  if (int e = sweep(kF64E0, true, D(L.e0), D(L.v), nullptr)) return e;
  ++g_launches;
  f64_lane_reduce_kernel<<<(unsigned)((B + 7) / 8), 256, 0, st>>>(D(L.e0), d2, nullptr, 0, B,
                                                                  out_cost, 1);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out_log_u, D(L.u), (size_t)B * d1 * 8, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(out_log_v, D(L.v), (size_t)B * d2 * 8, cudaMemcpyDeviceToDevice, st));
  if (out_residuals)
    CK(cudaMemcpyAsync(out_residuals, D(L.res), (size_t)B * 8, cudaMemcpyDeviceToDevice, st));
  if (out_iterations) *out_iterations = iters;
  int h[2] = {0, 0};
  CK(cudaMemcpyAsync(h, status, 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (h[0] == SINKHORN_STATUS_INVALID_HISTOGRAM)
    return fail(h[0], "invalid histogram (row " + std::to_string(h[1]) + ")");
  if (h[0] == SINKHORN_STATUS_INVALID_COST) return fail(h[0], "cost must be finite and >= 0");
  if (h[0] == SINKHORN_STATUS_NON_FINITE_OUTPUT) return fail(h[0], "NaN in batched solver state");
  return h[0];
}
}  // namespace
}  // extern "C++"

int32_t sinkhorn_backward_device_v1(int64_t B, int64_t d1, int64_t d2, double lambda,
                                    const float* log_u, const float* log_v,
                                    const float* upstream, float* out_grad_mu,
                                    float* out_grad_nu, int32_t* out_zero_mass_lane,
                                    void* workspace, size_t workspace_bytes, void* stream) {
  return backward_device<float>(B, d1, d2, lambda, log_u, log_v, upstream, out_grad_mu,
                                out_grad_nu, out_zero_mass_lane, workspace, workspace_bytes, stream);
}

int32_t sinkhorn_backward_f64_device_v1(int64_t B, int64_t d1, int64_t d2, double lambda,
                                        const double* log_u, const double* log_v,
                                        const double* upstream, double* out_grad_mu,
                                        double* out_grad_nu, int32_t* out_zero_mass_lane,
                                        void* workspace, size_t workspace_bytes, void* stream) {
  return backward_device<double>(B, d1, d2, lambda, log_u, log_v, upstream, out_grad_mu,
                                 out_grad_nu, out_zero_mass_lane, workspace, workspace_bytes,
                                 stream);
}

size_t sinkhorn_workspace_bytes_f64_v1(const sinkhorn_problem_v1* prob) {
  if (check_problem(prob) != 0) return 0;
  return f64_layout(*prob).total;
}

int32_t sinkhorn_forward_f64_device_v1(const sinkhorn_problem_v1* prob,
                                       const sinkhorn_options_v1* opt, const double* mu,
                                       const double* nu, const double* cost, double* out_cost,
                                       double* out_log_u, double* out_log_v,
                                       int32_t* out_iterations, double* out_residuals,
                                       void* workspace, size_t workspace_bytes, void* stream) {
  if (int e = check_problem(prob)) return e;
  if (prob->cost_kind == SINKHORN_COST_POINTS)
    return fail(SINKHORN_STATUS_BAD_ARGUMENT, "the float64 mode takes stored or grid costs");
  if (prob->B == 0) {   // ffi.ts:107-109
    if (out_iterations) *out_iterations = 0;
    return 0;
  }
  if (prob->d1 == 0 || prob->d2 == 0)
    return fail(SINKHORN_STATUS_INVALID_HISTOGRAM, "empty histogram cannot sum to 1");
  if (int e = check_options(opt)) return e;
  if (!mu || !nu || !out_cost || !out_log_u || !out_log_v ||
      (prob->cost_kind != SINKHORN_COST_GRID2D && !cost))
    return fail(SINKHORN_STATUS_BAD_ARGUMENT, "null pointer");
  return forward_f64_impl(*prob, *opt, mu, nu, cost, out_cost, out_log_u, out_log_v,
                          out_iterations, out_residuals, workspace, workspace_bytes,
                          static_cast<cudaStream_t>(stream));
}

size_t sinkhorn_half_sweep_workspace_bytes_v1(int64_t B, int64_t d1, int64_t d2) {
  sinkhorn_problem_v1 pr = {B, d1, d2, SINKHORN_COST_SHARED, 0, 0, 0.f, 0.f};
  if (check_problem(&pr) != 0) return 0;
  return make_layout(pr, device_info().sms).total;
}

int32_t sinkhorn_half_sweep_device_v1(int64_t B, int64_t d1, int64_t d2, double lambda,
                                      const float* log_x, const float* cost,
                                      const float* target, float* out, float* out_max,
                                      float* out_sum, void* workspace, size_t workspace_bytes,
                                      void* stream) {
  sinkhorn_problem_v1 pr = {B, d1, d2, SINKHORN_COST_SHARED, 0, 0, 0.f, 0.f};
  if (int e = check_problem(&pr)) return e;
  if (B == 0 || d2 == 0) return 0;
  if (!(std::isfinite(lambda) && lambda > 0))
    return fail(SINKHORN_STATUS_INVALID_CONFIG, "lam must be positive and finite");
  const bool partial = (out_max != nullptr || out_sum != nullptr);
  if (!log_x || !cost || (partial ? (!out_max || !out_sum) : (!out || !target)))
    return fail(SINKHORN_STATUS_BAD_ARGUMENT, "null pointer");
  Solve S;
  S.pr = pr;
  S.di = device_info();
  S.L = make_layout(pr, S.di.sms);
  S.ws = workspace;
  S.st = static_cast<cudaStream_t>(stream);
  S.lam = (float)lambda;
  S.cost = cost;
  const Layout& L = S.L;
  if (workspace == nullptr || workspace_bytes < L.total)
    return fail(SINKHORN_STATUS_WORKSPACE, "workspace too small");
  cudaStream_t st = S.st;
  int* status = at<int>(workspace, L.status);
  CK(cudaMemsetAsync(status, 0, 4, st));
  CK(cudaMemsetAsync(at<int>(workspace, L.counters), 0,
                     std::max<size_t>(L.counter_count, 1) * 4, st));
  {
    dim3 g((unsigned)((L.D2p + 31) / 32), (unsigned)((L.D1p + 31) / 32));
    ++g_launches;
    prep_cost_kernel<<<g, 256, 0, st>>>(cost, (int)d1, (int)d2, L.D1p, L.D2p,
                                         (float)(-1.4426950408889634 / lambda), S.F(L.a2),
                                         S.F(L.a2t), status);
    dim3 gx((unsigned)((L.D1p + 31) / 32), (unsigned)((L.Bp + 31) / 32));
    ++g_launches;
    import_potential_kernel<<<gx, 256, 0, st>>>(log_x, (int)B, (int)d1, L.Bp, L.D1p, L.sb1,
                                                 L.si1, S.F(L.f2));
    if (!partial) {
      dim3 gt((unsigned)((L.D2p + 31) / 32), (unsigned)((L.Bp + 31) / 32));
      ++g_launches;
      import_potential_kernel<<<gt, 256, 0, st>>>(target, (int)B, (int)d2, L.Bp, L.D2p, L.sb2,
                                                   L.si2, S.F(L.l2nu));
    }
    CK(cudaGetLastError());
  }
  if (int e = S.setup_maps()) return e;
  TiledArgs a = {&S.tm_a2, &S.tm_f2, (int)d1, (int)d2, L.D1p, L.D2p, S.F(L.l2nu), S.F(L.nu),
                 S.F(L.g2[0]), nullptr, nullptr, kResNone, nullptr, S.F(L.g2[0]), S.F(L.g2[1])};
  if (partial) {
    if (int e = launch_tiled<false, kModePartial>(L, workspace, S.di, a, pr, S.lam, st)) return e;
  } else {
    if (int e = launch_tiled<false, kModeUpdate>(L, workspace, S.di, a, pr, S.lam, st)) return e;
  }
  dim3 gv((unsigned)((d2 + 31) / 32), (unsigned)((B + 31) / 32));
  if (partial) {
    ++g_launches;
    export_potential_kernel<<<gv, 256, 0, st>>>(S.F(L.g2[0]), (int)B, (int)d2, L.sb2, L.si2,
                                                out_max, status, 1.0f, 0);
    ++g_launches;
    export_potential_kernel<<<gv, 256, 0, st>>>(S.F(L.g2[1]), (int)B, (int)d2, L.sb2, L.si2,
                                                out_sum, status, 1.0f, 0);
  } else {
    ++g_launches;
    export_potential_kernel<<<gv, 256, 0, st>>>(S.F(L.g2[0]), (int)B, (int)d2, L.sb2, L.si2,
                                                out, status, kLn2, 0);
  }
  CK(cudaGetLastError());
  int h = 0;
  if (int e = S.read_status(&h)) return e;
  return h == 0 ? 0 : fail(h, "device status " + std::to_string(h));
}

// ---- dC on the tensor cores (shared costs) -------------------------------------
namespace {
struct PlanLayout {
  size_t va = 0, uh = 0, ul = 0, al = 0, be = 0, part = 0, total = 0;
  long long kch = 0;
};
PlanLayout plan_layout(const sinkhorn_problem_v1& pr, int sms) {
  PlanLayout P;
  Carver c;
  P.kch = (pr.B + kUmBK - 1) / kUmBK;
  P.va = c.take((size_t)round_up(pr.d2, kUmBM) * P.kch * kUmBK * 4);
  P.uh = c.take((size_t)round_up(pr.d1, kUmBN) * P.kch * kUmBK * 4);
  P.ul = c.take((size_t)round_up(pr.d1, kUmBN) * P.kch * kUmBK * 4);
  P.al = c.take((size_t)pr.d1 * 4);
  P.be = c.take((size_t)pr.d2 * 4);
  P.part = c.take((size_t)sms * 2 * kUmBN * kUmBM * 4);
  P.total = c.take(256);
  return P;
}

int plan_grad_umma(const sinkhorn_problem_v1& pr, double lambda, const float* log_u,
                   const float* log_v, const float* cost, const float* up, float* dc, void* ws,
                   size_t ws_bytes, cudaStream_t st) {
  const DeviceInfo di = device_info();
  const PlanLayout P = plan_layout(pr, di.sms);
  if (ws == nullptr || ws_bytes < P.total) return fail(SINKHORN_STATUS_WORKSPACE, "workspace too small");
  const int B = (int)pr.B, d1 = (int)pr.d1, d2 = (int)pr.d2;
  float* al = at<float>(ws, P.al);
  float* be = at<float>(ws, P.be);
  g_launches += 3;
  plan_lane_max_kernel<<<grid_for((size_t)d1), 256, 0, st>>>(log_u, B, d1, al);
  plan_lane_max_kernel<<<grid_for((size_t)d2), 256, 0, st>>>(log_v, B, d2, be);
  const size_t nop = (size_t)(round_up(d2, kUmBM) + round_up(d1, kUmBN)) * P.kch * kUmBK;
  plan_operands_kernel<<<grid_for(nop), 256, 0, st>>>(log_u, log_v, up, al, be, B, d1, d2, P.kch,
                                                      at<float>(ws, P.va), at<float>(ws, P.uh),
                                                      at<float>(ws, P.ul));
  CK(cudaGetLastError());
  CUtensorMap ta, tbh, tbl;
  const size_t mt = (size_t)round_up(d2, kUmBM) / kUmBM, nt = (size_t)round_up(d1, kUmBN) / kUmBN;
  const size_t sub = (size_t)P.kch * kUmSub;
  bool ok = make_tmap_sw128(&ta, at<float>(ws, P.va), mt * sub * kUmBM, 32, 32, kUmBM);
  ok &= make_tmap_sw128(&tbh, at<float>(ws, P.uh), nt * sub * kUmBN, 32, 32, kUmBN);
  ok &= make_tmap_sw128(&tbl, at<float>(ws, P.ul), nt * sub * kUmBN, 32, 32, kUmBN);
  if (!ok) return fail(SINKHORN_STATUS_CUDA_ERROR, "cuTensorMapEncodeTiled failed (plan)");
  UmmaParams p = {};   // S[i][j] = sum_b U_bi V_bj: M = d2 (A = V), N = d1 (lanes = U)
  p.M = d2;
  p.N = d1;
  p.K = B;
  p.MT = (int)mt;
  p.NT = (int)nt;
  p.KCH = (int)P.kch;
  p.units = (long long)p.MT * p.NT * p.KCH;
  p.G = (int)std::min<long long>(di.sms, p.units);
  p.out = dc;
  p.ldo = d2;
  p.part = at<float>(ws, P.part);
  p.status = nullptr;
  if (int e = set_max_smem(reinterpret_cast<const void*>(&umma_gemm_kernel<false>), kUmSmemBytes)) return e;
  g_launches += 3;
  CK(launch_pdl(umma_gemm_kernel<false>, dim3(p.G), dim3(kUmThreads), kUmSmemBytes, st, ta, tbh, tbl, p));
  CK(launch_pdl(umma_fixup_kernel, dim3((unsigned)p.G), dim3(256), 0, st, p));
  plan_finish_kernel<<<grid_for((size_t)d1 * d2), 256, 0, st>>>(
      dc, cost, al, be, d1, d2, (float)(-kLog2e / lambda));
  CK(cudaGetLastError());
  return 0;
}
}  // namespace

int32_t sinkhorn_plan_grad_device_v1(const sinkhorn_problem_v1* prob, double lambda,
                                     const float* log_u, const float* log_v, const float* cost,
                                     const float* upstream, float* out_grad_cost, void* stream) {
  if (int e = check_problem(prob)) return e;
  if (prob->cost_kind == SINKHORN_COST_GRID2D || prob->cost_kind == SINKHORN_COST_POINTS)
    return fail(SINKHORN_STATUS_BAD_ARGUMENT, "grid / point costs are not materialised");
  if (!(std::isfinite(lambda) && lambda > 0))
    return fail(SINKHORN_STATUS_INVALID_CONFIG, "lam must be positive and finite");
  if (prob->d1 == 0 || prob->d2 == 0) return 0;
  if (!log_u || !log_v || !cost || !upstream || !out_grad_cost)
    return fail(SINKHORN_STATUS_BAD_ARGUMENT, "null pointer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const float k = (float)(-1.4426950408889634 / lambda);
  dim3 g((unsigned)((prob->d2 + 31) / 32), (unsigned)((prob->d1 + 7) / 8));
  // (the workspace variant below runs the shared-cost case on the tensor cores)
  if (prob->cost_kind == SINKHORN_COST_SHARED) {
    ++g_launches;
    plan_grad_shared_kernel<<<g, 256, 0, st>>>(log_u, log_v, cost, upstream, (int)prob->B,
                                                (int)prob->d1, (int)prob->d2, k, out_grad_cost);
  } else {
    if (prob->B == 0) return 0;
    g.z = lanes_in_launch(prob->B, 0);   // the kernel strides over the rest
    ++g_launches;
    const bool vec = prob->d2 % 4 == 0 && (reinterpret_cast<uintptr_t>(cost) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(out_grad_cost) & 15) == 0 &&
                     (reinterpret_cast<uintptr_t>(log_v) & 15) == 0;
    if (vec) {
      int dev = 0;
      CK(cudaGetDevice(&dev));
      int sms = 148;
      CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
      const long long rows = prob->B * prob->d1;
      const int grid = (int)std::min<long long>((rows + 7) / 8, (long long)sms * 8);
      plan_grad_per_sample_vec4_kernel<<<grid, 256, 0, st>>>(log_u, log_v, cost, upstream,
                                                              (int)prob->B, (int)prob->d1,
                                                              (int)prob->d2, k, out_grad_cost);
    } else {
      plan_grad_per_sample_kernel<<<g, 256, 0, st>>>(log_u, log_v, cost, upstream,
                                                      (int)prob->B, (int)prob->d1, (int)prob->d2,
                                                      k, out_grad_cost);
    }
  }
  CK(cudaGetLastError());
  return 0;
}

size_t sinkhorn_plan_grad_workspace_bytes_v1(const sinkhorn_problem_v1* prob) {
  if (check_problem(prob) != 0) return 0;
  if (prob->cost_kind != SINKHORN_COST_SHARED) return 256;
  return plan_layout(*prob, device_info().sms).total;
}

int32_t sinkhorn_plan_grad_ws_device_v1(const sinkhorn_problem_v1* prob, double lambda,
                                        const float* log_u, const float* log_v, const float* cost,
                                        const float* upstream, float* out_grad_cost,
                                        void* workspace, size_t workspace_bytes, void* stream) {
  if (int e = check_problem(prob)) return e;
  if (prob->cost_kind != SINKHORN_COST_SHARED || prob->B == 0 || prob->d1 == 0 || prob->d2 == 0)
    return sinkhorn_plan_grad_device_v1(prob, lambda, log_u, log_v, cost, upstream, out_grad_cost,
                                        stream);
  if (!(std::isfinite(lambda) && lambda > 0))
    return fail(SINKHORN_STATUS_INVALID_CONFIG, "lam must be positive and finite");
  if (!log_u || !log_v || !cost || !upstream || !out_grad_cost)
    return fail(SINKHORN_STATUS_BAD_ARGUMENT, "null pointer");
  return plan_grad_umma(*prob, lambda, log_u, log_v, cost, upstream, out_grad_cost, workspace,
                        workspace_bytes, static_cast<cudaStream_t>(stream));
}

void sinkhorn_set_residual_reducer_v1(sinkhorn_residual_reducer_v1 fn, void* user) {
  g_reducer = fn;
  g_reducer_user = user;
}

int32_t sinkhorn_e0_partial_device_v1(int64_t B, int64_t d1, int64_t d2, double lambda,
                                      const float* log_u, const float* log_v, const float* cost,
                                      float* out_log2, void* workspace, size_t workspace_bytes,
                                      void* stream) {
  sinkhorn_problem_v1 pr = {B, d1, d2, SINKHORN_COST_SHARED, 0, 0, 0.f, 0.f};
  if (int e = check_problem(&pr)) return e;
  if (B == 0) return 0;
  if (!(std::isfinite(lambda) && lambda > 0))
    return fail(SINKHORN_STATUS_INVALID_CONFIG, "lam must be positive and finite");
  if (!log_u || !log_v || !cost || !out_log2)
    return fail(SINKHORN_STATUS_BAD_ARGUMENT, "null pointer");
  Solve S;
  S.pr = pr;
  S.di = device_info();
  S.L = make_layout(pr, S.di.sms);
  S.ws = workspace;
  S.st = static_cast<cudaStream_t>(stream);
  S.lam = (float)lambda;
  S.cost = cost;
  const Layout& L = S.L;
  if (workspace == nullptr || workspace_bytes < L.total)
    return fail(SINKHORN_STATUS_WORKSPACE, "workspace too small");
  cudaStream_t st = S.st;
  int* status = at<int>(workspace, L.status);
  CK(cudaMemsetAsync(status, 0, 4, st));
  CK(cudaMemsetAsync(at<int>(workspace, L.counters), 0,
                     std::max<size_t>(L.counter_count, 1) * 4, st));
  if (d1 == 0 || d2 == 0) {
    if (int e = fill(out_log2, (size_t)B, neg_inf_host(), st)) return e;
    return 0;
  }
  {
    dim3 g((unsigned)((L.D2p + 31) / 32), (unsigned)((L.D1p + 31) / 32));
    ++g_launches;
    prep_cost_kernel<<<g, 256, 0, st>>>(cost, (int)d1, (int)d2, L.D1p, L.D2p,
                                         (float)(-1.4426950408889634 / lambda), S.F(L.a2),
                                         S.F(L.a2t), status);
    dim3 gx((unsigned)((L.D1p + 31) / 32), (unsigned)((L.Bp + 31) / 32));
    ++g_launches;
    import_potential_kernel<<<gx, 256, 0, st>>>(log_u, (int)B, (int)d1, L.Bp, L.D1p, L.sb1,
                                                 L.si1, S.F(L.f2));
    dim3 gv((unsigned)((L.D2p + 31) / 32), (unsigned)((L.Bp + 31) / 32));
    ++g_launches;
    import_potential_kernel<<<gv, 256, 0, st>>>(log_v, (int)B, (int)d2, L.Bp, L.D2p, L.sb2,
                                                 L.si2, S.F(L.g2[0]));
    CK(cudaGetLastError());
  }
  if (int e = S.setup_maps()) return e;
  TiledArgs a = {&S.tm_a2, &S.tm_f2, (int)d1, (int)d2, L.D1p, L.D2p, S.F(L.l2nu), S.F(L.nu),
                 nullptr, S.F(L.g2[0]), nullptr, kResNone, S.F(L.e0), nullptr, nullptr};
  if (int e = launch_tiled<false, kModeTail>(L, workspace, S.di, a, pr, S.lam, st)) return e;
  ++g_launches;
  e0_finalize_kernel<<<(unsigned)((B + 31) / 32), 256, 0, st>>>(S.F(L.e0), (int)B, (int)d2, 1,
                                                                 L.Bp, out_log2, status, 1);
  CK(cudaGetLastError());
  int h = 0;
  if (int e = S.read_status(&h)) return e;
  return h == 0 ? 0 : fail(h, "device status " + std::to_string(h));
}

// ---- layer 1: host float64 views, the exact ffi.ts contract -----------------
static bool view_ok(const sinkhorn_view_v1* v, int ndim, int64_t s0, int64_t s1) {
  if (!v || v->ndim != ndim) return false;
  if (v->shape[0] != s0 || (ndim == 2 && v->shape[1] != s1)) return false;
  const int64_t n = ndim == 2 ? s0 * s1 : s0;
  return n <= v->length && (n == 0 || v->data != nullptr);   // ffi.ts:33-38
}

namespace {
// Device scratch of the host-buffer symbols: grow-only, one per host thread
// and entry point, reused across calls (both symbols run on
// cudaStreamPerThread and synchronise before they return), so repeated calls
// never pay for a device allocation.
struct HostScratch {
  void* p = nullptr;
  size_t cap = 0;
  int dev = -1;
  ~HostScratch() {
    if (p) cudaFree(p);
  }
  cudaError_t get(size_t n, void** out) {
    int d = 0;
    cudaGetDevice(&d);
    if (p == nullptr || cap < n || dev != d) {
      if (p) cudaFree(p);
      p = nullptr;
      cap = 0;
      const cudaError_t e = cudaMalloc(&p, n);
      if (e != cudaSuccess) return e;
      cap = n;
      dev = d;
    }
    *out = p;
    return cudaSuccess;
  }
};
thread_local HostScratch g_host_fwd, g_host_bwd;

struct DevBuf {
  void* p = nullptr;
  cudaStream_t st = nullptr;
};
}  // namespace

int32_t sinkhorn_forward_v1(const sinkhorn_view_v1* mu, const sinkhorn_view_v1* nu,
                            const sinkhorn_view_v1* cost, double lambda, int32_t max_iters,
                            double tolerance, const sinkhorn_view_v1* out_cost,
                            const sinkhorn_view_v1* out_log_u, const sinkhorn_view_v1* out_log_v) {
  // ffi.ts:91-106 shape checks
  if (!mu || !nu || !cost || mu->ndim != 2 || nu->ndim != 2 || cost->ndim != 2)
    return fail(SINKHORN_STATUS_SHAPE_MISMATCH, "mu, nu and cost must be 2-D");
  const int64_t B = mu->shape[0], d1 = mu->shape[1], d2 = nu->shape[1];
  if (!view_ok(mu, 2, B, d1) || !view_ok(nu, 2, B, d2) || nu->shape[0] != B ||
      !view_ok(cost, 2, d1, d2) || !view_ok(out_cost, 1, B, 0) || !view_ok(out_log_u, 2, B, d1) ||
      !view_ok(out_log_v, 2, B, d2))
    return fail(SINKHORN_STATUS_SHAPE_MISMATCH, "view shapes disagree");
  if (B == 0) return 0;   // ffi.ts:107-109
  if (B > INT32_MAX || d1 > INT32_MAX || d2 > INT32_MAX)
    return fail(SINKHORN_STATUS_SHAPE_MISMATCH, "extent exceeds int32");
  if (d1 == 0 || d2 == 0)
    return fail(SINKHORN_STATUS_INVALID_HISTOGRAM, "empty histogram cannot sum to 1");
  cudaStream_t st = cudaStreamPerThread;
  const size_t n_mu = (size_t)B * d1, n_nu = (size_t)B * d2, n_c = (size_t)d1 * d2;
  sinkhorn_problem_v1 pr = {B, d1, d2, SINKHORN_COST_SHARED, 0, 0, 0.f, 0.f};
  const size_t ws_bytes = workspace_total(pr, device_info().sms);
  // one device allocation: f64 staging + f32 inputs/outputs + solver workspace
  Carver c;
  const size_t o_d64 = c.take(std::max(n_mu + n_nu + n_c, n_mu + n_nu + (size_t)B) * 8);
  const size_t o_f_mu = c.take(n_mu * 4), o_f_nu = c.take(n_nu * 4), o_f_c = c.take(n_c * 4);
  const size_t o_cost = c.take((size_t)B * 4), o_lu = c.take(n_mu * 4), o_lv = c.take(n_nu * 4);
  const size_t o_ws = c.take(ws_bytes);
  DevBuf buf;
  buf.st = st;
  CK(g_host_fwd.get(c.off, &buf.p));
  double* d64 = at<double>(buf.p, o_d64);
  CK(cudaMemcpyAsync(d64, mu->data, n_mu * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d64 + n_mu, nu->data, n_nu * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d64 + n_mu + n_nu, cost->data, n_c * 8, cudaMemcpyHostToDevice, st));
  // histogram validation in float64, exactly ffi.ts:53-63 (status 11)
  int* vstat = at<int>(buf.p, o_ws + make_layout(pr, device_info().sms).status);
  int* vbad = at<int>(buf.p, o_ws + make_layout(pr, device_info().sms).badrow);
  CK(cudaMemsetAsync(vstat, 0, 4, st));
  CK(cudaMemsetAsync(vbad, 0x7f, 4, st));
  ++g_launches;
  validate_rows_kernel<double><<<(unsigned)B, 256, 0, st>>>(d64, (int)d1, vstat, vbad);
  ++g_launches;
  validate_rows_kernel<double><<<(unsigned)B, 256, 0, st>>>(d64 + n_mu, (int)d2, vstat, vbad);
  CK(cudaGetLastError());
  int hs = 0;
  CK(cudaMemcpyAsync(&hs, vstat, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (hs != 0) return fail(hs, "invalid histogram");
  sinkhorn_options_v1 op = {lambda, max_iters, 10, tolerance, SINKHORN_FLAG_SKIP_VALIDATION};
  if (int e = check_options(&op)) return e;
  ++g_launches;
  f64_to_f32_kernel<<<grid_for(n_mu), 256, 0, st>>>(d64, at<float>(buf.p, o_f_mu), n_mu);
  ++g_launches;
  f64_to_f32_kernel<<<grid_for(n_nu), 256, 0, st>>>(d64 + n_mu, at<float>(buf.p, o_f_nu), n_nu);
  ++g_launches;
  f64_to_f32_kernel<<<grid_for(n_c), 256, 0, st>>>(d64 + n_mu + n_nu, at<float>(buf.p, o_f_c), n_c);
  CK(cudaGetLastError());
  int32_t iters = 0;
  int e = forward_impl(pr, op, at<float>(buf.p, o_f_mu), at<float>(buf.p, o_f_nu),
                       at<float>(buf.p, o_f_c), at<float>(buf.p, o_cost), at<float>(buf.p, o_lu),
                       at<float>(buf.p, o_lv), &iters, nullptr, at<void>(buf.p, o_ws), ws_bytes,
                       st);
  if (e != 0) return e;
  // outputs back as float64 (ffi.ts:123-133 writes in place)
  ++g_launches;
  f32_to_f64_kernel<<<grid_for(B), 256, 0, st>>>(at<float>(buf.p, o_cost), d64, (size_t)B);
  ++g_launches;
  f32_to_f64_kernel<<<grid_for(n_mu), 256, 0, st>>>(at<float>(buf.p, o_lu), d64 + B, n_mu);
  ++g_launches;
  f32_to_f64_kernel<<<grid_for(n_nu), 256, 0, st>>>(at<float>(buf.p, o_lv), d64 + B + n_mu, n_nu);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out_cost->data, d64, (size_t)B * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(out_log_u->data, d64 + B, n_mu * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(out_log_v->data, d64 + B + n_mu, n_nu * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return 0;
}

int32_t sinkhorn_backward_v1(const sinkhorn_view_v1* log_u, const sinkhorn_view_v1* log_v,
                             double lambda, const sinkhorn_view_v1* upstream,
                             const sinkhorn_view_v1* out_grad_mu,
                             const sinkhorn_view_v1* out_grad_nu) {
  // ffi.ts:151-165
  if (!log_u || !log_v || log_u->ndim != 2 || log_v->ndim != 2)
    return fail(SINKHORN_STATUS_SHAPE_MISMATCH, "potentials must be 2-D");
  const int64_t B = log_u->shape[0], d1 = log_u->shape[1], d2 = log_v->shape[1];
  if (log_v->shape[0] != B || !view_ok(log_u, 2, B, d1) || !view_ok(log_v, 2, B, d2) ||
      !view_ok(upstream, 1, B, 0) || !view_ok(out_grad_mu, 2, B, d1) ||
      !view_ok(out_grad_nu, 2, B, d2))
    return fail(SINKHORN_STATUS_SHAPE_MISMATCH, "view shapes disagree");
  if (B == 0) return 0;
  if (B > INT32_MAX || d1 > INT32_MAX || d2 > INT32_MAX)
    return fail(SINKHORN_STATUS_SHAPE_MISMATCH, "extent exceeds int32");
  cudaStream_t st = cudaStreamPerThread;
  const size_t n1 = (size_t)B * d1, n2 = (size_t)B * d2;
  DevBuf buf;
  buf.st = st;
  CK(g_host_bwd.get((2 * n1 + 2 * n2 + B) * 8 + 16, &buf.p));
  double* u = static_cast<double*>(buf.p);
  double* v = u + n1;
  double* up = v + n2;
  double* gu = up + B;
  double* gv = gu + n1;
  int* stat = reinterpret_cast<int*>(gv + n2);
  CK(cudaMemcpyAsync(u, log_u->data, n1 * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(v, log_v->data, n2 * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(up, upstream->data, (size_t)B * 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(stat, 0, 4, st));
  CK(cudaMemsetAsync(stat + 1, 0x7f, 4, st));
  ++g_launches;
  backward_kernel<double><<<dim3((unsigned)B, 2), 256, 0, st>>>(u, v, (int)d1, (int)d2, lambda,
                                                                up, gu, gv, stat, stat + 1);
  CK(cudaGetLastError());
  int h = 0;
  CK(cudaMemcpyAsync(&h, stat, 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (h != 0) return fail(h, "zero-mass lane");   // ffi.ts:177-179
  CK(cudaMemcpyAsync(out_grad_mu->data, gu, n1 * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(out_grad_nu->data, gv, n2 * 8, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return 0;
}

}  // extern "C"
#pragma GCC visibility pop
