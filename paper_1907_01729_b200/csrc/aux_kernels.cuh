// aux_kernels.cuh -- setup / validation / finalisation / backward kernels.
//
// None of these is on the per-iteration path; together they touch
// O(B*(d1+d2)) values (plus one pass over a shared cost) per solve.
#pragma once

#include "common.cuh"

namespace skb {


__global__ void fill_kernel(float* __restrict__ x, size_t n, float v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    x[i] = v;
}

// Per-row histogram validation (core.py:143-160, ffi.ts:53-63): finite,
// non-negative, |sum - 1| <= 1e-6 with the sum in fp64 and a fixed-order tree.
// One block per row; `bad_row` receives the first offending row (atomicMin).
template <typename T>
__global__ void __launch_bounds__(256) validate_rows_kernel(const T* __restrict__ m, int d,
                                                            int* status, int* bad_row) {
  __shared__ double s_sum[256];
  __shared__ int s_bad[256];
  const int b = blockIdx.x;
  const T* row = m + (size_t)b * d;
  double acc = 0.0;
  int bad = 0;
  for (int i = threadIdx.x; i < d; i += 256) {
    const double v = (double)row[i];
    if (!(v >= 0.0) || isinf(v)) bad = 1;   // NaN, -x, +-inf
    acc += v;
  }
  s_sum[threadIdx.x] = acc;
  s_bad[threadIdx.x] = bad;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      s_sum[threadIdx.x] += s_sum[threadIdx.x + w];
      s_bad[threadIdx.x] |= s_bad[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    if (s_bad[0] || !(fabs(s_sum[0] - 1.0) <= 1e-6)) {
      set_status(status, 11);
      atomicMin(bad_row, b);
    }
  }
}

// Marginal setup (batch.py:291-296): log2 marginal, linear marginal and the
// initial potential (0 on the support / -inf off it, or all -inf), written
// in the solver layout x[b*sb + i*si] with padding rows/lanes = (-inf, 0, -inf).
// Reads the (B, d) row-major input through a 32x32 shared tile so both the
// read and the (possibly transposed) write are coalesced.
__global__ void __launch_bounds__(256) prep_marginal_kernel(const float* __restrict__ m, int B,
                                                            int d, int Bp, int Dp, long long sb,
                                                            long long si, float* __restrict__ l2m,
                                                            float* __restrict__ lin,
                                                            float* __restrict__ pot0,
                                                            int pot_on_support) {
  __shared__ float tile[32][33];
  const int i0 = blockIdx.x * 32, b0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int r = ty; r < 32; r += 8) {
    const int b = b0 + r, i = i0 + tx;
    tile[r][tx] = (b < B && i < d) ? m[(size_t)b * d + i] : 0.f;
  }
  __syncthreads();
  const bool dim_major = (si != 1);
  for (int r = ty; r < 32; r += 8) {
    // dim-major: consecutive threads walk lanes; lane-major: walk dims
    const int b = dim_major ? (b0 + tx) : (b0 + r);
    const int i = dim_major ? (i0 + r) : (i0 + tx);
    if (b >= Bp || i >= Dp) continue;
    const float v = dim_major ? tile[tx][r] : tile[r][tx];
    const bool valid = (b < B && i < d);
    const size_t o = (size_t)b * sb + (size_t)i * si;
    const float mv = valid ? v : 0.f;
    l2m[o] = (valid && mv > 0.f) ? log2f(mv) : neg_inf();
    lin[o] = mv;
    pot0[o] = (valid && pot_on_support && mv > 0.f) ? 0.f : neg_inf();
  }
}

// Shared cost setup: A2 = c * k (k = -log2e/lambda) into [D1p][D2p] and its
// transpose into [D2p][D1p], -inf padding, plus CostMatrix validation
// (finite, >= 0; core.py:53-63) -> status 15.
__global__ void __launch_bounds__(256) prep_cost_kernel(const float* __restrict__ c, int d1,
                                                        int d2, int D1p, int D2p, float k,
                                                        float* __restrict__ a2,
                                                        float* __restrict__ a2t, int* status) {
  __shared__ float tile[32][33];
  const int j0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  bool bad = false;
  for (int r = ty; r < 32; r += 8) {
    const int i = i0 + r, j = j0 + tx;
    float v = neg_inf();
    if (i < d1 && j < d2) {
      const float cv = c[(size_t)i * d2 + j];
      if (!(cv >= 0.f) || isinf(cv)) bad = true;
      v = cv * k;
    }
    tile[r][tx] = v;
    if (i < D1p && j < D2p) a2[(size_t)i * D2p + j] = v;
  }
  if (bad) set_status(status, 15);
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int j = j0 + r, i = i0 + tx;
    if (j < D2p && i < D1p) a2t[(size_t)j * D1p + i] = tile[tx][r];
  }
}

// Per-sample cost validation (optional pass over B*d1*d2 values).
// HBM-bound (config 4: a 4.3 GB per-sample cost): float4 loads, four in flight
// per thread, after a scalar head up to the first 16-byte boundary.
__global__ void validate_cost_kernel(const float* __restrict__ c, size_t n, int* status) {
  auto ok = [](float v) { return v >= 0.f && v != __int_as_float(0x7f800000); };
  size_t head = ((16 - (reinterpret_cast<uintptr_t>(c) & 15)) & 15) / 4;
  if (head > n) head = n;
  const size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  const size_t nth = (size_t)gridDim.x * blockDim.x;
  bool good = tid >= head || ok(c[tid]);
  const float4* c4 = reinterpret_cast<const float4*>(c + head);
  const size_t n4 = (n - head) / 4;
  size_t i = tid;
  for (; i + 3 * nth < n4; i += 4 * nth) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldcs(c4 + i + u * nth);
#pragma unroll
    for (int u = 0; u < 4; ++u) good &= ok(v[u].x) & ok(v[u].y) & ok(v[u].z) & ok(v[u].w);
  }
  for (; i < n4; i += nth) {
    const float4 v = __ldcs(c4 + i);
    good &= ok(v.x) & ok(v.y) & ok(v.z) & ok(v.w);
  }
  const size_t tail = head + 4 * n4 + tid;
  if (tail < n) good &= ok(c[tail]);
  if (__any_sync(0xffffffffu, !good) && (threadIdx.x & 31) == 0) set_status(status, 15);
}

// Rows of n floats -> rows of ld floats (ld >= n), the tail zero: the fused
// per-sample pass's bulk copies need rows of whole 16-byte units.  A warp per
// row, grid-stride.
__global__ void __launch_bounds__(256) pad_rows_kernel(const float* __restrict__ src, long long rows,
                                                       int n, int ld, float* __restrict__ dst) {
  const int lane = threadIdx.x & 31;
  for (long long r = (blockIdx.x * 256LL + threadIdx.x) >> 5; r < rows;
       r += (long long)gridDim.x * 8) {
    const float* s = src + r * n;
    float* d = dst + r * ld;
    for (int j = lane; j < ld; j += 32) d[j] = j < n ? __ldcs(s + j) : 0.f;
  }
}

// Max over lanes of the residual vector (NaN wins), for the host's stopping test
// (batch.py:318-322).
__global__ void reduce_max_kernel(const float* __restrict__ res, int B, float* out) {
  __shared__ float s[256];
  float v = 0.f;
  for (int b = threadIdx.x; b < B; b += 256) {
    const float r = res[b];
    v = (r != r || v != v) ? __int_as_float(0x7fc00000) : fmaxf(v, r);
  }
  s[threadIdx.x] = v;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      const float a = s[threadIdx.x], bb = s[threadIdx.x + w];
      s[threadIdx.x] = (a != a || bb != bb) ? __int_as_float(0x7fc00000) : fmaxf(a, bb);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = s[0];
}

// E0 per lane (batch.py:334-337): cost_e0[b] = 2^(log2 sum_j 2^e0[j,b]).
// Block = 256 threads = 8 warps over 32 lanes; warps split j and merge their
// (max, sum) pairs in fixed order.
__global__ void __launch_bounds__(256) e0_finalize_kernel(const float* __restrict__ e0, int B,
                                                          int d2, long long sb, long long sj,
                                                          float* __restrict__ out_cost,
                                                          int* status, int out_log2) {
  __shared__ float sm[8][32], ss[8][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int b = blockIdx.x * 32 + lane;
  float m = kNegBig, s = 0.f;
  if (b < B) {
    for (int j = warp; j < d2; j += 8) {
      const float v = e0[(size_t)b * sb + (size_t)j * sj];
      if (v > m + kLazy) {
        s *= ex2(m - v);
        m = v;
      }
      s += ex2(v - m);
    }
  }
  sm[warp][lane] = m;
  ss[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && b < B) {
    for (int w = 1; w < 8; ++w) lse_merge(m, s, sm[w][lane], ss[w][lane]);
    if (out_log2) {      // partial (row-sharded) E0: log2 of this shard's sum
      out_cost[b] = lse_final(m, s);
    } else {
      const float cost = exp2f(lse_final(m, s));
      out_cost[b] = cost;
      if (!isfinite(cost)) set_status(status, 12);
    }
  }
}

// The same for lane-major E0 terms (sj == 1: lane b's terms contiguous):
// one warp per lane reads them coalesced, the (max, sum) pairs merged by a
// fixed xor butterfly (deterministic).  8 lanes per 256-thread block.
__global__ void __launch_bounds__(256) e0_finalize_rows_kernel(const float* __restrict__ e0, int B,
                                                               int d2, long long sb,
                                                               float* __restrict__ out_cost,
                                                               int* status, int out_log2) {
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (b >= B) return;
  const float* row = e0 + (size_t)b * sb;
  float m = kNegBig, s = 0.f;
  for (int j = lane; j < d2; j += 32) {
    const float v = __ldg(row + j);
    if (v > m + kLazy) {
      s *= ex2(m - v);
      m = v;
    }
    s += ex2(v - m);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const float mo = __shfl_xor_sync(0xffffffffu, m, off);
    const float so = __shfl_xor_sync(0xffffffffu, s, off);
    lse_merge(m, s, mo, so);
  }
  if (lane == 0) {
    if (out_log2) {
      out_cost[b] = lse_final(m, s);
    } else {
      const float cost = exp2f(lse_final(m, s));
      out_cost[b] = cost;
      if (!isfinite(cost)) set_status(status, 12);
    }
  }
}

// Solver layout (log2) -> caller layout (B, d) row-major natural log; NaN in
// the state is status 12 (batch.py:326-327 NaNProduced, ffi.ts:124-128).
__global__ void __launch_bounds__(256) export_potential_kernel(const float* __restrict__ x,
                                                               int B, int d, long long sb,
                                                               long long si,
                                                               float* __restrict__ out,
                                                               int* status, float scale,
                                                               int strict = 1) {
  __shared__ float tile[32][33];
  const int i0 = blockIdx.x * 32, b0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const bool dim_major = (si != 1);
  bool nan = false;
  for (int r = ty; r < 32; r += 8) {
    const int b = dim_major ? (b0 + tx) : (b0 + r);
    const int i = dim_major ? (i0 + r) : (i0 + tx);
    float v = 0.f;
    if (b < B && i < d) v = x[(size_t)b * sb + (size_t)i * si];
    if (dim_major) tile[tx][r] = v; else tile[r][tx] = v;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int b = b0 + r, i = i0 + tx;
    if (b < B && i < d) {
      const float v = tile[r][tx];
      // solver state: NaN, +inf or sentinel-scale (common.cuh); the half-sweep
      // API (fused_log_reduction) returns +inf like the reference and flags NaN only
      if (strict ? broken_state(v) : (v != v)) nan = true;
      out[(size_t)b * d + i] = v * scale;
    }
  }
  if (__any_sync(0xffffffffu, nan) && tx == 0) set_status(status, 12);
}

// Analytic backward (batch.py:352-375, ffi.ts:171-189): per lane row,
// grad = up[b] * lambda * (x - mean x), mean in fp64 with a fixed-order tree;
// any -inf -> status 13 and the first such lane.  grid (B, 2 sides).
template <typename T>
__global__ void __launch_bounds__(256) backward_kernel(const T* __restrict__ log_u,
                                                       const T* __restrict__ log_v, int d1,
                                                       int d2, double lam,
                                                       const T* __restrict__ up,
                                                       T* __restrict__ g_mu,
                                                       T* __restrict__ g_nu, int* status,
                                                       int* bad_lane) {
  __shared__ double s_sum[256];
  __shared__ int s_dead[256];
  const int b = blockIdx.x;
  const bool side_u = (blockIdx.y == 0);
  const int d = side_u ? d1 : d2;
  const T* x = (side_u ? log_u : log_v) + (size_t)b * d;
  T* g = (side_u ? g_mu : g_nu) + (size_t)b * d;
  double acc = 0.0;
  int dead = 0;
  for (int i = threadIdx.x; i < d; i += 256) {
    const double v = (double)x[i];
    if (isinf(v) && v < 0) dead = 1;
    acc += v;
  }
  s_sum[threadIdx.x] = acc;
  s_dead[threadIdx.x] = dead;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      s_sum[threadIdx.x] += s_sum[threadIdx.x + w];
      s_dead[threadIdx.x] |= s_dead[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (s_dead[0]) {
    if (threadIdx.x == 0) {
      set_status(status, 13);
      atomicMin(bad_lane, b);
    }
    return;
  }
  const double mean = s_sum[0] / (double)d;
  const double scale = (double)up[b] * lam;
  for (int i = threadIdx.x; i < d; i += 256) g[i] = (T)(scale * ((double)x[i] - mean));
}

// Caller layout (B, d) row-major natural log -> solver layout (log2), -inf padding.
__global__ void __launch_bounds__(256) import_potential_kernel(const float* __restrict__ in,
                                                               int B, int d, int Bp, int Dp,
                                                               long long sb, long long si,
                                                               float* __restrict__ x) {
  __shared__ float tile[32][33];
  const int i0 = blockIdx.x * 32, b0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int r = ty; r < 32; r += 8) {
    const int b = b0 + r, i = i0 + tx;
    tile[r][tx] = (b < B && i < d) ? in[(size_t)b * d + i] * kLog2e : neg_inf();
  }
  __syncthreads();
  const bool dim_major = (si != 1);
  for (int r = ty; r < 32; r += 8) {
    const int b = dim_major ? (b0 + tx) : (b0 + r);
    const int i = dim_major ? (i0 + r) : (i0 + tx);
    if (b >= Bp || i >= Dp) continue;
    x[(size_t)b * sb + (size_t)i * si] = dim_major ? tile[tx][r] : tile[r][tx];
  }
}

// Warm start: an imported log u stays -inf off the support (mu = 0), as the
// reference's initial potential does (batch.py:295).
__global__ void mask_potential_kernel(float* __restrict__ x, const float* __restrict__ lin,
                                      size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    if (!(lin[i] > 0.f)) x[i] = neg_inf();
}

// double <-> float conversions for the host-buffer (float64) ABI layer.
__global__ void f64_to_f32_kernel(const double* __restrict__ a, float* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    b[i] = (float)a[i];
}
__global__ void f32_to_f64_kernel(const float* __restrict__ a, double* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    b[i] = (double)a[i];
}

// Transport-plan gradient dC (core.py:363-368): for a shared cost
// dC[i,j] = sum_b up[b] * 2^(f2[b,i] + A2[i,j] + g2[b,j]) with natural-log
// inputs log_u/log_v (B, d) row-major; each plan entry is <= 1, so the sum is
// formed directly in the linear domain.  One thread per (i, j); lanes looped.
__global__ void __launch_bounds__(256) plan_grad_shared_kernel(
    const float* __restrict__ log_u, const float* __restrict__ log_v,
    const float* __restrict__ c, const float* __restrict__ up, int B, int d1, int d2, float k,
    float* __restrict__ dc) {
  const int j = blockIdx.x * 32 + (threadIdx.x & 31);
  const int i = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (i >= d1 || j >= d2) return;
  const float a = c[(size_t)i * d2 + j] * k;
  float acc = 0.f;
  for (int b = 0; b < B; ++b) {
    const float t = (log_u[(size_t)b * d1 + i] + log_v[(size_t)b * d2 + j]) * kLog2e + a;
    acc = fmaf(up[b], exp2f(t), acc);
  }
  dc[(size_t)i * d2 + j] = acc;
}

__global__ void __launch_bounds__(256) plan_grad_per_sample_kernel(
    const float* __restrict__ log_u, const float* __restrict__ log_v,
    const float* __restrict__ c, const float* __restrict__ up, int B, int d1, int d2, float k,
    float* __restrict__ dc) {
  const int j = blockIdx.x * 32 + (threadIdx.x & 31);
  const int i = blockIdx.y * 8 + (threadIdx.x >> 5);
  if (i >= d1 || j >= d2) return;
  for (int b = blockIdx.z; b < B; b += gridDim.z) {   // gridDim.z <= 65535 lanes at a time
    const size_t o = ((size_t)b * d1 + i) * d2 + j;
    const float t = (log_u[(size_t)b * d1 + i] + log_v[(size_t)b * d2 + j]) * kLog2e + c[o] * k;
    dc[o] = up[b] * exp2f(t);
  }
}

// The same, HBM-bound at config-4 size (4.3 GB read + 4.3 GB written): a warp
// per (lane, row) -- grid-stride over the B * d1 rows -- streams the row as
// float4 (d2 % 4 == 0, 16-byte aligned cost and output), evict-first.
__global__ void __launch_bounds__(256) plan_grad_per_sample_vec4_kernel(
    const float* __restrict__ log_u, const float* __restrict__ log_v,
    const float* __restrict__ c, const float* __restrict__ up, int B, int d1, int d2, float k,
    float* __restrict__ dc) {
  const int lane = threadIdx.x & 31;
  const long long rows = (long long)B * d1;
  const int q4 = d2 / 4;
  for (long long r = (long long)blockIdx.x * 8 + (threadIdx.x >> 5); r < rows;
       r += (long long)gridDim.x * 8) {
    const int b = (int)(r / d1);
    const float lu = log_u[r] * kLog2e, ub = up[b];
    const float4* cr = reinterpret_cast<const float4*>(c + r * d2);
    float4* dr = reinterpret_cast<float4*>(dc + r * d2);
    const float4* lv = reinterpret_cast<const float4*>(log_v + (size_t)b * d2);
    for (int j = lane; j < q4; j += 32) {
      const float4 cv = __ldcs(cr + j);
      const float4 v = __ldg(lv + j);
      float4 o;
      o.x = ub * exp2f(fmaf(v.x, kLog2e, lu) + cv.x * k);
      o.y = ub * exp2f(fmaf(v.y, kLog2e, lu) + cv.y * k);
      o.z = ub * exp2f(fmaf(v.z, kLog2e, lu) + cv.z * k);
      o.w = ub * exp2f(fmaf(v.w, kLog2e, lu) + cv.w * k);
      __stcs(dr + j, o);
    }
  }
}

}  // namespace skb
