// sweep_f64.cuh -- the float64 parity mode.
//
// The reference computes in float64 and stops at
// tolerance 1e-9 by default (core.py:85), which an fp32 solve cannot reach.
// This mode runs the reference's iteration (batch.py:264-349) in double on
// the device, in natural log, exactly as stated: two-pass log-sum-exp per
// output (max, then sum of exp), v first then u, lockstep residual checks,
// the stable E0 over A + log c.  It is the precision path, not the fast one:
// one warp per output, lanes striding the reduction with coalesced loads of
// a row-major operand G[p][q] and of the lane's potential x[b][q].
//
//   column half-sweep: G = A^T (d2 x d1), x = log_u, out = log_v (batch.py:315)
//   row half-sweep:    G = A   (d1 x d2), x = log_v, out = log_u (batch.py:316)
//
// Per-sample costs keep one A_b and one A_b^T per lane (built once per solve).
#pragma once

#include "common.cuh"

namespace skb {

enum F64Mode : int { kF64Update = 0, kF64Residual = 1, kF64E0 = 2 };

struct F64SweepParams {
  int B, P, Q;
  int b0;                 // first lane of this launch (grid.y <= 65535 lanes per launch)
  const double* G;        // [P][Q] (shared) or lane b at G + b * P * Q (per-sample)
  long long g_lane;       // 0 for a shared operand, P * Q per-sample
  const double* x;        // [B][Q] reduced-side potentials
  const double* target;   // [B][P] log marginal (UPDATE)
  double* out;            // [B][P] UPDATE: target - lse; RESIDUAL / E0: per-output terms
  const double* pot;      // [B][P] output-side potentials (RESIDUAL, E0)
  const double* marg;     // [B][P] linear marginal (RESIDUAL)
  double lam;             // E0: c = -G * lam
  const int* status;
};

__device__ __forceinline__ double d_neg_inf() { return __longlong_as_double(0xfff0000000000000ll); }

// lse over q of G[p][q] + x[b][q]; E0 mode adds log c = log(-G * lam).
template <int kMode>
__device__ __forceinline__ double f64_lse(const double* __restrict__ g, const double* __restrict__ x,
                                          int Q, double lam) {
  const int lane = lane_id();
  double m = d_neg_inf();
  for (int q = lane; q < Q; q += 32) {
    double t = g[q] + x[q];
    if (kMode == kF64E0) t += log(-g[q] * lam);
    m = fmax(m, t);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
  if (m == d_neg_inf()) return d_neg_inf();   // empty reduction (OnlineLseAccumulator.finalise)
  double s = 0.0;
  for (int q = lane; q < Q; q += 32) {
    double t = g[q] + x[q];
    if (kMode == kF64E0) t += log(-g[q] * lam);
    s += exp(t - m);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  return m + log(s);
}

// grid ((P + 7) / 8, B), block 256: one warp per (lane b, output p).
template <int kMode>
__global__ void __launch_bounds__(256) f64_sweep_kernel(const F64SweepParams p) {
  if (p.status != nullptr && *p.status != 0) return;
  const int b = p.b0 + blockIdx.y;
  const int o = blockIdx.x * 8 + warp_id();
  if (o >= p.P) return;
  const double* g = p.G + b * p.g_lane + (size_t)o * p.Q;
  const double* x = p.x + (size_t)b * p.Q;
  const double lse = f64_lse<kMode>(g, x, p.Q, p.lam);
  if (lane_id() != 0) return;
  const size_t i = (size_t)b * p.P + o;
  if (kMode == kF64Update) {
    const double t = p.target[i];
    p.out[i] = (t == d_neg_inf()) ? d_neg_inf() : t - lse;   // test_reduction.py:207-216
  } else if (kMode == kF64Residual) {   // batch.py:303-309
    p.out[i] = fabs(exp(p.pot[i] + lse) - p.marg[i]);
  } else {                              // E0 term S[b, j] + log_v[b, j] (batch.py:333-337)
    p.out[i] = lse + p.pot[i];
  }
}

// Per lane: max of the row and column residual terms (NaN propagates), or
// E0 = exp(LSE_j terms).  One warp per lane.
__global__ void __launch_bounds__(256) f64_lane_reduce_kernel(const double* __restrict__ a, int na,
                                                              const double* __restrict__ c, int nc,
                                                              int B, double* __restrict__ out,
                                                              int lse_mode) {
  const int b = blockIdx.x * 8 + warp_id();
  if (b >= B) return;
  const int lane = lane_id();
  if (!lse_mode) {
    double m = 0.0;
    bool nan = false;
    for (int k = lane; k < na; k += 32) {
      const double v = a[(size_t)b * na + k];
      nan |= (v != v);
      m = fmax(m, v);
    }
    for (int k = lane; k < nc; k += 32) {
      const double v = c[(size_t)b * nc + k];
      nan |= (v != v);
      m = fmax(m, v);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
    nan = __any_sync(0xffffffffu, nan);
    if (lane == 0) out[b] = nan ? __longlong_as_double(0x7ff8000000000000ll) : m;
    return;
  }
  double m = d_neg_inf();
  for (int k = lane; k < na; k += 32) m = fmax(m, a[(size_t)b * na + k]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, off));
  double s = 0.0;
  if (m != d_neg_inf())
    for (int k = lane; k < na; k += 32) s += exp(a[(size_t)b * na + k] - m);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) out[b] = (m == d_neg_inf()) ? 0.0 : exp(m + log(s));
}

// Setup: log marginals (log 0 = -inf), u0 = 0 on the support, v0 = -inf
// (batch.py:292-296).
__global__ void f64_prep_kernel(const double* __restrict__ mu, const double* __restrict__ nu,
                                int B, int d1, int d2, double* __restrict__ lmu,
                                double* __restrict__ lnu, double* __restrict__ u,
                                double* __restrict__ v) {
  const size_t n1 = (size_t)B * d1, n2 = (size_t)B * d2;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n1 + n2;
       i += (size_t)gridDim.x * blockDim.x) {
    if (i < n1) {
      const double m = mu[i];
      lmu[i] = m > 0.0 ? log(m) : d_neg_inf();
      u[i] = m > 0.0 ? 0.0 : d_neg_inf();
    } else {
      const size_t k = i - n1;
      const double m = nu[k];
      lnu[k] = m > 0.0 ? log(m) : d_neg_inf();
      v[k] = d_neg_inf();
    }
  }
}

// A = -c / lam and A^T for each of `lanes` cost matrices (1 shared or B
// per-sample; or the squared-Euclidean grid when c == nullptr), plus
// CostMatrix validation (finite, >= 0; core.py:53-63) -> status 15.
__global__ void __launch_bounds__(256) f64_cost_kernel(const double* __restrict__ c, int lanes,
                                                       int d1, int d2, double lam, int gnx,
                                                       double ghx2, double ghy2,
                                                       double* __restrict__ a,
                                                       double* __restrict__ at, int* status) {
  __shared__ double tile[32][33];
  const int j0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  bool bad = false;
  for (int l = blockIdx.z; l < lanes; l += gridDim.z) {   // gridDim.z <= 65535 lanes at a time
    const size_t base = (size_t)l * d1 * d2;
    for (int r = ty; r < 32; r += 8) {
      const int i = i0 + r, j = j0 + tx;
      double v = 0.0;
      if (i < d1 && j < d2) {
        double cv;
        if (c != nullptr) {
          cv = c[base + (size_t)i * d2 + j];
        } else {
          const double dx = (double)(i % gnx - j % gnx), dy = (double)(i / gnx - j / gnx);
          cv = ghx2 * dx * dx + ghy2 * dy * dy;
        }
        if (!(cv >= 0.0) || isinf(cv)) bad = true;
        v = -cv / lam;
        a[base + (size_t)i * d2 + j] = v;
      }
      tile[r][tx] = v;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
      const int j = j0 + r, i = i0 + tx;
      if (j < d2 && i < d1) at[base + (size_t)j * d1 + i] = tile[tx][r];
    }
    __syncthreads();
  }
  if (bad) set_status(status, 15);
}

// NaN anywhere in the potentials -> status 12 (batch.py:326-327).
__global__ void f64_nan_kernel(const double* __restrict__ u, size_t n1, const double* __restrict__ v,
                               size_t n2, int* status) {
  bool nan = false;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n1 + n2;
       i += (size_t)gridDim.x * blockDim.x) {
    const double x = i < n1 ? u[i] : v[i - n1];
    nan |= (x != x);
  }
  if (__any_sync(0xffffffffu, nan) && lane_id() == 0) set_status(status, 12);
}

}  // namespace skb
