// sweep_gemm.cuh -- large shared costs (BASELINE config 5) as two GEMMs per
// iteration.
//
// With K = 2^A2 (A2 = -c log2e / lambda <= 0, so K <= 1) and, per lane, the
// potentials scaled by their maximum, X_j = 2^(v_j - vmax_b) <= 1:
//     LSE_j(A2_ij + v_j)  = vmax_b + log2 S_i,   S = K X           (row sweep)
//     u_i = l2mu_i - lse_i,  a_i = 2^(u_i + vmax_b) = mu_i / S_i
//     LSE_i(A2_ij + u_i)  = log2 T_j - vmax_b,   T = K^T a         (column sweep)
//     v'_j = l2nu_j + vmax_b - log2 T_j
// which is the reference's iteration (batch.py:314-316) with the log-sum-exps
// shifted by vmax_b, a valid shift (no term exceeds 1).  The two contractions
// over the whole (B, d1, d2) space run on the tcgen05 tensor cores in 3xTF32
// (sweep_umma.cuh: K and its stored transpose streamed once per contraction,
// fp32-accurate products, promoted fp32 accumulation).  Range
// guards: a row with S_i < 2^-60 (its terms may have flushed to zero) is
// redone exactly in the log domain from the caller's cost; a column with
// T_j < 2^-60 or a non-finite update flags the solve for the exact rerun.
// E0 = sum_i a_i (K o C) X per lane: a third GEMM at the end.
#pragma once

#include "common.cuh"

namespace skb {

constexpr float kGemmMin = 8.673617379884035e-19f;   // 2^-60

// Per lane: vmax = max_j v_j (a finite floor), X_j = 2^(v_j - vmax).
// grid B, block 1024.
__global__ void __launch_bounds__(1024) gemm_scale_kernel(const float* __restrict__ v, int d,
                                                          float* __restrict__ X,
                                                          float* __restrict__ vmax) {
  __shared__ float sm[32];
  const int b = blockIdx.x;
  const float* vb = v + (size_t)b * d;
  float m = kNegBig;
  for (int j = threadIdx.x; j < d; j += 1024) m = fmaxf(m, vb[j]);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
  if (lane_id() == 0) sm[warp_id()] = m;
  __syncthreads();
  if (warp_id() == 0) {
    m = sm[lane_id()];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    if (lane_id() == 0) sm[0] = m;
  }
  __syncthreads();
  m = sm[0];
  if (threadIdx.x == 0) vmax[b] = m;
  float* xb = X + (size_t)b * d;
  for (int j = threadIdx.x; j < d; j += 1024) xb[j] = ex2(vb[j] - m);
}

struct GemmRowParams {
  int B, d1, d2;
  int b0;                // first lane of this launch (grid.y <= 65535 lanes per launch)
  const float* S;        // [B][d1] K X
  const float* vmax;     // [B]
  const float* l2mu;     // [B][d1]
  const float* mu;       // [B][d1]
  float* u;              // [B][d1] out
  float* a;              // [B][d1] out: 2^(u + vmax)
  int* nfall;            // fallback row count
  int* fall;             // [B*d1] fallback rows (b * d1 + i)
  float* res;            // [B] row residual (tail), nullable
  const int* status;
};

// u_i and a_i from the GEMM row sums; grid (x: grid-stride over d1, y: lane b).
__global__ void gemm_row_kernel(const GemmRowParams p) {
  if (p.status != nullptr && *p.status != 0) return;
  const int b = p.b0 + blockIdx.y;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < p.d1; i += gridDim.x * blockDim.x) {
    const size_t k = (size_t)b * p.d1 + i;
    const float S = p.S[k];
    const float m = p.mu[k];
    if (!(S >= kGemmMin) || !(S < 3.0e38f)) {
      if (m > 0.f) {   // zero-mass rows are -inf whatever S is
        p.fall[atomicAdd(p.nfall, 1)] = (int)k;
        continue;
      }
    }
    const float lse = p.vmax[b] + log2f(S);
    const float u = sweep_out(p.l2mu[k], lse);
    p.u[k] = u;
    p.a[k] = m > 0.f ? m / S : 0.f;
    if (p.res != nullptr) atomic_max_nonneg(&p.res[b], fabsf(exp2f(u + lse) - m));
  }
}

// The queued rows, exactly in the log domain: lse = LSE_j(c_ij * kscale + v_j)
// from the caller's cost row (two passes), one warp per row, grid-stride.
__global__ void __launch_bounds__(256) gemm_row_fallback_kernel(const GemmRowParams p,
                                                                const float* __restrict__ cost,
                                                                const float* __restrict__ v,
                                                                float kscale) {
  const int n = *p.nfall;
  const int lane = lane_id();
  for (int w = blockIdx.x * 8 + warp_id(); w < n; w += gridDim.x * 8) {
    const int k = p.fall[w];
    const int b = k / p.d1, i = k % p.d1;
    const float* crow = cost + (size_t)i * p.d2;
    const float* vb = v + (size_t)b * p.d2;
    float m = kNegBig;
    for (int j = lane; j < p.d2; j += 32) m = fmaxf(m, fmaf(crow[j], kscale, vb[j]));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
    float s = 0.f;
    for (int j = lane; j < p.d2; j += 32) s += ex2(fmaf(crow[j], kscale, vb[j]) - m);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
    if (lane == 0) {
      const float lse = lse_final(m, s);
      const float u = sweep_out(p.l2mu[k], lse);
      p.u[k] = u;
      p.a[k] = exp2f(u + p.vmax[b]);   // P_ij = a_i K_ij X_j; overflow -> caught by the column guard
      if (p.res != nullptr) atomic_max_nonneg(&p.res[b], fabsf(exp2f(u + lse) - p.mu[k]));
    }
  }
}

struct GemmColParams {
  int B, d2;
  int b0;                // first lane of this launch (grid.y <= 65535 lanes per launch)
  const float* T;        // [B][d2] K^T a
  const float* vmax;     // [B] shift of the a's (the row pass's vmax, or 0 for the first sweep)
  const float* v_old;    // [B][d2] (residual), nullable on the first sweep
  float* v_new;          // [B][d2]
  const float* l2nu;     // [B][d2]
  const float* nu;       // [B][d2]
  float* res;            // [B] column residual, nullable
  int* est_fail;
  const int* status;
};

// v'_j = l2nu_j + vmax_b - log2 T_j, column residual |2^(v_j - vmax + log2 T_j) - nu_j|.
// grid (x: grid-stride over d2, y: lane b).
__global__ void gemm_col_kernel(const GemmColParams p) {
  if (p.status != nullptr && *p.status != 0) return;
  const int b = p.b0 + blockIdx.y;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < p.d2; j += gridDim.x * blockDim.x) {
    const size_t k = (size_t)b * p.d2 + j;
    const float T = p.T[k];
    const float tgt = p.l2nu[k];
    const float lt = log2f(T);
    float vn = neg_inf();
    if (tgt != neg_inf()) {
      vn = tgt + p.vmax[b] - lt;
      if (!(T >= kGemmMin) || !(vn == vn) || isinf(vn)) *p.est_fail = 1;
    }
    if (p.res != nullptr)
      atomic_max_nonneg(&p.res[b], fabsf(exp2f(p.v_old[k] - p.vmax[b] + lt) - p.nu[k]));
    p.v_new[k] = vn;
  }
}

// a0 = 1 on the support of mu (u0 = 0 there), 0 off it (batch.py:295).
__global__ void gemm_first_a_kernel(const float* __restrict__ mu, size_t n, float* __restrict__ a) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    a[i] = mu[i] > 0.f ? 1.f : 0.f;
}

// E0_b = sum_ij P_ij c_ij = sum_i a_i SE[b][i] with SE = (K o C) X (P_ij =
// a_i K_ij X_j carries the shifts).  One block per lane, double accumulation.
__global__ void __launch_bounds__(256) gemm_e0_kernel(const float* __restrict__ a,
                                                      const float* __restrict__ SE, int d1,
                                                      float* __restrict__ out, int* status) {
  __shared__ double sm[8];
  const int b = blockIdx.x;
  double s = 0.0;
  for (int i = threadIdx.x; i < d1; i += 256) s += (double)a[(size_t)b * d1 + i] * SE[(size_t)b * d1 + i];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane_id() == 0) sm[warp_id()] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += sm[w];
    out[b] = (float)t;
    if (!isfinite((float)t)) set_status(status, 12);
  }
}

}  // namespace skb
