// sweep_lane.cuh -- K3: half-sweeps over per-sample stored costs (B, d1, d2).
//
// Each lane owns its own cost C_b, so nothing is reused across lanes and the
// sweep streams C_b from HBM once per half-sweep: 4 bytes per cell, the HBM
// roofline of BASELINE config 4.  Both orientations read C_b in its native
// row-major layout with 128-bit coalesced loads -- no transposed copy (the
// reference materialises At, batch.py:290):
//   column sweep (reduce over i, out j): a CTA owns 256*VEC consecutive
//       columns of one lane and walks the rows; a warp reads 512 contiguous
//       bytes per row.
//   row sweep (reduce over j, out i): one warp per row; lanes stride the row
//       with float4 loads and merge their (max, sum) pairs by shuffles.
// Potentials are lane-major here: x[b*ld + i] (a lane's vector is contiguous).
// The exponent argument c*kscale + x is one FFMA per cell (kscale = -log2e/lambda).
#pragma once

#include "common.cuh"

namespace skb {

struct LaneSweepParams {
  int d1, d2;            // rows / cols of each lane's cost
  int ldx, ldo;          // lane strides of the reduced-side and output-side vectors
  const float* cost;     // lane b at cost + b*d1*d2
  float kscale;          // -log2(e)/lambda
  const float* x;        // reduced-side potentials (log2)
  const float* target;   // output-side log2 marginal
  const float* marg;     // output-side linear marginal
  float* out;            // output-side potentials (UPDATE)
  const float* old;      // output-side current potentials (kResCol / TAIL)
  float* res;            // [B] residual (atomic max), nullable
  float* e0;             // output-side E0 log2 terms (TAIL)
  float* pmax;           // PARTIAL outputs
  float* psum;
  float* part;           // column split partials [B][nj][nsplit][3][256*VEC]
  int* counters;         // [B][nj]
  int nsplit;
  int res_kind;
  const int* status;     // abort early if an earlier stage failed validation
  int* vstatus;          // kValidate: the cost check rides on this sweep (status 15)
  int b0;                // first lane of this launch (grid.y <= 65535 lanes per launch)
};

// Streaming (evict-first, ld.global.cs) loads: each cost element is used once per sweep.
__device__ __forceinline__ float4 ld_stream4(const float* p) {
  return __ldcs(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ float ld_stream1(const float* p) { return __ldcs(p); }

// Online accumulation of a chunk of KC values into (m, s[, s2]).
template <int KC, bool kTail>
__device__ __forceinline__ void lane_consume(const float (&t)[KC], const float (&cv)[KC], float& m,
                                             float& s, float& s2) {
  float cm = kNegBig;
#pragma unroll
  for (int k = 0; k < KC; ++k) cm = fmaxf(cm, t[k]);
  if (cm > m + kLazy) {
    const float r = ex2(m - cm);
    s *= r;
    if (kTail) s2 *= r;
    m = cm;
  }
  float e[KC], e2[KC];
#pragma unroll
  for (int k = 0; k < KC; ++k) {
    e[k] = ex2(t[k] - m);
    if (kTail) e2[k] = e[k] * cv[k];
  }
#pragma unroll
  for (int w = 1; w < KC; w *= 2)
#pragma unroll
    for (int k = 0; k + w < KC; k += 2 * w) {
      e[k] += e[k + w];
      if (kTail) e2[k] += e2[k + w];
    }
  s += e[0];
  if (kTail) s2 += e2[0];
}

// ---------------------------------------------------------------------------
// column sweep: out[b, j] = target - log2 sum_i 2^(C_b[i,j]*k + x[b,i])
// grid (nsplit, B, nj); block 256; thread owns VEC consecutive columns.
// kValidate (the solve's first sweep): every cost element is read exactly
// once here, so the CostMatrix check (finite, >= 0; core.py:53-63) is done on
// the same loads instead of a separate 4.3 GB pass at config 4; status 15
// stops every later kernel of the solve.
template <int VEC, int kMode, bool kValidate = false>
__global__ void __launch_bounds__(256) lane_col_kernel(const LaneSweepParams p) {
  constexpr int NT = 256;
  constexpr int KC = 8;
  constexpr int XCH = 512;  // potentials staged through smem in chunks
  constexpr bool kTail = (kMode == kModeTail);
  constexpr int NV = kTail ? 3 : 2;
  __shared__ float sx[XCH];
  __shared__ float s_res;
  __shared__ int s_flag;

  pdl_wait();
  if (p.status != nullptr && *p.status != 0) return;

  const int split = blockIdx.x;
  const int b = p.b0 + blockIdx.y;
  const int jb = blockIdx.z;
  const int tid = threadIdx.x;
  const int j0 = jb * NT * VEC + tid * VEC;
  const int i_begin = int((long long)split * p.d1 / p.nsplit);
  const int i_end = int((long long)(split + 1) * p.d1 / p.nsplit);
  const float* C = p.cost + (size_t)b * p.d1 * p.d2;
  const float* xb = p.x + (size_t)b * p.ldx;
  const bool colok = j0 < p.d2;   // VEC columns all valid when d2 % VEC == 0

  float m[VEC], s[VEC], s2[VEC];
#pragma unroll
  for (int v = 0; v < VEC; ++v) { m[v] = kNegBig; s[v] = 0.f; s2[v] = 0.f; }
  bool good = true;   // kValidate
  auto check = [&](float c) {
    if constexpr (kValidate) good &= (c >= 0.f) & (c != __int_as_float(0x7f800000));
  };

  for (int ic = i_begin; ic < i_end; ic += XCH) {
    const int n = min(XCH, i_end - ic);
    __syncthreads();
    for (int i = tid; i < n; i += NT) sx[i] = xb[ic + i];
    __syncthreads();
    if (!colok) continue;
    int i = 0;
    for (; i + KC <= n; i += KC) {
      float cv[VEC][KC];
#pragma unroll
      for (int k = 0; k < KC; ++k) {
        const float* row = C + (size_t)(ic + i + k) * p.d2 + j0;
        if constexpr (VEC == 4) {
          const float4 v4 = ld_stream4(row);
          cv[0][k] = v4.x; cv[1 % VEC][k] = v4.y; cv[2 % VEC][k] = v4.z; cv[3 % VEC][k] = v4.w;
        } else {
          cv[0][k] = ld_stream1(row);
        }
      }
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        float t[KC];
#pragma unroll
        for (int k = 0; k < KC; ++k) {
          check(cv[v][k]);
          t[k] = fmaf(cv[v][k], p.kscale, sx[i + k]);
        }
        lane_consume<KC, kTail>(t, cv[v], m[v], s[v], s2[v]);
      }
    }
    for (; i < n; ++i) {  // row tail
      const float* row = C + (size_t)(ic + i) * p.d2 + j0;
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        float t[1] = {fmaf(row[v], p.kscale, sx[i])};
        float cv1[1] = {row[v]};
        check(row[v]);
        lane_consume<1, kTail>(t, cv1, m[v], s[v], s2[v]);
      }
    }
  }

  if constexpr (kValidate)
    if (__any_sync(0xffffffffu, !good) && (tid & 31) == 0) set_status(p.vstatus, 15);
  auto finish = [&]() {
    float rmax = 0.f;
    if (colok) {
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        const int j = j0 + v;
        const size_t o = (size_t)b * p.ldo + j;
        if (kMode == kModePartial) {
          p.pmax[o] = m[v];
          p.psum[o] = s[v];
          continue;
        }
        const float lse = lse_final(m[v], s[v]);
        if (kMode == kModeUpdate) {
          const float ov = sweep_out(p.target[o], lse);
          p.out[o] = ov;
          if (p.res != nullptr && p.res_kind == kResCol)
            rmax = fmaxf(rmax, fabsf(exp2f(p.old[o] + lse) - p.marg[o]));
          else if (p.res != nullptr && p.res_kind == kResRow)
            rmax = fmaxf(rmax, fabsf(exp2f(ov + lse) - p.marg[o]));
        } else {
          const float od = p.old[o];
          p.e0[o] = (s2[v] > 0.f) ? (m[v] + log2f(s2[v]) + od) : neg_inf();
          rmax = fmaxf(rmax, fabsf(exp2f(od + lse) - p.marg[o]));
        }
      }
    }
    if (p.res != nullptr && (kTail || p.res_kind != kResNone)) {
      if (tid == 0) s_res = 0.f;
      __syncthreads();
      if (rmax != rmax) rmax = __int_as_float(0x7fc00000);
      atomic_max_nonneg(&s_res, rmax);
      __syncthreads();
      if (tid == 0) atomic_max_nonneg(&p.res[b], s_res);
    }
  };

  if (p.nsplit == 1) {
    finish();
  } else {
    const int nj = gridDim.z;
    float* base = p.part + ((((size_t)b * nj + jb) * p.nsplit) * NV) * (NT * VEC);
    float* mine = base + (size_t)split * NV * (NT * VEC);
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
      mine[tid * VEC + v] = m[v];
      mine[NT * VEC + tid * VEC + v] = s[v];
      if (kTail) mine[2 * NT * VEC + tid * VEC + v] = s2[v];
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) {
      const int prev = atomicAdd(&p.counters[b * nj + jb], 1);
      s_flag = (prev == p.nsplit - 1);
    }
    __syncthreads();
    if (s_flag) {
      __threadfence();
#pragma unroll
      for (int v = 0; v < VEC; ++v) { m[v] = kNegBig; s[v] = 0.f; s2[v] = 0.f; }
      for (int sp = 0; sp < p.nsplit; ++sp) {   // ascending split order (batch.py:198-201)
        const float* src = base + (size_t)sp * NV * (NT * VEC);
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
          const float m2 = __ldcg(src + tid * VEC + v);
          const float sv = __ldcg(src + NT * VEC + tid * VEC + v);
          const float mn = fmaxf(m[v], m2);
          const float ra = ex2(m[v] - mn), rb = ex2(m2 - mn);
          s[v] = s[v] * ra + sv * rb;
          if (kTail) s2[v] = s2[v] * ra + __ldcg(src + 2 * NT * VEC + tid * VEC + v) * rb;
          m[v] = mn;
        }
      }
      finish();
      if (tid == 0) p.counters[b * nj + jb] = 0;
    }
  }
  pdl_launch_dependents();
}

// ---------------------------------------------------------------------------
// row sweep: out[b, i] = target - log2 sum_j 2^(C_b[i,j]*k + x[b,j])
// grid (ceil(d1/ROWS), B); block 256 = 8 warps; one warp per row.
template <int VEC>
__global__ void __launch_bounds__(256) lane_row_kernel(const LaneSweepParams p, int rows_per_cta) {
  __shared__ float s_res;
  pdl_wait();
  if (p.status != nullptr && *p.status != 0) return;

  const int b = p.b0 + blockIdx.y;
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const float* C = p.cost + (size_t)b * p.d1 * p.d2;
  const float* xb = p.x + (size_t)b * p.ldx;
  const int r0 = blockIdx.x * rows_per_cta;
  const int r1 = min(p.d1, r0 + rows_per_cta);
  float rmax = 0.f;
  if (threadIdx.x == 0) s_res = 0.f;

  for (int i = r0 + warp; i < r1; i += 8) {
    const float* row = C + (size_t)i * p.d2;
    float m = kNegBig, s = 0.f, s2 = 0.f;
    constexpr int STEP = 32 * VEC;
    int j = lane * VEC;
    // main body: 4 vector loads in flight per lane
    for (; j + 3 * STEP + VEC <= p.d2; j += 4 * STEP) {
      float t[4 * VEC], cv[4 * VEC];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if constexpr (VEC == 4) {
          const float4 c4 = ld_stream4(row + j + u * STEP);
          const float4 x4 = __ldg(reinterpret_cast<const float4*>(xb + j + u * STEP));
          cv[u * VEC + 0] = c4.x; cv[u * VEC + (1 % VEC)] = c4.y;
          cv[u * VEC + (2 % VEC)] = c4.z; cv[u * VEC + (3 % VEC)] = c4.w;
          t[u * VEC + 0] = fmaf(c4.x, p.kscale, x4.x);
          t[u * VEC + (1 % VEC)] = fmaf(c4.y, p.kscale, x4.y);
          t[u * VEC + (2 % VEC)] = fmaf(c4.z, p.kscale, x4.z);
          t[u * VEC + (3 % VEC)] = fmaf(c4.w, p.kscale, x4.w);
        } else {
          cv[u] = ld_stream1(row + j + u * STEP);
          t[u] = fmaf(cv[u], p.kscale, __ldg(xb + j + u * STEP));
        }
      }
      lane_consume<4 * VEC, false>(t, cv, m, s, s2);
    }
    for (; j < p.d2; j += STEP) {  // tail (VEC-aligned rows: d2 % VEC == 0)
#pragma unroll
      for (int v = 0; v < VEC; ++v) {
        if (j + v < p.d2) {
          float t[1] = {fmaf(row[j + v], p.kscale, xb[j + v])};
          float cv1[1] = {0.f};
          lane_consume<1, false>(t, cv1, m, s, s2);
        }
      }
    }
    // warp merge of (m, s) pairs: OnlineLseAccumulator.merge (batch.py:116-130)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const float m2 = __shfl_xor_sync(0xffffffffu, m, off);
      const float sv = __shfl_xor_sync(0xffffffffu, s, off);
      lse_merge(m, s, m2, sv);
    }
    if (lane == 0) {
      const size_t o = (size_t)b * p.ldo + i;
      const float lse = lse_final(m, s);
      const float ov = sweep_out(p.target[o], lse);
      p.out[o] = ov;
      if (p.res != nullptr && p.res_kind == kResRow)
        rmax = fmaxf(rmax, fabsf(exp2f(ov + lse) - p.marg[o]));
    }
  }
  if (p.res != nullptr && p.res_kind == kResRow) {
    __syncthreads();
    if (lane == 0) {
      if (rmax != rmax) rmax = __int_as_float(0x7fc00000);
      atomic_max_nonneg(&s_res, rmax);
    }
    __syncthreads();
    if (threadIdx.x == 0) atomic_max_nonneg(&p.res[b], s_res);
  }
  pdl_launch_dependents();
}

}  // namespace skb
