// sweep_small.cuh -- the whole solve for small shared / grid costs in ONE
// launch (batch.py:279-337 end to end).
//
// When d1*d2 is small (BASELINE config 1: d = 100) a sweep is a few hundred
// thousand cells and the tiled path is bound by its two launches per
// half-sweep, not by MUFU.  Here every CTA keeps the cost (both orientations,
// log2-scaled) and the potentials of its group of lanes in shared memory and
// runs all iterations itself: lanes are independent, so the only cross-CTA
// step is the lockstep stopping test every check_interval iterations
// (batch.py:318-322), a grid barrier on a cooperative launch.
//
// A lane group can be spread over a thread-block cluster of C CTAs: CTA r of
// the cluster owns the output slice [r*n/C, (r+1)*n/C) of every half-sweep
// (and only those rows of the cost), computes it exactly as a lone CTA would,
// and stores each new potential into every CTA's copy through distributed
// shared memory; a cluster barrier ends each half-sweep.  More SMs per lane,
// identical arithmetic.
//
// Work split inside a CTA: each (lane, output) unit is reduced by a group of
// S threads (S = 1..32, chosen on the host per orientation), element i read
// by thread s = i mod S.  The leading dimension of each cost orientation is
// ld = 32k + S, so the 32/S groups of a warp hit 32 distinct banks.  Every
// reduction is the exact two-pass one (max, then sum of 2^(x - max)), merged
// across the group with xor shuffles -- the same arithmetic as the tiled
// exact chunks, so results match the tiled path to fp32 rounding.
#pragma once

#include <cooperative_groups.h>

#include "common.cuh"

namespace skb {

struct SmallParams {
  const float* a2;    // [D1p][D2p] log2-scaled shared cost (null for grid costs)
  const float* a2t;   // [D2p][D1p]
  int D1p, D2p;
  int grid, gnx;      // grid cost recomputed into shared memory
  float gk, ghx2, ghy2;
  float cinv;         // cost = A2 * cinv (E0 weights)
  const float* l2mu;  // solver layout: element (b, i) at b * sb1 + i * si1
  const float* l2nu;  //                 element (b, j) at b * sb2 + j * si2
  const float* mu;
  const float* nu;
  const float* f2_init;   // warm start: log2 u in the solver layout (null: cold start)
  long long sb1, si1, sb2, si2;
  int B, d1, d2;
  int L;              // lanes per CTA (per cluster)
  int C;              // CTAs per cluster sharing a lane group (1 = no cluster)
  int Sc, Sr;         // threads per output: column sweep (reduces d1) / row sweep (reduces d2)
  int ldc, ldr;       // shared leading dims of A2T (column sweep) and A2 (row sweep)
  int max_iters, check_interval, checks;
  float tol;
  float* out_log_u;   // (B, d1) natural log
  float* out_log_v;   // (B, d2)
  float* out_cost;    // (B)
  float* res;         // (B) final residuals
  float* cta_res;     // [2][gridDim.x] per-check CTA maxima
  unsigned int* bar;  // grid-barrier counter (zero on entry)
  int* result;        // [0] iterations_run
  int* status;
  unsigned long long* dbg;   // optional timeline of CTA 0 (diagnostics), nullable
  const float* cps;   // per-sample costs (B, d1, d2) staged per lane (C = 1), else null
  float kscale;       // per-sample: A2 = c * kscale (-log2 e / lambda)
};

__host__ __device__ inline int small_slice(int n, int C, int r) { return (int)((long long)n * r / C); }
__host__ __device__ inline int small_rows(int n, int C) { return (n + C - 1) / C; }

struct SmallSmem {
  float* A;    // [rows of this CTA's d1 slice][ldr]  contiguous over j (row sweep)
  float* AT;   // [rows of this CTA's d2 slice][ldc]  contiguous over i (column sweep)
  float* f;    // [L][d1] log2 u
  float* g0;   // [L][d2] log2 v (ping-pong pair)
  float* g1;
  float* lmu;  // [L][d1]
  float* lnu;  // [L][d2]
  float* mu;   // [L][d1]
  float* nu;   // [L][d2]
  unsigned int* rres;   // [L] residual maxima (non-negative float bits)
  __host__ __device__ static size_t floats(int d1, int d2, int L, int ldc, int ldr, int C,
                                           bool ps = false) {
    return ((size_t)small_rows(d1, C) * ldr + (size_t)small_rows(d2, C) * ldc) * (ps ? L : 1) +
           (size_t)L * (3 * d1 + 5 * d2) + L + 8;
  }
  __device__ SmallSmem(float* base, const SmallParams& p, bool ps) {
    const size_t nl = ps ? (size_t)p.L : 1;   // per-sample: a cost per lane
    A = base;
    AT = A + (size_t)small_rows(p.d1, p.C) * p.ldr * nl;
    f = AT + (size_t)small_rows(p.d2, p.C) * p.ldc * nl;
    g0 = f + (size_t)p.L * p.d1;
    g1 = g0 + (size_t)p.L * p.d2;
    lmu = g1 + (size_t)p.L * p.d2;
    lnu = lmu + (size_t)p.L * p.d1;
    mu = lnu + (size_t)p.L * p.d2;
    nu = mu + (size_t)p.L * p.d1;
    rres = reinterpret_cast<unsigned int*>(nu + (size_t)p.L * p.d2);
  }
  __device__ float* g(int i) const { return i ? g1 : g0; }
};

// (max, sum 2^(row + x - max)[, sum of 2^(...) * row * cinv]) of one unit,
// reduced over the S threads of its group.  All 32 lanes of the warp call it.
template <int S, bool kTail>
__device__ __forceinline__ void small_unit_lse(const float* __restrict__ row,
                                               const float* __restrict__ x, int n, int s,
                                               bool active, float cinv, float& m_out,
                                               float& s_out, float& w_out) {
  float m0 = neg_inf(), m1 = neg_inf(), m2 = neg_inf(), m3 = neg_inf();
  if (active) {
    int i = s;
    for (; i + 3 * S < n; i += 4 * S) {
      m0 = fmaxf(m0, row[i] + x[i]);
      m1 = fmaxf(m1, row[i + S] + x[i + S]);
      m2 = fmaxf(m2, row[i + 2 * S] + x[i + 2 * S]);
      m3 = fmaxf(m3, row[i + 3 * S] + x[i + 3 * S]);
    }
    for (; i < n; i += S) m0 = fmaxf(m0, row[i] + x[i]);
  }
  float m = fmaxf(fmaxf(m0, m1), fmaxf(m2, m3));
#pragma unroll
  for (int o = 1; o < S; o <<= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  const float mm = (m == neg_inf()) ? 0.f : m;   // all terms -inf: the sum is 0
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f, w0 = 0.f, w1 = 0.f;
  if (active) {
    int i = s;
    for (; i + 3 * S < n; i += 4 * S) {
      const float e0 = ex2(row[i] + x[i] - mm);
      const float e1 = ex2(row[i + S] + x[i + S] - mm);
      const float e2 = ex2(row[i + 2 * S] + x[i + 2 * S] - mm);
      const float e3 = ex2(row[i + 3 * S] + x[i + 3 * S] - mm);
      s0 += e0;
      s1 += e1;
      s2 += e2;
      s3 += e3;
      if (kTail) {
        w0 = fmaf(e0, row[i] * cinv, w0);
        w1 = fmaf(e1, row[i + S] * cinv, w1);
        w0 = fmaf(e2, row[i + 2 * S] * cinv, w0);
        w1 = fmaf(e3, row[i + 3 * S] * cinv, w1);
      }
    }
    for (; i < n; i += S) {
      const float e = ex2(row[i] + x[i] - mm);
      s0 += e;
      if (kTail) w0 = fmaf(e, row[i] * cinv, w0);
    }
  }
  float sum = (s0 + s1) + (s2 + s3);
  float w = w0 + w1;
#pragma unroll
  for (int o = 1; o < S; o <<= 1) {
    sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (kTail) w += __shfl_xor_sync(0xffffffffu, w, o);
  }
  m_out = m;
  s_out = sum;
  w_out = w;
}

// Single pass shifted by an estimate of the result (the previous sweep's lse
// at this output, est = target - previous output): sum 2^(row + x - est).
// Accepted when the sum lies in [2^-60, 2^100] -- no term overflows and every
// term within 2^-60 of the largest is represented -- as the tiled and
// separable sweeps' estimate mode; the caller redoes the unit exactly
// otherwise (first iteration: no estimate).
template <int S>
__device__ __forceinline__ float small_unit_est(const float* __restrict__ row,
                                                const float* __restrict__ x, int n, int s,
                                                bool active, float est) {
  float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
  if (active) {
    int i = s;
    for (; i + 3 * S < n; i += 4 * S) {
      s0 += ex2(row[i] + x[i] - est);
      s1 += ex2(row[i + S] + x[i + S] - est);
      s2 += ex2(row[i + 2 * S] + x[i + 2 * S] - est);
      s3 += ex2(row[i + 3 * S] + x[i + 3 * S] - est);
    }
    for (; i < n; i += S) s0 += ex2(row[i] + x[i] - est);
  }
  float sum = (s0 + s1) + (s2 + s3);
#pragma unroll
  for (int o = 1; o < S; o <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  return sum;
}

// One half-sweep over the CTA's nl lanes and its output slice [o0, o1):
// out[l][o] = target - LSE_k(M[o - o0][k] + x[l][k]), stored locally and into
// every other CTA of the cluster (peer[r] = the same buffer in CTA r).
//   kRes 0: plain update; 1: row residual |2^(out + lse) - marg|;
//   2: column residual against `old` (the check sweep), 3: TAIL (residual
//   against `old` + the E0 term written to `out`, batch.py:329-337).
// prev: the previous potential of this orientation (the estimate source; may
// alias out -- each output is read by its own group before it is written).
template <int NT, int kRes, int S, bool kPS>
__device__ __forceinline__ void small_sweep_s(const float* __restrict__ M, int ld, int nout, int o0,
                                              int o1, int nin, int nl,
                                              const float* __restrict__ x,
                                              const float* __restrict__ target,
                                              const float* __restrict__ marg,
                                              const float* __restrict__ old, const float* prev,
                                              float* out, unsigned int* rres, float cinv,
                                              float* const* peers, const float* local_base, int C,
                                              int self, long long mls) {
  const int tid = threadIdx.x;
  constexpr int gpr = NT / S;   // groups per round
  const int s = tid % S;
  const int ns = o1 - o0;
  const int U = nl * ns;
  for (int base = 0; base < U; base += gpr) {
    const int u = base + tid / S;
    const bool active = u < U;
    const int l = active ? u / ns : 0;
    const int os = active ? u - l * ns : 0;
    const int o = o0 + os;
    const int idx = l * nout + o;
    const float* mrow = kPS ? M + (size_t)l * mls + (size_t)os * ld   // per-lane costs
                            : M + (size_t)os * ld;
    const float* xl = x + (size_t)l * nin;
    float m, sum, w = 0.f;
    bool exact = true;
    if constexpr (kRes != 3) {
      const float tg = active ? target[idx] : 0.f;
      const float est = active ? tg - prev[idx] : 0.f;
      const bool have = active && est - est == 0.f;   // finite (no NaN / inf)
      // zero-mass outputs stay -inf whatever the sum: no estimate needed
      const bool skip = active && tg == neg_inf();
      const bool any_est = __any_sync(0xffffffffu, have);
      if (any_est) {
        m = have ? est : 0.f;
        sum = small_unit_est<S>(mrow, xl, nin, s, active && have, m);
        const bool ok = !active || skip || (have && sum >= 0x1p-60f && sum <= 0x1p100f);
        exact = __any_sync(0xffffffffu, !ok);
      }
    }
    if (exact)
      small_unit_lse<S, kRes == 3>(mrow, xl, nin, s, active, cinv, m, sum, w);
    if (active && s == 0) {
      const float lse = lse_final(m, sum);
      float r = 0.f, v;
      if (kRes == 3) {
        const float ov = old[idx];
        v = (w > 0.f) ? (m + log2f(w) + ov) : neg_inf();
        r = fabsf(exp2f(ov + lse) - marg[idx]);
      } else {
        v = sweep_out(target[idx], lse);
        if (kRes == 1) r = fabsf(exp2f(v + lse) - marg[idx]);
        if (kRes == 2) r = fabsf(exp2f(old[idx] + lse) - marg[idx]);
      }
      out[idx] = v;
      if (C > 1) {
        const size_t off = (size_t)(out + idx - local_base);
        for (int q = 0; q < C; ++q)
          if (q != self) peers[q][off] = v;   // distributed shared memory
      }
      if (kRes != 0) {
        // NaN must win the max (batch.py:320 compares max <= tol, false for NaN)
        if (r != r) r = __int_as_float(0x7fc00000);
        atomicMax(&rres[l], __float_as_uint(r));
      }
    }
  }
}

// The group size S (threads per output, a power of two chosen on the host)
// as a template argument: unrolled shuffles, shift/mask indexing.
template <int NT, int kRes, bool kPS = false>
__device__ __forceinline__ void small_sweep(const float* __restrict__ M, int ld, int nout, int o0,
                                            int o1, int nin, int S, int nl,
                                            const float* __restrict__ x,
                                            const float* __restrict__ target,
                                            const float* __restrict__ marg,
                                            const float* __restrict__ old, const float* prev,
                                            float* out, unsigned int* rres, float cinv,
                                            float* const* peers, const float* local_base, int C,
                                            int self, long long mls = 0) {
#define SKB_SMALL_CASE(SS)                                                                      \
  case SS:                                                                                      \
    small_sweep_s<NT, kRes, SS, kPS>(M, ld, nout, o0, o1, nin, nl, x, target, marg, old, prev, out,  \
                                rres, cinv, peers, local_base, C, self, mls);                   \
    break;
  switch (S) {
    SKB_SMALL_CASE(1)
    SKB_SMALL_CASE(2)
    SKB_SMALL_CASE(4)
    SKB_SMALL_CASE(8)
    SKB_SMALL_CASE(16)
    default:
      small_sweep_s<NT, kRes, 32, kPS>(M, ld, nout, o0, o1, nin, nl, x, target, marg, old, prev, out,
                                  rres, cinv, peers, local_base, C, self, mls);
  }
#undef SKB_SMALL_CASE
}

// End of a half-sweep: every CTA of the cluster has stored its slice everywhere.
__device__ __forceinline__ void small_sync(int C) {
  if (C > 1) cooperative_groups::this_cluster().sync();
  else __syncthreads();
}

// kPS: per-sample costs (a cost per lane in shared memory); a separate
// instantiation so the shared-cost solver's code and registers are unchanged.
template <int NT, bool kPS = false>
__global__ void __launch_bounds__(NT, 2) small_solve_kernel(const SmallParams p) {
  extern __shared__ __align__(16) float small_smem[];
  const SmallSmem sm(small_smem, p, kPS);
  const int tid = threadIdx.x;
  const int C = p.C;
  const int crank = (C > 1) ? (int)cooperative_groups::this_cluster().block_rank() : 0;
  const int grp = blockIdx.x / C;
  const int b0 = grp * p.L;
  const int nl = min(p.L, p.B - b0);
  // this CTA's output slices of the column (over d2) and row (over d1) sweeps
  const int j0 = small_slice(p.d2, C, crank), j1 = small_slice(p.d2, C, crank + 1);
  const int i0 = small_slice(p.d1, C, crank), i1 = small_slice(p.d1, C, crank + 1);
  __shared__ int s_conv;
  __shared__ float* s_peer[8];
  if (C > 1 && tid < C)
    s_peer[tid] = cooperative_groups::this_cluster().map_shared_rank(small_smem, tid);

  // ---- stage this CTA's cost rows (both orientations) and the lanes ---------
  // A rows i in [i0, i1) (row sweep), AT rows j in [j0, j1) (column sweep)
  const int ni = i1 - i0, nj = j1 - j0;
  if (p.grid) {
    for (int e = tid; e < ni * p.d2; e += NT) {
      const int il = e / p.d2, j = e - il * p.d2, i = i0 + il;
      const int yi = i / p.gnx, xi = i - yi * p.gnx, yj = j / p.gnx, xj = j - yj * p.gnx;
      const float dx = float(xi) - float(xj), dy = float(yi) - float(yj);
      sm.A[(size_t)il * p.ldr + j] = p.gk * fmaf(p.ghx2, dx * dx, p.ghy2 * dy * dy);
    }
    for (int e = tid; e < nj * p.d1; e += NT) {
      const int jl = e / p.d1, i = e - jl * p.d1, j = j0 + jl;
      const int yi = i / p.gnx, xi = i - yi * p.gnx, yj = j / p.gnx, xj = j - yj * p.gnx;
      const float dx = float(xi) - float(xj), dy = float(yi) - float(yj);
      sm.AT[(size_t)jl * p.ldc + i] = p.gk * fmaf(p.ghx2, dx * dx, p.ghy2 * dy * dy);
    }
  } else if (kPS) {   // per-sample: each lane's own cost (C = 1), validated here
    bool bad = false;
    const size_t lc = (size_t)p.d1 * p.d2;
    for (long long e = tid; e < (long long)nl * lc; e += NT) {
      const int l = (int)(e / lc);
      const int k = (int)(e - (long long)l * lc);
      const int i = k / p.d2, j = k - i * p.d2;
      const float cv = p.cps[(size_t)(b0 + l) * lc + k];
      if (!(cv >= 0.f) || isinf(cv)) bad = true;
      const float a = cv * p.kscale;
      sm.A[(size_t)l * p.d1 * p.ldr + (size_t)i * p.ldr + j] = a;
      sm.AT[(size_t)l * p.d2 * p.ldc + (size_t)j * p.ldc + i] = a;
    }
    if (__any_sync(0xffffffffu, bad) && (tid & 31) == 0) set_status(p.status, 15);
  } else {
    for (int e = tid; e < ni * p.d2; e += NT) {
      const int il = e / p.d2, j = e - il * p.d2;
      sm.A[(size_t)il * p.ldr + j] = p.a2[(size_t)(i0 + il) * p.D2p + j];
    }
    for (int e = tid; e < nj * p.d1; e += NT) {
      const int jl = e / p.d1, i = e - jl * p.d1;
      sm.AT[(size_t)jl * p.ldc + i] = p.a2t[(size_t)(j0 + jl) * p.D1p + i];
    }
  }
  for (int e = tid; e < nl * p.d1; e += NT) {
    const int l = e / p.d1, i = e - l * p.d1;
    const size_t gi = (size_t)(b0 + l) * p.sb1 + (size_t)i * p.si1;
    sm.lmu[e] = p.l2mu[gi];
    sm.mu[e] = p.mu[gi];
    sm.f[e] = p.f2_init ? p.f2_init[gi] : ((p.mu[gi] > 0.f) ? 0.f : neg_inf());   // batch.py:295
  }
  for (int e = tid; e < nl * p.d2; e += NT) {
    const int l = e / p.d2, j = e - l * p.d2;
    const size_t gj = (size_t)(b0 + l) * p.sb2 + (size_t)j * p.si2;
    sm.lnu[e] = p.l2nu[gj];
    sm.nu[e] = p.nu[gj];
    sm.g0[e] = neg_inf();   // log v0 (batch.py:296): no estimate for the first column sweep
    sm.g1[e] = neg_inf();
  }
  small_sync(C);   // also publishes s_peer; every CTA of the cluster is running
  float* const* peers = s_peer;

  // ---- lockstep iteration (batch.py:314-324), v first then u ---------------
  unsigned int epoch = 0;
  int cur = 0;             // g[cur] holds log_v_k
  bool have_next = false;  // g[cur] already advanced by a check sweep
  int iters = 0, check_no = 0;
  const bool tl = p.dbg != nullptr && blockIdx.x == 0 && tid == 0;
  if (tl) p.dbg[0] = globaltimer_ns();
  for (int k = 1; k <= p.max_iters; ++k) {
    if (!have_next) {
      small_sweep<NT, 0, kPS>(sm.AT, p.ldc, p.d2, j0, j1, p.d1, p.Sc, nl, sm.f, sm.lnu, nullptr,
                         nullptr, sm.g(cur), sm.g(cur ^ 1), nullptr, 0.f, peers, small_smem, C,
                         crank,
                         kPS ? (long long)p.d2 * p.ldc : 0);
      if (tl && k <= 8) p.dbg[4 * k] = globaltimer_ns();
      small_sync(C);
      if (tl && k <= 8) p.dbg[4 * k + 1] = globaltimer_ns();
      cur ^= 1;
    }
    have_next = false;
    const bool last = (k == p.max_iters);
    const bool check = p.checks && (k % p.check_interval == 0) && !last;
    if (check || last) {
      for (int l = tid; l < nl; l += NT) sm.rres[l] = 0u;
      __syncthreads();
      small_sweep<NT, 1, kPS>(sm.A, p.ldr, p.d1, i0, i1, p.d2, p.Sr, nl, sm.g(cur), sm.lmu, sm.mu,
                         nullptr, sm.f, sm.f, sm.rres, 0.f, peers, small_smem, C, crank,
                         kPS ? (long long)p.d1 * p.ldr : 0);
    } else {
      small_sweep<NT, 0, kPS>(sm.A, p.ldr, p.d1, i0, i1, p.d2, p.Sr, nl, sm.g(cur), sm.lmu, nullptr,
                         nullptr, sm.f, sm.f, nullptr, 0.f, peers, small_smem, C, crank,
                         kPS ? (long long)p.d1 * p.ldr : 0);
    }
    if (tl && k <= 8) p.dbg[4 * k + 2] = globaltimer_ns();
    small_sync(C);
    if (tl && k <= 8) p.dbg[4 * k + 3] = globaltimer_ns();
    iters = k;
    if (check) {
      // column sweep k+1 doubles as the column residual of iteration k
      small_sweep<NT, 2, kPS>(sm.AT, p.ldc, p.d2, j0, j1, p.d1, p.Sc, nl, sm.f, sm.lnu, sm.nu,
                         sm.g(cur), sm.g(cur), sm.g(cur ^ 1), sm.rres, 0.f, peers, small_smem, C,
                         crank,
                         kPS ? (long long)p.d2 * p.ldc : 0);
      small_sync(C);
      // every CTA publishes the max over its lanes and slices; all CTAs read
      // all of them behind a grid barrier and take the same decision
      if (tid == 0) {
        unsigned int mx = 0u;
        for (int l = 0; l < nl; ++l) mx = max(mx, sm.rres[l]);
        p.cta_res[(check_no & 1) * gridDim.x + blockIdx.x] = __uint_as_float(mx);
      }
      grid_sync(p.bar, epoch);
      if (tid == 0) {
        unsigned int mx = 0u;
        for (int c = 0; c < (int)gridDim.x; ++c) {
          float v;
          asm volatile("ld.relaxed.gpu.global.f32 %0, [%1];"
                       : "=f"(v)
                       : "l"(p.cta_res + (check_no & 1) * gridDim.x + c));
          mx = max(mx, __float_as_uint(v));   // NaN bits exceed every finite value
        }
        s_conv = ((double)__uint_as_float(mx) <= (double)p.tol) ? 1 : 0;
      }
      __syncthreads();
      ++check_no;
      if (s_conv) break;   // keep g[cur] = log_v_k; the k+1 sweep is discarded
      cur ^= 1;
      have_next = true;
    }
  }

  // ---- tail: column residual + E0 terms, then export (batch.py:323-337) -----
  float* e0t = sm.g(cur ^ 1);
  small_sweep<NT, 3, kPS>(sm.AT, p.ldc, p.d2, j0, j1, p.d1, p.Sc, nl, sm.f, nullptr, sm.nu, sm.g(cur),
                     nullptr, e0t, sm.rres, p.cinv, peers, small_smem, C, crank,
                     kPS ? (long long)p.d2 * p.ldc : 0);
  small_sync(C);
  // the lane residual is the max over the cluster's slices (peer reads)
  if (C > 1 && crank == 0) {
    for (int l = tid; l < nl; l += NT) {
      unsigned int mx = sm.rres[l];
      for (int q = 1; q < C; ++q)
        mx = max(mx, *reinterpret_cast<const unsigned int*>(
                         peers[q] + (reinterpret_cast<const float*>(sm.rres + l) - small_smem)));
      sm.rres[l] = mx;
    }
  }
  small_sync(C);   // peers stay resident until the leader has read them
  if (crank == 0) {
    const int warp = tid >> 5, lane = tid & 31;
    for (int l = warp; l < nl; l += NT / 32) {
      float m = neg_inf();
      for (int j = lane; j < p.d2; j += 32) m = fmaxf(m, e0t[l * p.d2 + j]);
      for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      const float mm = (m == neg_inf()) ? 0.f : m;
      float s = 0.f;
      for (int j = lane; j < p.d2; j += 32) s += ex2(e0t[l * p.d2 + j] - mm);
      for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) {
        const float cost = exp2f(lse_final(m, s));
        p.out_cost[b0 + l] = cost;
        if (!isfinite(cost)) set_status(p.status, 12);
        p.res[b0 + l] = __uint_as_float(sm.rres[l]);
      }
    }
    bool nan = false;
    for (int e = tid; e < nl * p.d1; e += NT) {
      const float v = sm.f[e];
      nan |= broken_state(v);
      p.out_log_u[(size_t)b0 * p.d1 + e] = v * kLn2;
    }
    const float* gv = sm.g(cur);
    for (int e = tid; e < nl * p.d2; e += NT) {
      const float v = gv[e];
      nan |= broken_state(v);
      p.out_log_v[(size_t)b0 * p.d2 + e] = v * kLn2;
    }
    if (nan) set_status(p.status, 12);   // batch.py:326-327 NaNProduced (see broken_state)
  }
  if (blockIdx.x == 0 && tid == 0) p.result[0] = iters;
}

}  // namespace skb
