// sweep_sep.cuh -- separable half-sweep for squared-Euclidean grid costs.
//
// On an nx x ny grid (point k = y*nx + x) the log2-scaled cost splits as
//   A2(i, j) = Ax(ix, jx) + Ay(iy, jy),   Ax(a, b) = gk*hx^2*(a-b)^2, Ay likewise,
// so the half-sweep LSE over the nx*ny grid points nests into two 1-D LSEs:
//   T(iy, jx)  = LSE_ix( Ax(ix, jx) + x(iy, ix) )                    (step 1)
//   lse(jy,jx) = LSE_iy( Ay(iy, jy) + T(iy, jx) )                     (step 2)
// -- nx*ny*(nx+ny) exponentials per lane instead of (nx*ny)^2 (32x fewer at
// 64x64), the same value as batch.py:208-230's fused reduction up to fp32
// rounding (each nested LSE is shifted by its own maximum).  The cost is
// symmetric, so column and row sweeps are the same operator on different
// buffers.  The E0 pass (batch.py:329-337) uses the same nesting with the
// weights c = cx + cy carried as a weighted mean through step 1.
//
// One CTA owns (lane, block of NB jx columns): step 1 produces T(:, block),
// step 2 the outputs (:, block) -- the blocks of a lane share no work.  Both
// steps are the same "LSE-GEMM" over shared-memory operands, 4x4 outputs per
// thread (two passes: max, then sum of 2^(p + q - max)).
#pragma once

#include "common.cuh"

namespace skb {

struct SepParams {
  int nx, ny;
  float ax, ay;            // log2 factors: Ax(a, b) = ax * (a - b)^2
  float cinv;              // cost = A2 * cinv
  const float* x;          // input potential, lane-major: (b, k) at b * ld + k
  const float* target;
  const float* marg;
  const float* old;
  float* out;              // update: new potential; tail: E0 term per point
  float* res;              // [B] residual maxima
  int res_kind;
  int ld;
  int B;
  int nblk;                // jx blocks per lane
  int use_poly;            // part of the exponentials on the FMA pipe
  const float* est_src;    // previous potential of this orientation (estimate mode) or null
  unsigned int* redo;      // count of thread tiles redone exactly (statistics)
};

// Estimate mode: the shifted sum must stay inside [2^kSepLo, 2^kSepHi] so no
// term overflows and every term within 2^-60 of the largest is represented.
constexpr float kSepLo = 0x1p-60f, kSepHi = 0x1p100f;

// Thread tile: RM (=4) consecutive m by RN (2 or 4) consecutive n, NT threads.
template <int NB_, int RN_, int NT_>
struct SepShape {
  static constexpr int NB = NB_, RN = RN_, NT = NT_, RM = 4;
  static constexpr int TN = NB / RN;       // threads along n
  static constexpr int TM = NT / TN;       // threads along m
  static constexpr int MT = TM * RM;       // m extent per pass
  static constexpr int OUT = RM * RN;      // outputs per thread
  static constexpr int HP = RN / 2;        // output pairs per m row
#ifdef SKB_SEP_POLY
  static constexpr int POLY = SKB_SEP_POLY;
#else
  static constexpr int POLY = OUT / 8;     // pairs on the FMA-pipe polynomial (25%)
#endif
  static_assert(RN == 2 || RN == 4, "pairs of n");
  static_assert(NT % TN == 0, "whole m rows of threads");
};

// floats of shared memory for an nx x ny grid
__host__ __device__ inline int sep_ldm(int ny) { return (ny + 3) & ~3; }
template <class S>
__host__ __device__ inline size_t sep_smem_floats(int nx, int ny, bool tail) {
  const int ldm = sep_ldm(ny);
  return (size_t)nx * ldm          // XT [ix][iy]
         + (size_t)nx * S::NB      // Ax block [ix][n]
         + (size_t)ny * ldm        // Ay [iy][jy]
         + (size_t)ny * S::NB      // T [iy][n]
         + (tail ? (size_t)ny * S::NB : 0) + S::MT;   // pad: ragged m tiles read past the end
}

template <int RN>
__device__ __forceinline__ void sep_load_q(const float* q, uint64_t (&qp)[RN / 2]) {
  if constexpr (RN == 4) {
    const float4 v = *reinterpret_cast<const float4*>(q);
    qp[0] = pk2(v.x, v.y);
    qp[1] = pk2(v.z, v.w);
  } else {
    const float2 v = *reinterpret_cast<const float2*>(q);
    qp[0] = pk2(v.x, v.y);
  }
}

// out(m, n) over m in [m0, m0 + MT) and the block's n, reducing k in [0, K):
//   (max, sum) of P(k, m) + Q(k, n) [+ weighted sum].  kW: 0 none,
//   1 weight Q*cinv (step 1 tail), 2 weight R(k, n) + P*cinv (step 2 tail).
// Packed f32x2 arithmetic on output pairs (n, n+1); the max pass folds two
// k steps into one 3-input max; kPoly sends a quarter of the output pairs
// through the FMA-pipe polynomial instead of MUFU (as the tiled sweep).
// kEst: one pass shifted by the caller's estimate `mx` (no max pass); returns
// false when a shifted sum leaves [2^kSepLo, 2^kSepHi] -- the caller then
// redoes the tile exactly.
template <class S, int kW, bool kPoly, bool kEst = false>
__device__ __forceinline__ bool sep_lse_gemm(const float* __restrict__ PT, int ldp,
                                             const float* __restrict__ Q,
                                             const float* __restrict__ R, int K, int m0,
                                             float cinv, float (&mx)[S::OUT],
                                             float (&sm)[S::OUT], float (&w)[S::OUT]) {
  constexpr int RN = S::RN, HP = S::HP, NB = S::NB;
  const int tn = threadIdx.x % S::TN, tm = threadIdx.x / S::TN;
  const float* pp = PT + m0 + tm * 4;
  const float* qq = Q + tn * RN;
  int k = 0;
  if (!kEst) {
#pragma unroll
  for (int e = 0; e < S::OUT; ++e) mx[e] = neg_inf();
#pragma unroll 2
  for (; k + 1 < K; k += 2) {
    const float4 p0 = *reinterpret_cast<const float4*>(pp + (size_t)k * ldp);
    const float4 p1 = *reinterpret_cast<const float4*>(pp + (size_t)(k + 1) * ldp);
    uint64_t qa[HP], qb[HP];
    sep_load_q<RN>(qq + (size_t)k * NB, qa);
    sep_load_q<RN>(qq + (size_t)(k + 1) * NB, qb);
    const float pv0[4] = {p0.x, p0.y, p0.z, p0.w}, pv1[4] = {p1.x, p1.y, p1.z, p1.w};
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int h = 0; h < HP; ++h) {
        const uint64_t u = fadd2(qa[h], pk2(pv0[a], pv0[a]));
        const uint64_t v = fadd2(qb[h], pk2(pv1[a], pv1[a]));
        mx[a * RN + 2 * h] = fmax3(mx[a * RN + 2 * h], lo2(u), lo2(v));
        mx[a * RN + 2 * h + 1] = fmax3(mx[a * RN + 2 * h + 1], hi2(u), hi2(v));
      }
  }
  if (k < K) {
    const float4 p0 = *reinterpret_cast<const float4*>(pp + (size_t)k * ldp);
    uint64_t qa[HP];
    sep_load_q<RN>(qq + (size_t)k * NB, qa);
    const float pv[4] = {p0.x, p0.y, p0.z, p0.w};
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int h = 0; h < HP; ++h) {
        const uint64_t u = fadd2(qa[h], pk2(pv[a], pv[a]));
        mx[a * RN + 2 * h] = fmaxf(mx[a * RN + 2 * h], lo2(u));
        mx[a * RN + 2 * h + 1] = fmaxf(mx[a * RN + 2 * h + 1], hi2(u));
      }
  }
  }
  uint64_t nM[4][HP], acc[4][HP], wacc[4][HP];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int h = 0; h < HP; ++h) {
      const float m0v = mx[a * RN + 2 * h], m1v = mx[a * RN + 2 * h + 1];
      nM[a][h] = pk2(m0v == neg_inf() ? 0.f : -m0v, m1v == neg_inf() ? 0.f : -m1v);
      acc[a][h] = pk2(0.f, 0.f);
      wacc[a][h] = pk2(0.f, 0.f);
    }
  const uint64_t c2 = pk2(cinv, cinv);
#pragma unroll 2
  for (k = 0; k < K; ++k) {
    const float4 p = *reinterpret_cast<const float4*>(pp + (size_t)k * ldp);
    const float pv[4] = {p.x, p.y, p.z, p.w};
    uint64_t qp[HP], wq[HP], rp[HP];
    sep_load_q<RN>(qq + (size_t)k * NB, qp);
    if (kW == 1) {
#pragma unroll
      for (int h = 0; h < HP; ++h) wq[h] = ffma2(qp[h], c2, pk2(0.f, 0.f));
    }
    if (kW == 2) sep_load_q<RN>(R + tn * RN + (size_t)k * NB, rp);
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const uint64_t pb = pk2(pv[a], pv[a]);
#pragma unroll
      for (int h = 0; h < HP; ++h) {
        const uint64_t t = fadd2(fadd2(qp[h], pb), nM[a][h]);
        const uint64_t e = (kPoly && a * HP + h < S::POLY) ? ex2_poly2(t)
                                                            : pk2(ex2(lo2(t)), ex2(hi2(t)));
        acc[a][h] = fadd2(acc[a][h], e);
        if (kW == 1) wacc[a][h] = ffma2(e, wq[h], wacc[a][h]);
        if (kW == 2) wacc[a][h] = ffma2(e, ffma2(pb, c2, rp[h]), wacc[a][h]);
      }
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int h = 0; h < HP; ++h) {
      sm[a * RN + 2 * h] = lo2(acc[a][h]);
      sm[a * RN + 2 * h + 1] = hi2(acc[a][h]);
      w[a * RN + 2 * h] = lo2(wacc[a][h]);
      w[a * RN + 2 * h + 1] = hi2(wacc[a][h]);
    }
  bool ok = true;
  if (kEst) {
#pragma unroll
    for (int e = 0; e < S::OUT; ++e) ok &= (sm[e] >= kSepLo) && (sm[e] <= kSepHi);   // NaN fails
  }
  return ok;
}

template <int RN>
__device__ __forceinline__ void sep_ld_row(const float* src, float (&v)[RN]) {
  if constexpr (RN == 4) {
    const float4 t = __ldcg(reinterpret_cast<const float4*>(src));
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  } else {
    const float2 t = __ldcg(reinterpret_cast<const float2*>(src));
    v[0] = t.x; v[1] = t.y;
  }
}
template <int RN>
__device__ __forceinline__ void sep_st_row(float* dst, const float (&v)[RN]) {
  if constexpr (RN == 4) *reinterpret_cast<float4*>(dst) = make_float4(v[0], v[1], v[2], v[3]);
  else *reinterpret_cast<float2*>(dst) = make_float2(v[0], v[1]);
}

// The previous lse of this orientation at the thread's tile of grid points,
// lse = target - previous potential; false when any is not finite (zero-mass
// points, first sweeps): the tile then takes the exact two-pass path.
template <class S>
__device__ __forceinline__ bool sep_estimate(const SepParams& p, int b, int m0, int jx0,
                                             float (&est)[S::OUT]) {
  constexpr int RN = S::RN;
  const int tn = threadIdx.x % S::TN, tm = threadIdx.x / S::TN;
  bool ok = true;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int y = min(m0 + tm * 4 + a, p.ny - 1);
#pragma unroll
    for (int c = 0; c < RN; ++c) {
      const int x = min(jx0 + tn * RN + c, p.nx - 1);
      const size_t k = (size_t)b * p.ld + (size_t)y * p.nx + x;
      const float e = __ldcg(p.target + k) - __ldcg(p.est_src + k);
      est[a * RN + c] = e;
      ok &= isfinite(e);
    }
  }
  return ok;
}

template <class S, int kMode>
__global__ void __launch_bounds__(S::NT, (S::NT >= 256) ? 4 : 4) sep_sweep_kernel(const SepParams p) {
  constexpr bool kTail = (kMode == kModeTail);
  constexpr int NB = S::NB, RN = S::RN, NT = S::NT;
  extern __shared__ __align__(16) float sep_smem[];
  const int nx = p.nx, ny = p.ny, ldm = sep_ldm(ny);
  float* XT = sep_smem;
  float* AX = XT + (size_t)nx * ldm;
  float* AY = AX + (size_t)nx * NB;
  float* T = AY + (size_t)ny * ldm;
  float* R = T + (size_t)ny * NB;   // tail only
  __shared__ unsigned int s_res;
  const int tid = threadIdx.x;
  const int b = blockIdx.y;
  const int jx0 = blockIdx.x * NB;
  const float* xb = p.x + (size_t)b * p.ld;

  if (tid == 0) s_res = 0u;
  // cost factors first: they do not depend on the previous sweep (PDL overlap)
  for (int e = tid; e < nx * NB; e += NT) {
    const int ix = e / NB, n = e - ix * NB;
    const float d = float(ix - (jx0 + n));
    AX[e] = p.ax * (d * d);
  }
  for (int e = tid; e < ny * ldm; e += NT) {
    const int iy = e / ldm, jy = e - iy * ldm;
    const float d = float(iy - jy);
    AY[e] = p.ay * (d * d);
  }
  pdl_wait();   // x is the previous sweep's output
  // the lane's potential, transposed into XT[ix][iy]: consecutive threads take
  // consecutive rows iy (conflict-free transposed stores), every 16-byte load
  // of a batch in flight before the first store
  if ((nx & 3) == 0) {
    const int nx4 = nx >> 2, n4 = nx4 * ny;
    for (int base = 0; base < n4; base += NT * 4) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int idx = base + u * NT + tid;
        if (idx < n4) {
          const int ix4 = idx / ny, iy = idx - ix4 * ny;
          v[u] = __ldcg(reinterpret_cast<const float4*>(xb + (size_t)iy * nx) + ix4);
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int idx = base + u * NT + tid;
        if (idx < n4) {
          const int ix4 = idx / ny, iy = idx - ix4 * ny;
          float* d = XT + (size_t)(4 * ix4) * ldm + iy;
          d[0] = v[u].x;
          d[ldm] = v[u].y;
          d[2 * ldm] = v[u].z;
          d[3 * ldm] = v[u].w;
        }
      }
    }
  } else {
    for (int e = tid; e < nx * ny; e += NT) {
      const int iy = e / nx, ix = e - iy * nx;
      XT[(size_t)ix * ldm + iy] = __ldcg(xb + e);
    }
  }
  __syncthreads();
  pdl_launch_dependents();

  const int tn = tid % S::TN, tm = tid / S::TN;
  float mx[S::OUT], sm[S::OUT], w[S::OUT];
  // ---- step 1: T(iy, n) = LSE_ix(Ax(ix, n) + x(iy, ix)) --------------------
  for (int m0 = 0; m0 < ny; m0 += S::MT) {
    bool done = false;
    if (!kTail && p.est_src != nullptr) {
      // shift T(iy, n) by the previous lse at grid point (iy, n): T <= lse there
      done = sep_estimate<S>(p, b, m0, jx0, mx) &&
             (p.use_poly ? sep_lse_gemm<S, 0, true, true>(XT, ldm, AX, nullptr, nx, m0, p.cinv, mx, sm, w)
                         : sep_lse_gemm<S, 0, false, true>(XT, ldm, AX, nullptr, nx, m0, p.cinv, mx, sm, w));
      if (!done && p.redo) atomicAdd(p.redo, 1u);
    }
    if (done) {
    } else if (!kTail && p.use_poly)
      sep_lse_gemm<S, 0, true>(XT, ldm, AX, nullptr, nx, m0, p.cinv, mx, sm, w);
    else
      sep_lse_gemm<S, kTail ? 1 : 0, false>(XT, ldm, AX, nullptr, nx, m0, p.cinv, mx, sm, w);
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int iy = m0 + tm * 4 + a;
      if (iy >= ny) continue;
#pragma unroll
      for (int c = 0; c < RN; ++c) {
        const int e = a * RN + c;
        T[(size_t)iy * NB + tn * RN + c] = lse_final(mx[e], sm[e]);
        if (kTail) R[(size_t)iy * NB + tn * RN + c] = (sm[e] > 0.f) ? w[e] / sm[e] : 0.f;
      }
    }
  }
  __syncthreads();
  // ---- step 2: lse(jy, n) = LSE_iy(Ay(iy, jy) + T(iy, n)); epilogue --------
  float rmax = 0.f;
  for (int m0 = 0; m0 < ny; m0 += S::MT) {
    bool done = false;
    if (!kTail && p.est_src != nullptr) {
      done = sep_estimate<S>(p, b, m0, jx0, mx) &&
             (p.use_poly ? sep_lse_gemm<S, 0, true, true>(AY, ldm, T, R, ny, m0, p.cinv, mx, sm, w)
                         : sep_lse_gemm<S, 0, false, true>(AY, ldm, T, R, ny, m0, p.cinv, mx, sm, w));
      if (!done && p.redo) atomicAdd(p.redo, 1u);
    }
    if (done) {
    } else if (!kTail && p.use_poly)
      sep_lse_gemm<S, 0, true>(AY, ldm, T, R, ny, m0, p.cinv, mx, sm, w);
    else
      sep_lse_gemm<S, kTail ? 2 : 0, false>(AY, ldm, T, R, ny, m0, p.cinv, mx, sm, w);
    const int jxb = jx0 + tn * RN;
    if (!kTail && (nx % RN) == 0 && jxb + RN - 1 < nx) {
      // update epilogue, vector rows: every load of the tile issued first
      float tg[4][RN], mg[4][RN], od[4][RN];
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int jy = min(m0 + tm * 4 + a, ny - 1);
        const size_t off = (size_t)b * p.ld + (size_t)jy * nx + jxb;
        sep_ld_row<RN>(p.target + off, tg[a]);
        if (p.res_kind != kResNone) sep_ld_row<RN>(p.marg + off, mg[a]);
        if (p.res_kind == kResCol) sep_ld_row<RN>(p.old + off, od[a]);
      }
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int jy = m0 + tm * 4 + a;
        if (jy >= ny) continue;
        float nv[RN];
#pragma unroll
        for (int c = 0; c < RN; ++c) {
          const float lse = lse_final(mx[a * RN + c], sm[a * RN + c]);
          nv[c] = sweep_out(tg[a][c], lse);
          if (p.res_kind == kResRow) rmax = fmaxf(rmax, fabsf(exp2f(nv[c] + lse) - mg[a][c]));
          if (p.res_kind == kResCol) rmax = fmaxf(rmax, fabsf(exp2f(od[a][c] + lse) - mg[a][c]));
        }
        sep_st_row<RN>(p.out + (size_t)b * p.ld + (size_t)jy * nx + jxb, nv);
      }
      continue;
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int jy = m0 + tm * 4 + a;
      if (jy >= ny) continue;
#pragma unroll
      for (int c = 0; c < RN; ++c) {
        const int jx = jxb + c;
        if (jx >= nx) continue;
        const int e = a * RN + c;
        const size_t k = (size_t)b * p.ld + (size_t)jy * nx + jx;
        const float lse = lse_final(mx[e], sm[e]);
        if (kTail) {
          const float ov = p.old[k];
          p.out[k] = (w[e] > 0.f) ? (mx[e] + log2f(w[e]) + ov) : neg_inf();
          rmax = fmaxf(rmax, fabsf(exp2f(ov + lse) - p.marg[k]));
        } else {
          const float nv = sweep_out(p.target[k], lse);
          p.out[k] = nv;
          if (p.res_kind == kResRow) rmax = fmaxf(rmax, fabsf(exp2f(nv + lse) - p.marg[k]));
          if (p.res_kind == kResCol) rmax = fmaxf(rmax, fabsf(exp2f(p.old[k] + lse) - p.marg[k]));
        }
      }
    }
  }
  if (kTail || p.res_kind != kResNone) {
    // NaN must win the max (batch.py:320 compares max <= tol, false for NaN)
    if (rmax != rmax) rmax = __int_as_float(0x7fc00000);
    atomicMax(&s_res, __float_as_uint(rmax));
    __syncthreads();
    if (tid == 0) atomic_max_nonneg(&p.res[b], __uint_as_float(s_res));
  }
}

}  // namespace skb
