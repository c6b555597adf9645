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
// steps are the same "LSE-GEMM" out(m, n) = LSE_k(P(m, k) + Q(k, n)) over
// shared-memory operands, 4x2 outputs per thread:
//   step 1: P^T = x^T [ix][iy] (transposed on staging), Q = Ax block
//   step 2: P^T = Ay [iy][jy] (symmetric),               Q = T
// The Ax / Ay tables are built once per solve and arrive by cp.async (no
// per-CTA arithmetic, no registers) before the PDL wait.
#pragma once

#include "common.cuh"

namespace skb {

struct SepParams {
  int nx, ny;
  float cinv;              // cost = A2 * cinv
  const float* ax_tab;     // [nx][nblk*NB] Ax(ix, jx) (log2 units), padded columns finite
  const float* ay_tab;     // [ny][sep_ld(ny)] Ay(iy, jy)
  const float* xT;         // input potential transposed, lane-major: (b, ix, iy) at b*ld + ix*ny + iy
  float* outT;             // update: the new potential transposed (same layout), else null
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
  int b0;                  // first lane of this launch (grid.y <= 65535 lanes per launch)
  const float* est_src;    // previous potential of this orientation (estimate mode) or null
  unsigned int* redo;      // count of thread tiles redone exactly (statistics)
  unsigned long long* dbg; // optional per-CTA timeline (diagnostics), nullable
  float* tg;               // split sweeps: T per (lane, jx block) [B][nblk][ny][NB]
  float* rg;               // split sweeps, tail: the E0 weights R, same layout
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

// leading dimension (floats) of shared rows indexed by y: padded to 4
__host__ __device__ inline int sep_ld(int n) { return (n + 3) & ~3; }
template <class S>
__host__ __device__ inline size_t sep_smem_floats(int nx, int ny, bool tail) {
  const size_t xt = (size_t)nx * sep_ld(ny), ot = (size_t)S::NB * (ny + 1);
  return (xt > ot ? xt : ot)        // XT [ix][iy] / OT [n][jy]
         + (size_t)nx * S::NB      // Ax block [ix][n]
         + (size_t)ny * sep_ld(ny) // Ay [iy][jy]
         + (size_t)ny * S::NB      // T  [iy][n]
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

// Rows of `cols` floats from global (row stride gld) into shared memory (row
// stride sld): 16-byte cp.async when every row start is 16-byte aligned,
// 4-byte otherwise.  The caller commits the group.
template <int NT>
__device__ __forceinline__ void sep_stage_rows(float* dst, int sld, const float* src, size_t gld,
                                               int rows, int cols) {
  const bool v4 = ((cols | sld | (int)(gld & 3)) & 3) == 0 &&
                  (reinterpret_cast<uintptr_t>(src) & 15) == 0;
  if (v4) {
    const int c4 = cols >> 2;
    for (int e = threadIdx.x; e < rows * c4; e += NT) {
      const int r = e / c4, c = e - r * c4;
      cp_async16(dst + (size_t)r * sld + 4 * c, src + r * gld + 4 * c);
    }
  } else {
    for (int e = threadIdx.x; e < rows * cols; e += NT) {
      const int r = e / cols, c = e - r * cols;
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                       smem_u32(dst + (size_t)r * sld + c)),
                   "l"(src + r * gld + c)
                   : "memory");
    }
  }
}

template <class S, int kMode>
__global__ void __launch_bounds__(S::NT, 4) sep_sweep_kernel(const SepParams p) {
  constexpr bool kTail = (kMode == kModeTail);
  constexpr int NB = S::NB, RN = S::RN, NT = S::NT;
  extern __shared__ __align__(16) float sep_smem[];
  const int nx = p.nx, ny = p.ny, ldm = sep_ld(ny);
  float* XT = sep_smem;                      // [nx][ldm]
  float* AX = XT + (size_t)nx * ldm;         // [nx][NB]
  float* AY = AX + (size_t)nx * NB;          // [ny][ldm]
  float* T = AY + (size_t)ny * ldm;          // [ny][NB]
  float* R = T + (size_t)ny * NB;            // [ny][NB], tail only
  __shared__ unsigned int s_res;
  const int tid = threadIdx.x;
  const int b = p.b0 + blockIdx.y;
  const int jx0 = blockIdx.x * NB;

  if (tid == 0) s_res = 0u;
  const int cta = blockIdx.y * gridDim.x + blockIdx.x;
  if (p.dbg && tid == 0) {
    unsigned smid;
    asm("mov.u32 %0, %%smid;" : "=r"(smid));
    p.dbg[4 * cta] = globaltimer_ns();
    p.dbg[4 * cta + 3] = smid;
  }
  // everything arrives by cp.async: the cost factors before the PDL wait
  // (they do not depend on the previous sweep), then the lane's potential,
  // which the previous sweep also wrote transposed ([ix][iy]) for this copy
  sep_stage_rows<NT>(AX, NB, p.ax_tab + jx0, (size_t)p.nblk * NB, nx, NB);
  sep_stage_rows<NT>(AY, ldm, p.ay_tab, (size_t)ldm, ny, ny);
  cp_async_commit();
  pdl_wait();   // x is the previous sweep's output
  sep_stage_rows<NT>(XT, ldm, p.xT + (size_t)b * p.ld, (size_t)ny, nx, ny);
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  pdl_launch_dependents();
  if (p.dbg && tid == 0) p.dbg[4 * cta + 1] = globaltimer_ns();

  const int tn = tid % S::TN, tm = tid / S::TN;
  float mx[S::OUT], sm[S::OUT], w[S::OUT];
  // ---- step 1: T(iy, n) = LSE_ix(x(iy, ix) + Ax(ix, n)) --------------------
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
  // ---- step 2: lse(jy, n) = LSE_iy(Ay(jy, iy) + T(iy, n)); epilogue --------
  // The block's new potentials are also collected transposed in OT (XT is
  // dead after step 1) and written out as whole [jx][iy] rows below.
  float* OT = XT;
  const int kOtLd = ny + 1;   // odd: the thread tile's column stores spread over banks
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
#pragma unroll
        for (int c = 0; c < RN; ++c) OT[(tn * RN + c) * kOtLd + jy] = nv[c];
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
          OT[(tn * RN + c) * kOtLd + jy] = nv;
          if (p.res_kind == kResRow) rmax = fmaxf(rmax, fabsf(exp2f(nv + lse) - p.marg[k]));
          if (p.res_kind == kResCol) rmax = fmaxf(rmax, fabsf(exp2f(p.old[k] + lse) - p.marg[k]));
        }
      }
    }
  }
  if (!kTail) {   // the transposed copy the next sweep stages: coalesced rows
    __syncthreads();
    const int ncol = min(NB, nx - jx0);
    float* dst = p.outT + (size_t)b * p.ld + (size_t)jx0 * ny;
    for (int r = tid / 32; r < ncol; r += NT / 32)
      for (int jy = tid % 32; jy < ny; jy += 32) dst[(size_t)r * ny + jy] = OT[r * kOtLd + jy];
  }
  if (kTail || p.res_kind != kResNone) {
    // NaN must win the max (batch.py:320 compares max <= tol, false for NaN)
    if (rmax != rmax) rmax = __int_as_float(0x7fc00000);
    atomicMax(&s_res, __float_as_uint(rmax));
    __syncthreads();
    if (tid == 0) atomic_max_nonneg(&p.res[b], __uint_as_float(s_res));
  }
  if (p.dbg) {
    __syncthreads();
    if (tid == 0) p.dbg[4 * cta + 2] = globaltimer_ns();
  }
}

// ---------------------------------------------------------------------------
// Split separable sweep for grids whose lane potential and Ay table do not fit
// one CTA's shared memory (the fused kernel above stages 2 n^2 floats): the
// two nested LSE-GEMMs become two kernels with T in global memory, each CTA
// owning one 64-row m block (kSepBlk = S::MT) of its step --
//   step 1 (lane, jx block, iy block):  T(iy, n) = LSE_ix(x(iy, ix) + Ax(ix, n))
//   step 2 (lane, jx block, jy block):  lse(jy, n) = LSE_iy(Ay(iy, jy) + T(iy, n))
// -- so shared memory is O(n * 96) floats: grids up to ~590 x 450.  Same
// arithmetic, estimate mode and tail weights as the fused kernel.
template <class S>
__host__ __device__ inline size_t sep_split1_floats(int nx) {
  return (size_t)nx * S::MT + (size_t)nx * S::NB + S::MT;     // XT block [ix][64], Ax block
}
template <class S>
__host__ __device__ inline size_t sep_split2_floats(int ny, bool tail) {
  return (size_t)ny * S::MT + (size_t)ny * S::NB * (tail ? 2 : 1) + S::MT;   // Ay block, T (, R)
}

template <class S, int kMode>
__global__ void __launch_bounds__(S::NT, 2) sep_step1_kernel(const SepParams p) {
  constexpr bool kTail = (kMode == kModeTail);
  constexpr int NB = S::NB, RN = S::RN, NT = S::NT, MB = S::MT;
  extern __shared__ __align__(16) float sep_smem[];
  const int nx = p.nx, ny = p.ny;
  float* XT = sep_smem;                 // [nx][MB]: x(iy0 + m, ix) transposed
  float* AX = XT + (size_t)nx * MB;     // [nx][NB]
  const int b = p.b0 + blockIdx.z;
  const int jx0 = blockIdx.x * NB, iy0 = blockIdx.y * MB;
  const int niy = min(MB, ny - iy0);
  const int tid = threadIdx.x, tn = tid % S::TN, tm = tid / S::TN;
  sep_stage_rows<NT>(AX, NB, p.ax_tab + jx0, (size_t)p.nblk * NB, nx, NB);
  cp_async_commit();
  pdl_wait();   // x is the previous sweep's output
  sep_stage_rows<NT>(XT, MB, p.xT + (size_t)b * p.ld + iy0, (size_t)ny, nx, niy);
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  pdl_launch_dependents();
  float mx[S::OUT], sm[S::OUT], w[S::OUT];
  bool done = false;
  if (!kTail && p.est_src != nullptr) {
    done = sep_estimate<S>(p, b, iy0, jx0, mx) &&
           (p.use_poly ? sep_lse_gemm<S, 0, true, true>(XT, MB, AX, nullptr, nx, 0, p.cinv, mx, sm, w)
                       : sep_lse_gemm<S, 0, false, true>(XT, MB, AX, nullptr, nx, 0, p.cinv, mx, sm, w));
    if (!done && p.redo) atomicAdd(p.redo, 1u);
  }
  if (done) {
  } else if (!kTail && p.use_poly)
    sep_lse_gemm<S, 0, true>(XT, MB, AX, nullptr, nx, 0, p.cinv, mx, sm, w);
  else
    sep_lse_gemm<S, kTail ? 1 : 0, false>(XT, MB, AX, nullptr, nx, 0, p.cinv, mx, sm, w);
  float* T = p.tg + ((size_t)b * p.nblk + blockIdx.x) * ny * NB;
  float* R = kTail ? p.rg + ((size_t)b * p.nblk + blockIdx.x) * ny * NB : nullptr;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int m = tm * 4 + a;
    if (m >= niy) continue;
#pragma unroll
    for (int c = 0; c < RN; ++c) {
      const int e = a * RN + c;
      T[(size_t)(iy0 + m) * NB + tn * RN + c] = lse_final(mx[e], sm[e]);
      if (kTail) R[(size_t)(iy0 + m) * NB + tn * RN + c] = (sm[e] > 0.f) ? w[e] / sm[e] : 0.f;
    }
  }
}

template <class S, int kMode>
__global__ void __launch_bounds__(S::NT, 2) sep_step2_kernel(const SepParams p) {
  constexpr bool kTail = (kMode == kModeTail);
  constexpr int NB = S::NB, RN = S::RN, NT = S::NT, MB = S::MT;
  extern __shared__ __align__(16) float sep_smem[];
  const int nx = p.nx, ny = p.ny, ldm = sep_ld(ny);
  float* AY = sep_smem;                 // [ny][MB]: Ay(iy, jy0 + m)
  float* T = AY + (size_t)ny * MB;      // [ny][NB]
  float* R = T + (size_t)ny * NB;       // [ny][NB], tail only
  __shared__ unsigned int s_res;
  const int b = p.b0 + blockIdx.z;
  const int jx0 = blockIdx.x * NB, jy0 = blockIdx.y * MB;
  const int njy = min(MB, ny - jy0);
  const int tid = threadIdx.x, tn = tid % S::TN, tm = tid / S::TN;
  if (tid == 0) s_res = 0u;
  sep_stage_rows<NT>(AY, MB, p.ay_tab + jy0, (size_t)ldm, ny, njy);
  cp_async_commit();
  pdl_wait();   // T is step 1's output
  const size_t tb = ((size_t)b * p.nblk + blockIdx.x) * ny * NB;
  sep_stage_rows<NT>(T, NB, p.tg + tb, (size_t)NB, ny, NB);
  if (kTail) sep_stage_rows<NT>(R, NB, p.rg + tb, (size_t)NB, ny, NB);
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  pdl_launch_dependents();
  float mx[S::OUT], sm[S::OUT], w[S::OUT];
  bool done = false;
  if (!kTail && p.est_src != nullptr) {
    done = sep_estimate<S>(p, b, jy0, jx0, mx) &&
           (p.use_poly ? sep_lse_gemm<S, 0, true, true>(AY, MB, T, R, ny, 0, p.cinv, mx, sm, w)
                       : sep_lse_gemm<S, 0, false, true>(AY, MB, T, R, ny, 0, p.cinv, mx, sm, w));
    if (!done && p.redo) atomicAdd(p.redo, 1u);
  }
  if (done) {
  } else if (!kTail && p.use_poly)
    sep_lse_gemm<S, 0, true>(AY, MB, T, R, ny, 0, p.cinv, mx, sm, w);
  else
    sep_lse_gemm<S, kTail ? 2 : 0, false>(AY, MB, T, R, ny, 0, p.cinv, mx, sm, w);
  float rmax = 0.f;
  const int jxb = jx0 + tn * RN;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int m = tm * 4 + a;
    if (m >= njy) continue;
    const int jy = jy0 + m;
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
        p.outT[(size_t)b * p.ld + (size_t)jx * ny + jy] = nv;   // the next sweep's layout
        if (p.res_kind == kResRow) rmax = fmaxf(rmax, fabsf(exp2f(nv + lse) - p.marg[k]));
        if (p.res_kind == kResCol) rmax = fmaxf(rmax, fabsf(exp2f(p.old[k] + lse) - p.marg[k]));
      }
    }
  }
  if (kTail || p.res_kind != kResNone) {
    if (rmax != rmax) rmax = __int_as_float(0x7fc00000);
    atomicMax(&s_res, __float_as_uint(rmax));
    __syncthreads();
    if (tid == 0) atomic_max_nonneg(&p.res[b], __uint_as_float(s_res));
  }
}

// Per-lane transpose [ny][nx] -> [nx][ny] of a lane-major potential (the
// initial log u of the separable path; later sweeps write both layouts).
__global__ void sep_transpose_kernel(const float* __restrict__ src, float* __restrict__ dst,
                                     int B, int ld, int nx, int ny) {
  const size_t n = (size_t)B * nx * ny;
  for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < n;
       e += (size_t)gridDim.x * blockDim.x) {
    const int b = (int)(e / ((size_t)nx * ny));
    const int k = (int)(e - (size_t)b * nx * ny);
    const int iy = k / nx, ix = k - iy * nx;
    dst[(size_t)b * ld + (size_t)ix * ny + iy] = src[(size_t)b * ld + k];
  }
}

// The factor tables of one grid, built once per solve: Ax(ix, jx) for jx up to
// nblk*NB (padded columns hold finite values; their outputs are never stored)
// and Ay(iy, jy) with a leading dimension of sep_ld(ny).
__global__ void sep_tables_kernel(float* ax_tab, float* ay_tab, int nx, int ny, int axcols,
                                  float ax, float ay) {
  const int ldy = sep_ld(ny);
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < nx * axcols + ny * ldy;
       e += gridDim.x * blockDim.x) {
    if (e < nx * axcols) {
      const int i = e / axcols, j = e - i * axcols;
      const float d = float(i - j);
      ax_tab[e] = ax * (d * d);
    } else {
      const int f = e - nx * axcols;
      const int i = f / ldy, j = f - i * ldy;
      const float d = float(i - j);
      ay_tab[f] = ay * (d * d);
    }
  }
}

}  // namespace skb
