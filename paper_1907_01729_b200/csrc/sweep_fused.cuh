// sweep_fused.cuh -- one fused row->column pass per Sinkhorn iteration for a
// stored cost shared by every lane (BASELINE config 2).
//
// The reference runs an iteration as two half-sweeps (batch.py:314-316):
//     log_v = log_nu - LSE_i(A + log_u)        (column sweep)
//     log_u = log_mu - LSE_j(A + log_v)        (row sweep)
// each with one exponential per cell.  Here the column sweep of iteration
// k+1 is folded into the row sweep of iteration k.  After row i of lane b is
// reduced, with t_j = A2[i,j] + v_j, m = max_j t_j, e_j = 2^(t_j - m) and
// S = sum_j e_j:
//     u_i = l2mu_i - (m + log2 S)                         (the row sweep)
//     P_ij = 2^(u_i + A2[i,j] + v_j) = e_j * (mu_i / S)   (the plan entries)
// so the plan's column marginal colsum_j = sum_i P_ij needs no further
// exponential: it is an FFMA per cell on the e_j already in registers.  Then
//     LSE_i(A2[:,j] + u) = log2(colsum_j) - v_j
//     v'_j = l2nu_j - LSE_i(...) = v_j + l2nu_j - log2(colsum_j)
// which is the reference's column update, and |colsum_j - nu_j| is its column
// residual (batch.py:303-309).  One exponential per cell per iteration instead
// of two: the MUFU roofline of the whole iteration halves.
//
// Range: every P_ij <= mu_i <= 1, so the sums cannot overflow.  Terms below
// 2^-126 flush to zero; they are negligible against colsum_j unless colsum_j
// itself is tiny, so the merge checks colsum_j >= 2^-60 (relevant terms are
// then >= 2^-60 * 2^-24 / d1 >> 2^-126) and otherwise flags the solve, which
// the host reruns with the exact two-half-sweep path.  The row reduction is
// exact two-pass (max, then one exponential per cell) in registers.
//
// Decomposition: a CTA has 16 warps, one lane each (a "group" of 16 lanes);
// every warp reduces the same cost row for its own lane, so a cost row is
// staged once in shared memory (cp.async.bulk, a ring of kFusedStages rows)
// and read by 16 lanes.  The (group, row) units are split evenly over one CTA
// per SM (stream-K); each CTA writes the column partials of every group
// segment it covers, and fused_merge_kernel sums them in ascending CTA order
// (deterministic, like the reference's ascending span merge, batch.py:198-201)
// and applies the column update.  Lane-major buffers: x[b*ld + j].
//
// The same kernel with kRowOnly and the transposed cost runs the first column
// sweep (v_1 from u_0, batch.py:315), where no plan exists yet.
#pragma once

#include "common.cuh"

#include <type_traits>

namespace skb {

constexpr int kFusedWarps = 16;    // max lanes per group = warps per CTA
// Lanes per group for a row of nq chunks: 16 warps while the row's registers
// (potentials, plan partials, exponentials: 6 per chunk) fit in 128, else 12
// warps with up to 168 registers.
// Per-sample rows up to 2048 columns (fused_ps_kernel only): 8 warps.
__host__ __device__ constexpr int fused_warps(int nq) { return nq <= 13 ? 16 : nq <= 16 ? 12 : 8; }
constexpr int kFusedStages = 8;    // cost rows in flight per CTA
constexpr int kFusedMaxChunks = 16;  // row length <= 1024 columns
constexpr int kFusedMaxCtas = 1024;   // CTAs of one fused launch (sms x CTAs per SM)
constexpr float kFusedMinColsum = 8.673617379884035e-19f;   // 2^-60

struct FusedParams {
  int B;                  // lanes
  int nrows;              // output rows of this pass (d1 main pass, d2 row-only pass)
  int rowlen;             // padded row length = 64 * nq (= leading dim of x and of part rows)
  int nq;                 // 64-column chunks per row (<= NQ)
  long long U;            // units = groups * nrows
  int nct;                // CTAs
  int maxseg;             // partial slots per CTA
  const float* a2;        // [>= nrows][rowlen] rows streamed through the ring: log2 cost
                          // (A2, or A2^T for kRowOnly), or the kernel K = 2^A2 (kLin)
  const float* a2log;     // [>= nrows][rowlen] log2 cost rows (kLin's exact fallback)
  const float* x;         // [B][rowlen] reduced-side potentials (log2)
  const float* target;    // [B][ldo] output-side log2 marginal
  const float* marg;      // [B][ldo] output-side linear marginal
  float* out;             // [B][ldo] output-side potentials
  int ldo;
  float* part;            // [nct][maxseg][16][rowlen] plan column partials (main pass)
  float* res;             // [B] row residual, atomic max (nullable)
  float* e0;              // [B][ldo] log2 E0 row terms (nullable)
  float e0_log2scale;     // log2(lambda * ln2): c = -A2 * lambda * ln2
  const int* status;      // abort if validation failed
  int* est_fail;          // kLin: more fallback rows than a warp can queue -> exact rerun
  float* vmax_out;        // block pass, first sweep: [B][rowlen] filled with -(the lane's max log u0)
};

struct FusedMergeParams {
  int B, nrows, rowlen;   // rowlen = padded output length (ld of v, part rows)
  int nw;                 // lanes per group of the fused pass
  long long U;
  int nct, maxseg;
  const float* part;
  const float* v_old;     // [B][rowlen] v_k
  float* v_new;           // [B][rowlen] v_{k+1}
  const float* target;    // [B][rowlen] l2nu
  const float* marg;      // [B][rowlen] nu
  float* res;             // [B] column residual, atomic max (nullable)
  int* est_fail;          // set when a column's plan mass is below 2^-60
  int b0;                 // first lane of this launch (grid.y <= 65535 lanes per launch)
};

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// shared-window (u32) address forms, computed once per CTA
__device__ __forceinline__ void bulk_g2s_s(uint32_t dst, const void* src, uint32_t bytes,
                                           uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx_s(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait_s(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint64_t lds64(uint32_t addr) {
  uint64_t v;
  asm volatile("ld.shared.b64 %0, [%1];" : "=l"(v) : "r"(addr) : "memory");
  return v;
}

// Ring-slot release count.  Relaxed: a warp only counts itself after
// __syncwarp, when every lane has consumed its shared-memory reads of the slot;
// the last one fences the async proxy before the bulk copy overwrites it.
__device__ __forceinline__ int atom_add_relaxed_cta(int* addr, int v) {
  int old;
  asm volatile("atom.relaxed.cta.shared::cta.add.u32 %0, [%1], %2;"
               : "=r"(old) : "r"(smem_u32(addr)), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__host__ __device__ inline long long fused_seg_start(long long U, int nct, int c) {
  return (long long)c * U / nct;
}

template <int NQ>
__host__ __device__ constexpr size_t fused_smem_bytes() {
  return (size_t)kFusedStages * NQ * 64 * 4 + kFusedStages * 8;
}

constexpr float kFusedEstLo = 8.673617379884035e-19f;   // 2^-60
constexpr float kFusedEstHi = 1.2676506002282294e30f;   // 2^100

// The rows of one (lane group, row range) segment.  The main pass shifts each
// row's exponentials by the row's previous log-sum-exp (target - old u_i):
// the potentials move little between iterations, so the sum stays in
// [2^-60, 2^100] and no max pass is needed; a row outside that range (or with
// no previous value) is redone with the exact two-pass reduction from the
// staged cost row.  The row-only pass is always exact.
constexpr int kFusedRedoMax = 32;   // queued log-domain fallback rows per warp and segment

template <int NQ, int NW, bool kRowOnly, bool kTail, bool kLin>
__device__ __forceinline__ void fused_segment(const FusedParams& p, const float* ring,
                                              uint32_t full_s, int* rel, int* redo, int& r, int& s,
                                              uint32_t& par, int n, int g, int i_begin, int i_end,
                                              int sidx) {
  constexpr bool kGuard = false;   // every pass is instantiated for its exact chunk count
  const int rowlen = p.rowlen;
  const int warp = warp_id(), lane = lane_id();
  const int b = g * NW + warp;
  const bool act = b < p.B;   // warp-uniform; idle warps compute on -inf and store nothing
  auto chunk_on = [&](int q) { return !kGuard || q < p.nq; };
  const uint32_t row_bytes = (uint32_t)rowlen * 4u;

  uint64_t xv[NQ], acc[NQ];
  const float* x_b = p.x + (size_t)b * rowlen + 2 * lane;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    float2 v2 = make_float2(neg_inf(), neg_inf());
    if (act && chunk_on(q)) v2 = __ldg(reinterpret_cast<const float2*>(x_b + 64 * q));
    xv[q] = pk2(v2.x, v2.y);
    acc[q] = 0ull;
  }
  // kLin: the lane's potentials as X_j = 2^(v_j - vmax) <= 1, so a row's terms
  // 2^(A2_ij + v_j - vmax) = K_ij * X_j are products (no exponential per cell)
  float vmax = neg_inf();
  if constexpr (kLin) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) vmax = fmax3(vmax, lo2(xv[q]), hi2(xv[q]));
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, off));
    vmax = fmaxf(vmax, kNegBig);
#pragma unroll
    for (int q = 0; q < NQ; ++q) xv[q] = pk2(ex2(lo2(xv[q]) - vmax), ex2(hi2(xv[q]) - vmax));
  }
  // per-row scalars, 32 rows per window, prefetched one window ahead: target,
  // linear marginal and (main pass) the previous potential of the row
  const float* tg_b = p.target + (size_t)b * p.ldo;
  const float* mg_b = p.marg + (size_t)b * p.ldo;
  float* out_b = p.out + (size_t)b * p.ldo;
  float* e0_b = kTail ? p.e0 + (size_t)b * p.ldo : nullptr;
  auto ld_win = [&](int base, float& tw, float& mw, float& ow) {
    const int i = base + lane;
    const bool ok = act && i < i_end;
    tw = ok ? __ldg(tg_b + i) : 0.f;
    mw = (!kRowOnly && ok) ? __ldg(mg_b + i) : 0.f;
    ow = (!kRowOnly && ok) ? out_b[i] : 0.f;
  };
  float tw, mw, ow, tw_n, mw_n, ow_n;
  ld_win(i_begin, tw, mw, ow);
  ld_win(i_begin + 32, tw_n, mw_n, ow_n);
  float rres = 0.f, ob = 0.f;
  int nredo = 0;
  const float* ring_l = ring + 2 * lane;

  // two rows per trip: the accumulators alternate between two register sets
  // instead of being copied back at every loop edge
#pragma unroll 2
  for (int i = i_begin; i < i_end; ++i) {
    const int wi = (i - i_begin) & 31;
    const float tgt = __shfl_sync(0xffffffffu, tw, wi);
    const float mgl = __shfl_sync(0xffffffffu, mw, wi);
    const float uold = __shfl_sync(0xffffffffu, ow, wi);
    if (wi == 31) {
      tw = tw_n;
      mw = mw_n;
      ow = ow_n;
      ld_win(i + 33, tw_n, mw_n, ow_n);
    }
    const float* row = ring_l + s * rowlen;
    mbar_wait_s(full_s + 8u * (uint32_t)s, par);
    uint64_t t[NQ];
    float ms, S = 0.f;
    bool exact;
    // row epilogue: u_i, plan column partials acc += e * mu_i / S, tail terms
    // (called at the end of each branch below, so t never merges across them)
    auto finish = [&](float ms, float S) {
      const float lse = S > 0.f ? ms + lg2(S) : neg_inf();
      const float o = sweep_out(tgt, lse);
      if (lane == wi) ob = o;   // stored 32 rows at a time below
      if constexpr (!kRowOnly) {
        const float a = S > 0.f ? mgl * rcp_approx(S) : 0.f;   // mu_i / S: P_ij = e_j * a
        const uint64_t av2 = pk2(a, a);
#pragma unroll
        for (int q = 0; q < NQ; ++q) ffma2_acc(acc[q], t[q], av2);
        if constexpr (kTail) {
          rres = fmaxf(rres, fabsf(exp2f(o + lse) - mgl));
          // E0 row term: a * sum_j e_j * c_ij, c = -A2 * lambda * ln2
          float qs = 0.f;
#pragma unroll
          for (int q = 0; q < NQ; ++q) {
            const float2 av = *reinterpret_cast<const float2*>(row + 64 * q);
            // padding columns hold A2 = -inf
            qs = fmaf(lo2(t[q]), av.x > -3.0e38f ? -av.x : 0.f, qs);
            qs = fmaf(hi2(t[q]), av.y > -3.0e38f ? -av.y : 0.f, qs);
          }
#pragma unroll
          for (int off = 16; off > 0; off >>= 1) qs += __shfl_xor_sync(0xffffffffu, qs, off);
          if (act && lane == 0)
            e0_b[i] = (a > 0.f && qs > 0.f) ? log2f(a) + log2f(qs) + p.e0_log2scale : neg_inf();
        }
      }
    };

    if constexpr (kLin) {
      uint64_t s0 = 0ull, s1 = 0ull;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const float2 k2 = *reinterpret_cast<const float2*>(row + 64 * q);
        t[q] = fmul2(pk2(k2.x, k2.y), xv[q]);
        if (q & 1) s1 = fadd2(s1, t[q]);
        else       s0 = fadd2(s0, t[q]);
      }
      const uint64_t s01 = fadd2(s0, s1);
      S = lo2(s01) + hi2(s01);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) S += __shfl_xor_sync(0xffffffffu, S, off);
      // a row whose terms underflow (S < 2^-60) contributes nothing here and is
      // queued for the log-domain fallback after the segment (idle warps: all -inf)
      const bool ok = !act || S >= kFusedEstLo;
      if (!ok && lane == 0) {
        if (nredo < kFusedRedoMax) redo[nredo] = i;
        else *p.est_fail = 1;
      }
      nredo += ok ? 0 : 1;
      const float lse = vmax + lg2(S);
      if (lane == wi) ob = sweep_out(tgt, lse);
      const float a = ok ? mgl * rcp_approx(S) : 0.f;   // mu_i / S: P_ij = e_j * a
      const uint64_t av2 = pk2(a, a);
#pragma unroll
      for (int q = 0; q < NQ; ++q) ffma2_acc(acc[q], t[q], av2);
    } else {
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        if (chunk_on(q)) {
          const float2 a = *reinterpret_cast<const float2*>(row + 64 * q);
          t[q] = fadd2(pk2(a.x, a.y), xv[q]);
        }
      }
      ms = tgt - uold;
      exact = kRowOnly || !(ms > -3.0e38f && ms < 3.0e38f);
      if (!exact) {
        const uint64_t nm = pk2(-ms, -ms);
        uint64_t s0 = 0ull, s1 = 0ull;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const uint64_t d = fadd2(t[q], nm);
          t[q] = pk2(ex2(lo2(d)), ex2(hi2(d)));
          if (q & 1) s1 = fadd2(s1, t[q]);
          else       s0 = fadd2(s0, t[q]);
        }
        const uint64_t s01 = fadd2(s0, s1);
        S = lo2(s01) + hi2(s01);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) S += __shfl_xor_sync(0xffffffffu, S, off);
        // (idle warps never redo: their rows are all -inf)
        exact = act && !(S >= kFusedEstLo && S <= kFusedEstHi);
      }
      if (exact) {   // warp-uniform; rare after the first iterations
        float m0 = neg_inf(), m1 = neg_inf();
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          if (chunk_on(q)) {
            const float2 a = *reinterpret_cast<const float2*>(row + 64 * q);
            t[q] = fadd2(pk2(a.x, a.y), xv[q]);
            if (q & 1) m1 = fmax3(m1, lo2(t[q]), hi2(t[q]));
            else       m0 = fmax3(m0, lo2(t[q]), hi2(t[q]));
          }
        }
        float m = fmaxf(m0, m1);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
        ms = fmaxf(m, kNegBig);   // an all -inf row gives e = 0, S = 0
        const uint64_t nm = pk2(-ms, -ms);
        uint64_t s0 = 0ull, s1 = 0ull;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          if (chunk_on(q)) {
            const uint64_t d = fadd2(t[q], nm);
            t[q] = pk2(ex2(lo2(d)), ex2(hi2(d)));
            if (q & 1) s1 = fadd2(s1, t[q]);
            else       s0 = fadd2(s0, t[q]);
          }
        }
        const uint64_t s01 = fadd2(s0, s1);
        S = lo2(s01) + hi2(s01);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) S += __shfl_xor_sync(0xffffffffu, S, off);
      }
      finish(ms, S);
    }
    if (wi == 31 || i + 1 == i_end) {   // this window's u_i, one coalesced store
      const int i0 = i - wi;
      if (act && lane <= wi) out_b[i0 + lane] = ob;
    }
    // release the slot; the last warp to do so refills it with the row
    // kFusedStages stream positions ahead (no producer warp, no waiting)
    __syncwarp();
    if (lane == 0) {
      if (atom_add_relaxed_cta(&rel[s], 1) == NW - 1) {
        rel[s] = 0;
        if (r + kFusedStages < n) {
          fence_proxy_async();
          int nrow = i + kFusedStages;
          while (nrow >= p.nrows) nrow -= p.nrows;
          const uint32_t bar = full_s + 8u * (uint32_t)s;
          mbar_arrive_expect_tx_s(bar, row_bytes);
          bulk_g2s_s(smem_u32(ring + s * rowlen), p.a2 + (size_t)nrow * rowlen, row_bytes, bar);
        }
      }
    }
    ++r;
    if (++s == kFusedStages) {
      s = 0;
      par ^= 1u;
    }
  }

  if constexpr (kLin) {
    // queued rows in the log domain, from L2: A2 row + potentials, exact two-pass
    __syncwarp();
    const int nq_redo = nredo < kFusedRedoMax ? nredo : kFusedRedoMax;
    for (int k = 0; k < nq_redo; ++k) {
      const int i = redo[k];
      const float* arow = p.a2log + (size_t)i * rowlen + 2 * lane;
      uint64_t t[NQ];
      float m0 = neg_inf(), m1 = neg_inf();
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const float2 a = __ldg(reinterpret_cast<const float2*>(arow + 64 * q));
        const float2 v = __ldg(reinterpret_cast<const float2*>(x_b + 64 * q));
        t[q] = fadd2(pk2(a.x, a.y), pk2(v.x, v.y));
        if (q & 1) m1 = fmax3(m1, lo2(t[q]), hi2(t[q]));
        else       m0 = fmax3(m0, lo2(t[q]), hi2(t[q]));
      }
      float m = fmaxf(m0, m1);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
      const float ms = fmaxf(m, kNegBig);
      const uint64_t nm = pk2(-ms, -ms);
      uint64_t s0 = 0ull, s1 = 0ull;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const uint64_t d = fadd2(t[q], nm);
        t[q] = pk2(ex2(lo2(d)), ex2(hi2(d)));
        if (q & 1) s1 = fadd2(s1, t[q]);
        else       s0 = fadd2(s0, t[q]);
      }
      const uint64_t s01 = fadd2(s0, s1);
      float S = lo2(s01) + hi2(s01);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) S += __shfl_xor_sync(0xffffffffu, S, off);
      const float lse = S > 0.f ? ms + lg2(S) : neg_inf();
      if (lane == 0) out_b[i] = sweep_out(__ldg(tg_b + i), lse);
      const float a = S > 0.f ? __ldg(mg_b + i) * rcp_approx(S) : 0.f;
      const uint64_t av2 = pk2(a, a);
#pragma unroll
      for (int q = 0; q < NQ; ++q) ffma2_acc(acc[q], t[q], av2);
    }
  }
  if constexpr (!kRowOnly) {
    if (act) {
      float* dst = p.part + (((size_t)blockIdx.x * p.maxseg + sidx) * NW + warp) * (size_t)rowlen;
#pragma unroll
      for (int q = 0; q < NQ; ++q)
        *reinterpret_cast<float2*>(dst + 2 * lane + 64 * q) = make_float2(lo2(acc[q]), hi2(acc[q]));
    }
  }
  if constexpr (kTail) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) rres = fmaxf(rres, __shfl_xor_sync(0xffffffffu, rres, off));
    if (act && lane == 0) atomic_max_nonneg(&p.res[b], rres);
  }
}

// NQ chunks of 64 columns per row, instantiated for the exact chunk count
// (no per-chunk guards, so the chunks interleave freely).
// kTail (check and last iterations): row residual + E0 row terms as well.
// kLin (the other main passes): the ring streams K = 2^A2 rows and a row's
// terms are K_ij * 2^(v_j - vmax_b): products instead of exponentials.
template <int NQ, bool kRowOnly, bool kTail, bool kLin = false, int NW = fused_warps(NQ)>
__global__ void __launch_bounds__(NW * 32, 1) fused_pass_kernel(const FusedParams p) {
  extern __shared__ __align__(128) unsigned char fsm[];
  __shared__ int rel[kFusedStages];   // warps that released each ring slot
  __shared__ int redo_rows[kLin ? NW * kFusedRedoMax : 1];
  const int rowlen = p.rowlen;
  float* ring = reinterpret_cast<float*>(fsm);
  uint64_t* full = reinterpret_cast<uint64_t*>(fsm + (size_t)kFusedStages * rowlen * 4);
  const long long u0 = fused_seg_start(p.U, p.nct, blockIdx.x);
  const long long u1 = fused_seg_start(p.U, p.nct, blockIdx.x + 1);
  const int n = (int)(u1 - u0);

  if (threadIdx.x == 0) {
    for (int s = 0; s < kFusedStages; ++s) {
      mbar_init(&full[s], 1);
      rel[s] = 0;
    }
    fence_barrier_init();
  }
  __syncthreads();
  // the cost rows do not depend on the previous launch: start streaming them
  // before the programmatic-dependent-launch wait
  const int npre = n < kFusedStages ? n : kFusedStages;
  if (threadIdx.x == 0) {
    const uint32_t row_bytes = (uint32_t)rowlen * 4u;
    int row = (int)(u0 % p.nrows);
    for (int r = 0; r < npre; ++r) {
      mbar_arrive_expect_tx(&full[r], row_bytes);
      bulk_g2s(ring + (size_t)r * rowlen, p.a2 + (size_t)row * rowlen, row_bytes, &full[r]);
      if (++row == p.nrows) row = 0;
    }
  }
  pdl_wait();
  if (p.status != nullptr && *p.status != 0) {   // validation failed: drain and leave
    if (threadIdx.x == 0)
      for (int r = 0; r < npre; ++r) mbar_wait(&full[r], 0);
    __syncthreads();
    return;
  }

  int r = 0, s = 0;   // position in this CTA's row stream, its ring slot and phase
  uint32_t par = 0;
  const uint32_t full_s = smem_u32(full);
  long long u = u0;
  const int g_first = (int)(u0 / p.nrows);
  while (u < u1) {
    const int g = (int)(u / p.nrows);
    const int i_begin = (int)(u - (long long)g * p.nrows);
    const long long seg_end = (long long)(g + 1) * p.nrows < u1 ? (long long)(g + 1) * p.nrows : u1;
    const int i_end = (int)(seg_end - (long long)g * p.nrows);
    fused_segment<NQ, NW, kRowOnly, kTail, kLin>(p, ring, full_s, rel,
                                                 redo_rows + (kLin ? warp_id() * kFusedRedoMax : 0),
                                                 r, s, par, n, g, i_begin, i_end, g - g_first);
    u = seg_end;
  }
  pdl_launch_dependents();
}

// ---------------------------------------------------------------------------
// Per-sample costs (BASELINE config 4): the same fused row->column pass over
// each lane's own C_b, which is streamed from HBM once per iteration instead
// of twice (the two half-sweeps each read it).  Every warp streams its own
// lane's rows through a private ring of kPsStages slots (cp.async.bulk, one
// mbarrier per slot) and refills a slot as soon as it has consumed it.  Rows
// are reduced in the log domain, t_j = c_ij * (-log2e / lambda) + v_j, with
// the previous-lse shift and the exact fallback of the shared-cost pass.
constexpr int kPsStages = 4;
constexpr int kPsMaxChunks = 32;   // per-sample rows <= 2048 columns
// CTAs per SM of the per-sample pass: short rows (<= 256 columns) are bound by
// each warp's serial per-row chain, so two CTAs (32 warps) share an SM
__host__ __device__ constexpr int ps_ctas_per_sm(int nq) { return nq <= 4 ? 2 : 1; }
// ring slots per warp: ~192 KB of rows in flight per SM whatever the row
// length, capped at 32 (4 for 1024-column rows, 3 above)
__host__ __device__ constexpr int ps_stages(int nq) {
  return nq <= 16 ? (196608 / ps_ctas_per_sm(nq) / ((nq <= 13 ? 16 : 12) * nq * 256) > 32
                         ? 32
                         : (196608 / ps_ctas_per_sm(nq) / ((nq <= 13 ? 16 : 12) * nq * 256) <
                                    kPsStages
                                ? kPsStages
                                : 196608 / ps_ctas_per_sm(nq) / ((nq <= 13 ? 16 : 12) * nq * 256)))
                  : 3;
}

template <int NQ>
__host__ __device__ constexpr size_t fused_ps_smem_bytes() {
  return (size_t)fused_warps(NQ) * ps_stages(NQ) * (NQ * 64 * 4 + 8);
}

// kHalves = 2 or 4 (rows of 2049-4096 / 4097-8192 columns): that many warps
// per lane, each streaming and holding one slice of every row; the row's sums
// and maxima are combined through shared memory (fixed slice order, so every
// warp of the lane gets the same value) behind a named barrier per exchange.
template <int NQ, bool kTail, int NW = fused_warps(NQ), int kHalves = 1>
__global__ void __launch_bounds__(NW * 32, ps_ctas_per_sm(NQ)) fused_ps_kernel(const FusedParams p, const float* cost,
                                                              int d2, int ldc, float kscale) {
  extern __shared__ __align__(128) unsigned char fsm[];
  constexpr int rowlen = NQ * 64;          // columns held by one warp
  constexpr int kPsStages = ps_stages(NQ);
  constexpr int LPG = NW / kHalves;        // lanes per group
  const int warp = warp_id(), lane = lane_id();
  const int lw = warp % LPG, half = warp / LPG;
  const int col0 = half * rowlen;          // this warp's first column
  __shared__ float xch[kHalves > 1 ? LPG : 1][2][kHalves];   // [lane][parity][slice]
  int xc = 0;
  // exchange v among the lane's warps: parity double-buffering makes one
  // barrier per exchange enough (a warp cannot pass the next barrier before
  // every partner has read this one's values)
  auto exchange = [&](float v) -> int {
    const int par = xc & 1;
    ++xc;
    if (lane == 0) xch[lw][par][half] = v;
    asm volatile("bar.sync %0, %1;" ::"r"(1 + lw), "r"(32 * kHalves) : "memory");
    return par;
  };
  auto pair_sum = [&](float v) -> float {
    if constexpr (kHalves == 1) {
      return v;
    } else {
      const int par = exchange(v);
      float t = xch[lw][par][0];
#pragma unroll
      for (int h = 1; h < kHalves; ++h) t += xch[lw][par][h];
      return t;
    }
  };
  auto pair_max = [&](float v) -> float {
    if constexpr (kHalves == 1) {
      return v;
    } else {
      const int par = exchange(v);
      float t = xch[lw][par][0];
#pragma unroll
      for (int h = 1; h < kHalves; ++h) t = fmaxf(t, xch[lw][par][h]);
      return t;
    }
  };
  float* ring = reinterpret_cast<float*>(fsm) + (size_t)warp * kPsStages * rowlen;
  uint64_t* full = reinterpret_cast<uint64_t*>(fsm + (size_t)NW * kPsStages * rowlen * 4) +
                   warp * kPsStages;
  const long long u0 = fused_seg_start(p.U, p.nct, blockIdx.x);
  const long long u1 = fused_seg_start(p.U, p.nct, blockIdx.x + 1);
  const int n = (int)(u1 - u0);
  const int nrows = p.nrows;
  // cost rows of ldc floats (ldc = d2, or d2 rounded up to 4 in the solver's
  // zero-padded copy when d2 % 4 != 0: bulk copies move whole 16-byte units)
  const int ncopy = ldc - col0 < rowlen ? (ldc - col0 > 0 ? ldc - col0 : 0) : rowlen;
  const uint32_t row_bytes = (uint32_t)ncopy * 4u;   // this warp's part of a row
  const size_t lane_cells = (size_t)nrows * ldc;

  // columns past d2 are never written by the copies: zero them once so the
  // -inf potentials there meet a finite cost
  for (int k = lane; k < kPsStages * rowlen; k += 32)
    if ((k % rowlen) >= ncopy) ring[k] = 0.f;
  if (lane == 0) {
    for (int st = 0; st < kPsStages; ++st) mbar_init(&full[st], 1);
    fence_barrier_init();
  }
  __syncwarp();
  // producer state of this warp: stream position, group and row it loads next
  int pp = 0, pg = (int)(u0 / nrows), pi = (int)(u0 % nrows);
  auto produce = [&]() {   // lane 0: position pp into slot pp % kPsStages
    const int st = pp % kPsStages;
    const int b = pg * LPG + lw;
    if (b < p.B && row_bytes > 0) {
      mbar_arrive_expect_tx(&full[st], row_bytes);
      bulk_g2s(ring + st * rowlen, cost + b * lane_cells + (size_t)pi * ldc + col0, row_bytes,
               &full[st]);
    } else {
      mbar_arrive(&full[st]);   // idle lane: complete the phase without data
    }
    ++pp;
    if (++pi == nrows) {
      pi = 0;
      ++pg;
    }
  };
  const int npre = n < kPsStages ? n : kPsStages;
  if (lane == 0)
    for (int k = 0; k < npre; ++k) produce();   // the cost does not depend on the previous launch
  pdl_wait();
  const bool dead = p.status != nullptr && *p.status != 0;

  int r = 0;
  long long u = u0;
  const int g_first = (int)(u0 / nrows);
  const uint64_t ks2 = pk2(kscale, kscale);
  while (u < u1) {
    const int g = (int)(u / nrows);
    const int i_begin = (int)(u - (long long)g * nrows);
    const long long seg_end = (long long)(g + 1) * nrows < u1 ? (long long)(g + 1) * nrows : u1;
    const int i_end = (int)(seg_end - (long long)g * nrows);
    const int b = g * LPG + lw;
    const bool act = b < p.B && !dead;

    uint64_t xv[NQ], acc[NQ];
    const float* x_b = p.x + (size_t)b * p.rowlen + col0 + 2 * lane;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      float2 v2 = make_float2(neg_inf(), neg_inf());
      if (act && col0 + 2 * lane + 64 * q < d2)
        v2 = __ldg(reinterpret_cast<const float2*>(x_b + 64 * q));
      xv[q] = pk2(v2.x, v2.y);
      acc[q] = 0ull;
    }
    const float* tg_b = p.target + (size_t)b * p.ldo;
    const float* mg_b = p.marg + (size_t)b * p.ldo;
    float* out_b = p.out + (size_t)b * p.ldo;
    float* e0_b = kTail ? p.e0 + (size_t)b * p.ldo : nullptr;
    auto ld_win = [&](int base, float& tw, float& mw, float& ow) {
      const int i = base + lane;
      const bool ok = act && i < i_end;
      tw = ok ? __ldg(tg_b + i) : 0.f;
      mw = ok ? __ldg(mg_b + i) : 0.f;
      ow = ok ? out_b[i] : 0.f;
    };
    float tw, mw, ow, tw_n, mw_n, ow_n;
    ld_win(i_begin, tw, mw, ow);
    ld_win(i_begin + 32, tw_n, mw_n, ow_n);
    float rres = 0.f, ob = 0.f;

    for (int i = i_begin; i < i_end; ++i, ++r) {
      const int wi = (i - i_begin) & 31;
      const float tgt = __shfl_sync(0xffffffffu, tw, wi);
      const float mgl = __shfl_sync(0xffffffffu, mw, wi);
      const float uold = __shfl_sync(0xffffffffu, ow, wi);
      if (wi == 31) {
        tw = tw_n;
        mw = mw_n;
        ow = ow_n;
        ld_win(i + 33, tw_n, mw_n, ow_n);
      }
      const int st = r % kPsStages;
      mbar_wait(&full[st], (uint32_t)((r / kPsStages) & 1));
      const float* row = ring + st * rowlen + 2 * lane;
      uint64_t t[NQ];
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const float2 c2 = *reinterpret_cast<const float2*>(row + 64 * q);
        t[q] = ffma2(pk2(c2.x, c2.y), ks2, xv[q]);
      }
      float ms = tgt - uold;
      bool exact = !(ms > -3.0e38f && ms < 3.0e38f);
      float S = 0.f;
      if (!exact) {
        const uint64_t nm = pk2(-ms, -ms);
        uint64_t s0 = 0ull, s1 = 0ull;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const uint64_t d = fadd2(t[q], nm);
          t[q] = pk2(ex2(lo2(d)), ex2(hi2(d)));
          if (q & 1) fadd2_acc(s1, t[q]);
          else       fadd2_acc(s0, t[q]);
        }
        const uint64_t s01 = fadd2(s0, s1);
        S = lo2(s01) + hi2(s01);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) S += __shfl_xor_sync(0xffffffffu, S, off);
        S = pair_sum(S);
        exact = act && !(S >= kFusedEstLo && S <= kFusedEstHi);
      }
      if (exact) {   // warp-uniform; the first iteration and rare rows after it
        float m0 = neg_inf(), m1 = neg_inf();
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const float2 c2 = *reinterpret_cast<const float2*>(row + 64 * q);
          t[q] = ffma2(pk2(c2.x, c2.y), ks2, xv[q]);
          if (q & 1) m1 = fmax3(m1, lo2(t[q]), hi2(t[q]));
          else       m0 = fmax3(m0, lo2(t[q]), hi2(t[q]));
        }
        float m = fmaxf(m0, m1);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
        m = pair_max(m);
        ms = fmaxf(m, kNegBig);
        const uint64_t nm = pk2(-ms, -ms);
        uint64_t s0 = 0ull, s1 = 0ull;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const uint64_t d = fadd2(t[q], nm);
          t[q] = pk2(ex2(lo2(d)), ex2(hi2(d)));
          if (q & 1) fadd2_acc(s1, t[q]);
          else       fadd2_acc(s0, t[q]);
        }
        const uint64_t s01 = fadd2(s0, s1);
        S = lo2(s01) + hi2(s01);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) S += __shfl_xor_sync(0xffffffffu, S, off);
        S = pair_sum(S);
      }
      const float lse = S > 0.f ? ms + lg2(S) : neg_inf();
      const float o = sweep_out(tgt, lse);
      if (lane == wi) ob = o;
      const float a = S > 0.f ? mgl * rcp_approx(S) : 0.f;   // mu_i / S: P_ij = e_j * a
      const uint64_t av2 = pk2(a, a);
#pragma unroll
      for (int q = 0; q < NQ; ++q) ffma2_acc(acc[q], t[q], av2);
      if constexpr (kTail) {
        rres = fmaxf(rres, fabsf(exp2f(o + lse) - mgl));
        float qs = 0.f;   // E0 row term: a * sum_j e_j * c_ij
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const float2 c2 = *reinterpret_cast<const float2*>(row + 64 * q);
          qs = fmaf(lo2(t[q]), c2.x, qs);
          qs = fmaf(hi2(t[q]), c2.y, qs);
        }
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) qs += __shfl_xor_sync(0xffffffffu, qs, off);
        qs = pair_sum(qs);
        if (act && half == 0 && lane == 0)
          e0_b[i] = (a > 0.f && qs > 0.f) ? log2f(a) + log2f(qs) : neg_inf();
      }
      if (wi == 31 || i + 1 == i_end) {   // this window's u_i, one coalesced store
        if (act && half == 0 && lane <= wi) out_b[i - wi + lane] = ob;
      }
      // refill the slot just consumed with the position kPsStages ahead
      __syncwarp();
      if (lane == 0 && pp < n) {
        fence_proxy_async();
        produce();
      }
    }
    if (act) {
      float* dst = p.part + (((size_t)blockIdx.x * p.maxseg + (g - g_first)) * LPG + lw) *
                                (size_t)p.rowlen + col0;
#pragma unroll
      for (int q = 0; q < NQ; ++q)
        if (col0 + 2 * lane + 64 * q < p.rowlen)
          *reinterpret_cast<float2*>(dst + 2 * lane + 64 * q) = make_float2(lo2(acc[q]), hi2(acc[q]));
    }
    if constexpr (kTail) {
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) rres = fmaxf(rres, __shfl_xor_sync(0xffffffffu, rres, off));
      if (act && lane == 0) atomic_max_nonneg(&p.res[b], rres);
    }
    u = seg_end;
  }
  pdl_launch_dependents();
}

// ---------------------------------------------------------------------------
// The linear rows as two register-blocked GEMMs per block of 16 cost rows
// (fgemm_pass_kernel, the default for the non-check iterations of shared
// costs with d <= 1024).  A CTA owns 16 lanes (b) and walks blocks of 16 rows
// (i) of K = 2^A2, staged in shared memory (cp.async.bulk, double buffered):
//   S[i][b] = sum_j K[i][j] X[b][j]      16 x 16 outputs, the j range split
//                                        over 16 thread slices (4x4 blocking)
//   u, a[i][b] = mu / S                   one thread per output
//   T[b][j] += sum_i K[i][j] a[i][b]      every thread 4 lanes x NQ columns,
//                                        held in registers for the segment
// X[b][j] T[b][j] = sum_i P_ij is the plan column partial the merge kernel
// sums, exactly as the warp-per-row pass writes it.  There are no per-row shuffle reductions, so
// the loop is a plain FFMA2 / LDS.128 stream.  A row block with any S below
// 2^-60 (terms may have flushed) flags the solve for the exact rerun.
constexpr int kFgRows = 16;     // cost rows per block
constexpr int kFgLanes = 16;    // lanes per CTA
constexpr int kFgThreads = 256;

// Shared-memory strides chosen so the LDS.128s of a warp hit 8 distinct 16-byte
// bank groups: K rows padded by 8 floats (a thread's 4 rows interleaved by 4),
// X lane-pair rows carry a 4-float gap after every j slice plus 4 floats of pad.
__host__ __device__ constexpr int fg_stride(int nq) { return nq * 64 + 8; }
__host__ __device__ constexpr int fg_xstride(int nq) { return 2 * nq * 64 + 4 * 16 + 4; }

template <int NQ>
__host__ __device__ constexpr size_t fg_smem_bytes() {
  return (size_t)(kFgLanes / 2 * fg_xstride(NQ)            // X: 8 interleaved lane pairs
                  + 2 * kFgRows * fg_stride(NQ)            // two K blocks
                  + 16 * kFgRows * kFgLanes               // GEMM-1 slice partials
                  + kFgRows * kFgLanes + kFgLanes) * 4     // a, vmax
         + 2 * 8;                                         // mbarriers
}

// kTail (check and last iterations): GEMM 1 also accumulates
// SE = (K o C) X with c = -log2(K) * lambda ln2 recovered per cell, and the
// epilogue writes the row residual and the E0 row term a_i SE_i.
// kMode 0: an iteration; 1: a check / last iteration (kTail); 2: the first
// column sweep from u0 (kFirst): no GEMM 1, a_i = 2^(u0_i - umax_b) on the
// support, T = K^T a = 2^(-umax_b) sum_i K_ij 2^(u0_i), and -umax_b written to
// vmax_out so the merge's v' = v + l2nu - log2(T) starts from v = -umax_b.
template <int NQ, int kMode>
__global__ void __launch_bounds__(kFgThreads, 1) fgemm_pass_kernel(const FusedParams p, int nrb) {
  constexpr bool kTail = kMode == 1;
  constexpr bool kFirst = kMode == 2;
  extern __shared__ __align__(128) unsigned char fsm[];
  constexpr int STR = fg_stride(NQ);
  constexpr int XSTR = fg_xstride(NQ);    // a lane pair's interleaved row
  constexpr int SL = NQ * 4;              // j slice length (DP / 16)
  // X position of column j in a pair row: 2 j plus a 4-float gap per slice
  auto xpos = [](int j) { return 2 * j + 4 * (j / SL); };
  constexpr int DP = NQ * 64;
  float* Xs = reinterpret_cast<float*>(fsm);               // [8 lane pairs][XSTR]
  float* Ks = Xs + kFgLanes / 2 * XSTR;                     // [2][16 rows][STR]
  float* Sred = Ks + 2 * kFgRows * STR;                     // [16 slices][256]
  float* As = Sred + 16 * kFgRows * kFgLanes;               // [16 rows][16 lanes]
  float* Vm = As + kFgRows * kFgLanes;                      // [16]
  uint64_t* bar = reinterpret_cast<uint64_t*>(Vm + kFgLanes);
  const int t = threadIdx.x, warp = warp_id(), lane = lane_id();
  const long long u0 = fused_seg_start(p.U, p.nct, blockIdx.x);
  const long long u1 = fused_seg_start(p.U, p.nct, blockIdx.x + 1);
  const int n = (int)(u1 - u0);
  const uint32_t row_bytes = DP * 4u;

  if (t == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_barrier_init();
  }
  __syncthreads();
  // stream position k -> row block (u0 + k) % nrb; thread 0 issues its 16 row copies
  auto issue = [&](int k) {
    const int rb = (int)((u0 + k) % nrb);
    const int st = k & 1;
    mbar_arrive_expect_tx(&bar[st], kFgRows * row_bytes);
    for (int r = 0; r < kFgRows; ++r)
      bulk_g2s(Ks + (st * kFgRows + r) * STR, p.a2 + (size_t)(rb * kFgRows + r) * DP, row_bytes,
               &bar[st]);
  };
  if (t == 0) {
    issue(0);
    if (n > 1) issue(1);
  }
  pdl_wait();
  const bool dead = p.status != nullptr && *p.status != 0;

  // GEMM-1 roles: slice of the j range, 4 rows, 4 lanes
  const int ks = t >> 4, rq = (t >> 2) & 3, lq = t & 3;
  // GEMM-2 roles: 4 lanes, columns jc + 64 k
  const int l4 = t >> 6, jc = t & 63;
  int k = 0;   // stream position
  long long u = u0;
  const int g_first = (int)(u0 / nrb);
  while (u < u1) {
    const int g = (int)(u / nrb);
    const long long seg_end = (long long)(g + 1) * nrb < u1 ? (long long)(g + 1) * nrb : u1;
    const int b0 = g * kFgLanes;
    // this group's potentials as X = 2^(v - vmax) (warp w: lanes 2w, 2w+1)
    __syncthreads();
    if constexpr (kFirst) {   // umax_b over log u0; X = 1 (the partials are T itself)
      for (int h = 0; h < 2; ++h) {
        const int l = warp * 2 + h, b = b0 + l;
        float m = kNegBig;
        if (b < p.B)
          for (int i = lane; i < p.nrows; i += 32) m = fmaxf(m, p.out[(size_t)b * p.ldo + i]);
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
        for (int j = lane; j < DP; j += 32) Xs[(l >> 1) * XSTR + xpos(j) + (l & 1)] = 1.f;
        if (lane == 0) Vm[l] = m;
        // the group's CTA holding row block 0 publishes -umax as the merge's v
        if (b < p.B && (u - (long long)g * nrb) == 0)
          for (int j = lane; j < DP; j += 32) p.vmax_out[(size_t)b * DP + j] = -m;
      }
    } else
    for (int h = 0; h < 2; ++h) {
      const int l = warp * 2 + h, b = b0 + l;
      const float* v = p.x + (size_t)b * DP;
      float vr[DP / 32];   // the lane's potentials, one load each, all in flight
#pragma unroll
      for (int q = 0; q < DP / 32; ++q) vr[q] = b < p.B ? __ldg(v + lane + 32 * q) : neg_inf();
      float m = kNegBig;
#pragma unroll
      for (int q = 0; q < DP / 32; ++q) m = fmaxf(m, vr[q]);
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, off));
      // lane pairs interleaved: Xs[l / 2][j][l % 2], so GEMM 1 multiplies a K value
      // into two lanes with one FFMA2
#pragma unroll
      for (int q = 0; q < DP / 32; ++q) {
        const int j = lane + 32 * q;
        Xs[(l >> 1) * XSTR + xpos(j) + (l & 1)] = ex2(vr[q] - m);
      }
      if (lane == 0) Vm[l] = m;
    }
    uint64_t T[2][NQ];   // [lane pair][column k]: lanes 4 l4 + {0,1} and {2,3}
#pragma unroll
    for (int q = 0; q < NQ; ++q) T[0][q] = T[1][q] = 0ull;
    __syncthreads();

    for (; u < seg_end; ++u, ++k) {
      const int st = k & 1;
      const int rb = (int)(u - (long long)g * nrb);
      // this thread's epilogue scalars, requested now so the L2 latency hides under GEMM 1
      const int e_i = rb * kFgRows + (t >> 4), e_b = b0 + (t & 15);
      const bool e_ok = e_i < p.nrows && e_b < p.B && !dead;
      const size_t e_o = (size_t)e_b * p.ldo + e_i;
      const float e_mg = e_ok ? __ldg(p.marg + e_o) : 0.f;
      const float e_tg = e_ok ? (kFirst ? p.out[e_o] : __ldg(p.target + e_o)) : 0.f;   // kFirst: u0
      mbar_wait(&bar[st], (uint32_t)((k >> 1) & 1));
      const float* Kb = Ks + st * kFgRows * STR;
      float se_part[4][4];   // kTail: this thread's SE partials
      if constexpr (!kFirst) {
      // ---- GEMM 1: partial S over this thread's j slice, 4 rows x 2 lane pairs
      uint64_t acc[4][2], ace[4][2];
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[r][0] = acc[r][1] = ace[r][0] = ace[r][1] = 0ull;
      const int j0 = ks * (DP / 16);
      const float* xp0 = Xs + (lq * 2) * XSTR + 2 * j0 + 4 * ks;       // lanes 4 lq, 4 lq + 1
      const float* xp1 = Xs + (lq * 2 + 1) * XSTR + 2 * j0 + 4 * ks;   // lanes 4 lq + 2, + 3
#pragma unroll
      for (int jj = 0; jj < DP / 16; jj += 4) {
        float4 kr[4];
#pragma unroll
        for (int r = 0; r < 4; ++r)
          kr[r] = *reinterpret_cast<const float4*>(Kb + (rq + 4 * r) * STR + j0 + jj);
        // (x_l(j), x_l+1(j)) pairs for j = jj .. jj + 3
        const float4 xa = *reinterpret_cast<const float4*>(xp0 + 2 * jj);
        const float4 xb = *reinterpret_cast<const float4*>(xp0 + 2 * jj + 4);
        const float4 xc = *reinterpret_cast<const float4*>(xp1 + 2 * jj);
        const float4 xd = *reinterpret_cast<const float4*>(xp1 + 2 * jj + 4);
        const uint64_t p0[4] = {pk2(xa.x, xa.y), pk2(xa.z, xa.w), pk2(xb.x, xb.y), pk2(xb.z, xb.w)};
        const uint64_t p1[4] = {pk2(xc.x, xc.y), pk2(xc.z, xc.w), pk2(xd.x, xd.y), pk2(xd.z, xd.w)};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const float kv[4] = {kr[r].x, kr[r].y, kr[r].z, kr[r].w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const uint64_t kk = pk2(kv[e], kv[e]);
            ffma2_acc(acc[r][0], kk, p0[e]);
            ffma2_acc(acc[r][1], kk, p1[e]);
            if constexpr (kTail) {   // K c / (lambda ln2) = -K log2 K (0 where K flushed)
              const float kc = kv[e] > 0.f ? -kv[e] * lg2(kv[e]) : 0.f;
              const uint64_t kck = pk2(kc, kc);
              ffma2_acc(ace[r][0], kck, p0[e]);
              ffma2_acc(ace[r][1], kck, p1[e]);
            }
          }
        }
      }
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        float* o = Sred + ks * 256 + (rq + 4 * r) * 16 + lq * 4;
        *reinterpret_cast<float4*>(o) = make_float4(lo2(acc[r][0]), hi2(acc[r][0]), lo2(acc[r][1]),
                                                    hi2(acc[r][1]));
      }
      if constexpr (kTail) {   // the SE partials go through Sred after the S sums are read
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          se_part[r][0] = lo2(ace[r][0]);
          se_part[r][1] = hi2(ace[r][0]);
          se_part[r][2] = lo2(ace[r][1]);
          se_part[r][3] = hi2(ace[r][1]);
        }
      }
      __syncthreads();
      }
      // ---- row epilogue: thread t -> (row i, lane b)
      if constexpr (kFirst) {
        const int r = t >> 4, l = t & 15;
        As[r * 16 + l] = (e_ok && e_mg > 0.f) ? ex2(e_tg - Vm[l]) : 0.f;   // 2^(u0 - umax)
      } else {
        const int r = t >> 4, l = t & 15;
        float S = 0.f;
#pragma unroll
        for (int q = 0; q < 16; ++q) S += Sred[q * 256 + t];   // ascending slices
        float SE = 0.f;
        if constexpr (kTail) {
          __syncthreads();   // every S is read: reuse Sred for the SE partials
#pragma unroll
          for (int rr = 0; rr < 4; ++rr) {
            float* o = Sred + ks * 256 + (rq + 4 * rr) * 16 + lq * 4;
            *reinterpret_cast<float4*>(o) =
                make_float4(se_part[rr][0], se_part[rr][1], se_part[rr][2], se_part[rr][3]);
          }
          __syncthreads();
#pragma unroll
          for (int q = 0; q < 16; ++q) SE += Sred[q * 256 + t];
        }
        const int b = b0 + l;
        float a = 0.f;
        if (e_ok) {
          const size_t o = e_o;
          const float mg = e_mg;
          if (mg > 0.f && !(S >= kFusedEstLo)) *p.est_fail = 1;   // flushed terms: exact rerun
          const float lse = Vm[l] + lg2(S);
          const float u = sweep_out(e_tg, lse);
          p.out[o] = u;
          a = mg > 0.f ? mg * rcp_approx(S) : 0.f;
          if constexpr (kTail) {
            atomic_max_nonneg(&p.res[b], fabsf(exp2f(u + lse) - mg));
            // E0 row term a_i SE_i lambda ln2, log2 for e0_rows_finalize_kernel
            p.e0[o] = (a > 0.f && SE > 0.f) ? log2f(a) + log2f(SE) + p.e0_log2scale : neg_inf();
          }
        }
        As[r * 16 + l] = a;
      }
      __syncthreads();
      // ---- GEMM 2: T[lane][j] += sum_r K[r][j] a[r][lane]
#pragma unroll 8
      for (int r = 0; r < kFgRows; ++r) {
        const float4 a4 = *reinterpret_cast<const float4*>(As + r * 16 + l4 * 4);
        const uint64_t a01 = pk2(a4.x, a4.y), a23 = pk2(a4.z, a4.w);
        const float* kr = Kb + r * STR + jc;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const float kv = kr[64 * q];
          const uint64_t kk = pk2(kv, kv);
          ffma2_acc(T[0][q], kk, a01);
          ffma2_acc(T[1][q], kk, a23);
        }
      }
      __syncthreads();   // every thread is done with this K block and with As / Sred
      if (t == 0 && k + 2 < n) {
        fence_proxy_async();
        issue(k + 2);
      }
    }
    // plan column partials of this segment, part[cta][seg][lane][j] =
    // X[lane][j] * T[lane][j] = sum_i a_i K_ij X_j (the plan entries' sum)
    float* dst = p.part + ((size_t)blockIdx.x * p.maxseg + (g - g_first)) * kFgLanes * (size_t)DP;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int j = jc + 64 * q;
      const int l = l4 * 4;
      const float2 x01 = *reinterpret_cast<const float2*>(Xs + (l >> 1) * XSTR + xpos(j));
      const float2 x23 = *reinterpret_cast<const float2*>(Xs + ((l >> 1) + 1) * XSTR + xpos(j));
      dst[(size_t)(l + 0) * DP + j] = lo2(T[0][q]) * x01.x;
      dst[(size_t)(l + 1) * DP + j] = hi2(T[0][q]) * x01.y;
      dst[(size_t)(l + 2) * DP + j] = lo2(T[1][q]) * x23.x;
      dst[(size_t)(l + 3) * DP + j] = hi2(T[1][q]) * x23.y;
    }
  }
  pdl_launch_dependents();
}

// Column update from the plan partials: colsum_j = sum over the CTAs that
// covered lane b's group (ascending), v'_j = v_j + l2nu_j - log2(colsum_j),
// column residual |colsum_j - nu_j|.  grid (ceil(rowlen / 256), B).
__global__ void __launch_bounds__(256) fused_merge_kernel(const FusedMergeParams p) {
  __shared__ int s_off[kFusedMaxCtas];   // partial rows of this lane, ascending CTA
  __shared__ int s_c0, s_n;
  const int b = p.b0 + blockIdx.y;
  const int g = b / p.nw, w = b % p.nw;
  if (threadIdx.x == 0) {
    const long long ua = (long long)g * p.nrows, ub = ua + p.nrows - 1;
    s_c0 = (int)(((ua + 1) * p.nct - 1) / p.U);
    s_n = (int)(((ub + 1) * p.nct - 1) / p.U) - s_c0 + 1;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < s_n; t += blockDim.x) {   // every covering CTA has >= 1 unit
    const int c = s_c0 + t;
    const long long s0 = fused_seg_start(p.U, p.nct, c);
    s_off[t] = (int)(((long long)c * p.maxseg + (g - (int)(s0 / p.nrows))) * p.nw + w);
  }
  __syncthreads();
  pdl_wait();
  const int j = (blockIdx.x * 256 + threadIdx.x) * 2;   // two columns per thread
  float rr = 0.f;
  if (j < p.rowlen) {
    const int np = s_n;
    float2 cs = make_float2(0.f, 0.f);
    int k = 0;
    for (; k + 8 <= np; k += 8) {   // eight loads in flight, summed in ascending order
      float2 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        v[u] = __ldcg(reinterpret_cast<const float2*>(p.part + (size_t)s_off[k + u] * p.rowlen + j));
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        cs.x += v[u].x;
        cs.y += v[u].y;
      }
    }
    for (; k + 4 <= np; k += 4) {
      float2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        v[u] = __ldcg(reinterpret_cast<const float2*>(p.part + (size_t)s_off[k + u] * p.rowlen + j));
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        cs.x += v[u].x;
        cs.y += v[u].y;
      }
    }
    for (; k < np; ++k) {
      const float2 v = __ldcg(reinterpret_cast<const float2*>(p.part + (size_t)s_off[k] * p.rowlen + j));
      cs.x += v.x;
      cs.y += v.y;
    }
    const size_t o = (size_t)b * p.rowlen + j;
    const float2 tg = *reinterpret_cast<const float2*>(p.target + o);
    const float2 vo = *reinterpret_cast<const float2*>(p.v_old + o);
    float2 vn = make_float2(neg_inf(), neg_inf());
    bool bad = false;
    if (tg.x != neg_inf()) {
      vn.x = vo.x + tg.x - log2f(cs.x);
      bad |= !(cs.x >= kFusedMinColsum) || !(vn.x == vn.x);
    }
    if (tg.y != neg_inf()) {
      vn.y = vo.y + tg.y - log2f(cs.y);
      bad |= !(cs.y >= kFusedMinColsum) || !(vn.y == vn.y);
    }
    if (bad) *p.est_fail = 1;
    *reinterpret_cast<float2*>(p.v_new + o) = vn;
    if (p.res != nullptr) {
      const float2 mg = *reinterpret_cast<const float2*>(p.marg + o);
      rr = fmaxf(fabsf(cs.x - mg.x), fabsf(cs.y - mg.y));
    }
  }
  if (p.res != nullptr) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) rr = fmaxf(rr, __shfl_xor_sync(0xffffffffu, rr, off));
    if ((threadIdx.x & 31) == 0) atomic_max_nonneg(&p.res[b], rr);
  }
  pdl_launch_dependents();
}

// K = 2^A2 for the fused passes' linear rows (padding -inf -> 0).
__global__ void kernel_matrix_kernel(const float* __restrict__ a2, float* __restrict__ k, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    k[i] = ex2(a2[i]);
}

// E0 per lane from per-row log2 terms e0[b][i] (lane-major rows): one warp
// per lane, (max, sum) merge by shuffles.
__global__ void __launch_bounds__(256) e0_rows_finalize_kernel(const float* __restrict__ e0, int B,
                                                               int d, int ld,
                                                               float* __restrict__ out_cost,
                                                               int* status) {
  const int b = blockIdx.x * 8 + warp_id();
  if (b >= B) return;
  const float* row = e0 + (size_t)b * ld;
  float m = kNegBig, s = 0.f;
  for (int i = lane_id(); i < d; i += 32) {
    const float v = row[i];
    if (v > m + kLazy) {
      s *= ex2(m - v);
      m = v;
    }
    s += ex2(v - m);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, off);
    const float s2 = __shfl_xor_sync(0xffffffffu, s, off);
    lse_merge(m, s, m2, s2);
  }
  if (lane_id() == 0) {
    const float cost = exp2f(lse_final(m, s));
    out_cost[b] = cost;
    if (!isfinite(cost)) set_status(status, 12);
  }
}

}  // namespace skb
