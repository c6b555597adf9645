// sweep_tiled.cuh -- K1/K2/K4/K6: the fused online-logsumexp half-sweep for a
// cost shared by every lane (stored, TMA-staged) or recomputed on the fly
// (squared-Euclidean grid).
//
// One launch computes, for every lane b and output index p,
//     lse[b,p] = log2 sum_q 2^(G[q,p] + X[q,b])
// which is `_fused_lse` (batch.py:185-201) in log base 2, with
//   column sweep: G = A2 = -c*log2e/lambda,  X = f2 (log_u), p = j  (batch.py:315)
//   row sweep:    G = A2^T,                  X = g2 (log_v), p = i  (batch.py:316)
// and then one of three epilogues:
//   UPDATE : out[p,b] = target[p,b] - lse  (a half-sweep, batch.py:300-301),
//            optionally with the fused residual term (batch.py:303-309);
//   PARTIAL: the raw (max, sum) accumulator, merged across GPUs for row-sharded
//            solves exactly like OnlineLseAccumulator.merge (batch.py:116-130);
//   TAIL   : the final column pass: column residual plus the stable E0 term
//            log2 sum_q 2^(G+X) * c[q,p]  (batch.py:323-337), one pass for both.
//
// Data layout in HBM (all fp32, padded with -inf so padding contributes 0):
//   G  [Qp][Pp]  row-major (A2 or its transpose, built once per solve)
//   X, target, out, old, marg  [dim][Bp]  ("dim-major": a q-row holds all lanes)
// Work decomposition: tiles of BT lanes x PT outputs, each reduced over
// NQ = Qp/QC chunks of QC q's.  The (tile, chunk) "atoms" are split evenly over
// a grid of resident CTAs (stream-K); a tile cut between CTAs is merged by the
// last CTA to finish it, in ascending CTA order, so results are deterministic
// (the reference's ascending span merge, batch.py:198-201).
// Per CTA and atom, TMA brings one [QC][PT] tile of G and one [QC][BT] tile of X
// into shared memory; each G tile is reused by BT lanes, each X tile by PT
// outputs, so the kernel is bound by the MUFU ex2 rate, not by memory.
#pragma once

#include "common.cuh"

#include <type_traits>

namespace skb {


struct TiledSweepParams {
  int Qv, Pv;          // valid reduce / output extents (d)
  int Bp;              // padded lane count (row stride of dim-major buffers)
  int ntile_b, ntile_p, nq;
  long long W;         // stream-K units: virtual rows over all tiles = ntiles * (Qv + seg_x)
  int G;               // grid size (<= W / QC, so every CTA owns >= 1 chunk of rows)
  const float* target; // [Pp][Bp] log2 marginal of the output side
  const float* marg;   // [Pp][Bp] linear marginal of the output side (residuals)
  float* out;          // [Pp][Bp] updated potentials (UPDATE)
  const float* old;    // [Pp][Bp] current potentials of the output side (kResCol, TAIL)
  float* res;          // [Bp] per-lane residual, atomic max (nullable)
  float* e0;           // [Pp][Bp] per-output E0 log2 terms (TAIL)
  float* pmax;         // [Pp][Bp] (PARTIAL)
  float* psum;         // [Pp][Bp] (PARTIAL)
  float* part;         // stream-K partial slots [G][2][3][BT*PT]
  int* counters;       // [ntile_b * ntile_p], zero between launches
  int res_kind;
  float cinv;          // c = G * cinv (TAIL):  cinv = -lambda / log2e
  // on-the-fly grid cost: G[q,p] = gk * (hx2*dx^2 + hy2*dy^2), points k -> (k % nx, k / nx)
  int gnx;
  float gk, ghx2, ghy2;
  unsigned long long* dbg;   // optional per-CTA timing records (diagnostics), nullable
  int seg_x;                 // virtual rows charged per tile start (stream-K weighting)
  int fast32;                // W * G and every row index fit in 32 bits: 32-bit index math
  // Estimate mode: start every output's running max at the previous iteration's
  // log-sum-exp, target - est_old, and reduce each chunk in one pass.
  const float* est_old;      // output-side potentials before this sweep (nullable)
  int use_est;
  int use_poly;              // route kPolyPairs of the 8 output pairs through ex2_poly2
  int* est_fail;             // set when an estimate was > kEstSlack above the result
};

// Per-call fields of a sweep (the rest of TiledSweepParams is static over a
// solve and stays in constant / kernel-parameter space).
struct SweepDyn {
  float* out;
  const float* old;
  const float* est_old;
  int use_est;
  int res_kind;
};

__host__ __device__ inline SweepDyn dyn_of(const TiledSweepParams& p) {
  return SweepDyn{p.out, p.old, p.est_old, p.use_est, p.res_kind};
}

// One-pass chunks tolerate terms up to 2^kRedo above the running max (no fp32
// overflow for <= 2^20 terms); beyond that the warp redoes the chunk exactly.
constexpr float kRedo = 100.f;
// An estimate more than this above the final lse could have flushed
// significant terms: flag it and the host reruns the solve in exact mode.
constexpr float kEstSlack = 100.f;
constexpr float kParked = 1.0e30f;   // running max of outputs whose target is -inf
// Output pairs (of 8 per thread) whose exponentials run on the FMA pipe.
#ifndef SKB_POLY_PAIRS
#define SKB_POLY_PAIRS 2
#endif
constexpr int kPolyPairs = SKB_POLY_PAIRS;

#ifndef SKB_OCC_SMALL
#define SKB_OCC_SMALL 2   // resident 256-thread (64-lane) tiles per SM
#endif
template <int BT, int PT, int QC, int RB, int RP, int NSTAGE, bool kGrid, int kMode>
struct TiledSweep {
  static constexpr int NT = (BT / RB) * (PT / RP);
  static constexpr int NTB = BT / RB;          // threads along lanes (within a warp)
  static constexpr int NV = (kMode == kModeTail) ? 3 : 2;
  static constexpr int G_FLOATS = QC * PT;
  static constexpr int X_FLOATS = QC * BT;
  static constexpr int STAGE_FLOATS = G_FLOATS + X_FLOATS;
  static constexpr uint32_t TMA_BYTES = (kGrid ? 0 : G_FLOATS * 4) + X_FLOATS * 4;
  static constexpr int EST_FLOATS = 2 * RB * RP * NT;   // per-thread estimate rows (tg, old)
  static constexpr size_t SMEM_BYTES =
      size_t(NSTAGE) * STAGE_FLOATS * 4 + 64 * 8 /*bars*/ + BT * 4 +
      (kGrid ? (QC + PT) * 8 : 0) + size_t(EST_FLOATS) * 4;
  static_assert(NTB == 16 || NTB == 32, "lane-threads per (half) warp");
  static constexpr int OCC = (NT >= 512) ? 1 : SKB_OCC_SMALL;   // CTAs per SM the launch bounds target
  static_assert(NT % 32 == 0, "whole warps");
  static_assert(RB == 4 && RP == 4, "float4 tile loads");
  static_assert(QC % 4 == 0, "unroll");
};

// Stream-K split over reduction rows, weighted for segments: every tile is
// charged X = seg_x virtual rows at its start (the fixed cost of starting a
// segment: estimate loads, partial chunks, the piece epilogue), and the
// virtual row space W = ntiles * (Qv + X) is split evenly, so a CTA that
// crosses a tile boundary gets ~X fewer real rows.
__host__ __device__ __forceinline__ long long atom_begin(const TiledSweepParams& p, long long c) {
  if (p.fast32) {   // every product below fits in 32 bits (checked on the host)
    const unsigned v = (unsigned)c * (unsigned)p.W / (unsigned)p.G;
    const unsigned tq = (unsigned)(p.Qv + p.seg_x);
    const unsigned t = v / tq, off = v - t * tq;
    return (long long)(t * (unsigned)p.Qv + (off > (unsigned)p.seg_x ? off - p.seg_x : 0u));
  }
  const unsigned long long v = ((unsigned long long)c * (unsigned long long)p.W) /
                               (unsigned long long)p.G;
  const unsigned long long tq = (unsigned long long)(p.Qv + p.seg_x);
  const unsigned long long t = v / tq, off = v - t * tq;
  return (long long)(t * (unsigned long long)p.Qv +
                     (off > (unsigned long long)p.seg_x ? off - p.seg_x : 0ull));
}
// CTA owning real row a: the largest c with atom_begin(c) <= a.
__host__ __device__ __forceinline__ long long atom_owner(const TiledSweepParams& p, long long a) {
  if (p.fast32) {
    const unsigned t = (unsigned)a / (unsigned)p.Qv;
    const unsigned va = t * (unsigned)(p.Qv + p.seg_x) + p.seg_x + ((unsigned)a - t * (unsigned)p.Qv);
    return (long long)(((va + 1) * (unsigned)p.G - 1) / (unsigned)p.W);
  }
  const unsigned long long t = (unsigned long long)a / (unsigned long long)p.Qv;
  const unsigned long long va = t * (unsigned long long)(p.Qv + p.seg_x) + p.seg_x +
                                ((unsigned long long)a - t * (unsigned long long)p.Qv);
  return (long long)(((va + 1) * (unsigned long long)p.G - 1) / (unsigned long long)p.W);
}

// Finalise one output tile from per-thread accumulators (M, Sm, S2 hold the
// thread's RB x RP outputs).  Called by every thread of the CTA (it may sync).
template <int BT, int PT, int RB, int RP, int NT, int kMode>
__device__ __forceinline__ void tile_epilogue(const TiledSweepParams& p, const SweepDyn& d,
                                              int tid, int tb, int tp,
                                              int b0, int p0, int own_lo, const float* M,
                                              const float* Sm, const float* S2, float* s_res) {
  // tid/NT here are the block-local thread index and block size (the caller
  // passes the lane/output groups tb/tp of the sweep's thread map)
    if (p.res != nullptr && (kMode == kModeTail || d.res_kind != kResNone)) {
      for (int i = tid; i < BT; i += NT) s_res[i] = 0.f;
      __syncthreads();
    }
    float rmax[RB];
#pragma unroll
    for (int rb = 0; rb < RB; ++rb) rmax[rb] = 0.f;
    const int bb = b0 + tb * RB;
#pragma unroll
    for (int rp = 0; rp < RP; ++rp) {
      const int pp = p0 + tp * RP + rp;
      if (pp >= p.Pv || pp < own_lo) continue;
      const size_t row = size_t(pp) * p.Bp + bb;
      if constexpr (kMode == kModePartial) {
        *reinterpret_cast<float4*>(p.pmax + row) =
            make_float4(M[0 * RP + rp], M[1 * RP + rp], M[2 * RP + rp], M[3 * RP + rp]);
        *reinterpret_cast<float4*>(p.psum + row) =
            make_float4(Sm[0 * RP + rp], Sm[1 * RP + rp], Sm[2 * RP + rp], Sm[3 * RP + rp]);
        continue;
      } else {
      float lse[RB];
#pragma unroll
      for (int rb = 0; rb < RB; ++rb) lse[rb] = lse_final(M[rb * RP + rp], Sm[rb * RP + rp]);
      if (kMode == kModeUpdate) {
        const float4 tg = *reinterpret_cast<const float4*>(p.target + row);
        const float tv[4] = {tg.x, tg.y, tg.z, tg.w};
        if (d.use_est) {
          const float4 eo = *reinterpret_cast<const float4*>(d.est_old + row);
          const float ev[4] = {eo.x, eo.y, eo.z, eo.w};
          bool bad = false;
#pragma unroll
          for (int rb = 0; rb < RB; ++rb) {
            const float est = tv[rb] - ev[rb];
            if (tv[rb] != neg_inf() && isfinite(est) && !(lse[rb] >= est - kEstSlack)) bad = true;
          }
          if (bad) atomicOr(p.est_fail, 1);
        }
        float ov[4];
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) ov[rb] = sweep_out(tv[rb], lse[rb]);
        *reinterpret_cast<float4*>(d.out + row) = make_float4(ov[0], ov[1], ov[2], ov[3]);
        if (p.res != nullptr && d.res_kind != kResNone) {
          const float4 mg = *reinterpret_cast<const float4*>(p.marg + row);
          const float mv[4] = {mg.x, mg.y, mg.z, mg.w};
          float base[4] = {ov[0], ov[1], ov[2], ov[3]};
          if (d.res_kind == kResCol) {
            const float4 od = *reinterpret_cast<const float4*>(d.old + row);
            base[0] = od.x; base[1] = od.y; base[2] = od.z; base[3] = od.w;
          }
#pragma unroll
          for (int rb = 0; rb < RB; ++rb)
            rmax[rb] = fmaxf(rmax[rb], fabsf(exp2f(base[rb] + lse[rb]) - mv[rb]));
        }
      } else {  // TAIL: column residual against `old` and the E0 term
        const float4 od = *reinterpret_cast<const float4*>(d.old + row);
        const float4 mg = *reinterpret_cast<const float4*>(p.marg + row);
        const float ovv[4] = {od.x, od.y, od.z, od.w};
        const float mv[4] = {mg.x, mg.y, mg.z, mg.w};
        float ev[4];
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) {
          const float s2 = S2[rb * RP + rp];
          ev[rb] = (s2 > 0.f) ? (M[rb * RP + rp] + log2f(s2) + ovv[rb]) : neg_inf();
          rmax[rb] = fmaxf(rmax[rb], fabsf(exp2f(ovv[rb] + lse[rb]) - mv[rb]));
        }
        *reinterpret_cast<float4*>(p.e0 + row) = make_float4(ev[0], ev[1], ev[2], ev[3]);
      }
      }   // if constexpr (kMode == kModePartial) ... else
    }
    if (p.res != nullptr && (kMode == kModeTail || d.res_kind != kResNone)) {
#pragma unroll
      for (int rb = 0; rb < RB; ++rb) {
        // NaN must win the max (batch.py:320 compares max <= tol, false for NaN)
        const float v = (rmax[rb] != rmax[rb]) ? __int_as_float(0x7fc00000) : rmax[rb];
        atomic_max_nonneg(&s_res[tb * RB + rb], v);
      }
      __syncthreads();
      for (int i = tid; i < BT; i += NT) {
        if (b0 + i < p.Bp) atomic_max_nonneg(&p.res[b0 + i], s_res[i]);
      }
    }
  }

// Thread -> (lane group, output group) map shared by the sweep and the fixup:
// a warp covers 64 lanes x 8 outputs (16 lane-threads x 2 output-groups), so
// per row it reads 256 B of X and two 16 B G vectors (3 shared wavefronts);
// with BT=128 the warps split into two lane halves.
template <int BT, int RB, int NT>
__device__ __forceinline__ void thread_map(int tid, int& tb, int& tp) {
  constexpr int NTB = BT / RB;
  constexpr int NW = NT / 32;
  constexpr int WPH = NW / (NTB / 16);
  const int warp = tid >> 5, lane = tid & 31;
  tb = (warp / WPH) * 16 + (lane & 15);
  tp = (warp % WPH) * 2 + (lane >> 4);
}

// Shared-memory carve-up common to the sweep kernel and the persistent solve.
template <int BT, int PT, int QC, int RB, int RP, int NSTAGE, bool kGrid, int kMode>
struct SweepSmem {
  using S = TiledSweep<BT, PT, QC, RB, RP, NSTAGE, kGrid, kMode>;
  float* smem;
  uint64_t* bars;
  float* s_res;
  float* s_gq;   // grid mode: q coordinates (x, y) [QC][2]
  float* s_gp;   // grid mode: p coordinates [PT][2]
  float* est;    // estimate rows per thread: [2*RP][NT] float4 (target rows, old rows)
  __device__ explicit SweepSmem(uint8_t* raw) {
    smem = reinterpret_cast<float*>(raw);
    bars = reinterpret_cast<uint64_t*>(smem + NSTAGE * S::STAGE_FLOATS);
    s_res = reinterpret_cast<float*>(bars + 64);
    s_gq = s_res + BT;
    s_gp = s_gq + 2 * QC;
    est = s_gq + (kGrid ? 2 * (QC + PT) : 0);   // 16-byte aligned (all extents are multiples of 4)
  }
};

// One half-sweep over this CTA's stream-K range of (tile, row) work: the hot
// loop.  `seq` counts the TMA stages this CTA has consumed so far, so the
// mbarrier phases stay consistent when several sweeps run in one kernel.
template <int BT, int PT, int QC, int RB, int RP, int NSTAGE, bool kGrid, int kMode>
__device__ __forceinline__ void sweep_phase(const CUtensorMap* tmap_g, const CUtensorMap* tmap_x,
                                            const TiledSweepParams& p, const SweepDyn& d,
                                            const SweepSmem<BT, PT, QC, RB, RP, NSTAGE, kGrid, kMode>& sm,
                                            uint32_t& seq) {
  using S = TiledSweep<BT, PT, QC, RB, RP, NSTAGE, kGrid, kMode>;
  constexpr int NT = S::NT;
  constexpr int NV = S::NV;
  constexpr int NOUT = RB * RP;
  float* smem = sm.smem;
  uint64_t* bars = sm.bars;
  float* s_res = sm.s_res;
  float* s_gq = sm.s_gq;
  float* s_gp = sm.s_gp;

  const int tid = threadIdx.x;
  int tb, tp;   // lane group (b = tb*RB + rb), output group (p = tp*RP + rp)
  thread_map<BT, RB, NT>(tid, tb, tp);

  const long long c = blockIdx.x;
  const long long a_begin = atom_begin(p, c);     // first row (global row index)
  const long long a_end = atom_begin(p, c + 1);   // one past the last row
  const int nq = p.nq;
  const long long Qv = p.Qv;
  // global chunk index of a row: tile * nq + (q / QC)
  auto chunk_of = [&](long long r) {
    if (p.fast32) {
      const unsigned t = (unsigned)r / (unsigned)Qv;
      return (long long)(t * (unsigned)nq + ((unsigned)r - t * (unsigned)Qv) / QC);
    }
    const long long t = r / Qv;
    return t * nq + (r - t * Qv) / QC;
  };
  if (a_end <= a_begin) return;   // no rows for this CTA
  const long long g_first = chunk_of(a_begin);
  const int n_local = int(chunk_of(a_end - 1) - g_first + 1);

  // Output tile tp_idx covers [p0, p0 + PT) but owns (writes) [tp_idx*PT, ...):
  // the last tile is shifted left to end at Pv -- its start rounded up to a
  // float4 boundary (an unaligned start faulted for Pv % 4 != 0), so it may
  // reach 3 columns into the padding, whose outputs are clamped to Pv - 1 --
  // so no tile is partial (a
  // partial tile's few active warps are latency-bound and stretch the tail).
  auto atom_coords = [&](long long a, int& tile, int& qc, int& b0, int& p0) {
    tile = int((unsigned)a / (unsigned)nq);   // chunk indices fit in 32 bits
    qc = int(a - (long long)tile * nq);
    const int tb_idx = tile % p.ntile_b;     // lane tiles innermost: consecutive tiles share G
    const int tp_idx = tile / p.ntile_b;
    b0 = tb_idx * BT;
    p0 = (tp_idx == p.ntile_p - 1) ? max((p.Pv - PT + 3) & ~3, 0) : tp_idx * PT;
  };

  auto issue = [&](int l) {
    const long long a = g_first + l;
    int tile, qc, b0, p0;
    atom_coords(a, tile, qc, b0, p0);   // thread 0 only, NSTAGE ahead
    const int s = (seq + l) % NSTAGE;
    float* st = smem + s * S::STAGE_FLOATS;
    mbar_arrive_expect_tx(&bars[s], S::TMA_BYTES);
    if (!kGrid) tma_load_2d(st, tmap_g, p0, qc * QC, &bars[s]);
    tma_load_2d(st + S::G_FLOATS, tmap_x, b0, qc * QC, &bars[s]);
  };

  // Estimate rows (target, previous potential) of a tile's outputs, copied
  // asynchronously into this thread's slots of sm.est: issued a segment
  // ahead, so the loads never stall the hot loop and cost no registers.
  float* est_buf = sm.est;
  auto est_fetch = [&](int tile_n) {
    const int tb_n = tile_n % p.ntile_b, tp_n = tile_n / p.ntile_b;
    const int b0n = tb_n * BT;
    const int p0n = (tp_n == p.ntile_p - 1) ? max((p.Pv - PT + 3) & ~3, 0) : tp_n * PT;
#pragma unroll
    for (int rp = 0; rp < RP; ++rp) {
      const int pp = min(p0n + tp * RP + rp, p.Pv - 1);
      const size_t row = size_t(pp) * p.Bp + b0n + tb * RB;
      cp_async16(est_buf + (size_t(rp) * NT + tid) * 4, p.target + row);
      cp_async16(est_buf + (size_t(RP + rp) * NT + tid) * 4, d.est_old + row);
    }
    cp_async_commit();
  };
  // chunk coordinates walk incrementally (no per-chunk 64-bit division)
  int tile, qc, b0, p0;
  atom_coords(g_first, tile, qc, b0, p0);
  if (d.use_est) est_fetch(tile);
  const int last_tile = int(chunk_of(a_end - 1) / nq);

  if (p.dbg && tid == 0) p.dbg[12288 + blockIdx.x * 4 + 0] = globaltimer_ns();
  if (tid == 0) {
    for (int l = 0; l < NSTAGE && l < n_local; ++l) issue(l);
  }

  float M[NOUT], Sm[NOUT], S2[NOUT];
  auto reset_acc = [&]() {
#pragma unroll
    for (int o = 0; o < NOUT; ++o) {
      M[o] = kNegBig;
      Sm[o] = 0.f;
      S2[o] = 0.f;
    }
  };
  reset_acc();

  for (int l = 0; l < n_local; ++l) {
    if (l > 0 && ++qc == nq) {
      qc = 0;
      ++tile;
      const int tb_idx = tile % p.ntile_b, tp_idx = tile / p.ntile_b;
      b0 = tb_idx * BT;
      p0 = (tp_idx == p.ntile_p - 1) ? max((p.Pv - PT + 3) & ~3, 0) : tp_idx * PT;
    }
    // this CTA's rows inside the chunk: [k_lo, k_hi) relative to the chunk start
    const long long row0 = (long long)tile * Qv + (long long)qc * QC;
    const int chunk_rows = (int)(Qv - (long long)qc * QC < QC ? Qv - (long long)qc * QC : QC);
    const int k_lo = (int)(a_begin > row0 ? a_begin - row0 : 0);
    int k_hi = (int)(a_end - row0 < chunk_rows ? a_end - row0 : chunk_rows);
    // rows past Qv are -inf padding: round the natural chunk end up to a pair
    if (k_hi == chunk_rows) k_hi = min(QC, (k_hi + 1) & ~1);
    const int s = (seq + l) % NSTAGE;
    const uint32_t parity = ((seq + l) / NSTAGE) & 1;
    float* st = smem + s * S::STAGE_FLOATS;
    const float* Gs = st;
    const float* Xs = st + S::G_FLOATS;

    if (kGrid) {
      // Recompute this atom's [QC][PT] cost tile: never materialised in HBM.
      for (int i = tid; i < QC + PT; i += NT) {
        const int k = (i < QC) ? (qc * QC + i) : (p0 + i - QC);
        const int yk = k / p.gnx;
        const int xk = k - yk * p.gnx;
        float* dst = (i < QC) ? (s_gq + 2 * i) : (s_gp + 2 * (i - QC));
        dst[0] = float(xk);
        dst[1] = float(yk);
      }
      __syncthreads();
      float* Gw = st;
      for (int i = tid; i < QC * PT; i += NT) {
        const int qi = i / PT;
        const int pi = i - qi * PT;
        const float dx = s_gq[2 * qi] - s_gp[2 * pi];
        const float dy = s_gq[2 * qi + 1] - s_gp[2 * pi + 1];
        const bool valid = (qc * QC + qi) < p.Qv && (p0 + pi) < p.Pv;
        Gw[i] = valid ? p.gk * fmaf(p.ghx2, dx * dx, p.ghy2 * dy * dy) : neg_inf();
      }
    }
    const bool est_init = d.use_est && (l == 0 || qc == 0);
    if (p.dbg && tid == 0 && l == 0) p.dbg[12288 + blockIdx.x * 4 + 1] = globaltimer_ns();
    mbar_wait(&bars[s], parity);
    if (p.dbg && tid == 0 && l == 0) p.dbg[12288 + blockIdx.x * 4 + 2] = globaltimer_ns();
    if (est_init) {
      // segment start in estimate mode: running max := previous lse (target -
      // old), from the rows est_fetch staged; outputs with a -inf target never
      // need their lse (parked).  Then stage the next segment's rows.
      cp_async_wait_all();
#pragma unroll
      for (int rp = 0; rp < RP; ++rp) {
        const float4 tg = *reinterpret_cast<const float4*>(est_buf + (size_t(rp) * NT + tid) * 4);
        const float4 eo =
            *reinterpret_cast<const float4*>(est_buf + (size_t(RP + rp) * NT + tid) * 4);
        const float tv[4] = {tg.x, tg.y, tg.z, tg.w};
        const float ev[4] = {eo.x, eo.y, eo.z, eo.w};
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) {
          const float est = tv[rb] - ev[rb];
          M[rb * RP + rp] = (tv[rb] == neg_inf()) ? kParked : (isfinite(est) ? est : kNegBig);
        }
      }
      if (tile < last_tile) est_fetch(tile + 1);
    }
    if (kGrid) __syncthreads();

    // ---- consume: the hot loop --------------------------------------------
    // Rows beyond Qv are -inf in both tiles (padded buffers / recomputed tile),
    // so the chunk length can be rounded up to the unroll width.
    // a warp covers 2 output groups; skip it only if both are past Pv (uniform)
    const bool warp_active = __any_sync(0xffffffffu, (p0 + tp * RP) < p.Pv);
    if (warp_active) {
      // Outputs are handled in lane pairs (rb = 2h, 2h+1) so every add is a
      // packed FADD2 with the cost value broadcast: o = (2h + e) * RP + rp.
      uint64_t acc[2][RP], acc2[2][RP];
      // phase 3: one ex2 per cell; packed adds for t = g + x, t - M and the
      // chunk-local sums (which keep the fp32 error ~ sqrt(Q/QC))
      auto phase3 = [&](auto poly) {
        constexpr bool kPoly = decltype(poly)::value;
        uint64_t nM[2][RP];
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int rp = 0; rp < RP; ++rp) {
            nM[h][rp] = pk2(-M[(2 * h) * RP + rp], -M[(2 * h + 1) * RP + rp]);
            acc[h][rp] = 0ull;
            acc2[h][rp] = 0ull;
          }
#pragma unroll 4
        for (int k = k_lo; k < k_hi; ++k) {
          const float4 gv = *reinterpret_cast<const float4*>(Gs + k * PT + tp * RP);
          const float4 xv = *reinterpret_cast<const float4*>(Xs + k * BT + tb * RB);
          const float g[4] = {gv.x, gv.y, gv.z, gv.w};
          const uint64_t x2[2] = {pk2(xv.x, xv.y), pk2(xv.z, xv.w)};
          float cw[4];
          if (kMode == kModeTail) {
            // c = G * cinv; padding rows (G = -inf) must weigh 0, not +inf
#pragma unroll
            for (int rp = 0; rp < RP; ++rp) cw[rp] = (g[rp] == neg_inf()) ? 0.f : g[rp] * p.cinv;
          }
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int rp = 0; rp < RP; ++rp) {
              const uint64_t a = fadd2(fadd2(x2[h], pk2(g[rp], g[rp])), nM[h][rp]);
              const uint64_t e = (kPoly && h * RP + rp < kPolyPairs)
                                     ? ex2_poly2(a)
                                     : pk2(ex2(lo2(a)), ex2(hi2(a)));
              acc[h][rp] = fadd2(acc[h][rp], e);
              if (kMode == kModeTail) acc2[h][rp] = ffma2(e, pk2(cw[rp], cw[rp]), acc2[h][rp]);
            }
        }
      };
      bool exact = !d.use_est;
      if (!exact) {
        if (p.use_poly) phase3(std::true_type{}); else phase3(std::false_type{});
        // A term above 2^kRedo (or inf/NaN) means the shift was too low for
        // this chunk: discard it and redo the chunk exactly (warp-uniform).
        bool ok = true;
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int rp = 0; rp < RP; ++rp)
            ok = ok && (lo2(acc[h][rp]) <= 0x1p100f) && (hi2(acc[h][rp]) <= 0x1p100f);
        if (!__all_sync(0xffffffffu, ok)) {
          exact = true;
        } else {
          // Fold the chunk in.  Every chunk sum is <= 2^100 (checked above),
          // so a segment's running sum stays far below the fp32 range without
          // per-chunk renormalisation; the shift M stays the estimate.
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int rp = 0; rp < RP; ++rp) {
              const int o0 = (2 * h) * RP + rp, o1 = (2 * h + 1) * RP + rp;
              Sm[o0] += lo2(acc[h][rp]);
              Sm[o1] += hi2(acc[h][rp]);
              if (kMode == kModeTail) {
                S2[o0] += lo2(acc2[h][rp]);
                S2[o1] += hi2(acc2[h][rp]);
              }
            }
        }
      }
      if (exact) {
        // phase 1: exact max of this chunk, 2 rows per FMNMX3 (1 instr / cell)
        float cm[NOUT];
#pragma unroll
        for (int o = 0; o < NOUT; ++o) cm[o] = kNegBig;
        const int k_pairs_end = k_lo + ((k_hi - k_lo) & ~1);
#pragma unroll 2
        for (int k = k_lo; k < k_pairs_end; k += 2) {
          const float4 ga = *reinterpret_cast<const float4*>(Gs + k * PT + tp * RP);
          const float4 gb = *reinterpret_cast<const float4*>(Gs + (k + 1) * PT + tp * RP);
          const float4 xa = *reinterpret_cast<const float4*>(Xs + k * BT + tb * RB);
          const float4 xb = *reinterpret_cast<const float4*>(Xs + (k + 1) * BT + tb * RB);
          const float gav[4] = {ga.x, ga.y, ga.z, ga.w};
          const float gbv[4] = {gb.x, gb.y, gb.z, gb.w};
          const uint64_t xa2[2] = {pk2(xa.x, xa.y), pk2(xa.z, xa.w)};
          const uint64_t xb2[2] = {pk2(xb.x, xb.y), pk2(xb.z, xb.w)};
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int rp = 0; rp < RP; ++rp) {
              const uint64_t ta = fadd2(xa2[h], pk2(gav[rp], gav[rp]));
              const uint64_t tb2 = fadd2(xb2[h], pk2(gbv[rp], gbv[rp]));
              const int o0 = (2 * h) * RP + rp, o1 = (2 * h + 1) * RP + rp;
              cm[o0] = fmax3(cm[o0], lo2(ta), lo2(tb2));
              cm[o1] = fmax3(cm[o1], hi2(ta), hi2(tb2));
            }
        }
        if (k_pairs_end < k_hi) {   // odd row at a CTA boundary
          const int k = k_pairs_end;
          const float4 ga = *reinterpret_cast<const float4*>(Gs + k * PT + tp * RP);
          const float4 xa = *reinterpret_cast<const float4*>(Xs + k * BT + tb * RB);
          const float gav[4] = {ga.x, ga.y, ga.z, ga.w};
          const float xav[4] = {xa.x, xa.y, xa.z, xa.w};
#pragma unroll
          for (int rb = 0; rb < RB; ++rb)
#pragma unroll
            for (int rp = 0; rp < RP; ++rp)
              cm[rb * RP + rp] = fmaxf(cm[rb * RP + rp], gav[rp] + xav[rb]);
        }
        // phase 2: lazy online rescale (batch.py:98-105), warp-uniform so the
        // branch never diverges; the running max only moves when a chunk beats
        // it by more than kLazy, i.e. rarely after the first chunks.
#pragma unroll
        for (int o = 0; o < NOUT; ++o) {
          if (__any_sync(0xffffffffu, cm[o] > M[o] + kLazy)) {
            const float mn = fmaxf(M[o], cm[o]);
            const float r = ex2(M[o] - mn);
            Sm[o] *= r;
            if (kMode == kModeTail) S2[o] *= r;
            M[o] = mn;
          }
        }
        if (p.use_poly) phase3(std::true_type{}); else phase3(std::false_type{});
#pragma unroll
        for (int h = 0; h < 2; ++h)
#pragma unroll
          for (int rp = 0; rp < RP; ++rp) {
            const int o0 = (2 * h) * RP + rp, o1 = (2 * h + 1) * RP + rp;
            Sm[o0] += lo2(acc[h][rp]);
            Sm[o1] += hi2(acc[h][rp]);
            if (kMode == kModeTail) {
              S2[o0] += lo2(acc2[h][rp]);
              S2[o1] += hi2(acc2[h][rp]);
            }
          }
      }
    }
    __syncthreads();   // every warp is done with stage s
    if (tid == 0 && l + NSTAGE < n_local) issue(l + NSTAGE);
    if (p.dbg && tid == 0 && l < 16) p.dbg[8192 + blockIdx.x * 16 + l] = globaltimer_ns();

    // ---- segment end: finalize or hand over to the stream-K merge ---------
    const bool seg_end = (qc == nq - 1) || (l == n_local - 1);
    if (!seg_end) continue;
    const long long t_first = (long long)tile * Qv;   // first row of this tile
    const long long c_lo = atom_owner(p, t_first);
    const long long c_hi = atom_owner(p, t_first + Qv - 1);
    const int own_lo = (tile / p.ntile_b) * PT;
    if (c_lo == c_hi) {
      tile_epilogue<BT, PT, RB, RP, NT, kMode>(p, d, tid, tb, tp, b0, p0, own_lo, M, Sm, S2, s_res);
    } else {
      // split tile: leave this piece's (max, sum[, E0 sum]) for the merge
      const int slot = (a_begin >= t_first) ? 0 : 1;
      float* mine = p.part + ((c * 2 + slot) * NV) * (size_t)(BT * PT) + tid * NOUT;
#pragma unroll
      for (int o = 0; o < NOUT; o += 4) {
        __stcg(reinterpret_cast<float4*>(mine + o), make_float4(M[o], M[o + 1], M[o + 2], M[o + 3]));
        __stcg(reinterpret_cast<float4*>(mine + BT * PT + o),
               make_float4(Sm[o], Sm[o + 1], Sm[o + 2], Sm[o + 3]));
        if (NV == 3)
          __stcg(reinterpret_cast<float4*>(mine + 2 * BT * PT + o),
                 make_float4(S2[o], S2[o + 1], S2[o + 2], S2[o + 3]));
      }
    }
    reset_acc();
  }
  seq += n_local;
}

template <int BT, int PT, int QC, int RB, int RP, int NSTAGE, bool kGrid, int kMode>
__global__ void __launch_bounds__((BT / RB) * (PT / RP), ((BT / RB) * (PT / RP) >= 512) ? 1 : SKB_OCC_SMALL)
    tiled_sweep_kernel(const __grid_constant__ CUtensorMap tmap_g,
                       const __grid_constant__ CUtensorMap tmap_x, const TiledSweepParams p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const SweepSmem<BT, PT, QC, RB, RP, NSTAGE, kGrid, kMode> sm(smem_raw);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) mbar_init(&sm.bars[s], 1);
    fence_barrier_init();
    if (!kGrid) prefetch_tmap(&tmap_g);
    prefetch_tmap(&tmap_x);
  }
  __syncthreads();
  // Everything above overlaps the previous kernel's tail; inputs are read below.
  pdl_wait();
#ifndef SKB_PDL_LATE
  // let the dependent (fixup) grid launch now: its CTAs take SMs as ours
  // retire and wait in griddepcontrol.wait for this grid's completion
  pdl_launch_dependents();
#endif
  uint32_t seq = 0;
  if (p.dbg && threadIdx.x == 0) p.dbg[2 * blockIdx.x] = globaltimer_ns();
  sweep_phase<BT, PT, QC, RB, RP, NSTAGE, kGrid, kMode>(&tmap_g, &tmap_x, p, dyn_of(p), sm, seq);
  if (p.dbg) {
    __syncthreads();
    if (threadIdx.x == 0) p.dbg[2 * blockIdx.x + 1] = globaltimer_ns();
  }
#ifdef SKB_PDL_LATE
  pdl_launch_dependents();
#endif
}

// Merge the stream-K pieces of every split tile in ascending CTA order (the
// reference's ascending span merge, batch.py:198-201: deterministic) and run
// the tile epilogue.  One CTA per tile, same thread map as the sweep, so each
// thread merges exactly the outputs its counterpart accumulated.  Launched
// right after the sweep with programmatic dependent launch.
// Merge float4 groups [g0, g1) (4 outputs of one lane each) of split tile
// `tile`: every thread takes one group per round.  (Merging inside the sweep
// instead -- per-tile piece counters, the contributing CTAs each merging a
// share once the tile is complete -- measured slower on B200: 11.4 vs 10.0 ms
// at config 2, so the merge stays a separate PDL-launched pass.)
template <int BT, int PT, int QC, int RB, int RP, int kMode, int NB>
__device__ __forceinline__ void merge_tile_groups(const TiledSweepParams& p, const SweepDyn& d,
                                                  int tile, int g0, int g1, float* s_res) {
  constexpr int NT = (BT / RB) * (PT / RP);   // the sweep's threads per tile
  constexpr int NOUT = RB * RP;
  constexpr int NG = NOUT / 4;                // float4 groups per sweep thread (one per rb)
  constexpr int NV = (kMode == kModeTail) ? 3 : 2;
  constexpr int GRP = 8;                      // pieces whose loads are in flight together
  static_assert(RP == 4, "one float4 group = the RP outputs of one lane");
  const long long Qv = p.Qv;
  const long long t_first = (long long)tile * Qv;
  const long long c_lo = atom_owner(p, t_first);
  const long long c_hi = atom_owner(p, t_first + Qv - 1);
  if (c_lo == c_hi) return;   // finalised by the sweep itself (CTA-uniform)
  // only the tile's first piece can be its CTA's second slot (the CTA began
  // in an earlier tile); every later piece starts inside this tile
  const int sl0 = (atom_begin(p, c_lo) < t_first) ? 1 : 0;
  const int tb_idx = tile % p.ntile_b, tp_idx = tile / p.ntile_b;
  const int p0 = (tp_idx == p.ntile_p - 1) ? max((p.Pv - PT + 3) & ~3, 0) : tp_idx * PT;
  const int own_lo = tp_idx * PT;
  const bool want_res = p.res != nullptr && (kMode == kModeTail || d.res_kind != kResNone);
  for (int gb = g0; gb < g1; gb += NB) {
  const int e = gb + (int)threadIdx.x;             // float4 group within the tile
  const bool act = e < g1;
  const int vtid = (act ? e : g0) / NG, rb = (act ? e : g0) % NG;   // mirrored sweep thread, lane
  int tb, tp;
  thread_map<BT, RB, NT>(vtid, tb, tp);
  const int b = tb_idx * BT + tb * RB + rb;
  // epilogue inputs do not depend on the pieces: their loads go out first
  float tgv[4], eov[4], odv[4], mgv[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int pp = min(p0 + tp * RP + r, p.Pv - 1);
    const size_t o = size_t(pp) * p.Bp + b;
    tgv[r] = eov[r] = odv[r] = mgv[r] = 0.f;
    if (kMode == kModeUpdate) {
      tgv[r] = __ldg(p.target + o);
      if (d.use_est) eov[r] = d.est_old[o];
    }
    if (kMode == kModeTail || d.res_kind == kResCol) odv[r] = d.old[o];
    if (want_res) mgv[r] = __ldg(p.marg + o);
  }
  float M[4], Sm[4], S2[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    M[r] = kNegBig;
    Sm[r] = 0.f;
    S2[r] = 0.f;
  }
#pragma unroll 1
  for (long long c0 = c_lo; c0 <= c_hi; c0 += GRP) {
    float4 mv[GRP], sv[GRP], tv[GRP];
#pragma unroll
    for (int g = 0; g < GRP; ++g) {
      const long long cc = c0 + g;
      if (cc > c_hi || !act) break;
      const int sl = (cc == c_lo) ? sl0 : 0;
      const float* src = p.part + ((cc * 2 + sl) * NV) * (size_t)(BT * PT) + vtid * NOUT + rb * 4;
      mv[g] = __ldcg(reinterpret_cast<const float4*>(src));
      sv[g] = __ldcg(reinterpret_cast<const float4*>(src + BT * PT));
      if (NV == 3) tv[g] = __ldcg(reinterpret_cast<const float4*>(src + 2 * BT * PT));
    }
#pragma unroll
    for (int g = 0; g < GRP; ++g) {
      if (c0 + g > c_hi || !act) break;   // ascending piece order (batch.py:198-201)
      const float* m2 = reinterpret_cast<const float*>(&mv[g]);
      const float* s2 = reinterpret_cast<const float*>(&sv[g]);
      const float* t2 = reinterpret_cast<const float*>(&tv[g]);
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const float mn = fmaxf(M[r], m2[r]);
        const float ra = ex2(M[r] - mn), rb2 = ex2(m2[r] - mn);
        Sm[r] = Sm[r] * ra + s2[r] * rb2;
        if (NV == 3) S2[r] = S2[r] * ra + t2[r] * rb2;
        M[r] = mn;
      }
    }
  }
  // epilogue for lane b, outputs p0 + tp*RP + r
  if (want_res) {
    for (int i = threadIdx.x; i < BT; i += NB) s_res[i] = 0.f;
    __syncthreads();
  }
  float rmax = 0.f;
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int pp = p0 + tp * RP + r;
    if (!act || pp >= p.Pv || pp < own_lo) continue;
    const size_t o = size_t(pp) * p.Bp + b;
    if (kMode == kModePartial) {
      p.pmax[o] = M[r];
      p.psum[o] = Sm[r];
      continue;
    }
    const float lse = lse_final(M[r], Sm[r]);
    if (kMode == kModeUpdate) {
      const float tg = tgv[r];
      if (d.use_est) {
        const float est = tg - eov[r];
        if (tg != neg_inf() && isfinite(est) && !(lse >= est - kEstSlack)) atomicOr(p.est_fail, 1);
      }
      const float ov = sweep_out(tg, lse);
      d.out[o] = ov;
      if (want_res) {
        const float base = (d.res_kind == kResCol) ? odv[r] : ov;
        rmax = fmaxf(rmax, fabsf(exp2f(base + lse) - mgv[r]));
      }
    } else {   // TAIL
      const float od = odv[r];
      p.e0[o] = (S2[r] > 0.f) ? (M[r] + log2f(S2[r]) + od) : neg_inf();
      rmax = fmaxf(rmax, fabsf(exp2f(od + lse) - mgv[r]));
    }
  }
  if (want_res) {
    const float v = (rmax != rmax) ? __int_as_float(0x7fc00000) : rmax;
    atomic_max_nonneg(&s_res[b - tb_idx * BT], v);
    __syncthreads();
    for (int i = threadIdx.x; i < BT; i += NB) {
      const float rv = s_res[i];
      if (rv != 0.f) atomic_max_nonneg(&p.res[tb_idx * BT + i], rv);
    }
    __syncthreads();   // s_res is reused by the next chunk
  }
  }   // rounds of NB groups
}

template <int BT, int PT, int QC, int RB, int RP, int kMode, int NB>
__device__ __forceinline__ void fixup_chunk(const TiledSweepParams& p, const SweepDyn& d, int chunk,
                                            float* s_res) {
  constexpr int NT = (BT / RB) * (PT / RP);
  constexpr int GT = NT * (RB * RP / 4);      // float4 groups per tile
  static_assert(GT % NB == 0, "chunks align with tiles");
  constexpr int CPT = GT / NB;
  const int tile = chunk / CPT, g0 = (chunk % CPT) * NB;
  merge_tile_groups<BT, PT, QC, RB, RP, kMode, NB>(p, d, tile, g0, g0 + NB, s_res);
}

template <int BT, int PT, int QC, int RB, int RP, int kMode>
__global__ void __launch_bounds__(256) tiled_fixup_kernel(const TiledSweepParams p) {
  __shared__ float s_res[BT];
  pdl_wait();
#ifndef SKB_PDL_LATE
  pdl_launch_dependents();
#endif
  if (p.dbg && threadIdx.x == 0) p.dbg[4096 + 2 * blockIdx.x] = globaltimer_ns();
  fixup_chunk<BT, PT, QC, RB, RP, kMode, 256>(p, dyn_of(p), blockIdx.x, s_res);
  if (p.dbg) {
    __syncthreads();
    if (threadIdx.x == 0) p.dbg[4096 + 2 * blockIdx.x + 1] = globaltimer_ns();
  }
#ifdef SKB_PDL_LATE
  pdl_launch_dependents();
#endif
}

}  // namespace skb
