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

namespace skb {


struct TiledSweepParams {
  int Qv, Pv;          // valid reduce / output extents (d)
  int Bp;              // padded lane count (row stride of dim-major buffers)
  int ntile_b, ntile_p, nq;
  long long W;         // atoms = ntile_b * ntile_p * nq
  int G;               // grid size
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
};

template <int BT, int PT, int QC, int RB, int RP, int KC, int NSTAGE, bool kGrid, int kMode>
struct TiledSweep {
  static constexpr int NT = (BT / RB) * (PT / RP);
  static constexpr int NTB = BT / RB;          // threads along lanes (within a warp)
  static constexpr int NV = (kMode == kModeTail) ? 3 : 2;
  static constexpr int G_FLOATS = QC * PT;
  static constexpr int X_FLOATS = QC * BT;
  static constexpr int STAGE_FLOATS = G_FLOATS + X_FLOATS;
  static constexpr uint32_t TMA_BYTES = (kGrid ? 0 : G_FLOATS * 4) + X_FLOATS * 4;
  static constexpr size_t SMEM_BYTES =
      1024 /*align slack*/ + size_t(NSTAGE) * STAGE_FLOATS * 4 + 64 * 8 /*bars*/ + BT * 4 +
      (kGrid ? (QC + PT) * 8 : 0);
  static_assert(NTB == 16, "thread map assumes 16 lane-threads per half warp");
  static_assert(NT % 32 == 0, "whole warps");
  static_assert(RB == 4 && RP == 4, "float4 tile loads");
  static_assert(QC % KC == 0, "sub-chunks");
};

__device__ __forceinline__ long long atom_begin(long long c, long long W, long long G) {
  return (c * W) / G;
}
// CTA owning atom a: largest c with atom_begin(c) <= a.
__device__ __forceinline__ long long atom_owner(long long a, long long W, long long G) {
  return ((a + 1) * G - 1) / W;
}

template <int BT, int PT, int QC, int RB, int RP, int KC, int NSTAGE, bool kGrid, int kMode>
__global__ void __launch_bounds__((BT / RB) * (PT / RP), 1)
    tiled_sweep_kernel(const __grid_constant__ CUtensorMap tmap_g,
                       const __grid_constant__ CUtensorMap tmap_x, const TiledSweepParams p) {
  using S = TiledSweep<BT, PT, QC, RB, RP, KC, NSTAGE, kGrid, kMode>;
  constexpr int NT = S::NT;
  constexpr int NV = S::NV;
  constexpr int NOUT = RB * RP;

  extern __shared__ uint8_t smem_raw[];
  float* smem = reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NSTAGE * S::STAGE_FLOATS);
  float* s_res = reinterpret_cast<float*>(bars + 64);
  int* s_flag = reinterpret_cast<int*>(bars + 60);
  float* s_gq = s_res + BT;        // grid mode: q coordinates (x, y) [QC][2]
  float* s_gp = s_gq + 2 * QC;     // grid mode: p coordinates [PT][2]

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int tb = lane & 15;                 // lane-group index (b = tb*RB + rb)
  const int tp = warp * 2 + (lane >> 4);    // output-group index (p = tp*RP + rp)

  const long long W = p.W;
  const long long Gc = p.G;
  const long long c = blockIdx.x;
  const long long a_begin = atom_begin(c, W, Gc);
  const long long a_end = atom_begin(c + 1, W, Gc);
  const int n_local = int(a_end - a_begin);
  const int nq = p.nq;

  if (tid == 0) {
    for (int s = 0; s < NSTAGE; ++s) mbar_init(&bars[s], 1);
    fence_barrier_init();
    if (!kGrid) prefetch_tmap(&tmap_g);
    prefetch_tmap(&tmap_x);
  }
  __syncthreads();
  // Everything above overlaps the previous kernel's tail; inputs are read below.
  pdl_wait();

  auto atom_coords = [&](long long a, int& tile, int& qc, int& b0, int& p0) {
    tile = int(a / nq);
    qc = int(a - (long long)tile * nq);
    const int tb_idx = tile % p.ntile_b;     // lane tiles innermost: consecutive tiles share G
    const int tp_idx = tile / p.ntile_b;
    b0 = tb_idx * BT;
    p0 = tp_idx * PT;
  };

  auto issue = [&](int l) {
    const long long a = a_begin + l;
    int tile, qc, b0, p0;
    atom_coords(a, tile, qc, b0, p0);
    const int s = l % NSTAGE;
    float* st = smem + s * S::STAGE_FLOATS;
    mbar_arrive_expect_tx(&bars[s], S::TMA_BYTES);
    if (!kGrid) tma_load_2d(st, &tmap_g, p0, qc * QC, &bars[s]);
    tma_load_2d(st + S::G_FLOATS, &tmap_x, b0, qc * QC, &bars[s]);
  };

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

  // finalize one output tile from the accumulators in registers
  auto epilogue = [&](int b0, int p0) {
    if (p.res != nullptr && (kMode == kModeTail || p.res_kind != kResNone)) {
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
      if (pp >= p.Pv) continue;
      const size_t row = size_t(pp) * p.Bp + bb;
      if (kMode == kModePartial) {
        *reinterpret_cast<float4*>(p.pmax + row) =
            make_float4(M[0 * RP + rp], M[1 * RP + rp], M[2 * RP + rp], M[3 * RP + rp]);
        *reinterpret_cast<float4*>(p.psum + row) =
            make_float4(Sm[0 * RP + rp], Sm[1 * RP + rp], Sm[2 * RP + rp], Sm[3 * RP + rp]);
        continue;
      }
      float lse[RB];
#pragma unroll
      for (int rb = 0; rb < RB; ++rb) lse[rb] = lse_final(M[rb * RP + rp], Sm[rb * RP + rp]);
      if (kMode == kModeUpdate) {
        const float4 tg = *reinterpret_cast<const float4*>(p.target + row);
        const float tv[4] = {tg.x, tg.y, tg.z, tg.w};
        float ov[4];
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) ov[rb] = sweep_out(tv[rb], lse[rb]);
        *reinterpret_cast<float4*>(p.out + row) = make_float4(ov[0], ov[1], ov[2], ov[3]);
        if (p.res != nullptr && p.res_kind != kResNone) {
          const float4 mg = *reinterpret_cast<const float4*>(p.marg + row);
          const float mv[4] = {mg.x, mg.y, mg.z, mg.w};
          float base[4] = {ov[0], ov[1], ov[2], ov[3]};
          if (p.res_kind == kResCol) {
            const float4 od = *reinterpret_cast<const float4*>(p.old + row);
            base[0] = od.x; base[1] = od.y; base[2] = od.z; base[3] = od.w;
          }
#pragma unroll
          for (int rb = 0; rb < RB; ++rb)
            rmax[rb] = fmaxf(rmax[rb], fabsf(exp2f(base[rb] + lse[rb]) - mv[rb]));
        }
      } else {  // TAIL: column residual against `old` and the E0 term
        const float4 od = *reinterpret_cast<const float4*>(p.old + row);
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
    }
    if (p.res != nullptr && (kMode == kModeTail || p.res_kind != kResNone)) {
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
  };

  int cur_tile = -1;
  int seg_q0 = 0;
  for (int l = 0; l < n_local; ++l) {
    const long long a = a_begin + l;
    int tile, qc, b0, p0;
    atom_coords(a, tile, qc, b0, p0);
    if (tile != cur_tile) {
      cur_tile = tile;
      seg_q0 = qc;
    }
    const int s = l % NSTAGE;
    const uint32_t parity = (l / NSTAGE) & 1;
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
    mbar_wait(&bars[s], parity);
    if (kGrid) __syncthreads();

    // ---- consume: the hot loop --------------------------------------------
    const int kvalid = min(QC, p.Qv - qc * QC);
    const bool active = (p0 + tp * RP) < p.Pv;   // uniform per half-warp
    if (active) {
      for (int kk = 0; kk < kvalid; kk += KC) {
        float g[KC][RP], x[KC][RB];
#pragma unroll
        for (int k = 0; k < KC; ++k) {
          const float4 gv = *reinterpret_cast<const float4*>(Gs + (kk + k) * PT + tp * RP);
          const float4 xv = *reinterpret_cast<const float4*>(Xs + (kk + k) * BT + tb * RB);
          g[k][0] = gv.x; g[k][1] = gv.y; g[k][2] = gv.z; g[k][3] = gv.w;
          x[k][0] = xv.x; x[k][1] = xv.y; x[k][2] = xv.z; x[k][3] = xv.w;
        }
        float cw[KC][RP];
        if (kMode == kModeTail) {
          // c = G * cinv; padding rows (G = -inf) must weigh 0, not +inf
#pragma unroll
          for (int k = 0; k < KC; ++k)
#pragma unroll
            for (int rp = 0; rp < RP; ++rp)
              cw[k][rp] = (g[k][rp] == neg_inf()) ? 0.f : g[k][rp] * p.cinv;
        }
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) {
#pragma unroll
          for (int rp = 0; rp < RP; ++rp) {
            const int o = rb * RP + rp;
            float t[KC];
            float cm = kNegBig;
#pragma unroll
            for (int k = 0; k < KC; ++k) {
              t[k] = g[k][rp] + x[k][rb];
              cm = fmaxf(cm, t[k]);
            }
            if (cm > M[o] + kLazy) {   // lazy online rescale (batch.py:98-105)
              const float r = ex2(M[o] - cm);
              Sm[o] *= r;
              if (kMode == kModeTail) S2[o] *= r;
              M[o] = cm;
            }
            float e[KC], e2[KC];
#pragma unroll
            for (int k = 0; k < KC; ++k) {
              e[k] = ex2(t[k] - M[o]);
              if (kMode == kModeTail) e2[k] = e[k] * cw[k][rp];
            }
            // pairwise tree inside the chunk keeps the fp32 error ~ sqrt(Q/KC)
#pragma unroll
            for (int w = 1; w < KC; w *= 2)
#pragma unroll
              for (int k = 0; k + w < KC; k += 2 * w) {
                e[k] += e[k + w];
                if (kMode == kModeTail) e2[k] += e2[k + w];
              }
            Sm[o] += e[0];
            if (kMode == kModeTail) S2[o] += e2[0];
          }
        }
      }
    }
    __syncthreads();   // every warp is done with stage s
    if (tid == 0 && l + NSTAGE < n_local) issue(l + NSTAGE);

    // ---- segment end: finalize or hand over to the stream-K merge ---------
    const bool seg_end = (qc == nq - 1) || (l == n_local - 1);
    if (!seg_end) continue;
    const long long t_first = (long long)tile * nq;
    const long long c_lo = atom_owner(t_first, W, Gc);
    const long long c_hi = atom_owner(t_first + nq - 1, W, Gc);
    if (c_lo == c_hi) {
      epilogue(b0, p0);
    } else {
      const int slot = (a_begin >= t_first) ? 0 : 1;
      float* mine = p.part + ((c * 2 + slot) * NV) * (size_t)(BT * PT);
#pragma unroll
      for (int o = 0; o < NOUT; o += 4) {
        *reinterpret_cast<float4*>(mine + tid * NOUT + o) =
            make_float4(M[o], M[o + 1], M[o + 2], M[o + 3]);
        *reinterpret_cast<float4*>(mine + BT * PT + tid * NOUT + o) =
            make_float4(Sm[o], Sm[o + 1], Sm[o + 2], Sm[o + 3]);
        if (NV == 3)
          *reinterpret_cast<float4*>(mine + 2 * BT * PT + tid * NOUT + o) =
              make_float4(S2[o], S2[o + 1], S2[o + 2], S2[o + 3]);
      }
      __threadfence();
      __syncthreads();
      if (tid == 0) {
        const int pieces = int(c_hi - c_lo + 1);
        const int prev = atomicAdd(&p.counters[tile], 1);
        *s_flag = (prev == pieces - 1);
      }
      __syncthreads();
      if (*s_flag) {
        __threadfence();
        reset_acc();
        for (long long cc = c_lo; cc <= c_hi; ++cc) {
          const int sl = (atom_begin(cc, W, Gc) >= t_first) ? 0 : 1;
          const float* src = p.part + ((cc * 2 + sl) * NV) * (size_t)(BT * PT);
#pragma unroll
          for (int o = 0; o < NOUT; ++o) {
            const float m2 = __ldcg(src + tid * NOUT + o);
            const float s2v = __ldcg(src + BT * PT + tid * NOUT + o);
            const float mn = fmaxf(M[o], m2);
            const float ra = ex2(M[o] - mn), rb2 = ex2(m2 - mn);
            Sm[o] = Sm[o] * ra + s2v * rb2;
            if (NV == 3) S2[o] = S2[o] * ra + __ldcg(src + 2 * BT * PT + tid * NOUT + o) * rb2;
            M[o] = mn;
          }
        }
        epilogue(b0, p0);
        if (tid == 0) p.counters[tile] = 0;
      }
    }
    reset_acc();
    (void)seg_q0;
  }
  pdl_launch_dependents();
}

}  // namespace skb
