// persistent.cuh -- the whole lockstep iteration (batch.py:314-324) in one
// cooperative kernel for shared / grid costs.
//
// One CTA per SM (all resident: cooperative launch) runs every half-sweep as
//   stream-K sweep phase -> grid barrier -> fixup phase -> grid barrier
// instead of two kernel launches per half-sweep, so the ~400 launch gaps and
// ramp-up/tail bubbles of a 100-iteration solve disappear.  The convergence
// test (tolerance > 0) is evaluated on the device from the fused residuals:
// after the check sweep every CTA reads the same per-lane residuals and takes
// the same decision, so no host synchronisation is needed inside the loop.
//
// The loop is a small state machine around ONE inlined sweep_phase call site
// (one copy of the hot loop, the same register allocation as the standalone
// sweep kernel); every sweep variant's parameters are precomputed on the host
// into the kernel-parameter space and selected by index.
#pragma once

#include "sweep_tiled.cuh"

namespace skb {

struct PersistMaps {
  CUtensorMap a2;      // G for column sweeps (unused for grid costs)
  CUtensorMap a2t;     // G for row sweeps
  CUtensorMap f2;      // X for column sweeps
  CUtensorMap g2[2];   // X for row sweeps (ping-pong log_v buffers)
};

struct PersistParams {
  TiledSweepParams col;   // static part of every column sweep (reads f2, writes a g2 buffer)
  TiledSweepParams row;   // static part of every row sweep (reads a g2 buffer, writes f2)
  float* g2[2];
  float* f2;
  float* res;             // [Bp] fused residuals (zero on entry)
  int B, Bp;
  int max_iters, check_interval, est_from;
  double tol;
  unsigned int* bar;      // grid-barrier counter (zero on entry)
  int* result;            // out: [0] iterations_run, [1] index of the final log_v buffer
};

template <int BT, int PT, int QC, int RB, int RP, int NSTAGE, bool kGrid>
__global__ void __launch_bounds__((BT / RB) * (PT / RP), 1)
    persistent_solve_kernel(const __grid_constant__ PersistMaps maps,
                            const __grid_constant__ PersistParams P) {
  using SM = SweepSmem<BT, PT, QC, RB, RP, NSTAGE, kGrid, kModeUpdate>;
  constexpr int NT = (BT / RB) * (PT / RP);
  constexpr int CPT = RB * RP / 4;   // fixup chunks (of NT float4 groups) per tile
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const SM sm(smem_raw);
  __shared__ unsigned int s_max;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) mbar_init(&sm.bars[s], 1);
    fence_barrier_init();
    if (!kGrid) {
      prefetch_tmap(&maps.a2);
      prefetch_tmap(&maps.a2t);
    }
    prefetch_tmap(&maps.f2);
    prefetch_tmap(&maps.g2[0]);
    prefetch_tmap(&maps.g2[1]);
  }
  __syncthreads();
  uint32_t seq = 0;
  unsigned int epoch = 0;

  // state machine over the reference's loop (batch.py:314-324)
  enum : int { kColumn = 0, kRow = 1, kCheckColumn = 2 };
  const bool checks = P.tol > 0;
  int k = 1, cur = 0, step = kColumn, iters = 0;
  while (k <= P.max_iters) {
    const bool last = (k == P.max_iters);
    const bool check = checks && (k % P.check_interval == 0) && !last;
    const int est = (k >= P.est_from) ? 1 : 0;
    const bool row = (step == kRow);
    const int buf = row ? cur : (cur ^ 1);
    const int res = row ? ((check || last) ? 1 : 0) : (step == kCheckColumn ? 1 : 0);
    // two call sites (column / row) so each reads its static parameters
    // straight from the kernel-parameter bank
    // The parameter block is reached through a pointer made opaque in every
    // iteration, so no field is hoisted out of this loop and kept live across
    // the sweep (the hot loop needs all 128 registers of a 512-thread CTA).
    const TiledSweepParams* pp = row ? &P.row : &P.col;
    const CUtensorMap* tg = row ? &maps.a2t : &maps.a2;
    const CUtensorMap* tx = row ? &maps.g2[buf] : &maps.f2;
    asm volatile("" : "+l"(pp), "+l"(tg), "+l"(tx));
    const SweepDyn d = row ? SweepDyn{P.f2, nullptr, P.f2, est, res ? kResRow : kResNone}
                           : SweepDyn{P.g2[buf], P.g2[buf ^ 1], P.g2[buf ^ 1], est,
                                      res ? kResCol : kResNone};
    sweep_phase<BT, PT, QC, RB, RP, NSTAGE, kGrid, kModeUpdate>(tg, tx, *pp, d, sm, seq);
    grid_sync(P.bar, epoch);
    const int chunks = pp->ntile_b * pp->ntile_p * CPT;
    for (int ch = blockIdx.x; ch < chunks; ch += gridDim.x)
      fixup_chunk<BT, PT, QC, RB, RP, kModeUpdate, NT>(*pp, d, ch, sm.s_res);
    grid_sync(P.bar, epoch);

    if (step == kColumn) {
      cur ^= 1;
      step = kRow;
    } else if (step == kRow) {
      iters = k;
      if (check) {
        step = kCheckColumn;   // column sweep k+1 doubles as the column residual of k
      } else {
        ++k;
        step = kColumn;
      }
    } else {   // kCheckColumn: decide on the device, identically in every CTA
      float mx = 0.f;
      for (int b = threadIdx.x; b < P.B; b += NT) {
        float r;
        asm volatile("ld.relaxed.gpu.global.f32 %0, [%1];" : "=f"(r) : "l"(P.res + b));
        mx = (r != r || mx != mx) ? __int_as_float(0x7f800000) : fmaxf(mx, r);   // NaN: no stop
      }
      if (threadIdx.x == 0) s_max = 0u;
      __syncthreads();
      atomicMax(&s_max, __float_as_uint(mx));
      __syncthreads();
      const bool converged = (double)__uint_as_float(s_max) <= P.tol;
      grid_sync(P.bar, epoch);   // every CTA has read the residuals
      if (converged) break;      // keep g2[cur] = log_v_k; the k+1 sweep is discarded
      for (int b = blockIdx.x * NT + threadIdx.x; b < P.Bp; b += gridDim.x * NT) P.res[b] = 0.f;
      grid_sync(P.bar, epoch);
      cur ^= 1;                  // log_v_{k+1} is already computed
      ++k;
      step = kRow;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    P.result[0] = iters;
    P.result[1] = cur;
  }
}

}  // namespace skb
