// common.cuh -- sm_100a helpers shared by the Sinkhorn kernels.
//
// Everything the iteration computes lives in log base 2: potentials
// f2 = log_u * log2(e), costs A2 = -c * log2(e) / lambda, so every exponential
// is one MUFU.EX2 (ex2.approx.ftz.f32) and every log one MUFU.LG2.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace skb {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;
// Finite "minus infinity" for running maxima: keeps (m - m') finite so the
// online rescale never evaluates exp(-inf - -inf) = NaN (batch.py:106-110
// guards the same case with its _maybe_dead mask).
constexpr float kNegBig = -1.0e30f;
// Lazy rescale threshold (log2 units): the running max is only raised when a
// chunk exceeds it by more than this, so terms stay <= 2^8 and the sum of up
// to 2^20 of them cannot overflow fp32.
constexpr float kLazy = 8.0f;

// Half-sweep epilogues (see sweep_tiled.cuh) and fused residual terms.
enum SweepMode : int { kModeUpdate = 0, kModePartial = 1, kModeTail = 2 };
enum ResKind : int { kResNone = 0, kResRow = 1, kResCol = 2 };

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float lg2(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float neg_inf() { return __int_as_float(0xff800000); }

// ---- sm_100 packed fp32 (FADD2 / FFMA2) and 3-input max (FMNMX3) -----------
// Two fp32 lanes in one 64-bit register pair; a scalar operand packed as
// {g, g} is folded by ptxas into the instruction's broadcast form.
__device__ __forceinline__ uint64_t pk2(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float lo2(uint64_t v) {
  return __uint_as_float(static_cast<uint32_t>(v));
}
__device__ __forceinline__ float hi2(uint64_t v) {
  return __uint_as_float(static_cast<uint32_t>(v >> 32));
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
// In-place accumulators (read-write operand): the running sum keeps its
// register pair across loop iterations instead of being copied every step.
__device__ __forceinline__ void ffma2_acc(uint64_t& acc, uint64_t a, uint64_t b) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(a), "l"(b));
}
__device__ __forceinline__ void fadd2_acc(uint64_t& acc, uint64_t a) {
  asm("add.rn.f32x2 %0, %0, %1;" : "+l"(acc) : "l"(a));
}
__device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
// 2^a for a pair on the FMA pipe (FADD2/FFMA2 + integer exponent add), so a
// share of the exponentials bypasses the 16/clk/SM MUFU (FlashAttention-4's
// trick).  Degree-5 near-minimax polynomial on [-0.5, 0.5]: max relative
// error 2.1e-7 in fp32, on par with ex2.approx.  Inputs below -126 return a
// value <= 2^-126 (not exactly 0): only used where such terms are negligible
// against a running sum near 1 (the solver's sweeps, not the empty-reduction
// half-sweep API).
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b);
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c);
__device__ __forceinline__ uint64_t ex2_poly2(uint64_t a) {
  float lo, hi;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(a));
  const uint64_t x = pk2(fmaxf(lo, -126.f), fmaxf(hi, -126.f));
  const uint64_t t = fadd2(x, pk2(12582912.f, 12582912.f));        // 1.5 * 2^23: round
  const uint64_t j = fadd2(t, pk2(-12582912.f, -12582912.f));      // nearest integer
  const uint64_t f = ffma2(j, pk2(-1.f, -1.f), x);                  // x - j in [-1/2, 1/2]
  uint64_t p = ffma2(pk2(1.3276466634124517e-3f, 1.3276466634124517e-3f), f,
                     pk2(9.675540961325169e-3f, 9.675540961325169e-3f));
  p = ffma2(p, f, pk2(5.550713464617729e-2f, 5.550713464617729e-2f));
  p = ffma2(p, f, pk2(2.4022120237350464e-1f, 2.4022120237350464e-1f));
  p = ffma2(p, f, pk2(6.931469440460205e-1f, 6.931469440460205e-1f));
  p = ffma2(p, f, pk2(1.0000001192092896f, 1.0000001192092896f));
  // times 2^j: the integer j sits in t's low mantissa bits, so t << 23 is j << 23
  float p0, p1, t0, t1;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(p0), "=f"(p1) : "l"(p));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(t0), "=f"(t1) : "l"(t));
  return pk2(__uint_as_float(__float_as_uint(p0) + (__float_as_uint(t0) << 23)),
             __uint_as_float(__float_as_uint(p1) + (__float_as_uint(t1) << 23)));
}

__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}

// A potential (log2 units) is a broken state when it is NaN or +inf -- or at
// the scale of the finite -inf sentinel kNegBig, which only an empty
// reduction produces.  That is the case where a target with positive mass has
// no finite term in its reduction (every -c/lambda is -inf): the reference's
// next half-sweep then evaluates -inf + inf = NaN and batch_forward raises
// NaNProduced (batch.py:326-327), so the device reports status 12.
constexpr float kStateMax = 1.0e29f;
__device__ __forceinline__ bool broken_state(float v) { return !(v <= kStateMax); }

// (m, s) -> log2-sum-exp; an empty accumulator (s == 0) is -inf (batch.py:132-138).
__device__ __forceinline__ float lse_final(float m, float s) {
  return s > 0.0f ? m + log2f(s) : neg_inf();
}

// OnlineLseAccumulator.merge (batch.py:116-130) on (max, sum) pairs; both
// maxima are finite (>= kNegBig) by construction so no NaN guard is needed.
__device__ __forceinline__ void lse_merge(float& m, float& s, float m2, float s2) {
  float mn = fmaxf(m, m2);
  s = s * ex2(m - mn) + s2 * ex2(m2 - mn);
  m = mn;
}

// target - lse with the reference's zero-mass rule: a -inf target stays -inf
// (test_reduction.py:207-216) even where the reduction is also empty.
__device__ __forceinline__ float sweep_out(float target, float lse) {
  return target == neg_inf() ? neg_inf() : target - lse;
}

// Non-negative float max via integer atomics (order-independent, deterministic).
__device__ __forceinline__ void atomic_max_nonneg(float* addr, float v) {
  atomicMax(reinterpret_cast<unsigned int*>(addr), __float_as_uint(v));
}

// ---- programmatic dependent launch (griddepcontrol) ----------------------
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// ---- mbarrier + TMA ------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(tmap)) : "memory");
}

// 2-D tiled TMA load: box at (c0 = inner coordinate, c1 = outer) into smem,
// completing `bytes` on the mbarrier.
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const void* tmap, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(tmap)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ int warp_id() { return threadIdx.x >> 5; }
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// Grid-wide barrier for a cooperative launch: the counter only grows, so
// epoch e completes when it reaches e * gridDim.x.  The release reduction and
// the acquire load (which also invalidates L1) order every CTA's global
// writes before every later read; the async-proxy fence covers TMA reads of
// data written with ordinary stores.
__device__ __forceinline__ void grid_sync(unsigned int* counter, unsigned int& epoch) {
  asm volatile("fence.proxy.async.global;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    ++epoch;
    const unsigned int target = epoch * gridDim.x;
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(counter), "r"(1u) : "memory");
    unsigned int v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(counter) : "memory");
    } while (v < target);
  }
  __syncthreads();
}

// Status word: first error wins, in stream order, which reproduces the
// reference's check order (shapes on the host, then histograms ffi.ts:111-115,
// then the cost the CLI validates, core.py:53-63).
__device__ __forceinline__ void set_status(int* status, int code) { atomicCAS(status, 0, code); }

__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// 16-byte asynchronous global -> shared copy (LDGSTS, L2 only) and its wait.
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)),
               "l"(gmem_src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

}  // namespace skb
