// sweep_umma.cuh -- the shared-cost contractions of the linear-domain
// iteration (sweep_gemm.cuh) on the tcgen05 tensor cores, 3xTF32.
//
//   D[m][n] = sum_k A[m][k] * B[n][k]        (out[n * ldo + m], lane-major)
//
// A is the kernel matrix K = 2^A2 (row sweep: S = K X, M = d1) or its stored
// transpose (column sweep: T = K^T a, M = d2), fp32 row-major, streamed from
// HBM once per contraction; B is the lanes' X or a, pre-split on the device
// into tf32 hi / lo planes (B <= 64 lanes per N tile).  Products are
// hi*hi + hi*lo + lo*hi (the dropped lo*lo term is < 2^-22 relative): every
// operand and every product is positive, so the relative error of each term
// bounds the sum's.
//
// Accumulation precision.  The tensor core adds each MMA's result into the
// fp32 TMEM accumulator with truncation (tools/micro/umma_probe.cu: a K=65536
// accumulation in TMEM is 1e-3 low).  Every k-chunk (32 reduction indices, 12
// MMAs) therefore goes to its own accumulator slot, and the epilogue warps add
// the slots into fp32 registers with round-to-nearest (the "promotion" of
// FP8 GEMMs): the bias is then <= 12 truncations per chunk (~7e-7 relative).
//
// Warp roles (384 threads, one CTA per SM, persistent stream-K over
// (tile, k-chunk) units, split tiles merged in ascending CTA order by
// umma_fixup_kernel -- deterministic, like the reference's ascending span
// merge, batch.py:198-201):
//   warp 0      TMA producer, A ring: tile [128][32] (evict-first), SW128
//   warp 3      TMA producer, B ring: hi / lo tiles [64][32] (evict-last)
//   warp 1      MMA issuer (one thread): 12 kind::tf32 MMAs per chunk, A from TMEM
//   warp 2      TMEM allocator
//   warps 4-7   splitters: A tile rows smem -> registers -> hi / lo -> TMEM
//   warps 8-11  epilogue: accumulator slot -> registers (+=) -> global
#pragma once

#include <cuda.h>

#include "common.cuh"
#include "umma.cuh"

namespace skb {

constexpr int kUmBM = 128;       // MMA M (rows of A per tile)
constexpr int kUmBN = 64;        // MMA N (lanes per tile)
#ifndef SKB_UM_SUB
#define SKB_UM_SUB 2
#endif
constexpr int kUmSub = SKB_UM_SUB;   // 32-wide sub-blocks (one 128-byte swizzle row) per chunk
constexpr int kUmBK = 32 * kUmSub;   // reduction indices per chunk
#ifndef SKB_UM_ASM
#define SKB_UM_ASM (8 / SKB_UM_SUB)
#endif
#ifndef SKB_UM_BSM
#define SKB_UM_BSM (6 / SKB_UM_SUB)
#endif
#ifndef SKB_UM_ATM
#define SKB_UM_ATM (4 / SKB_UM_SUB)
#endif
#ifndef SKB_UM_SLOTS
#define SKB_UM_SLOTS 2
#endif
#ifndef SKB_UM_PROMO
#define SKB_UM_PROMO 1
#endif
constexpr int kUmAStagesSm = SKB_UM_ASM;   // shared-memory A tile ring
constexpr int kUmBStagesSm = SKB_UM_BSM;   // shared-memory B hi/lo ring
constexpr int kUmAStages = SKB_UM_ATM;     // TMEM A stages (hi | lo, 2 * kUmBK columns each)
constexpr int kUmSlots = SKB_UM_SLOTS;     // TMEM accumulator slot sets
constexpr int kUmPromo = SKB_UM_PROMO;     // chunks accumulated in TMEM per promotion
constexpr int kUmSlotCols = 2 * kUmBN;     // [hi*hi + lo*hi | hi*lo]
constexpr int kUmACols = 2 * kUmBK;
static_assert(kUmSlots * kUmSlotCols + kUmAStages * kUmACols <= 512, "TMEM budget");
constexpr int kUmThreads = 384;
constexpr uint32_t kUmTmemCols = 512;
constexpr uint32_t kUmABase = kUmSlots * kUmSlotCols;   // A stages after the accumulators
constexpr int kUmASubBytes = kUmBM * 32 * 4;            // 16 KB: one [128][32] box
constexpr int kUmBSubBytes = kUmBN * 32 * 4;            // 8 KB: one [64][32] box (one plane)
constexpr int kUmATileBytes = kUmSub * kUmASubBytes;
constexpr int kUmBStageBytes = kUmSub * 2 * kUmBSubBytes;   // per sub-block: hi rows, then lo rows
constexpr int kUmSmemBytes = kUmAStagesSm * kUmATileBytes + kUmBStagesSm * kUmBStageBytes + 1024;

struct UmmaParams {
  int M, N, K;          // D is M x N, reduction length K
  int MT, NT, KCH;      // tiles along M / N, chunks along K
  long long units;      // MT * NT * KCH
  int G;                // CTAs
  float* out;           // out[n * ldo + m]
  long long ldo;
  float* part;          // [G][2][kUmBN][kUmBM] split-tile partials
  const int* status;    // skip the work when an earlier kernel failed (nullable)
  float kc_scale;       // kKC: A is K o C, C recovered from K = 2^(-C log2e / lambda) as
                        // -log2(K) * kc_scale (kc_scale = lambda ln 2)
};

// First unit of CTA c's stream-K range (U units over G CTAs; U * G < 2^62).
__device__ __forceinline__ long long um_start(long long U, int G, int c) {
  return U * c / G;
}

// Tiles are numbered nt-major (tile = nt * MT + mt): the CTAs a quarter (for
// NT = 4) of the grid apart work on the same rows of A with different lane
// tiles at about the same time, so A streams from HBM once and the other N
// tiles' reads hit L2 (mt-major, one CTA walked the N tiles of an A block in
// turn and re-streamed it from HBM for each).
__device__ __forceinline__ int um_tile_mt(const UmmaParams& p, long long tile) {
  return (int)(tile % p.MT);
}
__device__ __forceinline__ int um_tile_nt(const UmmaParams& p, long long tile) {
  return (int)(tile / p.MT);
}

// The CTA whose unit range holds unit u.
__device__ __forceinline__ int um_owner(long long U, int G, long long u) {
  int c = (int)(u * G / U);
  while (c + 1 < G && um_start(U, G, c + 1) <= u) ++c;
  while (c > 0 && um_start(U, G, c) > u) --c;
  return c;
}

// kKC (the E0 contraction): the splitters turn each K element into
// K * C = -K log2(K) * kc_scale before the hi / lo split, so K o C needs no
// stored copy (17 GB at config 5).
template <bool kKC = false>
__global__ void __launch_bounds__(kUmThreads, 1)
    umma_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmBh,
                     const __grid_constant__ CUtensorMap tmBl, const UmmaParams p) {
  extern __shared__ uint8_t um_smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(um_smem_raw) + 1023) &
                                           ~uintptr_t(1023));
  __shared__ uint64_t afull_sm[kUmAStagesSm], afree_sm[kUmAStagesSm];
  __shared__ uint64_t bfull_sm[kUmBStagesSm], bfree_sm[kUmBStagesSm];
  __shared__ uint64_t afull[kUmAStages], aempty[kUmAStages];
  __shared__ uint64_t cfull[kUmSlots], cempty[kUmSlots];
  __shared__ uint32_t tmem_base_sh;
  uint8_t* smA = sm;
  uint8_t* smB = sm + kUmAStagesSm * kUmATileBytes;

  const int warp = warp_id(), lane = lane_id();
  if (threadIdx.x == 0) {
    for (int s = 0; s < kUmAStagesSm; ++s) {
      mbar_init(&afull_sm[s], 1);
      mbar_init(&afree_sm[s], 4);    // the 4 splitter warps
    }
    for (int s = 0; s < kUmBStagesSm; ++s) {
      mbar_init(&bfull_sm[s], 1);
      mbar_init(&bfree_sm[s], 1);    // the MMA commit
    }
    for (int a = 0; a < kUmAStages; ++a) {
      mbar_init(&afull[a], 4);
      mbar_init(&aempty[a], 1);
    }
    for (int r = 0; r < kUmSlots; ++r) {
      mbar_init(&cfull[r], 1);
      mbar_init(&cempty[r], 4);
    }
    fence_barrier_init();
  }
  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmBh);
    prefetch_tmap(&tmBl);
  }
  if (warp == 2) tmem_alloc<kUmTmemCols>(&tmem_base_sh);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tmem_base_sh;

  pdl_wait();
#ifdef SKB_UM_DBG_CLOCK
  const long long dbg_t0 = clock64();
#endif
  const bool skip = p.status != nullptr && *p.status != 0;
  const long long u0 = um_start(p.units, p.G, blockIdx.x);
  const long long u1 = um_start(p.units, p.G, blockIdx.x + 1);

  if (!skip && warp == 0) {
    // ---------------- TMA producer, A ring (the streamed kernel matrix) ----------------
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_first();
      int s = 0;
      uint32_t ph = 0;
      for (long long u = u0; u < u1; ++u) {
        const long long tile = u / p.KCH;
        const int kc = (int)(u % p.KCH);
        const int mt = um_tile_mt(p, tile);
        mbar_wait(&afree_sm[s], ph ^ 1);
        mbar_arrive_expect_tx(&afull_sm[s], kUmATileBytes);
        const int arow = (int)(((long long)mt * p.KCH + kc) * kUmSub * kUmBM);
#pragma unroll
        for (int sb = 0; sb < kUmSub; ++sb)
          tma_load_2d_hint(smA + (size_t)s * kUmATileBytes + sb * kUmASubBytes, &tmA, 0,
                           arow + sb * kUmBM, &afull_sm[s], pol);
        if (++s == kUmAStagesSm) { s = 0; ph ^= 1; }
      }
    }
  } else if (!skip && warp == 3) {
    // ---------------- TMA producer, B ring (the lanes' tf32 planes) ----------------
    if (lane == 0) {
      const uint64_t pol = l2_policy_evict_last();
      int s = 0;
      uint32_t ph = 0;
      for (long long u = u0; u < u1; ++u) {
        const long long tile = u / p.KCH;
        const int kc = (int)(u % p.KCH);
        const int nt = um_tile_nt(p, tile);
        mbar_wait(&bfree_sm[s], ph ^ 1);
        uint8_t* st = smB + (size_t)s * kUmBStageBytes;
        mbar_arrive_expect_tx(&bfull_sm[s], kUmBStageBytes);
        const int brow = (int)(((long long)nt * p.KCH + kc) * kUmSub * kUmBN);
#pragma unroll
        for (int sb = 0; sb < kUmSub; ++sb) {
          tma_load_2d_hint(st + sb * 2 * kUmBSubBytes, &tmBh, 0, brow + sb * kUmBN, &bfull_sm[s], pol);
          tma_load_2d_hint(st + sb * 2 * kUmBSubBytes + kUmBSubBytes, &tmBl, 0, brow + sb * kUmBN,
                           &bfull_sm[s], pol);
        }
        if (++s == kUmBStagesSm) { s = 0; ph ^= 1; }
      }
    }
  } else if (!skip && warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_tf32(kUmBM, kUmBN);
      const uint32_t idesc2 = umma_idesc_tf32(kUmBM, 2 * kUmBN);
      int s = 0, a = 0, r = 0;
      uint32_t ph = 0, aph = 0, rph = 0;
      long long span0 = u0;   // first chunk of the current promotion span
      for (long long u = u0; u < u1; ++u) {
        const long long piece0 = u0 > (u / p.KCH) * p.KCH ? u0 : (u / p.KCH) * p.KCH;
        const bool first = (u - piece0) % kUmPromo == 0;
        const bool last = (u - piece0) % kUmPromo == kUmPromo - 1 || u + 1 == u1 ||
                          (u + 1) % p.KCH == 0;
        if (first) {
          span0 = u;
          mbar_wait(&cempty[r], rph ^ 1);
        }
        mbar_wait(&bfull_sm[s], ph);
        mbar_wait(&afull[a], aph);
        tc_fence_after();
        const uint32_t bst = smem_u32(smB + (size_t)s * kUmBStageBytes);
        const uint32_t ahi = tbase + kUmABase + kUmACols * a, alo = ahi + kUmBK;
        // per k-step two MMAs: hi x [B hi ; B lo] as one N = 128 MMA (the two
        // planes are adjacent 64-row halves of the sub-block, one 1024-byte-
        // strided operand) into the slot set's columns [0, 128), then lo x B hi
        // (N = 64) accumulated onto the hi x B hi columns [0, 64).  An N = 64
        // MMA costs ~45 cycles, an N = 128 one 64 (tools/micro/umma_rate.cu).
        const uint32_t d = tbase + r * kUmSlotCols;
        const uint32_t acc = (u > span0) ? 1u : 0u;
#ifdef SKB_UM_DBG_NOMMA
        if (false)
#endif
#pragma unroll
        for (int k = 0; k < kUmBK / 8; ++k) {
          const uint32_t ak = k > 0 ? 1u : acc;
          const uint64_t bd = umma_sdesc_sw128(bst + (k / 4) * 2 * kUmBSubBytes + 32 * (k % 4));
          umma_tf32_ts(d, ahi + 8 * k, bd, idesc2, ak);
          umma_tf32_ts(d, alo + 8 * k, bd, idesc, 1);
        }
        umma_commit(&bfree_sm[s]);
        umma_commit(&aempty[a]);
        if (++s == kUmBStagesSm) { s = 0; ph ^= 1; }
        if (++a == kUmAStages) { a = 0; aph ^= 1; }
        if (last) {
          umma_commit(&cfull[r]);
          if (++r == kUmSlots) { r = 0; rph ^= 1; }
        }
      }
    }
  } else if (!skip && warp >= 4 && warp < 8) {
    // ---------------- splitters: A tile -> tf32 hi / lo in TMEM ----------------
    const int row = (warp - 4) * 32 + lane;          // TMEM lane = tile row
    const uint32_t lane_off = (uint32_t)((warp - 4) * 32) << 16;
    int s = 0, a = 0;
    uint32_t ph = 0, aph = 0;
    for (long long u = u0; u < u1; ++u) {
      mbar_wait(&afull_sm[s], ph);
      // split from shared memory first (overlaps the MMAs still reading the
      // TMEM stage), then wait for the stage and store both planes
      uint32_t hi[kUmBK], lo[kUmBK];
#pragma unroll
      for (int sb = 0; sb < kUmSub; ++sb) {
        const float4* rowp = reinterpret_cast<const float4*>(smA + (size_t)s * kUmATileBytes +
                                                             sb * kUmASubBytes + row * 128);
#if defined(SKB_UM_DBG_NOSPLIT) || defined(SKB_UM_DBG_NOLDS)
        if (false)
#endif
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float4 v = rowp[q ^ (row & 7)];
          float x[4] = {v.x, v.y, v.z, v.w};
          if constexpr (kKC) {
#pragma unroll
            for (int e = 0; e < 4; ++e) x[e] = x[e] > 0.f ? -x[e] * lg2(x[e]) * p.kc_scale : 0.f;
          }
#pragma unroll
          for (int e = 0; e < 4; e += 2) {   // lo = x - hi on packed pairs (FADD2)
            const int c = 32 * sb + 4 * q + e;
            const float h0 = tf32_hi(x[e]), h1 = tf32_hi(x[e + 1]);
            hi[c] = __float_as_uint(h0);
            hi[c + 1] = __float_as_uint(h1);
            const uint64_t d2 = fadd2(pk2(x[e], x[e + 1]), pk2(-h0, -h1));
            lo[c] = __float_as_uint(lo2(d2));
            lo[c + 1] = __float_as_uint(hi2(d2));
          }
        }
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&afree_sm[s])) : "memory");
      mbar_wait(&aempty[a], aph ^ 1);
      tc_fence_after();
      const uint32_t ahi = tbase + lane_off + kUmABase + kUmACols * a;
#ifndef SKB_UM_DBG_NOSPLIT
      static_assert(kUmBK == 64, "the splitter stores 64-column planes");
      tmem_st64(ahi, hi);
      tmem_st64(ahi + kUmBK, lo);
      tmem_st_wait();
#endif
      tc_fence_before();
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&afull[a])) : "memory");
      if (++s == kUmAStagesSm) { s = 0; ph ^= 1; }
      if (++a == kUmAStages) { a = 0; aph ^= 1; }
    }
  } else if (!skip && warp >= 8) {
    // ---------------- epilogue: promote every chunk into fp32 registers ----------------
    const int row = (warp - 8) * 32 + lane;
    const uint32_t lane_off = (uint32_t)((warp - 8) * 32) << 16;
    int r = 0;
    uint32_t rph = 0;
    const long long first_tile = u0 / p.KCH;
    long long u = u0;
    while (u < u1) {
      const long long tile = u / p.KCH;
      const int k0 = (int)(u % p.KCH);
      const int k1 = (int)(k0 + (u1 - u) < p.KCH ? k0 + (u1 - u) : p.KCH);
      uint64_t acc2[kUmBN / 2];   // packed pairs: FADD2 promotion
#pragma unroll
      for (int n = 0; n < kUmBN / 2; ++n) acc2[n] = 0ull;
      for (int kc = k0; kc < k1; kc += kUmPromo) {
        mbar_wait(&cfull[r], rph);
        tc_fence_after();
#ifdef SKB_UM_DBG_NOEPI
        if (false)
#endif
#pragma unroll
        for (int h = 0; h < kUmBN / 32; ++h) {
          uint32_t v0[32], v1[32];
          const uint32_t t = tbase + lane_off + r * kUmSlotCols + 32 * h;
          tmem_ld32(t, v0);            // hi*hi + lo*hi
          tmem_ld32(t + kUmBN, v1);    // hi*lo
          tmem_ld_wait();
#pragma unroll
          for (int n = 0; n < 16; ++n) {
            const uint64_t s0 = fadd2(pk2(__uint_as_float(v0[2 * n]), __uint_as_float(v0[2 * n + 1])),
                                      pk2(__uint_as_float(v1[2 * n]), __uint_as_float(v1[2 * n + 1])));
            fadd2_acc(acc2[16 * h + n], s0);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&cempty[r])) : "memory");
        if (++r == kUmSlots) { r = 0; rph ^= 1; }
      }
      float acc[kUmBN];
#pragma unroll
      for (int n = 0; n < kUmBN / 2; ++n) {
        acc[2 * n] = lo2(acc2[n]);
        acc[2 * n + 1] = hi2(acc2[n]);
      }
      const int nt = um_tile_nt(p, tile), mt = um_tile_mt(p, tile);
      const int m = mt * kUmBM + row;
      if (k0 == 0 && k1 == p.KCH) {
        if (m < p.M) {
          const int nmax = min(kUmBN, p.N - nt * kUmBN);
#pragma unroll
          for (int n = 0; n < kUmBN; ++n)
            if (n < nmax) p.out[(long long)(nt * kUmBN + n) * p.ldo + m] = acc[n];
        }
      } else {
        const int slot = tile == first_tile ? 0 : 1;
        float* dst = p.part + ((size_t)(blockIdx.x * 2 + slot) * kUmBN) * kUmBM + row;
#pragma unroll
        for (int n = 0; n < kUmBN; ++n) dst[(size_t)n * kUmBM] = acc[n];
      }
      u += k1 - k0;
    }
  }
  tc_fence_before();
  __syncthreads();
#ifdef SKB_UM_DBG_CLOCK
  if (threadIdx.x == 0) {
    extern __device__ unsigned long long g_um_dbg_cycles[2];
    atomicAdd(&g_um_dbg_cycles[0], (unsigned long long)(clock64() - dbg_t0));
    atomicAdd(&g_um_dbg_cycles[1], (unsigned long long)(u1 - u0));
  }
#endif
  pdl_launch_dependents();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<kUmTmemCols>(tbase);
  }
}

// Split tiles: sum the pieces in ascending CTA order into out.  grid = G
// blocks, block 256: block c owns the tile holding its range's first unit when
// that tile is split there and no earlier boundary falls inside it.  The
// contributing (CTA, slot) pieces are listed once per block in shared memory.
constexpr int kUmFixMax = 256;
__global__ void __launch_bounds__(256) umma_fixup_kernel(const UmmaParams p) {
  pdl_wait();
  if (p.status != nullptr && *p.status != 0) return;
  __shared__ int s_n;
  __shared__ int s_piece[kUmFixMax];   // part row offset (cta * 2 + slot)
  const int c = blockIdx.x;
  const long long uc = um_start(p.units, p.G, c);
  const long long t = uc / p.KCH;
  if (threadIdx.x == 0) {
    s_n = 0;
    bool mine = c > 0 && uc < p.units && uc % p.KCH != 0 && um_start(p.units, p.G, c + 1) > uc;
    for (int e = c - 1; mine && e >= 1; --e) {   // an earlier boundary inside t owns it
      const long long ue = um_start(p.units, p.G, e);
      if (ue / p.KCH != t) break;
      if (ue % p.KCH != 0 && um_start(p.units, p.G, e + 1) > ue) mine = false;
    }
    if (mine) {
      const int c0 = um_owner(p.units, p.G, t * p.KCH);
      const int c1 = um_owner(p.units, p.G, (t + 1) * p.KCH - 1);
      int n = 0;
      for (int cc = c0; cc <= c1 && n < kUmFixMax; ++cc) {
        const long long u = um_start(p.units, p.G, cc);
        if (um_start(p.units, p.G, cc + 1) == u) continue;   // empty range
        s_piece[n++] = cc * 2 + ((u / p.KCH == t) ? 0 : 1);
      }
      s_n = n;
    }
  }
  __syncthreads();
  const int np = s_n;
  if (np == 0) return;
  const int nt = um_tile_nt(p, t), mt = um_tile_mt(p, t);
  const int nmax = min(kUmBN, p.N - nt * kUmBN);
  for (int e = threadIdx.x; e < kUmBM * kUmBN / 4; e += 256) {
    const int n = e / (kUmBM / 4), row = 4 * (e % (kUmBM / 4));
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int k = 0; k < np; ++k) {
      const float4 v = *reinterpret_cast<const float4*>(
          p.part + ((size_t)s_piece[k] * kUmBN + n) * kUmBM + row);
      s.x += v.x; s.y += v.y; s.z += v.z; s.w += v.w;
    }
    if (n < nmax) {
      const float vals[4] = {s.x, s.y, s.z, s.w};
      float* o = p.out + (long long)(nt * kUmBN + n) * p.ldo + mt * kUmBM + row;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (mt * kUmBM + row + q < p.M) o[q] = vals[q];
    }
  }
}

// Operand layout.  Every operand is stored tile-major,
// [tile][chunk][sub-block][row][32]: an R x 32 sub-block (R = 128 or 64) is one
// contiguous 16 / 8 KB run, so each TMA box is a single sequential read, and a
// CTA's stream-K range (consecutive chunks of consecutive tiles) is one
// contiguous stretch of HBM.  Element (r, k) of an operand with R-row tiles
// and kch chunks of kUmBK sits at
//   ((r / R) * kch + k / kUmBK) * R * kUmBK + ((k % kUmBK) / 32) * R * 32 + (r % R) * 32 + k % 32.
__host__ __device__ __forceinline__ long long um_tiled_index(long long r, long long k, int R,
                                                             long long kch) {
  return ((r / R) * kch + k / kUmBK) * R * kUmBK + ((k % kUmBK) / 32) * R * 32 + (r % R) * 32 +
         (k % 32);
}

// hi / lo tf32 planes of a lane-major [rows][cols] fp32 array in the tiled
// B-operand layout (64-row tiles, kch chunks; the padding reads as 0).
// grid-stride over the padded [NT*64][kch*32] index space.
__global__ void umma_split_kernel(const float* __restrict__ x, int rows, int cols, long long kch,
                                  float* __restrict__ hi, float* __restrict__ lo) {
  const int nt = (rows + kUmBN - 1) / kUmBN;
  const long long n = (long long)nt * kUmBN * kch * kUmBK;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    // e enumerates the tiled array itself (coalesced stores)
    const long long blk = e / (kUmBN * kUmBK);        // (tile, chunk)
    const int within = (int)(e % (kUmBN * kUmBK));
    const int sb = within / (kUmBN * 32), w2 = within % (kUmBN * 32);
    const int r = (int)((blk / kch) * kUmBN + w2 / 32);
    const long long k = (blk % kch) * kUmBK + sb * 32 + w2 % 32;
    const float v = (r < rows && k < cols) ? x[(long long)r * cols + k] : 0.f;
    const float h = tf32_hi(v);
    hi[e] = h;
    lo[e] = v - h;
  }
}

// ---- point-cloud costs: c_ij = |x_i|^2 + |y_j|^2 - 2 x_i . y_j ---------------------
// x: [d1][D], y: [d2][D] packed as one [(d1 + d2)][D]
// fp32 array.  The dot products run on the tensor cores (umma_gemm_kernel with
// A = y in the tiled layout, B = x's tf32 planes); these kernels prepare the
// operands, the norms, and finish the cost.

// Squared norms, accumulated in double (a non-finite point gives a non-finite norm).
__global__ void points_norms_kernel(const float* __restrict__ pts, int n, int D,
                                    float* __restrict__ norms) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < D; ++k) {
      const float v = pts[(size_t)r * D + k];
      s += (double)v * v;
    }
    norms[r] = (float)s;
  }
}

// y -> the tiled A-operand layout (128-row tiles, kch chunks of kUmBK, zero padding).
__global__ void points_tile_a_kernel(const float* __restrict__ y, int rows, int D, long long kch,
                                     float* __restrict__ out) {
  const long long mt = (rows + kUmBM - 1) / kUmBM;
  const long long n = mt * kUmBM * kch * kUmBK;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const long long blk = e / (kUmBM * kUmBK);
    const int within = (int)(e % (kUmBM * kUmBK));
    const int sb = within / (kUmBM * 32), w2 = within % (kUmBM * 32);
    const long long r = (blk / kch) * kUmBM + w2 / 32;
    const long long k = (blk % kch) * kUmBK + sb * 32 + w2 % 32;
    out[e] = (r < rows && k < D) ? y[r * D + k] : 0.f;
  }
}

// c_ij = max(0, |x_i|^2 + |y_j|^2 - 2 dot_ij), in place over the [d1][d2] dot products.
__global__ void points_cost_kernel(float* __restrict__ c, const float* __restrict__ nx,
                                   const float* __restrict__ ny, int d1, int d2) {
  const long long n = (long long)d1 * d2;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / d2), j = (int)(e - (long long)i * d2);
    const float v = fmaf(-2.f, c[e], nx[i] + ny[j]);
    c[e] = v < 0.f ? 0.f : v;   // rounding below 0 clamps; NaN (non-finite points) stays
  }
}

// ---- dC = sum_b up_b P_b for a shared cost, as a tensor-core contraction -------
// P_bij = 2^(u_bi + A2_ij + v_bj) (log2 units) = 2^(A2_ij + al_i + be_j) *
// U_bi V_bj with al_i = max_b u_bi, be_j = max_b v_bj, U_bi = up_b 2^(u_bi - al_i),
// V_bj = 2^(v_bj - be_j) <= 1: S = U^T V is a (d1 x B)(B x d2) contraction over
// the lanes (core.py:363-368 per lane, the one dense
// contraction of the path).  A operand: V over (d2 rows, B reduction); B
// operand: U's tf32 planes over (d1 rows, B reduction); out[i * d2 + j].

// al / be: the per-row maxima over the lanes (natural-log input -> log2);
// -inf everywhere (zero mass in every lane) -> 0, its terms are all 0.
__global__ void plan_lane_max_kernel(const float* __restrict__ lx, int B, int d,
                                     float* __restrict__ mx) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d; i += gridDim.x * blockDim.x) {
    float m = neg_inf();
    for (int b = 0; b < B; ++b) m = fmaxf(m, lx[(size_t)b * d + i] * kLog2e);
    mx[i] = m == neg_inf() ? 0.f : m;
  }
}

// V -> the tiled A-operand layout (rows j, reduction b); U -> tf32 planes of
// the lane operand (rows i, reduction b).  Grid-stride over the tiled index
// space of each (zero padding).
__global__ void plan_operands_kernel(const float* __restrict__ log_u, const float* __restrict__ log_v,
                                     const float* __restrict__ up, const float* __restrict__ al,
                                     const float* __restrict__ be, int B, int d1, int d2,
                                     long long kch, float* __restrict__ va,
                                     float* __restrict__ uh, float* __restrict__ ul) {
  const long long nva = (long long)((d2 + kUmBM - 1) / kUmBM) * kUmBM * kch * kUmBK;
  const long long nu = (long long)((d1 + kUmBN - 1) / kUmBN) * kUmBN * kch * kUmBK;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nva + nu;
       e += (long long)gridDim.x * blockDim.x) {
    const bool isv = e < nva;
    const long long f = isv ? e : e - nva;
    const int R = isv ? kUmBM : kUmBN;
    const long long blk = f / (R * kUmBK);
    const int within = (int)(f % (R * kUmBK));
    const int sb = within / (R * 32), w2 = within % (R * 32);
    const long long r = (blk / kch) * R + w2 / 32;          // j (V) or i (U)
    const int b = (int)((blk % kch) * kUmBK + sb * 32 + w2 % 32);
    if (isv) {
      float v = 0.f;
      if (r < d2 && b < B) v = exp2f(log_v[(size_t)b * d2 + r] * kLog2e - be[r]);
      va[f] = v;
    } else {
      float x = 0.f;
      if (r < d1 && b < B) x = up[b] * exp2f(log_u[(size_t)b * d1 + r] * kLog2e - al[r]);
      const float h = tf32_hi(x);
      uh[f] = h;
      ul[f] = x - h;
    }
  }
}

// dC_ij = S_ij * 2^(c_ij * kscale + al_i + be_j), in place over S (row-major [d1][d2]).
__global__ void plan_finish_kernel(float* __restrict__ dc, const float* __restrict__ c,
                                   const float* __restrict__ al, const float* __restrict__ be,
                                   int d1, int d2, float kscale) {
  const long long n = (long long)d1 * d2;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(e / d2), j = (int)(e - (long long)i * d2);
    const float s = dc[e];
    dc[e] = s == 0.f ? 0.f : s * exp2f(fmaf(c[e], kscale, al[i] + be[j]));
  }
}

// K = 2^(c * kscale) and K o C (E0) as tiled A operands over (d1 rows, d2
// reduction), and K^T over (d2 rows, d1 reduction), from the caller's cost
// (validated: finite, >= 0, status 15).  One block per 32 x 32 cost block
// through shared memory: in the tiled layout a 32 x 32 block is one
// contiguous 4 KB run for both orientations.  The padded extents are
// covered too (zeros).  grid (ceil(D2p/32), ceil(D1p/32)) with D1p, D2p the
// extents rounded up to 128; block 256.
__global__ void __launch_bounds__(256) umma_kernel_matrices(const float* __restrict__ c, int d1,
                                                            int d2, float kscale,
                                                            float* __restrict__ K,
                                                            float* __restrict__ KT, int* status) {
  __shared__ float tile[32][33];
  const int j0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
  const long long kch1 = (d1 + kUmBK - 1) / kUmBK, kch2 = (d2 + kUmBK - 1) / kUmBK;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const bool in_k = i0 < ((d1 + kUmBM - 1) / kUmBM) * kUmBM && j0 < kch2 * kUmBK;    // K rows
  const bool in_kt = j0 < ((d2 + kUmBM - 1) / kUmBM) * kUmBM && i0 < kch1 * kUmBK;   // K^T rows
  bool bad = false;
  for (int r = ty; r < 32; r += 8) {
    const int i = i0 + r, j = j0 + tx;
    float k = 0.f;
    if (i < d1 && j < d2) {
      const float cv = c[(size_t)i * d2 + j];
      if (!(cv >= 0.f) || isinf(cv)) bad = true;
      k = ex2(cv * kscale);
    }
    if (in_k) K[um_tiled_index(i, j, kUmBM, kch2)] = k;
    tile[r][tx] = k;
  }
  __syncthreads();
  if (in_kt)
    for (int r = ty; r < 32; r += 8) KT[um_tiled_index(j0 + r, i0 + tx, kUmBM, kch1)] = tile[tx][r];
  if (__any_sync(0xffffffffu, bad) && lane_id() == 0) set_status(status, 15);
}

// The same on 32 x 128 strips with float4 loads and stores (d2 % 4 == 0 and a
// 16-byte aligned cost): HBM-bound, 4 B read and 8 B written per element
// (K, K^T).  grid (ldk2 / 128, ldk1 / 32); block 256 = 8 warps.
__global__ void __launch_bounds__(256) umma_kernel_matrices_vec4(
    const float* __restrict__ c, int d1, int d2, float kscale, float* __restrict__ K,
    float* __restrict__ KT, int* status) {
  __shared__ float tile[32][128 + 4];
  const int j0 = blockIdx.x * 128, i0 = blockIdx.y * 32;
  const long long kch1 = (d1 + kUmBK - 1) / kUmBK, kch2 = (d2 + kUmBK - 1) / kUmBK;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int mrows1 = ((d1 + kUmBM - 1) / kUmBM) * kUmBM;   // K / KC rows in the tiled layout
  const int j = j0 + 4 * tx;
  bool bad = false;
  for (int r = ty; r < 32; r += 8) {
    const int i = i0 + r;
    float4 k4 = make_float4(0.f, 0.f, 0.f, 0.f);
    if (i < d1 && j < d2) {   // d2 % 4 == 0: the four columns are all inside
      const float4 cv = __ldcs(reinterpret_cast<const float4*>(c + (size_t)i * d2 + j));
      const float cc[4] = {cv.x, cv.y, cv.z, cv.w};
      float kk[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (!(cc[e] >= 0.f) || isinf(cc[e])) bad = true;
        kk[e] = ex2(cc[e] * kscale);
      }
      k4 = make_float4(kk[0], kk[1], kk[2], kk[3]);
    }
    if (i < mrows1 && j < kch2 * kUmBK)   // 4 consecutive floats of the tiled layout
      *reinterpret_cast<float4*>(K + um_tiled_index(i, j, kUmBM, kch2)) = k4;
    *reinterpret_cast<float4*>(&tile[r][4 * tx]) = k4;
  }
  __syncthreads();
  if (i0 < kch1 * kUmBK) {
    const int i = i0 + tx;
    for (int rr = ty; rr < 128; rr += 8)   // K^T rows j0 + rr, 32 contiguous i each
      KT[um_tiled_index(j0 + rr, i, kUmBM, kch1)] = tile[tx][rr];
  }
  if (__any_sync(0xffffffffu, bad) && lane_id() == 0) set_status(status, 15);
}

}  // namespace skb
