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
//   warp 0      TMA producer: A tile [128][32] + B hi/lo tiles [64][32], SW128
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
constexpr int kUmBK = 32;        // reduction indices per chunk (one 128-byte swizzle row)
constexpr int kUmStages = 4;     // shared-memory stages
constexpr int kUmAStages = 3;    // TMEM A stages (hi + lo, 64 columns each)
constexpr int kUmSlots = 4;      // TMEM accumulator slots (64 columns each)
constexpr int kUmThreads = 384;
constexpr uint32_t kUmTmemCols = 512;
constexpr uint32_t kUmABase = kUmSlots * kUmBN;   // A stages after the accumulator slots
constexpr int kUmATileBytes = kUmBM * kUmBK * 4;  // 16 KB
constexpr int kUmBTileBytes = kUmBN * kUmBK * 4;  // 8 KB
constexpr int kUmStageBytes = kUmATileBytes + 2 * kUmBTileBytes;
constexpr int kUmSmemBytes = kUmStages * kUmStageBytes + 1024;

struct UmmaParams {
  int M, N, K;          // D is M x N, reduction length K
  int MT, NT, KCH;      // tiles along M / N, chunks along K
  long long units;      // MT * NT * KCH
  int G;                // CTAs
  float* out;           // out[n * ldo + m]
  long long ldo;
  float* part;          // [G][2][kUmBN][kUmBM] split-tile partials
  const int* status;    // skip the work when an earlier kernel failed (nullable)
};

__device__ __forceinline__ long long um_start(long long U, int G, int c) {
  return (long long)((__int128)U * c / G);
}

// The CTA whose unit range holds unit u.
__device__ __forceinline__ int um_owner(long long U, int G, long long u) {
  int c = (int)((__int128)u * G / U);
  while (c + 1 < G && um_start(U, G, c + 1) <= u) ++c;
  while (c > 0 && um_start(U, G, c) > u) --c;
  return c;
}

__global__ void __launch_bounds__(kUmThreads, 1)
    umma_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmBh,
                     const __grid_constant__ CUtensorMap tmBl, const UmmaParams p) {
  extern __shared__ uint8_t um_smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(um_smem_raw) + 1023) &
                                           ~uintptr_t(1023));
  __shared__ uint64_t full[kUmStages], kfree[kUmStages];
  __shared__ uint64_t afull[kUmAStages], aempty[kUmAStages];
  __shared__ uint64_t cfull[kUmSlots], cempty[kUmSlots];
  __shared__ uint32_t tmem_base_sh;

  const int warp = warp_id(), lane = lane_id();
  if (threadIdx.x == 0) {
    for (int s = 0; s < kUmStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&kfree[s], 4 + 1);   // 4 splitter warps (A) + the MMA commit (B)
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
  const bool skip = p.status != nullptr && *p.status != 0;
  const long long u0 = um_start(p.units, p.G, blockIdx.x);
  const long long u1 = um_start(p.units, p.G, blockIdx.x + 1);

  if (!skip && warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (long long u = u0; u < u1; ++u) {
        const long long tile = u / p.KCH;
        const int kc = (int)(u % p.KCH);
        const int nt = (int)(tile % p.NT), mt = (int)(tile / p.NT);
        mbar_wait(&kfree[s], ph ^ 1);
        uint8_t* st = sm + (size_t)s * kUmStageBytes;
        mbar_arrive_expect_tx(&full[s], kUmStageBytes);
        tma_load_2d(st, &tmA, kc * kUmBK, mt * kUmBM, &full[s]);
        tma_load_2d(st + kUmATileBytes, &tmBh, kc * kUmBK, nt * kUmBN, &full[s]);
        tma_load_2d(st + kUmATileBytes + kUmBTileBytes, &tmBl, kc * kUmBK, nt * kUmBN, &full[s]);
        if (++s == kUmStages) { s = 0; ph ^= 1; }
      }
    }
  } else if (!skip && warp == 1) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      const uint32_t idesc = umma_idesc_tf32(kUmBM, kUmBN);
      int s = 0, a = 0, r = 0;
      uint32_t ph = 0, aph = 0, rph = 0;
      for (long long u = u0; u < u1; ++u) {
        mbar_wait(&cempty[r], rph ^ 1);
        mbar_wait(&full[s], ph);
        mbar_wait(&afull[a], aph);
        tc_fence_after();
        const uint32_t sb = smem_u32(sm + (size_t)s * kUmStageBytes);
        const uint32_t bh = sb + kUmATileBytes, bl = bh + kUmBTileBytes;
        const uint32_t ahi = tbase + kUmABase + 64 * a, alo = ahi + 32;
        const uint32_t d = tbase + r * kUmBN;
#pragma unroll
        for (int k = 0; k < kUmBK / 8; ++k) {
          umma_tf32_ts(d, ahi + 8 * k, umma_sdesc_sw128(bh + 32 * k), idesc, k > 0);
          umma_tf32_ts(d, ahi + 8 * k, umma_sdesc_sw128(bl + 32 * k), idesc, 1);
          umma_tf32_ts(d, alo + 8 * k, umma_sdesc_sw128(bh + 32 * k), idesc, 1);
        }
        umma_commit(&kfree[s]);
        umma_commit(&aempty[a]);
        umma_commit(&cfull[r]);
        if (++s == kUmStages) { s = 0; ph ^= 1; }
        if (++a == kUmAStages) { a = 0; aph ^= 1; }
        if (++r == kUmSlots) { r = 0; rph ^= 1; }
      }
    }
  } else if (!skip && warp >= 4 && warp < 8) {
    // ---------------- splitters: A tile -> tf32 hi / lo in TMEM ----------------
    const int row = (warp - 4) * 32 + lane;          // TMEM lane = tile row
    const uint32_t lane_off = (uint32_t)((warp - 4) * 32) << 16;
    int s = 0, a = 0;
    uint32_t ph = 0, aph = 0;
    for (long long u = u0; u < u1; ++u) {
      mbar_wait(&full[s], ph);
      const float4* rowp =
          reinterpret_cast<const float4*>(sm + (size_t)s * kUmStageBytes + row * 128);
      uint32_t hi[32], lo[32];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 v = rowp[q ^ (row & 7)];
        const float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float h = tf32_hi(x[e]);
          hi[4 * q + e] = __float_as_uint(h);
          lo[4 * q + e] = __float_as_uint(x[e] - h);
        }
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&kfree[s])) : "memory");
      mbar_wait(&aempty[a], aph ^ 1);
      tc_fence_after();
      const uint32_t ahi = tbase + lane_off + kUmABase + 64 * a;
      tmem_st32(ahi, hi);
      tmem_st32(ahi + 32, lo);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&afull[a])) : "memory");
      if (++s == kUmStages) { s = 0; ph ^= 1; }
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
      float acc[kUmBN];
#pragma unroll
      for (int n = 0; n < kUmBN; ++n) acc[n] = 0.f;
      for (int kc = k0; kc < k1; ++kc) {
        mbar_wait(&cfull[r], rph);
        tc_fence_after();
#pragma unroll
        for (int h = 0; h < kUmBN / 32; ++h) {
          uint32_t v[32];
          tmem_ld32(tbase + lane_off + r * kUmBN + 32 * h, v);
          tmem_ld_wait();
#pragma unroll
          for (int n = 0; n < 32; ++n) acc[32 * h + n] += __uint_as_float(v[n]);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&cempty[r])) : "memory");
        if (++r == kUmSlots) { r = 0; rph ^= 1; }
      }
      const int nt = (int)(tile % p.NT), mt = (int)(tile / p.NT);
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
  pdl_launch_dependents();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<kUmTmemCols>(tbase);
  }
}

// Split tiles: sum the pieces in ascending CTA order into out.  grid = tiles,
// block 256; unsplit tiles return at once.
__global__ void __launch_bounds__(256) umma_fixup_kernel(const UmmaParams p) {
  pdl_wait();
  if (p.status != nullptr && *p.status != 0) return;
  const long long t = blockIdx.x;
  const long long uf = t * p.KCH, ul = uf + p.KCH - 1;
  const int c0 = um_owner(p.units, p.G, uf), c1 = um_owner(p.units, p.G, ul);
  if (c0 == c1) return;
  const int nt = (int)(t % p.NT), mt = (int)(t / p.NT);
  const int nmax = min(kUmBN, p.N - nt * kUmBN);
  for (int e = threadIdx.x; e < kUmBM * kUmBN; e += 256) {
    const int n = e / kUmBM, row = e % kUmBM;
    const int m = mt * kUmBM + row;
    float s = 0.f;
    for (int c = c0; c <= c1; ++c) {
      const long long uc = um_start(p.units, p.G, c);
      if (um_start(p.units, p.G, c + 1) == uc) continue;   // empty range
      const int slot = (uc / p.KCH == t) ? 0 : 1;
      s += p.part[((size_t)(c * 2 + slot) * kUmBN + n) * kUmBM + row];
    }
    if (n < nmax && m < p.M) p.out[(long long)(nt * kUmBN + n) * p.ldo + m] = s;
  }
}

// hi / lo tf32 planes [rows][ld] of a lane-major [rows][cols] fp32 array (ld >=
// cols; the padding columns are written as 0).
__global__ void umma_split_kernel(const float* __restrict__ x, long long rows, int cols, int ld,
                                  float* __restrict__ hi, float* __restrict__ lo) {
  const long long n = rows * ld;
  for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n;
       k += (long long)gridDim.x * blockDim.x) {
    const long long b = k / ld;
    const int j = (int)(k - b * ld);
    const float v = j < cols ? x[b * cols + j] : 0.f;
    const float h = tf32_hi(v);
    hi[k] = h;
    lo[k] = v - h;
  }
}

// K = 2^(c * kscale), K o C (E0) row-major [d1][ldk2] and K^T [d2][ldk1] from
// the caller's cost (validated: finite, >= 0, status 15), 32 x 32 tiles
// through shared memory so both the row-major and the transposed stores are
// coalesced.  grid (ceil(d2/32), ceil(d1/32)), block 256.
__global__ void __launch_bounds__(256) umma_kernel_matrices(const float* __restrict__ c, int d1,
                                                            int d2, int ldk1, int ldk2, float kscale,
                                                            float* __restrict__ K, float* __restrict__ KC,
                                                            float* __restrict__ KT, int* status) {
  __shared__ float tile[32][33];
  const int j0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  bool bad = false;
  for (int r = ty; r < 32; r += 8) {
    const int i = i0 + r, j = j0 + tx;
    float k = 0.f;
    if (i < d1 && j < d2) {
      const float cv = c[(size_t)i * d2 + j];
      if (!(cv >= 0.f) || isinf(cv)) bad = true;
      k = ex2(cv * kscale);
      K[(size_t)i * ldk2 + j] = k;
      KC[(size_t)i * ldk2 + j] = k * cv;
    } else if (i < d1 && j < ldk2) {
      K[(size_t)i * ldk2 + j] = 0.f;
      KC[(size_t)i * ldk2 + j] = 0.f;
    }
    tile[r][tx] = k;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int j = j0 + r, i = i0 + tx;
    if (j < d2 && i < ldk1) KT[(size_t)j * ldk1 + i] = i < d1 ? tile[tx][r] : 0.f;
  }
  if (__any_sync(0xffffffffu, bad) && lane_id() == 0) set_status(status, 15);
}

}  // namespace skb
