// Probe of the tcgen05 pieces the 3xTF32 contraction kernels rely on:
// TMA SWIZZLE_128B tiles as K-major UMMA operands, kind::tf32 MMAs in SS and
// TS (A in TMEM) form, tcgen05.st / tcgen05.ld layouts, and how the tensor
// core reduces fp32 operand bits to tf32 (truncation or rounding).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_1907_01729_b200/csrc \
//        -o umma_probe umma_probe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "umma.cuh"

using namespace skb;

constexpr int M = 128, N = 64, KC = 32;

__global__ void __launch_bounds__(128) probe(const __grid_constant__ CUtensorMap tmA,
                                             const __grid_constant__ CUtensorMap tmB,
                                             const float* __restrict__ Ag, float* D1, float* D2,
                                             float* D3, int reps) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  float* sA = reinterpret_cast<float*>(sm);                  // 16 KB
  float* sB = reinterpret_cast<float*>(sm + 16384);          // 8 KB
  float* sBh = reinterpret_cast<float*>(sm + 16384 + 8192);  // 8 KB
  float* sBl = reinterpret_cast<float*>(sm + 16384 + 16384); // 8 KB
  __shared__ uint64_t bar[4];
  __shared__ uint32_t tbase;
  const int w = warp_id(), t = threadIdx.x;
  if (t == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  if (w == 1) tmem_alloc<512>(&tbase);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tbase;
  if (t == 0) {
    mbar_arrive_expect_tx(&bar[0], (M + N) * KC * 4);
    tma_load_2d(sA, &tmA, 0, 0, &bar[0]);
    tma_load_2d(sB, &tmB, 0, 0, &bar[0]);
  }
  mbar_wait(&bar[0], 0);
  const uint32_t idesc = umma_idesc_tf32(M, N);
  // --- SS
  if (t == 0) {
    tc_fence_after();
    for (int k = 0; k < KC / 8; ++k)
      umma_tf32_ss(tb + 0, umma_sdesc_sw128(smem_u32(sA) + 32 * k),
                   umma_sdesc_sw128(smem_u32(sB) + 32 * k), idesc, k > 0);
    umma_commit(&bar[1]);
  }
  // --- TS: A rows from global into TMEM columns 64.., hi at 192.., lo at 224..
  {
    uint32_t r[32], h[32], l[32];
    for (int k = 0; k < 32; ++k) {
      const float x = Ag[t * KC + k];
      r[k] = __float_as_uint(x);
      h[k] = __float_as_uint(tf32_hi(x));
      l[k] = __float_as_uint(x - tf32_hi(x));
    }
    const uint32_t lane = (uint32_t)(32 * w) << 16;
    tmem_st32(tb + lane + 64, r);
    tmem_st32(tb + lane + 192, h);
    tmem_st32(tb + lane + 224, l);
    tmem_st_wait();
    // B split in smem (elementwise: the swizzled layout is preserved)
    for (int i = t; i < N * KC; i += 128) {
      const float x = sB[i];
      sBh[i] = tf32_hi(x);
      sBl[i] = x - tf32_hi(x);
    }
    fence_proxy_async();
  }
  tc_fence_before();
  __syncthreads();
  if (t == 0) {
    tc_fence_after();
    for (int k = 0; k < KC / 8; ++k)
      umma_tf32_ts(tb + 128, tb + 64 + 8 * k, umma_sdesc_sw128(smem_u32(sB) + 32 * k), idesc,
                   k > 0);
    umma_commit(&bar[2]);
    for (int rep = 0; rep < reps; ++rep)
    for (int k = 0; k < KC / 8; ++k) {
      umma_tf32_ts(tb + 256, tb + 192 + 8 * k, umma_sdesc_sw128(smem_u32(sBh) + 32 * k), idesc,
                   (k | rep) > 0);
      umma_tf32_ts(tb + 256, tb + 192 + 8 * k, umma_sdesc_sw128(smem_u32(sBl) + 32 * k), idesc, 1);
      umma_tf32_ts(tb + 256, tb + 224 + 8 * k, umma_sdesc_sw128(smem_u32(sBh) + 32 * k), idesc, 1);
    }
    umma_commit(&bar[3]);
  }
  __syncwarp();
  mbar_wait(&bar[1], 0);
  mbar_wait(&bar[2], 0);
  mbar_wait(&bar[3], 0);
  tc_fence_after();
  const uint32_t lane = (uint32_t)(32 * w) << 16;
  float* outs[3] = {D1, D2, D3};
  const int cols[3] = {0, 128, 256};
  for (int o = 0; o < 3; ++o)
    for (int half = 0; half < 2; ++half) {
      uint32_t r[32];
      tmem_ld32(tb + lane + cols[o] + 32 * half, r);
      tmem_ld_wait();
      for (int c = 0; c < 32; ++c) outs[o][t * N + 32 * half + c] = __uint_as_float(r[c]);
    }
  tc_fence_before();
  __syncthreads();
  if (w == 1) tmem_dealloc<512>(tb);
}

static PFN_cuTensorMapEncodeTiled_v12000 encode() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}

static void make_map(CUtensorMap* m, const float* base, int rows, int cols, int box_rows) {
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 4};
  cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); exit(1); }
}

static float trunc19(float x) {
  uint32_t u; memcpy(&u, &x, 4); u &= 0xFFFFE000u; memcpy(&x, &u, 4); return x;
}
static float rn19(float x) {
  uint32_t u; memcpy(&u, &x, 4);
  u = (u + 0xFFFu + ((u >> 13) & 1u)) & 0xFFFFE000u;
  memcpy(&x, &u, 4); return x;
}

int main() {
  std::vector<float> A(M * KC), B(N * KC);
  srand(7);
  for (auto& x : A) x = (float)rand() / RAND_MAX * 0.999f + 1e-3f;
  for (auto& x : B) x = (float)rand() / RAND_MAX * 0.999f + 1e-3f;
  float *dA, *dB, *d1, *d2, *d3;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&d1, M * N * 4); cudaMalloc(&d2, M * N * 4); cudaMalloc(&d3, M * N * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  CUtensorMap tA, tB;
  make_map(&tA, dA, M, KC, M);
  make_map(&tB, dB, N, KC, N);
  const int smem = 1024 + 16384 + 3 * 8192;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int reps_list[5] = {1, 16, 256, 2048, 8192};
  for (int ri = 1; ri < 5; ++ri) {
    probe<<<1, 128, smem>>>(tA, tB, dA, d1, d2, d3, reps_list[ri]);
    cudaDeviceSynchronize();
    std::vector<float> h(M * N);
    cudaMemcpy(h.data(), d3, M * N * 4, cudaMemcpyDeviceToHost);
    double emax = 0, emean = 0;
    for (int m = 0; m < M; ++m) for (int n = 0; n < N; ++n) {
      double ex = 0; for (int k = 0; k < KC; ++k) ex += (double)A[m * KC + k] * B[n * KC + k];
      ex *= reps_list[ri];
      double r = (h[m * N + n] - ex) / ex; emax = fmax(emax, fabs(r)); emean += r;
    }
    printf("reps %d (K=%d): 3xTF32 max rel err %.3e mean signed %.3e\n", reps_list[ri], 32 * reps_list[ri], emax, emean / (M * N));
  }
  probe<<<1, 128, smem>>>(tA, tB, dA, d1, d2, d3, 1);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  std::vector<float> h1(M * N), h2(M * N), h3(M * N);
  cudaMemcpy(h1.data(), d1, M * N * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(h2.data(), d2, M * N * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(h3.data(), d3, M * N * 4, cudaMemcpyDeviceToHost);
  double e1[3] = {0, 0, 0}, e2[3] = {0, 0, 0}, e3 = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double ex = 0, tr = 0, rn = 0;
      for (int k = 0; k < KC; ++k) {
        ex += (double)A[m * KC + k] * B[n * KC + k];
        tr += (double)trunc19(A[m * KC + k]) * trunc19(B[n * KC + k]);
        rn += (double)rn19(A[m * KC + k]) * rn19(B[n * KC + k]);
      }
      const double refs[3] = {ex, tr, rn};
      for (int i = 0; i < 3; ++i) {
        e1[i] = fmax(e1[i], fabs(h1[m * N + n] - refs[i]) / ex);
        e2[i] = fmax(e2[i], fabs(h2[m * N + n] - refs[i]) / ex);
      }
      e3 = fmax(e3, fabs(h3[m * N + n] - ex) / ex);
    }
  printf("SS  max rel err vs exact %.3e  vs trunc %.3e  vs rn %.3e\n", e1[0], e1[1], e1[2]);
  printf("TS  max rel err vs exact %.3e  vs trunc %.3e  vs rn %.3e\n", e2[0], e2[1], e2[2]);
  printf("3xTF32 TS max rel err vs exact %.3e\n", e3);
  printf("sample D1[0][0]=%.8f D2[0][0]=%.8f D3[5][7]=%.8f\n", h1[0], h2[0], h3[5 * N + 7]);
  const bool ok = e1[0] < 2e-3 && e2[0] < 2e-3 && e3 < 1e-6;
  printf(ok ? "PROBE OK\n" : "PROBE FAIL\n");
  return ok ? 0 : 2;
}
