// Stand-alone timing of the 3xTF32 contraction kernel (sweep_umma.cuh) on a
// config-5-like shape, for tuning its pipeline depths without the solver.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I../../paper_1907_01729_b200/csrc [-DSKB_UM_...] -o umma_gemm_bench umma_gemm_bench.cu -lcuda
//   ./umma_gemm_bench M K N reps
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "umma.cuh"
#include "sweep_umma.cuh"

__device__ unsigned long long g_um_dbg_cycles[2];

using namespace skb;

static PFN_cuTensorMapEncodeTiled_v12000 encode() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
}
static void make_map(CUtensorMap* m, const float* base, size_t rows, int box_rows) {
  cuuint64_t dims[2] = {32, (cuuint64_t)rows};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)base, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); exit(1); }
}

__global__ void fill_tiled(float* a, long long n, unsigned seed) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    unsigned h = (unsigned)(i * 2654435761u) ^ seed;
    h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    a[i] = 0.25f + (h & 0xFFFFFF) * (1.0f / 16777216.0f);
  }
}

__global__ void split_planes(float* h, float* l, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const float x = h[i];
    h[i] = tf32_hi(x);
    l[i] = x - tf32_hi(x);
  }
}

int main(int argc, char** argv) {
  const int M = argc > 1 ? atoi(argv[1]) : 16384;
  const int K = argc > 2 ? atoi(argv[2]) : 65536;
  const int N = argc > 3 ? atoi(argv[3]) : 64;
  const int reps = argc > 4 ? atoi(argv[4]) : 10;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  UmmaParams p = {};
  p.M = M; p.N = N; p.K = K;
  p.MT = (M + kUmBM - 1) / kUmBM;
  p.NT = (N + kUmBN - 1) / kUmBN;
  p.KCH = (K + kUmBK - 1) / kUmBK;
  p.units = (long long)p.MT * p.NT * p.KCH;
  p.G = (int)std::min<long long>(sms, p.units);
  const size_t na = (size_t)p.MT * p.KCH * kUmBM * kUmBK, nb = (size_t)p.NT * p.KCH * kUmBN * kUmBK;
  float *A, *Bh, *Bl, *out, *part;
  cudaMalloc(&A, na * 4); cudaMalloc(&Bh, nb * 4); cudaMalloc(&Bl, nb * 4);
  cudaMalloc(&out, (size_t)M * N * 4); cudaMalloc(&part, (size_t)p.G * 2 * kUmBN * kUmBM * 4);
  fill_tiled<<<1184, 256>>>(A, (long long)na, 1u);
  fill_tiled<<<1184, 256>>>(Bh, (long long)nb, 2u);
  split_planes<<<1184, 256>>>(Bh, Bl, (long long)nb);   // Bh -> (hi, lo)
  p.out = out; p.ldo = M; p.part = part; p.status = nullptr;
  CUtensorMap ta, tbh, tbl;
  make_map(&ta, A, na / 32, kUmBM);
  make_map(&tbh, Bh, nb / 32, kUmBN);
  make_map(&tbl, Bl, nb / 32, kUmBN);
  cudaFuncSetAttribute(umma_gemm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kUmSmemBytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) {
    umma_gemm_kernel<false><<<p.G, kUmThreads, kUmSmemBytes>>>(ta, tbh, tbl, p);
    umma_fixup_kernel<<<p.G, 256>>>(p);
  }
  cudaError_t err = cudaDeviceSynchronize();
  if (err != cudaSuccess) { printf("error %s\n", cudaGetErrorString(err)); return 1; }
  unsigned long long zero2[2] = {0, 0};
  cudaMemcpyToSymbol(g_um_dbg_cycles, zero2, 16);
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) umma_gemm_kernel<false><<<p.G, kUmThreads, kUmSmemBytes>>>(ta, tbh, tbl, p);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  ms /= reps;
  unsigned long long cyc[2];
  cudaMemcpyFromSymbol(cyc, g_um_dbg_cycles, 16);
  if (cyc[1]) printf("cycles per chunk (per CTA, incl. fill/drain): %.1f  implied SM clock %.0f MHz\n",
                     (double)cyc[0] / cyc[1], (double)cyc[0] / p.G / reps / (ms * 1e3));
  umma_fixup_kernel<<<p.G, 256>>>(p);
  cudaDeviceSynchronize();
  // spot-check a few outputs against a double reference (the tiled A layout)
  std::vector<float> hA(na), hB(nb), hO((size_t)M * N);
  cudaMemcpy(hA.data(), A, na * 4, cudaMemcpyDeviceToHost);
  std::vector<float> hBl(nb);
  cudaMemcpy(hB.data(), Bh, nb * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(hBl.data(), Bl, nb * 4, cudaMemcpyDeviceToHost);
  for (size_t i = 0; i < nb; ++i) hB[i] += hBl[i];
  cudaMemcpy(hO.data(), out, (size_t)M * N * 4, cudaMemcpyDeviceToHost);
  double emax = 0;
  for (int t = 0; t < 16; ++t) {
    const int m = (int)((t * 7919LL) % M), n = (t * 13) % N;
    double ref = 0;
    for (int k = 0; k < K; ++k)
      ref += (double)hA[um_tiled_index(m, k, kUmBM, p.KCH)] * hB[um_tiled_index(n, k, kUmBN, p.KCH)];
    emax = fmax(emax, fabs(hO[(size_t)n * M + m] - ref) / ref);
  }
  const double gb = (double)M * K * 4 / 1e9;
  printf("M %d K %d N %d  SUB %d ASM %d BSM %d ATM %d SLOTS %d PROMO %d: %.3f ms/launch  A %.1f GB/s  max rel err %.2e\n",
         M, K, N, kUmSub, kUmAStagesSm, kUmBStagesSm, kUmAStages, kUmSlots, kUmPromo, ms, gb / (ms * 1e-3), emax);
  return 0;
}
