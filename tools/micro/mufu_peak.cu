// Sustained MUFU.EX2 throughput on one B200 (ex2.approx.ftz.f32), with and
// without an FADD per exponential -- the ceiling the sweep roofline divides by.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_peak mufu_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int kAdd>
__global__ void __launch_bounds__(256) ex2_loop(float* out, int iters, float seed) {
  float v[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = seed * (threadIdx.x + i) * 1e-9f;
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float y;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(v[i]));
      if (kAdd) acc += y;
      v[i] = kAdd ? v[i] : y * -1e-3f;
    }
  }
  float s = acc;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += v[i];
  if (s == 12345.f) out[0] = s;
}

int main() {
  float* out;
  cudaMalloc(&out, 4);
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int iters = 4096;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int blocksPerSm : {4, 8}) {
    for (int mode = 0; mode < 2; ++mode) {
      const int grid = sms * blocksPerSm;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (mode == 0) ex2_loop<0><<<grid, 256>>>(out, iters, 1.f);
        else ex2_loop<1><<<grid, 256>>>(out, iters, 1.f);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double ex2 = (double)grid * 256 * iters * 16;
        if (rep)
          printf("blocks/SM %d mode %s: %.3f Tex2/s = %.2f ex2/clk/SM at %.0f MHz max\n",
                 blocksPerSm, mode ? "ex2+fadd" : "ex2-chain", ex2 / ms / 1e9,
                 ex2 / (ms * 1e-3) / sms / (clk * 1e3), clk / 1e3);
      }
    }
  }
  return 0;
}
