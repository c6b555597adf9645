// Raw tcgen05.mma issue/throughput rates for the shapes the 3xTF32
// contraction can use (no data movement: operands stay in place).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_1907_01729_b200/csrc \
//        -o umma_rate umma_rate.cu
#include <cuda_runtime.h>

#include <cstdio>

#include "common.cuh"
#include "umma.cuh"

using namespace skb;

__device__ __forceinline__ void umma_f16_ss(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// mode: 0 TS same acc, 1 TS 3 accs interleaved, 2 SS same acc, 3 SS 3 accs, 4 f16 SS
template <int MODE, int N>
__global__ void __launch_bounds__(128, 1) rate(int iters, unsigned long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t tb_sh;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp_id() == 0) tmem_alloc<512>(&tb_sh);
  for (int i = threadIdx.x; i < 32768 / 4; i += 128) reinterpret_cast<float*>(sm)[i] = 0.5f;
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tb_sh;
  if (threadIdx.x == 0) {
    const uint32_t idesc = MODE == 4 ? ((1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | (8u << 24))
                                     : umma_idesc_tf32(128, N);
    const uint64_t ad = umma_sdesc_sw128(smem_u32(sm));
    const uint64_t bd = umma_sdesc_sw128(smem_u32(sm + 16384));
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 12; ++k) {
        const uint32_t d = (MODE == 1 || MODE == 3) ? tb + (k % 3) * 64 : tb;
        if (MODE <= 1) umma_tf32_ts(d, tb + 256 + 8 * (k & 3), bd, idesc, 1);
        else if (MODE <= 3) umma_tf32_ss(d, ad, bd, idesc, 1);
        else umma_f16_ss(d, ad, bd, idesc, 1);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    cyc[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp_id() == 0) tmem_dealloc<512>(tb);
}

template <int MODE, int N>
void run(const char* name, int blocks) {
  unsigned long long* d;
  cudaMalloc(&d, 8 * 148);
  const int iters = 2000;
  cudaFuncSetAttribute(rate<MODE, N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  rate<MODE, N><<<blocks, 128, 80 * 1024>>>(iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h = 0;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("%-28s N=%3d blocks %3d: %s  %.1f cycles per MMA\n", name, N, blocks, cudaGetErrorString(e),
         (double)h / (iters * 12.0));
  cudaFree(d);
}

int main() {
  for (int blocks : {1, 148}) {
    run<0, 64>("TS tf32 one accumulator", blocks);
    run<1, 64>("TS tf32 three accumulators", blocks);
    run<0, 128>("TS tf32 one accumulator", blocks);
    run<0, 256>("TS tf32 one accumulator", blocks);
    run<2, 64>("SS tf32 one accumulator", blocks);
    run<3, 64>("SS tf32 three accumulators", blocks);
    run<2, 128>("SS tf32 one accumulator", blocks);
    run<2, 256>("SS tf32 one accumulator", blocks);
    run<4, 64>("SS f16 one accumulator", blocks);
    run<4, 256>("SS f16 one accumulator", blocks);
  }
  return 0;
}
