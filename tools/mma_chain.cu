// Microbenchmark: tcgen05.mma issue/latency for short-N MMAs. One CTA per SM, one thread
// issues NMMA kind::f16 MMAs (M=128, N=NN, K=16, A/B from smem) spread round-robin over
// CH independent TMEM accumulators, then commits and waits. Prints cycles per MMA.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2405_10853_b200/csrc tools/mma_chain.cu -o tools/mma_chain
#include <cstdio>
#include <cuda.h>
#include "common.cuh"
#include "sm100.cuh"
using namespace fb;
using namespace fb::sm100;

template <int NN, int CH>
__global__ void __launch_bounds__(128, 1) chain_kernel(long long* out, int nmma) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* base = sm + ((1024 - (smem_u32(sm) & 1023)) & 1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(base)[i] = 0;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(&slot, 512);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t id = idesc_bf16_f32(128, NN, 0, 0);
    const uint64_t ad = smem_desc_sw128(smem_u32(base), 16, 1024), bd = smem_desc_sw128(smem_u32(base) + 32768, 16, 1024);
    long long t0 = clock64();
    for (int i = 0; i < nmma; i += CH) {
#pragma unroll
      for (int c = 0; c < CH; ++c) umma_f16(tmem + c * NN, ad + ((i & 3) * 2), bd + ((i & 3) * 2), id, i > 0);
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int NN, int CH>
void run(long long* d) {
  auto k = chain_kernel<NN, CH>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 66 * 1024);
  const int n = 512;
  k<<<148, 128, 66 * 1024>>>(d, n);
  k<<<148, 128, 66 * 1024>>>(d, n);
  long long c;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const double math = 128.0 * NN / 256.0;  // cycles of tensor work per MMA at full rate
  printf("N=%3d chains=%d: %.1f cycles/MMA (full-rate math %.0f) err=%s\n", NN, CH, (double)c / n, math,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  run<64, 1>(d); run<64, 2>(d); run<64, 4>(d);
  run<128, 1>(d); run<128, 2>(d); run<128, 4>(d);
  run<256, 1>(d); run<256, 2>(d);
  return 0;
}
