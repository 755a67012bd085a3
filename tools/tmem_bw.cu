// Microbenchmark: tcgen05.ld / tcgen05.st throughput per SM (32x32b.x32: 4 KB per warp op).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2405_10853_b200/csrc tools/tmem_bw.cu -o tools/tmem_bw
#include <cstdio>
#include "common.cuh"
#include "sm100.cuh"
using namespace fb;
using namespace fb::sm100;

template <int NW, bool ST, int INFL = 1>
__global__ void __launch_bounds__(NW * 32, 1) tmem_kernel(long long* out, float* sink, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 64;
  uint32_t r[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) r[i] = i;
  float acc = 0.f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (ST) {
      tmem_st_32x32b_x32(tmem + (it & 1) * 32, r);
      tmem_st_wait();
    } else {
      if (INFL == 1) {
        tmem_ld_32x32b_x32(tmem + (it & 1) * 32, r);
        tmem_ld_wait();
        acc += __uint_as_float(r[it & 31]);
      } else {
        uint32_t r2[32];
        tmem_ld_32x32b_x32(tmem, r);
        tmem_ld_32x32b_x32(tmem + 32, r2);
        tmem_ld_wait();
        acc += __uint_as_float(r[it & 31]) + __uint_as_float(r2[(it + 1) & 31]);
        ++it;
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = t1 - t0;
  if (acc == 12345.f) sink[0] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(slot, 512); }
}

template <int NW, bool ST, int INFL = 1>
void run(long long* d, float* s) {
  const int iters = 4096;
  tmem_kernel<NW, ST, INFL><<<148, NW * 32>>>(d, s, iters);
  tmem_kernel<NW, ST, INFL><<<148, NW * 32>>>(d, s, iters);
  long long c;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  const double bytes = (double)NW * iters * 4096;
  printf("%s infl=%d warps=%2d: %.1f B/cycle/SM  (%s)\n", ST ? "st" : "ld", INFL, NW, bytes / c, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* d;
  float* s;
  cudaMalloc(&d, 8);
  cudaMalloc(&s, 8);
  run<4, false>(d, s); run<8, false>(d, s); run<16, false>(d, s);
  run<4, false, 2>(d, s); run<8, false, 2>(d, s); run<16, false, 2>(d, s);
  run<4, true>(d, s); run<8, true>(d, s); run<16, true>(d, s);
  return 0;
}
