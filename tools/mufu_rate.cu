// Microbenchmark: ex2.approx.ftz.f32 (MUFU.EX2) and FFMA2 throughput per SM, cycles per warp instruction.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mufu_rate.cu -o tools/mufu_rate
#include <cstdio>
template <int NW, int MODE>
__global__ void __launch_bounds__(NW * 32, 1) k(float* out, long long* cyc, int iters) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (MODE == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      else asm volatile("fma.rn.f32 %0, %0, 0.999, 0.0001;" : "+f"(a[i]));
    }
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
template <int NW, int MODE>
void run(float* o, long long* c) {
  const int iters = 2048;
  k<NW, MODE><<<148, NW * 32>>>(o, c, iters);
  k<NW, MODE><<<148, NW * 32>>>(o, c, iters);
  long long h;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  const double winstr = (double)NW * iters * 16;  // warp instructions per SM
  printf("%s warps=%2d: %.2f cycles per warp-instr per SM (%.2f per SMSP)\n", MODE ? "FFMA" : "MUFU.EX2", NW, h / winstr,
         4 * h / winstr);
}
int main() {
  float* o; long long* c;
  cudaMalloc(&o, 148 * 1024 * 4); cudaMalloc(&c, 8);
  run<4, 0>(o, c); run<8, 0>(o, c); run<16, 0>(o, c);
  run<4, 1>(o, c); run<8, 1>(o, c); run<16, 1>(o, c);
  return 0;
}
