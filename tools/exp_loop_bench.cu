// Microbenchmark of the attention-forward softmax exp loop body (FFMA2/FADD2 + MUFU.EX2 +
// F2FP + FADD2 sum) per element, with NW warps per SM. Prints cycles per element per warp.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2405_10853_b200/csrc tools/exp_loop_bench.cu -o tools/exp_loop_bench
#include <cstdio>
#include "common.cuh"
__device__ __forceinline__ unsigned long long u64of(float2 v) { return *reinterpret_cast<unsigned long long*>(&v); }
__device__ __forceinline__ float2 f2of(unsigned long long v) { return *reinterpret_cast<float2*>(&v); }
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(u64of(a)), "l"(u64of(b)), "l"(u64of(c)));
  return f2of(r);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  unsigned long long r;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(u64of(a)), "l"(u64of(b)));
  return f2of(r);
}
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
template <int NW, int MODE>
__global__ void __launch_bounds__(NW * 32, 1) k(float* out, long long* cyc, int iters) {
  __shared__ float4 colb4[32];
  __shared__ uint32_t pks[NW * 32 * 33];
  if (threadIdx.x < 32) colb4[threadIdx.x] = make_float4(threadIdx.x * 0.01f, 0.02f, 0.03f, 0.04f);
  __syncthreads();
  uint32_t v[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) v[i] = __float_as_uint(-0.01f * (threadIdx.x + i));
  const float2 c2 = make_float2(0.1f, 0.1f);
  float2 sh = make_float2(-1.0f, -1.0f);
  float2 ps[4] = {};
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t pk[32];
#pragma unroll
    for (int u = 0; u < 64; u += 4) {
      const float4 cb = colb4[u >> 2];
      float2 a0 = ffma2(make_float2(__uint_as_float(v[u]), __uint_as_float(v[u + 1])), c2, fadd2(make_float2(cb.x, cb.y), sh));
      float2 a1 = ffma2(make_float2(__uint_as_float(v[u + 2]), __uint_as_float(v[u + 3])), c2, fadd2(make_float2(cb.z, cb.w), sh));
      float2 p0, p1;
      if (MODE == 0) {
        p0 = make_float2(ex2(a0.x), ex2(a0.y));
        p1 = make_float2(ex2(a1.x), ex2(a1.y));
      } else {
        p0 = a0; p1 = a1;
      }
      ps[(u >> 2) & 3] = fadd2(ps[(u >> 2) & 3], fadd2(p0, p1));
      pk[u >> 1] = fb::pack_bf16(p0.x, p0.y);
      pk[(u >> 1) + 1] = fb::pack_bf16(p1.x, p1.y);
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) pks[threadIdx.x * 33 + i] = pk[i];
    sh.x += 1e-7f; sh.y = sh.x;
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = ps[0].x + ps[1].y + ps[2].x + ps[3].y + __uint_as_float(pks[threadIdx.x]);
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
}
template <int NW, int MODE>
void run(float* o, long long* c) {
  const int iters = 512;
  k<NW, MODE><<<148, NW * 32>>>(o, c, iters);
  k<NW, MODE><<<148, NW * 32>>>(o, c, iters);
  long long h;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%s warps/SM=%2d: %.2f cycles per element per warp (MUFU bound 8 x warps/SMSP = %d) %s\n",
         MODE ? "no-exp" : "exp", NW, (double)h / (iters * 64.0), 8 * NW / 4, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  float* o; long long* c;
  cudaMalloc(&o, 148 * 1024 * 4); cudaMalloc(&c, 8);
  run<4, 0>(o, c); run<8, 0>(o, c); run<4, 1>(o, c); run<8, 1>(o, c);
  return 0;
}
