// Check of the A-from-TMEM ("TS") tcgen05.mma layout used by the attention kernels:
// A [128 x 64] bf16 written to TMEM with tcgen05.st (lane = row, 32-bit column c holds
// k = 2c (low half) and 2c+1 (high half)), B [64 n x 64 k] K-major SW128 in smem,
// D = A B^T over 4 MMAs (K = 16 each, A column offset +8 per MMA). Prints max |err|.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2405_10853_b200/csrc tools/ts_mma_test.cu -o tools/ts_mma_test
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include "common.cuh"
#include "sm100.cuh"
using namespace fb;
using namespace fb::sm100;

__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a), "l"(bdesc), "r"(idesc), "r"(acc)
      : "memory");
}

__global__ void __launch_bounds__(128, 1) ts_kernel(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D) {
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024 - (smem_u32(sm_raw) & 1023)) & 1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  // B: 64 rows (n) x 64 k bf16 = 128 B per row, SW128: 16 B chunk c of row r at (c ^ (r & 7))
  for (int i = tid; i < 64 * 8; i += 128) {
    const int r = i / 8, c = i % 8;
    *reinterpret_cast<uint4*>(sm + r * 128 + ((c ^ (r & 7)) << 4)) = *reinterpret_cast<const uint4*>(B + r * 64 + c * 8);
  }
  if (tid == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc(&slot, 128);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  // A row tid -> TMEM lane tid, columns [64, 96)
  uint32_t a[32];
#pragma unroll
  for (int c = 0; c < 32; ++c) a[c] = pack_bf16(__bfloat162float(A[tid * 64 + 2 * c]), __bfloat162float(A[tid * 64 + 2 * c + 1]));
  tmem_st_32x32b_x32(tmem + ((uint32_t)(warp * 32) << 16) + 64, a);
  tmem_st_wait();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    constexpr uint32_t id = idesc_bf16_f32(128, 64, 0, 0);
    const uint64_t bd = smem_desc_sw128(smem_u32(sm), 16, 1024);
    for (int kk = 0; kk < 4; ++kk) umma_ts(tmem, tmem + 64 + 8 * kk, bd + ((kk * 32) >> 4), id, kk > 0);
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t d0[32], d1[32];
  tmem_ld_32x32b_x32(tmem + ((uint32_t)(warp * 32) << 16), d0);
  tmem_ld_32x32b_x32(tmem + ((uint32_t)(warp * 32) << 16) + 32, d1);
  tmem_ld_wait();
  for (int c = 0; c < 32; ++c) {
    D[tid * 64 + c] = __uint_as_float(d0[c]);
    D[tid * 64 + 32 + c] = __uint_as_float(d1[c]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 128); }
}

int main() {
  const int M = 128, N = 64, K = 64;
  __nv_bfloat16 *hA = (__nv_bfloat16*)malloc(M * K * 2), *hB = (__nv_bfloat16*)malloc(N * K * 2);
  float* hD = (float*)malloc(M * N * 4);
  srand(1);
  for (int i = 0; i < M * K; ++i) hA[i] = __float2bfloat16((rand() % 17 - 8) / 8.0f);
  for (int i = 0; i < N * K; ++i) hB[i] = __float2bfloat16((rand() % 17 - 8) / 8.0f);
  __nv_bfloat16 *dA, *dB;
  float* dD;
  cudaMalloc(&dA, M * K * 2); cudaMalloc(&dB, N * K * 2); cudaMalloc(&dD, M * N * 4);
  cudaMemcpy(dA, hA, M * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, N * K * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(ts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 20 * 1024);
  ts_kernel<<<1, 128, 20 * 1024>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(hD, dD, M * N * 4, cudaMemcpyDeviceToHost);
  double err = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double r = 0;
      for (int k = 0; k < K; ++k) r += (double)__bfloat162float(hA[m * K + k]) * __bfloat162float(hB[n * K + k]);
      err = fmax(err, fabs(r - hD[m * N + n]));
    }
  printf("TS mma: %s, max |err| = %g (D[0]=%g)\n", cudaGetErrorString(e), err, hD[0]);
  return 0;
}
