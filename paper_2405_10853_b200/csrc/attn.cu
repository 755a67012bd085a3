// Fused causal self-attention with ALiBi, forward and backward (flash-style, no
// T x T materialisation).
//
// Reference: Block.forward attention  fedforge/model.py:92-98
//   scores = q k^T / sqrt(dh) + bias,  bias[h,i,j] = -slope_h (i - j) (j <= i), -inf above
//   slope_h = 2^(-8 (h+1) / H)        model.py:46-50 (used for every H, incl. H = 12)
// The (H, ctx, ctx) f32 bias buffer of the reference (model.py:115-121) is never
// built: the bias is one FFMA per score in registers.
//
// Layout: qkv is the qkv-GEMM output [B*T][3d] bf16 (q | k | v, head h at columns
// h*dh), o is [B*T][d] bf16 — exactly the attn_proj GEMM operand — so no permutes.
// The softmax runs in base 2 (scores pre-multiplied by log2 e) and the saved
// row statistic is lse2 = max + log2(sum) in base-2 units ([B][H][T] f32).
//
// Tensor-core path (round 1): mma.sync m16n8k16 bf16 -> f32 with ldmatrix from
// XOR-swizzled shared memory and cp.async double buffering of K/V (fwd) and
// Q/dO (bwd). Forward: CTA = 64*NW query rows x one (b, h); backward: CTA = 64
// keys, dK/dV accumulated in registers, dQ accumulated in f32 with vector atomics.
#include "common.cuh"

namespace fb {

__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void ldsm_x4(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(saddr), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__device__ __forceinline__ uint32_t pack2(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

// swizzled [rows][DH] bf16 tile: 16-byte chunk c of row r lives at chunk c ^ (r & 7)
template <int DH>
__device__ __forceinline__ uint32_t swz(uint32_t base, int row, int col) {
  return base + row * (DH * 2) + ((((col >> 3) ^ (row & 7))) << 4) + ((col & 7) << 1);
}

// cooperative cp.async of `rows` rows (global row stride ld elements) into a swizzled tile
template <int DH>
__device__ __forceinline__ void load_tile(uint32_t sbase, const __nv_bfloat16* g, int64_t ld, int rows, int tid,
                                          int nthr) {
  constexpr int CPR = DH / 8;
  for (int idx = tid; idx < rows * CPR; idx += nthr) {
    const int r = idx / CPR, c = idx % CPR;
    cp_async16(sbase + r * (DH * 2) + ((c ^ (r & 7)) << 4), g + (int64_t)r * ld + c * 8);
  }
}

__device__ __forceinline__ float alibi_slope_log2(int h, int H, int use_alibi) {
  return use_alibi ? exp2f(-8.0f * (float)(h + 1) / (float)H) * 1.4426950408889634f : 0.0f;
}

// ------------------------------------------------------------------ forward
template <int DH, int NW>
__global__ void __launch_bounds__(NW * 32) attn_fwd_kernel(const __nv_bfloat16* __restrict__ qkv,
                                                           __nv_bfloat16* __restrict__ out, float* __restrict__ lse2,
                                                           int T, int H, float scale_log2, int use_alibi) {
  constexpr int BQ = 16 * NW;
  constexpr int BKV = 64;
  constexpr int NT = DH / 8;  // dh n-tiles
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sQ = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t sK0 = sQ + BQ * DH * 2;
  const uint32_t sV0 = sK0 + 2 * BKV * DH * 2;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int qb = gridDim.x - 1 - blockIdx.x;  // heavy (late) blocks first
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const int d = H * DH;
  const int64_t ld = 3 * (int64_t)d;
  const int q0 = qb * BQ;
  const __nv_bfloat16* Qg = qkv + ((int64_t)b * T + q0) * ld + h * DH;
  const __nv_bfloat16* Kg = qkv + (int64_t)b * T * ld + d + h * DH;
  const __nv_bfloat16* Vg = Kg + d;
  const float sl = alibi_slope_log2(h, H, use_alibi);

  load_tile<DH>(sQ, Qg, ld, BQ, tid, NW * 32);
  load_tile<DH>(sK0, Kg, ld, BKV, tid, NW * 32);
  load_tile<DH>(sV0, Vg, ld, BKV, tid, NW * 32);
  cp_commit();
  cp_wait<0>();
  __syncthreads();

  uint32_t qf[DH / 16][4];
#pragma unroll
  for (int kk = 0; kk < DH / 16; ++kk)
    ldsm_x4(qf[kk], swz<DH>(sQ, w * 16 + (lane & 7) + 8 * ((lane >> 3) & 1), kk * 16 + 8 * (lane >> 4)));

  float o[NT][4];
#pragma unroll
  for (int i = 0; i < NT; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  const int qrow0 = q0 + w * 16 + (lane >> 2);
  const int nkv = (q0 + BQ) / BKV;

  for (int j = 0; j < nkv; ++j) {
    const int buf = j & 1;
    if (j + 1 < nkv) {
      const int nb = buf ^ 1;
      load_tile<DH>(sK0 + nb * BKV * DH * 2, Kg + (int64_t)(j + 1) * BKV * ld, ld, BKV, tid, NW * 32);
      load_tile<DH>(sV0 + nb * BKV * DH * 2, Vg + (int64_t)(j + 1) * BKV * ld, ld, BKV, tid, NW * 32);
    }
    cp_commit();
    const uint32_t sK = sK0 + buf * BKV * DH * 2, sV = sV0 + buf * BKV * DH * 2;
    float s[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) s[i][0] = s[i][1] = s[i][2] = s[i][3] = 0.f;
#pragma unroll
    for (int kk = 0; kk < DH / 16; ++kk) {
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        uint32_t r[4];
        ldsm_x4(r, swz<DH>(sK, np * 16 + (lane & 7) + 8 * (lane >> 4), kk * 16 + 8 * ((lane >> 3) & 1)));
        mma16816(s[2 * np], qf[kk], r[0], r[1]);
        mma16816(s[2 * np + 1], qf[kk], r[2], r[3]);
      }
    }
    const bool diag = (j + 1) * BKV > q0 + w * 16;  // this tile may cross the diagonal for this warp
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = j * BKV + nt * 8 + 2 * (lane & 3) + (e & 1);
        const int qr = qrow0 + 8 * (e >> 1);
        float v = s[nt][e] * scale_log2 - sl * (float)(qr - key);
        if (diag && key > qr) v = -INFINITY;
        s[nt][e] = v;
      }
      mx0 = fmaxf(mx0, fmaxf(s[nt][0], s[nt][1]));
      mx1 = fmaxf(mx1, fmaxf(s[nt][2], s[nt][3]));
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
    const float a0 = exp2f(m0 - mn0), a1 = exp2f(m1 - mn1);
    m0 = mn0;
    m1 = mn1;
    float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      s[nt][0] = exp2f(s[nt][0] - mn0);
      s[nt][1] = exp2f(s[nt][1] - mn0);
      s[nt][2] = exp2f(s[nt][2] - mn1);
      s[nt][3] = exp2f(s[nt][3] - mn1);
      rs0 += s[nt][0] + s[nt][1];
      rs1 += s[nt][2] + s[nt][3];
    }
    l0 = l0 * a0 + rs0;
    l1 = l1 * a1 + rs1;
#pragma unroll
    for (int i = 0; i < NT; ++i) {
      o[i][0] *= a0; o[i][1] *= a0; o[i][2] *= a1; o[i][3] *= a1;
    }
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t pa[4] = {pack2(s[2 * kk][0], s[2 * kk][1]), pack2(s[2 * kk][2], s[2 * kk][3]),
                        pack2(s[2 * kk + 1][0], s[2 * kk + 1][1]), pack2(s[2 * kk + 1][2], s[2 * kk + 1][3])};
#pragma unroll
      for (int dp = 0; dp < DH / 16; ++dp) {
        uint32_t r[4];
        ldsm_x4_t(r, swz<DH>(sV, kk * 16 + (lane & 7) + 8 * ((lane >> 3) & 1), dp * 16 + 8 * (lane >> 4)));
        mma16816(o[2 * dp], pa, r[0], r[1]);
        mma16816(o[2 * dp + 1], pa, r[2], r[3]);
      }
    }
    cp_wait<0>();
    __syncthreads();
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float il0 = 1.f / l0, il1 = 1.f / l1;
  __nv_bfloat16* O0 = out + ((int64_t)b * T + qrow0) * d + h * DH;
  __nv_bfloat16* O1 = O0 + 8 * (int64_t)d;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int c = nt * 8 + 2 * (lane & 3);
    *reinterpret_cast<uint32_t*>(O0 + c) = pack2(o[nt][0] * il0, o[nt][1] * il0);
    *reinterpret_cast<uint32_t*>(O1 + c) = pack2(o[nt][2] * il1, o[nt][3] * il1);
  }
  if ((lane & 3) == 0) {
    float* L = lse2 + (int64_t)bh * T;
    L[qrow0] = m0 + log2f(l0);
    L[qrow0 + 8] = m1 + log2f(l1);
  }
}

// ------------------------------------------------------------------ backward
// D[bh][t] = sum_c dO * O, one warp per (row, head), 8-byte vector loads; the same warp
// zeroes that (row, head) slice of the f32 dQ accumulator (saves a memset pass).
__global__ void attn_bwd_dot_kernel(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dO,
                                    float* __restrict__ D, float* __restrict__ dq, int B, int T, int H, int dh) {
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (gw >= B * T * H) return;
  const int h = gw % H, row = gw / H;  // row = b*T + t
  const int d = H * dh;
  const __nv_bfloat16* a = o + (int64_t)row * d + h * dh;
  const __nv_bfloat16* g = dO + (int64_t)row * d + h * dh;
  float s = 0.f;
  for (int c = 4 * lane; c < dh; c += 128) {
    const uint2 av = *reinterpret_cast<const uint2*>(a + c), gv = *reinterpret_cast<const uint2*>(g + c);
    const __nv_bfloat162* ap = reinterpret_cast<const __nv_bfloat162*>(&av);
    const __nv_bfloat162* gp = reinterpret_cast<const __nv_bfloat162*>(&gv);
    const float2 a0 = __bfloat1622float2(ap[0]), a1 = __bfloat1622float2(ap[1]);
    const float2 g0 = __bfloat1622float2(gp[0]), g1 = __bfloat1622float2(gp[1]);
    s += a0.x * g0.x + a0.y * g0.y + a1.x * g1.x + a1.y * g1.y;
    if (dq) *reinterpret_cast<float4*>(dq + (int64_t)row * d + h * dh + c) = make_float4(0.f, 0.f, 0.f, 0.f);
  }
  s = warp_sum(s);
  if (lane == 0) {
    const int b = row / T, t = row % T;
    D[((int64_t)b * H + h) * T + t] = s;
  }
}

template <int DH>
__global__ void __launch_bounds__(128) attn_bwd_kernel(const __nv_bfloat16* __restrict__ qkv,
                                                       const __nv_bfloat16* __restrict__ dO,
                                                       const float* __restrict__ lse2, const float* __restrict__ Dd,
                                                       float* __restrict__ dq_acc, __nv_bfloat16* __restrict__ dqkv,
                                                       int T, int H, float scale_log2, float scale, int use_alibi) {
  constexpr int BKV = 64, BQ = 64, NT = DH / 8;
  extern __shared__ __align__(128) uint8_t smem[];
  const uint32_t sK = (uint32_t)__cvta_generic_to_shared(smem);
  const uint32_t sV = sK + BKV * DH * 2;
  const uint32_t sQ0 = sV + BKV * DH * 2;          // [2][BQ][DH]
  const uint32_t sO0 = sQ0 + 2 * BQ * DH * 2;       // dO [2][BQ][DH]
  const uint32_t sS = sO0 + 2 * BQ * DH * 2;        // dS^T [BKV][BQ] bf16
  float* sL = reinterpret_cast<float*>(smem + (BKV * DH * 2) * 2 + 4 * BQ * DH * 2 + BKV * BQ * 2);  // [2][BQ]
  float* sD = sL + 2 * BQ;                                                                          // [2][BQ]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int kb = blockIdx.x, bh = blockIdx.y, b = bh / H, h = bh % H;
  const int d = H * DH;
  const int64_t ld = 3 * (int64_t)d;
  const int k0 = kb * BKV;
  const __nv_bfloat16* Qg = qkv + (int64_t)b * T * ld + h * DH;
  const __nv_bfloat16* Kg = Qg + d + (int64_t)k0 * ld;
  const __nv_bfloat16* Vg = Kg + d;
  const __nv_bfloat16* dOg = dO + (int64_t)b * T * d + h * DH;
  const float* Lg = lse2 + (int64_t)bh * T;
  const float* Dg = Dd + (int64_t)bh * T;
  const float sl = alibi_slope_log2(h, H, use_alibi);
  const int first = k0 / BQ, nq = T / BQ;

  load_tile<DH>(sK, Kg, ld, BKV, tid, 128);
  load_tile<DH>(sV, Vg, ld, BKV, tid, 128);
  load_tile<DH>(sQ0, Qg + (int64_t)first * BQ * ld, ld, BQ, tid, 128);
  load_tile<DH>(sO0, dOg + (int64_t)first * BQ * d, d, BQ, tid, 128);
  if (tid < BQ) { sL[tid] = Lg[first * BQ + tid]; sD[tid] = Dg[first * BQ + tid]; }
  cp_commit();

  float dv[NT][4], dk[NT][4];
#pragma unroll
  for (int i = 0; i < NT; ++i) {
#pragma unroll
    for (int e = 0; e < 4; ++e) { dv[i][e] = 0.f; dk[i][e] = 0.f; }
  }
  const int key0 = k0 + w * 16 + (lane >> 2);  // rows of this thread: key0, key0 + 8

  for (int it = first; it < nq; ++it) {
    const int buf = (it - first) & 1;
    cp_wait<0>();
    __syncthreads();
    if (it + 1 < nq) {
      const int nb = buf ^ 1;
      load_tile<DH>(sQ0 + nb * BQ * DH * 2, Qg + (int64_t)(it + 1) * BQ * ld, ld, BQ, tid, 128);
      load_tile<DH>(sO0 + nb * BQ * DH * 2, dOg + (int64_t)(it + 1) * BQ * d, d, BQ, tid, 128);
      if (tid < BQ) { sL[nb * BQ + tid] = Lg[(it + 1) * BQ + tid]; sD[nb * BQ + tid] = Dg[(it + 1) * BQ + tid]; }
    }
    cp_commit();
    const uint32_t sQ = sQ0 + buf * BQ * DH * 2, sO = sO0 + buf * BQ * DH * 2;
    const float* L = sL + buf * BQ;
    const float* Dv = sD + buf * BQ;
    const int q0 = it * BQ;
    // S^T = K Q^T and dP^T = V dO^T  (16 keys x 64 queries per warp)
    float s[8][4], dp[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
#pragma unroll
      for (int e = 0; e < 4; ++e) { s[i][e] = 0.f; dp[i][e] = 0.f; }
    }
#pragma unroll
    for (int kk = 0; kk < DH / 16; ++kk) {
      uint32_t kf[4], vf[4];
      ldsm_x4(kf, swz<DH>(sK, w * 16 + (lane & 7) + 8 * ((lane >> 3) & 1), kk * 16 + 8 * (lane >> 4)));
      ldsm_x4(vf, swz<DH>(sV, w * 16 + (lane & 7) + 8 * ((lane >> 3) & 1), kk * 16 + 8 * (lane >> 4)));
#pragma unroll
      for (int np = 0; np < 4; ++np) {
        uint32_t r[4], g[4];
        ldsm_x4(r, swz<DH>(sQ, np * 16 + (lane & 7) + 8 * (lane >> 4), kk * 16 + 8 * ((lane >> 3) & 1)));
        ldsm_x4(g, swz<DH>(sO, np * 16 + (lane & 7) + 8 * (lane >> 4), kk * 16 + 8 * ((lane >> 3) & 1)));
        mma16816(s[2 * np], kf, r[0], r[1]);
        mma16816(s[2 * np + 1], kf, r[2], r[3]);
        mma16816(dp[2 * np], vf, g[0], g[1]);
        mma16816(dp[2 * np + 1], vf, g[2], g[3]);
      }
    }
    // P^T, dS^T
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int ql = nt * 8 + 2 * (lane & 3) + (e & 1);
        const int q = q0 + ql;
        const int key = key0 + 8 * (e >> 1);
        float p = 0.f;
        if (q >= key) p = exp2f(s[nt][e] * scale_log2 - sl * (float)(q - key) - L[ql]);
        s[nt][e] = p;
        dp[nt][e] = p * (dp[nt][e] - Dv[ql]);
      }
    }
    // dV += P^T dO ; dK += dS^T Q   (A operands straight from the C fragments)
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      uint32_t pa[4] = {pack2(s[2 * kk][0], s[2 * kk][1]), pack2(s[2 * kk][2], s[2 * kk][3]),
                        pack2(s[2 * kk + 1][0], s[2 * kk + 1][1]), pack2(s[2 * kk + 1][2], s[2 * kk + 1][3])};
      uint32_t da[4] = {pack2(dp[2 * kk][0], dp[2 * kk][1]), pack2(dp[2 * kk][2], dp[2 * kk][3]),
                        pack2(dp[2 * kk + 1][0], dp[2 * kk + 1][1]), pack2(dp[2 * kk + 1][2], dp[2 * kk + 1][3])};
#pragma unroll
      for (int dq = 0; dq < DH / 16; ++dq) {
        uint32_t r[4], g[4];
        ldsm_x4_t(g, swz<DH>(sO, kk * 16 + (lane & 7) + 8 * ((lane >> 3) & 1), dq * 16 + 8 * (lane >> 4)));
        ldsm_x4_t(r, swz<DH>(sQ, kk * 16 + (lane & 7) + 8 * ((lane >> 3) & 1), dq * 16 + 8 * (lane >> 4)));
        mma16816(dv[2 * dq], pa, g[0], g[1]);
        mma16816(dv[2 * dq + 1], pa, g[2], g[3]);
        mma16816(dk[2 * dq], da, r[0], r[1]);
        mma16816(dk[2 * dq + 1], da, r[2], r[3]);
      }
    }
    // dS^T -> smem [64 keys][64 queries]
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const int r0 = w * 16 + (lane >> 2);
      const int c = nt * 8 + 2 * (lane & 3);
      asm volatile("st.shared.b32 [%0], %1;" ::"r"(sS + r0 * 128 + ((nt ^ (r0 & 7)) << 4) + ((c & 7) << 1)),
                   "r"(pack2(dp[nt][0], dp[nt][1])));
      const int r1 = r0 + 8;
      asm volatile("st.shared.b32 [%0], %1;" ::"r"(sS + r1 * 128 + ((nt ^ (r1 & 7)) << 4) + ((c & 7) << 1)),
                   "r"(pack2(dp[nt][2], dp[nt][3])));
    }
    __syncthreads();
    // dQ[q0 + w*16 .. +15] += dS K * scale
    uint32_t af[4][4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const int kr = kk * 16 + (lane & 7) + 8 * (lane >> 4);
      const int qc = w * 16 + 8 * ((lane >> 3) & 1);
      ldsm_x4_t(af[kk], sS + kr * 128 + (((qc >> 3) ^ (kr & 7)) << 4));
    }
    float* dqrow0 = dq_acc + ((int64_t)b * T + q0 + w * 16 + (lane >> 2)) * d + h * DH;
    float* dqrow1 = dqrow0 + 8 * (int64_t)d;
#pragma unroll
    for (int dq = 0; dq < DH / 16; ++dq) {
      float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        uint32_t r[4];
        ldsm_x4_t(r, swz<DH>(sK, kk * 16 + (lane & 7) + 8 * ((lane >> 3) & 1), dq * 16 + 8 * (lane >> 4)));
        mma16816(acc[0], af[kk], r[0], r[1]);
        mma16816(acc[1], af[kk], r[2], r[3]);
      }
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int c = dq * 16 + hh * 8 + 2 * (lane & 3);
        atomicAdd(reinterpret_cast<float2*>(dqrow0 + c), make_float2(acc[hh][0] * scale, acc[hh][1] * scale));
        atomicAdd(reinterpret_cast<float2*>(dqrow1 + c), make_float2(acc[hh][2] * scale, acc[hh][3] * scale));
      }
    }
  }
  cp_wait<0>();
  // dK (scaled) and dV -> dqkv
  __nv_bfloat16* dK0 = dqkv + ((int64_t)b * T + key0) * ld + d + h * DH;
  __nv_bfloat16* dK1 = dK0 + 8 * ld;
  __nv_bfloat16* dV0 = dK0 + d;
  __nv_bfloat16* dV1 = dK1 + d;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int c = nt * 8 + 2 * (lane & 3);
    *reinterpret_cast<uint32_t*>(dK0 + c) = pack2(dk[nt][0] * scale, dk[nt][1] * scale);
    *reinterpret_cast<uint32_t*>(dK1 + c) = pack2(dk[nt][2] * scale, dk[nt][3] * scale);
    *reinterpret_cast<uint32_t*>(dV0 + c) = pack2(dv[nt][0], dv[nt][1]);
    *reinterpret_cast<uint32_t*>(dV1 + c) = pack2(dv[nt][2], dv[nt][3]);
  }
}

// dqkv[:, 0:d] = bf16(dq accumulator): 8 columns per thread (two 16-byte loads, one 16-byte store)
__global__ void dq_finalize_kernel(const float* __restrict__ acc, __nv_bfloat16* __restrict__ dqkv, int rows, int d) {
  const int64_t n8 = (int64_t)rows * d / 8;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = 8 * i, r = e / d, c = e % d;
    const float4 x = *reinterpret_cast<const float4*>(acc + e), y = *reinterpret_cast<const float4*>(acc + e + 4);
    *reinterpret_cast<uint4*>(dqkv + r * 3 * d + c) =
        make_uint4(pack_bf16(x.x, x.y), pack_bf16(x.z, x.w), pack_bf16(y.x, y.y), pack_bf16(y.z, y.w));
  }
}

template <int DH>
int attn_fwd_tc_launch(const void* qkv, void* o, float* lse, int B, int T, int H, int use_alibi, cudaStream_t st);

template <int DH>
static int attn_fwd_launch(const void* qkv, void* o, float* lse, int B, int T, int H, int use_alibi, cudaStream_t st) {
  if (T % 256 == 0) return attn_fwd_tc_launch<DH>(qkv, o, lse, B, T, H, use_alibi, st);  // tcgen05 path
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)DH);
  if (T % 128 == 0) {
    constexpr int NW = 8;
    const int shm = (16 * NW + 4 * 64) * DH * 2;
    auto k = attn_fwd_kernel<DH, NW>;
    FB_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, shm));
    k<<<dim3(T / (16 * NW), B * H), NW * 32, shm, st>>>((const __nv_bfloat16*)qkv, (__nv_bfloat16*)o, lse, T, H,
                                                       scale_log2, use_alibi);
  } else {
    constexpr int NW = 4;
    const int shm = (16 * NW + 4 * 64) * DH * 2;
    auto k = attn_fwd_kernel<DH, NW>;
    FB_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, shm));
    k<<<dim3(T / (16 * NW), B * H), NW * 32, shm, st>>>((const __nv_bfloat16*)qkv, (__nv_bfloat16*)o, lse, T, H,
                                                       scale_log2, use_alibi);
  }
  FB_LAUNCH_CHECK();
  return FB_OK;
}

template <int DH>
int attn_bwd_tc_launch(const void* qkv, const void* dO, const float* lse, const float* Dbuf, float* dq, void* dqkv,
                       int B, int T, int H, int use_alibi, cudaStream_t st);

template <int DH>
static int attn_bwd_launch(const void* qkv, const void* o, const void* dO, const float* lse, void* dqkv, float* work,
                           int B, int T, int H, int use_alibi, cudaStream_t st) {
  const int d = H * DH;
  float* Dbuf = work;
  float* dq = work + (int64_t)B * H * T;
  const int nw = B * T * H;
  attn_bwd_dot_kernel<<<(nw + 7) / 8, 256, 0, st>>>((const __nv_bfloat16*)o, (const __nv_bfloat16*)dO, Dbuf, dq, B, T, H,
                                                    DH);
  FB_LAUNCH_CHECK();
  if (T % 128 == 0) {  // tcgen05 path
    int rc = attn_bwd_tc_launch<DH>(qkv, dO, lse, Dbuf, dq, dqkv, B, T, H, use_alibi, st);
    if (rc) return rc;
    dq_finalize_kernel<<<kNumSMs * 8, 256, 0, st>>>(dq, (__nv_bfloat16*)dqkv, B * T, d);
    FB_LAUNCH_CHECK();
    return FB_OK;
  }
  const int shm = 2 * 64 * DH * 2 + 4 * 64 * DH * 2 + 64 * 64 * 2 + 4 * 64 * 4;
  auto k = attn_bwd_kernel<DH>;
  FB_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, shm));
  const float scale = 1.0f / sqrtf((float)DH);
  k<<<dim3(T / 64, B * H), 128, shm, st>>>((const __nv_bfloat16*)qkv, (const __nv_bfloat16*)dO, lse, Dbuf, dq,
                                          (__nv_bfloat16*)dqkv, T, H, 1.4426950408889634f * scale, scale, use_alibi);
  FB_LAUNCH_CHECK();
  dq_finalize_kernel<<<kNumSMs * 8, 256, 0, st>>>(dq, (__nv_bfloat16*)dqkv, B * T, d);
  FB_LAUNCH_CHECK();
  return FB_OK;
}

}  // namespace fb

using namespace fb;

extern "C" int fb_attn_fwd(const void* d_qkv, void* d_o, float* d_lse, int B, int T, int H, int dh, int use_alibi,
                           void* stream) {
  FB_REQUIRE(B > 0 && H > 0 && T > 0 && T % 64 == 0, "attn_fwd: T must be a positive multiple of 64 (T=%d)", T);
  cudaStream_t st = (cudaStream_t)stream;
  // algorithmic flops: causal lower triangle, QK^T and PV (2*T*d per layer-token fwd)
  const double fl = 2.0 * 2.0 * B * H * (double)T * (T + 1) / 2.0 * dh;
  const int pi = prof_on() ? prof_start(1, st) : -1;
  int rc = FB_UNSUPPORTED;
  if (dh == 64) rc = attn_fwd_launch<64>(d_qkv, d_o, d_lse, B, T, H, use_alibi, st);
  else if (dh == 128) rc = attn_fwd_launch<128>(d_qkv, d_o, d_lse, B, T, H, use_alibi, st);
  prof_stop(1, pi, st, fl);
  if (rc != FB_UNSUPPORTED) return rc;
  set_error("attn_fwd: head dim %d unsupported (64 or 128)", dh);
  return FB_UNSUPPORTED;
}

extern "C" int fb_attn_bwd(const void* d_qkv, const void* d_o, const void* d_do, const float* d_lse, void* d_dqkv,
                           float* d_work, int B, int T, int H, int dh, int use_alibi, void* stream) {
  FB_REQUIRE(B > 0 && H > 0 && T > 0 && T % 64 == 0, "attn_bwd: T must be a positive multiple of 64 (T=%d)", T);
  FB_REQUIRE(d_work != nullptr, "attn_bwd: needs a work buffer of B*H*T + B*T*H*dh floats");
  cudaStream_t st = (cudaStream_t)stream;
  const double fl = 2.0 * 2.0 * 2.0 * B * H * (double)T * (T + 1) / 2.0 * dh;  // bwd = 2x fwd
  const int pi = prof_on() ? prof_start(2, st) : -1;
  int rc = FB_UNSUPPORTED;
  if (dh == 64) rc = attn_bwd_launch<64>(d_qkv, d_o, d_do, d_lse, d_dqkv, d_work, B, T, H, use_alibi, st);
  else if (dh == 128) rc = attn_bwd_launch<128>(d_qkv, d_o, d_do, d_lse, d_dqkv, d_work, B, T, H, use_alibi, st);
  prof_stop(2, pi, st, fl);
  if (rc != FB_UNSUPPORTED) return rc;
  set_error("attn_bwd: head dim %d unsupported (64 or 128)", dh);
  return FB_UNSUPPORTED;
}
