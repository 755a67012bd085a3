// Causal ALiBi attention on the CUDA cores, for the shapes the tcgen05 kernels do not
// tile: any head dim (the reference's desk / recipe configs use dh 4..32, fedforge
// configs/desk-small.json) and any sequence length (T % 128 != 0). Same math and the
// same base-2 lse convention as attn_tc.cu / attn_bwd_tc.cu, so either backward can
// follow either forward.
//
// Reference: fedforge/model.py:92-98 (scores = q k^T / sqrt(dh) + bias, softmax, PV),
// bias model.py:46-72 (slope_h = 2^(-8(h+1)/H), -slope (i-j) below the diagonal).
//
// One warp per (b, h, row). Lanes split the head dim (lane owns c = lane + 32 e), so a
// score is one warp reduction; keys (forward, dQ) or queries (dK/dV) are walked in
// ascending order, so every output is a fixed-order sum: the backward is deterministic
// (no atomics).
#include "common.cuh"

namespace fb {

constexpr float kLog2e = 1.4426950408889634f;

template <int NE>
__device__ __forceinline__ void load_head(const __nv_bfloat16* __restrict__ p, int dh, int lane, float (&x)[NE],
                                          float scale = 1.f) {
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const int c = lane + 32 * e;
    x[e] = c < dh ? __bfloat162float(p[c]) * scale : 0.f;
  }
}

template <int NE>
__device__ __forceinline__ float dot_head(const float (&a)[NE], const __nv_bfloat16* __restrict__ p, int dh,
                                          int lane) {
  float s = 0.f;
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const int c = lane + 32 * e;
    if (c < dh) s = fmaf(a[e], __bfloat162float(p[c]), s);
  }
  return warp_sum(s);
}

// o = softmax(q k^T * scale + bias) v ; lse2 = log2 sum exp2 of the base-2 scores
template <int NE>
__global__ void __launch_bounds__(256) attn_fwd_generic_kernel(const __nv_bfloat16* __restrict__ qkv,
                                                               __nv_bfloat16* __restrict__ o, float* __restrict__ lse2,
                                                               int B, int T, int H, int dh, int use_alibi) {
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (gw >= (int64_t)B * H * T) return;
  const int i = (int)(gw % T);
  const int bh = (int)(gw / T);
  const int h = bh % H, b = bh / H;
  const int d = H * dh;
  const int64_t ld = 3 * (int64_t)d;
  const __nv_bfloat16* base = qkv + (int64_t)b * T * ld + h * dh;
  const float sc = kLog2e / sqrtf((float)dh);
  const float sl = use_alibi ? exp2f(-8.0f * (float)(h + 1) / (float)H) * kLog2e : 0.f;
  float q[NE], acc[NE];
  load_head(base + (int64_t)i * ld, dh, lane, q, sc);
#pragma unroll
  for (int e = 0; e < NE; ++e) acc[e] = 0.f;
  float m = -INFINITY, l = 0.f;
  for (int j = 0; j <= i; ++j) {
    const __nv_bfloat16* kr = base + (int64_t)j * ld + d;
    const float s = dot_head(q, kr, dh, lane) - sl * (float)(i - j);
    const float mn = fmaxf(m, s);
    const float corr = exp2f(m - mn), p = exp2f(s - mn);
    l = l * corr + p;
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const int c = lane + 32 * e;
      acc[e] = acc[e] * corr + (c < dh ? p * __bfloat162float(kr[d + c]) : 0.f);
    }
    m = mn;
  }
  const float inv = 1.f / l;
  __nv_bfloat16* orow = o + ((int64_t)b * T + i) * d + h * dh;
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const int c = lane + 32 * e;
    if (c < dh) orow[c] = __float2bfloat16_rn(acc[e] * inv);
  }
  if (lane == 0) lse2[gw] = m + log2f(l);
}

// D[b][h][i] = sum_c dO * O (bf16 inputs, f32 sum)
__global__ void attn_rowdot_generic_kernel(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dO,
                                           float* __restrict__ D, int B, int T, int H, int dh) {
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (gw >= (int64_t)B * H * T) return;
  const int i = (int)(gw % T);
  const int bh = (int)(gw / T);
  const int h = bh % H, b = bh / H;
  const int64_t off = ((int64_t)b * T + i) * H * dh + h * dh;
  float s = 0.f;
  for (int c = lane; c < dh; c += 32) s = fmaf(__bfloat162float(o[off + c]), __bfloat162float(dO[off + c]), s);
  s = warp_sum(s);
  if (lane == 0) D[gw] = s;
}

// dQ_i = scale * sum_{j <= i} P_ij (dP_ij - D_i) k_j,   dP_ij = dO_i . v_j
template <int NE>
__global__ void __launch_bounds__(256) attn_bwd_dq_generic_kernel(const __nv_bfloat16* __restrict__ qkv,
                                                                  const __nv_bfloat16* __restrict__ dO,
                                                                  const float* __restrict__ lse2,
                                                                  const float* __restrict__ D,
                                                                  __nv_bfloat16* __restrict__ dqkv, int B, int T,
                                                                  int H, int dh, int use_alibi) {
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (gw >= (int64_t)B * H * T) return;
  const int i = (int)(gw % T);
  const int bh = (int)(gw / T);
  const int h = bh % H, b = bh / H;
  const int d = H * dh;
  const int64_t ld = 3 * (int64_t)d;
  const __nv_bfloat16* base = qkv + (int64_t)b * T * ld + h * dh;
  const float sc = kLog2e / sqrtf((float)dh);
  const float sl = use_alibi ? exp2f(-8.0f * (float)(h + 1) / (float)H) * kLog2e : 0.f;
  float q[NE], g[NE], acc[NE];
  load_head(base + (int64_t)i * ld, dh, lane, q, sc);
  load_head(dO + ((int64_t)b * T + i) * d + h * dh, dh, lane, g);
#pragma unroll
  for (int e = 0; e < NE; ++e) acc[e] = 0.f;
  const float lse = lse2[gw], Di = D[gw];
  for (int j = 0; j <= i; ++j) {
    const __nv_bfloat16* kr = base + (int64_t)j * ld + d;
    const float p = exp2f(dot_head(q, kr, dh, lane) - sl * (float)(i - j) - lse);
    const float ds = p * (dot_head(g, kr + d, dh, lane) - Di);
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const int c = lane + 32 * e;
      if (c < dh) acc[e] = fmaf(ds, __bfloat162float(kr[c]), acc[e]);
    }
  }
  const float scale = 1.f / sqrtf((float)dh);
  __nv_bfloat16* out = dqkv + ((int64_t)b * T + i) * ld + h * dh;
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const int c = lane + 32 * e;
    if (c < dh) out[c] = __float2bfloat16_rn(acc[e] * scale);
  }
}

// dK_j = scale * sum_{i >= j} dS_ij q_i ,  dV_j = sum_{i >= j} P_ij dO_i
template <int NE>
__global__ void __launch_bounds__(256) attn_bwd_dkdv_generic_kernel(const __nv_bfloat16* __restrict__ qkv,
                                                                    const __nv_bfloat16* __restrict__ dO,
                                                                    const float* __restrict__ lse2,
                                                                    const float* __restrict__ D,
                                                                    __nv_bfloat16* __restrict__ dqkv, int B, int T,
                                                                    int H, int dh, int use_alibi) {
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (gw >= (int64_t)B * H * T) return;
  const int j = (int)(gw % T);
  const int bh = (int)(gw / T);
  const int h = bh % H, b = bh / H;
  const int d = H * dh;
  const int64_t ld = 3 * (int64_t)d;
  const __nv_bfloat16* base = qkv + (int64_t)b * T * ld + h * dh;
  const __nv_bfloat16* gbase = dO + (int64_t)b * T * d + h * dh;
  const float sc = kLog2e / sqrtf((float)dh);
  const float sl = use_alibi ? exp2f(-8.0f * (float)(h + 1) / (float)H) * kLog2e : 0.f;
  float k[NE], v[NE], dk[NE], dv[NE];
  load_head(base + (int64_t)j * ld + d, dh, lane, k, sc);
  load_head(base + (int64_t)j * ld + 2 * d, dh, lane, v);
#pragma unroll
  for (int e = 0; e < NE; ++e) dk[e] = dv[e] = 0.f;
  const int64_t bh0 = (int64_t)bh * T;
  for (int i = j; i < T; ++i) {
    const __nv_bfloat16* qr = base + (int64_t)i * ld;
    const __nv_bfloat16* gr = gbase + (int64_t)i * d;
    const float p = exp2f(dot_head(k, qr, dh, lane) - sl * (float)(i - j) - lse2[bh0 + i]);
    const float ds = p * (dot_head(v, gr, dh, lane) - D[bh0 + i]);
#pragma unroll
    for (int e = 0; e < NE; ++e) {
      const int c = lane + 32 * e;
      if (c < dh) {
        dv[e] = fmaf(p, __bfloat162float(gr[c]), dv[e]);
        dk[e] = fmaf(ds, __bfloat162float(qr[c]), dk[e]);
      }
    }
  }
  const float scale = 1.f / sqrtf((float)dh);
  __nv_bfloat16* out = dqkv + ((int64_t)b * T + j) * ld + h * dh;
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const int c = lane + 32 * e;
    if (c < dh) {
      out[d + c] = __float2bfloat16_rn(dk[e] * scale);
      out[2 * d + c] = __float2bfloat16_rn(dv[e]);
    }
  }
}

#define FB_GENERIC_NE(dh, CALL)  \
  do {                           \
    if ((dh) <= 32) {            \
      CALL(1);                   \
    } else if ((dh) <= 64) {     \
      CALL(2);                   \
    } else if ((dh) <= 128) {    \
      CALL(4);                   \
    } else {                     \
      CALL(8);                   \
    }                            \
  } while (0)

int attn_fwd_generic(const void* qkv, void* o, float* lse, int B, int T, int H, int dh, int use_alibi,
                     cudaStream_t st) {
  FB_REQUIRE(dh >= 1 && dh <= 256, "attn: head dim %d outside [1, 256]", dh);
  const int64_t rows = (int64_t)B * H * T;
  const int grid = (int)((rows + 7) / 8);
#define CALL(NE)                                                                                          \
  attn_fwd_generic_kernel<NE><<<grid, 256, 0, st>>>((const __nv_bfloat16*)qkv, (__nv_bfloat16*)o, lse, B, T, \
                                                    H, dh, use_alibi)
  FB_GENERIC_NE(dh, CALL);
#undef CALL
  FB_LAUNCH_CHECK();
  return FB_OK;
}

// D (work[0 : B*H*T]) is recomputed here unless the caller says it is ready
int attn_bwd_generic(const void* qkv, const void* o, const void* dO, const float* lse, void* dqkv, float* work, int B,
                     int T, int H, int dh, int use_alibi, int d_ready, cudaStream_t st) {
  FB_REQUIRE(dh >= 1 && dh <= 256, "attn: head dim %d outside [1, 256]", dh);
  const int64_t rows = (int64_t)B * H * T;
  const int grid = (int)((rows + 7) / 8);
  if (!d_ready) {
    attn_rowdot_generic_kernel<<<grid, 256, 0, st>>>((const __nv_bfloat16*)o, (const __nv_bfloat16*)dO, work, B, T,
                                                     H, dh);
    FB_LAUNCH_CHECK();
  }
#define CALL(NE)                                                                                             \
  attn_bwd_dq_generic_kernel<NE><<<grid, 256, 0, st>>>((const __nv_bfloat16*)qkv, (const __nv_bfloat16*)dO, lse, \
                                                       work, (__nv_bfloat16*)dqkv, B, T, H, dh, use_alibi);     \
  attn_bwd_dkdv_generic_kernel<NE><<<grid, 256, 0, st>>>((const __nv_bfloat16*)qkv, (const __nv_bfloat16*)dO,     \
                                                         lse, work, (__nv_bfloat16*)dqkv, B, T, H, dh, use_alibi)
  FB_GENERIC_NE(dh, CALL);
#undef CALL
  FB_LAUNCH_CHECK();
  return FB_OK;
}

}  // namespace fb
