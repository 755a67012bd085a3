// Dense bf16 GEMM on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// Replaces every nn.Linear of the reference TinyLM (fedforge/model.py:82-86, :114)
// in forward (X W^T), dgrad (dY W) and wgrad (dY^T X) form, with the elementwise
// work that follows each one fused into the TMEM drain (GELU-erf, dGELU, residual
// add, fp32 wgrad accumulation across micro-batches).
//
// Kernel anatomy (persistent, warp-specialised, one CTA per SM):
//   warp 0      TMA producer: STAGES-deep ring of {A 128x64, B BNx64} bf16 tiles,
//               128B-swizzled, K-major or MN-major (3-D tensor map so an MN-major
//               tile is a single TMA), completion via mbarrier expect_tx
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (128xBNx16 UMMAs),
//               tcgen05.commit frees smem slots / publishes finished accumulators
//   warps 2-9   epilogue (two warps per TMEM lane quadrant, one column half each):
//               tcgen05.ld 32x32b.x32 -> registers -> fused op (packed f32x2 math) ->
//               swizzled smem staging -> TMA bulk tensor store
//   TMEM        2 x BN fp32 columns: the accumulator is double-buffered so the
//               epilogue of tile i overlaps the main loop of tile i+1
// The 2-SM variant (gemm_bf16_tc2_kernel, cta_group::2, 256 x 256 tiles) is used whenever
// its tiles fill the 74 CTA pairs; ragged last waves are split along K (last-wave split).
// D = rowsum(dO o O) of the attention backward can ride on the out-projection dgrad
// epilogue (FB_EPI_BF16_ROWDOT).
#include <cudaTypedefs.h>
#include <stdlib.h>

#include "common.cuh"
#include "sm100.cuh"

namespace fb {
using namespace sm100;

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int kGemmThreads = 320;  // TMA warp, MMA warp, 8 epilogue warps (2 per TMEM lane quadrant)

template <int BN>
struct GemmCfg {
  static constexpr int STAGES = BN == 256 ? 4 : 6;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*barriers*/ + 1024 /*align slack*/;
  static constexpr int TMEM_COLS = 2 * BN;
};

// Grouped raster: tiles walk GROUP_M m-blocks at a time (m fastest), so the ~148 concurrently
// resident tiles touch GROUP_M A blocks and a few B blocks that stay L2-resident.
constexpr int kGroupM = 16;
__device__ __forceinline__ void tile_coords(int tile, int num_m, int num_n, int& mb, int& nb, int kGroupM = 16) {
  const int group_size = kGroupM * num_n;
  const int g = tile / group_size;
  const int first_m = g * kGroupM;
  const int gm = min(num_m - first_m, kGroupM);
  const int idx = tile - g * group_size;
  mb = first_m + idx % gm;
  nb = idx / gm;
}

struct EpiArgs {
  void* C;
  int64_t ldc;
  const void* aux;
  void* aux_out;
  int64_t ld_aux;
  int ksplit;            // > 1: work unit u = (split, tile); split s writes C + s * split_stride
  int64_t split_stride;  // elements
  // Last-wave split (2-SM kernel only; tail_split > 1 enables it): tiles [0, full_tiles) are
  // whole-K units that fill complete waves of the 74 CTA pairs; each remaining tile is cut
  // into tail_split K ranges whose raw f32 partials go to a [piece][256][256] workspace,
  // reduced in fixed order by tail_reduce_kernel (deterministic).
  int full_tiles;
  int tail_split;
  void* tail_ws;         // f32 [pieces][256][256]
  int units;             // work units of the launch
  int group_m;           // raster group height (2-SM kernel)
  int rd_T, rd_dh;       // FB_EPI_BF16_ROWDOT: sequence length, head dim
  // MN-major operand whose MN extent is not a multiple of 64 (1-SM kernel only): its map is
  // 2-D {mn, K} and each 64-wide MN chunk of a stage is its own TMA, so the chunks past mn
  // are zero-filled by the TMA bounds check instead of reading the next K row
  int a_2d, b_2d;
};

// work unit -> (tile, first k-block, k-block count, tail piece or -1), 2-SM kernel
__device__ __forceinline__ void unit_coords2(int u, int num_tiles, int num_kb, const EpiArgs& e, int& tile, int& kb0,
                                             int& nkb, int& piece) {
  if (e.tail_split > 1) {
    piece = -1;
    if (u < e.full_tiles) {
      tile = u;
      kb0 = 0;
      nkb = num_kb;
      return;
    }
    const int v = u - e.full_tiles;
    tile = e.full_tiles + v / e.tail_split;
    const int per = (num_kb + e.tail_split - 1) / e.tail_split;
    kb0 = (v % e.tail_split) * per;
    nkb = min(num_kb, kb0 + per) - kb0;
    piece = v;
    return;
  }
  tile = u % num_tiles;
  const int sp = u / num_tiles;
  const int per = (num_kb + e.ksplit - 1) / e.ksplit;
  kb0 = sp * per;
  nkb = min(num_kb, kb0 + per) - kb0;
  piece = -1;
}

// work unit -> (tile, first k-block, k-block count)
__device__ __forceinline__ void unit_coords(int u, int num_tiles, int num_kb, int ksplit, int& tile, int& kb0, int& nkb) {
  tile = u % num_tiles;
  const int s = u / num_tiles;
  const int per = (num_kb + ksplit - 1) / ksplit;
  kb0 = s * per;
  nkb = min(num_kb, kb0 + per) - kb0;
}

// Exact-erf GELU (reference: F.gelu, fedforge/model.py:101) on the FMA pipe.
// Phi(x) = 1 - h (x >= 0) or h (x < 0), h = erfc(|x|/sqrt2)/2 from the Chebyshev-fitted
// erfc of Numerical Recipes (relative error < 1.2e-7 everywhere, i.e. float-exact):
//   erfc(z) = t exp(-z^2 + P(t)), t = 1 / (1 + z/2)
// with log2(e) and the 1/2 folded into P's coefficients so exp is one ex2. About half the
// instructions of erff(), which mattered: the GELU GEMM runs at the power cap.
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float norm_cdf(float x) {
  const float t = rcp_approx(fmaf(fabsf(x), 0.353553391f, 1.0f));  // 1 / (1 + |x| / (2 sqrt2))
  float q = 0.246517298f;
  q = fmaf(q, t, -1.18611495f);
  q = fmaf(q, t, 2.14747446f);
  q = fmaf(q, t, -1.63775315f);
  q = fmaf(q, t, 0.402321582f);
  q = fmaf(q, t, -0.26875686f);
  q = fmaf(q, t, 0.139630057f);
  q = fmaf(q, t, 0.539700616f);
  q = fmaf(q, t, 1.4427292f);
  q = fmaf(q, t, -2.82574822f);                          // log2(e) * c0 - 1  (the 1/2)
  const float h = t * ex2_approx(fmaf(x * x, -0.72134752f, q));  // - z^2 log2(e), z^2 = x^2 / 2
  return x >= 0.f ? 1.0f - h : h;
}
__device__ __forceinline__ float gelu_erf(float x) { return x * norm_cdf(x); }
__device__ __forceinline__ float gelu_erf_grad(float x) {
  // Phi(x) + x phi(x), phi(x) = exp(-x^2/2) / sqrt(2 pi)
  return fmaf(x, ex2_approx(fmaf(x * x, -0.72134752f, -1.32574806f)), norm_cdf(x));
}

// Pair forms on the packed f32x2 pipe (FFMA2 / FMUL2, sm_100): each lane rounds exactly like
// the scalar FFMA / FMUL above, so the results are bit-identical, at about 60% of the issue
// slots. The fused GELU / dGELU GEMMs are epilogue-heavy and run at the power cap.
__device__ __forceinline__ float2 f2_fma(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(r)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
        "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return *reinterpret_cast<float2*>(&r);
}
__device__ __forceinline__ float2 f2_mul(float2 a, float2 b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;"
      : "=l"(r)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)));
  return *reinterpret_cast<float2*>(&r);
}
__device__ __forceinline__ float2 f2s(float c) { return make_float2(c, c); }
// Phi(x) for two values; xx = x * x (shared with the dGELU density term)
__device__ __forceinline__ float2 norm_cdf2(float2 x, float2 xx) {
  const float2 t = make_float2(rcp_approx(fmaf(fabsf(x.x), 0.353553391f, 1.0f)),
                               rcp_approx(fmaf(fabsf(x.y), 0.353553391f, 1.0f)));
  float2 q = f2_fma(f2s(0.246517298f), t, f2s(-1.18611495f));
  q = f2_fma(q, t, f2s(2.14747446f));
  q = f2_fma(q, t, f2s(-1.63775315f));
  q = f2_fma(q, t, f2s(0.402321582f));
  q = f2_fma(q, t, f2s(-0.26875686f));
  q = f2_fma(q, t, f2s(0.139630057f));
  q = f2_fma(q, t, f2s(0.539700616f));
  q = f2_fma(q, t, f2s(1.4427292f));
  q = f2_fma(q, t, f2s(-2.82574822f));
  const float2 a = f2_fma(xx, f2s(-0.72134752f), q);
  const float2 h = f2_mul(t, make_float2(ex2_approx(a.x), ex2_approx(a.y)));
  return make_float2(x.x >= 0.f ? 1.0f - h.x : h.x, x.y >= 0.f ? 1.0f - h.y : h.y);
}
__device__ __forceinline__ float2 gelu_erf2(float2 x) { return f2_mul(x, norm_cdf2(x, f2_mul(x, x))); }
#ifndef FB_EXP_DGELU3
// gelu'(x) = Phi(x) + x phi(x) with ONE shared exponential E = 2^(-x^2 log2(e) / 2): phi = E / sqrt(2 pi)
// and h = t E R(t), where R(t) = 2^P(t) of the erfc fit above is itself fitted as a degree-10
// polynomial in t (f32 Horner, relative error <= 2.4e-7 on t in [0, 1]): 2 MUFU ops per value
// (rcp, ex2) instead of 3 — the dGELU GEMM's epilogue is MUFU-heavy.
__device__ __forceinline__ float2 gelu_erf_grad2(float2 x) {
  const float2 xx = f2_mul(x, x);
  const float2 a = f2_mul(xx, f2s(-0.72134752f));
  const float2 E = make_float2(ex2_approx(a.x), ex2_approx(a.y));
  const float2 t = make_float2(rcp_approx(fmaf(fabsf(x.x), 0.353553391f, 1.0f)),
                               rcp_approx(fmaf(fabsf(x.y), 0.353553391f, 1.0f)));
  float2 r = f2_fma(f2s(0.0160564873f), t, f2s(-0.0902611241f));
  r = f2_fma(r, t, f2s(0.190638140f));
  r = f2_fma(r, t, f2s(-0.163145512f));
  r = f2_fma(r, t, f2s(0.0217379313f));
  r = f2_fma(r, t, f2s(-0.0107644396f));
  r = f2_fma(r, t, f2s(0.0418829955f));
  r = f2_fma(r, t, f2s(0.0883701667f));
  r = f2_fma(r, t, f2s(0.123389557f));
  r = f2_fma(r, t, f2s(0.141048372f));
  r = f2_fma(r, t, f2s(0.141047388f));
  const float2 h = f2_mul(f2_mul(t, E), r);
  const float2 phi = make_float2(x.x >= 0.f ? 1.0f - h.x : h.x, x.y >= 0.f ? 1.0f - h.y : h.y);
  return f2_fma(f2_mul(x, f2s(0.398942280f)), E, phi);
}
#else
__device__ __forceinline__ float2 gelu_erf_grad2(float2 x) {
  const float2 xx = f2_mul(x, x);
  const float2 a = f2_fma(xx, f2s(-0.72134752f), f2s(-1.32574806f));
  return f2_fma(x, make_float2(ex2_approx(a.x), ex2_approx(a.y)), norm_cdf2(x, xx));
}
#endif

// FB_EPI_CE_EXP (LM head + cross-entropy, model.py:226-229): the 32 logits of this chunk
// become e = exp(x - m) with m the chunk max (so e in (0, 1] keeps bf16 precision), and the
// chunk's (m, sum e) pair goes to aux_out[(col / 32) * M + row] (a warp's 32 rows are
// contiguous). The f32 logits never reach HBM; fb_lmhead_ce turns the pairs into the row's
// log-sum-exp and rescales e into the gradient in place.
__device__ __forceinline__ void ce_exp_chunk(const EpiArgs& e, int64_t row, bool in, int col, int N, float (&v)[32]) {
  constexpr float kL2e = 1.4426950408889634f;
  float m = -INFINITY;
#pragma unroll
  for (int i = 0; i < 32; ++i) m = (col + i < N) ? fmaxf(m, v[i]) : m;
  const float ml = m * kL2e;
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const float x = (col + i < N) ? ex2_approx(fmaf(v[i], kL2e, -ml)) : 0.f;
    v[i] = x;
    s += x;
  }
  if (in) reinterpret_cast<float2*>(e.aux_out)[(int64_t)(col >> 5) * e.ld_aux + row] = make_float2(m, s);
}

// Process 32 consecutive columns [col, col+32) of one row held in registers.
template <int EPI>
__device__ __forceinline__ void epilogue_chunk(const EpiArgs& e, int64_t row, int col, int N, const uint32_t (&r)[32]) {
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
  const bool full = col + 32 <= N;
  if constexpr (EPI == FB_EPI_CE_EXP) ce_exp_chunk(e, row, true, col, N, v);
  if constexpr (EPI == FB_EPI_BF16 || EPI == FB_EPI_GELU || EPI == FB_EPI_DGELU || EPI == FB_EPI_CE_EXP) {
    __nv_bfloat16* C = reinterpret_cast<__nv_bfloat16*>(e.C) + row * e.ldc + col;
    float o[32];
    if constexpr (EPI == FB_EPI_GELU) {
      __nv_bfloat16* P = reinterpret_cast<__nv_bfloat16*>(e.aux_out) + row * e.ld_aux + col;
      if (full) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 pk = make_uint4(pack_bf16(v[8 * q], v[8 * q + 1]), pack_bf16(v[8 * q + 2], v[8 * q + 3]),
                                pack_bf16(v[8 * q + 4], v[8 * q + 5]), pack_bf16(v[8 * q + 6], v[8 * q + 7]));
          *reinterpret_cast<uint4*>(P + 8 * q) = pk;
        }
      } else {
        _Pragma("unroll") for (int i = 0; i < 32; ++i) if (col + i < N) P[i] = __float2bfloat16_rn(v[i]);
      }
      // GELU of the bf16-rounded pre-activation so forward and backward see the same input
#pragma unroll
      for (int i = 0; i < 32; ++i) o[i] = gelu_erf(__bfloat162float(__float2bfloat16_rn(v[i])));
    } else if constexpr (EPI == FB_EPI_DGELU) {
      const __nv_bfloat16* P = reinterpret_cast<const __nv_bfloat16*>(e.aux) + row * e.ld_aux + col;
      if (full) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 pk = *reinterpret_cast<const uint4*>(P + 8 * q);
          const __nv_bfloat16* pb = reinterpret_cast<const __nv_bfloat16*>(&pk);
#pragma unroll
          for (int i = 0; i < 8; ++i) o[8 * q + i] = v[8 * q + i] * gelu_erf_grad(__bfloat162float(pb[i]));
        }
      } else {
        _Pragma("unroll") for (int i = 0; i < 32; ++i) o[i] = (col + i < N) ? v[i] * gelu_erf_grad(__bfloat162float(P[i])) : 0.f;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) o[i] = v[i];
    }
    if (full) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 pk = make_uint4(pack_bf16(o[8 * q], o[8 * q + 1]), pack_bf16(o[8 * q + 2], o[8 * q + 3]),
                              pack_bf16(o[8 * q + 4], o[8 * q + 5]), pack_bf16(o[8 * q + 6], o[8 * q + 7]));
        *reinterpret_cast<uint4*>(C + 8 * q) = pk;
      }
    } else {
      _Pragma("unroll") for (int i = 0; i < 32; ++i) if (col + i < N) C[i] = __float2bfloat16_rn(o[i]);
    }
  } else {
    float* C = reinterpret_cast<float*>(e.C) + row * e.ldc + col;
    if constexpr (EPI == FB_EPI_ACC_F32) {
      if (full) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          float4 c = *reinterpret_cast<const float4*>(C + 4 * q);
          v[4 * q] += c.x; v[4 * q + 1] += c.y; v[4 * q + 2] += c.z; v[4 * q + 3] += c.w;
        }
      } else {
        _Pragma("unroll") for (int i = 0; i < 32; ++i) if (col + i < N) v[i] += C[i];
      }
    } else if constexpr (EPI == FB_EPI_RESID_F32 || EPI == FB_EPI_RESID_F32_BF16) {
      const float* R = reinterpret_cast<const float*>(e.aux) + row * e.ld_aux + col;
      if (full) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          float4 c = *reinterpret_cast<const float4*>(R + 4 * q);
          v[4 * q] += c.x; v[4 * q + 1] += c.y; v[4 * q + 2] += c.z; v[4 * q + 3] += c.w;
        }
      } else {
        _Pragma("unroll") for (int i = 0; i < 32; ++i) if (col + i < N) v[i] += R[i];
      }
      if constexpr (EPI == FB_EPI_RESID_F32_BF16) {
        __nv_bfloat16* Ob = reinterpret_cast<__nv_bfloat16*>(e.aux_out) + row * e.ldc + col;
        if (full) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 pk = make_uint4(pack_bf16(v[8 * q], v[8 * q + 1]), pack_bf16(v[8 * q + 2], v[8 * q + 3]),
                                  pack_bf16(v[8 * q + 4], v[8 * q + 5]), pack_bf16(v[8 * q + 6], v[8 * q + 7]));
            *reinterpret_cast<uint4*>(Ob + 8 * q) = pk;
          }
        } else {
          _Pragma("unroll") for (int i = 0; i < 32; ++i) if (col + i < N) Ob[i] = __float2bfloat16_rn(v[i]);
        }
      }
    }
    if (full) {
#pragma unroll
      for (int q = 0; q < 8; ++q)
        *reinterpret_cast<float4*>(C + 4 * q) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    } else {
      _Pragma("unroll") for (int i = 0; i < 32; ++i) if (col + i < N) C[i] = v[i];
    }
  }
}

template <int BN, int A_MN, int B_MN, int EPI>
__global__ void __launch_bounds__(kGemmThreads, 1)
    gemm_bf16_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M,
                        int N, int K, EpiArgs ep) {
  using Cfg = GemmCfg<BN>;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023) & ~1023u) - raw_addr);
  uint8_t* tiles = smem;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_m = (M + BM - 1) / BM;
  const int num_n = (N + BN - 1) / BN;
  const int num_tiles = num_m * num_n;
  const int num_kb = (K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 8);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      int stage = 0;
      uint32_t phase = 0;
      for (int u = blockIdx.x; u < num_tiles * ep.ksplit; u += gridDim.x) {
        int tile, kb0, nkb;
        unit_coords(u, num_tiles, num_kb, ep.ksplit, tile, kb0, nkb);
        int mb, nb;
        tile_coords(tile, num_m, num_n, mb, nb);
        const int m0 = mb * BM;
        const int n0 = nb * BN;
        for (int kb = kb0; kb < kb0 + nkb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = tiles + stage * Cfg::STAGE_BYTES;
          uint8_t* sb = sa + Cfg::A_BYTES;
          mbar_arrive_expect_tx(&full_bar[stage], Cfg::STAGE_BYTES);
          const int k0 = kb * BK;
          if (A_MN && ep.a_2d) {
            for (int c = 0; c < BM / 64; ++c) tma_load_2d(sa + c * (64 * BK * 2), &tmA, &full_bar[stage], m0 + 64 * c, k0);
          } else if (A_MN) {
            tma_load_3d(sa, &tmA, &full_bar[stage], 0, k0, m0 / 64);
          } else {
            tma_load_2d(sa, &tmA, &full_bar[stage], k0, m0);
          }
          if (B_MN && ep.b_2d) {
            for (int c = 0; c < BN / 64; ++c) tma_load_2d(sb + c * (64 * BK * 2), &tmB, &full_bar[stage], n0 + 64 * c, k0);
          } else if (B_MN) {
            tma_load_3d(sb, &tmB, &full_bar[stage], 0, k0, n0 / 64);
          } else {
            tma_load_2d(sb, &tmB, &full_bar[stage], k0, n0);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t idesc = idesc_bf16_f32(BM, BN, A_MN, B_MN);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int u = blockIdx.x; u < num_tiles * ep.ksplit; u += gridDim.x, ++it) {
      int tile, kb0, nkb;
      unit_coords(u, num_tiles, num_kb, ep.ksplit, tile, kb0, nkb);
      const int buf = it & 1;
      const uint32_t use = it >> 1;
      mbar_wait(&tempty_bar[buf], (use & 1) ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_base + buf * BN;
      for (int kb = 0; kb < nkb; ++kb) {
        mbar_wait(&full_bar[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t sa = smem_u32(tiles + stage * Cfg::STAGE_BYTES);
          const uint32_t sb = sa + Cfg::A_BYTES;
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            // K-major SW128: rows 128B apart, 8-row atoms SBO=1024; k-step = +32B
            // MN-major SW128: 64-elem MN chunks LBO=64*128B, 8-k-row groups SBO=1024; k-step = +2048B
            const uint64_t ad = A_MN ? smem_desc_sw128(sa + kk * 2048, BK * 128, 1024)
                                     : smem_desc_sw128(sa + kk * 32, 16, 1024);
            const uint64_t bd = B_MN ? smem_desc_sw128(sb + kk * 2048, BK * 128, 1024)
                                     : smem_desc_sw128(sb + kk * 32, 16, 1024);
            umma_f16(d_tmem, ad, bd, idesc, (kb | kk) != 0);
          }
          umma_commit(&empty_bar[stage]);
        }
        __syncwarp();
        if (++stage == STAGES) { stage = 0; phase ^= 1; }
      }
      if (lane == 0) umma_commit(&tfull_bar[buf]);
      __syncwarp();
    }
  } else {
    // ---------------- epilogue warps 2..9: quadrant = warp & 3, column half = (warp - 2) >> 2 ----------------
    const int quad = warp & 3;  // TMEM lane quadrant this warp may access
    const int half = (warp - 2) >> 2;
    int it = 0;
    for (int u = blockIdx.x; u < num_tiles * ep.ksplit; u += gridDim.x, ++it) {
      int tile, kb0, nkb;
      unit_coords(u, num_tiles, num_kb, ep.ksplit, tile, kb0, nkb);
      EpiArgs eu = ep;
      eu.C = (char*)ep.C + (u / num_tiles) * ep.split_stride *
                               (EPI == FB_EPI_BF16 || EPI == FB_EPI_GELU || EPI == FB_EPI_DGELU || EPI == FB_EPI_CE_EXP ? 2 : 4);
      int mb, nb;
      tile_coords(tile, num_m, num_n, mb, nb);
      const int m0 = mb * BM;
      const int n0 = nb * BN;
      const int buf = it & 1;
      const uint32_t use = it >> 1;
      mbar_wait(&tfull_bar[buf], use & 1);
      tc_fence_after();
      const int64_t row = m0 + quad * 32 + lane;
      const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + buf * BN + half * (BN / 2);
#pragma unroll 1
      for (int c = 0; c < BN / 64; ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(taddr + c * 32, r);
        tmem_ld_wait();
        if (c == BN / 64 - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty_bar[buf]);
        }
        const int col = n0 + half * (BN / 2) + c * 32;
        if (row < M && col < N) epilogue_chunk<EPI>(eu, row, col, N, r);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
  }
}

// ---------------------------------------------------------------------------------------
// TMA-store epilogue (2-SM kernel). Each epilogue warp owns a 4 KB staging tile in smem:
// its 32 TMEM lanes (= 32 output rows) x one 32-column chunk, written with 16-byte
// st.shared in the swizzle the output tensor map uses (f32: 128 B rows, SWIZZLE_128B;
// bf16: 64 B rows, SWIZZLE_64B -> conflict-free), then ONE cp.async.bulk.tensor store per
// chunk and output. The TMA engine writes whole lines and clips the M / N tails, so the
// warps never issue per-row global stores. The previous chunk's store drains (read side)
// while the next chunk is pulled from TMEM and computed.
constexpr int kStageEpi = 4096;

__device__ __forceinline__ void stg_put_f32(uint8_t* stg, int r, int j, float a, float b, float c, float d) {
  *reinterpret_cast<float4*>(stg + r * 128 + ((j ^ (r & 7)) << 4)) = make_float4(a, b, c, d);
}
__device__ __forceinline__ void stg_put_bf16(uint8_t* stg, int r, int j, const float* f) {
  *reinterpret_cast<uint4*>(stg + r * 64 + ((j ^ ((r >> 1) & 3)) << 4)) =
      make_uint4(pack_bf16(f[0], f[1]), pack_bf16(f[2], f[3]), pack_bf16(f[4], f[5]), pack_bf16(f[6], f[7]));
}

struct EpiMaps {
  CUtensorMap C;     // {N, M, splits} box {32, 32, 1}
  CUtensorMap Aux;   // bf16 second output (GELU pre-activation, RESID_F32_BF16 copy), {N, M, 1}
  CUtensorMap Part;  // f32 last-wave partials {256, 256, pieces} box {32, 32, 1}
};

// Raw f32 accumulator chunk -> last-wave partial workspace (no epilogue op).
__device__ __forceinline__ void partial_chunk_tma(const CUtensorMap* map, uint8_t* stg, int lane, int x, int y, int z,
                                                  const uint32_t (&r)[32]) {
  if (lane == 0) bulk_wait_read<0>();
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 8; ++j)
    stg_put_f32(stg, lane, j, __uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]), __uint_as_float(r[4 * j + 2]),
                __uint_as_float(r[4 * j + 3]));
  fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) {
    tma_store_3d(map, stg, x, y, z);
    bulk_commit();
  }
}

// Per-row epilogue inputs that do not depend on the accumulator (dGELU pre-activation,
// residual stream): loaded for the NEXT chunk (and the tile's first chunk before its
// accumulator is ready), so the load latency hides behind the current chunk / the main loop.
// At C2 / C3 widths (K = 512 / 768) the main loop of a tile is short and the epilogue with
// an exposed ~1 us load per chunk was the bound.
template <int EPI>
constexpr bool kEpiPrefetch = EPI == FB_EPI_DGELU || EPI == FB_EPI_RESID_F32 || EPI == FB_EPI_RESID_F32_BF16;
template <int EPI>
__device__ __forceinline__ void epi_prefetch(const EpiArgs& e, int64_t row, int col, int M, int N, uint4 (&pf)[8]) {
  if constexpr (kEpiPrefetch<EPI>) {
    if (row < M && col + 32 <= N) {
      if constexpr (EPI == FB_EPI_DGELU) {
        const uint4* P = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(e.aux) + row * e.ld_aux + col);
#pragma unroll
        for (int q = 0; q < 4; ++q) pf[q] = P[q];
      } else {
        const uint4* R = reinterpret_cast<const uint4*>(reinterpret_cast<const float*>(e.aux) + row * e.ld_aux + col);
#pragma unroll
        for (int q = 0; q < 8; ++q) pf[q] = R[q];
      }
    }
  }
}

// One 32-column chunk of one warp: lane = row (row0 + lane), r[] = TMEM accumulator values.
template <int EPI>
__device__ __forceinline__ void epilogue_chunk_tma(const EpiArgs& e, const EpiMaps& mp, uint8_t* stg, int lane,
                                                   int64_t row, int row0, int col, int split, int M, int N,
                                                   const uint32_t (&r)[32], float& rd, const uint4 (&pf)[8]) {
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
  const bool in = row < M;
  const bool full = col + 32 <= N;
  // ---- inputs (per-row reads; the M / N tails read nothing) ----
  if constexpr (EPI == FB_EPI_ACC_F32 || EPI == FB_EPI_RESID_F32 || EPI == FB_EPI_RESID_F32_BF16) {
    const float* R = EPI == FB_EPI_ACC_F32 ? reinterpret_cast<const float*>(e.C) + row * e.ldc + col
                                           : reinterpret_cast<const float*>(e.aux) + row * e.ld_aux + col;
    if (in && full) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 c = EPI == FB_EPI_ACC_F32 ? *reinterpret_cast<const float4*>(R + 4 * q)
                                               : *reinterpret_cast<const float4*>(&pf[q]);
        v[4 * q] += c.x; v[4 * q + 1] += c.y; v[4 * q + 2] += c.z; v[4 * q + 3] += c.w;
      }
    } else if (in) {
      _Pragma("unroll") for (int i = 0; i < 32; ++i) if (col + i < N) v[i] += R[i];
    }
  }
  if constexpr (EPI == FB_EPI_CE_EXP) ce_exp_chunk(e, row, in, col, N, v);
  uint32_t pre[16];  // GELU: bf16 pre-activation pairs (stored as aux_out; gelu sees the rounded value)
  if constexpr (EPI == FB_EPI_GELU) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      pre[i] = pack_bf16(v[2 * i], v[2 * i + 1]);
#ifdef FB_EXP_GELU_ID
      const float2 g = make_float2(__uint_as_float(pre[i] << 16), __uint_as_float(pre[i] & 0xFFFF0000u));
#else
      const float2 g = gelu_erf2(make_float2(__uint_as_float(pre[i] << 16), __uint_as_float(pre[i] & 0xFFFF0000u)));
#endif
      v[2 * i] = g.x;
      v[2 * i + 1] = g.y;
    }
  } else if constexpr (EPI == FB_EPI_DGELU) {
    const __nv_bfloat16* P = reinterpret_cast<const __nv_bfloat16*>(e.aux) + row * e.ld_aux + col;
    if (in && full) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 pk = pf[q];
        const __nv_bfloat16* pb = reinterpret_cast<const __nv_bfloat16*>(&pk);
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
#ifdef FB_EXP_GELU_ID
          const float2 g = make_float2(__bfloat162float(pb[i]), __bfloat162float(pb[i + 1]));
#else
          const float2 g = gelu_erf_grad2(make_float2(__bfloat162float(pb[i]), __bfloat162float(pb[i + 1])));
#endif
          const float2 o = f2_mul(make_float2(v[8 * q + i], v[8 * q + i + 1]), g);
          v[8 * q + i] = o.x;
          v[8 * q + i + 1] = o.y;
        }
      }
    } else {
      _Pragma("unroll") for (int i = 0; i < 32; ++i) v[i] = (in && col + i < N) ? v[i] * gelu_erf_grad(__bfloat162float(P[i])) : 0.f;
    }
  }
  if constexpr (EPI == FB_EPI_BF16_ROWDOT) {  // rd += bf16(dO) . O over these 32 columns of the head
    if (in && full) {
      const __nv_bfloat16* O = reinterpret_cast<const __nv_bfloat16*>(e.aux) + row * e.ld_aux + col;
      float acc = 0.f;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 pk = *reinterpret_cast<const uint4*>(O + 8 * q);
        const __nv_bfloat162* ob = reinterpret_cast<const __nv_bfloat162*>(&pk);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 o2 = __bfloat1622float2(ob[i]);
          const float2 g2 = __bfloat1622float2(__floats2bfloat162_rn(v[8 * q + 2 * i], v[8 * q + 2 * i + 1]));
          acc = fmaf(g2.x, o2.x, acc);
          acc = fmaf(g2.y, o2.y, acc);
        }
      }
      rd += acc;
    }
  }
  // ---- staging (the previous chunk's bulk store must have read the tile) ----
  if (lane == 0) bulk_wait_read<0>();
  __syncwarp();
  constexpr bool kBf16Out = EPI == FB_EPI_BF16 || EPI == FB_EPI_GELU || EPI == FB_EPI_DGELU || EPI == FB_EPI_BF16_ROWDOT ||
                            EPI == FB_EPI_CE_EXP;
  if constexpr (kBf16Out) {
#pragma unroll
    for (int j = 0; j < 4; ++j) stg_put_bf16(stg, lane, j, v + 8 * j);
    if constexpr (EPI == FB_EPI_GELU) {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        *reinterpret_cast<uint4*>(stg + 2048 + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4)) =
            make_uint4(pre[4 * j], pre[4 * j + 1], pre[4 * j + 2], pre[4 * j + 3]);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) stg_put_f32(stg, lane, j, v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
  }
  fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) {
    tma_store_3d(&mp.C, stg, col, row0, split);
#ifndef FB_EXP_NO_AUX
    if constexpr (EPI == FB_EPI_GELU) tma_store_3d(&mp.Aux, stg + 2048, col, row0, 0);
#endif
    bulk_commit();
  }
  if constexpr (EPI == FB_EPI_RESID_F32_BF16) {  // second output reuses the tile once the f32 store read it
    if (lane == 0) bulk_wait_read<0>();
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 4; ++j) stg_put_bf16(stg, lane, j, v + 8 * j);
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_store_3d(&mp.Aux, stg, col, row0, 0);
      bulk_commit();
    }
  }
}

// ---------------------------------------------------------------------------------------
// 2-SM variant: a CTA pair (cluster of 2 on one TPC) computes a 256 x 256 tile with
// tcgen05.mma.cta_group::2 (M = 256). Each CTA stages its 128 rows of A and its 128 of
// the 256 B rows, so per-SM operand traffic drops from 48 KB to 32 KB per 64-deep
// k-block and 6 stages fit. The leader CTA (rank 0) issues all MMAs; accumulator rows
// land in each CTA's own TMEM, and each CTA drains its own 128 rows.
constexpr int kStages2 = 6;
constexpr int kStage2Bytes = 2 * BM * BK * 2;  // A half + B half
constexpr int kSmem2 = kStages2 * kStage2Bytes + 8 * 4096 + 1024 + 1024;  // tiles, epilogue staging, barriers, align

template <int A_MN, int B_MN, int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kGemmThreads, 1)
    gemm_bf16_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M,
                         int N, int K, EpiArgs ep, const __grid_constant__ EpiMaps maps) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_addr = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_addr + 1023) & ~1023u) - raw_addr);
  uint8_t* tiles = smem;
  uint8_t* staging = smem + kStages2 * kStage2Bytes;  // 8 epilogue warps x kStageEpi
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(staging + 8 * kStageEpi);
  uint64_t* empty_bar = full_bar + kStages2;
  uint64_t* tfull_bar = empty_bar + kStages2;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int cluster = blockIdx.x >> 1, nclusters = gridDim.x >> 1;
  const int num_m = (M + 255) / 256;
  const int num_n = (N + 255) / 256;
  const int num_tiles = num_m * num_n;
  const int num_kb = (K + BK - 1) / BK;
  // epilogue inputs one chunk ahead only where the main loop is short (C2 / C3: dGELU +17%,
  // out-projection residual +5%); at K = 2048 the early loads measured 1-4% slower
  const bool early = K <= 1024;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    tma_prefetch(&maps.C);
    for (int s = 0; s < kStages2; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull_bar[b], 1);
      mbar_init(&tempty_bar[b], 16);  // 8 epilogue warps x 2 CTAs
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_2sm(tmem_slot, 512);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = cluster; u < ep.units; u += nclusters) {
        int tile, kb0, nkb, piece;
        unit_coords2(u, num_tiles, num_kb, ep, tile, kb0, nkb, piece);
        int mb, nb;
        tile_coords(tile, num_m, num_n, mb, nb, ep.group_m);
        const int m0 = mb * 256 + rank * 128;
        const int n0 = nb * 256 + rank * 128;
        for (int kb = kb0; kb < kb0 + nkb; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = tiles + stage * kStage2Bytes;
          uint8_t* sb = sa + BM * BK * 2;
          if (leader) mbar_arrive_expect_tx(&full_bar[stage], 2 * kStage2Bytes);
          const int k0 = kb * BK;
          if (A_MN) tma_load_3d_2sm(sa, &tmA, &full_bar[stage], 0, k0, m0 / 64);
          else      tma_load_2d_2sm(sa, &tmA, &full_bar[stage], k0, m0);
          if (B_MN) tma_load_3d_2sm(sb, &tmB, &full_bar[stage], 0, k0, n0 / 64);
          else      tma_load_2d_2sm(sb, &tmB, &full_bar[stage], k0, n0);
          if (++stage == kStages2) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      constexpr uint32_t idesc = idesc_bf16_f32(256, 256, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int u = cluster; u < ep.units; u += nclusters, ++it) {
        int tile, kb0, nkb, piece;
        unit_coords2(u, num_tiles, num_kb, ep, tile, kb0, nkb, piece);
        const int buf = it & 1;
        const uint32_t use = it >> 1;
        mbar_wait(&tempty_bar[buf], (use & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + buf * 256;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          if (lane == 0) {
            const uint32_t sa = smem_u32(tiles + stage * kStage2Bytes);
            const uint32_t sb = sa + BM * BK * 2;
#pragma unroll
            for (int kk = 0; kk < BK / 16; ++kk) {
              const uint64_t ad = A_MN ? smem_desc_sw128(sa + kk * 2048, BK * 128, 1024)
                                       : smem_desc_sw128(sa + kk * 32, 16, 1024);
              const uint64_t bd = B_MN ? smem_desc_sw128(sb + kk * 2048, BK * 128, 1024)
                                       : smem_desc_sw128(sb + kk * 32, 16, 1024);
              umma_f16_2sm(d_tmem, ad, bd, idesc, (kb | kk) != 0);
            }
            umma_commit_2sm_mc(&empty_bar[stage]);
          }
          __syncwarp();
          if (++stage == kStages2) { stage = 0; phase ^= 1; }
        }
        if (lane == 0) umma_commit_2sm_mc(&tfull_bar[buf]);
        __syncwarp();
      }
    }
  } else {
    const int quad = warp & 3;
    const int half = (warp - 2) >> 2;
    uint8_t* stg = staging + (warp - 2) * kStageEpi;
    int it = 0;
    for (int u = cluster; u < ep.units; u += nclusters, ++it) {
      int tile, kb0, nkb, piece;
      unit_coords2(u, num_tiles, num_kb, ep, tile, kb0, nkb, piece);
      int mb, nb;
      tile_coords(tile, num_m, num_n, mb, nb, ep.group_m);
      const int m0 = mb * 256 + rank * 128;
      const int n0 = nb * 256 + half * 128;
      const int buf = it & 1;
      const uint32_t use = it >> 1;
      const int row0 = m0 + quad * 32;
      uint4 pf[8];
      if (piece < 0 && early) epi_prefetch<EPI>(ep, row0 + lane, n0, M, N, pf);
      mbar_wait(&tfull_bar[buf], use & 1);
      tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(quad * 32) << 16) + buf * 256 + half * 128;
      float rd = 0.f;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(taddr + c * 32, r);
        uint4 cur[8];
        if (early) {
#pragma unroll
          for (int q = 0; q < 8; ++q) cur[q] = pf[q];
          if (c < 3 && piece < 0) epi_prefetch<EPI>(ep, row0 + lane, n0 + (c + 1) * 32, M, N, pf);
        } else if (piece < 0) {
          epi_prefetch<EPI>(ep, row0 + lane, n0 + c * 32, M, N, cur);
        }
        tmem_ld_wait();
        if (c == 3) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_leader(&tempty_bar[buf]);
        }
        const int col = n0 + c * 32;
        if (row0 < M && col < N) {
          if (piece >= 0)
            partial_chunk_tma(&maps.Part, stg, lane, col - nb * 256, row0 - mb * 256, piece, r);
          else
            epilogue_chunk_tma<EPI>(ep, maps, stg, lane, row0 + lane, row0, col, u / num_tiles, M, N, r, rd, cur);
        }
        if constexpr (EPI == FB_EPI_BF16_ROWDOT) {  // head boundary: D[b][h][t] of this lane's row
          if ((col + 32) % ep.rd_dh == 0) {
            const int row = row0 + lane;
            if (row < M && col < N) {
              const int T = ep.rd_T, nh = N / ep.rd_dh;
              reinterpret_cast<float*>(ep.aux_out)[((int64_t)(row / T) * nh + col / ep.rd_dh) * T + row % T] = rd;
            }
            rd = 0.f;
          }
        }
      }
    }
    if (lane == 0) bulk_wait_read<0>();
    __syncwarp();
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_2sm(tmem_base, 512);
  }
}

// ---------------------------------------------------------------------------------------
// host side
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static thread_local void* g_split_ws = nullptr;  // split-K workspace for the current call
static thread_local int g_split_n = 1;
static thread_local void* g_tail_ws = nullptr;  // last-wave split for the current call
static thread_local int g_tail_full = 0, g_tail_split = 1;
static thread_local int g_rd_T = 0, g_rd_dh = 0;  // fb_gemm_bf16_rowdot for the current call
int g_gemm_2sm = 1;  // fb_gemm_set_2sm() toggles it (A/B tests)
int g_group_m_forced = 0;  // fb_gemm_set_group_m(): raster group override (A/B tests)

static int get_encoder() {
  if (g_encode) return FB_OK;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  FB_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  if (!fn || q != cudaDriverEntryPointSuccess) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return FB_CUDA_ERROR;
  }
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return FB_OK;
}

// K-major operand stored [rows][ld] (K contiguous): box {64 k, box_rows}
static int make_map_kmajor(CUtensorMap* m, const void* ptr, int rows, int K, int64_t ld, int box_rows) {
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled(K-major rows=%d K=%d ld=%lld) failed: %d", rows, K, (long long)ld, (int)r);
    return FB_CUDA_ERROR;
  }
  return FB_OK;
}

// MN-major operand stored [K][ld] (MN contiguous), viewed 3-D {64 mn, K, mn/64}
static int make_map_mnmajor(CUtensorMap* m, const void* ptr, int mn, int K, int64_t ld, int box_mn) {
  cuuint64_t dims[3] = {64, (cuuint64_t)K, (cuuint64_t)(mn / 64)};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 2, 128};
  cuuint32_t box[3] = {64, (cuuint32_t)BK, (cuuint32_t)(box_mn / 64)};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled(MN-major mn=%d K=%d ld=%lld) failed: %d", mn, K, (long long)ld, (int)r);
    return FB_CUDA_ERROR;
  }
  return FB_OK;
}

// Ragged MN-major operand [K][ld] (mn % 64 != 0): 2-D {mn, K}, box {64 mn, 64 k}, one TMA per chunk
static int make_map_mnmajor_2d(CUtensorMap* m, const void* ptr, int mn, int K, int64_t ld) {
  cuuint64_t dims[2] = {(cuuint64_t)mn, (cuuint64_t)K};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)BK};
  cuuint32_t es[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled(MN-major 2-D mn=%d K=%d ld=%lld) failed: %d", mn, K, (long long)ld, (int)r);
    return FB_CUDA_ERROR;
  }
  return FB_OK;
}

template <int BN, int A_MN, int B_MN, int EPI>
static int launch_gemm_t(const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K, const EpiArgs& ep,
                         cudaStream_t st) {
  using Cfg = GemmCfg<BN>;
  auto kern = gemm_bf16_tc_kernel<BN, A_MN, B_MN, EPI>;
  static bool attr_set = false;  // per instantiation
  if (!attr_set) {
    FB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM));
    attr_set = true;
  }
  const int tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN) * ep.ksplit;
  const int grid = tiles < kNumSMs ? tiles : kNumSMs;
  kern<<<grid, kGemmThreads, Cfg::SMEM, st>>>(ta, tb, M, N, K, ep);
  FB_LAUNCH_CHECK();
  return FB_OK;
}

// Output map for the TMA-store epilogue: {N, M, splits}, box {32 cols, 32 rows, 1}.
static int make_out_map(CUtensorMap* m, void* ptr, bool bf16, int M, int N, int64_t ld, int splits,
                        int64_t split_stride) {
  const int es = bf16 ? 2 : 4;
  cuuint64_t dims[3] = {(cuuint64_t)N, (cuuint64_t)M, (cuuint64_t)splits};
  cuuint64_t strides[2] = {(cuuint64_t)ld * es, (cuuint64_t)(splits > 1 ? split_stride : (int64_t)M * ld) * es};
  cuuint32_t box[3] = {32, 32, 1};
  cuuint32_t el[3] = {1, 1, 1};
  CUresult r = g_encode(m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, ptr, dims,
                        strides, box, el, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        bf16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled(output M=%d N=%d ld=%lld) failed: %d", M, N, (long long)ld, (int)r);
    return FB_CUDA_ERROR;
  }
  return FB_OK;
}

template <int A_MN, int B_MN, int EPI>
static int launch_gemm2_t(const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K, const EpiArgs& ep,
                          cudaStream_t st) {
  constexpr bool kBf16Out = EPI == FB_EPI_BF16 || EPI == FB_EPI_GELU || EPI == FB_EPI_DGELU || EPI == FB_EPI_BF16_ROWDOT ||
                            EPI == FB_EPI_CE_EXP;
  EpiMaps maps;
  int rc = make_out_map(&maps.C, ep.C, kBf16Out, M, N, ep.ldc, ep.ksplit, ep.split_stride);
  if (rc) return rc;
  if (EPI == FB_EPI_GELU || EPI == FB_EPI_RESID_F32_BF16) {
    rc = make_out_map(&maps.Aux, ep.aux_out, true, M, N, EPI == FB_EPI_GELU ? ep.ld_aux : ep.ldc, 1, 0);
    if (rc) return rc;
  } else {
    maps.Aux = maps.C;
  }
  if (ep.tail_split > 1) {
    const int pieces = (((M + 255) / 256) * ((N + 255) / 256) - ep.full_tiles) * ep.tail_split;
    rc = make_out_map(&maps.Part, ep.tail_ws, false, 256, 256, 256, pieces, 65536);
    if (rc) return rc;
  } else {
    maps.Part = maps.C;
  }
  auto kern = gemm_bf16_tc2_kernel<A_MN, B_MN, EPI>;
  static bool attr_set = false;
  if (!attr_set) {
    FB_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem2));
    attr_set = true;
  }
  EpiArgs e2 = ep;
  const int tiles = ((M + 255) / 256) * ((N + 255) / 256);
  e2.units = ep.tail_split > 1 ? ep.full_tiles + (tiles - ep.full_tiles) * ep.tail_split : tiles * ep.ksplit;
  const int clusters = e2.units < kNumSMs / 2 ? e2.units : kNumSMs / 2;
  kern<<<2 * clusters, kGemmThreads, kSmem2, st>>>(ta, tb, M, N, K, e2, maps);
  FB_LAUNCH_CHECK();
  return FB_OK;
}

template <int A_MN, int B_MN>
static int dispatch_epi2(int epi, const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K,
                         const EpiArgs& ep, cudaStream_t st) {
  switch (epi) {
    case FB_EPI_BF16: return launch_gemm2_t<A_MN, B_MN, FB_EPI_BF16>(ta, tb, M, N, K, ep, st);
    case FB_EPI_F32: return launch_gemm2_t<A_MN, B_MN, FB_EPI_F32>(ta, tb, M, N, K, ep, st);
    case FB_EPI_ACC_F32: return launch_gemm2_t<A_MN, B_MN, FB_EPI_ACC_F32>(ta, tb, M, N, K, ep, st);
    case FB_EPI_RESID_F32: return launch_gemm2_t<A_MN, B_MN, FB_EPI_RESID_F32>(ta, tb, M, N, K, ep, st);
    case FB_EPI_GELU: return launch_gemm2_t<A_MN, B_MN, FB_EPI_GELU>(ta, tb, M, N, K, ep, st);
    case FB_EPI_DGELU: return launch_gemm2_t<A_MN, B_MN, FB_EPI_DGELU>(ta, tb, M, N, K, ep, st);
    case FB_EPI_RESID_F32_BF16: return launch_gemm2_t<A_MN, B_MN, FB_EPI_RESID_F32_BF16>(ta, tb, M, N, K, ep, st);
    case FB_EPI_BF16_ROWDOT: return launch_gemm2_t<A_MN, B_MN, FB_EPI_BF16_ROWDOT>(ta, tb, M, N, K, ep, st);
    case FB_EPI_CE_EXP:
      if constexpr (A_MN == 0 && B_MN == 0) return launch_gemm2_t<0, 0, FB_EPI_CE_EXP>(ta, tb, M, N, K, ep, st);
      break;
  }
  set_error("unknown epilogue %d", epi);
  return FB_BAD_ARG;
}

template <int BN, int A_MN, int B_MN>
static int dispatch_epi(int epi, const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K,
                        const EpiArgs& ep, cudaStream_t st) {
  switch (epi) {
    case FB_EPI_BF16: return launch_gemm_t<BN, A_MN, B_MN, FB_EPI_BF16>(ta, tb, M, N, K, ep, st);
    case FB_EPI_F32: return launch_gemm_t<BN, A_MN, B_MN, FB_EPI_F32>(ta, tb, M, N, K, ep, st);
    case FB_EPI_ACC_F32: return launch_gemm_t<BN, A_MN, B_MN, FB_EPI_ACC_F32>(ta, tb, M, N, K, ep, st);
    case FB_EPI_RESID_F32: return launch_gemm_t<BN, A_MN, B_MN, FB_EPI_RESID_F32>(ta, tb, M, N, K, ep, st);
    case FB_EPI_GELU: return launch_gemm_t<BN, A_MN, B_MN, FB_EPI_GELU>(ta, tb, M, N, K, ep, st);
    case FB_EPI_DGELU: return launch_gemm_t<BN, A_MN, B_MN, FB_EPI_DGELU>(ta, tb, M, N, K, ep, st);
    case FB_EPI_RESID_F32_BF16: return launch_gemm_t<BN, A_MN, B_MN, FB_EPI_RESID_F32_BF16>(ta, tb, M, N, K, ep, st);
    case FB_EPI_CE_EXP:
      if constexpr (A_MN == 0 && B_MN == 0) return launch_gemm_t<BN, 0, 0, FB_EPI_CE_EXP>(ta, tb, M, N, K, ep, st);
      break;
  }
  set_error("unknown epilogue %d", epi);
  return FB_BAD_ARG;
}

}  // namespace fb

namespace fb {
extern int g_gemm_2sm;
extern int g_group_m_forced;
int raster_group_m(int K, int num_n);
int gemm_dispatch(int key, int epilogue, const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K,
                  const EpiArgs& ep, cudaStream_t st);
}
using namespace fb;

extern "C" int fb_gemm_bf16(int M, int N, int K, const void* d_A, int64_t lda, int a_major, const void* d_B,
                            int64_t ldb, int b_major, void* d_C, int64_t ldc, int epilogue, const void* d_aux,
                            void* d_aux_out, int64_t ld_aux, void* stream) {
  FB_REQUIRE(M > 0 && N > 0 && K > 0, "gemm: non-positive shape %d x %d x %d", M, N, K);
  FB_REQUIRE(d_A && d_B && d_C, "gemm: null operand");
  FB_REQUIRE(((uintptr_t)d_A % 16 == 0) && ((uintptr_t)d_B % 16 == 0) && ((uintptr_t)d_C % 16 == 0),
             "gemm: operands must be 16-byte aligned");
  FB_REQUIRE(lda % 8 == 0 && ldb % 8 == 0, "gemm: lda/ldb must be multiples of 8 elements");
  FB_REQUIRE(ldc % 8 == 0, "gemm: ldc must be a multiple of 8 elements");
  const bool need_aux = epilogue == FB_EPI_RESID_F32 || epilogue == FB_EPI_DGELU || epilogue == FB_EPI_RESID_F32_BF16;
  const bool need_aux_out = epilogue == FB_EPI_GELU || epilogue == FB_EPI_RESID_F32_BF16 || epilogue == FB_EPI_CE_EXP;
  FB_REQUIRE(epilogue != FB_EPI_CE_EXP || (a_major == 0 && b_major == 0 && ld_aux >= M),
             "gemm: the CE epilogue needs K-major operands and ld_aux >= M (stats row stride)");
  FB_REQUIRE(!need_aux || d_aux, "gemm: epilogue %d needs aux", epilogue);
  FB_REQUIRE(!need_aux_out || d_aux_out, "gemm: epilogue %d needs aux_out", epilogue);
  FB_REQUIRE(!need_aux_out || ((uintptr_t)d_aux_out % 8 == 0 && (epilogue != FB_EPI_GELU || ld_aux % 8 == 0)),
             "gemm: aux_out must be 16-byte aligned with ld_aux %% 8 == 0");
  int rc = get_encoder();
  if (rc) return rc;
  // 2-SM 256x256 tiles when they fill the 74 CTA pairs; else 1-SM 128x256, else 128x128
  const int tiles2 = ((M + 255) / 256) * ((N + 255) / 256);
  const int ks = g_split_ws ? g_split_n : 1;
  const bool a_2d = a_major && M % 64, b_2d = b_major && N % 64;
#ifndef FB_OLD_KSPLIT
  // a split-K call keeps the 2-SM kernel even when its units do not fill the first wave
  const bool use2 = g_gemm_2sm && M >= 256 && N >= 256 && (tiles2 * ks >= kNumSMs / 2 || ks > 1) && !a_2d && !b_2d;
#else
  const bool use2 = g_gemm_2sm && M >= 256 && N >= 256 && tiles2 * ks >= kNumSMs / 2 && !a_2d && !b_2d;
#endif
  const int tiles256 = ((M + BM - 1) / BM) * ((N + 255) / 256) * ks;
  const int BN = (use2 || (N >= 256 && tiles256 >= kNumSMs)) ? 256 : 128;
  CUtensorMap ta, tb;
  rc = a_2d ? make_map_mnmajor_2d(&ta, d_A, M, K, lda)
     : a_major ? make_map_mnmajor(&ta, d_A, M, K, lda, BM) : make_map_kmajor(&ta, d_A, M, K, lda, BM);
  if (rc) return rc;
  const int bbox = use2 ? 128 : BN;  // 2-SM: each CTA stages 128 of the 256 B rows
  rc = b_2d ? make_map_mnmajor_2d(&tb, d_B, N, K, ldb)
     : b_major ? make_map_mnmajor(&tb, d_B, N, K, ldb, bbox) : make_map_kmajor(&tb, d_B, N, K, ldb, bbox);
  if (rc) return rc;
  if (epilogue == FB_EPI_BF16_ROWDOT && (!use2 || g_rd_T <= 0)) {
    set_error("gemm: the row-dot epilogue needs the 2-SM kernel (fb_gemm_bf16_rowdot)");
    return FB_UNSUPPORTED;
  }
  EpiArgs ep{d_C, ldc, d_aux, d_aux_out, ld_aux, 1, 0, 0, 1, nullptr, 0, raster_group_m(K, (N + 255) / 256),
             g_rd_T, g_rd_dh, (int)a_2d, (int)b_2d};
  if (g_tail_ws && use2) {  // set by fb_gemm_bf16_splitk for this call only
    ep.full_tiles = g_tail_full;
    ep.tail_split = g_tail_split;
    ep.tail_ws = g_tail_ws;
  }
  if (g_split_ws) {  // set by fb_gemm_bf16_splitk for this call only
    ep.ksplit = g_split_n;
    ep.C = g_split_ws;
    ep.ldc = N;
    ep.split_stride = (int64_t)M * N;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int key = (BN == 256 ? 4 : 0) | (a_major ? 2 : 0) | (b_major ? 1 : 0);
  const int pi = prof_on() ? prof_start(0, st) : -1;
  if (use2) {
    const int k2 = (a_major ? 2 : 0) | (b_major ? 1 : 0);
    rc = k2 == 0 ? dispatch_epi2<0, 0>(epilogue, ta, tb, M, N, K, ep, st)
       : k2 == 1 ? dispatch_epi2<0, 1>(epilogue, ta, tb, M, N, K, ep, st)
       : k2 == 2 ? dispatch_epi2<1, 0>(epilogue, ta, tb, M, N, K, ep, st)
                 : dispatch_epi2<1, 1>(epilogue, ta, tb, M, N, K, ep, st);
  } else {
    rc = gemm_dispatch(key, epilogue, ta, tb, M, N, K, ep, st);
  }
  prof_stop(0, pi, st, 2.0 * M * N * (double)K);
  return rc;
}

namespace fb {
extern int g_gemm_2sm;
extern int g_group_m_forced;
int gemm_dispatch(int key, int epilogue, const CUtensorMap& ta, const CUtensorMap& tb, int M, int N, int K,
                  const EpiArgs& ep, cudaStream_t st) {
  switch (key) {
    case 0: return dispatch_epi<128, 0, 0>(epilogue, ta, tb, M, N, K, ep, st);
    case 1: return dispatch_epi<128, 0, 1>(epilogue, ta, tb, M, N, K, ep, st);
    case 2: return dispatch_epi<128, 1, 0>(epilogue, ta, tb, M, N, K, ep, st);
    case 3: return dispatch_epi<128, 1, 1>(epilogue, ta, tb, M, N, K, ep, st);
    case 4: return dispatch_epi<256, 0, 0>(epilogue, ta, tb, M, N, K, ep, st);
    case 5: return dispatch_epi<256, 0, 1>(epilogue, ta, tb, M, N, K, ep, st);
    case 6: return dispatch_epi<256, 1, 0>(epilogue, ta, tb, M, N, K, ep, st);
    case 7: return dispatch_epi<256, 1, 1>(epilogue, ta, tb, M, N, K, ep, st);
  }
  return FB_BAD_ARG;
}
}  // namespace fb

extern "C" int fb_gemm_bf16_rowdot(int M, int N, int K, const void* d_A, int64_t lda, int a_major, const void* d_B,
                                   int64_t ldb, int b_major, void* d_C, int64_t ldc, const void* d_O, int64_t ld_o,
                                   float* d_D, int T, int dh, void* stream) {
  FB_REQUIRE(d_O && d_D && T > 0 && M % T == 0, "rowdot: needs O, D and M %% T == 0");
  FB_REQUIRE(dh >= 32 && dh % 32 == 0 && 128 % dh == 0 && N % dh == 0, "rowdot: head dim %d unsupported", dh);
  FB_REQUIRE(ld_o % 8 == 0 && (uintptr_t)d_O % 16 == 0, "rowdot: O must be 16-byte aligned rows");
  const int tiles2 = ((M + 255) / 256) * ((N + 255) / 256);
  if (!(g_gemm_2sm && M >= 256 && N >= 256 && tiles2 >= kNumSMs / 2)) {
    set_error("rowdot: the 2-SM kernel does not apply to %d x %d", M, N);
    return FB_UNSUPPORTED;
  }
  g_rd_T = T;
  g_rd_dh = dh;
  const int rc = fb_gemm_bf16(M, N, K, d_A, lda, a_major, d_B, ldb, b_major, d_C, ldc, FB_EPI_BF16_ROWDOT, d_O, d_D,
                              ld_o, stream);
  g_rd_T = g_rd_dh = 0;
  return rc;
}

extern "C" int fb_gemm_set_group_m(int group_m) {
  FB_REQUIRE(group_m >= 0 && group_m <= 1024, "bad group_m %d", group_m);
  fb::g_group_m_forced = group_m;
  return FB_OK;
}

extern "C" int fb_gemm_set_2sm(int enable) {
  fb::g_gemm_2sm = enable ? 1 : 0;
  return FB_OK;
}

namespace fb {
// C[m][n] (+)= sum_s W[s][m][n] in fixed split order (deterministic)
__global__ void splitk_reduce_kernel(const float* __restrict__ W, int S, int64_t MN, int N, float* __restrict__ C,
                                     int64_t ldc, int accumulate) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < MN / 4; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = 4 * i, m = e / N, n = e % N;
    float4 acc = *reinterpret_cast<const float4*>(W + e);
    for (int s = 1; s < S; ++s) {
      const float4 v = *reinterpret_cast<const float4*>(W + s * MN + e);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    float4* c = reinterpret_cast<float4*>(C + m * ldc + n);
    if (accumulate) {
      const float4 o = *c;
      acc.x += o.x; acc.y += o.y; acc.z += o.z; acc.w += o.w;
    }
    *c = acc;
  }
}

// Last-wave split: C[tile] (+)= sum_s part[(tile - F) * S + s] in fixed order, for the tiles
// [F, num_tiles) of the 2-SM raster (deterministic). Block x = tail tile, y = row slab.
__global__ void tail_reduce_kernel(const float* __restrict__ W, int S, int F, int num_m, int num_n, int group_m, int M,
                                   int N, float* __restrict__ C, int64_t ldc, int accumulate) {
  int mb, nb;
  tile_coords(F + blockIdx.x, num_m, num_n, mb, nb, group_m);
  const float* w0 = W + (int64_t)blockIdx.x * S * 65536;
  for (int i = blockIdx.y * blockDim.x + threadIdx.x; i < 256 * 64; i += gridDim.y * blockDim.x) {
    const int r = i >> 6, c = (i & 63) * 4;
    const int m = mb * 256 + r, n = nb * 256 + c;
    if (m >= M || n >= N) continue;
    float4 acc = *reinterpret_cast<const float4*>(w0 + r * 256 + c);
    for (int sp = 1; sp < S; ++sp) {
      const float4 v = *reinterpret_cast<const float4*>(w0 + (int64_t)sp * 65536 + r * 256 + c);
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    float4* cp = reinterpret_cast<float4*>(C + (int64_t)m * ldc + n);
    if (accumulate) {
      const float4 o = *cp;
      acc.x = o.x + acc.x; acc.y = o.y + acc.y; acc.z = o.z + acc.z; acc.w = o.w + acc.w;
    }
    *cp = acc;
  }
}

// Raster group height of the 2-SM kernel. Short K: 16 m-blocks (the A panels of a group are
// small and stay in L2 across its waves). Long K (>= 4096, panels >= 2 MB): a wave of the 74
// CTA pairs covers whole rows of n-blocks, so every A and B k-slice is shared by the tiles
// that read it at the same time and no panel is re-fetched from DRAM in a later wave.
int raster_group_m(int K, int num_n) {
  if (g_group_m_forced > 0) return g_group_m_forced;  // fb_gemm_set_group_m (A/B experiments)
  if (K >= 4096 && num_n <= kNumSMs / 2) return (kNumSMs / 2 + num_n - 1) / num_n;
  return kGroupM;
}

// Plan the last-wave split of a 2-SM GEMM with `tiles` 256x256 tiles and num_kb k-blocks:
// returns S > 1 (and F) when cutting the ragged last wave into S K-ranges beats running it
// whole by >= 4% of the launch, within `max_pieces` workspace tiles.
static int plan_tail_split(int tiles, int num_kb, int max_pieces, int& F) {
  const int P = kNumSMs / 2;
  F = (tiles / P) * P;
  const int R = tiles - F;
  if (R == 0) return 1;
  const double base = F / (double)P + 1.0;
  int best = 1;
  double best_t = base;
  for (int S = 2; S <= 16; ++S) {
    const int per = (num_kb + S - 1) / S;
    if (num_kb - (S - 1) * per < 4 || R * S > max_pieces) break;
    const double t = F / (double)P + (double)((R * S + P - 1) / P) / S + 0.01 * S;
    if (t < best_t) { best_t = t; best = S; }
  }
  return best_t <= 0.96 * base ? best : 1;
}

// Full split-K for the 2-SM kernel (fewer output tiles than CTA pairs): the split S minimises
// waves(S) * (k-blocks per unit + 2) + partial traffic, in units of one 256x256x64 k-block of a
// CTA pair (~2.2 MB of HBM traffic at the power-capped clock). Filling the first wave is not
// enough: 4 tiles x 19 splits = 76 units is two waves for two units (51% busy), 4 x 18 = 72 one.
static int plan_ksplit(int tiles, int num_kb, int64_t mn, int max_split) {
  const int P = kNumSMs / 2;
  int best = 1;
  double best_t = 1e30;
  // S = 1 with fewer tiles than CTA pairs would leave the 2-SM kernel; start at 2 then
  for (int S = tiles < P && max_split >= 2 ? 2 : 1; S <= std::min(max_split, 64); ++S) {
    const int per = (num_kb + S - 1) / S;
    if (S > 1 && (per < 16 || (S - 1) * per >= num_kb)) break;
    const int waves = (tiles * S + P - 1) / P;
    const double t = waves * (per + 2.0) + (S > 1 ? (S + 2) * (double)mn * 4 / 2.2e6 + 8.0 : 0.0);
    if (t < best_t) { best_t = t; best = S; }
  }
  return best;
}
}  // namespace fb

// Split-K GEMM for short-M/N, long-K products (weight gradients over many tokens):
// ksplit partial f32 products into d_ws (ksplit * M * N floats), then a fixed-order
// reduction into C (f32; += when epilogue == FB_EPI_ACC_F32). ksplit <= 0 picks a split
// that fills the 148 SMs.
extern "C" int fb_gemm_bf16_splitk(int M, int N, int K, const void* d_A, int64_t lda, int a_major, const void* d_B,
                                   int64_t ldb, int b_major, void* d_C, int64_t ldc, int epilogue, int ksplit,
                                   void* d_ws, int64_t ws_bytes, void* stream) {
  FB_REQUIRE(epilogue == FB_EPI_F32 || epilogue == FB_EPI_ACC_F32, "split-K supports the f32 / acc_f32 epilogues");
  FB_REQUIRE(N % 4 == 0 && ldc % 4 == 0, "split-K needs N and ldc multiples of 4");
  const int tiles2 = ((M + 255) / 256) * ((N + 255) / 256);
  const int num_kb = (K + BK - 1) / BK;
  if (ksplit <= 0) {
    // 2-SM raster with a full first wave: split only the ragged last wave (tile-local partials)
    const bool ragged = (a_major && M % 64) || (b_major && N % 64);  // 1-SM kernel only
    if (g_gemm_2sm && M >= 256 && N >= 256 && tiles2 >= kNumSMs / 2 && d_ws && !ragged) {
      int F = 0;
      const int S = plan_tail_split(tiles2, num_kb, (int)(ws_bytes / (65536 * 4)), F);
      if (S > 1) {
        g_tail_ws = d_ws;
        g_tail_full = F;
        g_tail_split = S;
        int rc = fb_gemm_bf16(M, N, K, d_A, lda, a_major, d_B, ldb, b_major, d_C, ldc, epilogue, nullptr, nullptr, 0,
                              stream);
        g_tail_ws = nullptr;
        g_tail_full = 0;
        g_tail_split = 1;
        if (rc) return rc;
        fb::tail_reduce_kernel<<<dim3(tiles2 - F, 16), 256, 0, (cudaStream_t)stream>>>(
            (const float*)d_ws, S, F, (M + 255) / 256, (N + 255) / 256, raster_group_m(K, (N + 255) / 256), M, N,
            (float*)d_C, ldc,
            epilogue == FB_EPI_ACC_F32);
        FB_LAUNCH_CHECK();
        return FB_OK;
      }
    }
    ksplit = 1;
#ifndef FB_OLD_KSPLIT
    if (g_gemm_2sm && M >= 256 && N >= 256 && tiles2 < kNumSMs / 2 && !ragged && d_ws)
      ksplit = plan_ksplit(tiles2, num_kb, (int64_t)M * N, (int)std::min<int64_t>(64, ws_bytes / ((int64_t)M * N * 4)));
    else
#endif
    while (tiles2 * ksplit < kNumSMs / 2 && num_kb / (ksplit + 1) >= 16) ++ksplit;
  }
  // every split must own >= 1 k-block (ceil-sized splits: the last ones could be empty)
  while (ksplit > 1 && (ksplit - 1) * ((num_kb + ksplit - 1) / ksplit) >= num_kb) --ksplit;
  if (ksplit <= 1) return fb_gemm_bf16(M, N, K, d_A, lda, a_major, d_B, ldb, b_major, d_C, ldc, epilogue, nullptr,
                                       nullptr, 0, stream);
  FB_REQUIRE(d_ws && ws_bytes >= (int64_t)ksplit * M * N * 4, "split-K workspace too small (%d splits)", ksplit);
  g_split_ws = d_ws;
  g_split_n = ksplit;
  int rc = fb_gemm_bf16(M, N, K, d_A, lda, a_major, d_B, ldb, b_major, d_ws, N, FB_EPI_F32, nullptr, nullptr, 0, stream);
  g_split_ws = nullptr;
  g_split_n = 1;
  if (rc) return rc;
  fb::splitk_reduce_kernel<<<fb::kNumSMs * 4, 256, 0, (cudaStream_t)stream>>>(
      (const float*)d_ws, ksplit, (int64_t)M * N, N, (float*)d_C, ldc, epilogue == FB_EPI_ACC_F32);
  FB_LAUNCH_CHECK();
  return FB_OK;
}
