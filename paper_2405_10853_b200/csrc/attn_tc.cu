// Causal ALiBi attention FORWARD on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// Reference: fedforge/model.py:92-98 (scores/sqrt(dh) + alibi bias, softmax, PV) with
// slope_h = 2^(-8(h+1)/H) (model.py:46-50). Output/lse contract identical to
// attn_fwd_kernel in attn.cu (o [B*T][d] bf16, lse2 [B][H][T] base-2).
//
// CTA = 128 query rows of one (b, h); KV tiles of 128 keys, causal (tiles 0..qb).
//   warp 0     TMA producer: Q once, K/V double-buffered. One 3-D tensor map
//              {64, B*T, 3d/64} over the qkv buffer serves Q, K and V: the smem image
//              [dh/64][128 rows][64] is a K-major operand for Q and K and an MN-major
//              operand for V, so no transposes are ever materialised.
//   warp 1     TMEM owner + single-thread tcgen05.mma issuer:
//              S = Q K^T  (M=128, N=128, K=dh)       -> TMEM cols [0,128)
//              O_j = P V  (M=128, N=dh,  K=128 keys)  -> TMEM cols [128, 128+dh)
//   warps 2-5  softmax: thread = query row = TMEM lane. Two passes over S in TMEM
//              (row max, then exp2 + row sum + bf16 P into a 128B-swizzled K-major smem
//              tile), then O_acc = O_acc * alpha + O_j in registers.
#include <cudaTypedefs.h>

#include "common.cuh"
#include "sm100.cuh"

namespace fb {
using namespace sm100;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

template <int DH>
struct AttnTcCfg {
  static constexpr int BM = 128, BN = 128;
  static constexpr int TILE = 128 * DH * 2;  // one 128-row x DH bf16 tile
  static constexpr int Q_OFF = 0;
  static constexpr int K_OFF = Q_OFF + TILE;          // [2] stages
  static constexpr int V_OFF = K_OFF + 2 * TILE;      // [2] stages
  static constexpr int P_OFF = V_OFF + 2 * TILE;      // 128 x 128 bf16
  static constexpr int BAR_OFF = P_OFF + 128 * 128 * 2;
  static constexpr int SMEM = BAR_OFF + 256 + 1024;
  static constexpr uint32_t TMEM_COLS = 256;
};

template <int DH>
__global__ void __launch_bounds__(192, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tm, __nv_bfloat16* __restrict__ out,
                       float* __restrict__ lse2, int T, int H, float scale_log2, int use_alibi) {
  using Cf = AttnTcCfg<DH>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023) & ~1023u) - raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Cf::BAR_OFF);
  uint64_t* q_full = bar + 0;
  uint64_t* k_full = bar + 1;   // [2]
  uint64_t* v_full = bar + 3;   // [2]
  uint64_t* kv_empty = bar + 5; // [2]
  uint64_t* s_full = bar + 7;
  uint64_t* s_empty = bar + 8;
  uint64_t* p_full = bar + 9;
  uint64_t* o_full = bar + 10;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 12);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nq = T / 128;
  const int qb = nq - 1 - blockIdx.x;  // heavy tiles first
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const int d = H * DH;
  const int row0 = b * T;              // first row of this sequence in [B*T]
  const int q0 = qb * 128;
  const int ntiles = qb + 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm);
    mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_empty, 4);
    mbar_init(p_full, 4);
    mbar_init(o_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, Cf::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sQ = smem_u32(smem + Cf::Q_OFF), sK = smem_u32(smem + Cf::K_OFF),
                 sV = smem_u32(smem + Cf::V_OFF), sP = smem_u32(smem + Cf::P_OFF);

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      const int zq = (0 * d + h * DH) / 64, zk = (1 * d + h * DH) / 64, zv = (2 * d + h * DH) / 64;
      mbar_arrive_expect_tx(q_full, Cf::TILE);
      tma_load_3d(smem + Cf::Q_OFF, &tm, q_full, 0, row0 + q0, zq);
      for (int j = 0; j < ntiles; ++j) {
        const int s = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        mbar_wait(&kv_empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&k_full[s], Cf::TILE);
        tma_load_3d(smem + Cf::K_OFF + s * Cf::TILE, &tm, &k_full[s], 0, row0 + j * 128, zk);
        mbar_arrive_expect_tx(&v_full[s], Cf::TILE);
        tma_load_3d(smem + Cf::V_OFF + s * Cf::TILE, &tm, &v_full[s], 0, row0 + j * 128, zv);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      constexpr uint32_t idS = idesc_bf16_f32(128, 128, 0, 0);
      constexpr uint32_t idO = idesc_bf16_f32(128, DH, 0, 1);
      const uint32_t tS = tmem, tO = tmem + 128;
      mbar_wait(q_full, 0);
      for (int j = 0; j < ntiles; ++j) {
        const int s = j & 1;
        const uint32_t ph = (j >> 1) & 1;
        mbar_wait(&k_full[s], ph);
        mbar_wait(s_empty, (j & 1) ^ 1);
        tc_fence_after();
        const uint32_t kb = sK + s * Cf::TILE;
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const uint32_t off = (kk >> 2) * (128 * 128) + (kk & 3) * 32;
          umma_f16(tS, smem_desc_sw128(sQ + off, 16, 1024), smem_desc_sw128(kb + off, 16, 1024), idS, kk > 0);
        }
        umma_commit(s_full);
        mbar_wait(p_full, j & 1);  // P_j written and O rescaled by the softmax warps
        mbar_wait(&v_full[s], ph);
        tc_fence_after();
        const uint32_t vb = sV + s * Cf::TILE;
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // 128 keys / 16
          const uint32_t poff = (kk >> 2) * (128 * 128) + (kk & 3) * 32;
          umma_f16(tO, smem_desc_sw128(sP + poff, 16, 1024), smem_desc_sw128(vb + kk * 2048, 128 * 128, 1024), idO,
                   (j | kk) > 0);
        }
        umma_commit(o_full);
        umma_commit(&kv_empty[s]);
      }
    }
  } else {
    // ---------------- softmax warps 2..5 ----------------
    const int quad = warp & 3;
    const int r = quad * 32 + lane;  // row within the tile == TMEM lane
    const int qi = q0 + r;           // query position
    const uint32_t tS = tmem + ((uint32_t)(quad * 32) << 16);
    const uint32_t tO = tS + 128;
    const float sl = use_alibi ? exp2f(-8.0f * (float)(h + 1) / (float)H) * 1.4426950408889634f : 0.0f;
    float m = -INFINITY, l = 0.f;
    const uint32_t prow = sP + r * 128;
    for (int j = 0; j < ntiles; ++j) {
      const int k0 = j * 128;
      const bool diag = (j == ntiles - 1);
      mbar_wait(s_full, j & 1);
      tc_fence_after();
      // pass 1: row max of the scaled, biased, masked scores
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tS + c * 32, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int kj = k0 + c * 32 + i;
          float x = __uint_as_float(v[i]) * scale_log2 - sl * (float)(qi - kj);
          if (diag && kj > qi) x = -INFINITY;
          mx = fmaxf(mx, x);
        }
      }
      const float m_new = fmaxf(m, mx);
      const float alpha = ex2(m - m_new);
      // pass 2: P = exp2(x - m_new) -> bf16 -> swizzled K-major smem tile; row sum
      float rs = 0.f;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tS + c * 32, v);
        tmem_ld_wait();
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float p[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int kj = k0 + c * 32 + q * 8 + i;
            const float x = __uint_as_float(v[q * 8 + i]) * scale_log2 - sl * (float)(qi - kj);
            p[i] = (diag && kj > qi) ? 0.f : ex2(x - m_new);
            rs += p[i];
          }
          const int kc = c * 4 + q;  // 8-key chunk 0..15
          const uint32_t addr = prow + (kc >> 3) * (128 * 128) + (((kc & 7) ^ (r & 7)) << 4);
          asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(pack_bf16(p[0], p[1])),
                       "r"(pack_bf16(p[2], p[3])), "r"(pack_bf16(p[4], p[5])), "r"(pack_bf16(p[6], p[7])));
        }
      }
      l = l * alpha + rs;
      m = m_new;
      // rescale the TMEM accumulator O by alpha once PV_{j-1} has landed (skip when no row moved)
      if (j > 0) {
        mbar_wait(o_full, (j - 1) & 1);
        tc_fence_after();
        if (__any_sync(0xffffffffu, alpha != 1.0f)) {
#pragma unroll
          for (int c = 0; c < DH / 32; ++c) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(tO + c * 32, v);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
            tmem_st_32x32b_x32(tO + c * 32, v);
          }
          tmem_st_wait();
        }
      }
      tc_fence_before();
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(s_empty);
        mbar_arrive(p_full);
      }
    }
    mbar_wait(o_full, (ntiles - 1) & 1);
    tc_fence_after();
    const float il = 1.0f / l;
    __nv_bfloat16* orow = out + ((int64_t)row0 + qi) * d + h * DH;
#pragma unroll
    for (int c = 0; c < DH / 32; ++c) {
      uint32_t v[32];
      tmem_ld_32x32b_x32(tO + c * 32, v);
      tmem_ld_wait();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float* f = reinterpret_cast<const float*>(v) + 8 * q;
        uint4 pk = make_uint4(pack_bf16(f[0] * il, f[1] * il), pack_bf16(f[2] * il, f[3] * il),
                              pack_bf16(f[4] * il, f[5] * il), pack_bf16(f[6] * il, f[7] * il));
        *reinterpret_cast<uint4*>(orow + c * 32 + 8 * q) = pk;
      }
    }
    lse2[(int64_t)bh * T + qi] = m + log2f(l);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, Cf::TMEM_COLS);
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 g_enc_attn = nullptr;

template <int DH>
int attn_fwd_tc_launch(const void* qkv, void* o, float* lse, int B, int T, int H, int use_alibi, cudaStream_t st) {
  using Cf = AttnTcCfg<DH>;
  if (!g_enc_attn) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    FB_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn) {
      set_error("cuTensorMapEncodeTiled unavailable");
      return FB_CUDA_ERROR;
    }
    g_enc_attn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const int d = H * DH;
  CUtensorMap tm;
  cuuint64_t dims[3] = {64, (cuuint64_t)B * T, (cuuint64_t)(3 * d / 64)};
  cuuint64_t strides[2] = {(cuuint64_t)3 * d * 2, 128};
  cuuint32_t box[3] = {64, 128, DH / 64};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_enc_attn(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(qkv), dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("attn tensor map encode failed: %d", (int)r);
    return FB_CUDA_ERROR;
  }
  auto k = attn_fwd_tc_kernel<DH>;
  FB_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM));
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)DH);
  k<<<dim3(T / 128, B * H), 192, Cf::SMEM, st>>>(tm, (__nv_bfloat16*)o, lse, T, H, scale_log2, use_alibi);
  FB_LAUNCH_CHECK();
  return FB_OK;
}

template int attn_fwd_tc_launch<64>(const void*, void*, float*, int, int, int, int, cudaStream_t);
template int attn_fwd_tc_launch<128>(const void*, void*, float*, int, int, int, int, cudaStream_t);

}  // namespace fb
