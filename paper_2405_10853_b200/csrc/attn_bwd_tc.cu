// Causal ALiBi attention BACKWARD on tcgen05 / TMEM / TMA.
//
// Reference: gradient of fedforge/model.py:92-98 (scores/sqrt(dh) + ALiBi bias, softmax,
// PV); the bias is constant, so dq = dS k / sqrt(dh), dk = dS^T q / sqrt(dh),
// dv = P^T dO, dS = P o (dP - D), D = rowsum(dO o O) (precomputed).
//
// CTA = 128 keys of one (b, h); loop over the causal query tiles i >= kb.
//   warp 0     TMA producer: K, V once; Q_i and dO_i per tile (single buffer, each
//              refilled as soon as its last MMA reader commits). One 3-D tensor map
//              {64, B*T, 3d/64} over qkv (K-major for S/dP, MN-major for dK/dQ's B)
//              and one {64, B*T, d/64} over dO.
//   warp 1     TMEM owner + single-thread tcgen05.mma issuer, per tile:
//                S^T  = K  Q^T   (M=128 keys, N=128 q, K=dh)  -> TMEM [0,128)
//                dP^T = V  dO^T  (M=128 keys, N=128 q, K=dh)  -> TMEM [128,256)
//                dV  += P^T dO   (M=128 keys, N=dh, K=128 q)  -> TMEM [256, 256+dh)
//                dK  += dS^T Q   (M=128 keys, N=dh, K=128 q)  -> TMEM [256+dh, 256+2dh)
//                dQ   = dS  K    (M=128 q, N=dh, K=128 keys)  -> TMEM [128, 128+dh) (aliases dP^T)
//              dS for dQ is the SAME swizzled smem image as dS^T, read as an MN-major A.
//   warps 2-5  thread = TMEM lane: (a) key row: P^T = exp2(S^T c - sl (q-k) - lse2_q) masked,
//              dS^T = P^T (dP^T - D_q) -> bf16 K-major smem tiles; (b) query row: drain dQ
//              (x 1/sqrt(dh)) into the f32 dq accumulator with vector reductions.
//   end        dK (x 1/sqrt(dh)), dV -> bf16 rows of dqkv.
#include <cudaTypedefs.h>

#include "common.cuh"
#include "sm100.cuh"

namespace fb {
using namespace sm100;

__device__ __forceinline__ float ex2b(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

template <int DH>
struct AttnBwdCfg {
  static constexpr int TILE = 128 * DH * 2;
  static constexpr int K_OFF = 0;
  static constexpr int V_OFF = K_OFF + TILE;
  static constexpr int Q_OFF = V_OFF + TILE;      // [2] stages
  static constexpr int O_OFF = Q_OFF + 2 * TILE;  // dO [2] stages
  static constexpr int PS_OFF = O_OFF + 2 * TILE; // P^T, then dS^T (128x128 bf16, shared)
  static constexpr int L_OFF = PS_OFF + 32768;    // e[128], D[128]
  static constexpr int BAR_OFF = L_OFF + 2 * 128 * 4;
  static constexpr int SMEM = BAR_OFF + 160 + 1024;  // 17 mbarriers + TMEM slot; 1 KB alignment slack
};

template <int DH>
__global__ void __launch_bounds__(320, 1)
    attn_bwd_tc_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                       const __grid_constant__ CUtensorMap tm_dq, const float* __restrict__ lse2, const float* __restrict__ Dd, float* __restrict__ dq_acc,
                       __nv_bfloat16* __restrict__ dqkv, int T, int H, float scale_log2, float scale, int use_alibi) {
  using Cf = AttnBwdCfg<DH>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023) & ~1023u) - raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Cf::BAR_OFF);
  uint64_t* kv_full = bar + 0;
  uint64_t* q_full = bar + 1;    // [2]
  uint64_t* o_full = bar + 3;    // [2]
  uint64_t* q_empty = bar + 5;   // [2]
  uint64_t* o_empty = bar + 7;   // [2]
  uint64_t* s_full = bar + 9;
  uint64_t* p_full = bar + 10;
  uint64_t* p_free = bar + 11;
  uint64_t* ds_full = bar + 12;
  uint64_t* ds_free = bar + 13;
  uint64_t* dq_full = bar + 14;
  uint64_t* dq_empty = bar + 15;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 16);
  float* sE = reinterpret_cast<float*>(smem + Cf::L_OFF);  // [128]
  float* sD = sE + 128;                                      // [128]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nq = T / 128;
  const int kb = blockIdx.x;  // kb = 0 has the most query tiles: launched first
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const int d = H * DH;
  const int row0 = b * T;
  const int k0 = kb * 128;
  const int first = kb, ntiles = nq - kb;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_qkv);
    tma_prefetch(&tm_do);
    mbar_init(kv_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&o_full[s], 1);
      mbar_init(&q_empty[s], 1);
      mbar_init(&o_empty[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(p_full, 8);
    mbar_init(p_free, 1);
    mbar_init(ds_full, 8);
    mbar_init(ds_free, 1);
    mbar_init(dq_full, 1);
    mbar_init(dq_empty, 8);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sK = smem_u32(smem + Cf::K_OFF), sV = smem_u32(smem + Cf::V_OFF), sQ0 = smem_u32(smem + Cf::Q_OFF),
                 sO0 = smem_u32(smem + Cf::O_OFF), sPS = smem_u32(smem + Cf::PS_OFF);

  if (warp == 0) {
    if (lane == 0) {
      const int zq = (h * DH) / 64, zk = (d + h * DH) / 64, zv = (2 * d + h * DH) / 64, zo = (h * DH) / 64;
      mbar_arrive_expect_tx(kv_full, 2 * Cf::TILE);
      tma_load_3d(smem + Cf::K_OFF, &tm_qkv, kv_full, 0, row0 + k0, zk);
      tma_load_3d(smem + Cf::V_OFF, &tm_qkv, kv_full, 0, row0 + k0, zv);
      for (int t = 0; t < ntiles; ++t) {
        const int s = t & 1;
        const uint32_t ph = (t >> 1) & 1;
        const int q0 = (first + t) * 128;
        mbar_wait(&q_empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&q_full[s], Cf::TILE);
        tma_load_3d(smem + Cf::Q_OFF + s * Cf::TILE, &tm_qkv, &q_full[s], 0, row0 + q0, zq);
        mbar_wait(&o_empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&o_full[s], Cf::TILE);
        tma_load_3d(smem + Cf::O_OFF + s * Cf::TILE, &tm_do, &o_full[s], 0, row0 + q0, zo);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idSP = idesc_bf16_f32(128, 128, 0, 0);  // S^T, dP^T: K-major A and B
      constexpr uint32_t idKV = idesc_bf16_f32(128, DH, 0, 1);   // dV, dK: K-major A, MN-major B
      constexpr uint32_t idQ = idesc_bf16_f32(128, DH, 1, 1);    // dQ: MN-major A (dS), MN-major B (K)
      const uint32_t tS = tmem, tP = tmem + 128, tV = tmem + 256, tK = tmem + 256 + DH, tQ = tmem + 128;
      mbar_wait(kv_full, 0);
      for (int t = 0; t < ntiles; ++t) {
        const int s = t & 1;
        const uint32_t ph = t & 1, sph = (t >> 1) & 1;
        const uint32_t sQ = sQ0 + s * Cf::TILE, sO = sO0 + s * Cf::TILE;
        mbar_wait(&q_full[s], sph);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {  // S^T = K Q^T
          const uint32_t off = (kk >> 2) * (128 * 128) + (kk & 3) * 32;
          umma_f16(tS, smem_desc_sw128(sK + off, 16, 1024), smem_desc_sw128(sQ + off, 16, 1024), idSP, kk > 0);
        }
        mbar_wait(&o_full[s], sph);
        mbar_wait(dq_empty, ph ^ 1);  // dP^T columns still hold dQ of the previous tile until drained
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {  // dP^T = V dO^T
          const uint32_t off = (kk >> 2) * (128 * 128) + (kk & 3) * 32;
          umma_f16(tP, smem_desc_sw128(sV + off, 16, 1024), smem_desc_sw128(sO + off, 16, 1024), idSP, kk > 0);
        }
        umma_commit(s_full);
        mbar_wait(p_full, ph);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // dV += P^T dO   (K = 128 queries)
          const uint32_t aoff = (kk >> 2) * (128 * 128) + (kk & 3) * 32;
          umma_f16(tV, smem_desc_sw128(sPS + aoff, 16, 1024), smem_desc_sw128(sO + kk * 2048, 128 * 128, 1024), idKV,
                   (t | kk) > 0);
        }
        umma_commit(p_free);
        umma_commit(&o_empty[s]);
        mbar_wait(ds_full, ph);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // dK += dS^T Q
          const uint32_t aoff = (kk >> 2) * (128 * 128) + (kk & 3) * 32;
          umma_f16(tK, smem_desc_sw128(sPS + aoff, 16, 1024), smem_desc_sw128(sQ + kk * 2048, 128 * 128, 1024), idKV,
                   (t | kk) > 0);
        }
        umma_commit(&q_empty[s]);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // dQ = dS K   (K = 128 keys), dS read as MN-major
          umma_f16(tQ, smem_desc_sw128(sPS + kk * 2048, 128 * 128, 1024),
                   smem_desc_sw128(sK + kk * 2048, 128 * 128, 1024), idQ, kk > 0);
        }
        umma_commit(ds_free);
        umma_commit(dq_full);
      }
    }
  } else {
    // warps 2-5 (g = 0) and 6-9 (g = 1): each warpgroup owns half of the 128 query
    // columns of S^T / dP^T and half of the dh columns of dQ / dK / dV.
    const int g = (warp - 2) >> 2;
    const int quad = warp & 3;
    const int r = quad * 32 + lane;  // TMEM lane: key row (P/dS phase) / query row (dQ drain)
    const int kj = k0 + r;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const uint32_t tS = tmem + lane_off + 64 * g, tP = tmem + 128 + lane_off + 64 * g;
    const uint32_t tQ = tmem + 128 + lane_off + (DH / 2) * g;
    const float sl = use_alibi ? exp2f(-8.0f * (float)(h + 1) / (float)H) * 1.4426950408889634f : 0.0f;
    const float slk = sl * (float)kj;
    const uint32_t prow = sPS + r * 128;
    const int tid = threadIdx.x - 64;  // 0..255
    for (int t = 0; t < ntiles; ++t) {
      const uint32_t ph = t & 1;
      const int q0 = (first + t) * 128;
      const bool diag = (t == 0);
      float* Eb = sE;  // e_q = sl * q + lse2_q  (x = S c + sl k - e_q)
      float* Db = sD;
      asm volatile("bar.sync 1, 256;" ::: "memory");  // everyone is done with the previous tile's e/D
      if (tid < 128) Eb[tid] = sl * (float)(q0 + tid) + lse2[(int64_t)bh * T + q0 + tid];
      else Db[tid - 128] = Dd[(int64_t)bh * T + q0 + tid - 128];
      asm volatile("bar.sync 1, 256;" ::: "memory");
      mbar_wait(s_full, ph);
      mbar_wait(ds_free, ph ^ 1);  // the shared P/dS tile is no longer read by dQ of the previous tile
      tc_fence_after();
      uint32_t dsp[32];  // dS^T packed bf16x2, written after dV consumed P^T
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t sv[32], pv[32];
        tmem_ld_32x32b_x32(tS + c * 32, sv);
        tmem_ld_32x32b_x32(tP + c * 32, pv);
        tmem_ld_wait();
        const int qb = 64 * g + 32 * c;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float p[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int ql = qb + q * 8 + i;
            const float x = fmaf(__uint_as_float(sv[q * 8 + i]), scale_log2, slk - Eb[ql]);
            p[i] = (diag && q0 + ql < kj) ? 0.f : ex2b(x);
            sv[q * 8 + i] = __float_as_uint(p[i] * (__uint_as_float(pv[q * 8 + i]) - Db[ql]));
          }
#pragma unroll
          for (int i = 0; i < 4; ++i)
            dsp[c * 16 + q * 4 + i] = pack_bf16(__uint_as_float(sv[q * 8 + 2 * i]), __uint_as_float(sv[q * 8 + 2 * i + 1]));
          const int kc = (qb >> 3) + q;
          const uint32_t sw = (kc >> 3) * (128 * 128) + (((kc & 7) ^ (r & 7)) << 4);
          asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(prow + sw), "r"(pack_bf16(p[0], p[1])),
                       "r"(pack_bf16(p[2], p[3])), "r"(pack_bf16(p[4], p[5])), "r"(pack_bf16(p[6], p[7])));
        }
      }
      tc_fence_before();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      // dV has consumed P^T: overwrite the shared tile with dS^T
      mbar_wait(p_free, ph);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int kc = ((64 * g + 32 * c) >> 3) + q;
          const uint32_t sw = (kc >> 3) * (128 * 128) + (((kc & 7) ^ (r & 7)) << 4);
          asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(prow + sw), "r"(dsp[c * 16 + q * 4]),
                       "r"(dsp[c * 16 + q * 4 + 1]), "r"(dsp[c * 16 + q * 4 + 2]), "r"(dsp[c * 16 + q * 4 + 3]));
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(ds_full);
      // drain this warpgroup's half of dQ (thread = query row r of this tile): TMEM -> 128B-swizzled
      // smem (the P/dS tile is free once dQ_t has completed) -> TMA bulk reduce-add into the f32 dq
      // accumulator, one 128 x 32 box per chunk (replaces per-thread red.global traffic).
      mbar_wait(dq_full, ph);
      tc_fence_after();
      const uint32_t stage = sPS + g * 16384;
#pragma unroll 1
      for (int c = 0; c < DH / 64; ++c) {
        uint32_t v[32];
        tmem_ld_32x32b_x32(tQ + c * 32, v);
        tmem_ld_wait();
        if (c > 0) {  // the previous box must have been read out of smem
          if (quad == 0 && lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          asm volatile("bar.sync %0, 128;" ::"r"(2 + g) : "memory");
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint32_t addr = stage + r * 128 + ((q ^ (r & 7)) << 4);
          asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "f"(__uint_as_float(v[4 * q]) * scale),
                       "f"(__uint_as_float(v[4 * q + 1]) * scale), "f"(__uint_as_float(v[4 * q + 2]) * scale),
                       "f"(__uint_as_float(v[4 * q + 3]) * scale));
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync %0, 128;" ::"r"(2 + g) : "memory");
        if (quad == 0 && lane == 0) {
          asm volatile(
              "cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                  reinterpret_cast<uint64_t>(&tm_dq)),
              "r"(stage), "r"(h * DH + (DH / 2) * g + c * 32), "r"(row0 + q0)
              : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
      // the P/dS tile is reused by the next tile's P: wait until TMA has read the staging box
      if (quad == 0 && lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      asm volatile("bar.sync %0, 128;" ::"r"(2 + g) : "memory");
      asm volatile("bar.sync 1, 256;" ::: "memory");  // both staging halves drained before any next-tile P write
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dq_empty);
    }
    // dK, dV: the last dK/dV MMAs completed before the last dq_full
    const int64_t ld = 3 * (int64_t)d;
    __nv_bfloat16* dkrow = dqkv + ((int64_t)row0 + kj) * ld + d + h * DH + (DH / 2) * g;
    __nv_bfloat16* dvrow = dkrow + d;
#pragma unroll 1
    for (int c = 0; c < DH / 64; ++c) {
      uint32_t kv[32], vv[32];
      const uint32_t col = (DH / 2) * g + c * 32;
      tmem_ld_32x32b_x32(tmem + 256 + DH + lane_off + col, kv);
      tmem_ld_32x32b_x32(tmem + 256 + lane_off + col, vv);
      tmem_ld_wait();
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float* fk = reinterpret_cast<const float*>(kv) + 8 * q;
        const float* fv = reinterpret_cast<const float*>(vv) + 8 * q;
        *reinterpret_cast<uint4*>(dkrow + c * 32 + 8 * q) =
            make_uint4(pack_bf16(fk[0] * scale, fk[1] * scale), pack_bf16(fk[2] * scale, fk[3] * scale),
                       pack_bf16(fk[4] * scale, fk[5] * scale), pack_bf16(fk[6] * scale, fk[7] * scale));
        *reinterpret_cast<uint4*>(dvrow + c * 32 + 8 * q) = make_uint4(
            pack_bf16(fv[0], fv[1]), pack_bf16(fv[2], fv[3]), pack_bf16(fv[4], fv[5]), pack_bf16(fv[6], fv[7]));
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 g_enc_bwd = nullptr;

static int encode_rows_map(CUtensorMap* m, const void* base, int64_t rows, int cols, int box_chunks) {
  cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)(cols / 64)};
  cuuint64_t strides[2] = {(cuuint64_t)cols * 2, 128};
  cuuint32_t box[3] = {64, 128, (cuuint32_t)box_chunks};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_enc_bwd(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("attn bwd tensor map encode failed: %d", (int)r);
    return FB_CUDA_ERROR;
  }
  return FB_OK;
}

template <int DH>
int attn_bwd_tc_launch(const void* qkv, const void* dO, const float* lse, const float* Dbuf, float* dq, void* dqkv,
                       int B, int T, int H, int use_alibi, cudaStream_t st) {
  using Cf = AttnBwdCfg<DH>;
  if (!g_enc_bwd) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    FB_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn) {
      set_error("cuTensorMapEncodeTiled unavailable");
      return FB_CUDA_ERROR;
    }
    g_enc_bwd = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  }
  const int d = H * DH;
  CUtensorMap tq, to;
  int rc = encode_rows_map(&tq, qkv, (int64_t)B * T, 3 * d, DH / 64);
  if (rc) return rc;
  rc = encode_rows_map(&to, dO, (int64_t)B * T, d, DH / 64);
  if (rc) return rc;
  CUtensorMap tdq;
  {
    cuuint64_t dims[2] = {(cuuint64_t)d, (cuuint64_t)B * T};
    cuuint64_t strides[1] = {(cuuint64_t)d * 4};
    cuuint32_t box[2] = {32, 128};
    cuuint32_t es[2] = {1, 1};
    CUresult r = g_enc_bwd(&tdq, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dq, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("attn bwd dq tensor map encode failed: %d", (int)r);
      return FB_CUDA_ERROR;
    }
  }
  auto k = attn_bwd_tc_kernel<DH>;
  FB_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM));
  const float scale = 1.0f / sqrtf((float)DH);
  k<<<dim3(T / 128, B * H), 320, Cf::SMEM, st>>>(tq, to, tdq, lse, Dbuf, dq, (__nv_bfloat16*)dqkv, T, H,
                                                 1.4426950408889634f * scale, scale, use_alibi);
  FB_LAUNCH_CHECK();
  return FB_OK;
}

template int attn_bwd_tc_launch<64>(const void*, const void*, const float*, const float*, float*, void*, int, int, int,
                                    int, cudaStream_t);
template int attn_bwd_tc_launch<128>(const void*, const void*, const float*, const float*, float*, void*, int, int,
                                     int, int, cudaStream_t);

}  // namespace fb
