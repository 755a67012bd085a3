// Causal ALiBi attention FORWARD on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// Reference: fedforge/model.py:92-98 (scores/sqrt(dh) + alibi bias, softmax, PV) with
// slope_h = 2^(-8(h+1)/H) (model.py:46-50). Outputs: o [B*T][d] bf16 and
// lse2 [B][H][T] (base-2 log-sum-exp, consumed by the backward).
//
// CTA = a PAIR of 128-row query tiles of one (b, h) (ping-pong; the last pair holds one
// tile when T % 256 == 128), KV tiles of 64 keys, causal. Heaviest pairs launch first.
//   warp 8     TMA producer: Q once, K and V double-buffered with separate barriers, K
//              loaded ahead of V. One 3-D tensor map {64, B*T, 3d/64} serves K and V:
//              the smem image [dh/64][rows][64] is K-major for K and MN-major for V, so
//              no transposes are ever materialised.
//   warp 9     TMEM owner + single-thread tcgen05.mma issuer. S = Q K^T for both Q tiles
//              is issued one KV tile ahead into double-buffered TMEM columns, then
//              O_g += P_g V (accumulated in TMEM).
//   warps 0-3 (Q tile 0), 4-7 (Q tile 1): softmax, thread = query row = TMEM lane.
//              exp2 with the ALiBi bias folded into one FFMA, bf16 P into a 128B-swizzled
//              K-major smem tile, lazy (threshold 8, log2 units) in-TMEM rescale of O.
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
#ifdef FB_ATTN_TRACE
__device__ unsigned long long g_attn_trace_fwd[2048];
__device__ __forceinline__ unsigned long long gtimer_f() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define FTRACE(slot) do { if (blockIdx.x == 0 && blockIdx.y == 5 && (slot) < 2048) g_attn_trace_fwd[(slot)] = gtimer_f(); } while (0)
#else
#define FTRACE(slot) do {} while (0)
#endif
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Layout: a CTA owns TWO 128-query tiles (rows q0..q0+255) that ping-pong on the tensor
// core. KV tiles are 64 keys in an NST-deep ring: a step's MMAs take ~0.6 us while a K/V
// TMA load takes ~1 us, so two stages left the MMA warp waiting on loads (measured with
// tools/attn_trace_fwd.py). P is single-buffered per Q tile: PV(j) finishes long before
// the softmax of step j+1 writes P again.
template <int DH>
struct AttnTcCfg {
  static constexpr int BN = 64;
  static constexpr int NST = DH == 128 ? 4 : 8;  // K/V ring depth
  static constexpr int QT = 128 * DH * 2;      // one 128-row Q tile
  static constexpr int KT = BN * DH * 2;       // one 64-row K (or V) tile
  static constexpr int PT = 128 * BN * 2;      // one P tile (128 q x 64 keys)
  static constexpr int Q_OFF = 0;              // [2] Q tiles
  static constexpr int K_OFF = 2 * QT;         // [NST] stages
  static constexpr int V_OFF = K_OFF + NST * KT;  // [NST] stages
  static constexpr int P_OFF = V_OFF + NST * KT;  // [2 Q tiles] P tiles
  static constexpr int BAR_OFF = P_OFF + 2 * PT;
  static constexpr int SMEM = BAR_OFF + 512 + 1024;  // (13 + 4 NST) mbarriers + TMEM slot; alignment slack
  static_assert(SMEM <= 232448, "attention forward smem");
};

// Warp roles. The issue scheduler favours HIGH warp ids, so the two single-thread control
// warps (TMA producer, MMA issuer) sit above the eight softmax warps: at ids 0/1 they were
// starved by the softmax warps sharing their SM sub-partition (MMA issue stretched to
// ~70 cycles per instruction; tools/attn_trace_fwd.py).
constexpr int kProducerWarp = 8, kMmaWarp = 9;

// Pipeline (per KV step j of Q tile g, b = j & 1; key tiles walk from the diagonal down):
//   MMA:     S_g(j+1) -> TMEM S[g][b^1]   (runs ahead: S is double-buffered)
//            PV_g(j)  -> TMEM O[g]        (after P_g(j) is in smem buffer [g][b])
//   softmax: S[g][b] -> P[g][b]; O rescaled only when the row max grows by > 8 (log2)
template <int DH>
__global__ void __launch_bounds__(320, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmq, const __grid_constant__ CUtensorMap tm,
                       __nv_bfloat16* __restrict__ out, float* __restrict__ lse2, uint8_t* __restrict__ live_map,
                       int T, int H, float scale_log2, int use_alibi) {
  using Cf = AttnTcCfg<DH>;
  constexpr int BN = Cf::BN;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023) & ~1023u) - raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Cf::BAR_OFF);
  constexpr int NST = Cf::NST;
  uint64_t* q_full = bar + 0;
  uint64_t* k_full = bar + 1;             // [NST]
  uint64_t* k_empty = k_full + NST;       // [NST]
  uint64_t* v_full = k_empty + NST;       // [NST]
  uint64_t* v_empty = v_full + NST;       // [NST]
  uint64_t* s_full = v_empty + NST;       // [g][b]
  uint64_t* s_empty = s_full + 4;         // [g][b]
  uint64_t* p_full = s_empty + 4;         // [g]
  uint64_t* pv_done = p_full + 2;         // [g]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pv_done + 2);
  uint8_t* dead_flag = reinterpret_cast<uint8_t*>(tmem_slot + 1);  // [g][warp of the group]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int npair = (T + 255) / 256;
  const int pb = npair - 1 - blockIdx.x;  // heavy pairs first
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const int d = H * DH;
  const int row0 = b * T;
  const int q0 = pb * 256;
  const bool has1 = q0 + 256 <= T;        // T % 256 == 128: the last pair has only Q tile 0
  const int nkv0 = (q0 + 128) / BN;      // KV tiles for Q tile 0
  const int nkv = has1 ? (q0 + 256) / BN : nkv0;  // KV tiles for the whole pair
  // KV tiles are visited from the diagonal DOWN (key tile nkv-1-t at step t): with ALiBi the
  // row max is found in the first tile, so the lazy O rescale almost never fires. Q tile 0
  // joins once the walk reaches its last key tile (start0 steps in).
  const int start0 = nkv - nkv0;

  if (warp == kProducerWarp && lane == 0) {
    tma_prefetch(&tm);
    tma_prefetch(&tmq);
    mbar_init(q_full, 1);
    for (int i = 0; i < NST; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 4);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&p_full[i], 4);
      mbar_init(&pv_done[i], 1);
    }
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sQ = smem_u32(smem + Cf::Q_OFF), sK = smem_u32(smem + Cf::K_OFF),
                 sV = smem_u32(smem + Cf::V_OFF), sP = smem_u32(smem + Cf::P_OFF);

  if (warp == kProducerWarp) {
    if (lane == 0) {
      const int zq = (h * DH) / 64, zk = (d + h * DH) / 64, zv = (2 * d + h * DH) / 64;
      mbar_arrive_expect_tx(q_full, (has1 ? 2 : 1) * Cf::QT);
      tma_load_3d(smem + Cf::Q_OFF, &tmq, q_full, 0, row0 + q0, zq);
      if (has1) tma_load_3d(smem + Cf::Q_OFF + Cf::QT, &tmq, q_full, 0, row0 + q0 + 128, zq);
      // K runs one tile ahead of V: order K0, K1, V0, K2, V1, ... (K stages free right after the S MMAs)
      auto load_k = [&](int j) {
        const int s = j % NST;
        mbar_wait(&k_empty[s], ((j / NST) & 1) ^ 1);
        mbar_arrive_expect_tx(&k_full[s], Cf::KT);
        tma_load_3d(smem + Cf::K_OFF + s * Cf::KT, &tm, &k_full[s], 0, row0 + (nkv - 1 - j) * BN, zk);
      };
      auto load_v = [&](int j) {
        const int s = j % NST;
        mbar_wait(&v_empty[s], ((j / NST) & 1) ^ 1);
        mbar_arrive_expect_tx(&v_full[s], Cf::KT);
        tma_load_3d(smem + Cf::V_OFF + s * Cf::KT, &tm, &v_full[s], 0, row0 + (nkv - 1 - j) * BN, zv);
      };
      load_k(0);
      for (int j = 0; j < nkv; ++j) {
        if (j + 1 < nkv) load_k(j + 1);
        load_v(j);
      }
    }
  } else if (warp == kMmaWarp) {
    if (lane == 0) {
      constexpr uint32_t idS = idesc_bf16_f32(128, BN, 0, 0);
      constexpr uint32_t idO = idesc_bf16_f32(128, DH, 0, 1);
      // TMEM: S[g][b] at 64 (2g + b); O[g] at 256 + DH g
      auto issue_s = [&](int g, int j, int t) {  // j: Q tile g's own tile count, t: KV stage counter
        const int bb = j & 1;
        mbar_wait(&s_empty[2 * g + bb], ((j >> 1) & 1) ^ 1);
        FTRACE((t - 1) * 16 + 8 + g);
        tc_fence_after();
        const uint32_t qb = sQ + g * Cf::QT, kb = sK + (t % NST) * Cf::KT;
        // K-major SW128 operands: 16-wide k steps are +32 B inside a 64-column chunk, chunks
        // are (rows x 128 B) apart
        const uint64_t qd = smem_desc_sw128(qb, 16, 1024), kd = smem_desc_sw128(kb, 16, 1024);
        constexpr int NK = DH / 16;
        uint64_t ad[NK], bd[NK];
#pragma unroll
        for (int kk = 0; kk < NK; ++kk) {
          ad[kk] = qd + ((uint64_t)((kk >> 2) * (128 * 128) + (kk & 3) * 32) >> 4);
          bd[kk] = kd + ((uint64_t)((kk >> 2) * (BN * 128) + (kk & 3) * 32) >> 4);
        }
        if constexpr (NK == 8) umma_f16_x8(tmem + 64 * (2 * g + bb), ad, bd, idS, 0);
        else umma_f16_x4(tmem + 64 * (2 * g + bb), *reinterpret_cast<uint64_t(*)[4]>(ad),
                         *reinterpret_cast<uint64_t(*)[4]>(bd), idS, 0);
        umma_commit(&s_full[2 * g + bb]);
      };
      auto issue_s_both = [&](int j) {  // S(j) for the active Q tiles, then release the K stage
        mbar_wait(&k_full[j % NST], (j / NST) & 1);
        FTRACE((j - 1) * 16 + 7);
        if (j >= start0) issue_s(0, j - start0, j);
        if (has1) issue_s(1, j, j);
        umma_commit(&k_empty[j % NST]);
      };
      uint32_t o_acc[2] = {0u, 0u};  // O_g holds a PV product
      auto issue_pv = [&](int g, int j, int t) {
        mbar_wait(&p_full[g], j & 1);
        FTRACE(t * 16 + 10 + 2 * g);
        mbar_wait(&v_full[t % NST], (t / NST) & 1);
        FTRACE(t * 16 + 11 + 2 * g);
        // all four warps found every p of their rows exactly 0: the block adds nothing to O
        const bool dead = *reinterpret_cast<volatile uint32_t*>(dead_flag + 4 * g) == 0x01010101u;
        if (live_map)
          live_map[((int64_t)bh * (T / 128) + (q0 >> 7) + g) * (T / BN) + (g ? nkv : nkv0) - 1 - j] = dead ? 0 : 1;
        if (dead) {
          umma_commit(&pv_done[g]);
          return;
        }
        tc_fence_after();
        const uint32_t pbuf = sP + g * Cf::PT, vb = sV + (t % NST) * Cf::KT;
        // P: K-major (k step +32 B); V: MN-major (k step = 16 key rows = +2048 B)
        const uint64_t pd = smem_desc_sw128(pbuf, 16, 1024), vd = smem_desc_sw128(vb, BN * 128, 1024);
        uint64_t ad[4], bd[4];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          ad[kk] = pd + (uint64_t)((kk * 32) >> 4);
          bd[kk] = vd + (uint64_t)((kk * 2048) >> 4);
        }
        umma_f16_x4(tmem + 256 + DH * g, ad, bd, idO, o_acc[g]);
        o_acc[g] = 1u;
        umma_commit(&pv_done[g]);
      };
      mbar_wait(q_full, 0);
      issue_s_both(0);
      for (int j = 0; j < nkv; ++j) {
        if (j + 1 < nkv) issue_s_both(j + 1);  // run S ahead by one tile
        FTRACE(j * 16 + 0);
        if (j >= start0) issue_pv(0, j - start0, j);
        FTRACE(j * 16 + 1);
        if (has1) issue_pv(1, j, j);
        FTRACE(j * 16 + 2);
        umma_commit(&v_empty[j % NST]);
      }
    }
  } else {
    // ---------------- softmax warpgroups: warps 0-3 -> Q tile 0, warps 4-7 -> Q tile 1 ----------------
    const int g = warp >> 2;
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const int qi = q0 + 128 * g + r;
    const int ntile = g ? (has1 ? nkv : 0) : nkv0;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const uint32_t tO = tmem + lane_off + 256 + DH * g;
    const float sl = use_alibi ? exp2f(-8.0f * (float)(h + 1) / (float)H) * 1.4426950408889634f : 0.0f;
    float m = -1e30f, l = 0.f;  // finite: a row whose first (diagonal) tile is fully masked keeps alpha = 1, p = 0
    for (int j = 0; j < ntile; ++j) {
      const int k0 = (ntile - 1 - j) * BN;  // diagonal tile first: the running max settles at once
      const int bb = j & 1;
      const bool diag = k0 + BN > qi - r;  // tile reaches this Q tile's diagonal
      const uint32_t tS = tmem + lane_off + 64 * (2 * g + bb);
      const uint32_t prow = sP + g * Cf::PT + r * 128;
      mbar_wait(&s_full[2 * g + bb], (j >> 1) & 1);
      if (quad == 0 && lane == 0) FTRACE((j + (g ? 0 : start0)) * 16 + 3 + 2 * g);
      tc_fence_after();
      uint32_t v[64];
      tmem_ld_32x32b_x32(tS, *reinterpret_cast<uint32_t(*)[32]>(&v[0]));
      tmem_ld_32x32b_x32(tS + 32, *reinterpret_cast<uint32_t(*)[32]>(&v[32]));
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[2 * g + bb]);  // S buffer free for S(j+2)
      const float base = sl * (float)(k0 - qi);
      float pm[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) pm[u] = -INFINITY;
      if (diag) {
#pragma unroll
        for (int i = 0; i < 64; ++i) {
          float x = fmaf(__uint_as_float(v[i]), scale_log2, fmaf(sl, (float)i, base));
          x = (k0 + i > qi) ? -INFINITY : x;
          v[i] = __float_as_uint(x);
          pm[i & 7] = fmaxf(pm[i & 7], x);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 64; ++i) {
          const float x = fmaf(__uint_as_float(v[i]), scale_log2, fmaf(sl, (float)i, base));
          v[i] = __float_as_uint(x);
          pm[i & 7] = fmaxf(pm[i & 7], x);
        }
      }
      const float mx = fmaxf(fmaxf(fmaxf(pm[0], pm[1]), fmaxf(pm[2], pm[3])), fmaxf(fmaxf(pm[4], pm[5]), fmaxf(pm[6], pm[7])));
      // Dead rows: every x < m - 127, so every p = ex2.approx.ftz(x - m) is exactly 0 (the
      // ALiBi bias drives far keys there). A warp whose 32 rows are all dead skips the exps;
      // a block dead in all four warps skips its PV MMA and is marked for the backward.
      // Bit-identical to computing it: the skipped terms are exact zeros.
      const bool wdead = __all_sync(0xffffffffu, mx < m - 127.0f);
      // lazy rescale (FA4-style): keep the running max unless it grows by more than 8 (log2 units)
      const float m_new = (mx > m + 8.0f) ? mx : m;
      const float alpha = ex2(m - m_new);
      // P buffer [g] was last read by PV(j-1); O then holds exactly PV(0..j-1)
      if (j >= 1) mbar_wait(&pv_done[g], (j - 1) & 1);
      if (lane == 0) dead_flag[4 * g + quad] = wdead ? 1 : 0;
      if (wdead) {
#pragma unroll
        for (int q = 0; q < 8; ++q)
          asm volatile("st.shared.v4.b32 [%0], {%1,%1,%1,%1};" ::"r"(prow + ((q ^ (r & 7)) << 4)), "r"(0u));
        fence_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[g]);
        continue;
      }
      float ps[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float p[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          p[i] = ex2(__uint_as_float(v[8 * q + i]) - m_new);
          ps[i] += p[i];
        }
        const uint32_t addr = prow + (((q) ^ (r & 7)) << 4);
        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(pack_bf16(p[0], p[1])),
                     "r"(pack_bf16(p[2], p[3])), "r"(pack_bf16(p[4], p[5])), "r"(pack_bf16(p[6], p[7])));
      }
      const float rs = ((ps[0] + ps[1]) + (ps[2] + ps[3])) + ((ps[4] + ps[5]) + (ps[6] + ps[7]));
      l = l * alpha + rs;
      m = m_new;
      if (j > 0 && __any_sync(0xffffffffu, alpha != 1.0f)) {
        tc_fence_after();  // O holds exactly PV(0..j-1) (waited above)
#pragma unroll
        for (int c = 0; c < DH / 32; ++c) {
          uint32_t o[32];
          tmem_ld_32x32b_x32(tO + c * 32, o);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          tmem_st_32x32b_x32(tO + c * 32, o);
        }
        tmem_st_wait();
      }
      tc_fence_before();
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[g]);
      if (quad == 0 && lane == 0) FTRACE((j + (g ? 0 : start0)) * 16 + 4 + 2 * g);
    }
    if (ntile > 0) {  // warps of an absent second Q tile (T % 256 == 128) have nothing to write
      const int jl = ntile - 1;
      mbar_wait(&pv_done[g], jl & 1);
      tc_fence_after();
      const float il = 1.0f / l;
      __nv_bfloat16* orow = out + ((int64_t)row0 + qi) * d + h * DH;
#pragma unroll
      for (int c = 0; c < DH / 32; ++c) {
        uint32_t o[32];
        tmem_ld_32x32b_x32(tO + c * 32, o);
        tmem_ld_wait();
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float* f = reinterpret_cast<const float*>(o) + 8 * q;
          uint4 pk = make_uint4(pack_bf16(f[0] * il, f[1] * il), pack_bf16(f[2] * il, f[3] * il),
                                pack_bf16(f[4] * il, f[5] * il), pack_bf16(f[6] * il, f[7] * il));
          *reinterpret_cast<uint4*>(orow + c * 32 + 8 * q) = pk;
        }
      }
      lse2[(int64_t)bh * T + qi] = m + log2f(l);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 g_enc_attn = nullptr;

template <int DH>
int attn_fwd_tc_launch(const void* qkv, void* o, float* lse, uint8_t* live, int B, int T, int H, int use_alibi,
                       cudaStream_t st) {
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
  CUtensorMap tmq, tm;
  cuuint64_t dims[3] = {64, (cuuint64_t)B * T, (cuuint64_t)(3 * d / 64)};
  cuuint64_t strides[2] = {(cuuint64_t)3 * d * 2, 128};
  cuuint32_t es[3] = {1, 1, 1};
  for (int which = 0; which < 2; ++which) {
    cuuint32_t box[3] = {64, (cuuint32_t)(which ? Cf::BN : 128), DH / 64};  // Q: 128 rows, K/V: 64 rows
    CUresult r = g_enc_attn(which ? &tm : &tmq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(qkv), dims,
                            strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("attn tensor map encode failed: %d", (int)r);
      return FB_CUDA_ERROR;
    }
  }
  auto k = attn_fwd_tc_kernel<DH>;
  FB_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM));
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)DH);
  k<<<dim3((T + 255) / 256, B * H), 320, Cf::SMEM, st>>>(tmq, tm, (__nv_bfloat16*)o, lse, live, T, H, scale_log2,
                                                          use_alibi);
  FB_LAUNCH_CHECK();
  return FB_OK;
}

#ifdef FB_ATTN_TRACE
extern "C" int fb_attn_trace_read_fwd(unsigned long long* out, int n) {
  return cudaMemcpyFromSymbol(out, g_attn_trace_fwd, n * sizeof(unsigned long long)) == cudaSuccess ? 0 : 2;
}
#endif
template int attn_fwd_tc_launch<64>(const void*, void*, float*, uint8_t*, int, int, int, int, cudaStream_t);
template int attn_fwd_tc_launch<128>(const void*, void*, float*, uint8_t*, int, int, int, int, cudaStream_t);

}  // namespace fb
