// Causal ALiBi attention FORWARD on the 5th-generation tensor cores (tcgen05 + TMEM + TMA).
//
// Reference: fedforge/model.py:92-98 (scores/sqrt(dh) + alibi bias, softmax, PV) with
// slope_h = 2^(-8(h+1)/H) (model.py:46-50). Outputs: o [B*T][d] bf16 and
// lse2 [B][H][T] (base-2 log-sum-exp, consumed by the backward).
//
// CTA = a PAIR of 128-row query tiles g = 0, 1 of one (b, h) (the last pair holds one tile
// when T % 256 == 128); KV tiles of 128 keys walked from the diagonal DOWN, so the row max
// settles in the first tile and the lazy O rescale almost never fires. Heaviest pairs
// launch first.
//   TMEM (512 columns): S_g = Q_g K^T at [128 g, 128 g + 128) f32; the softmax writes
//   P_g (bf16 pairs) back over S_g's lower 64 columns, and PV reads it from there as an
//   A-from-TMEM MMA, so P never touches shared memory. O_g at 256 + DH g.
//   Why: the previous design (64-key tiles, P staged in smem, SS MMAs) was bound by smem
//   bandwidth: an N=64 SS MMA reads 6 KB of operands for 32 cycles of math and measured
//   48.7 cycles (tools/mma_chain.cu); the P stores added another quarter of the traffic.
//   warp 8     TMA producer: Q once, then K(t), V(t) into NST-deep rings.
//   warp 9     TMEM owner + single-thread MMA issuer. Per step t and tile g, once P_g(t) is
//              in TMEM: PV_g(t), then S_g(t+1) (tcgen05 MMAs execute in issue order, so
//              S_g(t+1) overwrites P_g(t) only after PV_g(t) has read it).
//   warps 0-3 (g = 0), 4-7 (g = 1): softmax, thread = query row = TMEM lane: exp2 with the
//              ALiBi bias folded into one FFMA, lazy (threshold 8, log2 units) in-TMEM
//              rescale of O, exact dead-block detection (below).
// The issue scheduler favours high warp ids, so the two single-thread control warps sit
// above the softmax warps.
#include <cudaTypedefs.h>

#include <type_traits>

#include "common.cuh"
#include "sm100.cuh"

namespace fb {
using namespace sm100;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// D[tmem] (+)= A[tmem] * B[smem]: A (M x 16) from TMEM, lane = row, 8 columns of bf16 pairs
// (layout checked by tools/ts_mma_test.cu)
__device__ __forceinline__ void umma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// Packed f32x2 math (FFMA2 / FADD2 on sm_100) and the 3-input max (FMNMX3): the softmax is
// issue-bound next to the MUFU, so every element-wise op counts.
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
__device__ __forceinline__ float2 fsub2(float2 a, float2 b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(u64of(a)), "l"(u64of(b)));
  return f2of(r);
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(u64of(a)), "l"(u64of(b)));
  return f2of(r);
}
// 2^x for a pair on the FMA pipe (FA4's MUFU offload): x = j + f with j = rint(x) (the 1.5*2^23
// magic add), 2^f on [-0.5, 0.5] by a degree-3 minimax polynomial (max rel. error 7.5e-5, far
// below the bf16 rounding of P), 2^j spliced into the exponent field. x is clamped at -127, where
// the spliced scale is exactly 0: like ex2.approx.ftz, every x <= -127 gives an exact 0.
__device__ __forceinline__ float2 exp2_poly2(float2 x) {
  x = make_float2(fmaxf(x.x, -127.f), fmaxf(x.y, -127.f));
  const float2 magic = make_float2(12582912.f, 12582912.f);
  const float2 t = fadd2(x, magic);
  const float2 f = fsub2(x, fsub2(t, magic));  // f = x - rint(x), exact
  float2 pp = ffma2(make_float2(0.055172716f, 0.055172716f), f, make_float2(0.24261133f, 0.24261133f));
  pp = ffma2(pp, f, make_float2(0.69326079f, 0.69326079f));
  pp = ffma2(pp, f, make_float2(0.99992806f, 0.99992806f));
  const float2 sc = make_float2(__uint_as_float((__float_as_uint(t.x) << 23) + 0x3F800000u),
                                __uint_as_float((__float_as_uint(t.y) << 23) + 0x3F800000u));
  return fmul2(pp, sc);
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
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

template <int DH>
struct AttnTcCfg {
  static constexpr int BN = 128;                 // keys per KV tile
  static constexpr int NST = DH == 128 ? 2 : 4;  // K and V ring depth
  static constexpr int QT = 128 * DH * 2;        // one 128-row Q tile
  static constexpr int KT = BN * DH * 2;         // one K (or V) tile
  static constexpr int Q_OFF = 0;                // [2] Q tiles
  static constexpr int K_OFF = 2 * QT;           // [NST]
  static constexpr int V_OFF = K_OFF + NST * KT; // [NST]
  static constexpr int CB_OFF = V_OFF + NST * KT;  // column bias table sl * i, i < BN (f32)
  static constexpr int BAR_OFF = CB_OFF + BN * 4;
  static constexpr int SMEM = BAR_OFF + 256 + 1024;
  static_assert(SMEM <= 232448, "attention forward smem");
};

constexpr int kProducerWarp = 8, kMmaWarp = 9;

template <int DH>
__global__ void __launch_bounds__(320, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tmq, const __grid_constant__ CUtensorMap tm,
                       const __grid_constant__ CUtensorMap tmo,
                       __nv_bfloat16* __restrict__ out, float* __restrict__ lse2, uint8_t* __restrict__ live_map,
                       int T, int H, float scale_log2, int use_alibi) {
  using Cf = AttnTcCfg<DH>;
  constexpr int BN = Cf::BN, NST = Cf::NST;
  // measured (tools/attn_bench.py, isolated, C3 / C4 head shapes): every 3rd pair at dh 64
  // (0.123 vs 0.1255 ms off, 0.132 at every 2nd), every 8th at dh 128 (0.172 vs 0.174, 0.187 at
  // every 2nd): the softmax is latency-bound more than MUFU-bound, so only a small share pays
#ifndef FB_POLY64
#define FB_POLY64 3
#endif
#ifndef FB_POLY128
#define FB_POLY128 8
#endif
  constexpr int kPolyEvery = DH == 64 ? FB_POLY64 : FB_POLY128;
  // dh 64: S_g 128 + O_g 64 columns leave room for P_g in its own 64 columns [384 + 64 g), so S_g(t+1)
  // need not wait for PV_g(t); dh 128 writes P over S_g's lower half
#ifdef FB_EXP_NOSEPP
  constexpr int kSepP = 0;
#else
  constexpr int kSepP = DH == 64 ? 1 : 0;
#endif
  constexpr uint32_t kPOff = kSepP ? 384 : 0;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023) & ~1023u) - raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Cf::BAR_OFF);
  uint64_t* q_full = bar + 0;
  uint64_t* k_full = bar + 1;          // [NST]
  uint64_t* k_empty = k_full + NST;    // [NST]
  uint64_t* v_full = k_empty + NST;    // [NST]
  uint64_t* v_empty = v_full + NST;    // [NST]
  uint64_t* s_full = v_empty + NST;    // [g]  S_g(t) in TMEM (committed after PV_g(t-1))
  uint64_t* p_full = s_full + 2;       // [g]  P_g(t) in TMEM (4 warps)
  uint64_t* o_done = p_full + 2;       // [g]  every PV_g done
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);
  uint8_t* dead_flag = reinterpret_cast<uint8_t*>(tmem_slot + 1);  // [g][warp of the group]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int npair = (T + 255) / 256;
  const int pb = npair - 1 - blockIdx.x;  // heavy pairs first
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const int d = H * DH;
  const int row0 = b * T;
  const int q0 = pb * 256;
  const bool has1 = q0 + 256 <= T;
  const int nkv0 = (q0 + 128) / BN;               // key tiles of Q tile 0
  const int nkv = has1 ? (q0 + 256) / BN : nkv0;  // key tiles of the pair
  const int start0 = nkv - nkv0;                  // Q tile 0 joins the diagonal-down walk here

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
    for (int g = 0; g < 2; ++g) {
      mbar_init(&s_full[g], 1);
      mbar_init(&p_full[g], 4);
      mbar_init(&o_done[g], 1);
    }
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tmem_alloc(tmem_slot, 512);
  const float sl = use_alibi ? exp2f(-8.0f * (float)(h + 1) / (float)H) * 1.4426950408889634f : 0.0f;
  float* colb = reinterpret_cast<float*>(smem + Cf::CB_OFF);
  if (threadIdx.x < BN) colb[threadIdx.x] = sl * (float)threadIdx.x;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t sQ = smem_u32(smem + Cf::Q_OFF), sK = smem_u32(smem + Cf::K_OFF), sV = smem_u32(smem + Cf::V_OFF);

  if (warp == kProducerWarp) {
    if (lane == 0) {
      const int zq = (h * DH) / 64, zk = (d + h * DH) / 64, zv = (2 * d + h * DH) / 64;
      mbar_arrive_expect_tx(q_full, (has1 ? 2 : 1) * Cf::QT);
      tma_load_3d(smem + Cf::Q_OFF, &tmq, q_full, 0, row0 + q0, zq);
      if (has1) tma_load_3d(smem + Cf::Q_OFF + Cf::QT, &tmq, q_full, 0, row0 + q0 + 128, zq);
      for (int t = 0; t < nkv; ++t) {
        const int s = t % NST;
        const uint32_t ph = ((t / NST) & 1) ^ 1;
        const int krow = row0 + (nkv - 1 - t) * BN;
        mbar_wait(&k_empty[s], ph);
        mbar_arrive_expect_tx(&k_full[s], Cf::KT);
        tma_load_3d(smem + Cf::K_OFF + s * Cf::KT, &tm, &k_full[s], 0, krow, zk);
        mbar_wait(&v_empty[s], ph);
        mbar_arrive_expect_tx(&v_full[s], Cf::KT);
        tma_load_3d(smem + Cf::V_OFF + s * Cf::KT, &tm, &v_full[s], 0, krow, zv);
      }
    }
  } else if (warp == kMmaWarp) {
    if (lane == 0) {
      constexpr uint32_t idS = idesc_bf16_f32(128, BN, 0, 0);  // Q (K-major) x K (K-major)
      constexpr uint32_t idO = idesc_bf16_f32(128, DH, 0, 1);  // P (TMEM) x V (MN-major)
      auto active = [&](int g, int t) { return g ? has1 : (t >= start0); };
      auto issue_s = [&](int g, int t) {
        mbar_wait(&k_full[t % NST], (t / NST) & 1);
        tc_fence_after();
        const uint64_t qd = smem_desc_sw128(sQ + g * Cf::QT, 16, 1024);
        const uint64_t kd = smem_desc_sw128(sK + (t % NST) * Cf::KT, 16, 1024);
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk)  // K-major SW128: k steps +32 B, 64-column chunks (rows x 128 B) apart
          umma_f16(tmem + 128 * g, qd + (uint64_t)(((kk >> 2) * (128 * 128) + (kk & 3) * 32) >> 4),
                   kd + (uint64_t)(((kk >> 2) * (BN * 128) + (kk & 3) * 32) >> 4), idS, kk > 0);
      };
      uint32_t o_acc[2] = {0u, 0u};
      // P_g(t) released by the softmax: returns whether the whole block is dead
      auto wait_p = [&](int g, int t) {
        const int j = g ? t : t - start0;
        mbar_wait(&p_full[g], j & 1);
        FTRACE(t * 16 + 8 + g);
        // all four warps found every p of their rows exactly 0: the block adds nothing to O
        const bool dead = *reinterpret_cast<volatile uint32_t*>(dead_flag + 4 * g) == 0x01010101u;
        if (live_map) {
          uint8_t* e = live_map + ((int64_t)bh * (T / 128) + (q0 >> 7) + g) * (T / 64) + 2 * (nkv - 1 - t);
          e[0] = e[1] = dead ? 0 : 1;
        }
        mbar_wait(&v_full[t % NST], (t / NST) & 1);
        return dead;
      };
      auto mma_pv = [&](int g, int t) {
        tc_fence_after();
        const uint64_t vd = smem_desc_sw128(sV + (t % NST) * Cf::KT, BN * 128, 1024);
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk)  // V MN-major: 16 keys = 16 rows x 128 B
          umma_ts(tmem + 256 + DH * g, tmem + kPOff + 64 * g * kSepP + 128 * g * (1 - kSepP) + 8 * kk,
                  vd + (uint64_t)((kk * 2048) >> 4), idO, o_acc[g] | (uint32_t)(kk > 0));
        o_acc[g] = 1u;
      };
      mbar_wait(q_full, 0);
      for (int g = 0; g < 2; ++g)
        if (active(g, 0)) {
          issue_s(g, 0);
          umma_commit(&s_full[g]);
        }
      umma_commit(&k_empty[0]);
      for (int t = 0; t < nkv; ++t) {
        for (int g = 0; g < 2; ++g) {
          const bool now = active(g, t), next = t + 1 < nkv && active(g, t + 1);
          if constexpr (kSepP) {
            // P has its own columns: S_g(t+1) goes in first (the next softmax starts one PV
            // earlier), PV_g(t) behind it, and o_done[g] tells the softmax when O and the P
            // columns are free again
            const bool dead = now && wait_p(g, t);
            if (next) {
              issue_s(g, t + 1);
              umma_commit(&s_full[g]);
              FTRACE(t * 16 + 12 + g);
            }
            if (now) {
              if (!dead) mma_pv(g, t);
              umma_commit(&o_done[g]);
              FTRACE(t * 16 + 10 + g);
            }
          } else {
            if (now && !wait_p(g, t)) mma_pv(g, t);
            FTRACE(t * 16 + 10 + g);
            if (next) {
              issue_s(g, t + 1);
              umma_commit(&s_full[g]);  // also covers PV_g(t): the softmax may rescale O / overwrite P
              FTRACE(t * 16 + 12 + g);
            } else if (now) {
              umma_commit(&o_done[g]);
            }
          }
        }
        umma_commit(&v_empty[t % NST]);
        if (t + 1 < nkv) umma_commit(&k_empty[(t + 1) % NST]);
      }
    }
  } else {
    // ---------------- softmax: warps 0-3 -> Q tile 0, warps 4-7 -> Q tile 1 ----------------
    const int g = warp >> 2;
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const int qi = q0 + 128 * g + r;
    const int ntile = g ? (has1 ? nkv : 0) : nkv0;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const uint32_t tS = tmem + lane_off + 128 * g;
    const uint32_t tP = kSepP ? tmem + lane_off + kPOff + 64 * g : tS;  // own columns, or over S's lower 64
    const uint32_t tO = tmem + lane_off + 256 + DH * g;
    // Scores in log2 units: x_i = s_i c + sl (k0 + i - qi) = y_i + base with the
    // tile-independent y_i = s_i c + colb[i] (colb = sl i, an smem broadcast table) and the
    // per-row, per-tile scalar base = sl (k0 - qi); the max and the exp argument then work
    // on y with base folded into one scalar.
    const float2 c2 = make_float2(scale_log2, scale_log2);
    const float4* colb4 = reinterpret_cast<const float4*>(colb);
    float m = -1e30f, l = 0.f;
    for (int j = 0; j < ntile; ++j) {
      const int k0 = (ntile - 1 - j) * BN;
      const bool diag = (j == 0);  // Q tiles and key tiles are both 128 wide: only the first crosses
      mbar_wait(&s_full[g], j & 1);
      if (quad == 0 && lane == 0) FTRACE((j + (g ? 0 : start0)) * 16 + 0 + g);
      tc_fence_after();
      uint32_t v[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) tmem_ld_32x32b_x32(tS + 32 * c, *reinterpret_cast<uint32_t(*)[32]>(&v[32 * c]));
      tmem_ld_wait();
      const float base = sl * (float)(k0 - qi);
      float pm[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
      auto scan = [&](auto diag_t) {  // y = s c + colb (masked above the diagonal), running maxima
        constexpr bool kDiag = decltype(diag_t)::value;
#pragma unroll
        for (int i = 0; i < 128; i += 4) {
          const float4 cb = colb4[i >> 2];
          float2 y0 = ffma2(make_float2(__uint_as_float(v[i]), __uint_as_float(v[i + 1])), c2, make_float2(cb.x, cb.y));
          float2 y1 = ffma2(make_float2(__uint_as_float(v[i + 2]), __uint_as_float(v[i + 3])), c2, make_float2(cb.z, cb.w));
          if constexpr (kDiag) {  // key k0 + i > qi  <=>  i > r (k0 = qi - r on the diagonal tile)
            if (i > r) y0.x = -INFINITY;
            if (i + 1 > r) y0.y = -INFINITY;
            if (i + 2 > r) y1.x = -INFINITY;
            if (i + 3 > r) y1.y = -INFINITY;
          }
          v[i] = __float_as_uint(y0.x);
          v[i + 1] = __float_as_uint(y0.y);
          v[i + 2] = __float_as_uint(y1.x);
          v[i + 3] = __float_as_uint(y1.y);
          pm[(i >> 2) & 3] = fmax3(pm[(i >> 2) & 3], fmax3(y0.x, y0.y, y1.x), y1.y);
        }
      };
      if (diag) scan(std::true_type{});
      else scan(std::false_type{});
      const float mx = fmax3(pm[0], pm[1], fmaxf(pm[2], pm[3])) + base;
      if (quad == 0 && lane == 0) FTRACE((j + (g ? 0 : start0)) * 16 + 2 + g);
      // Dead rows: every x < m - 127, so every p = ex2.approx.ftz(x - m) is exactly 0 (the
      // ALiBi bias drives far keys there). A warp whose 32 rows are all dead skips the exps;
      // a block dead in all four warps skips its PV MMA and is marked for the backward.
      // Bit-identical to computing it: the skipped terms are exact zeros.
      const bool wdead = __all_sync(0xffffffffu, mx < m - 127.0f);
      if (kSepP && j > 0) {  // PV_g(j-1) done: O = PV(0..j-1) and the P columns are free
        mbar_wait(&o_done[g], (j - 1) & 1);
        tc_fence_after();
      }
      if (lane == 0) dead_flag[4 * g + quad] = wdead ? 1 : 0;
      if (wdead) {
        uint32_t z[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) z[i] = 0u;
        tmem_st_32x32b_x32(tP, z);
        tmem_st_32x32b_x32(tP + 32, z);
      } else {
        // lazy rescale (FA4-style): keep the running max unless it grows by more than 8 (log2 units)
        const float m_new = (mx > m + 8.0f) ? mx : m;
        const float alpha = ex2(m - m_new);
        const float2 sh = make_float2(base - m_new, base - m_new);  // x - m_new = y + sh
        float2 ps[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        // P (bf16 pairs) over S's lower 64 columns: all of S is in registers by now
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t pk[32];
#pragma unroll
          for (int c = 0; c < 32; ++c) {
            const int i = 64 * hh + 2 * c;
            const float2 a = fadd2(make_float2(__uint_as_float(v[i]), __uint_as_float(v[i + 1])), sh);
            // every kPolyEvery-th pair on the FMA pipe: the MUFU (16 ex2 / clk / SM) bounds the
            // softmax, at dh 64 by twice the MMA time
            const float2 p = (kPolyEvery > 0 && c % kPolyEvery == kPolyEvery - 1) ? exp2_poly2(a)
                                                                                 : make_float2(ex2(a.x), ex2(a.y));
            ps[c & 3] = fadd2(ps[c & 3], p);
            pk[c] = pack_bf16(p.x, p.y);
          }
          tmem_st_32x32b_x32(tP + 32 * hh, pk);
        }
        const float2 s01 = fadd2(fadd2(ps[0], ps[1]), fadd2(ps[2], ps[3]));
        const float rs = s01.x + s01.y;
        l = l * alpha + rs;
        m = m_new;
        // O holds exactly PV(0..j-1): s_full(j) was committed after PV(j-1) (dh 128) or
        // o_done was waited for above (dh 64)
        if (j > 0 && __any_sync(0xffffffffu, alpha != 1.0f)) {
#pragma unroll
          for (int c = 0; c < DH / 32; ++c) {
            uint32_t o[32];
            tmem_ld_32x32b_x32(tO + c * 32, o);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tmem_st_32x32b_x32(tO + c * 32, o);
          }
        }
      }
      if (quad == 0 && lane == 0) FTRACE((j + (g ? 0 : start0)) * 16 + 4 + g);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[g]);
      if (quad == 0 && lane == 0) FTRACE((j + (g ? 0 : start0)) * 16 + 6 + g);
    }
    if (ntile > 0) {  // warps of an absent second Q tile (T % 256 == 128) have nothing to write
      mbar_wait(&o_done[g], kSepP ? ((ntile - 1) & 1) : 0);
      tc_fence_after();
      const float il = 1.0f / l;
      // O staged in this group's Q tile (free once every PV_g, hence every S_g, completed) in
      // the 128B-swizzled [chunk][row][64] layout it was loaded in, then one TMA bulk store
      uint8_t* stg = smem + Cf::Q_OFF + g * Cf::QT;
#pragma unroll
      for (int c = 0; c < DH / 32; ++c) {
        uint32_t o[32];
        tmem_ld_32x32b_x32(tO + c * 32, o);
        tmem_ld_wait();
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float* f = reinterpret_cast<const float*>(o) + 8 * q;
          const int jj = (c & 1) * 4 + q;
          *reinterpret_cast<uint4*>(stg + (c >> 1) * (128 * 128) + r * 128 + ((jj ^ (r & 7)) << 4)) =
              make_uint4(pack_bf16(f[0] * il, f[1] * il), pack_bf16(f[2] * il, f[3] * il),
                         pack_bf16(f[4] * il, f[5] * il), pack_bf16(f[6] * il, f[7] * il));
        }
      }
      lse2[(int64_t)bh * T + qi] = m + log2f(l);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync %0, 128;" ::"r"(2 + g) : "memory");
      if (quad == 0 && lane == 0) {
        tma_store_3d(&tmo, stg, 0, row0 + q0 + 128 * g, (h * DH) / 64);
        bulk_commit();
        bulk_wait_read<0>();
      }
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
    cuuint32_t box[3] = {64, (cuuint32_t)(which ? Cf::BN : 128), DH / 64};  // Q: 128 rows, K/V: BN rows
    CUresult r = g_enc_attn(which ? &tm : &tmq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(qkv), dims,
                            strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("attn tensor map encode failed: %d", (int)r);
      return FB_CUDA_ERROR;
    }
  }
  CUtensorMap tmo;  // O store boxes: 128 rows x DH (DH / 64 chunks of 64 columns), 128B swizzle
  {
    cuuint64_t odims[3] = {64, (cuuint64_t)B * T, (cuuint64_t)(d / 64)};
    cuuint64_t ostrides[2] = {(cuuint64_t)d * 2, 128};
    cuuint32_t obox[3] = {64, 128, DH / 64};
    CUresult r = g_enc_attn(&tmo, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, o, odims, ostrides, obox, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("attn output tensor map encode failed: %d", (int)r);
      return FB_CUDA_ERROR;
    }
  }
  auto k = attn_fwd_tc_kernel<DH>;
  FB_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM));
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)DH);
  k<<<dim3((T + 255) / 256, B * H), 320, Cf::SMEM, st>>>(tmq, tm, tmo, (__nv_bfloat16*)o, lse, live, T, H, scale_log2,
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
