// Causal ALiBi attention BACKWARD on tcgen05 / TMEM / TMA.
//
// Reference: gradient of fedforge/model.py:92-98 (scores/sqrt(dh) + ALiBi bias, softmax,
// PV); the bias is constant, so dq = dS k / sqrt(dh), dk = dS^T q / sqrt(dh),
// dv = P^T dO, dS = P o (dP - D), D = rowsum(dO o O) (from the out-projection dgrad
// epilogue, or the pre-pass in attn.cu).
//
// CTA = 128 keys of one (b, h); loop over the causal query tiles. Two kernels:
//   dh = 128  attn_bwd_tc64_kernel: 64-query tiles, P^T in TMEM (dV as an A-from-TMEM
//             MMA), 3-stage Q/dO ring, dQ^T = K^T dS^T in its own TMEM columns, one TMA
//             bulk reduce-add per warpgroup per tile, software pipeline across query
//             tiles (elementwise of tile t+1 overlaps the MMAs of tile t).
//   dh = 64   attn_bwd_tcd64_kernel: 128-query tiles, dQ = dS K with dS^T read as an
//             MN-major A operand, P/dS share a double-buffered smem tile.
// Warp roles in both: warp 0 TMA producer, warp 1 TMEM owner + single-thread MMA issuer,
// warps 2-9 elementwise (thread = TMEM lane).
#include <cudaTypedefs.h>
#include <stdlib.h>

#include <type_traits>

#include "common.cuh"
#include "sm100.cuh"

namespace fb {
using namespace sm100;

#ifdef FB_ATTN_TRACE
__device__ unsigned long long g_attn_trace[4096];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TRACE(slot) do { if (blockIdx.x == 4 && blockIdx.y == 5) g_attn_trace[(slot)] = gtimer(); } while (0)
#else
#define TRACE(slot) do {} while (0)
#endif

__device__ __forceinline__ float ex2b(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// packed f32x2 (FFMA2 / FADD2 / FMUL2): per-lane identical to the scalar ops, half the issue slots
__device__ __forceinline__ float2 pk_fma(float2 a, float2 b, float2 c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(r)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
        "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return *reinterpret_cast<float2*>(&r);
}
__device__ __forceinline__ float2 pk_sub(float2 a, float2 b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;"
      : "=l"(r)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)));
  return *reinterpret_cast<float2*>(&r);
}
__device__ __forceinline__ float2 pk_mul(float2 a, float2 b) {
  unsigned long long r;
  asm("mul.rn.f32x2 %0, %1, %2;"
      : "=l"(r)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)));
  return *reinterpret_cast<float2*>(&r);
}
// D[tmem] (+)= A[tmem] * B[smem]: A (M x 16) from TMEM, lane = row, 8 columns of bf16 pairs
__device__ __forceinline__ void umma_ts_b(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

// Live query tiles of one key block, from the forward's dead-block map (attn_tc.cu): a
// forward block (128 queries x 64 keys) whose every p was exactly 0 has P = 0 and dS = 0
// here too (lse >= the forward's running max), so its MMAs and exps are skipped. Warp 0
// ballots the map into a compact list tl[0..n) of tile offsets from `first`; every role then
// walks the same list. qshift: log2(query tile / 128) + 1 maps a tile to its forward row
// block (64-row tiles: >> 1, 128-row tiles: >> 0).
__device__ __forceinline__ void build_live_list(const uint8_t* __restrict__ live, int bh, int T, int kb, int first,
                                                int ntiles, int qshift, uint8_t* tl, uint32_t* nlive) {
  const int lane = threadIdx.x & 31;
  int n = 0;
  for (int base = 0; base < ntiles; base += 32) {
    const int t = base + lane;
    bool ok = t < ntiles;
    if (ok && live) {
      const uint8_t* row = live + ((int64_t)bh * (T / 128) + ((first + t) >> qshift)) * (T / 64) + 2 * kb;
      ok = (row[0] | row[1]) != 0;
    }
    const uint32_t m = __ballot_sync(0xffffffffu, ok);
    if (ok) tl[n + __popc(m & ((1u << lane) - 1u))] = (uint8_t)t;
    n += __popc(m);
  }
  if (lane == 0) *nlive = (uint32_t)n;
}

// dQ box out: TMA reduce-add into the f32 accumulator (z = 0), or, in deterministic mode, a
// plain TMA store into key block kb's own partial slab (z = kb) that dq_finalize_det_kernel
// sums in ascending kb order (the reduce-adds of different key blocks land in arrival order).
__device__ __forceinline__ void dq_out_box(const CUtensorMap* map, uint32_t src, int x, int y, int kb, int det) {
  if (det)
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(src), "r"(x), "r"(y), "r"(kb)
                 : "memory");
  else
    asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(src), "r"(x), "r"(y), "r"(0)
                 : "memory");
}

// ---------------------------------------------------------------------------------------
// dh = 128 variant with 64-query tiles and a software pipeline across query tiles:
//   MMA order per tile t:  [pds_full(t)]  S^T(t+1), dP^T(t+1)  dV(t)  dK(t)  [dq_empty(t-1)] dQ^T(t)
//   so the elementwise phase of tile t+1 overlaps the dV/dK/dQ MMAs of tile t.
//   dQ^T = K^T dS^T (M = dh = 128, N = 64 queries, K = 128 keys) has its own TMEM columns;
//   it is drained by the compute warps of the NEXT tile through a dedicated smem staging
//   box and ONE TMA bulk reduce-add per tile (dq rows [q0, q0+64) x 128 cols).
//   P^T (bf16 pairs) goes to TMEM and dV = P^T dO is an A-from-TMEM MMA; the 32 KB of
//   smem that P^T no longer needs buy a third Q / dO stage, so the loads of tile t+2 are
//   not gated by the dV / dK MMAs of tile t.
//   TMEM: S^T [0,64)  dP^T [64,128)  dQ^T [128,192)  P^T[2] [192,256)  dV [256,384)  dK [384,512).
struct AttnBwd64Cfg {
  static constexpr int DH = 128;
  static constexpr int NQ = 3;                   // Q / dO ring depth
  static constexpr int KT = 128 * DH * 2;        // K or V tile (128 keys)
  static constexpr int QT = 64 * DH * 2;         // Q or dO tile (64 queries)
  static constexpr int PT = 128 * 64 * 2;        // dS^T tile (128 keys x 64 q)
  static constexpr int K_OFF = 0;
  static constexpr int V_OFF = K_OFF + KT;
  static constexpr int Q_OFF = V_OFF + KT;       // [NQ]
  static constexpr int O_OFF = Q_OFF + NQ * QT;  // [NQ]
  static constexpr int S_OFF = O_OFF + NQ * QT;  // [2]
  static constexpr int X_OFF = S_OFF + 2 * PT;   // dQ staging: 64 rows x 128 f32
  static constexpr int L_OFF = X_OFF + 64 * DH * 4;  // e[2][64], D[2][64]
  static constexpr int BAR_OFF = L_OFF + 4 * 64 * 4;
  static constexpr int SMEM = BAR_OFF + 512 + 1024;  // mbarriers, TMEM slot, live count + list; align
  static_assert(SMEM <= 232448, "attention bwd (dh 128) smem");
};

__global__ void __launch_bounds__(320, 1)
    attn_bwd_tc64_kernel(const __grid_constant__ CUtensorMap tm_kv, const __grid_constant__ CUtensorMap tm_q,
                         const __grid_constant__ CUtensorMap tm_do, const __grid_constant__ CUtensorMap tm_dq,
                         const __grid_constant__ CUtensorMap tm_dkv,
                         const float* __restrict__ lse2, const uint8_t* __restrict__ live, const float* __restrict__ Dd,
                         __nv_bfloat16* __restrict__ dqkv, int T, int H, float scale_log2, float scale, int use_alibi,
                         int det) {
  using Cf = AttnBwd64Cfg;
  constexpr int DH = Cf::DH;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023) & ~1023u) - raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Cf::BAR_OFF);
  uint64_t* kv_full = bar + 0;
  uint64_t* q_full = bar + 1;     // [NQ]
  uint64_t* o_full = bar + 4;     // [NQ]
  uint64_t* q_empty = bar + 7;    // [NQ]
  uint64_t* o_empty = bar + 10;   // [NQ]
  uint64_t* s_full = bar + 13;
  uint64_t* pds_full = bar + 14;
  uint64_t* pds_free = bar + 15;  // [2]
  uint64_t* dq_full = bar + 17;
  uint64_t* dq_empty = bar + 18;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 20);
  uint32_t* nlive_p = tmem_slot + 1;
  uint8_t* tl = reinterpret_cast<uint8_t*>(tmem_slot + 2);
  float* sE0 = reinterpret_cast<float*>(smem + Cf::L_OFF);  // e[2][64] (double-buffered)
  float* sD0 = sE0 + 128;                                     // D[2][64]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kb = blockIdx.x;
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const int d = H * DH;
  const int row0 = b * T;
  const int k0 = kb * 128;
  const int first = 2 * kb, ntiles = T / 64 - 2 * kb;  // causal: query tiles of 64 from the block's diagonal

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_kv);
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_do);
    tma_prefetch(&tm_dq);
    mbar_init(kv_full, 1);
    for (int s = 0; s < Cf::NQ; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&o_full[s], 1);
      mbar_init(&q_empty[s], 1);
      mbar_init(&o_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) mbar_init(&pds_free[s], 1);
    mbar_init(s_full, 1);
    mbar_init(pds_full, 8);
    mbar_init(dq_full, 1);
    mbar_init(dq_empty, 8);
    fence_barrier_init();
#ifndef FB_EXP_LATE_KV
    // K / V of this key block are needed whatever is live: start them before the TMEM
    // allocation, the live-list build and the CTA barrier
    {
      const int zk = (d + h * DH) / 64, zv = (2 * d + h * DH) / 64;
      mbar_arrive_expect_tx(kv_full, 2 * Cf::KT);
      tma_load_3d(smem + Cf::K_OFF, &tm_kv, kv_full, 0, row0 + k0, zk);
      tma_load_3d(smem + Cf::V_OFF, &tm_kv, kv_full, 0, row0 + k0, zv);
    }
#endif
  }
  if (warp == 2) build_live_list(live, bh, T, kb, first, ntiles, 1, tl, nlive_p);
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int nlive = (int)*nlive_p;
  const uint32_t sK = smem_u32(smem + Cf::K_OFF), sV = smem_u32(smem + Cf::V_OFF), sQ0 = smem_u32(smem + Cf::Q_OFF),
                 sO0 = smem_u32(smem + Cf::O_OFF), sS0 = smem_u32(smem + Cf::S_OFF), sX = smem_u32(smem + Cf::X_OFF);

  if (warp == 0) {
    if (lane == 0) {
      const int zq = (h * DH) / 64, zo = (h * DH) / 64;
#ifdef FB_EXP_LATE_KV
      const int zk = (d + h * DH) / 64, zv = (2 * d + h * DH) / 64;
      mbar_arrive_expect_tx(kv_full, 2 * Cf::KT);
      tma_load_3d(smem + Cf::K_OFF, &tm_kv, kv_full, 0, row0 + k0, zk);
      tma_load_3d(smem + Cf::V_OFF, &tm_kv, kv_full, 0, row0 + k0, zv);
#endif
      for (int t = 0; t < nlive; ++t) {
        const int s = t % Cf::NQ;
        const uint32_t ph = (t / Cf::NQ) & 1;
        const int q0 = (first + tl[t]) * 64;
        mbar_wait(&q_empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&q_full[s], Cf::QT);
        tma_load_3d(smem + Cf::Q_OFF + s * Cf::QT, &tm_q, &q_full[s], 0, row0 + q0, zq);
        mbar_wait(&o_empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&o_full[s], Cf::QT);
        tma_load_3d(smem + Cf::O_OFF + s * Cf::QT, &tm_do, &o_full[s], 0, row0 + q0, zo);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idSP = idesc_bf16_f32(128, 64, 0, 0);  // S^T, dP^T: M=128 keys, N=64 q, K=dh
      constexpr uint32_t idKV = idesc_bf16_f32(128, DH, 0, 1);  // dV, dK: K-major A (P^T/dS^T), MN-major B
      constexpr uint32_t idQ = idesc_bf16_f32(128, 64, 1, 1);   // dQ^T = K^T dS^T: MN-major A and B
      const uint32_t tS = tmem, tP = tmem + 64, tQ = tmem + 128, tPT = tmem + 192, tV = tmem + 256, tK = tmem + 384;
      auto issue_sp = [&](int t) {
        const int s = t % Cf::NQ;
        const uint32_t sph = (t / Cf::NQ) & 1;
        const uint32_t sQ = sQ0 + s * Cf::QT, sO = sO0 + s * Cf::QT;
        mbar_wait(&q_full[s], sph);
        mbar_wait(&o_full[s], sph);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const uint32_t aoff = (kk >> 2) * (128 * 128) + (kk & 3) * 32;
          const uint32_t boff = (kk >> 2) * (64 * 128) + (kk & 3) * 32;
          umma_f16(tS, smem_desc_sw128(sK + aoff, 16, 1024), smem_desc_sw128(sQ + boff, 16, 1024), idSP, kk > 0);
          umma_f16(tP, smem_desc_sw128(sV + aoff, 16, 1024), smem_desc_sw128(sO + boff, 16, 1024), idSP, kk > 0);
        }
        umma_commit(s_full);
      };
      mbar_wait(kv_full, 0);  // also when no tile is live: the K/V loads must land before exit
      if (nlive > 0) issue_sp(0);
      for (int t = 0; t < nlive; ++t) {
        const int s = t % Cf::NQ, b2 = t & 1;
        const uint32_t ph = t & 1;
        const uint32_t sQ = sQ0 + s * Cf::QT, sO = sO0 + s * Cf::QT;
        const uint32_t sS = sS0 + b2 * Cf::PT;
        mbar_wait(pds_full, ph);  // S^T/dP^T(t) consumed; P^T(t), dS^T(t) in smem
        TRACE(16 * t + 0);
        if (t + 1 < nlive) issue_sp(t + 1);
        TRACE(16 * t + 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)  // dV += P^T dO   (K = 64 queries; P^T from TMEM)
          umma_ts_b(tV, tPT + 32 * b2 + 8 * kk, smem_desc_sw128(sO + kk * 2048, 64 * 128, 1024), idKV, (t | kk) > 0);
        umma_commit(&o_empty[s]);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)  // dK += dS^T Q
          umma_f16(tK, smem_desc_sw128(sS + kk * 32, 16, 1024), smem_desc_sw128(sQ + kk * 2048, 64 * 128, 1024), idKV,
                   (t | kk) > 0);
        umma_commit(&q_empty[s]);
        TRACE(16 * t + 2);
        mbar_wait(dq_empty, ph ^ 1);  // dQ^T(t-1) drained
        TRACE(16 * t + 3);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)  // dQ^T = K^T dS^T   (K = 128 keys)
          umma_f16(tQ, smem_desc_sw128(sK + kk * 2048, 128 * 128, 1024), smem_desc_sw128(sS + kk * 2048, 8192, 1024),
                   idQ, kk > 0);
        umma_commit(dq_full);
        umma_commit(&pds_free[b2]);
      }
    }
  } else {
    // compute warps: g = warpgroup (query-column half), quad = TMEM lane quadrant
    const int g = (warp - 2) >> 2;
    const int quad = warp & 3;
    const int r = quad * 32 + lane;  // TMEM lane: key row (elementwise) / dh index (dQ^T drain)
    const int kj = k0 + r;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const float sl = use_alibi ? exp2f(-8.0f * (float)(h + 1) / (float)H) * 1.4426950408889634f : 0.0f;
    const float slk = sl * (float)kj;
    const int tid = threadIdx.x - 64;  // 0..255
    float* Xs = reinterpret_cast<float*>(smem + Cf::X_OFF);
    auto drain = [&](int t) {  // dQ^T(t) -> staging [64 q][128 dh] -> TMA reduce-add into dq rows
      // each warpgroup g drains its own 32 query rows (one 32 x 128 reduce box, its own named
      // barrier), so the two groups do not wait for each other's elementwise skew
      const int q0 = (first + tl[t]) * 64;
      mbar_wait(dq_full, t & 1);
      tc_fence_after();
      uint32_t v[32];
      tmem_ld_32x32b_x32(tmem + 128 + lane_off + 32 * g, v);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dq_empty);
      // this group's staging box of the previous reduce must have been read by TMA
      if ((tid & 127) == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      asm volatile("bar.sync %0, 128;" ::"r"(2 + g) : "memory");
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        const float2 sv2 = pk_mul(make_float2(__uint_as_float(v[i]), __uint_as_float(v[i + 1])), make_float2(scale, scale));
        Xs[(32 * g + i) * DH + r] = sv2.x;
        Xs[(32 * g + i + 1) * DH + r] = sv2.y;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync %0, 128;" ::"r"(2 + g) : "memory");
      if ((tid & 127) == 0) {
        dq_out_box(&tm_dq, sX + g * 32 * DH * 4, h * DH, row0 + q0 + 32 * g, kb, det);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    };
    // e/D of tile t live in buffer t & 1; tile t+1's are prefetched before drain(t-1), whose
    // warpgroup barriers publish them (all readers of that buffer finished tile t-1 earlier)
    auto load_ed = [&](int t) {
      const int q0 = (first + tl[t]) * 64;
      float* E = sE0 + (t & 1) * 64;
      float* Dv = sD0 + (t & 1) * 64;
      // warpgroup g reads only queries [32g, 32g + 32) of the tile, so it loads that half itself
      // (published to its readers by its own drain barriers)
      const int j = tid & 127, qq = 32 * g + (j & 31);
      if (j < 32) E[qq] = sl * (float)(q0 + qq) + lse2[(int64_t)bh * T + q0 + qq];
      else if (j < 64) Dv[qq] = Dd[(int64_t)bh * T + q0 + qq];
    };
    if (nlive > 0) load_ed(0);
    asm volatile("bar.sync 1, 256;" ::: "memory");
    for (int t = 0; t < nlive; ++t) {
      const int s = t & 1;
      const uint32_t ph = t & 1;
      const int q0 = (first + tl[t]) * 64;
      const bool diag = (tl[t] < 2);  // the two 64-row tiles that cross the key block's diagonal
      const float* sE = sE0 + (t & 1) * 64;
      const float* sD = sD0 + (t & 1) * 64;
      if (warp == 2 && lane == 0) TRACE(16 * t + 4);
      mbar_wait(s_full, ph);
      if (warp == 2 && lane == 0) TRACE(16 * t + 5);
      tc_fence_after();
      uint32_t sv[32], pv[32];
      tmem_ld_32x32b_x32(tmem + lane_off + 32 * g, sv);
      tmem_ld_32x32b_x32(tmem + 64 + lane_off + 32 * g, pv);
      tmem_ld_wait();
      // P^T / dS^T buffers [s] were last read by the MMAs of tile t-2
      if (t >= 2) mbar_wait(&pds_free[s], ((t >> 1) & 1) ^ 1);
      const uint32_t srow = sS0 + s * Cf::PT + r * 128;
      uint32_t ptm[16];  // this group's 32 queries of P^T as bf16 pairs -> TMEM (A of the dV MMA)
      // the causal mask only touches the two diagonal tiles: the other tiles run a mask-free copy
      auto elementwise = [&](auto diag_t) {
      constexpr bool kDiag = decltype(diag_t)::value;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        float p[8], ds[8];
        const float4 e0 = *reinterpret_cast<const float4*>(sE + 32 * g + q * 8);
        const float4 e1 = *reinterpret_cast<const float4*>(sE + 32 * g + q * 8 + 4);
        const float4 d0 = *reinterpret_cast<const float4*>(sD + 32 * g + q * 8);
        const float4 d1 = *reinterpret_cast<const float4*>(sD + 32 * g + q * 8 + 4);
        const float ev[8] = {e0.x, e0.y, e0.z, e0.w, e1.x, e1.y, e1.z, e1.w};
        const float dv[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
          const float2 be = pk_sub(make_float2(slk, slk), make_float2(ev[i], ev[i + 1]));
          const float2 x = pk_fma(make_float2(__uint_as_float(sv[q * 8 + i]), __uint_as_float(sv[q * 8 + i + 1])),
                                  make_float2(scale_log2, scale_log2), be);
          const int ql = 32 * g + q * 8 + i;
          p[i] = (kDiag && q0 + ql < kj) ? 0.f : ex2b(x.x);
          p[i + 1] = (kDiag && q0 + ql + 1 < kj) ? 0.f : ex2b(x.y);
          const float2 dd = pk_sub(make_float2(__uint_as_float(pv[q * 8 + i]), __uint_as_float(pv[q * 8 + i + 1])),
                                   make_float2(dv[i], dv[i + 1]));
          const float2 d2 = pk_mul(make_float2(p[i], p[i + 1]), dd);
          ds[i] = d2.x;
          ds[i + 1] = d2.y;
        }
        const int kc = 4 * g + q;
        const uint32_t sw = ((kc ^ (r & 7)) << 4);
#pragma unroll
        for (int i = 0; i < 4; ++i) ptm[4 * q + i] = pack_bf16(p[2 * i], p[2 * i + 1]);
        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(srow + sw), "r"(pack_bf16(ds[0], ds[1])),
                     "r"(pack_bf16(ds[2], ds[3])), "r"(pack_bf16(ds[4], ds[5])), "r"(pack_bf16(ds[6], ds[7])));
      }
      };
      if (diag) elementwise(std::true_type{});
      else elementwise(std::false_type{});
      tmem_st_32x32b_x16(tmem + 192 + 32 * s + 16 * g + lane_off, ptm);
      tmem_st_wait();
      tc_fence_before();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(pds_full);
      if (warp == 2 && lane == 0) TRACE(16 * t + 6);
      if (t + 1 < nlive) load_ed(t + 1);
      if (t > 0) drain(t - 1);  // overlaps the MMAs of tile t
      else asm volatile("bar.sync 1, 256;" ::: "memory");  // publish e/D(1) on the first tile
      if (warp == 2 && lane == 0) TRACE(16 * t + 7);
    }
    if (nlive > 0) drain(nlive - 1);
#ifdef FB_EXP_FULL_WAIT
    if ((tid & 127) == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
#else
    // exit only needs the staging box read (the reduce-adds complete with the grid)
    if ((tid & 127) == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
#endif
    // dK, dV (the last dK/dV MMAs completed before the last dq_full): staged in the now idle
    // Q / dO rings in the 128B-swizzled [chunk][key][64] layout of the K tile, then one TMA
    // bulk store per matrix (coalesced, asynchronous) instead of per-row global stores
    uint8_t* stK = smem + Cf::Q_OFF;
    uint8_t* stV = smem + Cf::O_OFF;
#pragma unroll 1
    for (int c = 0; c < DH / 64; ++c) {
      uint32_t kv[32], vv[32];
      const uint32_t col = (DH / 2) * g + c * 32;
      tmem_ld_32x32b_x32(tmem + 384 + lane_off + col, kv);
      tmem_ld_32x32b_x32(tmem + 256 + lane_off + col, vv);
      tmem_ld_wait();
      if (nlive == 0) {  // every query of this key block was dead: dK = dV = 0
#pragma unroll
        for (int i = 0; i < 32; ++i) kv[i] = vv[i] = 0u;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float* fk = reinterpret_cast<const float*>(kv) + 8 * q;
        const float* fv = reinterpret_cast<const float*>(vv) + 8 * q;
        const int jj = 4 * c + q;  // 16-byte piece of this row within chunk g
        const uint32_t off = g * (128 * 128) + r * 128 + ((jj ^ (r & 7)) << 4);
        *reinterpret_cast<uint4*>(stK + off) =
            make_uint4(pack_bf16(fk[0] * scale, fk[1] * scale), pack_bf16(fk[2] * scale, fk[3] * scale),
                       pack_bf16(fk[4] * scale, fk[5] * scale), pack_bf16(fk[6] * scale, fk[7] * scale));
        *reinterpret_cast<uint4*>(stV + off) = make_uint4(
            pack_bf16(fv[0], fv[1]), pack_bf16(fv[2], fv[3]), pack_bf16(fv[4], fv[5]), pack_bf16(fv[6], fv[7]));
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("bar.sync 1, 256;" ::: "memory");
    if (tid == 0) {
      tma_store_3d(&tm_dkv, stK, 0, row0 + k0, (d + h * DH) / 64);
      tma_store_3d(&tm_dkv, stV, 0, row0 + k0, (2 * d + h * DH) / 64);
      bulk_commit();
      bulk_wait_read<0>();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ---------------------------------------------------------------------------------------
// dh = 64 variant of the pipelined backward: 128-query tiles, dQ = dS K (M = 128 queries,
// A = the dS^T smem image read MN-major) in its own TMEM columns, two 128 x 32 TMA
// reduce boxes per tile (one per warpgroup), same cross-tile pipeline as tc64.
//   TMEM: S^T [0,128)  dP^T [128,256)  dQ [256,320)  dV [320,384)  dK [384,448).
struct AttnBwdD64Cfg {
  static constexpr int DH = 64;
  static constexpr int KT = 128 * DH * 2;        // K or V tile (128 keys)
  static constexpr int QT = 128 * DH * 2;        // Q or dO tile (128 queries)
  static constexpr int PT = 128 * 128 * 2;       // P^T or dS^T tile
  static constexpr int K_OFF = 0;
  static constexpr int V_OFF = K_OFF + KT;
  static constexpr int Q_OFF = V_OFF + KT;       // [2]
  static constexpr int O_OFF = Q_OFF + 2 * QT;   // [2]
  static constexpr int P_OFF = O_OFF + 2 * QT;   // [2] P^T, then dS^T (shared per buffer)
  static constexpr int X_OFF = P_OFF + 2 * PT;   // dQ staging: 2 boxes of 128 rows x 32 f32 (swizzled)
  static constexpr int L_OFF = X_OFF + 128 * DH * 4;
  static constexpr int BAR_OFF = L_OFF + 2 * 128 * 4;
  static constexpr int SMEM = BAR_OFF + 512 + 1024;
  static_assert(SMEM <= 232448, "attention bwd (dh 64) smem");
};

__global__ void __launch_bounds__(320, 1)
    attn_bwd_tcd64_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                          const __grid_constant__ CUtensorMap tm_dq, const __grid_constant__ CUtensorMap tm_dkv, const float* __restrict__ lse2,
                          const uint8_t* __restrict__ live, const float* __restrict__ Dd,
                          __nv_bfloat16* __restrict__ dqkv, int T, int H,
                          float scale_log2, float scale, int use_alibi, int det) {
  using Cf = AttnBwdD64Cfg;
  constexpr int DH = Cf::DH;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw + 1023) & ~1023u) - raw);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Cf::BAR_OFF);
  uint64_t* kv_full = bar + 0;
  uint64_t* q_full = bar + 1;     // [2]
  uint64_t* o_full = bar + 3;     // [2]
  uint64_t* q_empty = bar + 5;    // [2]
  uint64_t* o_empty = bar + 7;    // [2]
  uint64_t* s_full = bar + 9;
  uint64_t* p_full = bar + 10;
  uint64_t* pds_free = bar + 11;  // [2]
  uint64_t* dq_full = bar + 13;
  uint64_t* dq_empty = bar + 14;
  uint64_t* p_free = bar + 15;
  uint64_t* ds_full = bar + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 17);
  uint32_t* nlive_p = tmem_slot + 1;
  uint8_t* tl = reinterpret_cast<uint8_t*>(tmem_slot + 2);
  float* sE = reinterpret_cast<float*>(smem + Cf::L_OFF);
  float* sD = sE + 128;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kb = blockIdx.x;
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const int d = H * DH;
  const int row0 = b * T;
  const int k0 = kb * 128;
  const int first = kb, ntiles = T / 128 - kb;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_qkv);
    tma_prefetch(&tm_do);
    tma_prefetch(&tm_dq);
    mbar_init(kv_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&o_full[s], 1);
      mbar_init(&q_empty[s], 1);
      mbar_init(&o_empty[s], 1);
      mbar_init(&pds_free[s], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(p_full, 8);
    mbar_init(p_free, 1);
    mbar_init(ds_full, 8);
    mbar_init(dq_full, 1);
    mbar_init(dq_empty, 8);
    fence_barrier_init();
  }
  if (warp == 2) build_live_list(live, bh, T, kb, first, ntiles, 0, tl, nlive_p);
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int nlive = (int)*nlive_p;
  const uint32_t sK = smem_u32(smem + Cf::K_OFF), sV = smem_u32(smem + Cf::V_OFF), sQ0 = smem_u32(smem + Cf::Q_OFF),
                 sO0 = smem_u32(smem + Cf::O_OFF), sP0 = smem_u32(smem + Cf::P_OFF), sX = smem_u32(smem + Cf::X_OFF);

  if (warp == 0) {
    if (lane == 0) {
      const int zq = (h * DH) / 64, zk = (d + h * DH) / 64, zv = (2 * d + h * DH) / 64, zo = (h * DH) / 64;
      mbar_arrive_expect_tx(kv_full, 2 * Cf::KT);
      tma_load_3d(smem + Cf::K_OFF, &tm_qkv, kv_full, 0, row0 + k0, zk);
      tma_load_3d(smem + Cf::V_OFF, &tm_qkv, kv_full, 0, row0 + k0, zv);
      for (int t = 0; t < nlive; ++t) {
        const int s = t & 1;
        const uint32_t ph = (t >> 1) & 1;
        const int q0 = (first + tl[t]) * 128;
        mbar_wait(&q_empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&q_full[s], Cf::QT);
        tma_load_3d(smem + Cf::Q_OFF + s * Cf::QT, &tm_qkv, &q_full[s], 0, row0 + q0, zq);
        mbar_wait(&o_empty[s], ph ^ 1);
        mbar_arrive_expect_tx(&o_full[s], Cf::QT);
        tma_load_3d(smem + Cf::O_OFF + s * Cf::QT, &tm_do, &o_full[s], 0, row0 + q0, zo);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idSP = idesc_bf16_f32(128, 128, 0, 0);
      constexpr uint32_t idKV = idesc_bf16_f32(128, DH, 0, 1);
      constexpr uint32_t idQ = idesc_bf16_f32(128, DH, 1, 1);
      const uint32_t tS = tmem, tP = tmem + 128, tQ = tmem + 256, tV = tmem + 320, tK = tmem + 384;
      auto issue_sp = [&](int t) {
        const int s = t & 1;
        const uint32_t sph = (t >> 1) & 1;
        const uint32_t sQ = sQ0 + s * Cf::QT, sO = sO0 + s * Cf::QT;
        mbar_wait(&q_full[s], sph);
        mbar_wait(&o_full[s], sph);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          const uint32_t off = (kk & 3) * 32;
          umma_f16(tS, smem_desc_sw128(sK + off, 16, 1024), smem_desc_sw128(sQ + off, 16, 1024), idSP, kk > 0);
          umma_f16(tP, smem_desc_sw128(sV + off, 16, 1024), smem_desc_sw128(sO + off, 16, 1024), idSP, kk > 0);
        }
        umma_commit(s_full);
      };
      mbar_wait(kv_full, 0);  // also when no tile is live: the K/V loads must land before exit
      if (nlive > 0) issue_sp(0);
      for (int t = 0; t < nlive; ++t) {
        const int s = t & 1;
        const uint32_t ph = t & 1;
        const uint32_t sQ = sQ0 + s * Cf::QT, sO = sO0 + s * Cf::QT;
        const uint32_t sP = sP0 + s * Cf::PT, sS = sP;  // dS^T overwrites P^T after dV
        mbar_wait(p_full, ph);
        if (t + 1 < nlive) issue_sp(t + 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // dV += P^T dO  (K = 128 queries)
          const uint32_t aoff = (kk >> 2) * (128 * 128) + (kk & 3) * 32;
          umma_f16(tV, smem_desc_sw128(sP + aoff, 16, 1024), smem_desc_sw128(sO + kk * 2048, 128 * 128, 1024), idKV,
                   (t | kk) > 0);
        }
        umma_commit(&o_empty[s]);
        umma_commit(p_free);
        mbar_wait(ds_full, ph);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {  // dK += dS^T Q
          const uint32_t aoff = (kk >> 2) * (128 * 128) + (kk & 3) * 32;
          umma_f16(tK, smem_desc_sw128(sS + aoff, 16, 1024), smem_desc_sw128(sQ + kk * 2048, 128 * 128, 1024), idKV,
                   (t | kk) > 0);
        }
        umma_commit(&q_empty[s]);
        mbar_wait(dq_empty, ph ^ 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)  // dQ = dS K  (K = 128 keys); dS read as MN-major
          umma_f16(tQ, smem_desc_sw128(sS + kk * 2048, 128 * 128, 1024), smem_desc_sw128(sK + kk * 2048, 128 * 128, 1024),
                   idQ, kk > 0);
        umma_commit(dq_full);
        umma_commit(&pds_free[s]);
      }
    }
  } else {
    const int g = (warp - 2) >> 2;
    const int quad = warp & 3;
    const int r = quad * 32 + lane;  // TMEM lane: key row (elementwise) / query row (dQ drain)
    const int kj = k0 + r;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const float sl = use_alibi ? exp2f(-8.0f * (float)(h + 1) / (float)H) * 1.4426950408889634f : 0.0f;
    const float slk = sl * (float)kj;
    const int tid = threadIdx.x - 64;
    const uint32_t xbox = sX + g * 16384;  // this warpgroup's 128 x 32 f32 staging box
    auto drain = [&](int t) {
      const int q0 = (first + tl[t]) * 128;
      mbar_wait(dq_full, t & 1);
      tc_fence_after();
      uint32_t v[32];
      tmem_ld_32x32b_x32(tmem + 256 + lane_off + 32 * g, v);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dq_empty);
      if (quad == 0 && lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      asm volatile("bar.sync %0, 128;" ::"r"(2 + g) : "memory");
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t addr = xbox + r * 128 + ((q ^ (r & 7)) << 4);
        asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "f"(__uint_as_float(v[4 * q]) * scale),
                     "f"(__uint_as_float(v[4 * q + 1]) * scale), "f"(__uint_as_float(v[4 * q + 2]) * scale),
                     "f"(__uint_as_float(v[4 * q + 3]) * scale));
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("bar.sync %0, 128;" ::"r"(2 + g) : "memory");
      if (quad == 0 && lane == 0) {
        dq_out_box(&tm_dq, xbox, h * DH + 32 * g, row0 + q0, kb, det);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    };
    for (int t = 0; t < nlive; ++t) {
      const int s = t & 1;
      const uint32_t ph = t & 1;
      const int q0 = (first + tl[t]) * 128;
      const bool diag = (tl[t] == 0);
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (tid < 128) sE[tid] = sl * (float)(q0 + tid) + lse2[(int64_t)bh * T + q0 + tid];
      else sD[tid - 128] = Dd[(int64_t)bh * T + q0 + tid - 128];
      asm volatile("bar.sync 1, 256;" ::: "memory");
      mbar_wait(s_full, ph);
      tc_fence_after();
      uint32_t sv[2][32], pv[2][32];
      tmem_ld_32x32b_x32(tmem + lane_off + 64 * g, sv[0]);
      tmem_ld_32x32b_x32(tmem + lane_off + 64 * g + 32, sv[1]);
      tmem_ld_32x32b_x32(tmem + 128 + lane_off + 64 * g, pv[0]);
      tmem_ld_32x32b_x32(tmem + 128 + lane_off + 64 * g + 32, pv[1]);
      tmem_ld_wait();
      if (t >= 2) mbar_wait(&pds_free[s], ((t >> 1) & 1) ^ 1);
      const uint32_t prow = sP0 + s * Cf::PT + r * 128;
      uint32_t dsp[32];  // dS^T packed bf16x2, written once dV has consumed P^T
      // the causal mask only touches the diagonal tile: the other tiles run a mask-free copy
      auto elementwise = [&](auto diag_t) {
        constexpr bool kDiag = decltype(diag_t)::value;
#pragma unroll
        for (int c = 0; c < 2; ++c) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            float p[8], ds[8];
            const int qb = 64 * g + 32 * c + q * 8;
            const float4 e0 = *reinterpret_cast<const float4*>(sE + qb), e1 = *reinterpret_cast<const float4*>(sE + qb + 4);
            const float4 d0 = *reinterpret_cast<const float4*>(sD + qb), d1 = *reinterpret_cast<const float4*>(sD + qb + 4);
            const float ev[8] = {e0.x, e0.y, e0.z, e0.w, e1.x, e1.y, e1.z, e1.w};
            const float dv[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
#pragma unroll
            for (int i = 0; i < 8; i += 2) {  // packed f32x2, per-lane identical to the scalar form
              const int ql = qb + i;
              const float2 be = pk_sub(make_float2(slk, slk), make_float2(ev[i], ev[i + 1]));
              const float2 x = pk_fma(make_float2(__uint_as_float(sv[c][q * 8 + i]), __uint_as_float(sv[c][q * 8 + i + 1])),
                                      make_float2(scale_log2, scale_log2), be);
              p[i] = (kDiag && q0 + ql < kj) ? 0.f : ex2b(x.x);
              p[i + 1] = (kDiag && q0 + ql + 1 < kj) ? 0.f : ex2b(x.y);
              const float2 d2 = pk_mul(make_float2(p[i], p[i + 1]),
                                       pk_sub(make_float2(__uint_as_float(pv[c][q * 8 + i]),
                                                          __uint_as_float(pv[c][q * 8 + i + 1])),
                                              make_float2(dv[i], dv[i + 1])));
              ds[i] = d2.x;
              ds[i + 1] = d2.y;
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) dsp[c * 16 + q * 4 + i] = pack_bf16(ds[2 * i], ds[2 * i + 1]);
            const int kc = 8 * g + 4 * c + q;  // 8-query chunk 0..15
            const uint32_t sw = (kc >> 3) * (128 * 128) + (((kc & 7) ^ (r & 7)) << 4);
            asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(prow + sw), "r"(pack_bf16(p[0], p[1])),
                         "r"(pack_bf16(p[2], p[3])), "r"(pack_bf16(p[4], p[5])), "r"(pack_bf16(p[6], p[7])));
          }
        }
      };
      if (diag) elementwise(std::true_type{});
      else elementwise(std::false_type{});
      tc_fence_before();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      mbar_wait(p_free, ph);  // dV(t) has read P^T: overwrite with dS^T
#pragma unroll
      for (int c = 0; c < 2; ++c) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int kc = 8 * g + 4 * c + q;
          const uint32_t sw = (kc >> 3) * (128 * 128) + (((kc & 7) ^ (r & 7)) << 4);
          asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(prow + sw), "r"(dsp[c * 16 + q * 4]),
                       "r"(dsp[c * 16 + q * 4 + 1]), "r"(dsp[c * 16 + q * 4 + 2]), "r"(dsp[c * 16 + q * 4 + 3]));
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(ds_full);
      if (t > 0) drain(t - 1);
    }
    if (nlive > 0) drain(nlive - 1);
    if (quad == 0 && lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    // dK / dV staged in the idle Q / dO buffers (128B-swizzled [key][64]), two TMA bulk stores
    uint8_t* stK = smem + Cf::Q_OFF;
    uint8_t* stV = smem + Cf::O_OFF;
    uint32_t kv[32], vv[32];
    tmem_ld_32x32b_x32(tmem + 384 + lane_off + 32 * g, kv);
    tmem_ld_32x32b_x32(tmem + 320 + lane_off + 32 * g, vv);
    tmem_ld_wait();
    if (nlive == 0) {  // every query of this key block was dead: dK = dV = 0
#pragma unroll
      for (int i = 0; i < 32; ++i) kv[i] = vv[i] = 0u;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float* fk = reinterpret_cast<const float*>(kv) + 8 * q;
      const float* fv = reinterpret_cast<const float*>(vv) + 8 * q;
      const int jj = 4 * g + q;
      const uint32_t off = r * 128 + ((jj ^ (r & 7)) << 4);
      *reinterpret_cast<uint4*>(stK + off) =
          make_uint4(pack_bf16(fk[0] * scale, fk[1] * scale), pack_bf16(fk[2] * scale, fk[3] * scale),
                     pack_bf16(fk[4] * scale, fk[5] * scale), pack_bf16(fk[6] * scale, fk[7] * scale));
      *reinterpret_cast<uint4*>(stV + off) = make_uint4(pack_bf16(fv[0], fv[1]), pack_bf16(fv[2], fv[3]),
                                                        pack_bf16(fv[4], fv[5]), pack_bf16(fv[6], fv[7]));
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("bar.sync 1, 256;" ::: "memory");
    if (tid == 0) {
      tma_store_3d(&tm_dkv, stK, 0, row0 + k0, (d + h * DH) / 64);
      tma_store_3d(&tm_dkv, stV, 0, row0 + k0, (2 * d + h * DH) / 64);
      bulk_commit();
      bulk_wait_read<0>();
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

static int encode_box(CUtensorMap* m, const void* base, int64_t rows, int cols, int box_rows, int box_chunks) {
  cuuint64_t dims[3] = {64, (cuuint64_t)rows, (cuuint64_t)(cols / 64)};
  cuuint64_t strides[2] = {(cuuint64_t)cols * 2, 128};
  cuuint32_t box[3] = {64, (cuuint32_t)box_rows, (cuuint32_t)box_chunks};
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

static int attn_bwd_tc64_launch(const void* qkv, const void* dO, const float* lse, const uint8_t* live,
                                const float* Dbuf, float* dq,
                                void* dqkv, int B, int T, int H, int use_alibi, int det, cudaStream_t st) {
  using Cf = AttnBwd64Cfg;
  constexpr int DH = 128;
  const int d = H * DH;
  CUtensorMap tkv, tq, to, tdq;
  int rc = encode_box(&tkv, qkv, (int64_t)B * T, 3 * d, 128, DH / 64);
  if (rc) return rc;
  rc = encode_box(&tq, qkv, (int64_t)B * T, 3 * d, 64, DH / 64);
  if (rc) return rc;
  rc = encode_box(&to, dO, (int64_t)B * T, d, 64, DH / 64);
  if (rc) return rc;
  {
    // {d, B*T, slabs}: slabs = 1 (reduce-add accumulator) or T/128 (deterministic per-key-block partials)
    const int slabs = det ? T / 128 : 1;
    cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)B * T, (cuuint64_t)slabs};
    cuuint64_t strides[2] = {(cuuint64_t)d * 4, (cuuint64_t)B * T * d * 4};
    cuuint32_t box[3] = {DH, 32, 1};  // one 32-query box per warpgroup
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = g_enc_bwd(&tdq, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, dq, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("attn bwd dq tensor map encode failed: %d", (int)r);
      return FB_CUDA_ERROR;
    }
  }
  CUtensorMap tdkv;  // dK / dV store boxes: 128 keys x 128 dh (two 64-column chunks), 128B swizzle
  rc = encode_box(&tdkv, dqkv, (int64_t)B * T, 3 * d, 128, DH / 64);
  if (rc) return rc;
  auto k = attn_bwd_tc64_kernel;
  FB_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM));
  const float scale = 1.0f / sqrtf((float)DH);
  k<<<dim3(T / 128, B * H), 320, Cf::SMEM, st>>>(tkv, tq, to, tdq, tdkv, lse, live, Dbuf, (__nv_bfloat16*)dqkv, T, H,
                                                 1.4426950408889634f * scale, scale, use_alibi, det);
  FB_LAUNCH_CHECK();
  return FB_OK;
}

static int attn_bwd_tcd64_launch(const void* qkv, const void* dO, const float* lse, const uint8_t* live,
                                 const float* Dbuf, float* dq,
                                 void* dqkv, int B, int T, int H, int use_alibi, int det, cudaStream_t st) {
  using Cf = AttnBwdD64Cfg;
  constexpr int DH = 64;
  const int d = H * DH;
  CUtensorMap tq, to, tdq;
  int rc = encode_box(&tq, qkv, (int64_t)B * T, 3 * d, 128, 1);
  if (rc) return rc;
  rc = encode_box(&to, dO, (int64_t)B * T, d, 128, 1);
  if (rc) return rc;
  {
    const int slabs = det ? T / 128 : 1;
    cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)B * T, (cuuint64_t)slabs};
    cuuint64_t strides[2] = {(cuuint64_t)d * 4, (cuuint64_t)B * T * d * 4};
    cuuint32_t box[3] = {32, 128, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = g_enc_bwd(&tdq, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, dq, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("attn bwd dq tensor map encode failed: %d", (int)r);
      return FB_CUDA_ERROR;
    }
  }
  CUtensorMap tdkv;  // dK / dV store boxes: 128 keys x 64 dh, 128B swizzle
  rc = encode_box(&tdkv, dqkv, (int64_t)B * T, 3 * d, 128, 1);
  if (rc) return rc;
  auto k = attn_bwd_tcd64_kernel;
  FB_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM));
  const float scale = 1.0f / sqrtf((float)DH);
  k<<<dim3(T / 128, B * H), 320, Cf::SMEM, st>>>(tq, to, tdq, tdkv, lse, live, Dbuf, (__nv_bfloat16*)dqkv, T, H,
                                                 1.4426950408889634f * scale, scale, use_alibi, det);
  FB_LAUNCH_CHECK();
  return FB_OK;
}

template <int DH>
int attn_bwd_tc_launch(const void* qkv, const void* dO, const float* lse, const uint8_t* live, const float* Dbuf,
                       float* dq, void* dqkv, int B, int T, int H, int use_alibi, int det, cudaStream_t st) {
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
  FB_REQUIRE(T <= 16384, "attn_bwd: T=%d above 16384", T);
  if (DH == 128) return attn_bwd_tc64_launch(qkv, dO, lse, live, Dbuf, dq, dqkv, B, T, H, use_alibi, det, st);
  if (DH == 64) return attn_bwd_tcd64_launch(qkv, dO, lse, live, Dbuf, dq, dqkv, B, T, H, use_alibi, det, st);
  return FB_UNSUPPORTED;
}

template int attn_bwd_tc_launch<64>(const void*, const void*, const float*, const uint8_t*, const float*, float*,
                                    void*, int, int, int, int, int, cudaStream_t);
template int attn_bwd_tc_launch<128>(const void*, const void*, const float*, const uint8_t*, const float*, float*,
                                     void*, int, int, int, int, int, cudaStream_t);

}  // namespace fb

#ifdef FB_ATTN_TRACE
extern "C" int fb_attn_trace_read(unsigned long long* out, int n) {
  return cudaMemcpyFromSymbol(out, fb::g_attn_trace, n * sizeof(unsigned long long)) == cudaSuccess ? 0 : 2;
}
#endif
