// Causal ALiBi attention BACKWARD on tcgen05 / TMEM / TMA.
//
// Reference: gradient of fedforge/model.py:92-98 (scores/sqrt(dh) + ALiBi bias, softmax,
// PV); the bias is constant, so dq = dS k / sqrt(dh), dk = dS^T q / sqrt(dh),
// dv = P^T dO, dS = P o (dP - D), D = rowsum(dO o O) (from the out-projection dgrad
// epilogue, or the pre-pass in attn.cu).
//
// CTA = 128 keys of one (b, h); loop over the causal query tiles. Two kernels:
//   dh = 128  attn_bwd_tc64_kernel: 64-query tiles, P^T in TMEM (dV as an A-from-TMEM
//             MMA), 2-stage Q/dO ring, dQ^T = K^T dS^T in its own TMEM columns, one
//             ordered dQ box per warpgroup per tile (dq_order), software pipeline across
//             query tiles (elementwise of tile t+1 overlaps the MMAs of tile t).
//   dh = 64   attn_bwd_tcd64_kernel: 128-query tiles, P^T in TMEM (A-from-TMEM dV), dS^T in a
//             double-buffered smem tile, dQ = dS K with dS^T read as an MN-major A operand.
// Warp roles in both: warp 0 TMA producer, warp 1 TMEM owner + single-thread MMA issuer,
// warps 2-9 elementwise (thread = TMEM lane), warps 10-11 ordered dQ output (dq_order).
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
#ifdef FB_ATTN_PROF  // per-CTA start / end / ns spent in sem_wait_eq / SM id (tools/attn_dq_prof.py)
__device__ unsigned long long g_attn_prof[8192 * 8];
__device__ __forceinline__ unsigned long long ptimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define PROF_CTA() (blockIdx.y * gridDim.x + blockIdx.x)
#define PROF_T0(v) const unsigned long long v = ptimer()
#define PROF_ADD(slot, v) do { if (PROF_CTA() < 8192) atomicAdd(&g_attn_prof[PROF_CTA() * 8 + (slot)], ptimer() - (v)); } while (0)
#else
#define PROF_T0(v) do {} while (0)
#define PROF_ADD(slot, v) do {} while (0)
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

// Ordered dQ accumulation (deterministic, no memset and no finalize pass).
// The dQ rows of 128-query block m receive one partial from every live key block kb <= m, and
// they arrive in DESCENDING kb order: CTA kb walks its query tiles upward from its diagonal, so
// the CTA of the larger kb reaches block m first (FA4's causal semaphore order). Every dQ box
// has a counter; the CTA of kb waits until it equals the number of live kb' in (kb, m], then
//   first contributor (count 0): TMA store of its partial into the f32 accumulator;
//   middle:                      TMA reduce-add (after the previous one COMPLETED);
//   last (no live kb' < kb):     acc + own partial in registers, bf16 straight into dqkv.
// A contributor bumps the counter one tile later, once its bulk op completed (the wait sits
// where the staging box is recycled anyway). The sum order is fixed by the live map alone, so
// dQ is bitwise reproducible. dq_order returns count | (last << 8) for (block m, key block kb);
// kb = -1 counts every live key block of row block m. One full warp calls it.
__device__ __forceinline__ uint32_t dq_order(const uint8_t* __restrict__ live, int bh, int T, int m, int kb) {
  const int lane = threadIdx.x & 31;
  uint32_t before = 0;
  bool later = false;
  for (int base = 0; base <= m; base += 32) {
    const int k = base + lane;
    bool ok = k <= m;
    if (ok && live) {
      const uint8_t* row = live + ((int64_t)bh * (T / 128) + m) * (T / 64) + 2 * k;
      ok = (row[0] | row[1]) != 0;
    }
    before += __popc(__ballot_sync(0xffffffffu, ok && k > kb));
    later |= __ballot_sync(0xffffffffu, ok && k < kb) != 0u;
  }
  return before | (later ? 0u : 0x100u);
}
// the same for one (m, kb) per lane (no ballot): the dQ warps tabulate 32 tiles at a time. The
// map row is read as 32-bit words (two key blocks each), all loads in flight together.
__device__ __forceinline__ uint32_t dq_order_lane(const uint8_t* __restrict__ live, int bh, int T, int m, int kb) {
  uint32_t before = 0;
  bool later = false;
  if (!live) {
    before = (uint32_t)(m > kb ? m - kb : 0);
    later = kb > 0;
  } else {
    const uint8_t* row = live + ((int64_t)bh * (T / 128) + m) * (T / 64);
    if ((T & 255) == 0) {
      const uint32_t* w = reinterpret_cast<const uint32_t*>(row);
      const int nw = m / 2 + 1;  // words holding key blocks 0..m
#pragma unroll 8
      for (int i = 0; i < nw; ++i) {
        const uint32_t x = __ldg(w + i);
#pragma unroll
        for (int hf = 0; hf < 2; ++hf) {
          const int k = 2 * i + hf;
          const bool ok = k <= m && ((x >> (16 * hf)) & 0xffffu) != 0u;
          before += (ok && k > kb) ? 1u : 0u;
          later |= ok && k < kb;
        }
      }
    } else {
      for (int k = 0; k <= m; ++k) {
        const bool ok = (row[2 * k] | row[2 * k + 1]) != 0;
        before += (ok && k > kb) ? 1u : 0u;
        later |= ok && k < kb;
      }
    }
  }
  return before | (later ? 0u : 0x100u);
}

// spin (one thread) until *p == v; a count above v or ~2^32 cycles without progress is a bug: trap
// instead of hanging the GPU
__device__ __forceinline__ void sem_wait_eq(const uint32_t* p, uint32_t v) {
#ifdef FB_ATTN_PROF
  const unsigned long long p0 = ptimer();
#endif
  const long long t0 = clock64();
  while (true) {
    uint32_t x;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(x) : "l"(p) : "memory");
    if (x == v) break;
    if (x > v || clock64() - t0 > (1ll << 32)) __trap();
    __nanosleep(64);
  }
  asm volatile("fence.proxy.async.global;" ::: "memory");  // later TMA reduce-adds see the acquired data
#ifdef FB_ATTN_PROF
  if (PROF_CTA() < 8192) atomicAdd(&g_attn_prof[PROF_CTA() * 8 + 2], ptimer() - p0);
#endif
}
// after cp.async.bulk.wait_group 0: publish this thread's completed bulk writes, bump the counter
__device__ __forceinline__ void sem_release(uint32_t* p) {
  asm volatile("fence.proxy.async.global;" ::: "memory");
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}
// a staged dQ box out (not the last contributor): TMA store for the first, reduce-add otherwise
__device__ __forceinline__ void dq_out_box(const CUtensorMap* map, uint32_t src, int x, int y, bool first) {
  if (first)
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(src), "r"(x), "r"(y), "r"(0)
                 : "memory");
  else
    asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(src), "r"(x), "r"(y), "r"(0)
                 : "memory");
}
// Row block kb of dQ gets no partial at all when every key block of it was dead (possible only
// if even the diagonal underflowed): the CTA of key block kb writes those rows' zeros. Called by
// whole warps (nthr threads, tid 0..nthr-1).
__device__ __forceinline__ void zero_dead_rows(const uint8_t* __restrict__ live, int bh, int T, int kb, int DH, int H,
                                               int row0, int h, __nv_bfloat16* __restrict__ dqkv, int tid, int nthr) {
  if (!live) return;
  if ((dq_order(live, bh, T, kb, -1) & 0xffu) != 0u) return;  // warp-uniform
  for (int e = tid; e < 128 * DH / 8; e += nthr) {
    const int rr = e / (DH / 8), c = (e % (DH / 8)) * 8;
    *reinterpret_cast<uint4*>(dqkv + (int64_t)(row0 + kb * 128 + rr) * (3 * H * DH) + h * DH + c) = make_uint4(0, 0, 0, 0);
  }
}

// ---------------------------------------------------------------------------------------
// dh = 128 variant with 64-query tiles and a software pipeline across query tiles:
//   MMA order per tile t:  [pds_full(t)]  S^T(t+1), dP^T(t+1)  dV(t)  dK(t)  [dq_empty(t-1)] dQ^T(t)
//   so the elementwise phase of tile t+1 overlaps the dV/dK/dQ MMAs of tile t.
//   dQ^T = K^T dS^T (M = dh = 128, N = 64 queries, K = 128 keys) has its own TMEM columns;
//   it is drained by the compute warps of the NEXT tile into their warpgroup's 32 x 128 f32
//   staging box (double-buffered) and handed to a dQ warp, which adds it in the fixed
//   order of dq_order. P^T (bf16 pairs) goes to TMEM and dV = P^T dO is an A-from-TMEM MMA;
//   the 32 KB of smem that P^T no longer needs hold the second staging buffer (the Q / dO
//   ring is 2 deep).
//   TMEM: S^T [0,64)  dP^T [64,128)  dQ^T [128,192)  P^T[2] [192,256)  dV [256,384)  dK [384,512).
// dQ staging buffers per warpgroup in the dh 128 kernel: 2 (the Q / dO ring gives up its third
// stage for them) measured 0.977 vs 1.003 ms at the C4 shape with 1 buffer and NQ = 3
#define DQ128_NBUF 2
struct AttnBwd64Cfg {
  static constexpr int DH = 128;
  static constexpr int NQ = DQ128_NBUF == 2 ? 2 : 3;  // Q / dO ring depth
  static constexpr int KT = 128 * DH * 2;        // K or V tile (128 keys)
  static constexpr int QT = 64 * DH * 2;         // Q or dO tile (64 queries)
  static constexpr int PT = 128 * 64 * 2;        // dS^T tile (128 keys x 64 q)
  static constexpr int K_OFF = 0;
  static constexpr int V_OFF = K_OFF + KT;
  static constexpr int Q_OFF = V_OFF + KT;       // [NQ]
  static constexpr int O_OFF = Q_OFF + NQ * QT;  // [NQ]
  static constexpr int S_OFF = O_OFF + NQ * QT;  // [2]
  static constexpr int X_OFF = S_OFF + 2 * PT;   // dQ staging: [DQ128_NBUF][64 rows x 128 f32]
  static constexpr int L_OFF = X_OFF + DQ128_NBUF * 64 * DH * 4;  // e[2][64], D[2][64]
  static constexpr int BAR_OFF = L_OFF + 4 * 64 * 4;
  static constexpr int SMEM = BAR_OFF + 512 + 1024;  // mbarriers, TMEM slot, live count + list; align
  static_assert(SMEM <= 232448, "attention bwd (dh 128) smem");
};

__global__ void __launch_bounds__(384, 1)
    attn_bwd_tc64_kernel(const __grid_constant__ CUtensorMap tm_kv, const __grid_constant__ CUtensorMap tm_q,
                         const __grid_constant__ CUtensorMap tm_do, const __grid_constant__ CUtensorMap tm_dq,
                         const __grid_constant__ CUtensorMap tm_dkv,
                         const float* __restrict__ lse2, const uint8_t* __restrict__ live, const float* __restrict__ Dd,
                         __nv_bfloat16* __restrict__ dqkv, float* __restrict__ dqacc, uint32_t* __restrict__ sem,
                         int T, int H, float scale_log2, float scale, int use_alibi) {
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
  uint64_t* staged = bar + 56;  // [g][buffer] warpgroup g's dQ box is staged (4 warp arrivals)
  uint64_t* sfree = bar + 60;   // [g][buffer] dQ warp g is done with that staging buffer
  float* sE0 = reinterpret_cast<float*>(smem + Cf::L_OFF);  // e[2][64] (double-buffered)
  float* sD0 = sE0 + 128;                                     // D[2][64]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kb = blockIdx.x;
#ifdef FB_ATTN_PROF
  if (threadIdx.x == 0 && PROF_CTA() < 8192) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_attn_prof[PROF_CTA() * 8 + 0] = ptimer();
    g_attn_prof[PROF_CTA() * 8 + 3] = smid;
  }
#endif
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const int d = H * DH;
  const int row0 = b * T;
  const int k0 = kb * 128;
  const int first = 2 * kb, ntiles = T / 64 - 2 * kb;  // causal: query tiles of 64 from the block's diagonal

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_kv);
    tma_prefetch(&tm_q);
    tma_prefetch(&tm_do);
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
    for (int i = 0; i < 4; ++i) {
      mbar_init(&staged[i], 4);
      mbar_init(&sfree[i], 1);
    }
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
  } else if (warp >= 10) {
    // dQ warps: warp 10 + g turns warpgroup g's staged 32 x 128 boxes into dQ in the fixed order
    // of dq_order: TMA store (first) / reduce-add (middle), bumping the box counter once the op
    // completed, or acc + box -> bf16 dqkv (last). The counter waits, bulk-op completions and
    // release fences stay off the compute warps.
    const int g = warp - 10;
    uint32_t ords = 0;  // lane l: dq_order of tile (t & ~31) + l
    for (int t = 0; t < nlive; ++t) {
      const int q0 = (first + tl[t]) * 64, qrow = q0 + 32 * g;
      const int sb = DQ128_NBUF == 2 ? (t & 1) : 0;
      const uint32_t sph = DQ128_NBUF == 2 ? ((t >> 1) & 1) : (t & 1);
      const float* Xg = reinterpret_cast<const float*>(smem + Cf::X_OFF) + (sb * 64 + g * 32) * DH;
      if ((t & 31) == 0 && t + lane < nlive) ords = dq_order_lane(live, bh, T, (first + tl[t + lane]) >> 1, kb);
      const uint32_t ord = __shfl_sync(0xffffffffu, ords, t & 31), cnt = ord & 0xffu;
      uint32_t* bsem = sem + (int64_t)bh * (T / 32) + qrow / 32;
      mbar_wait(&staged[2 * g + sb], sph);
      if (lane == 0 && cnt) sem_wait_eq(bsem, cnt);  // every larger live key block has added its partial
      __syncwarp();
      if (ord & 0x100u) {  // last contributor: dQ = acc + partial, bf16 (lane: 4 dh columns x 32 rows)
        const int c = 4 * lane;
        const float* acc = dqacc + (int64_t)(row0 + qrow) * d + h * DH + c;
        __nv_bfloat16* out = dqkv + (int64_t)(row0 + qrow) * (3 * d) + h * DH + c;
        float4 a[32];  // every accumulator load in flight at once (one L2 round trip per box)
#pragma unroll
        for (int i = 0; i < 32; ++i)
          a[i] = cnt ? __ldcg(reinterpret_cast<const float4*>(acc + (int64_t)i * d)) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          float4 x = *reinterpret_cast<const float4*>(Xg + i * DH + c);
          if (cnt) x = make_float4(a[i].x + x.x, a[i].y + x.y, a[i].z + x.z, a[i].w + x.w);
          *reinterpret_cast<uint2*>(out + (int64_t)i * (3 * d)) = make_uint2(pack_bf16(x.x, x.y), pack_bf16(x.z, x.w));
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sfree[2 * g + sb]);
      } else if (lane == 0) {
        dq_out_box(&tm_dq, smem_u32(Xg), h * DH, row0 + qrow, cnt == 0);
        bulk_commit();
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        mbar_arrive(&sfree[2 * g + sb]);
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        sem_release(bsem);  // at once: the next key block waits on it
      }
      __syncwarp();
    }
    if (g == 0) zero_dead_rows(live, bh, T, kb, DH, H, row0, h, dqkv, lane, 32);
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
    auto drain = [&](int t) {  // dQ^T(t) -> warpgroup g's 32 x 128 staging box, handed to dQ warp g
      mbar_wait(dq_full, t & 1);
      tc_fence_after();
      uint32_t v[32];
      tmem_ld_32x32b_x32(tmem + 128 + lane_off + 32 * g, v);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dq_empty);
      PROF_T0(pf);
      const int sb = DQ128_NBUF == 2 ? (t & 1) : 0;
      mbar_wait(&sfree[2 * g + sb], (DQ128_NBUF == 2 ? ((t >> 1) & 1) : (t & 1)) ^ 1);  // dQ warp g is done with it
      float* Xb = Xs + sb * 64 * DH;
      if (lane == 0 && quad == 0) PROF_ADD(6, pf);
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        const float2 sv2 = pk_mul(make_float2(__uint_as_float(v[i]), __uint_as_float(v[i + 1])), make_float2(scale, scale));
        Xb[(32 * g + i) * DH + r] = sv2.x;
        Xb[(32 * g + i + 1) * DH + r] = sv2.y;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the TMA reads the box
      __syncwarp();
      if (lane == 0) mbar_arrive(&staged[2 * g + sb]);
      // publishes the e/D that load_ed wrote just before (read in the next tile's elementwise)
      asm volatile("bar.sync %0, 128;" ::"r"(2 + g) : "memory");
    };
    // e/D of tile t live in buffer t & 1; tile t+1's are prefetched before drain(t-1), whose
    // warpgroup barrier publishes them (all readers of that buffer finished tile t-1 earlier)
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
#ifdef FB_ATTN_PROF
  if (threadIdx.x == 0 && PROF_CTA() < 8192) g_attn_prof[PROF_CTA() * 8 + 1] = ptimer();
#endif
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ---------------------------------------------------------------------------------------
// dh = 64 variant of the pipelined backward: 128-query tiles, dQ = dS K (M = 128 queries,
// A = the dS^T smem image read MN-major) in its own TMEM columns, two 128 x 32 dQ boxes per
// tile (one per warpgroup). MMA order per tile t: [p_full(t)] dV(t) (P^T from TMEM)
// S^T/dP^T(t+1) dK(t) [dq_empty] dQ(t): the compute warps never wait for dV before writing
// dS^T (round 1 shared one smem tile between P^T and dS^T and stalled on it every tile).
//   TMEM: S^T [0,128)  dP^T [128,256)  dQ [256,320)  dV [320,384)  dK [384,448)  P^T [448,512).
// dQ staging buffers per warpgroup in the dh 64 kernel: 2 measured 10% slower (the extra 32 KB of
// smem takes the L1 the E/D and map loads use)
#define DQ_NBUF 1
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
  static constexpr int X_OFF = P_OFF + 2 * PT;   // dQ staging [2 buffers][2 groups][128 rows x 32 f32] (swizzled)
  static constexpr int L_OFF = X_OFF + DQ_NBUF * 128 * DH * 4;
  static constexpr int BAR_OFF = L_OFF + 2 * 128 * 4;
  static constexpr int SMEM = BAR_OFF + 512 + 1024;
  static_assert(SMEM <= 232448, "attention bwd (dh 64) smem");
};

__global__ void __launch_bounds__(384, 1)
    attn_bwd_tcd64_kernel(const __grid_constant__ CUtensorMap tm_qkv, const __grid_constant__ CUtensorMap tm_do,
                          const __grid_constant__ CUtensorMap tm_dq, const __grid_constant__ CUtensorMap tm_dkv,
                          const float* __restrict__ lse2,
                          const uint8_t* __restrict__ live, const float* __restrict__ Dd,
                          __nv_bfloat16* __restrict__ dqkv, float* __restrict__ dqacc,
                          uint32_t* __restrict__ sem, int T, int H, float scale_log2, float scale, int use_alibi) {
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
  uint64_t* p_full = bar + 10;    // P^T(t) in TMEM and dS^T(t) in smem (8 compute warps)
  uint64_t* pds_free = bar + 11;  // [2]
  uint64_t* dq_full = bar + 13;
  uint64_t* dq_empty = bar + 14;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 17);
  uint32_t* nlive_p = tmem_slot + 1;
  uint8_t* tl = reinterpret_cast<uint8_t*>(tmem_slot + 2);
  uint64_t* staged = bar + 35;  // [g][buffer] warpgroup g's dQ box is staged (4 warp arrivals)
  uint64_t* sfree = bar + 39;   // [g][buffer] dQ warp g is done with that staging buffer
  float* sE = reinterpret_cast<float*>(smem + Cf::L_OFF);
  float* sD = sE + 128;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int kb = blockIdx.x;
#ifdef FB_ATTN_PROF
  if (threadIdx.x == 0 && PROF_CTA() < 8192) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_attn_prof[PROF_CTA() * 8 + 0] = ptimer();
    g_attn_prof[PROF_CTA() * 8 + 3] = smid;
  }
#endif
  const int bh = blockIdx.y, b = bh / H, h = bh % H;
  const int d = H * DH;
  const int row0 = b * T;
  const int k0 = kb * 128;
  const int first = kb, ntiles = T / 128 - kb;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_qkv);
    tma_prefetch(&tm_do);
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
    mbar_init(dq_full, 1);
    mbar_init(dq_empty, 8);
    for (int i = 0; i < 4; ++i) {
      mbar_init(&staged[i], 4);
      mbar_init(&sfree[i], 1);
    }
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
      const uint32_t tS = tmem, tP = tmem + 128, tQ = tmem + 256, tV = tmem + 320, tK = tmem + 384, tPT = tmem + 448;
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
        const uint32_t sS = sP0 + s * Cf::PT;  // dS^T(t)
        mbar_wait(p_full, ph);  // P^T(t) in TMEM, dS^T(t) in smem
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)  // dV += P^T dO  (K = 128 queries; P^T from TMEM)
          umma_ts_b(tV, tPT + 8 * kk, smem_desc_sw128(sO + kk * 2048, 128 * 128, 1024), idKV, (t | kk) > 0);
        umma_commit(&o_empty[s]);
        // S^T / dP^T(t+1) after dV(t): s_full(t+1) then also covers dV(t)'s read of P^T(t), which the
        // compute warps overwrite with P^T(t+1)
        if (t + 1 < nlive) issue_sp(t + 1);
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
  } else if (warp >= 10) {
    // dQ warps: warp 10 + g turns warpgroup g's staged 128 x 32 boxes (dh columns 32g..32g+31)
    // into dQ in the fixed order of dq_order, as in the dh 128 kernel; the staging is
    // double-buffered here (box t in buffer t & 1), so one slow box does not stall the compute warps
    const int g = warp - 10;
    uint32_t ords = 0;  // lane l: dq_order of tile (t & ~31) + l
    for (int t = 0; t < nlive; ++t) {
      const int q0 = (first + tl[t]) * 128, sb = DQ_NBUF == 2 ? (t & 1) : 0;
      const uint32_t xbox = sX + sb * 32768 + g * 16384;
      if ((t & 31) == 0 && t + lane < nlive) ords = dq_order_lane(live, bh, T, first + tl[t + lane], kb);
      const uint32_t ord = __shfl_sync(0xffffffffu, ords, t & 31), cnt = ord & 0xffu;
      uint32_t* bsem = sem + ((int64_t)bh * (T / 128) + q0 / 128) * 2 + g;
      mbar_wait(&staged[2 * g + sb], DQ_NBUF == 2 ? ((t >> 1) & 1) : (t & 1));
      if (lane == 0 && cnt) sem_wait_eq(bsem, cnt);
      __syncwarp();
      if (ord & 0x100u) {  // last contributor: lane owns rows lane + 32k, 32 columns each
#pragma unroll 1
        for (int k0 = 0; k0 < 4; k0 += 2) {  // two rows (16 accumulator loads in flight) at a time
          float4 a[16];
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            const float* acc = dqacc + (int64_t)(row0 + q0 + lane + 32 * (k0 + kk)) * d + h * DH + 32 * g;
#pragma unroll
            for (int q = 0; q < 8; ++q)
              a[8 * kk + q] = cnt ? __ldcg(reinterpret_cast<const float4*>(acc) + q) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            const int r = lane + 32 * (k0 + kk);
            __nv_bfloat16* out = dqkv + (int64_t)(row0 + q0 + r) * (3 * d) + h * DH + 32 * g;
#pragma unroll
            for (int q = 0; q < 8; q += 2) {
              float4 x0, x1;
              asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                           : "=f"(x0.x), "=f"(x0.y), "=f"(x0.z), "=f"(x0.w)
                           : "r"(xbox + r * 128 + ((q ^ (r & 7)) << 4)));
              asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                           : "=f"(x1.x), "=f"(x1.y), "=f"(x1.z), "=f"(x1.w)
                           : "r"(xbox + r * 128 + (((q + 1) ^ (r & 7)) << 4)));
              const float4 a0 = a[8 * kk + q], a1 = a[8 * kk + q + 1];
              if (cnt) {
                x0 = make_float4(a0.x + x0.x, a0.y + x0.y, a0.z + x0.z, a0.w + x0.w);
                x1 = make_float4(a1.x + x1.x, a1.y + x1.y, a1.z + x1.z, a1.w + x1.w);
              }
              *reinterpret_cast<uint4*>(out + 4 * q) =
                  make_uint4(pack_bf16(x0.x, x0.y), pack_bf16(x0.z, x0.w), pack_bf16(x1.x, x1.y), pack_bf16(x1.z, x1.w));
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sfree[2 * g + sb]);
      } else if (lane == 0) {
        dq_out_box(&tm_dq, xbox, h * DH + 32 * g, row0 + q0, cnt == 0);
        bulk_commit();
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        mbar_arrive(&sfree[2 * g + sb]);
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        sem_release(bsem);
      }
      __syncwarp();
    }
    if (g == 0) zero_dead_rows(live, bh, T, kb, DH, H, row0, h, dqkv, lane, 32);
  } else {
    const int g = (warp - 2) >> 2;
    const int quad = warp & 3;
    const int r = quad * 32 + lane;  // TMEM lane: key row (elementwise) / query row (dQ drain)
    const int kj = k0 + r;
    const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
    const float sl = use_alibi ? exp2f(-8.0f * (float)(h + 1) / (float)H) * 1.4426950408889634f : 0.0f;
    const float slk = sl * (float)kj;
    const int tid = threadIdx.x - 64;
    auto drain = [&](int t) {  // dQ(t) -> warpgroup g's staging box, handed to dQ warp g
      mbar_wait(dq_full, t & 1);
      tc_fence_after();
      uint32_t v[32];
      tmem_ld_32x32b_x32(tmem + 256 + lane_off + 32 * g, v);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dq_empty);
      PROF_T0(pf);
      const int sb = DQ_NBUF == 2 ? (t & 1) : 0;
      const uint32_t xbox = sX + sb * 32768 + g * 16384;  // this warpgroup's 128 x 32 f32 box
      mbar_wait(&sfree[2 * g + sb], (DQ_NBUF == 2 ? ((t >> 1) & 1) : (t & 1)) ^ 1);  // dQ warp g is done with it
      if (lane == 0 && quad == 0) PROF_ADD(6, pf);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t addr = xbox + r * 128 + ((q ^ (r & 7)) << 4);
        asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "f"(__uint_as_float(v[4 * q]) * scale),
                     "f"(__uint_as_float(v[4 * q + 1]) * scale), "f"(__uint_as_float(v[4 * q + 2]) * scale),
                     "f"(__uint_as_float(v[4 * q + 3]) * scale));
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the TMA reads the box
      __syncwarp();
      if (lane == 0) mbar_arrive(&staged[2 * g + sb]);
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
      uint32_t ptm[32];  // this group's 64 queries of P^T as bf16 pairs -> TMEM (A of the dV MMA)
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
            for (int i = 0; i < 4; ++i) ptm[c * 16 + q * 4 + i] = pack_bf16(p[2 * i], p[2 * i + 1]);
            const int kc = 8 * g + 4 * c + q;  // 8-query chunk 0..15
            const uint32_t sw = (kc >> 3) * (128 * 128) + (((kc & 7) ^ (r & 7)) << 4);
            asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(prow + sw), "r"(pack_bf16(ds[0], ds[1])),
                         "r"(pack_bf16(ds[2], ds[3])), "r"(pack_bf16(ds[4], ds[5])), "r"(pack_bf16(ds[6], ds[7])));
          }
        }
      };
      if (diag) elementwise(std::true_type{});
      else elementwise(std::false_type{});
      // P^T(t) over P^T(t-1): dV(t-1) finished before s_full(t) fired (it was issued before S^T(t))
      tmem_st_32x32b_x32(tmem + 448 + 32 * g + lane_off, ptm);
      tmem_st_wait();
      tc_fence_before();
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      if (t > 0) drain(t - 1);
    }
    if (nlive > 0) drain(nlive - 1);
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
#ifdef FB_ATTN_PROF
  if (threadIdx.x == 0 && PROF_CTA() < 8192) g_attn_prof[PROF_CTA() * 8 + 1] = ptimer();
#endif
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 g_enc_bwd = nullptr;

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

// {d, rows, 1} f32 map with box_cols x box_rows boxes (the dQ accumulator)
static int encode_f32_box(CUtensorMap* m, void* base, int64_t rows, int d, int box_cols, int box_rows,
                          CUtensorMapSwizzle swz) {
  cuuint64_t dims[3] = {(cuuint64_t)d, (cuuint64_t)rows, 1};
  cuuint64_t strides[2] = {(cuuint64_t)d * 4, (cuuint64_t)rows * d * 4};
  cuuint32_t box[3] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_enc_bwd(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("attn bwd dq tensor map encode failed: %d", (int)r);
    return FB_CUDA_ERROR;
  }
  return FB_OK;
}

static int attn_bwd_tc64_launch(const void* qkv, const void* dO, const float* lse, const uint8_t* live,
                                const float* Dbuf, float* dq, uint32_t* sem,
                                void* dqkv, int B, int T, int H, int use_alibi, cudaStream_t st) {
  using Cf = AttnBwd64Cfg;
  constexpr int DH = 128;
  const int d = H * DH;
  CUtensorMap tkv, tq, to;
  int rc = encode_box(&tkv, qkv, (int64_t)B * T, 3 * d, 128, DH / 64);
  if (rc) return rc;
  rc = encode_box(&tq, qkv, (int64_t)B * T, 3 * d, 64, DH / 64);
  if (rc) return rc;
  rc = encode_box(&to, dO, (int64_t)B * T, d, 64, DH / 64);
  if (rc) return rc;
  CUtensorMap tdq;  // the f32 accumulator of the ordered dQ partials: one 32 x 128 box per warpgroup
  rc = encode_f32_box(&tdq, dq, (int64_t)B * T, d, DH, 32, CU_TENSOR_MAP_SWIZZLE_NONE);
  if (rc) return rc;
  CUtensorMap tdkv;  // dK / dV store boxes: 128 keys x 128 dh (two 64-column chunks), 128B swizzle
  rc = encode_box(&tdkv, dqkv, (int64_t)B * T, 3 * d, 128, DH / 64);
  if (rc) return rc;
  auto k = attn_bwd_tc64_kernel;
  FB_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM));
  const float scale = 1.0f / sqrtf((float)DH);
  k<<<dim3(T / 128, B * H), 384, Cf::SMEM, st>>>(tkv, tq, to, tdq, tdkv, lse, live, Dbuf, (__nv_bfloat16*)dqkv, dq,
                                                 sem, T, H, 1.4426950408889634f * scale, scale, use_alibi);
  FB_LAUNCH_CHECK();
  return FB_OK;
}

static int attn_bwd_tcd64_launch(const void* qkv, const void* dO, const float* lse, const uint8_t* live,
                                 const float* Dbuf, float* dq, uint32_t* sem,
                                 void* dqkv, int B, int T, int H, int use_alibi, cudaStream_t st) {
  using Cf = AttnBwdD64Cfg;
  constexpr int DH = 64;
  const int d = H * DH;
  CUtensorMap tq, to;
  int rc = encode_box(&tq, qkv, (int64_t)B * T, 3 * d, 128, 1);
  if (rc) return rc;
  rc = encode_box(&to, dO, (int64_t)B * T, d, 128, 1);
  if (rc) return rc;
  CUtensorMap tdq;  // the f32 accumulator of the ordered dQ partials: 128 x 32 boxes, 128B swizzle
  rc = encode_f32_box(&tdq, dq, (int64_t)B * T, d, 32, 128, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  CUtensorMap tdkv;  // dK / dV store boxes: 128 keys x 64 dh, 128B swizzle
  rc = encode_box(&tdkv, dqkv, (int64_t)B * T, 3 * d, 128, 1);
  if (rc) return rc;
  auto k = attn_bwd_tcd64_kernel;
  FB_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM));
  const float scale = 1.0f / sqrtf((float)DH);
  k<<<dim3(T / 128, B * H), 384, Cf::SMEM, st>>>(tq, to, tdq, tdkv, lse, live, Dbuf, (__nv_bfloat16*)dqkv, dq, sem,
                                                 T, H, 1.4426950408889634f * scale, scale, use_alibi);
  FB_LAUNCH_CHECK();
  return FB_OK;
}

template <int DH>
int attn_bwd_tc_launch(const void* qkv, const void* dO, const float* lse, const uint8_t* live, const float* Dbuf,
                       float* dq, uint32_t* sem, void* dqkv, int B, int T, int H, int use_alibi, cudaStream_t st) {
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
  // the box counters of dq_order start at 0 (B*H*T/32 words: 32 KB at the C4 shape)
  FB_CUDA_TRY(cudaMemsetAsync(sem, 0, sizeof(uint32_t) * (size_t)B * H * (T / 32), st));
  if (DH == 128) return attn_bwd_tc64_launch(qkv, dO, lse, live, Dbuf, dq, sem, dqkv, B, T, H, use_alibi, st);
  if (DH == 64) return attn_bwd_tcd64_launch(qkv, dO, lse, live, Dbuf, dq, sem, dqkv, B, T, H, use_alibi, st);
  return FB_UNSUPPORTED;
}

template int attn_bwd_tc_launch<64>(const void*, const void*, const float*, const uint8_t*, const float*, float*,
                                    uint32_t*, void*, int, int, int, int, cudaStream_t);
template int attn_bwd_tc_launch<128>(const void*, const void*, const float*, const uint8_t*, const float*, float*,
                                     uint32_t*, void*, int, int, int, int, cudaStream_t);

}  // namespace fb

#ifdef FB_ATTN_PROF
extern "C" int fb_attn_prof_read(unsigned long long* out, int n) {
  return cudaMemcpyFromSymbol(out, fb::g_attn_prof, n * sizeof(unsigned long long)) == cudaSuccess ? 0 : 2;
}
extern "C" int fb_attn_prof_clear() {
  static unsigned long long z[8192 * 8];
  return cudaMemcpyToSymbol(fb::g_attn_prof, z, sizeof(z)) == cudaSuccess ? 0 : 2;
}
#endif
#ifdef FB_ATTN_TRACE
extern "C" int fb_attn_trace_read(unsigned long long* out, int n) {
  return cudaMemcpyFromSymbol(out, fb::g_attn_trace, n * sizeof(unsigned long long)) == cudaSuccess ? 0 : 2;
}
#endif
