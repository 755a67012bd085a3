// K13: fused pseudo-gradient aggregation + server outer step, one HBM pass.
//
// Reference math (fedforge/fedopt.py):
//   delta_k = f64(w) - f64(w_k)                                  trainer.py:352
//   deterministic finalize: pairwise tree over n_k*delta_k in id order, / total  fedopt.py:135-143
//   streaming finalize:     running sum in arrival order, / total               fedopt.py:95, 144
//   single contribution:    delta_0 unchanged                                   fedopt.py:133-134
//   m' = f32(mu*f64(m) + pg); w' = f32(f64(w) - eta*(mu*f64(m') + pg)) [Nesterov]
//                                  or f32(f64(w) - eta*f64(m'))                  fedopt.py:189-196
// All arithmetic uses explicit round-to-nearest f64 intrinsics (no FMA contraction)
// so results are bit-identical to numpy's.
//
// B200 design: memory-bound streaming kernel. Each thread owns 4 consecutive
// parameters (128-bit loads of every client vector, w and m; 128-bit streaming
// stores of w', m'); grid = 148 SMs x 8 resident CTAs, grid-stride. The
// pairwise tree is evaluated on the fly with a binary-counter stack of depth
// <= 7 (same association as the level-by-level pairing), so K clients cost K
// loads and no extra traffic. Algorithmic bytes: (4K + 16) N. The client loads
// are issued in batches of KB before any f64 math, with KB x VEC chosen per tree
// depth so that 128-256 B per thread are in flight: 73-82% of HBM for K = 8..64.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "sm100.cuh"

namespace fb {

// Bulk-staged input streams (K <= 8, n % 4 == 0, 16-byte aligned): a CTA's chunk of 1024
// parameters of every client, of w and of m arrives by one 4 KB cp.async.bulk each into a 2-stage
// smem ring (mbarrier complete_tx), issued a chunk ahead by thread 0, instead of per-thread 128-bit
// loads: every read stream gets deep, register-free memory-level parallelism, with 2 CTAs (16
// warps of f64 math) per SM. Same per-element math, same vector -> thread mapping: bit-identical.
// C4 (K 8, 1.339 B): 12.9 -> 11.1 ms = 77% -> 90% of HBM; K 4: 62% -> 79%. Clients only / 3 stages
// 80%; one CTA per SM with 3-4 stages 48-56% (8 warps cannot keep up with the f64 math).
// The kernel takes any VEC (chunk = 256 VEC), but only K <= 8 pays: K 9-16 staged in 512-chunks
// measured equal to the register kernel (74%), K 17-40 in 256-chunks slower (55% vs 77%), so the
// launch keeps the bulk path for K <= 8.
constexpr int kBulkStages = 2;
constexpr int kBulkMaxK = 8;
// A/B switch for the bulk-staged path (any value but "0" turns it off)
static bool getenv_flag(const char* name) {
  const char* v = getenv(name);
  return v && v[0] && !(v[0] == '0' && v[1] == 0);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   sm100::smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(sm100::smem_u32(bar))
               : "memory");
}

template <typename TIn>
struct AggParams {
  const TIn* src[FB_MAX_CLIENTS];
  double nk[FB_MAX_CLIENTS];
  double pk[FB_MAX_CLIENTS];  // n_k / sum n (f64), for the round-norm telemetry
  float* wrep[FB_MAX_REPLICAS];  // extra destinations of w' (peer GPUs' replicas over NVLink)
  int nrep;
};

// stats layout (f64): 0 |pg|^2, 1 |w'|^2, 2 |m'|^2, 3 |w|^2, 4 |sum p_k w_k|^2, 5 |w - sum p_k w_k|^2,
// 6 + k: |w_k|^2 (only with per-client norms)  -- compute_round_norms, fedforge/metrics.py:177-215
constexpr int kStatsFixed = 6;

// binary-counter stack of partial sums; D = floor(log2(K)) + 1 levels suffice
template <int kStack>
struct TreeAcc {
  double slot[kStack];
  __device__ __forceinline__ void push(double t, int k) {
    // k = index of this term; slots occupied = bits of k
    double carry = t;
    bool done = false;
#pragma unroll
    for (int L = 0; L < kStack; ++L) {
      if (!done) {
        if ((k >> L) & 1) {
          carry = __dadd_rn(slot[L], carry);
        } else {
          slot[L] = carry;
          done = true;
        }
      }
    }
  }
  __device__ __forceinline__ double result(int K) const {
    // merge occupied slots right-to-left: lowest level is the rightmost block
    double acc = 0.0;
    bool have = false;
#pragma unroll
    for (int L = 0; L < kStack; ++L) {
      if ((K >> L) & 1) {
        acc = have ? __dadd_rn(slot[L], acc) : slot[L];
        have = true;
      }
    }
    return acc;
  }
};

template <typename TIn>
__device__ __forceinline__ double delta_of(const TIn* p, int64_t j, double wg);
template <>
__device__ __forceinline__ double delta_of<float>(const float* p, int64_t j, double wg) {
  return __dsub_rn(wg, (double)__ldg(p + j));
}
template <>
__device__ __forceinline__ double delta_of<double>(const double* p, int64_t j, double) {
  return __ldg(p + j);
}

struct StepOut {
  float w, m;
  double pg;
};

__device__ __forceinline__ StepOut outer_step(float w32, float m32, double pg, double eta, double mu,
                                              int nesterov) {
  StepOut o;
  double m64 = __dadd_rn(__dmul_rn(mu, (double)m32), pg);
  o.m = __double2float_rn(m64);
  double upd;
  if (nesterov)
    upd = __dmul_rn(eta, __dadd_rn(__dmul_rn(mu, (double)o.m), pg));
  else
    upd = __dmul_rn(eta, (double)o.m);
  o.w = __double2float_rn(__dsub_rn((double)w32, upd));
  o.pg = pg;
  return o;
}

template <typename TIn, int VEC, int D, int STATS, int KB = 8, int BULK = 0>
__global__ void __launch_bounds__(256, 2) fedagg_kernel(AggParams<TIn> P, int K, int deterministic,
                                                     double inv_total_unused, double total,
                                                     const float* __restrict__ w,
                                                     const float* __restrict__ m,
                                                     float* __restrict__ w_out,
                                                     float* __restrict__ m_out, int64_t n,
                                                     double eta, double mu, int nesterov,
                                                     double* stats, unsigned long long* first_bad,
                                                     double* __restrict__ pg_out, int client_norms,
                                                     int n_fixed) {
  __shared__ double red[kStatsFixed + FB_MAX_CLIENTS][8];
  double s_pg = 0.0, s_w = 0.0, s_m = 0.0, s_w0 = 0.0, s_avg = 0.0, s_dif = 0.0;
  const int lane_ = threadIdx.x & 31, wid_ = threadIdx.x >> 5;
  if (client_norms) {
    for (int i = threadIdx.x; i < FB_MAX_CLIENTS * 8; i += blockDim.x) red[kStatsFixed + i / 8][i % 8] = 0.0;
    __syncthreads();
  }
  unsigned long long bad = ~0ull;
  const int64_t nvec = n / VEC;
  // BULK: input chunks staged in smem (bulk_g2s); iteration `it` of this CTA covers
  // parameters [c * CH, (c + 1) * CH) with c = blockIdx.x + it * gridDim.x
  extern __shared__ __align__(128) uint8_t agg_stage[];
  __shared__ __align__(8) uint64_t agg_full[kBulkStages];
  // chunks, the last one possibly partial (n % 4 == 0 keeps every copy a multiple of 16 bytes)
  constexpr int CH = 256 * VEC;  // parameters per CTA iteration (256 threads x VEC)
  const int slots = K + 2;        // stage layout: K clients, then w, then m, CH floats each
  const int64_t nchunk = BULK ? (n + CH - 1) / CH : 0;
  auto issue_chunk = [&](int64_t it) {  // thread 0: chunk `it` into stage it % kBulkStages
    const int64_t c = (int64_t)blockIdx.x + it * gridDim.x;
    if (c >= nchunk) return;
    const int st = (int)(it % kBulkStages);
    const uint32_t bytes = (uint32_t)(std::min<int64_t>(CH, n - c * CH) * 4);
    sm100::mbar_arrive_expect_tx(&agg_full[st], (uint32_t)slots * bytes);
    uint8_t* base = agg_stage + (size_t)st * slots * CH * 4;
    for (int k = 0; k < K; ++k)
      bulk_g2s(base + (size_t)k * CH * 4, reinterpret_cast<const float*>(P.src[k]) + c * CH, bytes, &agg_full[st]);
    bulk_g2s(base + (size_t)K * CH * 4, w + c * CH, bytes, &agg_full[st]);
    bulk_g2s(base + (size_t)(K + 1) * CH * 4, m + c * CH, bytes, &agg_full[st]);
  };
  if constexpr (BULK) {
    if (threadIdx.x == 0) {
      for (int i = 0; i < kBulkStages; ++i) sm100::mbar_init(&agg_full[i], 1);
      sm100::fence_barrier_init();
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int i = 0; i < kBulkStages - 1; ++i) issue_chunk(i);
  }
  int64_t it = 0;
  // With STATS the per-client norms are reduced across the warp (warp_sum), so every lane of a
  // warp runs the same trip count: lanes past the end recompute the last vector (valid reads)
  // and neither store nor count it. Without STATS the loop is the plain grid-stride one. BULK:
  // every thread of the CTA runs every chunk of the CTA (the stage barriers), masked past the end.
  for (int64_t v0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
       BULK ? ((int64_t)blockIdx.x + it * gridDim.x < nchunk) : (STATS ? (v0 - lane_ < nvec) : (v0 < nvec));
       v0 += (int64_t)gridDim.x * blockDim.x, ++it) {
    const bool act = !(STATS || BULK) || v0 < nvec;
    const float* stage = nullptr;
    if constexpr (BULK) {
      // every thread of the CTA runs the same iterations (whole chunks): the barrier frees stage
      // (it - 1) % 2 for chunk it + 1
      __syncthreads();
      if (threadIdx.x == 0) issue_chunk(it + kBulkStages - 1);
      sm100::mbar_wait(&agg_full[it % kBulkStages], (uint32_t)((it / kBulkStages) & 1));
      stage = reinterpret_cast<const float*>(agg_stage) + (size_t)(it % kBulkStages) * slots * CH + VEC * threadIdx.x;
    }
    const int64_t v = act ? v0 : nvec - 1;
    const int64_t j0 = v * VEC;
    float wv[VEC], mv[VEC];
    if constexpr (BULK) {
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        wv[e] = stage[K * CH + e];
        mv[e] = stage[(K + 1) * CH + e];
      }
    } else if constexpr (VEC == 4) {
      float4 a = ld_stream_f4(w + j0), b = ld_stream_f4(m + j0);
      wv[0] = a.x; wv[1] = a.y; wv[2] = a.z; wv[3] = a.w;
      mv[0] = b.x; mv[1] = b.y; mv[2] = b.z; mv[3] = b.w;
    } else if constexpr (VEC == 2) {
      float2 a = __ldg(reinterpret_cast<const float2*>(w + j0)), b = __ldg(reinterpret_cast<const float2*>(m + j0));
      wv[0] = a.x; wv[1] = a.y;
      mv[0] = b.x; mv[1] = b.y;
    } else {
#pragma unroll
      for (int e = 0; e < VEC; ++e) { wv[e] = w[j0 + e]; mv[e] = m[j0 + e]; }
    }
    double pg[VEC];
    if constexpr (sizeof(TIn) == 4) {
      // all client loads of a batch of KB clients are issued before any f64 math; the launch
      // picks KB x VEC so that >= 128-256 B per thread are in flight (measured, C5 sweep)
      TreeAcc<D> acc[VEC];
      double sum[VEC], avg[VEC];
#pragma unroll
      for (int e = 0; e < VEC; ++e) { sum[e] = 0.0; avg[e] = 0.0; }
      for (int k0 = 0; k0 < K; k0 += KB) {
        float c[KB][VEC];
#pragma unroll
        for (int j = 0; j < KB; ++j) {
          if (k0 + j < K) {
            const float* src = reinterpret_cast<const float*>(P.src[k0 + j]) + j0;
            if constexpr (BULK) {
#pragma unroll
              for (int e = 0; e < VEC; ++e) c[j][e] = stage[(k0 + j) * CH + e];
            } else if constexpr (VEC == 4) {
              float4 t = ld_stream_f4(src);
              c[j][0] = t.x; c[j][1] = t.y; c[j][2] = t.z; c[j][3] = t.w;
            } else if constexpr (VEC == 2) {
              float2 t = __ldg(reinterpret_cast<const float2*>(src));
              c[j][0] = t.x; c[j][1] = t.y;
            } else {  // unaligned inputs: scalar loads, same math (stats included)
              c[j][0] = __ldg(src);
            }
          }
        }
#pragma unroll
        for (int j = 0; j < KB; ++j) {
          if (k0 + j < K) {
            const int k = k0 + j;
            const float* cv = c[j];
            if (STATS) {
              double ck = 0.0;
#pragma unroll
              for (int e = 0; e < VEC; ++e) {
                avg[e] += P.pk[k] * (double)cv[e];
                ck += (double)cv[e] * (double)cv[e];
              }
              if (client_norms) {
                ck = warp_sum(act ? ck : 0.0);
                if (lane_ == 0) red[kStatsFixed + k][wid_] += ck;
              }
            }
#pragma unroll
            for (int e = 0; e < VEC; ++e) {
              const double dk = __dsub_rn((double)wv[e], (double)cv[e]);
              if (K == 1) {
                sum[e] = dk;
              } else if (deterministic) {
                acc[e].push(__dmul_rn(P.nk[k], dk), k);
              } else {
                sum[e] = __dadd_rn(sum[e], __dmul_rn(P.nk[k], dk));
              }
            }
          }
        }
      }
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        pg[e] = (K == 1) ? sum[e] : __ddiv_rn(deterministic ? acc[e].result(K) : sum[e], total);
        if (STATS && act) {
          const double w0 = (double)wv[e];
          s_w0 += w0 * w0;
          s_avg += avg[e] * avg[e];
          s_dif += (w0 - avg[e]) * (w0 - avg[e]);
        }
      }
    } else if (K == 1) {
#pragma unroll
      for (int e = 0; e < VEC; ++e) pg[e] = delta_of<TIn>(P.src[0], j0 + e, (double)wv[e]);
    } else if (deterministic) {
      TreeAcc<D> acc[VEC];
      for (int k = 0; k < K; ++k) {
#pragma unroll
        for (int e = 0; e < VEC; ++e) acc[e].push(__dmul_rn(P.nk[k], delta_of<TIn>(P.src[k], j0 + e, (double)wv[e])), k);
      }
#pragma unroll
      for (int e = 0; e < VEC; ++e) pg[e] = __ddiv_rn(acc[e].result(K), total);
    } else {
      double sum[VEC];
#pragma unroll
      for (int e = 0; e < VEC; ++e) sum[e] = 0.0;
      for (int k = 0; k < K; ++k) {
#pragma unroll
        for (int e = 0; e < VEC; ++e)
          sum[e] = __dadd_rn(sum[e], __dmul_rn(P.nk[k], delta_of<TIn>(P.src[k], j0 + e, (double)wv[e])));
      }
#pragma unroll
      for (int e = 0; e < VEC; ++e) pg[e] = __ddiv_rn(sum[e], total);
    }
    if (pg_out && act) {
#pragma unroll
      for (int e = 0; e < VEC; ++e) pg_out[j0 + e] = pg[e];
    }
    if (!w_out) {
      if (STATS && act) {
#pragma unroll
        for (int e = 0; e < VEC; ++e) s_pg += pg[e] * pg[e];
      }
      continue;
    }
    float wo[VEC], mo[VEC];
#pragma unroll
    for (int e = 0; e < VEC; ++e) {
      StepOut o = outer_step(wv[e], mv[e], pg[e], eta, mu, nesterov);
      wo[e] = o.w;
      mo[e] = o.m;
      if (STATS && act) {
        s_pg += pg[e] * pg[e];
        s_w += (double)o.w * (double)o.w;
        s_m += (double)o.m * (double)o.m;
      }
      if (act && !(isfinite(o.w) && isfinite(o.m)) && (unsigned long long)(j0 + e) < bad)
        bad = (unsigned long long)(j0 + e);
    }
    if (!act) continue;
    if constexpr (VEC == 4) {
      st_stream_f4(w_out + j0, make_float4(wo[0], wo[1], wo[2], wo[3]));
      st_stream_f4(m_out + j0, make_float4(mo[0], mo[1], mo[2], mo[3]));
      for (int i = 0; i < P.nrep; ++i) st_stream_f4(P.wrep[i] + j0, make_float4(wo[0], wo[1], wo[2], wo[3]));
    } else if constexpr (VEC == 2) {
      *reinterpret_cast<float2*>(w_out + j0) = make_float2(wo[0], wo[1]);
      *reinterpret_cast<float2*>(m_out + j0) = make_float2(mo[0], mo[1]);
      for (int i = 0; i < P.nrep; ++i) *reinterpret_cast<float2*>(P.wrep[i] + j0) = make_float2(wo[0], wo[1]);
    } else {
#pragma unroll
      for (int e = 0; e < VEC; ++e) {
        w_out[j0 + e] = wo[e];
        m_out[j0 + e] = mo[e];
        for (int i = 0; i < P.nrep; ++i) P.wrep[i][j0 + e] = wo[e];
      }
    }
  }
  // scalar tail (only when VEC > 1 and n % VEC != 0)
  if (VEC > 1 && blockIdx.x == 0 && threadIdx.x < (n % VEC)) {
    int64_t j = nvec * VEC + threadIdx.x;
    double wg = (double)w[j];
    double pgv;
    if (K == 1) {
      pgv = delta_of<TIn>(P.src[0], j, wg);
    } else if (deterministic) {
      TreeAcc<D> acc;
      for (int k = 0; k < K; ++k) acc.push(__dmul_rn(P.nk[k], delta_of<TIn>(P.src[k], j, wg)), k);
      pgv = __ddiv_rn(acc.result(K), total);
    } else {
      double s = 0.0;
      for (int k = 0; k < K; ++k) s = __dadd_rn(s, __dmul_rn(P.nk[k], delta_of<TIn>(P.src[k], j, wg)));
      pgv = __ddiv_rn(s, total);
    }
    if (pg_out) pg_out[j] = pgv;
    s_pg += pgv * pgv;
    if (STATS && sizeof(TIn) == 4) {
      double avg = 0.0;
      for (int k = 0; k < K; ++k) {
        const double ck = (double)reinterpret_cast<const float*>(P.src[k])[j];
        avg += P.pk[k] * ck;
        if (client_norms) atomicAdd(&red[kStatsFixed + k][wid_], ck * ck);
      }
      s_w0 += wg * wg;
      s_avg += avg * avg;
      s_dif += (wg - avg) * (wg - avg);
    }
    if (w_out) {
      StepOut o = outer_step(w[j], m[j], pgv, eta, mu, nesterov);
      w_out[j] = o.w;
      m_out[j] = o.m;
      for (int i = 0; i < P.nrep; ++i) P.wrep[i][j] = o.w;
      s_w += (double)o.w * (double)o.w;
      s_m += (double)o.m * (double)o.m;
      if (!(isfinite(o.w) && isfinite(o.m)) && (unsigned long long)j < bad) bad = (unsigned long long)j;
    }
  }
  if (first_bad) {
    // warp-min then one atomic per warp
    for (int o = 16; o > 0; o >>= 1) {
      unsigned long long t = __shfl_xor_sync(0xffffffffu, bad, o);
      bad = t < bad ? t : bad;
    }
    if ((threadIdx.x & 31) == 0 && bad != ~0ull) atomicMin(first_bad, bad);
  }
  if (STATS && stats) {
    double v[kStatsFixed] = {s_pg, s_w, s_m, s_w0, s_avg, s_dif};
#pragma unroll
    for (int i = 0; i < kStatsFixed; ++i) {
      v[i] = warp_sum(v[i]);
      if (lane_ == 0) red[i][wid_] = v[i];
    }
    __syncthreads();
    // only the entries the caller sized d_stats for: n_fixed (3 or 6) + K client norms
    const int nstat = client_norms ? kStatsFixed + K : n_fixed;
    for (int i = threadIdx.x; i < nstat; i += blockDim.x) {
      double t = 0.0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[i][w];
      atomicAdd(stats + i, t);
    }
  }
}

template <typename TIn>
static int launch_fedagg(const TIn* const* src, const int64_t* n_k, int K, int deterministic,
                         const float* w, const float* m, float* w_out, float* m_out, int64_t n,
                         double eta, double mu, int nesterov, double* stats, int64_t* first_bad,
                         double* pg_out, int stats_mode, cudaStream_t st, float* const* w_rep = nullptr,
                         int n_rep = 0) {
  FB_REQUIRE(K >= 1 && K <= FB_MAX_CLIENTS, "n_clients=%d outside [1, %d]", K, FB_MAX_CLIENTS);
  FB_REQUIRE(n > 0, "model length must be positive, got %lld", (long long)n);
  FB_REQUIRE(eta > 0.0, "server eta must be > 0, got %g", eta);
  FB_REQUIRE(mu >= 0.0 && mu < 1.0, "server mu must be in [0, 1), got %g", mu);
  AggParams<TIn> P;
  FB_REQUIRE(n_rep >= 0 && n_rep <= FB_MAX_REPLICAS, "n_replicas=%d outside [0, %d]", n_rep, FB_MAX_REPLICAS);
  FB_REQUIRE(n_rep == 0 || w_out, "w' replicas need w_out");
  P.nrep = n_rep;
  for (int i = 0; i < n_rep; ++i) {
    FB_REQUIRE(w_rep[i] != nullptr, "replica %d: null pointer", i);
    P.wrep[i] = w_rep[i];
  }
  double total = 0.0;
  int64_t itotal = 0;
  FB_REQUIRE((w_out == nullptr) == (m_out == nullptr), "w_out and m_out must both be set or both NULL");
  FB_REQUIRE(w_out || pg_out || stats, "nothing to compute");
  bool aligned = ((uintptr_t)w % 16 == 0) && ((uintptr_t)m % 16 == 0) && ((uintptr_t)w_out % 16 == 0) &&
                 ((uintptr_t)m_out % 16 == 0) && ((uintptr_t)pg_out % 8 == 0);
  for (int i = 0; i < n_rep; ++i) aligned = aligned && ((uintptr_t)w_rep[i] % 16 == 0);
  for (int k = 0; k < K; ++k) {
    FB_REQUIRE(n_k[k] >= 1, "client %d: n_k must be >= 1, got %lld", k, (long long)n_k[k]);
    FB_REQUIRE(src[k] != nullptr, "client %d: null pointer", k);
    P.src[k] = src[k];
    P.nk[k] = (double)n_k[k];
    itotal += n_k[k];
    P.pk[k] = 0.0;
    aligned = aligned && ((uintptr_t)src[k] % 16 == 0);
  }
  total = (double)itotal;
  for (int k = 0; k < K; ++k) P.pk[k] = (double)n_k[k] / total;
  // stats_mode: 1 = 3 doubles (|pg|^2, |w'|^2, |m'|^2); 4 = the 6 fixed round-norm entries;
  // 2 (with 1) = 6 fixed + K per-client entries
  const int client_norms = (stats_mode & 2) ? 1 : 0;
  const int n_fixed = (stats_mode & 6) ? kStatsFixed : 3;
  if (stats) FB_CUDA_TRY(cudaMemsetAsync(stats, 0, (n_fixed + (client_norms ? K : 0)) * sizeof(double), st));
  if (first_bad) FB_CUDA_TRY(cudaMemsetAsync(first_bad, 0x7f, sizeof(int64_t), st));
  const int threads = 256;
  const int depth = K <= 1 ? 1 : K <= 3 ? 2 : K <= 7 ? 3 : K <= 15 ? 4 : K <= 31 ? 5 : K <= 63 ? 6 : 7;
#define FB_AGG_LAUNCH(VEC_, D_, KB_)                                                                     \
  do {                                                                                                   \
    int64_t work = (n / VEC_ + threads - 1) / threads;                                                   \
    int blocks = (int)(work < kNumSMs * 8 ? (work > 0 ? work : 1) : kNumSMs * 8);                        \
    if (stats)                                                                                           \
      fedagg_kernel<TIn, VEC_, D_, 1, KB_><<<blocks, threads, 0, st>>>(P, K, deterministic, 0.0, total, w, m, w_out, \
                                                               m_out, n, eta, mu, nesterov, stats,         \
                                                               (unsigned long long*)first_bad, pg_out,     \
                                                               client_norms, n_fixed);                     \
    else                                                                                                 \
    fedagg_kernel<TIn, VEC_, D_, 0, KB_><<<blocks, threads, 0, st>>>(P, K, deterministic, 0.0, total, w, m, w_out, \
                                                             m_out, n, eta, mu, nesterov, stats,         \
                                                             (unsigned long long*)first_bad, pg_out,     \
                                                             client_norms, n_fixed);                     \
  } while (0)
  if constexpr (sizeof(TIn) == 4) {
    if (aligned && K <= kBulkMaxK && n % 4 == 0 && !getenv_flag("FB_AGG_NO_BULK")) {
      const int vec = 4;
      const int64_t nchunk = (n + 256 * vec - 1) / (256 * vec);
      const int smem = kBulkStages * (K + 2) * 256 * vec * 4;
      const int blocks = (int)std::min<int64_t>(nchunk, kNumSMs * (smem <= 110 * 1024 ? 2 : 1));  // all resident
#define FB_AGG_BULK(VEC_, D_, KB_, S_)                                                                          \
  do {                                                                                                          \
    auto kf = fedagg_kernel<float, VEC_, D_, S_, KB_, 1>;                                                       \
    FB_CUDA_TRY(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));                   \
    kf<<<blocks, threads, smem, st>>>(P, K, deterministic, 0.0, total, w, m, w_out, m_out, n, eta, mu, nesterov, \
                                      stats, (unsigned long long*)first_bad, pg_out, client_norms, n_fixed);    \
  } while (0)
      // tree depth D >= floor(log2 K) + 1
      if (K <= 7) {
        if (stats) FB_AGG_BULK(4, 3, 8, 1); else FB_AGG_BULK(4, 3, 8, 0);
      } else {
        if (stats) FB_AGG_BULK(4, 4, 8, 1); else FB_AGG_BULK(4, 4, 8, 0);
      }
#undef FB_AGG_BULK
      FB_LAUNCH_CHECK();
      return FB_OK;
    }
  }
  if (aligned && sizeof(TIn) == 4) {
    switch (depth) {
      case 1: case 2: case 3: FB_AGG_LAUNCH(4, 3, 8); break;
      case 4: FB_AGG_LAUNCH(4, 4, 8); break;
      case 5: FB_AGG_LAUNCH(4, 5, 16); break;   // K 16-31: 16 x 16 B in flight per thread
      default: FB_AGG_LAUNCH(2, 7, 32); break;  // K 32-64: 32 x 8 B (the 7-deep tree needs VEC 2)
    }
  } else {
    FB_AGG_LAUNCH(1, 7, 8);
  }
#undef FB_AGG_LAUNCH
  FB_LAUNCH_CHECK();
  return FB_OK;
}

// AggregatorState.weighted_sum (fedopt.py:95): sum_k n_k * (w - w_k) in arrival order, f64,
// the reference's running accumulator itself (no division, no tree).
template <typename TIn>
__global__ void weighted_sum_kernel(AggParams<TIn> P, int K, const float* __restrict__ w, int64_t n,
                                    double* __restrict__ out) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
    const double wg = (double)w[j];
    double s = 0.0;
    for (int k = 0; k < K; ++k) s = __dadd_rn(s, __dmul_rn(P.nk[k], delta_of<TIn>(P.src[k], j, wg)));
    out[j] = s;
  }
}

template <typename TIn>
static int launch_weighted_sum(const void* const* src, const int64_t* n_k, int K, const float* w, int64_t n,
                               double* out, cudaStream_t st) {
  FB_REQUIRE(K >= 1 && K <= FB_MAX_CLIENTS, "n_clients=%d outside [1, %d]", K, FB_MAX_CLIENTS);
  FB_REQUIRE(n > 0 && out && (w || sizeof(TIn) == 8), "weighted_sum: bad args");
  AggParams<TIn> P;
  P.nrep = 0;
  for (int k = 0; k < K; ++k) {
    FB_REQUIRE(src[k] != nullptr && n_k[k] >= 1, "client %d: null pointer or n_k < 1", k);
    P.src[k] = reinterpret_cast<const TIn*>(src[k]);
    P.nk[k] = (double)n_k[k];
    P.pk[k] = 0.0;
  }
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, kNumSMs * 8);
  weighted_sum_kernel<TIn><<<(int)blocks, 256, 0, st>>>(P, K, w, n, out);
  FB_LAUNCH_CHECK();
  return FB_OK;
}

}  // namespace fb

extern "C" int fb_fedagg_weighted_sum(const void* const* d_src, int src_is_f64_delta, const int64_t* n_k,
                                      int n_clients, const float* d_w, int64_t n, double* d_out, void* stream) {
  return src_is_f64_delta
             ? fb::launch_weighted_sum<double>(d_src, n_k, n_clients, d_w, n, d_out, (cudaStream_t)stream)
             : fb::launch_weighted_sum<float>(d_src, n_k, n_clients, d_w, n, d_out, (cudaStream_t)stream);
}

extern "C" int fb_fedagg_step_f32(const float* const* d_client_w, const int64_t* n_k, int n_clients,
                                  int deterministic, const float* d_w, const float* d_m, float* d_w_out,
                                  float* d_m_out, int64_t n, double eta, double mu, int nesterov,
                                  double* d_stats, int64_t* d_first_bad, double* d_pg_out,
                                  void* stream) {
  return fb::launch_fedagg<float>(d_client_w, n_k, n_clients, deterministic, d_w, d_m, d_w_out, d_m_out, n,
                                  eta, mu, nesterov, d_stats, d_first_bad, d_pg_out, 1, (cudaStream_t)stream);
}

// Multi-GPU fused round end over NVLink peer memory (dist.PeerAggregator): the client
// pointers may be peer-GPU addresses (symmetric memory), so the kernel pulls every
// client's slice of this rank's shard straight over NVLink, and w' is stored both to
// w_out and to every replica (the other ranks' copies of the global model) - the
// all-to-all, the reduction and the all-gather in one pass. Same arithmetic and client
// order as fb_fedagg_step_f32, so the result is bit-identical to one GPU.
extern "C" int fb_fedagg_step_f32_peers(const float* const* d_client_w, const int64_t* n_k, int n_clients,
                                        int deterministic, const float* d_w, const float* d_m, float* d_w_out,
                                        float* d_m_out, float* const* d_w_replicas, int n_replicas, int64_t n,
                                        double eta, double mu, int nesterov, double* d_stats,
                                        int64_t* d_first_bad, void* stream) {
  return fb::launch_fedagg<float>(d_client_w, n_k, n_clients, deterministic, d_w, d_m, d_w_out, d_m_out, n, eta, mu,
                                  nesterov, d_stats, d_first_bad, nullptr, 4, (cudaStream_t)stream, d_w_replicas,
                                  n_replicas);
}

// Peer-memory round end plus the per-client round telemetry: d_stats[6 + K] as in
// fb_fedagg_round_norms_f32, each entry this rank's shard's contribution (sum over ranks).
extern "C" int fb_fedagg_round_norms_f32_peers(const float* const* d_client_w, const int64_t* n_k, int n_clients,
                                               int deterministic, const float* d_w, const float* d_m, float* d_w_out,
                                               float* d_m_out, float* const* d_w_replicas, int n_replicas, int64_t n,
                                               double eta, double mu, int nesterov, double* d_stats,
                                               int64_t* d_first_bad, void* stream) {
  FB_REQUIRE(d_stats != nullptr, "fb_fedagg_round_norms_f32_peers needs d_stats (6 + K doubles)");
  return fb::launch_fedagg<float>(d_client_w, n_k, n_clients, deterministic, d_w, d_m, d_w_out, d_m_out, n, eta, mu,
                                  nesterov, d_stats, d_first_bad, nullptr, 3, (cudaStream_t)stream, d_w_replicas,
                                  n_replicas);
}

extern "C" int fb_fedagg_round_norms_f32(const float* const* d_client_w, const int64_t* n_k, int n_clients,
                                         int deterministic, const float* d_w, const float* d_m, float* d_w_out,
                                         float* d_m_out, int64_t n, double eta, double mu, int nesterov,
                                         double* d_stats, int64_t* d_first_bad, void* stream) {
  FB_REQUIRE(d_stats != nullptr, "fb_fedagg_round_norms_f32 needs d_stats (6 + K doubles)");
  return fb::launch_fedagg<float>(d_client_w, n_k, n_clients, deterministic, d_w, d_m, d_w_out, d_m_out, n, eta, mu,
                                  nesterov, d_stats, d_first_bad, nullptr, 3, (cudaStream_t)stream);
}

extern "C" int fb_fedagg_step_f64delta(const double* const* d_deltas, const int64_t* n_k, int n_clients,
                                       int deterministic, const float* d_w, const float* d_m, float* d_w_out,
                                       float* d_m_out, int64_t n, double eta, double mu, int nesterov,
                                       double* d_stats, int64_t* d_first_bad, double* d_pg_out,
                                       void* stream) {
  return fb::launch_fedagg<double>(d_deltas, n_k, n_clients, deterministic, d_w, d_m, d_w_out, d_m_out, n,
                                   eta, mu, nesterov, d_stats, d_first_bad, d_pg_out, 1, (cudaStream_t)stream);
}
