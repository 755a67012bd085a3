// K10-K12: gradient norm, clip decision and the fused AdamW step over the flat
// parameter vector, plus the device data feed.
//
// Reference: adamw_step  fedforge/localopt.py:61-96 (f64 math, f32 moments,
//            update rounded to f32 before it is applied);  clip_grad localopt.py:132-143;
//            l2_norm params.py:126-133;  BatchIterator.next_batch data.py:152-161.
//
// B200 design: the parameters, gradients and both moments are single flat f32
// buffers in manifest order, so the "multi-tensor" AdamW is one streaming pass
// with 128-bit accesses over 4 arrays (30 B/param incl. the bf16 shadow write).
// Every f64 operation uses an explicit _rn intrinsic in numpy's evaluation order,
// so identical inputs give bit-identical outputs. Reductions use a fixed grid
// (FB_RED_BLOCKS) with per-block partials and a fixed-order final sum, making
// them run-to-run deterministic; the clip decision stays on the device (no host
// synchronisation inside a local step).
#include "common.cuh"

namespace fb {

__global__ void __launch_bounds__(256) sumsq_partials_kernel(const float* __restrict__ x, int64_t n,
                                                             double* __restrict__ part) {
  __shared__ double sh[8];
  double s = 0.0;
  const int64_t nvec = n / 4;
  const bool al = ((uintptr_t)x % 16) == 0;
  if (al) {
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += (int64_t)gridDim.x * blockDim.x) {
      float4 a = ld_stream_f4(x + 4 * v);
      s += (double)a.x * a.x + (double)a.y * a.y + (double)a.z * a.z + (double)a.w * a.w;
    }
    for (int64_t j = 4 * nvec + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
      s += (double)x[j] * x[j];
  } else {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
      s += (double)x[j] * x[j];
  }
  s = block_sum(s, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = s;
}

__global__ void sum_partials_kernel(const double* __restrict__ part, int np, double* out) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) s += part[i];
  s = block_sum(s, sh);
  if (threadIdx.x == 0) *out = s;
}

__global__ void step_prepare_kernel(const double* __restrict__ part, double lr, double bc1, double bc2,
                                    double clip_norm, fb_step_ctl* ctl) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int i = threadIdx.x; i < FB_RED_BLOCKS; i += blockDim.x) s += part[i];
  s = block_sum(s, sh);
  if (threadIdx.x == 0) {
    double raw = __dsqrt_rn(s);
    ctl->lr = lr;
    ctl->bc1 = bc1;
    ctl->bc2 = bc2;
    ctl->grad_sumsq = s;
    ctl->clip_active = raw > clip_norm ? 1 : 0;
    ctl->clip_scale = raw > clip_norm ? __ddiv_rn(clip_norm, raw) : 1.0;
  }
}

struct AdamWScalars {
  double b1, omb1, b2, omb2, eps, wd;
};

__device__ __forceinline__ void adamw_one(float& p32, float g32, float& m1_32, float& m2_32, const AdamWScalars& c,
                                          double lr, double bc1, double bc2, int clip, double cs, double& su,
                                          double& sp) {
  if (clip) g32 = __double2float_rn(__dmul_rn((double)g32, cs));
  const double g = (double)g32;
  const double p = (double)p32;
  const double m1 = __dadd_rn(__dmul_rn(c.b1, (double)m1_32), __dmul_rn(c.omb1, g));
  const double m2 = __dadd_rn(__dmul_rn(c.b2, (double)m2_32), __dmul_rn(__dmul_rn(c.omb2, g), g));
  const double m1h = __ddiv_rn(m1, bc1);
  const double m2h = __ddiv_rn(m2, bc2);
  const double u64 = __dmul_rn(lr, __dadd_rn(__ddiv_rn(m1h, __dadd_rn(__dsqrt_rn(m2h), c.eps)), __dmul_rn(c.wd, p)));
  const float u = __double2float_rn(u64);
  p32 = __double2float_rn(__dsub_rn(p, (double)u));
  m1_32 = __double2float_rn(m1);
  m2_32 = __double2float_rn(m2);
  su += (double)u * (double)u;
  sp += (double)p32 * (double)p32;
}

__global__ void __launch_bounds__(256) adamw_kernel(float* __restrict__ p, const float* __restrict__ g,
                                                    float* __restrict__ m1, float* __restrict__ m2,
                                                    __nv_bfloat16* __restrict__ shadow, int64_t n, AdamWScalars c,
                                                    const fb_step_ctl* __restrict__ ctl, double* part_u,
                                                    double* part_p, unsigned long long* first_bad, int vec) {
  __shared__ double sh[8];
  const double lr = ctl->lr, bc1 = ctl->bc1, bc2 = ctl->bc2, cs = ctl->clip_scale;
  const int clip = ctl->clip_active;
  double su = 0.0, sp = 0.0;
  unsigned long long bad = ~0ull;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t done = 0;
  if (vec) {
    const int64_t nvec = n / 4;
    for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < nvec; v += stride) {
      const int64_t j = 4 * v;
      float4 pv = *reinterpret_cast<const float4*>(p + j);
      float4 gv = ld_stream_f4(g + j);
      float4 av = *reinterpret_cast<const float4*>(m1 + j);
      float4 bv = *reinterpret_cast<const float4*>(m2 + j);
      adamw_one(pv.x, gv.x, av.x, bv.x, c, lr, bc1, bc2, clip, cs, su, sp);
      adamw_one(pv.y, gv.y, av.y, bv.y, c, lr, bc1, bc2, clip, cs, su, sp);
      adamw_one(pv.z, gv.z, av.z, bv.z, c, lr, bc1, bc2, clip, cs, su, sp);
      adamw_one(pv.w, gv.w, av.w, bv.w, c, lr, bc1, bc2, clip, cs, su, sp);
      st_stream_f4(p + j, pv);
      st_stream_f4(m1 + j, av);
      st_stream_f4(m2 + j, bv);
      if (shadow) {
        __nv_bfloat162 lo = __floats2bfloat162_rn(pv.x, pv.y), hi = __floats2bfloat162_rn(pv.z, pv.w);
        uint2 pk;
        pk.x = *reinterpret_cast<uint32_t*>(&lo);
        pk.y = *reinterpret_cast<uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(shadow + j) = pk;
      }
      if (!(isfinite(pv.x) && isfinite(pv.y) && isfinite(pv.z) && isfinite(pv.w))) {
        int64_t b = !isfinite(pv.x) ? j : !isfinite(pv.y) ? j + 1 : !isfinite(pv.z) ? j + 2 : j + 3;
        if ((unsigned long long)b < bad) bad = (unsigned long long)b;
      }
    }
    done = 4 * nvec;
  }
  for (int64_t j = done + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
    float pj = p[j], a = m1[j], b = m2[j];
    adamw_one(pj, g[j], a, b, c, lr, bc1, bc2, clip, cs, su, sp);
    p[j] = pj;
    m1[j] = a;
    m2[j] = b;
    if (shadow) shadow[j] = __float2bfloat16_rn(pj);
    if (!isfinite(pj) && (unsigned long long)j < bad) bad = (unsigned long long)j;
  }
  if (first_bad) {
    for (int o = 16; o > 0; o >>= 1) {
      unsigned long long t = __shfl_xor_sync(0xffffffffu, bad, o);
      bad = t < bad ? t : bad;
    }
    if ((threadIdx.x & 31) == 0 && bad != ~0ull) atomicMin(first_bad, bad);
  }
  su = block_sum(su, sh);
  sp = block_sum(sp, sh);
  if (threadIdx.x == 0) {
    if (part_u) part_u[blockIdx.x] = su;
    if (part_p) part_p[blockIdx.x] = sp;
  }
}

__global__ void cast_bf16_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ y, int64_t n) {
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
    y[j] = __float2bfloat16_rn(x[j]);
}

__global__ void gather_batch_kernel(const uint16_t* __restrict__ corpus, const int64_t* __restrict__ order,
                                    int64_t n_order, int64_t cursor, int batch, int T, int32_t* __restrict__ tok) {
  const int i = blockIdx.x;
  const int64_t row = order[(cursor + i) % n_order];
  const uint16_t* src = corpus + row * (int64_t)T;
  for (int t = threadIdx.x; t < T; t += blockDim.x) tok[(int64_t)i * T + t] = (int32_t)src[t];
}

}  // namespace fb

using namespace fb;

extern "C" int fb_sumsq_partials(const float* d_x, int64_t n, double* d_partials, void* stream) {
  FB_REQUIRE(n > 0 && d_x && d_partials, "fb_sumsq_partials: bad args");
  sumsq_partials_kernel<<<FB_RED_BLOCKS, 256, 0, (cudaStream_t)stream>>>(d_x, n, d_partials);
  FB_LAUNCH_CHECK();
  return FB_OK;
}

extern "C" int fb_sum_partials(const double* d_partials, int n_partials, double* d_out, void* stream) {
  FB_REQUIRE(n_partials > 0 && d_partials && d_out, "fb_sum_partials: bad args");
  sum_partials_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(d_partials, n_partials, d_out);
  FB_LAUNCH_CHECK();
  return FB_OK;
}

extern "C" int fb_step_prepare(const double* d_partials, double lr, double bc1, double bc2, double clip_norm,
                               fb_step_ctl* d_ctl, void* stream) {
  FB_REQUIRE(d_partials && d_ctl, "fb_step_prepare: null pointer");
  FB_REQUIRE(clip_norm > 0, "max_norm must be positive, got %g", clip_norm);
  step_prepare_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(d_partials, lr, bc1, bc2, clip_norm, d_ctl);
  FB_LAUNCH_CHECK();
  return FB_OK;
}

extern "C" int fb_adamw_step(float* d_p, const float* d_g, float* d_m1, float* d_m2, void* d_shadow_bf16, int64_t n,
                             fb_adamw_cfg cfg, const fb_step_ctl* d_ctl, double* d_part_u, double* d_part_p,
                             int64_t* d_first_bad, void* stream) {
  FB_REQUIRE(n > 0 && d_p && d_g && d_m1 && d_m2 && d_ctl, "fb_adamw_step: bad args");
  FB_REQUIRE(cfg.beta1 >= 0 && cfg.beta1 < 1 && cfg.beta2 >= 0 && cfg.beta2 < 1, "betas must be in [0, 1)");
  FB_REQUIRE(cfg.eps > 0 && cfg.weight_decay >= 0, "bad eps / weight_decay");
  AdamWScalars c{cfg.beta1, 1.0 - cfg.beta1, cfg.beta2, 1.0 - cfg.beta2, cfg.eps, cfg.weight_decay};
  cudaStream_t st = (cudaStream_t)stream;
  if (d_first_bad) FB_CUDA_TRY(cudaMemsetAsync(d_first_bad, 0x7f, sizeof(int64_t), st));
  int vec = ((uintptr_t)d_p % 16 == 0) && ((uintptr_t)d_g % 16 == 0) && ((uintptr_t)d_m1 % 16 == 0) &&
            ((uintptr_t)d_m2 % 16 == 0) && ((uintptr_t)d_shadow_bf16 % 8 == 0);
  adamw_kernel<<<FB_RED_BLOCKS, 256, 0, st>>>(d_p, d_g, d_m1, d_m2, (__nv_bfloat16*)d_shadow_bf16, n, c, d_ctl,
                                              d_part_u, d_part_p, (unsigned long long*)d_first_bad, vec);
  FB_LAUNCH_CHECK();
  return FB_OK;
}

extern "C" int fb_cast_bf16(const float* d_x, void* d_y, int64_t n, void* stream) {
  FB_REQUIRE(n > 0 && d_x && d_y, "fb_cast_bf16: bad args");
  cast_bf16_kernel<<<kNumSMs * 8, 256, 0, (cudaStream_t)stream>>>(d_x, (__nv_bfloat16*)d_y, n);
  FB_LAUNCH_CHECK();
  return FB_OK;
}

extern "C" int fb_gather_batch(const uint16_t* d_corpus, const int64_t* d_order, int64_t n_order, int64_t cursor,
                               int batch, int T, int32_t* d_tok, void* stream) {
  FB_REQUIRE(n_order > 0 && batch > 0 && T > 0 && cursor >= 0, "fb_gather_batch: bad args");
  gather_batch_kernel<<<batch, 256, 0, (cudaStream_t)stream>>>(d_corpus, d_order, n_order, cursor, batch, T, d_tok);
  FB_LAUNCH_CHECK();
  return FB_OK;
}
