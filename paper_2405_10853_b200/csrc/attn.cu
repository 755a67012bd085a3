// Causal self-attention with ALiBi: entry points and small helpers.
//
// Reference: Block.forward attention  fedforge/model.py:92-98
//   scores = q k^T / sqrt(dh) + bias,  bias[h,i,j] = -slope_h (i - j) (j <= i), -inf above
//   slope_h = 2^(-8 (h+1) / H)        model.py:46-50 (used for every H, incl. H = 12)
// The (H, ctx, ctx) f32 bias buffer of the reference (model.py:115-121) is never built:
// the bias is one FFMA per score in registers.
//
// Layout: qkv is the qkv-GEMM output [B*T][3d] bf16 (q | k | v, head h at columns h*dh),
// o is [B*T][d] bf16 (the attn_proj GEMM operand), lse2 [B][H][T] f32 in base-2 units.
// The kernels themselves are tcgen05/TMEM/TMA (attn_tc.cu forward, attn_bwd_tc.cu
// backward); this file holds the D = rowsum(dO o O) pre-pass, the dQ f32 -> bf16
// finalisation and the C-ABI dispatch. Tensor-core path: T % 128 == 0, dh in {64, 128};
// every other shape (the reference's desk configs: dh 4..32, short or ragged T) runs the
// CUDA-core kernels of attn_generic.cu (fixed order by construction). Both backwards are
// bitwise reproducible: the tensor-core one adds the key blocks' dQ partials in a fixed
// (descending key block) order and writes bf16 dQ itself (attn_bwd_tc.cu, dq_order).
#include "common.cuh"

namespace fb {

// D[bh][t] = sum_c dO * O, one warp per (row, head), 8-byte vector loads
__global__ void attn_bwd_dot_kernel(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dO,
                                    float* __restrict__ D, int B, int T, int H, int dh) {
  const int gw = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (gw >= B * T * H) return;
  const int h = gw % H, row = gw / H;  // row = b*T + t
  const int d = H * dh;
  const __nv_bfloat16* a = o + (int64_t)row * d + h * dh;
  const __nv_bfloat16* g = dO + (int64_t)row * d + h * dh;
  float s = 0.f;
  for (int c = 4 * lane; c < dh; c += 128) {
    const uint2 av = *reinterpret_cast<const uint2*>(a + c), gv = *reinterpret_cast<const uint2*>(g + c);
    const __nv_bfloat162* ap = reinterpret_cast<const __nv_bfloat162*>(&av);
    const __nv_bfloat162* gp = reinterpret_cast<const __nv_bfloat162*>(&gv);
    const float2 a0 = __bfloat1622float2(ap[0]), a1 = __bfloat1622float2(ap[1]);
    const float2 g0 = __bfloat1622float2(gp[0]), g1 = __bfloat1622float2(gp[1]);
    s += a0.x * g0.x + a0.y * g0.y + a1.x * g1.x + a1.y * g1.y;
  }
  s = warp_sum(s);
  if (lane == 0) {
    const int b = row / T, t = row % T;
    D[((int64_t)b * H + h) * T + t] = s;
  }
}

int attn_fwd_generic(const void* qkv, void* o, float* lse, int B, int T, int H, int dh, int use_alibi,
                     cudaStream_t st);
int attn_bwd_generic(const void* qkv, const void* o, const void* dO, const float* lse, void* dqkv, float* work, int B,
                     int T, int H, int dh, int use_alibi, int d_ready, cudaStream_t st);
int g_deterministic = 0;  // fb_set_deterministic (the Python package turns it on at load)

static bool tc_shape(int T, int dh) { return (dh == 64 || dh == 128) && T % 128 == 0; }

template <int DH>
int attn_fwd_tc_launch(const void* qkv, void* o, float* lse, uint8_t* live, int B, int T, int H, int use_alibi,
                       cudaStream_t st);
template <int DH>
int attn_bwd_tc_launch(const void* qkv, const void* dO, const float* lse, const uint8_t* live, const float* Dbuf,
                       float* dq, uint32_t* sem, void* dqkv, int B, int T, int H, int use_alibi, cudaStream_t st);

template <int DH>
static int attn_bwd_launch(const void* qkv, const void* o, const void* dO, const float* lse, const uint8_t* live,
                           void* dqkv, float* work, int B, int T, int H, int use_alibi, int flags, cudaStream_t st) {
  const int d = H * DH;
  float* Dbuf = work;                                           // [B*H*T]
  float* dq = work + (int64_t)B * H * T;                        // [B*T][d] f32 partial sums
  uint32_t* sem = reinterpret_cast<uint32_t*>(dq + (int64_t)B * T * d);  // [B*H*T/32] box counters
  if (!(flags & FB_ATTN_D_READY)) {
    const int nw = B * T * H;
    attn_bwd_dot_kernel<<<(nw + 7) / 8, 256, 0, st>>>((const __nv_bfloat16*)o, (const __nv_bfloat16*)dO, Dbuf, B, T,
                                                      H, DH);
    FB_LAUNCH_CHECK();
  }
  // dQ is written into dqkv by the backward itself (ordered partials, attn_bwd_tc.cu dq_order):
  // no accumulator memset, no finalize pass
  return attn_bwd_tc_launch<DH>(qkv, dO, lse, live, Dbuf, dq, sem, dqkv, B, T, H, use_alibi, st);
}

}  // namespace fb

using namespace fb;

extern "C" int fb_attn_fwd(const void* d_qkv, void* d_o, float* d_lse, uint8_t* d_live, int B, int T, int H, int dh,
                           int use_alibi, void* stream) {
  FB_REQUIRE(B > 0 && H > 0 && T > 0 && dh > 0, "attn_fwd: bad shape B=%d T=%d H=%d dh=%d", B, T, H, dh);
  cudaStream_t st = (cudaStream_t)stream;
  if (!tc_shape(T, dh)) return attn_fwd_generic(d_qkv, d_o, d_lse, B, T, H, dh, use_alibi, st);
  // algorithmic flops: causal lower triangle, QK^T and PV (2*T*d per layer-token fwd)
  const double fl = 2.0 * 2.0 * B * H * (double)T * (T + 1) / 2.0 * dh;
  const int pi = prof_on() ? prof_start(1, st) : -1;
  int rc = dh == 64 ? attn_fwd_tc_launch<64>(d_qkv, d_o, d_lse, d_live, B, T, H, use_alibi, st)
                    : attn_fwd_tc_launch<128>(d_qkv, d_o, d_lse, d_live, B, T, H, use_alibi, st);
  prof_stop(1, pi, st, fl);
  return rc;
}

extern "C" int fb_attn_bwd(const void* d_qkv, const void* d_o, const void* d_do, const float* d_lse,
                           const uint8_t* d_live, void* d_dqkv, float* d_work, int B, int T, int H, int dh, int use_alibi,
                           void* stream) {
  return fb_attn_bwd_ex(d_qkv, d_o, d_do, d_lse, d_live, d_dqkv, d_work, B, T, H, dh, use_alibi, 0, stream);
}

extern "C" int fb_attn_bwd_ex(const void* d_qkv, const void* d_o, const void* d_do, const float* d_lse,
                              const uint8_t* d_live, void* d_dqkv, float* d_work, int B, int T, int H, int dh,
                              int use_alibi, int flags, void* stream) {
  FB_REQUIRE(B > 0 && H > 0 && T > 0 && dh > 0, "attn_bwd: bad shape B=%d T=%d H=%d dh=%d", B, T, H, dh);
  FB_REQUIRE(d_work != nullptr, "attn_bwd: needs a work buffer of B*H*T + B*T*H*dh floats");
  cudaStream_t st = (cudaStream_t)stream;
  if (!tc_shape(T, dh))
    return attn_bwd_generic(d_qkv, d_o, d_do, d_lse, d_dqkv, d_work, B, T, H, dh, use_alibi, flags & FB_ATTN_D_READY,
                            st);
  const double fl = 2.0 * 2.0 * 2.0 * B * H * (double)T * (T + 1) / 2.0 * dh;  // bwd = 2x fwd
  const int pi = prof_on() ? prof_start(2, st) : -1;
  int rc = dh == 64
               ? attn_bwd_launch<64>(d_qkv, d_o, d_do, d_lse, d_live, d_dqkv, d_work, B, T, H, use_alibi, flags, st)
               : attn_bwd_launch<128>(d_qkv, d_o, d_do, d_lse, d_live, d_dqkv, d_work, B, T, H, use_alibi, flags, st);
  prof_stop(2, pi, st, fl);
  return rc;
}

extern "C" int fb_set_deterministic(int enable) {
  fb::g_deterministic = enable ? 1 : 0;  // every kernel is fixed-order in both modes (ABI 3)
  return FB_OK;
}

extern "C" int64_t fb_attn_bwd_work_floats(int B, int T, int H, int dh) {
  if (B <= 0 || T <= 0 || H <= 0 || dh <= 0) return 0;
  // D [B*H*T] + dQ partial sums [B*T*H*dh] + box counters [B*H*ceil(T/32)] (u32)
  return (int64_t)B * H * T + (int64_t)B * T * H * dh + (int64_t)B * H * ((T + 31) / 32);
}
