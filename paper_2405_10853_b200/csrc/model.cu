// Native TinyLM runtime: one call = one micro-batch forward+backward, or one
// whole local optimizer step. Replaces LossEvaluator.loss_and_grad
// (fedforge/model.py:237-250) and the body of train_round's step loop
// (fedforge/trainer.py:78-101).
//
// Everything lives in caller-owned device memory: flat f32 master / grad / m1 / m2
// and a bf16 shadow of the master in the reference's manifest order (no
// flatten copies: GEMMs read weights at manifest offsets of the shadow and the
// wgrad epilogues accumulate straight into the flat f32 gradient), plus one
// workspace carved below. No host synchronisation: the clip decision, the LR
// and the telemetry stay on the device.
#include <algorithm>
#include <vector>

#include "common.cuh"

namespace fb {

struct Layout {
  int64_t embed, pos, lnf_w, lnf_b, head, total;
  struct Blk { int64_t ln1_w, ln1_b, qkv, proj, ln2_w, ln2_b, fc, proj2; };
  std::vector<Blk> blk;
};

static Layout layout_of(const fb_model_cfg& c) {
  Layout L;
  const int64_t V = c.vocab, d = c.d_model;
  int64_t o = 0;
  L.embed = o; o += V * d;
  L.pos = -1;
  if (!c.use_alibi) { L.pos = o; o += (int64_t)c.ctx * d; }
  for (int i = 0; i < c.n_layers; ++i) {
    Layout::Blk b;
    b.ln1_w = o; o += d;
    b.ln1_b = o; o += d;
    b.qkv = o; o += 3 * d * d;
    b.proj = o; o += d * d;
    b.ln2_w = o; o += d;
    b.ln2_b = o; o += d;
    b.fc = o; o += 4 * d * d;
    b.proj2 = o; o += 4 * d * d;
    L.blk.push_back(b);
  }
  L.lnf_w = o; o += d;
  L.lnf_b = o; o += d;
  L.head = o; o += V * d;
  L.total = o;
  return L;
}

// bump allocator over the workspace (dry run when base == nullptr)
struct Arena {
  uint8_t* base;
  int64_t off = 0;
  template <typename T>
  T* take(int64_t n) {
    off = (off + 255) & ~int64_t(255);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += n * (int64_t)sizeof(T);
    return p;
  }
};

struct Acts {  // per-layer saved activations
  float *x_in, *mean1, *rstd1, *x_mid, *mean2, *rstd2, *lse;
  __nv_bfloat16 *ln1, *qkv, *ao, *ln2, *pre, *act;
  uint8_t* live;  // attention dead-block map [B][H][T/128][T/64] (forward writes, backward reads)
};

// split-K partials of the weight-gradient GEMMs: auto-split stops once the 74 CTA pairs are
// busy, so splits * M * N <= (74 + tiles) * 256 * 256 < 16 M floats for every shape
constexpr int64_t kSplitKFloats = 16ll << 20;

struct WS {
  std::vector<Acts> L;
  float *x_out, *meanf, *rstdf, *ce_work, *dx, *dln, *attn_work, *ln_work, *splitk;
  __nv_bfloat16 *lnf, *dlogits, *dxb, *dao, *dqkv, *dfc;
  uint8_t* emb_work;  // sorted-token embedding backward (fb_embed_bwd_sorted)
  int64_t emb_work_bytes;
  int chunk;
};

static WS carve(const fb_model_cfg& c, int B, int T, Arena& A) {
  WS w;
  const int64_t M = (int64_t)B * T, d = c.d_model, V = c.vocab, H = c.n_heads;
  for (int l = 0; l < c.n_layers; ++l) {
    Acts a;
    a.x_in = A.take<float>(M * d);
    a.mean1 = A.take<float>(M);
    a.rstd1 = A.take<float>(M);
    a.ln1 = A.take<__nv_bfloat16>(M * d);
    a.qkv = A.take<__nv_bfloat16>(M * 3 * d);
    a.ao = A.take<__nv_bfloat16>(M * d);
    a.lse = A.take<float>(B * H * T);
    a.live = A.take<uint8_t>((int64_t)B * H * ((T + 127) / 128) * ((T + 63) / 64));
    a.x_mid = A.take<float>(M * d);
    a.mean2 = A.take<float>(M);
    a.rstd2 = A.take<float>(M);
    a.ln2 = A.take<__nv_bfloat16>(M * d);
    a.pre = A.take<__nv_bfloat16>(M * 4 * d);
    a.act = A.take<__nv_bfloat16>(M * 4 * d);
    w.L.push_back(a);
  }
  w.x_out = A.take<float>(M * d);
  w.meanf = A.take<float>(M);
  w.rstdf = A.take<float>(M);
  w.lnf = A.take<__nv_bfloat16>(M * d);
#ifndef FB_LMHEAD_CHUNK
#define FB_LMHEAD_CHUNK 32768
#endif
  w.chunk = (int)std::min<int64_t>(M, FB_LMHEAD_CHUNK);
  w.ce_work = A.take<float>(fb_lmhead_ce_work_floats(w.chunk, (int)V));  // chunk (max, sum) pairs + lse
  w.dlogits = A.take<__nv_bfloat16>((int64_t)w.chunk * V);
  w.dx = A.take<float>(M * d);
  w.dxb = A.take<__nv_bfloat16>(M * d);
  w.dln = A.take<float>(M * d);
  w.dao = A.take<__nv_bfloat16>(M * d);
  w.dqkv = A.take<__nv_bfloat16>(M * 3 * d);
  w.dfc = A.take<__nv_bfloat16>(M * 4 * d);
  w.attn_work = A.take<float>(fb_attn_bwd_work_floats(B, T, (int)H, (int)(d / H)));
  w.ln_work = A.take<float>(2 * 592 * d);
  w.splitk = A.take<float>(kSplitKFloats);
  w.emb_work_bytes = fb_embed_bwd_work_bytes((int)M, (int)V);
  w.emb_work = A.take<uint8_t>(w.emb_work_bytes);
  return w;
}

// The GEMM operands are read by TMA, whose row pitch must be a multiple of 16 bytes: every
// bf16 activation / weight row is d, 3d, 4d or V elements wide and every manifest offset is a
// multiple of d, so d % 8 == 0 and V % 8 == 0 are the only shape constraints. Attention runs
// on tcgen05 for dh in {64, 128} with T % 128 == 0 and on the CUDA-core kernels otherwise.
static int check_cfg(const fb_model_cfg& c, int B, int T) {
  FB_REQUIRE(c.vocab > 0 && c.n_layers >= 0 && c.d_model > 0 && c.n_heads > 0, "bad model config");
  FB_REQUIRE(c.d_model % c.n_heads == 0, "d_model=%d not divisible by n_heads=%d", c.d_model, c.n_heads);
  const int dh = c.d_model / c.n_heads;
  if (c.d_model % 8 || c.vocab % 8 || dh > 256) {
    set_error("GPU path needs d_model %% 8 == 0, vocab %% 8 == 0 and head dim <= 256 (got d=%d dh=%d V=%d)",
              c.d_model, dh, c.vocab);
    return FB_UNSUPPORTED;
  }
  FB_REQUIRE(B > 0 && T >= 2 && T <= c.ctx, "sequence length %d outside [2, context_len=%d]", T, c.ctx);
  return FB_OK;
}

static bool attn_tc_shape(int T, int dh) { return (dh == 64 || dh == 128) && T % 128 == 0; }

}  // namespace fb

using namespace fb;

extern "C" int fb_gemm_bf16(int, int, int, const void*, int64_t, int, const void*, int64_t, int, void*, int64_t, int,
                            const void*, void*, int64_t, void*);
extern "C" int fb_gemm_bf16_rowdot(int, int, int, const void*, int64_t, int, const void*, int64_t, int, void*, int64_t,
                                   const void*, int64_t, float*, int, int, void*);
extern "C" int fb_attn_bwd_ex(const void*, const void*, const void*, const float*, const uint8_t*, void*, float*, int,
                              int, int, int, int, int, void*);
extern "C" int fb_gemm_bf16_splitk(int, int, int, const void*, int64_t, int, const void*, int64_t, int, void*, int64_t,
                                   int, int, void*, int64_t, void*);

#define TRY(x)            \
  do {                    \
    int _rc = (x);        \
    if (_rc) return _rc;  \
  } while (0)

extern "C" int64_t fb_model_n_params(const fb_model_cfg* cfg) { return layout_of(*cfg).total; }

extern "C" int64_t fb_model_workspace_bytes(const fb_model_cfg* cfg, int batch, int T) {
  Arena A{nullptr};
  carve(*cfg, batch, T, A);
  return (A.off + 256 + 255) & ~int64_t(255);
}

extern "C" int fb_model_fwd_bwd(const fb_model_cfg* cfgp, const float* P, const void* shadow, float* G,
                                const int32_t* tok, int B, int T, float grad_scale, double* row_loss, int want_grad,
                                void* ws, int64_t ws_bytes, void* stream) {
  const fb_model_cfg& c = *cfgp;
  TRY(check_cfg(c, B, T));
  FB_REQUIRE(ws && ws_bytes >= fb_model_workspace_bytes(cfgp, B, T), "workspace too small");
  FB_REQUIRE(!want_grad || G, "want_grad needs a gradient buffer");
  cudaStream_t st = (cudaStream_t)stream;
  const Layout Lo = layout_of(c);
  Arena A{reinterpret_cast<uint8_t*>(ws)};
  WS w = carve(c, B, T, A);
  const int M = B * T, d = c.d_model, V = c.vocab, H = c.n_heads, dh = d / H;
  const __nv_bfloat16* S = reinterpret_cast<const __nv_bfloat16*>(shadow);

  // ---------------- forward ----------------
  TRY(fb_embed_fwd(tok, P + Lo.embed, Lo.pos >= 0 ? P + Lo.pos : nullptr, c.n_layers ? w.L[0].x_in : w.x_out, M, T,
                   d, st));
  for (int l = 0; l < c.n_layers; ++l) {
    const Layout::Blk& b = Lo.blk[l];
    Acts& a = w.L[l];
    float* x_next = (l + 1 < c.n_layers) ? w.L[l + 1].x_in : w.x_out;
    TRY(fb_ln_fwd(a.x_in, P + b.ln1_w, P + b.ln1_b, a.ln1, a.mean1, a.rstd1, M, d, st));
    TRY(fb_gemm_bf16(M, 3 * d, d, a.ln1, d, 0, S + b.qkv, d, 0, a.qkv, 3 * d, FB_EPI_BF16, nullptr, nullptr, 0, st));
    TRY(fb_attn_fwd(a.qkv, a.ao, a.lse, a.live, B, T, H, dh, c.use_alibi, st));
    TRY(fb_gemm_bf16(M, d, d, a.ao, d, 0, S + b.proj, d, 0, a.x_mid, d, FB_EPI_RESID_F32, a.x_in, nullptr, d, st));
    TRY(fb_ln_fwd(a.x_mid, P + b.ln2_w, P + b.ln2_b, a.ln2, a.mean2, a.rstd2, M, d, st));
    TRY(fb_gemm_bf16(M, 4 * d, d, a.ln2, d, 0, S + b.fc, d, 0, a.act, 4 * d, FB_EPI_GELU, nullptr, a.pre, 4 * d, st));
    TRY(fb_gemm_bf16(M, d, 4 * d, a.act, 4 * d, 0, S + b.proj2, 4 * d, 0, x_next, d, FB_EPI_RESID_F32, a.x_mid,
                     nullptr, d, st));
  }
  TRY(fb_ln_fwd(w.x_out, P + Lo.lnf_w, P + Lo.lnf_b, w.lnf, w.meanf, w.rstdf, M, d, st));
  // LM head + CE fused (no f32 logits): dlogits(bf16) of each row chunk, then the head backward
  for (int r0 = 0; r0 < M; r0 += w.chunk) {
    const int rows = std::min(w.chunk, M - r0);
    TRY(fb_lmhead_ce(w.lnf + (int64_t)r0 * d, S + Lo.head, tok, r0, rows, T, V, d, grad_scale, want_grad, w.dlogits,
                     w.ce_work, fb_lmhead_ce_work_floats(w.chunk, V), row_loss, st));
    if (want_grad) {
      // d(lnf) = dlogits . W_head ; dW_head += dlogits^T . lnf
      TRY(fb_gemm_bf16_splitk(rows, d, V, w.dlogits, V, 0, S + Lo.head, d, 1, w.dln + (int64_t)r0 * d, d,
                              FB_EPI_F32, 0, w.splitk, kSplitKFloats * 4, st));
      TRY(fb_gemm_bf16(V, d, rows, w.dlogits, V, 1, w.lnf + (int64_t)r0 * d, d, 1, G + Lo.head, d, FB_EPI_ACC_F32,
                       nullptr, nullptr, 0, st));
    }
  }
  if (!want_grad) return FB_OK;

  auto wgrad = [&](int Mg, int Ng, const __nv_bfloat16* A, int64_t lda, const __nv_bfloat16* Bm, int64_t ldb,
                   float* Cg) {
    return fb_gemm_bf16_splitk(Mg, Ng, M, A, lda, 1, Bm, ldb, 1, Cg, Ng, FB_EPI_ACC_F32, 0, w.splitk,
                               kSplitKFloats * 4, st);
  };
  // ---------------- backward ----------------
  TRY(fb_ln_bwd(w.x_out, P + Lo.lnf_w, w.meanf, w.rstdf, w.dln, nullptr, w.dx, w.dxb, G + Lo.lnf_w, G + Lo.lnf_b,
                w.ln_work, M, d, st));
  for (int l = c.n_layers - 1; l >= 0; --l) {
    const Layout::Blk& b = Lo.blk[l];
    Acts& a = w.L[l];
    // MLP: x_next = x_mid + proj2(gelu(fc(ln2(x_mid))))
    TRY(fb_gemm_bf16(M, 4 * d, d, w.dxb, d, 0, S + b.proj2, 4 * d, 1, w.dfc, 4 * d, FB_EPI_DGELU, a.pre, nullptr,
                     4 * d, st));
    TRY(wgrad(d, 4 * d, w.dxb, d, a.act, 4 * d, G + b.proj2));
    TRY(fb_gemm_bf16(M, d, 4 * d, w.dfc, 4 * d, 0, S + b.fc, d, 1, w.dln, d, FB_EPI_F32, nullptr, nullptr, 0, st));
    TRY(wgrad(4 * d, d, w.dfc, 4 * d, a.ln2, d, G + b.fc));
    TRY(fb_ln_bwd(a.x_mid, P + b.ln2_w, a.mean2, a.rstd2, w.dln, w.dx, w.dx, w.dxb, G + b.ln2_w, G + b.ln2_b,
                  w.ln_work, M, d, st));
    // attention: x_mid = x_in + proj(attn(ln1(x_in)))
    // dO = dY W_proj; its epilogue also forms the attention backward's D = rowsum(dO o O)
    int aflags = FB_ATTN_D_READY;
    int rc = attn_tc_shape(T, dh)
                 ? fb_gemm_bf16_rowdot(M, d, d, w.dxb, d, 0, S + b.proj, d, 1, w.dao, d, a.ao, d, w.attn_work, T, dh, st)
                 : FB_UNSUPPORTED;
    if (rc == FB_UNSUPPORTED) {
      aflags = 0;
      rc = fb_gemm_bf16(M, d, d, w.dxb, d, 0, S + b.proj, d, 1, w.dao, d, FB_EPI_BF16, nullptr, nullptr, 0, st);
    }
    TRY(rc);
    TRY(wgrad(d, d, w.dxb, d, a.ao, d, G + b.proj));
    TRY(fb_attn_bwd_ex(a.qkv, a.ao, w.dao, a.lse, a.live, w.dqkv, w.attn_work, B, T, H, dh, c.use_alibi, aflags, st));
    TRY(fb_gemm_bf16(M, d, 3 * d, w.dqkv, 3 * d, 0, S + b.qkv, d, 1, w.dln, d, FB_EPI_F32, nullptr, nullptr, 0, st));
    TRY(wgrad(3 * d, d, w.dqkv, 3 * d, a.ln1, d, G + b.qkv));
    TRY(fb_ln_bwd(a.x_in, P + b.ln1_w, a.mean1, a.rstd1, w.dln, w.dx, w.dx, w.dxb, G + b.ln1_w, G + b.ln1_b,
                  w.ln_work, M, d, st));
  }
  TRY(fb_embed_bwd_sorted(tok, w.dx, G + Lo.embed, Lo.pos >= 0 ? G + Lo.pos : nullptr, M, T, d, V, w.emb_work,
                          w.emb_work_bytes, st));
  return FB_OK;
}

namespace fb {
__global__ void tele_finalize_kernel(const double* __restrict__ row_loss, int n_rows, double loss_scale,
                                     const fb_step_ctl* ctl, const double* __restrict__ part_u,
                                     const double* __restrict__ part_p, const int64_t* first_bad, int64_t n,
                                     double* tele) {
  __shared__ double sh[32];
  double a = 0.0, u = 0.0, p = 0.0;
  for (int i = threadIdx.x; i < n_rows; i += blockDim.x) a += row_loss[i];
  for (int i = threadIdx.x; i < FB_RED_BLOCKS; i += blockDim.x) { u += part_u[i]; p += part_p[i]; }
  a = block_sum(a, sh);
  u = block_sum(u, sh);
  p = block_sum(p, sh);
  if (threadIdx.x == 0) {
    tele[0] = a * loss_scale;
    tele[1] = ctl->grad_sumsq;
    tele[2] = u;
    tele[3] = p;
    tele[4] = ctl->lr;
    tele[5] = (*first_bad < n) ? (double)*first_bad : -1.0;
  }
}
}  // namespace fb

extern "C" int fb_train_step(const fb_model_cfg* cfgp, float* P, void* shadow, float* G, float* m1, float* m2,
                             const fb_data_desc* data, fb_adamw_cfg opt, double lr, double bc1, double bc2,
                             double* tele, double* scratch, double* row_loss, void* ws, int64_t ws_bytes,
                             void* stream) {
  const fb_model_cfg& c = *cfgp;
  const fb_data_desc& D = *data;
  cudaStream_t st = (cudaStream_t)stream;
  FB_REQUIRE(D.micro >= 1 && D.batch >= 1, "micro_batches and batch_size must be >= 1");
  const int fuse = D.fuse > 1 ? (D.fuse < D.micro ? D.fuse : D.micro) : 1;
  // one forward/backward pass covers `fuse` consecutive micro-batches (the last pass the remainder
  // when fuse does not divide micro): micro-batch i's rows are order[cursor + i*B + r], so pass j
  // is the contiguous cursor range [cursor + j*fuse*B, + its rows); the per-token gradient scale
  // below does not depend on the passes
  const int B = D.batch * fuse, T = D.seq_len, M = B * T, passes = (D.micro + fuse - 1) / fuse;
  const int64_t n = layout_of(c).total;
  double* part_g = scratch;
  double* part_u = scratch + FB_RED_BLOCKS;
  double* part_p = scratch + 2 * FB_RED_BLOCKS;
  int64_t* first_bad = reinterpret_cast<int64_t*>(scratch + 3 * FB_RED_BLOCKS);
  fb_step_ctl* ctl = reinterpret_cast<fb_step_ctl*>(scratch + 3 * FB_RED_BLOCKS + 2);
  // token ids for the micro-batch live at the end of the workspace
  const int64_t need = fb_model_workspace_bytes(cfgp, B, T);
  FB_REQUIRE(ws_bytes >= need + (int64_t)M * 4 + 256, "workspace too small for the step");
  int32_t* tok = reinterpret_cast<int32_t*>(reinterpret_cast<uint8_t*>(ws) + ((need + 255) & ~int64_t(255)));
  FB_CUDA_TRY(cudaMemsetAsync(G, 0, sizeof(float) * (size_t)n, st));
  const float gscale = (float)(1.0 / ((double)D.batch * (T - 1)) / D.micro);
  for (int j = 0; j < passes; ++j) {
    const int Bj = D.batch * std::min(fuse, D.micro - j * fuse);  // rows of this pass
    TRY(fb_gather_batch(D.d_corpus, D.d_order, D.n_order, D.cursor + (int64_t)j * B, Bj, T, tok, st));
    TRY(fb_model_fwd_bwd(cfgp, P, shadow, G, tok, Bj, T, gscale, row_loss + (int64_t)j * M, 1, ws, need, st));
  }
  TRY(fb_sumsq_partials(G, n, part_g, st));
  TRY(fb_step_prepare(part_g, lr, bc1, bc2, opt.clip_norm, ctl, st));
  TRY(fb_adamw_step(P, G, m1, m2, shadow, n, opt, ctl, part_u, part_p, first_bad, st));
  tele_finalize_kernel<<<1, 1024, 0, st>>>(row_loss, D.micro * D.batch * T, 1.0 / ((double)D.batch * (T - 1)) / D.micro, ctl,
                                           part_u, part_p, first_bad, n, tele);
  FB_LAUNCH_CHECK();
  return FB_OK;
}
