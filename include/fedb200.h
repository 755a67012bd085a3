/*
 * libfedb200 — C ABI of the B200-native (sm_100a) federated-round hot path.
 *
 * Drop-in boundary for the reference `fedforge` (arXiv 2405.10853). The reference
 * has no FFI of its own (pure Python over numpy / torch-CPU), so each entry point
 * below names the Python call site it replaces; the Python shim
 * `paper_2405_10853_b200` binds these through ctypes.
 *
 * Conventions
 *   - plain pointers and sizes; every pointer argument named d_* is DEVICE memory
 *     owned by the caller; the library never allocates or frees in a hot call
 *   - every entry returns int (fb_status); fb_last_error() has the message
 *   - every entry takes an explicit CUDA stream (cudaStream_t passed as void*)
 *   - entries are reentrant; no global mutable state except a tensor-map cache
 */
#ifndef FEDB200_H
#define FEDB200_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

enum fb_status { FB_OK = 0, FB_BAD_ARG = 1, FB_CUDA_ERROR = 2, FB_NONFINITE = 3, FB_UNSUPPORTED = 4 };

#define FB_ABI_VERSION 3  /* 2: fused LM-head CE replaces fb_ce_fwd_bwd; fb_data_desc.fuse; deterministic attention bwd.
                             3: attention bwd always fixed-order (ordered dQ partials), d_work adds box counters */
#define FB_MAX_CLIENTS 64
#define FB_MAX_REPLICAS 8  /* w' destinations besides w_out (peer GPUs), fb_fedagg_step_f32_peers */
#define FB_RED_BLOCKS 1184 /* fixed reduction grid: 148 SMs x 8, deterministic partials */

const char* fb_last_error(void);
int fb_abi_version(void);
int fb_device_check(void); /* FB_OK iff device 0 is sm_100 (B200) */

/* ---- server: aggregation + outer optimizer (K13) ---------------------------------
 * Replaces AggregatorState.finalize  (fedforge/fedopt.py:129-144)
 *      then server_step              (fedforge/fedopt.py:167-201)
 * client weights w_k (f32) arrive in the order the pairwise tree / running sum uses
 * (deterministic: ascending client id; streaming: arrival order). The f64 pseudo-
 * gradient  sum_k n_k (f64(w) - f64(w_k)) / sum n_k  and the outer step run in f64
 * registers; m' is rounded to f32 before it feeds w' (fedopt.py:189-196).
 * d_stats (optional, 3 doubles): ||pg||^2, ||w'||^2, ||m'||^2.
 * d_first_bad (optional, 1 int64): lowest index with a non-finite w' or m' (or n).
 * d_pg_out (optional, n doubles): the f64 pseudo-gradient itself (AggregatorState.finalize).
 * d_w_out/d_m_out may be NULL to only materialise the pseudo-gradient.
 * Returns FB_OK; the caller checks d_first_bad (no host sync inside). */
int fb_fedagg_step_f32(const float* const* d_client_w, const int64_t* n_k, int n_clients,
                       int deterministic, const float* d_w, const float* d_m, float* d_w_out,
                       float* d_m_out, int64_t n, double eta, double mu, int nesterov,
                       double* d_stats, int64_t* d_first_bad, double* d_pg_out, void* stream);
/* Multi-GPU variant (one rank's shard): client pointers may be NVLink peer addresses and
 * w' is also stored to n_replicas peer copies of the global model, so the round-end
 * all-to-all, fused step and all-gather are one kernel. Bit-identical to the above.
 * d_stats (optional) here holds 6 doubles: the 3 above, then this shard's |w|^2,
 * |sum p_k w_k|^2, |w - sum p_k w_k|^2 (summed over ranks -> compute_round_norms). */
int fb_fedagg_step_f32_peers(const float* const* d_client_w, const int64_t* n_k, int n_clients,
                             int deterministic, const float* d_w, const float* d_m, float* d_w_out,
                             float* d_m_out, float* const* d_w_replicas, int n_replicas, int64_t n,
                             double eta, double mu, int nesterov, double* d_stats, int64_t* d_first_bad,
                             void* stream);
/* Same fused step plus the round telemetry of compute_round_norms (fedforge/metrics.py:177-215)
 * as side reductions of the same HBM pass: d_stats[6 + K] = |pg|^2, |w'|^2, |m'|^2, |w|^2,
 * |sum p_k w_k|^2, |w - sum p_k w_k|^2, then |w_k|^2 per client (p_k = n_k / sum n). */
int fb_fedagg_round_norms_f32(const float* const* d_client_w, const int64_t* n_k, int n_clients,
                              int deterministic, const float* d_w, const float* d_m, float* d_w_out,
                              float* d_m_out, int64_t n, double eta, double mu, int nesterov,
                              double* d_stats, int64_t* d_first_bad, void* stream);
/* Both: the peer-memory round end with the 6 + K round-norm stats of this rank's shard. */
int fb_fedagg_round_norms_f32_peers(const float* const* d_client_w, const int64_t* n_k, int n_clients,
                                    int deterministic, const float* d_w, const float* d_m, float* d_w_out,
                                    float* d_m_out, float* const* d_w_replicas, int n_replicas, int64_t n,
                                    double eta, double mu, int nesterov, double* d_stats,
                                    int64_t* d_first_bad, void* stream);
/* Same contract for reference-format f64 deltas (ClientUpdate.delta, fedopt.py:26-46). */
int fb_fedagg_step_f64delta(const double* const* d_deltas, const int64_t* n_k, int n_clients,
                            int deterministic, const float* d_w, const float* d_m, float* d_w_out,
                            float* d_m_out, int64_t n, double eta, double mu, int nesterov,
                            double* d_stats, int64_t* d_first_bad, double* d_pg_out, void* stream);

/* AggregatorState.weighted_sum (fedopt.py:95): d_out[n] (f64) = sum_k n_k * delta_k in the
 * given (arrival) order, delta_k = f64(w) - f64(w_k) for f32 client weights (src_is_f64_delta
 * = 0, d_w needed) or the f64 deltas themselves (1). Bitwise the reference's running sum. */
int fb_fedagg_weighted_sum(const void* const* d_src, int src_is_f64_delta, const int64_t* n_k,
                           int n_clients, const float* d_w, int64_t n, double* d_out, void* stream);

/* ---- client optimizer (K10-K12) --------------------------------------------------- */
/* d_partials[FB_RED_BLOCKS] = per-block sum of x^2 (f64). l2_norm: params.py:126-133 */
int fb_sumsq_partials(const float* d_x, int64_t n, double* d_partials, void* stream);
/* one block: sum the partials in fixed order -> d_out[0] (f64) */
int fb_sum_partials(const double* d_partials, int n_partials, double* d_out, void* stream);

typedef struct {
  double beta1, beta2, eps, weight_decay, clip_norm;
} fb_adamw_cfg; /* AdamWConfig, localopt.py:22-38 */

/* Per-step device control block: written by fb_step_prepare on device, read by AdamW. */
typedef struct {
  double lr, bc1, bc2;       /* lr_at(offset+s); 1-beta1^t; 1-beta2^t (host-computed) */
  double grad_sumsq;         /* ||g||^2 of the micro-batch-mean gradient */
  double clip_scale;         /* max_norm/raw when raw > max_norm */
  int32_t clip_active;       /* raw > max_norm (strict, localopt.py:140) */
  int32_t pad;
} fb_step_ctl;

/* Reduce d_partials (grad sum of squares) -> ctl->grad_sumsq, clip decision. */
int fb_step_prepare(const double* d_partials, double lr, double bc1, double bc2,
                    double clip_norm, fb_step_ctl* d_ctl, void* stream);
/* Fused AdamW over the flat vector (localopt.py:61-96, clip localopt.py:132-143):
 * f64 math, f32 p/m1/m2, optional bf16 shadow of p'. Per-block partials of ||u||^2
 * and ||p'||^2 go to d_part_u / d_part_p ([FB_RED_BLOCKS] each, optional);
 * d_first_bad (optional) gets the lowest index with non-finite p'. */
int fb_adamw_step(float* d_p, const float* d_g, float* d_m1, float* d_m2, void* d_shadow_bf16,
                  int64_t n, fb_adamw_cfg cfg, const fb_step_ctl* d_ctl, double* d_part_u,
                  double* d_part_p, int64_t* d_first_bad, void* stream);
/* f32 -> bf16 copy (shadow weights at round start) */
int fb_cast_bf16(const float* d_x, void* d_y, int64_t n, void* stream);

/* ---- dense GEMM on tcgen05 (K3, K5, K6, K7, LM head) -------------------------------
 * D[m,n] = sum_k A(m,k) * B(n,k), bf16 inputs, fp32 accumulation in TMEM.
 * a_major/b_major: 0 = K-major (A stored [M][lda], B stored [N][ldb]),
 *                  1 = MN-major (A stored [K][lda], B stored [K][ldb]).
 * Epilogues (fused in the TMEM->register drain): */
enum fb_epilogue {
  FB_EPI_BF16 = 0,       /* C(bf16) = acc */
  FB_EPI_F32 = 1,        /* C(f32) = acc */
  FB_EPI_ACC_F32 = 2,    /* C(f32) += acc   (wgrad micro-batch accumulation) */
  FB_EPI_RESID_F32 = 3,  /* C(f32) = aux(f32) + acc  (residual add; aux may alias C) */
  FB_EPI_GELU = 4,       /* C(bf16) = gelu_erf(acc); aux_out(bf16) = acc (pre-activation) */
  FB_EPI_DGELU = 5,      /* C(bf16) = acc * gelu_erf'(aux(bf16)) */
  FB_EPI_RESID_F32_BF16 = 6, /* C(f32) = aux(f32) + acc and aux_out(bf16) = same */
  FB_EPI_BF16_ROWDOT = 7,    /* C(bf16) = acc and per-head row dots with aux: fb_gemm_bf16_rowdot only */
  FB_EPI_CE_EXP = 8          /* LM head for fb_lmhead_ce: C(bf16) = exp(acc - m_c) per 32-column chunk c,
                                aux_out(float2)[c * ld_aux + row] = (m_c, sum of the chunk's exps);
                                K-major operands only */
};
/* 1 (default): use the 2-SM cta_group::2 256x256-tile kernel where the tile count fills the
 * 74 CTA pairs; 0: 1-SM kernels only (A/B comparison and tests) */
int fb_gemm_set_2sm(int enable);
/* A/B experiments: force the 2-SM raster group height (0 = automatic). */
int fb_gemm_set_group_m(int group_m);
int fb_gemm_bf16(int M, int N, int K, const void* d_A, int64_t lda, int a_major,
                 const void* d_B, int64_t ldb, int b_major, void* d_C, int64_t ldc, int epilogue,
                 const void* d_aux, void* d_aux_out, int64_t ld_aux, void* stream);

/* Split-K variant for short-M/N, long-K products (weight gradients over many tokens):
 * ksplit partial f32 products go to d_ws (ksplit*M*N floats) and are reduced in fixed
 * split order into C (+= for FB_EPI_ACC_F32) — deterministic. ksplit <= 0: auto. */
int fb_gemm_bf16_splitk(int M, int N, int K, const void* d_A, int64_t lda, int a_major,
                        const void* d_B, int64_t ldb, int b_major, void* d_C, int64_t ldc, int epilogue,
                        int ksplit, void* d_ws, int64_t ws_bytes, void* stream);

/* Attention-backward pre-pass fused into the out-projection dgrad (dO = dY W_proj):
 * C(bf16) = dO and D[b][h][t] = sum_{c in head h} bf16(dO)[row][c] * O[row][c] (row = b*T + t,
 * f32 [B][H][T], the rowsum(dO o O) of the attention backward, model.py:92-98). Runs on the
 * 2-SM kernel only (each epilogue warp drains 128 head-aligned columns of its rows);
 * returns FB_UNSUPPORTED (nothing launched) when that kernel does not apply, so the caller
 * falls back to fb_gemm_bf16 + fb_attn_bwd's own pre-pass. Needs 128 % dh == 0, dh % 32 == 0. */
int fb_gemm_bf16_rowdot(int M, int N, int K, const void* d_A, int64_t lda, int a_major,
                        const void* d_B, int64_t ldb, int b_major, void* d_C, int64_t ldc,
                        const void* d_O, int64_t ld_o, float* d_D, int T, int dh, void* stream);

/* ---- transformer pieces (model.py:75-150, :222-229) --------------------------------- */
int fb_embed_fwd(const int32_t* d_tok, const float* d_emb, const float* d_pos, float* d_x,
                 int n_tok, int T, int d, void* stream);
/* gemb[tok[r]] += dx[r] (and gpos[r % T] += dx[r]) with f32 atomics: arrival-order sums,
 * not bitwise reproducible run to run. The runtime uses fb_embed_bwd_sorted. */
int fb_embed_bwd(const int32_t* d_tok, const float* d_dx, float* d_gemb, float* d_gpos,
                 int n_tok, int T, int d, int vocab, void* stream);
/* Deterministic embedding backward (model.py:109 / :145 grads): token ids are
 * stably radix-sorted with their positions; a run of equal ids is cut into 8 contiguous
 * ranges of ascending positions, each summed in order, the range sums added in order and
 * once into gemb (one thread per column when d % 8 != 0); positions are summed in ascending
 * batch row. Bitwise reproducible. d_work: fb_embed_bwd_work_bytes(n_tok, vocab) bytes. */
int64_t fb_embed_bwd_work_bytes(int n_tok, int vocab);
int fb_embed_bwd_sorted(const int32_t* d_tok, const float* d_dx, float* d_gemb, float* d_gpos,
                        int n_tok, int T, int d, int vocab, void* d_work, int64_t work_bytes,
                        void* stream);
/* LayerNorm eps 1e-5 (model.py:81,84,113): y(bf16) = LN(x), saves mean/rstd */
int fb_ln_fwd(const float* d_x, const float* d_gamma, const float* d_beta, void* d_y_bf16,
              float* d_mean, float* d_rstd, int rows, int d, void* stream);
/* dx(f32) = dres(f32, optional) + LN'(dy); optional bf16 copy of dx; dgamma/dbeta +=.
 * d_work: 2 * 592 * d floats of scratch (per-CTA dgamma/dbeta partials) */
int fb_ln_bwd(const float* d_x, const float* d_gamma, const float* d_mean, const float* d_rstd,
              const float* d_dy, const float* d_dres, float* d_dx, void* d_dx_bf16,
              float* d_dgamma, float* d_dbeta, float* d_work, int rows, int d, void* stream);
/* Causal attention with the reference's ALiBi slopes 2^(-8(h+1)/H) (model.py:46-65, 92-98).
 * qkv: [B*T][3d] bf16 (q|k|v, head h at columns h*dh); o: [B*T][d] bf16; lse: [B][H][T] f32
 * (base 2). d_live (optional, uint8 [B][H][T/128][T/64]): the forward marks each causal
 * block of 128 queries x 64 keys live (1) or dead (0: every softmax weight underflowed to
 * exactly 0, which ALiBi causes far from the diagonal) and skips the dead blocks' PV; the
 * backward skips the MMAs of blocks the map says are dead. Results are bit-identical with
 * and without the map. tcgen05 kernels for T % 128 == 0 and dh in {64, 128}; any other
 * shape (dh <= 256, any T) runs fixed-order CUDA-core kernels (d_live unused). */
int fb_attn_fwd(const void* d_qkv, void* d_o, float* d_lse, uint8_t* d_live, int B, int T, int H,
                int dh, int use_alibi, void* stream);
int fb_attn_bwd(const void* d_qkv, const void* d_o, const void* d_do, const float* d_lse,
                const uint8_t* d_live, void* d_dqkv, float* d_work, int B, int T, int H, int dh,
                int use_alibi, void* stream);
/* flags: FB_ATTN_D_READY = d_work[0 : B*H*T] already holds D = rowsum(dO o O)
 * (fb_gemm_bf16_rowdot), so the backward skips its D pre-pass. */
enum { FB_ATTN_D_READY = 1 };
int fb_attn_bwd_ex(const void* d_qkv, const void* d_o, const void* d_do, const float* d_lse,
                   const uint8_t* d_live, void* d_dqkv, float* d_work, int B, int T, int H, int dh,
                   int use_alibi, int flags, void* stream);
/* Kept for ABI compatibility: every kernel is fixed-order (bitwise reproducible, the reference's
 * test_trainer.py:56-63 replay contract) whatever the flag. The tcgen05 attention backward adds
 * each query block's per-key-block dQ partials in descending key-block order (per-box counters in
 * d_work) and writes bf16 dQ itself; ABI 2's slab buffer and finalize pass are gone. */
int fb_set_deterministic(int enable);
/* floats of d_work that fb_attn_bwd / fb_attn_bwd_ex need: D [B*H*T], dQ partial sums [B*T*H*dh],
 * box counters [B*H*ceil(T/32)] */
int64_t fb_attn_bwd_work_floats(int B, int T, int H, int dh);
/* Fused LM head + mean next-token cross-entropy (model.py:114, :150, :226-229) for
 * rows [row0, row0 + rows) of a B x T batch: logits = x W^T on tcgen05 with the FB_EPI_CE_EXP
 * epilogue (no f32 logits in HBM: bf16 e = exp(x - m_chunk) plus (m, sum) per 32-column chunk),
 * then per row lse and loss = lse - x[target] (target logit recomputed in f32 from the same bf16
 * operands; 0 on each sequence's last position, which is not scored) -> d_row_loss[row0 + r]
 * (f64), and, when want_grad, dlogits(bf16) = scale * (softmax - onehot) written in place of e
 * (the target entry from the f32 target logit). d_x: [rows][d] bf16; d_w: [V][d] bf16;
 * d_work: fb_lmhead_ce_work_floats(rows, V) floats. V % 8 == 0, d % 8 == 0. */
int64_t fb_lmhead_ce_work_floats(int rows, int V);
int fb_lmhead_ce(const void* d_x, const void* d_w, const int32_t* d_tok, int row0, int rows, int T, int V, int d,
                 float scale, int want_grad, void* d_dlogits, float* d_work, int64_t work_floats,
                 double* d_row_loss, void* stream);

/* ---- data feed: BatchIterator.next_batch on device (data.py:152-161) ----------------
 * rows = order[(cursor + i) mod n_order]; tok[i][t] = corpus[rows[i]*T + t] */
int fb_gather_batch(const uint16_t* d_corpus, const int64_t* d_order, int64_t n_order,
                    int64_t cursor, int batch, int T, int32_t* d_tok, void* stream);


/* ---- native runtime: whole TinyLM micro-batch and whole local step ----------------
 * TinyLMConfig (model.py:28-43). Flat parameter layout = the reference manifest
 * order (model.py:184-190): embed, [pos_embed], per block {ln1.w, ln1.b, qkv, attn_proj,
 * ln2.w, ln2.b, mlp_fc, mlp_proj}, ln_f.w, ln_f.b, head. GPU path constraints (TMA row
 * pitch): d_model % 8 == 0, vocab % 8 == 0, head dim <= 256; any T in [2, ctx]. */
typedef struct {
  int32_t vocab, ctx, n_layers, d_model, n_heads, use_alibi;
} fb_model_cfg;

int64_t fb_model_n_params(const fb_model_cfg* cfg);
/* bytes of device workspace for one micro-batch of `batch` sequences of length T */
int64_t fb_model_workspace_bytes(const fb_model_cfg* cfg, int batch, int T);
/* Forward (+ backward when want_grad) of one micro-batch: LossEvaluator.loss_and_grad
 * (model.py:237-250). Gradients ACCUMULATE into d_grad (f32, manifest order), scaled by
 * grad_scale (1 / (B*(T-1)) / n_micro); per-row CE goes to d_row_loss[B*T] (f64,
 * 0 on each sequence's last position). d_shadow = bf16 copy of d_params. */
int fb_model_fwd_bwd(const fb_model_cfg* cfg, const float* d_params, const void* d_shadow, float* d_grad,
                     const int32_t* d_tok, int batch, int T, float grad_scale, double* d_row_loss,
                     int want_grad, void* d_ws, int64_t ws_bytes, void* stream);

typedef struct {
  const uint16_t* d_corpus; /* token stream (uint16, data.py:57) */
  const int64_t* d_order;   /* this client's sample order (data.py:141-144) */
  int64_t n_order;          /* n_k */
  int32_t seq_len, batch, micro;
  int32_t fuse;             /* micro-batches per forward/backward pass (0 or 1 = one; the last pass takes
                               the remainder when fuse does not divide micro): the same rows and the same
                               per-token gradient scale, so the same step; fewer, larger GEMMs / attention
                               grids. Workspace for batch * fuse rows */
  int64_t cursor;           /* sample cursor at the start of this step */
} fb_data_desc;

/* One local optimizer step of train_round (trainer.py:78-101): micro-batch fwd/bwd with
 * gradient accumulation, global-norm clip decision on device, fused AdamW (+ bf16
 * shadow), telemetry into d_tele[8]: {sum of micro mean losses / micro, ||g||^2,
 * ||u||^2, ||w'||^2, lr, first non-finite param index (as double, or -1)}.
 * d_scratch: FB_RED_BLOCKS*2 + 8 doubles + sizeof(fb_step_ctl); d_row_loss: micro*B*T doubles. */
int fb_train_step(const fb_model_cfg* cfg, float* d_params, void* d_shadow, float* d_grad, float* d_m1,
                  float* d_m2, const fb_data_desc* data, fb_adamw_cfg opt, double lr, double bc1, double bc2,
                  double* d_tele, double* d_scratch, double* d_row_loss, void* d_ws, int64_t ws_bytes,
                  void* stream);


/* ---- live kernel profiling (used by bench.py inside its timed region) --------------
 * While enabled, every fb_gemm_bf16 / fb_attn_* launch is bracketed by CUDA events on
 * its own stream (first max_launches launches per category). fb_profile_end syncs
 * and returns per category {total ms, timed launches, algorithmic flops} for
 * categories 0 = GEMM, 1 = attention fwd, 2 = attention bwd in out[0..8], and the
 * number of launches seen per category (timed or past the cap) in out[9..11]. */
int fb_profile_begin(int max_launches);
int fb_profile_end(double* out12);

#ifdef __cplusplus
}
#endif
#endif
