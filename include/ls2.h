/*
 * ls2.h — C ABI of the B200 (sm_100a) LightSeq2 training hot path.
 *
 * Every entry point takes plain device pointers, sizes, dtype codes and a
 * cudaStream_t passed as void*.  All calls are asynchronous (enqueue only),
 * allocate nothing and never synchronize, so they are CUDA-Graph capturable.
 * Return value: LS2_OK or an LS2_ERR_* status; ls2_last_error() gives text.
 * Status codes map 1:1 onto the reference's exception taxonomy
 * (/root/reference/pkg/src/ftrain/errors.py:4-57).
 *
 * Each function cites the reference operator it replaces
 * (F/ = /root/reference/pkg/src/ftrain/).
 */
#ifndef LS2_H
#define LS2_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* element types */
enum {
  LS2_F16 = 0,
  LS2_BF16 = 1,
  LS2_F32 = 2,
  LS2_F64 = 3,
  LS2_I32 = 4                 /* collectives only (the non-finite counter) */
};

/* status codes (F/errors.py) */
enum {
  LS2_OK = 0,
  LS2_ERR_SHAPE = 1,          /* ShapeMismatch */
  LS2_ERR_TOKEN = 2,          /* TokenOutOfRange */
  LS2_ERR_SEQLEN = 3,         /* SequenceTooLong */
  LS2_ERR_DEGENERATE = 4,     /* DegenerateRow */
  LS2_ERR_ALLMASKED = 5,      /* AllMaskedRow */
  LS2_ERR_TARGET = 6,         /* TargetOutOfRange */
  LS2_ERR_DTYPE = 7,          /* unsupported dtype combination (ShapeMismatch) */
  LS2_ERR_CUDA = 8,           /* CUDA runtime error */
  LS2_ERR_CUBLAS = 9          /* cuBLAS error */
};

/* softmax mask kinds (F/kernels.py:113-144) */
enum {
  LS2_MASK_NONE = 0,
  LS2_MASK_CAUSAL = 1,        /* keep col <= row % lq                          */
  LS2_MASK_PADDING = 2,       /* keep col < valid_len[row / (heads * lq)]     */
  LS2_MASK_DENSE = 3          /* uint8 keep[rows, cols]                        */
};

/* softmax reduction strategies (F/kernels.py:23-24,80-106): AUTO = the shape rule
 * (register template while the row fits, else one CTA per row); SERIAL = the
 * register template where it fits; TREE = one CTA per row (3 passes).  Both keep
 * f64 partition sums, so outputs agree to 1 ULP (T/test_kernels.py:160-171). */
enum {
  LS2_SOFTMAX_AUTO = 0,
  LS2_SOFTMAX_SERIAL = 1,     /* "row_serial"        */
  LS2_SOFTMAX_TREE = 2        /* "row_parallel_tree" */
};

const char* ls2_last_error(void);
int ls2_version(void);
/* dst[i] <- src[i] (nbytes[i] bytes, multiples of 8, 8-byte aligned), i < n <= 8, in ONE
 * launch; src may be pinned host memory (UVA).  The engine's per-step H2D inputs (batch
 * + dropout seed tables) enter a captured step as one kernel node.  Replaces the
 * reference's per-array host->device hand-off of a step's batch (F/engine.py:130-148). */
int ls2_copy_spans(void* const* dst, const void* const* src, const int64_t* nbytes, int n,
                   void* stream);
int ls2_num_kernels_launched(int64_t* out);   /* launches since load (host counter) */

/* ---- counter RNG / dropout masks: F/numerics.py:139-163, F/kernels.py:155-166 ----
 * keep bit i (byte i>>3, bit i&7) == (splitmix64(seed + i*phi) >> 11) >= thresh,
 * thresh = ceil(p * 2^53).  Bit-identical to rand_uniform_array(seed,0,n) >= p. */
int ls2_rand_uniform(double* out, uint64_t seed, int64_t start, int64_t n, void* stream);
int ls2_dropout_bits(uint8_t* bits, int64_t n, uint64_t seed, const uint64_t* seed_ptr, uint64_t thresh, void* stream);
/* every dropout site of a step in one launch (mask bank): desc rows {seed slot,
 * elements, first 32-bit word} (int64, sorted by first word, <= 64 sites); site s
 * writes the keep bits of its elements [0, n_s) (seed seeds[slot_s]) from word
 * first_s of `base` (4-byte aligned, bit i&31 of word i>>5), zero past n_s.
 * stamp/want (optional device scalars): nothing is drawn when *stamp == *want
 * (the bits of that step were already drawn, e.g. beside the previous Adam). */
int ls2_dropout_bits_multi(const int64_t* desc, int nsites, int64_t total_words, uint8_t* base,
                           const uint64_t* seeds, uint64_t thresh, const int64_t* stamp,
                           const int64_t* want, void* stream);
/* the same with at most ctas_per_sm resident CTAs of 256 per SM (0: full
 * occupancy): the engine draws the next step's bank with 1 CTA per SM beside
 * the HBM-bound optimizer, so the two kernels share every SM */
int ls2_dropout_bits_multi_ex(const int64_t* desc, int nsites, int64_t total_words,
                              uint8_t* base, const uint64_t* seeds, uint64_t thresh,
                              const int64_t* stamp, const int64_t* want, int ctas_per_sm,
                              void* stream);
int ls2_bits_to_dense(const uint8_t* bits, void* dense, int dtype, int64_t n, void* stream);
int ls2_dense_to_bits(const void* dense, int dtype, uint8_t* bits, int64_t n, void* stream);

/* ---- fused elementwise tails ----
 * bias+dropout+residual  (F/kernels.py:367-382):
 *   y = keep*(x+bias)*scale + res, keep bits generated (gen=1) or read (gen=0).
 * x,bias,res share dtype tin; y has tout.  scale = f32/f64(1/(1-p)); p==0 -> use_drop=0. */
int ls2_bias_dropout_residual_fwd(const void* x, const void* bias, const void* res, void* y,
                                  uint8_t* keep_bits, int64_t rows, int64_t cols,
                                  int use_drop, int gen, uint64_t seed, const uint64_t* seed_ptr, uint64_t thresh,
                                  double scale, int tin, int tout, void* stream);
/* backward (F/gradients.py:147-159): dx = keep*dy*scale; dbias = column sums of dx
 * (deterministic two-stage; beta=1 accumulates into dbias); dres is dy itself.
 * ws: workspace of ls2_colsum_ws_bytes(rows, cols) bytes. */
int ls2_bias_dropout_residual_bwd(const void* dy, const uint8_t* keep_bits, void* dx,
                                  void* dbias, int tbias, int beta_bias, void* ws,
                                  int64_t rows, int64_t cols, int use_drop, double scale,
                                  int tin, int tout, void* stream);
/* bias+relu+dropout (F/kernels.py:385-403): y = keep*relu(x+b)*scale, relu bit = (x+b)>0 */
int ls2_bias_relu_dropout_fwd(const void* x, const void* bias, void* y, uint8_t* keep_bits,
                              uint8_t* relu_bits, int64_t rows, int64_t cols, int use_drop,
                              int gen, uint64_t seed, const uint64_t* seed_ptr, uint64_t thresh, double scale,
                              int tin, int tout, void* stream);
/* backward (F/gradients.py:162-172) */
int ls2_bias_relu_dropout_bwd(const void* dy, const uint8_t* keep_bits, const uint8_t* relu_bits,
                              void* dx, void* dbias, int tbias, int beta_bias, void* ws,
                              int64_t rows, int64_t cols, int use_drop, double scale,
                              int tin, int tout, void* stream);
int64_t ls2_colsum_ws_bytes(int64_t rows, int64_t cols);
/* deterministic column sums of x[rows, cols] into out[cols] (beta=1 accumulates);
 * used for the bqkv / cross.bq / cross_kv.b gradients (F/model.py:501,726,258) */
int ls2_colsum(const void* x, int tin, void* out, int tout, int beta, void* ws,
               int64_t rows, int64_t cols, void* stream);
/* y[r, c] += bias[c]  (in place; x dtype == bias dtype) */
int ls2_bias_add(void* x, const void* bias, int64_t rows, int64_t cols, int dtype, void* stream);

/* ---- LayerNorm: F/kernels.py:235-270 / F/gradients.py:103-144 ----
 * stats (mu, sigma) have dtype tstat (F32 or F64).  degenerate: optional int*
 * set to 1 when eps == 0 and a row has zero variance. */
int ls2_layernorm_fwd(const void* x, const void* w, const void* b, void* y, void* mu,
                      void* sigma, int* degenerate, int64_t rows, int64_t cols, double eps,
                      int tin, int tout, int tstat, void* stream);
/* dx = LN input grad (+ dres if non-null); dw, db column sums (beta=1 accumulates),
 * dtype tparam.  ws of ls2_layernorm_bwd_ws_bytes(rows, cols) bytes. */
int64_t ls2_layernorm_bwd_ws_bytes(int64_t rows, int64_t cols);
int ls2_layernorm_bwd(const void* dy, const void* x, const void* w, const void* mu,
                      const void* sigma, const void* dres, void* dx, void* dw, void* db,
                      int tparam, int beta_param, void* ws, int64_t rows, int64_t cols,
                      int tin, int tout, int tstat, void* stream);

/* fused bias+dropout+residual -> LayerNorm (F/kernels.py:367-382 then :235-270):
 * yres = keep*(x+bias)*dscale + res (stored), u = LN(yres) with (mu, sigma);
 * use_drop: 0 none, 1 draw keep bits into keep_bits, 2 read keep_bits (mask bank);
 * needs cols % 8 == 0, cols <= 1024, 16-byte aligned operands (else LS2_ERR_SHAPE). */
int ls2_bdr_layernorm_fwd(const void* x, const void* bias, const void* res, void* yres,
                          uint8_t* keep_bits, const void* w, const void* b, void* u, void* mu,
                          void* sigma, int64_t rows, int64_t cols, double eps, int use_drop,
                          uint64_t seed, const uint64_t* seed_ptr, uint64_t thresh, double dscale,
                          int tin, int tout, int tstat, void* stream);
/* fused LayerNorm backward (+ dres) -> bias+dropout+residual backward
 * (F/gradients.py:103-144 then :147-159): dx = LN'(dy) + dres (stored), dproj =
 * keep*dx*dscale (stored), and dw, db, dbias column sums (bit k of beta_mask: accumulate) */
int ls2_layernorm_bwd_bdr(const void* dy, const void* x, const void* w, const void* mu,
                          const void* sigma, const void* dres, void* dx, const uint8_t* keep_bits,
                          void* dproj, int use_drop, double dscale, void* dw, void* db,
                          void* dbias, int tparam, int beta_mask, void* ws, int64_t rows,
                          int64_t cols, int tin, int tout, int tstat, void* stream);

/* ---- softmax family: F/kernels.py:277-331 / F/gradients.py:77-100 ----
 * x rows are the flattened leading dims; mask per LS2_MASK_*.  in_scale
 * multiplies x before the softmax (folds 1/sqrt(hd)); out may alias x.
 * all_masked: optional int* set when a row has no kept element. */
int ls2_softmax_fwd(const void* x, void* y, int64_t rows, int64_t cols, int mask_kind,
                    int64_t lq, int64_t heads, const int64_t* valid_lens,
                    const uint8_t* dense_keep, double in_scale, int* all_masked,
                    int tin, int tout, void* stream);
/* dx = out_scale * q*(dy - sum dy*q); dx may alias dy */
int ls2_softmax_bwd(const void* dy, const void* q, void* dx, int64_t rows, int64_t cols,
                    double out_scale, int tin, int tout, void* stream);
int ls2_log_softmax_fwd(const void* h, void* y, int64_t rows, int64_t cols, int tin,
                        int tout, void* stream);
/* the same with an explicit LS2_SOFTMAX_* strategy (the `strategy=` argument) */
int ls2_softmax_fwd_strategy(const void* x, void* y, int64_t rows, int64_t cols, int mask_kind,
                             int64_t lq, int64_t heads, const int64_t* valid_lens,
                             const uint8_t* dense_keep, double in_scale, int* all_masked,
                             int strategy, int tin, int tout, void* stream);
int ls2_log_softmax_fwd_strategy(const void* h, void* y, int64_t rows, int64_t cols, int strategy,
                                 int tin, int tout, void* stream);

/* ---- fused short-sequence attention (fp16, head dim 64, Lq/Lk <= 128) ----
 * Replaces scores = QK^T/sqrt(hd) -> softmax_forward(mask) -> P V -> merge heads
 * (F/model.py:362-376) and its backward (F/model.py:482-495, F/gradients.py:77-100).
 * Operands are addressed per (b, h) as base + b*L*ld + h*64 (row stride ld), so Q/K/V
 * are read straight from the fused projection and outputs land in merged layouts.
 * probs: [B, H, Lq, Lk] (written by fwd, read by bwd). mask: NONE/CAUSAL/PADDING. */
int ls2_attention_supported(int64_t lq, int64_t lk, int64_t hd, int dtype);
int ls2_attention_fwd(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v,
                      int64_t ldv, void* probs, void* o, int64_t ldo, int64_t batch,
                      int64_t heads, int64_t lq, int64_t lk, int64_t hd, int mask_kind,
                      const int64_t* lens, double scale, void* stream);
int ls2_attention_bwd(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v,
                      int64_t ldv, const void* probs, const void* dout, int64_t lddo, void* dq,
                      int64_t lddq, void* dk, int64_t lddk, void* dv, int64_t lddv,
                      int64_t batch, int64_t heads, int64_t lq, int64_t lk, int64_t hd,
                      double scale, void* stream);
/* the same, also leaving the projection biases' gradient partials: row b of
 * csq / csk / csv (f64, row pitch ld*, columns h*64..h*64+63) = column sums over
 * the sequence of the stored dQ / dK / dV of (b, h); any may be NULL.  Summing
 * the B rows (fixed order) gives dbias — the engine's deferred finish does it. */
int ls2_attention_bwd_bias(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v,
                           int64_t ldv, const void* probs, const void* dout, int64_t lddo,
                           void* dq, int64_t lddq, void* dk, int64_t lddk, void* dv, int64_t lddv,
                           int64_t batch, int64_t heads, int64_t lq, int64_t lk, int64_t hd,
                           double scale, double* csq, int64_t ldcsq, double* csk, int64_t ldcsk,
                           double* csv, int64_t ldcsv, void* stream);

/* ---- fused attention on tcgen05/TMEM/TMA (fp16, head dim 64, Lq/Lk <= 64) ----
 * Same operation and operand addressing as ls2_attention_fwd / _bwd_bias (F/model.py:
 * 362-376, 482-495; F/kernels.py:277-307; F/gradients.py:77-100), but the forward
 * keeps only per-row softmax statistics instead of the [B, H, Lq, Lk]
 * probabilities: stats = float2[B*H*Lq] (row max of the scaled masked scores,
 * 1 / row sum); the backward recomputes P from Q, K and the stats (bit-identical
 * to the forward's P) and therefore needs the same mask.  Operand pointers and
 * row pitches must be 16-byte aligned.  LS2_ATTN_TC=0 disables (supported -> 0). */
int ls2_attention_tc_supported(int64_t lq, int64_t lk, int64_t hd, int dtype);
/* debugging aid: per-CTA phase timestamps (globaltimer ns, u64[grid][8]) of the
 * following attention_tc launches are written to buf (NULL turns it off) */
int ls2_attention_tc_trace(void* buf);
int ls2_attention_tc_fwd(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v,
                         int64_t ldv, void* stats, void* o, int64_t ldo, int64_t batch,
                         int64_t heads, int64_t lq, int64_t lk, int64_t hd, int mask_kind,
                         const int64_t* lens, double scale, void* stream);
int ls2_attention_tc_bwd(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v,
                         int64_t ldv, const void* stats, const void* dout, int64_t lddo, void* dq,
                         int64_t lddq, void* dk, int64_t lddk, void* dv, int64_t lddv,
                         int64_t batch, int64_t heads, int64_t lq, int64_t lk, int64_t hd,
                         int mask_kind, const int64_t* lens, double scale, double* csq,
                         int64_t ldcsq, double* csk, int64_t ldcsk, double* csv, int64_t ldcsv,
                         void* stream);
/* the same with the forward's output O (ctx, [B, Lq, H*64] at row stride ldo): required by
 * the flash kernels (self-attention 128 < Lq == Lk <= 512: 128-row blocks, K / V
 * streamed through TMA rings, scores never in HBM; stats are then [B][H][Lq][4] floats
 * (max, 1/sum, D = rowsum(dO * O), -), and the bias partials have one row per
 * (batch, 128-row block)); shorter rows ignore O */
int ls2_attention_tc_bwd_o(const void* q, int64_t ldq, const void* k, int64_t ldk, const void* v,
                           int64_t ldv, const void* o, int64_t ldo, void* stats, const void* dout,
                           int64_t lddo, void* dq, int64_t lddq, void* dk, int64_t lddk, void* dv,
                           int64_t lddv, int64_t batch, int64_t heads, int64_t lq, int64_t lk,
                           int64_t hd, int mask_kind, const int64_t* lens, double scale,
                           double* csq, int64_t ldcsq, double* csk, int64_t ldcsk, double* csv,
                           int64_t ldcsv, void* stream);

/* ---- label-smoothed CE: F/kernels.py:338-360, F/gradients.py:47-74 ----
 * row_stats (double[rows*2]) receives per-row (loss, correct) partials;
 * out3 (double[3]) = (loss_sum, token_count, correct) after the fixed-order reduce. */
int ls2_ls_ce_fwd(const void* logq, const int64_t* targets, double* row_stats, double* out3,
                  int* bad_target, int64_t rows, int64_t v, double alpha, int64_t pad_id,
                  int has_pad, int tin, void* stream);
int ls2_ls_ce_bwd(const void* probs, const int64_t* targets, void* dh, int* bad_target,
                  int64_t rows, int64_t v, double alpha, int64_t pad_id, int has_pad,
                  double grad_scale, int tin, int tout, void* stream);
/* fused criterion (F/model.py:908-932): logits -> (loss, count, correct) and, when
 * dlogits != NULL, dlogits = (softmax - a/V - (1-a)[k]) * grad_scale written over
 * the row (may alias logits).  logq_out (optional) receives log-softmax. */
int ls2_criterion_fused(const void* logits, const int64_t* targets, void* dlogits,
                        void* logq_out, double* row_stats, double* out3, int* bad_target,
                        int64_t rows, int64_t v, double alpha, int64_t pad_id, int has_pad,
                        double grad_scale, int t_logits, void* stream);
/* the same over rows of pitch ld >= v (ld = v rounded up to a multiple of 8, for
 * vocabularies like BERT's 30522): columns [v, ld) are ignored on read and hold
 * don't-care values in dlogits; 16-bit logits, two rows must fit in 200 KB */
int ls2_criterion_fused_ld(const void* logits, int64_t ld, const int64_t* targets, void* dlogits,
                           double* row_stats, double* out3, int* bad_target, int64_t rows,
                           int64_t v, double alpha, int64_t pad_id, int has_pad,
                           double grad_scale, int t_logits, void* stream);

/* ---- embedding: F/kernels.py:203-228 / F/gradients.py:20-44 ---- */
int ls2_embedding_fwd(const void* emb, const void* pos, const int64_t* tokens, void* y,
                      uint8_t* keep_bits, int* bad_token, int64_t batch, int64_t len,
                      int64_t d, int64_t vocab, double emb_scale, int use_drop, int gen,
                      uint64_t seed, const uint64_t* seed_ptr, uint64_t thresh, double drop_scale, int tin, int tout,
                      void* stream);
/* dE[tok] += emb_scale*keep*dy*drop_scale (atomic scatter, tgrad F32/F64);
 * dP[l] (beta_pos: 0 write rows [0,len) and zero [len,max_len), 1 accumulate) */
int ls2_embedding_bwd(const void* dy, const int64_t* tokens, const uint8_t* keep_bits,
                      void* dE, void* dP, int tgrad, int beta_pos, int64_t batch,
                      int64_t len, int64_t d, int64_t max_len, double emb_scale,
                      int use_drop, double drop_scale, int tin, void* stream);

/* ---- workspace trainer: F/trainer.py:125-181, F/engine.py:152-157 ----
 * hyper: f32 constants precomputed on the host exactly as numpy does:
 *   [lr, beta1, 1-beta1, beta2, 1-beta2, eps, wd, loss_scale]
 * bc: (f32(1-beta1^t), f32(1-beta2^t)) table of bc_len rows indexed by t,
 *   followed by beta1, beta2 as two f64 values; for t >= bc_len the kernel
 *   forms f32(1 - beta^t) itself in f64.  The step t is either `t_host` (>0)
 *   or read as *applied + 1 from the device counter.
 * skip: the update is skipped when *nonfinite != 0 or (loss && !isfinite(*loss)). */
int ls2_adam(uint16_t* p16, const uint16_t* g16, float* m, float* v, int64_t n,
             const float* hyper, const float* bc_table, int64_t bc_len, int64_t t_host,
             const int64_t* applied, const int* nonfinite, const double* loss, void* stream);
/* ls2_adam over the rank's shard of a sharded-optimizer step: spans = n_spans {offset,
 * length} int64 pairs (device) of the flat workspace, max_len = the longest span */
int ls2_adam_spans(uint16_t* p16, const uint16_t* g16, float* m, float* v, const int64_t* spans,
                   int64_t n_spans, int64_t max_len, const float* hyper, const float* bc_table,
                   int64_t bc_len, int64_t t_host, const int64_t* applied, const int* nonfinite,
                   const double* loss, void* stream);
int ls2_sgd(uint16_t* p16, const uint16_t* g16, float* vel, int64_t n, const float* hyper,
            const int* nonfinite, const double* loss, void* stream);
/* applied += (nonfinite==0 && loss finite)  — one thread */
int ls2_step_commit(int64_t* applied, const int* nonfinite, const double* loss,
                    int* applied_flag, void* stream);
/* step_commit and the step report {loss sum, tokens, correct, applied, non-finite}
 * (f64 x 5, the train-step D2H source) in one launch; totals = (loss, count, correct).
 * applied == NULL: the report alone (the engine issues it before the optimizer, so the
 * host reads the step's metrics while the update still runs); report may be pinned host
 * memory (UVA), written directly by the kernel */
int ls2_step_report(int64_t* applied, const int* nonfinite, const double* totals, double* report,
                    void* stream);
/* g16 = RNE(acc32 * f32(loss_scale / max(count,1)) * post), count = out3[1] (device) or
 * count_host (>=0); nonfinite += #non-finite g16 (NULL to skip) */
int ls2_scale_narrow(const float* acc32, uint16_t* g16, int64_t n, double loss_scale,
                     const double* out3, int64_t count_host, float post, int* nonfinite,
                     void* stream);
int ls2_count_nonfinite_f16(const uint16_t* g16, int64_t n, int* nonfinite, void* stream);
/* deferred column-sum finishes fused with the narrow: desc rows {dst, cols, part, nblk,
 * stride, k} (int64), chunks {desc index, first column} (int32, one CTA per 64 columns);
 * g16[dst + c] = RNE(f32(sum_g partial[part + g*stride + k*cols + c]) * scale) */
int ls2_finish_narrow(const int64_t* desc, const int32_t* chunks, int64_t n_chunks,
                      const double* partial_base, uint16_t* g16, double loss_scale,
                      const double* out3, int64_t count_host, float post, int* nonfinite,
                      void* stream);
/* the same column sums unscaled into the fp32 accumulator: acc32[dst + c] = f32(sum_g ...)
 * (data parallelism reduces them in fp32 with the rest of the bucket, then narrows) */
int ls2_finish_acc32(const int64_t* desc, const int32_t* chunks, int64_t n_chunks,
                     const double* partial_base, float* acc32, void* stream);
/* number of partial rows the column-sum producers write (0: shape not deferrable) */
int ls2_colsum_nblk(int64_t rows, int64_t cols, int dtype);
int ls2_layernorm_bwd_nblk(int64_t rows, int64_t cols);

/* ---- GEMM on cuBLAS (F/kernels.py:413-447), row-major semantics ----
 * C[b] = alpha * op(A[b]) @ op(B[b]) + beta * C[b], batch index b = (i, j) with
 * i < n1, j < n2 and element offsets i*sX1 + j*sX2.  Compute fp32 (fp64 for F64),
 * never TF32.  Types: (A,B) same; C may be wider (F16/BF16 in -> F32 out). */
void* ls2_blas_create(void);
void ls2_blas_destroy(void* h);
int ls2_gemm(void* h, int trans_a, int trans_b, int64_t m, int64_t n, int64_t k,
             double alpha, const void* A, int64_t lda, int64_t sA1, int64_t sA2,
             const void* B, int64_t ldb, int64_t sB1, int64_t sB2, double beta, void* C,
             int64_t ldc, int64_t sC1, int64_t sC2, int64_t n1, int64_t n2, int tab, int tc,
             void* ptr_scratch, int ptrs_ready, void* stream);
/* count (<= 64) independent products of one shape, C_i = alpha op(A_i) op(B_i)
 * + beta C_i, as ONE cuBLAS pointer-array batch.  a_list / b_list / c_list are
 * HOST arrays of device pointers; they reach the device through a kernel's
 * parameters (graph-capturable), ptr_scratch: >= 3*count device pointers;
 * ptrs_ready=1: ptr_scratch already holds this list (cached per address list).
 * Used to issue a step's weight-gradient GEMMs batched across layers
 * (replaces the per-layer dW = dy^T x of F/model.py:451,461,479,500,678,688,706). */
int ls2_gemm_list(void* h, int trans_a, int trans_b, int64_t m, int64_t n, int64_t k,
                  double alpha, const void* const* a_list, int64_t lda,
                  const void* const* b_list, int64_t ldb, double beta, void* const* c_list,
                  int64_t ldc, int count, int tab, int tc, void* ptr_scratch,
                  int ptrs_ready, void* stream);
/* bytes of device scratch ls2_gemm needs for pointer-array batches
 * (ptrs_ready=1: the caller guarantees ptr_scratch already holds this call's
 *  A/B/C pointer arrays, e.g. cached per static arena address) */
int64_t ls2_gemm_scratch_bytes(int64_t n1, int64_t n2);
/* dense GEMM on tcgen05/TMEM/TMA (hand-written, gemm_tc.cu), the row-major
 * convention of ls2_gemm_lt: C[m x n] = alpha*op(A)@op(B) (+ bias[n]) (+ C when beta = 1),
 * A/B fp16 or bf16, C the same type or f32, fp32 accumulation in tensor memory.
 * split = 0 picks the cluster split-K factor (1/2/4/8; small-output, long-K products
 * reduce the partial tiles through DSMEM in rank order, deterministic); split = -1 the
 * persistent one-SM kernel (double-buffered TMEM accumulator); -2 / -3 the cta_group::2
 * kernels over SM pairs (256-row tiles; -2 one tile per pair, K-major A and B only;
 * -3 persistent with a TMA-store epilogue, every operand layout, n % 128 == 0).
 * ls2_gemm_tc_supported: 1 when the shape/dtype/alignment is covered (n a multiple of 128,
 * 16-byte aligned operands, ld multiples of 8; m and k arbitrary). */
int ls2_gemm_tc_supported(int trans_a, int trans_b, int64_t m, int64_t n, int64_t k,
                          const void* A, int64_t lda, const void* B, int64_t ldb, double beta,
                          const void* C, int64_t ldc, int tab, int tc);
int ls2_gemm_tc(int trans_a, int trans_b, int64_t m, int64_t n, int64_t k, double alpha,
                const void* A, int64_t lda, const void* B, int64_t ldb, double beta, void* C,
                int64_t ldc, const void* bias, int tab, int tc, int split, void* stream);
/* weight-gradient form of ls2_gemm_tc: C (f32) = A^T B (+ C when beta), A [k x m],
 * B [k x n] fp16 row-major.  ls2_wgrad_tc_split returns the split factor it uses,
 * or 0 when m, n are not multiples of 128. */
int ls2_wgrad_tc_split(int64_t m, int64_t n, int64_t k);
int ls2_wgrad_tc(const void* A, int64_t lda, const void* B, int64_t ldb, float* C, int64_t ldc,
                 int64_t m, int64_t n, int64_t k, int beta, void* stream);
/* GEMM on cuBLASLt that also writes a bias gradient from its epilogue (BGRADA/B):
 * which = 0 -> bgrad[i] = sum_k op(A)[i, k] (length m), 1 -> bgrad[j] = sum_k op(B)[k, j]
 * (length n); bgrad has type tc (fp32 accumulation).  The weight gradient dW = dY^T X
 * with which = 0 yields the layer's bias gradient sum_rows dY in the same pass
 * (F/model.py:501,726,766).  LS2_ERR_CUBLAS if Lt has no algorithm for it. */
int ls2_gemm_lt_bgrad(void* h, int trans_a, int trans_b, int64_t m, int64_t n, int64_t k,
                      double alpha, const void* A, int64_t lda, const void* B, int64_t ldb,
                      double beta, void* C, int64_t ldc, void* bgrad, int which, int tab, int tc,
                      void* stream);
/* plain GEMM on cuBLASLt with an optional fused bias epilogue (C += bias[n] per row);
 * LS2_ERR_CUBLAS if no Lt algorithm supports the combination (caller falls back) */
int ls2_gemm_lt(void* h, int trans_a, int trans_b, int64_t m, int64_t n, int64_t k, double alpha,
                const void* A, int64_t lda, const void* B, int64_t ldb, double beta, void* C,
                int64_t ldc, const void* bias, int tab, int tc, void* stream);

/* ---- data-parallel exchange: NCCL over NVLink/NVSwitch ----
 * Replaces the reference's "already-reduced gradients" contract (F/engine.py:4-7,
 * SPEC.md:569).  libnccl.so.2 is bound at run time (the copy already loaded by
 * torch.distributed when present).  ls2_comm_allreduce is a stream-ordered sum
 * (in place when send == recv) and may be captured into a CUDA graph. */
int ls2_comm_load(const char* path);
int ls2_comm_version(int* out);
int ls2_comm_unique_id(uint8_t* out128);
int ls2_comm_init(void** comm_out, int nranks, int rank, const uint8_t* id128, int device);
int ls2_comm_allreduce(void* comm, const void* send, void* recv, int64_t count, int dtype,
                       void* stream);
/* sharded-optimizer exchange (SPEC.md:573 makes the 1/N element shard legal):
 * reduce-scatter (sum; rank r gets [r*count, (r+1)*count) of the sum, in place when
 * recv == send + rank*count) and all-gather (in place when send == recv + rank*count) */
int ls2_comm_reduce_scatter(void* comm, const void* send, void* recv, int64_t count, int dtype,
                            void* stream);
int ls2_comm_all_gather(void* comm, const void* send, void* recv, int64_t count, int dtype,
                        void* stream);
int ls2_comm_destroy(void* comm);

#ifdef __cplusplus
}
#endif
#endif /* LS2_H */
