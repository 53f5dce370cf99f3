/*
 * mecefo.h — C-ABI of the B200-native MeCeFO degraded-step engine.
 *
 * Drop-in boundary for the step / failure-handling path of the reference CPU
 * simulator `faultsim` (pkg/src/faultsim, arXiv 2510.16415). The reference is
 * pure Python over float64 numpy arrays; its "FFI" is the module-level
 * function surface that `faultsim.harness` dispatches through by attribute
 * lookup (harness.py:209-249). Each entry point below names the reference
 * function it replaces (file:line under pkg/src/faultsim/).
 *
 * Conventions
 *  - All tensor arguments are caller-owned DEVICE pointers (e.g. PyTorch
 *    allocations), row-major, plus sizes and a cudaStream_t passed as void*.
 *    Nothing here allocates device memory except mecefo_engine_create (a small
 *    RoPE table); scratch space comes from a caller-provided workspace.
 *  - Activations that feed GEMMs are in the engine's compute precision
 *    (MECEFO_PREC_BF16 -> tcgen05 tensor cores, MECEFO_PREC_F32 -> fp32 FFMA
 *    path for the 1e-4 parity mode). Master weights, the residual stream,
 *    gradients and optimizer state are fp32.
 *  - Gradient outputs ACCUMULATE: g += alpha * dL/dW. alpha carries the
 *    Eq. (1) 1/|N_{l,#}| factor (cluster.py:292-322); a rank outside an active
 *    set simply passes NULL for that gradient (select, never multiply, so a
 *    non-finite value on an excluded rank cannot leak).
 *  - Every call is stream-ordered and asynchronous; no host synchronisation.
 *  - Return value: MECEFO_OK or an error code mirroring the reference's
 *    exception classes (errors.py:8-33); mecefo_last_error() gives the text.
 */
#ifndef MECEFO_H
#define MECEFO_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  MECEFO_OK = 0,
  MECEFO_ERR_CONTRACT = 1,      /* errors.py:12 ContractViolation */
  MECEFO_ERR_NUMERICAL = 2,     /* errors.py:16 NumericalFailure */
  MECEFO_ERR_SVD_NOCONV = 3,    /* errors.py:20 SvdConvergenceError */
  MECEFO_ERR_UNRECOVERABLE = 4, /* errors.py:28 UnrecoverableRankError */
  MECEFO_ERR_CONSISTENCY = 5,   /* errors.py:32 ConsistencyError */
  MECEFO_ERR_CONFIG = 6,        /* errors.py:8 ConfigError */
  MECEFO_ERR_CUDA = 7           /* CUDA runtime failure (no reference analogue) */
};

enum { MECEFO_PREC_F32 = 0, MECEFO_PREC_BF16 = 1 };

/* Bits of the engine's device status word (sticky until reset). The kernels
 * never read or write out of range on bad input: a token id outside
 * [0, vocab) gathers a zero row and is skipped by the scatter-add, a bad
 * target contributes loss 0 and a zero dlogits row. The host reads the word at
 * iteration boundaries and raises what the reference raises:
 *   BAD_TOKEN / BAD_TARGET -> ContractViolation (model.py:463, 505 IndexError)
 *   NONFINITE_GRAD         -> NumericalFailure  (optim.py:55-57 _check_grad) */
enum { MECEFO_STATUS_BAD_TOKEN = 1, MECEFO_STATUS_BAD_TARGET = 2, MECEFO_STATUS_NONFINITE_GRAD = 4 };

/* model.py:30-31 CACHE_FULL / CACHE_FFN_INPUT_ONLY */
enum { MECEFO_CACHE_FULL = 0, MECEFO_CACHE_FFN_INPUT_ONLY = 1 };

/* model.py:40-61 ModelConfig (+ the engine's compute precision). */
typedef struct {
  int64_t vocab, hidden, heads, ffn, layers, seq_len;
  int32_t rope;
  int32_t precision;
} mecefo_dims;

typedef struct mecefo_engine mecefo_engine;

/* model.py:64-90 LayerWeights, in the engine's HBM layout: q,k,v stacked as
 * one (3m, m) matrix and gate,up stacked as one (2f, m) matrix — exactly the
 * canonical parameter order of model.py:35, so a flat parameter buffer in
 * that order provides these views without copies. *_c are the operand copies
 * in compute precision (the masters themselves in fp32 mode). */
typedef struct {
  const float* w_qkv;
  const float* w_o;
  const float* norm_mha;
  const float* w_gu;
  const float* w_down;
  const float* norm_ffn;
  const void* w_qkv_c;
  const void* w_o_c;
  const void* w_gu_c;
  const void* w_down_c;
} mecefo_layer_weights;

/* model.py:376-381 BlockCache. x and x1 (fp32, (tokens, hidden)) are the
 * whole lean cache; the remaining fields are used only by CACHE_FULL. */
typedef struct {
  float* x;
  float* x1;
  void* h1;
  float* inv1;
  void* qkv;
  void* ctx;
  float* lse;
  void* h2;
  float* inv2;
  void* gu;
  void* act;
} mecefo_block_cache;

/* Per-layer gradient accumulators (fp32, canonical shapes); NULL = skip. */
typedef struct {
  float* qkv;      /* (3m, m): q, k, v */
  float* o;        /* (m, m) */
  float* norm_mha; /* (m) */
  float alpha_mha;
  float* gu;       /* (2f, m): gate, up */
  float* down;     /* (m, f) */
  float* norm_ffn; /* (m) */
  float alpha_ffn;
} mecefo_layer_grads;

/* approx.py:45-63 ProjectionCache.basis, per kind in FFN_KINDS order
 * (gate, up, down): V1 (in, rank_pad) and its transpose (rank_pad, in) in
 * compute precision, zero beyond rank[k] = min(r, in) (approx.py:79). */
typedef struct {
  int32_t rank[3];
  int32_t rank_pad;
  const void* v1[3];
  const void* v1t[3];
  /* optional: gate and up bases packed side by side, v1_gu = [V1_gate | V1_up]
   * (in, 2 rank_pad), and v1t_gu = [V1_gate^T ; V1_up^T] (2 rank_pad, in).
   * When set, the gate/up low-rank Wgrads run as one merged chain. */
  const void* v1_gu;
  const void* v1t_gu;
} mecefo_projection;

/* AdamW segment: one named parameter of the flat buffer (optim.py:75-93). */
typedef struct {
  int64_t offset;
  int64_t numel;
  float step_size; /* lr / (1 - beta1^t) */
  float inv_bc2;   /* 1 / (1 - beta2^t) */
  float lr_wd;     /* lr * weight_decay */
  int32_t pad;
} mecefo_adam_segment;

const char* mecefo_last_error(void);
const char* mecefo_version(void);

/* dims->ffn may be any width (model.py:40-61 accepts e.g. LLaMA-1B's 5461):
 * the engine rounds it up to mecefo_padded_ffn(ffn), a multiple of 8 (16-byte
 * bf16 rows for TMA). Every ffn-dimensioned buffer the caller passes (W_gate /
 * W_up rows, W_down columns and row stride, the FFN activations and their
 * gradients, the down-projection basis rows) uses the padded width with the
 * pad rows/columns zero — exact: they contribute nothing and their gradients
 * stay zero. */
int64_t mecefo_padded_ffn(int64_t ffn);
int mecefo_engine_create(mecefo_engine** out, const mecefo_dims* dims);
int mecefo_engine_destroy(mecefo_engine* e);
/* Device pointer to the engine's int32 status word (MECEFO_STATUS_* bits);
 * stream-ordered reset. */
int mecefo_status_device(mecefo_engine* e, int32_t** device_status);
int mecefo_status_reset(mecefo_engine* e, void* stream);
/* Stream-ordered copy of the status word into (pinned) host memory; graph-capturable. */
int mecefo_status_snapshot(mecefo_engine* e, int32_t* host_status, void* stream);
/* Stream-ordered zero fill of a device range (gradient / loss accumulators). */
int mecefo_memset_zero(void* device_ptr, size_t bytes, void* stream);

/* Workspace bytes needed by any call below at `tokens` rows and padded rank. */
size_t mecefo_workspace_bytes(const mecefo_engine* e, int64_t tokens, int32_t rank_pad);

/* model.py:398-418 forward_block. Reads cache->x, writes cache->x1, y and
 * (mode == FULL) the full-cache fields. y may alias the next block's x. */
int mecefo_forward_block(mecefo_engine* e, const mecefo_layer_weights* lw, mecefo_block_cache* cache, float* y,
                         void* y_c, int64_t tokens, int32_t mode, void* ws, size_t ws_bytes, void* stream);

/* forward_block of a chain of blocks (model.py:461-463 calls them in turn):
 * as mecefo_forward_block, plus
 *   flags & MECEFO_FWD_H1_READY: cache->h1 / cache->inv1 already hold this
 *     block's rmsnorm(x) * norm_mha and 1/rms (written by the previous block
 *     of the chain), so its own norm pass is skipped;
 *   next_norm_gain != NULL: the block also writes the NEXT block's
 *     h1 = rmsnorm(y) * next_norm_gain into next_h1 (compute precision) and
 *     1/rms into next_inv1 — fused into the residual down-projection when
 *     hidden = 512 (one kernel owns whole rows), a separate pass otherwise.
 * Same results as calling mecefo_forward_block per block. */
#define MECEFO_FWD_H1_READY 1
int mecefo_forward_block_chained(mecefo_engine* e, const mecefo_layer_weights* lw, mecefo_block_cache* cache,
                                 float* y, int64_t tokens, int32_t mode, int32_t flags, const float* next_norm_gain,
                                 void* next_h1, float* next_inv1, void* ws, size_t ws_bytes, void* stream);

/* approx.py:99-134 backward_block_neighbor: skip the MHA backward, recompute
 * the FFN from x1, FFN Wgrads low-rank through `proj` (NULL = exact Wgrads,
 * the proj=None branch), dx = dy + dx1_ffn. dy_c: optional compute-precision
 * copy of dy; dx_c: optional compute-precision copy of dx (next GEMM). */
int mecefo_backward_block_neighbor(mecefo_engine* e, const mecefo_layer_weights* lw,
                                   const mecefo_block_cache* cache, const float* dy, const void* dy_c, float* dx,
                                   void* dx_c, const mecefo_layer_grads* grads, const mecefo_projection* proj,
                                   int64_t tokens, void* ws, size_t ws_bytes, void* stream);

/* model.py:421-437 backward_block_exact (requires a FULL cache). */
int mecefo_backward_block_exact(mecefo_engine* e, const mecefo_layer_weights* lw, const mecefo_block_cache* cache,
                                const float* dy, const void* dy_c, float* dx, void* dx_c,
                                const mecefo_layer_grads* grads, int64_t tokens, void* ws, size_t ws_bytes,
                                void* stream);

/* model.py:207-225 ffn_forward == approx.py:90-96 recompute_ffn. Outputs in
 * compute precision (h2, gate, up, act, down) and fp32 inv_rms2; any output
 * pointer may be NULL except those needed downstream. */
int mecefo_recompute_ffn(mecefo_engine* e, const mecefo_layer_weights* lw, const float* x1, int64_t tokens,
                         void* h2, float* inv_rms2, void* gate, void* up, void* act, float* down, void* ws,
                         size_t ws_bytes, void* stream);

/* approx.py:24-42 lowrank_wgrad(g_y (out,b), x (in,b), v1 (in,r)) ->
 * (out, in) = g_y (x^T v1) v1^T, all operands in compute precision, out fp32
 * (out += alpha * result). */
int mecefo_lowrank_wgrad(mecefo_engine* e, const void* g_y, const void* x, const void* v1, float* out,
                         int64_t n_out, int64_t n_in, int64_t batch, int64_t rank, float alpha, void* ws,
                         size_t ws_bytes, void* stream);

/* model.py:463 embedding gather: x[t] = embedding[tokens[t]]. */
int mecefo_embedding_forward(mecefo_engine* e, const int64_t* tokens, const float* embedding, float* x,
                             int64_t n_tokens, void* stream);

/* model.py:469-471 + 492-509: xf = rmsnorm(x_last) * final_norm; logits =
 * xf unembedding^T; mean CE -> loss[0]; dlogits = (softmax-onehot)/n written
 * in place over `logits` (compute precision, (tokens, vocab)). */
int mecefo_head_forward_loss(mecefo_engine* e, const float* x_last, const float* final_norm, const void* unemb_c,
                             const int64_t* targets, int64_t tokens, void* xf, float* inv_f, void* logits,
                             float* loss, void* ws, size_t ws_bytes, void* stream);

/* model.py:469-471: xf = rmsnorm(x_last) * final_norm; logits = xf unembedding^T. */
int mecefo_head_logits(mecefo_engine* e, const float* x_last, const float* final_norm, const void* unemb_c,
                       int64_t tokens, void* xf, float* inv_f, void* logits, void* stream);

/* model.py:492-509 cross_entropy: loss[0] = mean CE; logits are overwritten
 * in place with dlogits = (softmax - onehot) / tokens. */
int mecefo_cross_entropy(mecefo_engine* e, void* logits, const int64_t* targets, int64_t tokens, float* loss,
                         void* ws, size_t ws_bytes, void* stream);

/* cross_entropy over `tokens / group_rows` stacked microbatches (logical
 * ranks) at once: each group's dlogits are scaled by 1/group_rows and
 * loss[g] is group g's mean, exactly as separate per-rank calls. */
int mecefo_cross_entropy_grouped(mecefo_engine* e, void* logits, const int64_t* targets, int64_t tokens,
                                 int64_t group_rows, float* loss, void* ws, size_t ws_bytes, void* stream);

/* model.py:469-471 + 492-509 for `tokens / group_rows` stacked ranks: final
 * norm + logits GEMM, then the fused softmax-CE pass (dlogits in place,
 * loss[g] = mean loss of group g). */
int mecefo_head_forward_loss_grouped(mecefo_engine* e, const float* x_last, const float* final_norm,
                                     const void* unemb_c, const int64_t* targets, int64_t tokens, int64_t group_rows,
                                     void* xf, float* inv_f, void* logits, float* loss, void* ws, size_t ws_bytes,
                                     void* stream);

/* model.py:476-483 head_backward (+ accumulate into g_final_norm/g_unemb). */
int mecefo_head_backward(mecefo_engine* e, const float* x_last, const float* final_norm, const float* inv_f,
                         const void* xf, const void* dlogits, const void* unemb_c, float* dx, void* dx_c,
                         float* g_final_norm, float* g_unemb, float alpha, int64_t tokens, void* ws, size_t ws_bytes,
                         void* stream);

/* model.py:486-489 embedding_backward: g[tokens[t]] += alpha * dx0[t]. */
int mecefo_embedding_backward(mecefo_engine* e, const int64_t* tokens, const float* dx0, float* g_emb,
                              float alpha, int64_t n_tokens, void* stream);

/* cluster.py:292-322 Eq. (1) helper on a flat fp32 range: out = beta*out + alpha*src. */
int mecefo_scale_accumulate(const float* src, float* out, int64_t n, float alpha, float beta, void* stream);

/* fp32 -> compute-precision copy (weights' operand shadows). */
int mecefo_cast(mecefo_engine* e, const float* src, void* dst, int64_t n, void* stream);

/* Gradient exchange in bf16 (cluster.py:292-322 Eq. (1) on the wire): the
 * pre-weighted fp32 bucket -> bf16 before the all-reduce, and the reduced
 * bf16 bucket -> fp32 for the optimizer. */
int mecefo_cast_bf16(const float* src, void* dst_bf16, int64_t n, void* stream);
int mecefo_widen_bf16(const void* src_bf16, float* dst, int64_t n, void* stream);

/* optim.py:55-57 _check_grad as a device flag: flag[0] |= any(!isfinite(v)). */
int mecefo_nonfinite(const float* v, int64_t n, int32_t* flag, void* stream);

/* optim.py:96-103 apply_step with AdamW (optim.py:75-93) over a flat buffer;
 * skipped parameters are omitted from `segs`. `segs` is a DEVICE array;
 * total_numel = sum of the segments' numel (profiler byte count only).
 * shadow (optional) receives the updated weights in compute precision.
 * _check_grad (optim.py:55-57) is fused into the read of g: a non-finite
 * gradient sets MECEFO_STATUS_NONFINITE_GRAD in the engine's status word. */
int mecefo_adamw_step(mecefo_engine* e, const mecefo_adam_segment* segs, int32_t nseg, int64_t total_numel, float* w,
                      const float* grad, float* m, float* v, void* shadow, float beta1, float beta2, float eps,
                      void* stream);

/* Generic C[M,N] (+)= alpha * A B^T on the engine's GEMM path (used by the
 * projection refresh, linalg.py:97-142). a_kmajor: A(i,k) at a[i*lda+k],
 * else a[k*lda+i]; likewise B(n,k). C fp32 (ldc), beta in {0,1}. */
int mecefo_gemm(mecefo_engine* e, int64_t M, int64_t N, int64_t K, const void* a, int64_t lda, int32_t a_kmajor,
                const void* b, int64_t ldb, int32_t b_kmajor, float* c, int64_t ldc, float alpha, float beta,
                void* stream);

/* FFN intermediates of a lean block kept for its deferred weight gradients
 * (approx.py:125-126 binds the low-rank wgrad inside ffn_backward; running it
 * later for all lean layers at once changes no arithmetic). Caller buffers,
 * compute precision, tokens rows. */
typedef struct mecefo_ffn_saved {
  void* h2;    /* (tokens, hidden): RMSNorm(x1), model.py:213 */
  void* act;   /* (tokens, ffn): silu(gate) * up, model.py:216 */
  void* dcat;  /* (tokens, 2 ffn): [d_gate | d_up], model.py:251-253 */
} mecefo_ffn_saved;

/* approx.py:99-134 backward_block_neighbor WITHOUT the FFN weight gradients:
 * dx, the norm_ffn grad (gr->norm_ffn, gr->alpha_ffn) and the intermediates in
 * `saved`; dy_c (compute precision) must stay alive until
 * mecefo_lowrank_wgrads_batched consumed it. */
int mecefo_backward_block_neighbor_main(mecefo_engine* e, const mecefo_layer_weights* lw,
                                        const mecefo_block_cache* c, const float* dy, const void* dy_c, float* dx,
                                        void* dx_c, const mecefo_layer_grads* gr, const mecefo_ffn_saved* saved,
                                        int64_t tokens, void* workspace, size_t workspace_bytes, void* stream);

/* One lean block's deferred low-rank FFN weight gradients (approx.py:24-42 for
 * gate, up and down; model.py:247, 255-256): grad += alpha * d2^T (inp V1) V1^T. */
typedef struct mecefo_lowrank_job {
  const void* dy_c;               /* (tokens, hidden) compute precision */
  mecefo_ffn_saved saved;
  const mecefo_projection* proj;
  float* grad_gu;                 /* (2 ffn, hidden) fp32 [gate; up] grads, accumulated */
  float* grad_down;               /* (hidden, ffn) fp32, accumulated */
  float alpha;                    /* Eq. (1) weight of the FFN kinds */
} mecefo_lowrank_job;

/* All jobs (HOST array) in as few launches as possible: bf16 with a rank_pad
 * multiple of 128 runs each product of up to 8 blocks as ONE grouped tcgen05
 * launch; otherwise one chain per job. */
size_t mecefo_lowrank_batched_workspace_bytes(const mecefo_engine* e, int64_t tokens, int32_t rank_pad,
                                             int32_t count);
int mecefo_lowrank_wgrads_batched(mecefo_engine* e, const mecefo_lowrank_job* jobs, int32_t count, int64_t tokens,
                                  void* workspace, size_t workspace_bytes, void* stream);

/* One matrix of a batched projection refresh (approx.py:66-87 refreshes
 * every (layer, kind) basis of a rank at once; each is linalg.py:97-142). */
typedef struct mecefo_subspace_job {
  const float* w;  /* rows x cols fp32, row stride ldw */
  int64_t rows, cols, ldw;
  int32_t k;       /* block width r + oversample (linalg.py:115), r <= k <= cols */
  int32_t r;       /* basis rank */
  float* v;        /* cols x k (ld k) scratch: in = orthonormal start block
                      (linalg.py:117), out = the iterated orthonormal block */
  float* v1;       /* cols x r (ld r) out: Ritz vectors of the r largest Ritz
                      values, descending (linalg.py:124-131) */
  float* theta;    /* r out (optional, may be NULL): those Ritz values */
} mecefo_subspace_job;

/* Block power iteration + Rayleigh-Ritz for `count` matrices at once
 * (linalg.py:119-131 with QR as CholeskyQR: fp32 GEMMs; fp64 k x k Cholesky
 * and Jacobi eigensolve on the device; no host round trip). `jobs` is a HOST
 * array. Fixed `iterations` (the budgeted refresh; costmodel.py:41 charges
 * 30). k <= 512. */
size_t mecefo_subspace_workspace_bytes(const mecefo_subspace_job* jobs, int32_t count);
int mecefo_subspace_iteration_batched(mecefo_engine* e, const mecefo_subspace_job* jobs, int32_t count,
                                      int32_t iterations, void* workspace, size_t workspace_bytes, void* stream);

/* One matrix of a CONVERGED projection refresh (linalg.py:97-142): the
 * orthonormal top-r right singular basis of W, returned once every kept Ritz
 * pair satisfies ||W^T W v - theta v|| <= tol * theta_max (linalg.py:131-135),
 * in float64. Host array of jobs; device pointers inside. */
typedef struct mecefo_refresh_job {
  const float* w;     /* rows x cols fp32, row stride ldw */
  int64_t rows, cols, ldw;
  int32_t r;          /* basis rank, 1 <= r <= cols (approx.py:79: min(r, in)) */
  int32_t k;          /* block width r + oversample, r <= k <= min(cols, 1024) */
  const double* v0;   /* cols x k (ld k) orthonormal start block: QR of the
                         seeded Gaussian (linalg.py:117) */
  float* v1;          /* out: cols x r (ld r) basis, fp32 */
  double* v1_f64;     /* optional out: the same in fp64 */
  double* theta;      /* optional out: the r Ritz values (sigma^2), descending */
  double residual;    /* out (host): final relative residual */
  int32_t products;   /* out (host): block products with W^T W (or W W^T) spent */
  int32_t converged;  /* out (host): 1 if residual <= tol */
  int32_t rr_steps;   /* out (host): Rayleigh-Ritz steps */
  int32_t jacobi_sweeps; /* out (host): Jacobi sweeps over all Ritz solves */
} mecefo_refresh_job;

/* Chebyshev-filtered block subspace iteration with Rayleigh-Ritz, all
 * matrices of a refresh batched per phase (fp64 DMMA GEMMs, CholeskyQR2,
 * Jacobi Ritz solve), wide matrices iterated on W W^T and checked on W^T W.
 * At most max_products block products per matrix (the reference's
 * max_iterations budget, one product per iteration there). Synchronises the
 * stream once per outer iteration. MECEFO_ERR_SVD_NOCONV (SvdConvergenceError)
 * if any job misses tol; each job's residual/products are filled in either way. */
size_t mecefo_refresh_workspace_bytes(const mecefo_refresh_job* jobs, int32_t count);
int mecefo_refresh_converged(mecefo_engine* e, mecefo_refresh_job* jobs, int32_t count, double tol,
                             int32_t max_products, void* workspace, size_t workspace_bytes, void* stream);

/* Number of kernels this library has launched (evidence counter). */
int64_t mecefo_launch_count(void);

/* Launch profiler (CUDA events around every kernel group, tagged with its
 * algorithmic FLOPs and HBM bytes). enable(1) clears and starts recording,
 * enable(0) stops; record(i) synchronizes on record i's end event. */
int mecefo_profile_enable(int32_t on);
int64_t mecefo_profile_count(void);
int mecefo_profile_record(int64_t i, const char** tag, float* ms, double* flops, double* bytes);

#ifdef __cplusplus
}
#endif

#endif /* MECEFO_H */
