/*
 * fixedfanin.h — C ABI of the B200-native fixed fan-in (uniform sparsity) sparse
 * output layer of arXiv 2306.03725 ("Towards Memory-Efficient Training for
 * Extremely Large Output Spaces", §3.2 "uniform sparsity").
 *
 * Citations: P:n = line n of the paper's LaTeX source (reference PAPER.md);
 * S:n = line n of the reference SPEC.md; readings R1..R23 are listed in DESIGN.md.
 *
 * Notation: L_global labels; this handle owns the contiguous
 * label rows [row_begin, row_begin + L_local) ("label shard"); every label has
 * exactly k connections ("fan-in", the paper's s) into a layer of width m
 * (the paper's feature/intermediate dimension); B = mini-batch.
 *
 * Layouts (all row-major, C order):
 *   W   float   [L_local][k]   weights        (the paper's `weights`  s x L, transposed; R2)
 *   idx int32_t [L_local][k]   source columns (the paper's `indices`  s x L, transposed; R2)
 *   bias, mb, vb float [L_local];  mW, vW float [L_local][k]  (Adam moments)
 *   h   float [B][m]  input of the sparse layer (`features`)
 *   y   float [B][L_local]   scores (`output`)
 *   dh  float [B][m]  gradient w.r.t. h (Alg. 2), THIS SHARD's partial sum
 *   labels: CSR over the batch — lbl_ptr int32 [B+1], lbl_ids int32 [lbl_ptr[B]] GLOBAL
 *           label ids of the positives of each instance (y in {0,1}^L stored sparse,
 *           P:92-97).  Ids outside this shard's rows are ignored (that is what makes
 *           label sharding transparent); ids outside [0, L_global) -> FF_ERR_RANGE
 *           (reported asynchronously, see fixedfanin_check).
 *
 * Memory ownership: the caller owns every buffer, including the workspace (one
 * device allocation of fixedfanin_workspace_size() bytes that holds all layer state
 * and scratch).  The library never allocates or frees device memory.
 * Pointers are DEVICE pointers unless the name ends in _host.
 * Asynchrony: every call enqueues its work on `stream` and returns without
 * synchronizing, except get_params/set_params/check (documented below).  Host-side
 * argument validation is synchronous and returns an error code before any work is
 * enqueued.  Not thread-safe per handle; distinct handles are independent.
 * Errors: status codes only (no exceptions cross the ABI); fixedfanin_last_error()
 * returns a thread-local message for the last non-OK status.
 */
#ifndef FIXEDFANIN_H
#define FIXEDFANIN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* ff_stream_t;   /* == cudaStream_t; NULL = legacy default stream */
typedef struct ff_layer ff_layer;

typedef enum {
    FF_OK = 0,
    FF_ERR_ARG = 1,        /* null pointer, bad shape, B > max_batch, K > max_topk, K > L_global   */
    FF_ERR_CONFIG = 2,     /* invalid ff_config (k > m, k > FF_MAX_FANIN, prune count < 1 or
                              m - k < prune count when redistribution is requested, ...)          */
    FF_ERR_RANGE = 3,      /* idx outside [0,m) or duplicate idx in a row (set_params);
                              label id outside [0, L_global) (reported by fixedfanin_check)       */
    FF_ERR_NONFINITE = 4,  /* non-finite score/gradient seen with FF_FLAG_CHECK_FINITE           */
    FF_ERR_CUDA = 5,       /* a CUDA runtime error (launch failure, async fault)                 */
    FF_ERR_STATE = 6       /* call order violated (adam_step without a preceding backward, ...)  */
} ff_status;

/* Compile-time limits of this build (checked at create). */
#define FF_MAX_FANIN 64     /* k <= 64 (the paper's largest, 64 nnz/label): a label
                               row is one or two warp-wide 128-B lines per array               */
#define FF_MAX_BATCH 1024   /* B <= 1024: processed as ceil(B/32) 32-sample lane groups       */
#define FF_MAX_TOPK 8       /* K <= 8 (the paper reports P@1/3/5)                  */

/* ff_config.flags */
#define FF_FLAG_CHECK_FINITE 1u  /* raise FF_ERR_NONFINITE on a non-finite score/gradient     */
#define FF_FLAG_STORE_GRADS 2u   /* fused train_step also stores dW/db (for get_grads/tests)  */
#define FF_FLAG_NO_PIPE 4u       /* use the generic fused kernel even where the pipelined one
                                    applies (k = 32, B <= 32); same results, for A/B tests     */
#define FF_STEP_AUTO UINT64_MAX  /* dense forward / model step `step`: key the dropout on the dense
                                  layer's device Adam counter + 1 (CUDA-graph capturable)      */
#define FF_FLAG_DENSE_SIMT 8u    /* ff_dense_config.flags: FP32 FMA forward instead of the
                                    tcgen05 3xTF32 tensor-core forward (B <= 32), for A/B tests */

/* ff_config.loss: the one-vs-all binary loss whose gradient the backward pass consumes */
#define FF_LOSS_BCE 0            /* binary cross-entropy with logits (the north star's) */
#define FF_LOSS_SQH 1            /* squared hinge max(0, 1 - y yhat)^2, y = +-1, whose
                                    exact zeros are skipped (implicit negative mining, §3.3)     */

/* ff_config.dh_mode */
#define FF_DH_ATOMIC 0           /* dh by coalesced red.global.add (Alg. 2 with atomics) */
#define FF_DH_CSC 1              /* dh by a transposed (CSC) index gather, rebuilt after redistribution;
                                    deterministic, and the faster BCE mode on B200       */
#define FF_DH_HYBRID 2           /* columns c < hybrid_frac*m by red (the L1->L2 write path), the rest by
                                    the CSC gather (the read path): both paths busy at once */

typedef struct {
    int64_t L_global;    /* total labels, 1 <= L_global < 2^31 (32-bit label ids)   */
    int64_t row_begin;   /* first global label row owned by this handle                         */
    int64_t L_local;     /* rows owned, 0 <= L_local, row_begin + L_local <= L_global,          */
                         /* L_local * k < 2^31 (32-bit connection offsets; else FF_ERR_CONFIG)  */
    int32_t m;           /* width of h, 1 <= m < 2^31                                           */
    int32_t k;           /* connections per label, 1 <= k <= min(m, FF_MAX_FANIN)               */
    int32_t max_batch;   /* largest B that will be passed, 1..FF_MAX_BATCH                      */
    int32_t max_topk;    /* largest K that will be passed to predict_topk, 1..FF_MAX_TOPK       */
    int32_t max_nnz;     /* largest lbl_ptr[B] for the *_host entry points (0 -> 64*max_batch)  */
    int32_t dh_mode;     /* FF_DH_ATOMIC (0, the default; best for FF_LOSS_SQH), FF_DH_CSC or     */
                         /* FF_DH_HYBRID                                                         */
    uint64_t seed;       /* Philox key for init and redistribution (R13)                        */
    float init_scale;    /* W init U(-a, a); 0 -> a = fp32(1/sqrt(k)) (R17)                     */
    float beta1, beta2, eps;   /* Adam; 0 -> 0.9 / 0.999 / 1e-8 (R6)                            */
    float prune_frac;    /* SET fraction alpha, p = floor(alpha*k) per row; 0 -> 0.1    */
    uint32_t flags;      /* FF_FLAG_*                                                           */
    int32_t loss;        /* FF_LOSS_BCE (default) or FF_LOSS_SQH                                */
    float hybrid_frac;   /* FF_DH_HYBRID: fraction of the columns reduced by red; 0 -> 0.5        */
} ff_config;

/* Bytes of device workspace the layer needs for `cfg` (host-only, no CUDA calls). */
ff_status fixedfanin_workspace_size(const ff_config* cfg, size_t* bytes_host);

/* Carve `workspace` (device, >= workspace_size bytes, 256-B aligned) and initialize the
 * layer on `stream`: idx rows = k distinct uniform draws from [0,m) and W ~ U(-a,a) from
 * the Philox streams keyed (seed, global row) (R13, R17); bias, moments = 0;
 * t = 0.  *out_host receives the handle (host memory, freed by destroy).               */
ff_status fixedfanin_create(const ff_config* cfg, void* workspace, size_t bytes,
                            ff_stream_t stream, ff_layer** out_host);

/* Free the host handle.  Does not touch the workspace (the caller owns it). */
ff_status fixedfanin_destroy(ff_layer* layer);

/* Overwrite the state from device arrays (any pointer may be NULL = keep).  Synchronizes
 * `stream`, validates idx (range, no duplicates within a row) -> FF_ERR_RANGE (state is
 * left modified but invalid in that case).  t_host: new Adam step count (NULL = keep). */
ff_status fixedfanin_set_params(ff_layer* layer, const float* W, const int32_t* idx,
                                const float* bias, const float* mW, const float* vW,
                                const float* mb, const float* vb, const int64_t* t_host,
                                ff_stream_t stream);

/* Copy the state into device arrays (any pointer may be NULL = skip); *t_host = Adam t
 * (read back from the device counter).  Synchronizes `stream`.                          */
ff_status fixedfanin_get_params(ff_layer* layer, float* W, int32_t* idx, float* bias,
                                float* mW, float* vW, float* mb, float* vb, int64_t* t_host,
                                ff_stream_t stream);

/* Alg. 1 + bias: y[b][j] = bias[j] + sum_i W[j][i] * h[b][idx[j][i]],
 * for b < B, j < L_local.  0 <= B <= max_batch (B = 0 is a no-op).                   */
ff_status fixedfanin_forward(ff_layer* layer, const float* h, int32_t B, float* y,
                             ff_stream_t stream);

/* Loss gradient — BCE g = grad_scale*(sigmoid(y) - t) (R4, R5), or with
 * FF_LOSS_SQH g = grad_scale*(-2 t' max(0, 1 - t' y)), t' = +-1 — then
 * Alg. 3 dW[j][i] = sum_b g[b][j] h[b][idx[j][i]], db[j] = sum_b g[b][j]
 * (kept in the workspace for adam_step/get_grads), and Alg. 2
 * dh[b][c] = sum_{(j,i): idx[j][i]=c} W[j][i] g[b][j] (overwritten).  `y` must be the
 * scores of the same h (e.g. from fixedfanin_forward).  loss (device float[1] or NULL)
 * = grad_scale * sum_{b,j} softplus(y) - t*y  (BCE)  or  max(0, 1 - t' y)^2  (SQH).
 * Exact-zero gradients (SQH) are skipped: no dh reductions / CSC gathers for them
 * (the paper's Alg. 2 early exit); results equal the unskipped sums.       */
ff_status fixedfanin_backward(ff_layer* layer, const float* h, const float* y, int32_t B,
                              const int32_t* lbl_ptr, const int32_t* lbl_ids,
                              float grad_scale, float* dh, float* loss, ff_stream_t stream);

/* Copy the gradients of the last backward (or train_step with FF_FLAG_STORE_GRADS). */
ff_status fixedfanin_get_grads(ff_layer* layer, float* dW, float* db, ff_stream_t stream);

/* t += 1; Adam (R6, R7) over W (with dW) and bias (with db). FF_ERR_STATE if
 * no backward ran since the last adam_step.                                          */
ff_status fixedfanin_adam_step(ff_layer* layer, float lr, ff_stream_t stream);

/* The fused training step: forward, BCE gradient, dW, db, dh (pre-update W) and Adam
 * (t += 1) in one pass over the label rows; y, g, dW are never written to HBM.
 * dh (device [B][m]) overwritten; loss as in backward (NULL = skip).
 * CUDA-graph capturable: it only enqueues kernels on `stream` (no host synchronisation),
 * and the Adam step counter t and its bias corrections live on the device (advanced by the
 * step's first kernel), so replays of a captured step take consecutive t.  A captured
 * step reads h / labels from the captured addresses (copy new batches into them).      */
ff_status fixedfanin_train_step(ff_layer* layer, const float* h, int32_t B,
                                const int32_t* lbl_ptr, const int32_t* lbl_ids,
                                float grad_scale, float lr, float* dh, float* loss,
                                ff_stream_t stream);

/* Same as train_step with HOST inputs/outputs (end-to-end path): copies h_host [B][m]
 * and the label CSR (host) into one of two workspace staging slots on a library-owned copy
 * stream (so that, with pinned memory, the next call's copy overlaps this call's kernels;
 * `stream` waits for the copy with an event), runs the fused step on `stream`, then returns
 * the loss (if loss_host != NULL) and dh (if dh_host != NULL) on `stream`.  A page-locked
 * loss_host is written by a one-thread kernel store (mapped memory, no copy-engine
 * operation); a pageable one by cudaMemcpyAsync.  dh_host == NULL skips the [B][m] copy-out
 * of dh (it is still computed).  The host inputs must stay
 * unmodified, and the host outputs are valid, once `stream` is synchronized.
 * lbl_ptr_host[B] <= max_nnz (read on the host for the copy size).                      */
ff_status fixedfanin_train_step_host(ff_layer* layer, const float* h_host, int32_t B,
                                     const int32_t* lbl_ptr_host, const int32_t* lbl_ids_host,
                                     float grad_scale, float lr, float* dh_host,
                                     float* loss_host, ff_stream_t stream);

/* SET prune/regrow, per row (R8): the p = floor(prune_frac*k)
 * slots of smallest (|W|, slot) are replaced by p distinct indices drawn uniformly from
 * [0,m) minus the row's current set, from the Philox stream keyed (seed, step, global
 * row) (R10-R13); W = mW = vW = 0 in those slots (R11).  The CSC index (dh_mode 1) is
 * rebuilt.  FF_ERR_CONFIG if p < 1 or m - k < p.                                       */
ff_status fixedfanin_redistribute(ff_layer* layer, uint64_t step, ff_stream_t stream);

/* Top-K prediction: per instance the K labels of this shard with the largest
 * scores, ordered by (score desc, global id asc) (R15).  scores [B][K] float,
 * ids [B][K] int32 GLOBAL ids.  1 <= K <= min(max_topk, L_local).  A NaN score never
 * enters the top K; with FF_FLAG_CHECK_FINITE a non-finite score raises FF_ERR_NONFINITE
 * at the next fixedfanin_check.                                                         */
ff_status fixedfanin_predict_topk(ff_layer* layer, const float* h, int32_t B, int32_t K,
                                  float* scores, int32_t* ids, ff_stream_t stream);

/* Shortlist scoring (restricting scoring to a label shortlist is "a trivial
 * matrix slicing operation"): for every candidate entry p of instance b,
 * cand_ptr[b] <= p < cand_ptr[b+1] (CSR, int32, device),
 *   scores[p] = y[b, cand_ids[p]] = bias_j + sum_i W[j][i] * h[b][idx[j][i]]  (Alg. 1)
 * bit-identical to the score the forward / predict_topk compute for the same (b, j).
 * h float [B][m] row-major (device).  cand_ids are GLOBAL label ids; entries whose label
 * is not in this shard's rows are written as +0 (so the shards' outputs sum to the full
 * result); ids outside [0, L_global) are written as NaN and reported as FF_ERR_RANGE by
 * fixedfanin_check.  B >= 0 (no max_batch limit: no workspace is used).  cand_ids and
 * scores may be NULL when the list is empty (cand_ptr[B] == 0).                        */
ff_status fixedfanin_score_shortlist(ff_layer* layer, const float* h, int32_t B,
                                     const int32_t* cand_ptr, const int32_t* cand_ids,
                                     float* scores, ff_stream_t stream);

/* Precision at K, Eq. (1): for each instance b the number of its predicted
 * labels ids[b][0..K) (e.g. from predict_topk / merge_topk; GLOBAL ids) that are positives
 * in the label CSR (lbl_ptr [B+1], lbl_ids, device), hits [B] int32 (or NULL), and
 * mean = (1/B) sum_b hits[b] / K (float[1], or NULL), dividing by K even when an instance
 * has fewer than K positives (R16).  The mean is summed in a fixed order (deterministic).
 * Stateless; 1 <= K <= 32, B >= 0 (B = 0 gives mean 0).                                   */
ff_status fixedfanin_precision_at_k(const int32_t* ids, int32_t B, int32_t K, const int32_t* lbl_ptr,
                                    const int32_t* lbl_ids, int32_t* hits, float* mean,
                                    ff_stream_t stream);

/* Merge per-shard top-K lists: in_scores/in_ids [P][B][K] (device) -> out [B][K] under
 * the same total order.  Stateless.  1 <= K <= FF_MAX_TOPK, 1 <= P <= 1024.            */
ff_status fixedfanin_merge_topk(const float* in_scores, const int32_t* in_ids, int32_t P,
                                int32_t B, int32_t K, float* out_scores, int32_t* out_ids,
                                ff_stream_t stream);

/* ======================================================================================
 * NEXT-2: the intermediate layer of the proposed architecture (Fig. 2,
 * P:1013-1022): fixed features x -> input dropout -> dense W_d
 * -> ReLU (R18) -> the fixed fan-in layer.  Readings R25-R28.
 * Layouts: x float [B][d] (d = feature dimension: 512 Slice / 768 Cascade),
 *          Wd float [d][m] (input-feature major), bd float [m], h and dh float [B][m].
 * One ff_dense handle = the dense layer or one column shard of it (col_begin, m_global):
 * under label sharding rank r owns the columns [m_global r / P, m_global (r+1) / P) of Wd,
 * bd and their Adam state; h is all-gathered and dh reduce-scattered.
 * Same conventions as above: caller-owned workspace, async on `stream`, status codes.
 * ====================================================================================== */
typedef struct ff_dense ff_dense;

typedef struct {
    int32_t d;           /* input feature dimension, >= 1                                       */
    int32_t m;           /* output columns of this handle, >= 1 (the fixed fan-in layer's m,   */
                         /* or a column shard of it: see col_begin / m_global)                  */
    int32_t max_batch;   /* largest B, 1..FF_MAX_BATCH                                          */
    int32_t col_begin;   /* column shard: this handle owns the global columns  */
                         /* [col_begin, col_begin + m) of Wd, bd; 0 for the whole layer          */
    uint64_t seed;       /* Philox key: Wd init (domain 4, R27) and dropout masks (domain 3, R25) */
    float init_scale;    /* Wd ~ U(-a, a); 0 -> a = fp32(sqrt(6 / (d + m))) (Glorot uniform, R27) */
    float dropout;       /* input dropout rate p in [0, 1) (0.1 Amazon-670K)         */
    float beta1, beta2, eps;   /* Adam; 0 -> 0.9 / 0.999 / 1e-8 (R6)                            */
    uint32_t flags;      /* FF_FLAG_STORE_GRADS: keep dWd/dbd for fixedfanin_dense_get_grads    */
    int32_t m_global;    /* width of the whole layer (0 -> m); col_begin + m <= m_global.  The   */
                         /* init draws global column c's word and the Glorot scale uses m_global,*/
                         /* so the column shards of a layer concatenate to the unsharded layer  */
} ff_dense_config;

/* Bytes of device workspace for `cfg` (host-only).  FF_ERR_CONFIG on a bad config.       */
ff_status fixedfanin_dense_workspace_size(const ff_dense_config* cfg, size_t* bytes_host);

/* Carve `workspace` (>= workspace_size bytes, 256-B aligned) and initialize on `stream`:
 * Wd[f][c] = a * (2 * ((u >> 8) * 2^-24) - 1) in fp32, u = word g of the Philox stream
 * (ctr = (g/4, f, 0, 4), key = seed), g = col_begin + c the global column (R27); bd =
 * moments = 0; t = 0.                                                                    */
ff_status fixedfanin_dense_create(const ff_dense_config* cfg, void* workspace, size_t bytes,
                                  ff_stream_t stream, ff_dense** out_host);
ff_status fixedfanin_dense_destroy(ff_dense* dense);

/* Overwrite / read the state (any pointer NULL = keep / skip); both synchronize `stream`.
 * Wd, mWd, vWd [d][m]; bd, mbd, vbd [m]; t_host = the dense layer's Adam step count.     */
ff_status fixedfanin_dense_set_params(ff_dense* dense, const float* Wd, const float* bd,
                                      const float* mWd, const float* vWd, const float* mbd,
                                      const float* vbd, const int64_t* t_host, ff_stream_t stream);
ff_status fixedfanin_dense_get_params(ff_dense* dense, float* Wd, float* bd, float* mWd,
                                      float* vWd, float* mbd, float* vbd, int64_t* t_host,
                                      ff_stream_t stream);

/* Forward: xt = dropout(x) if train (R25: sample b, feature f is kept iff
 * (u >> 8) * 2^-24 >= p for u = word f of the Philox stream (ctr = (f/4, b, step, 3),
 * key = seed), kept values scaled by fp32(1/(1-p))), else xt = x;
 * z[b][c] = bd[c] + sum_f xt[b][f] Wd[f][c] (f ascending); h = max(z, 0).  Writes h
 * [B][m] if h != NULL and keeps xt and h for the backward.  0 <= B <= max_batch.
 * step == FF_STEP_AUTO: the key is the dense layer's device Adam counter + 1 (the step the
 * following backward_adam takes), read on the device.                                    */
ff_status fixedfanin_dense_forward(ff_dense* dense, const float* x, int32_t B, uint64_t step,
                                   int32_t train, float* h, ff_stream_t stream);

/* Backward + Adam of the last training forward (same B): dz = dh * [z > 0] (R26),
 * dWd[f][c] = sum_b xt[b][f] dz[b][c], dbd[c] = sum_b dz[b][c], then t += 1 and Adam
 * (R6, R28: the dense layer's own t) over Wd and bd.  dh float [B][m] — under
 * label sharding, the all-reduced sum of the shards' dh.  FF_ERR_STATE without a
 * preceding training forward.                                                            */
ff_status fixedfanin_dense_backward_adam(ff_dense* dense, const float* dh, int32_t B, float lr,
                                         ff_stream_t stream);

/* dWd [d][m], dbd [m] of the last backward (needs FF_FLAG_STORE_GRADS, else FF_ERR_STATE). */
ff_status fixedfanin_dense_get_grads(ff_dense* dense, float* dWd, float* dbd, ff_stream_t stream);

/* One training step of the whole architecture on one GPU (unsharded `layer`, same m):
 * dense forward with dropout (step keys the masks) -> the fixed fan-in layer's fused
 * train_step -> dense backward + Adam.  h and dh never leave the layer's internal
 * h|dh column lines (no [B][m] round trip).  loss as in fixedfanin_train_step.
 * With step == FF_STEP_AUTO the step is CUDA-graph capturable: both layers' Adam counters
 * and the dropout key live on the device (the layer's k_prep advances both counters).    */
ff_status fixedfanin_model_train_step(ff_dense* dense, ff_layer* layer, const float* x, int32_t B,
                                      uint64_t step, const int32_t* lbl_ptr,
                                      const int32_t* lbl_ids, float grad_scale, float lr,
                                      float* loss, ff_stream_t stream);

/* Inference of the architecture: dense forward without dropout, then predict_topk.       */
ff_status fixedfanin_model_predict_topk(ff_dense* dense, ff_layer* layer, const float* x,
                                        int32_t B, int32_t K, float* scores, int32_t* ids,
                                        ff_stream_t stream);

/* Synchronize `stream` and report asynchronous errors raised by earlier calls
 * (FF_ERR_RANGE for bad label ids, FF_ERR_NONFINITE, FF_ERR_CUDA); clears them.       */
ff_status fixedfanin_check(ff_layer* layer, ff_stream_t stream);

/* Kernel timing for benchmarks: between profile_begin and profile_end every train_step
 * (and train_step_host, backward) records a CUDA event pair around each launch of its
 * fused row kernel on the call's stream (one launch per step, or one per label tile in
 * FF_DH_CSC mode; at most max_launches pairs).  profile_end synchronizes on the last event
 * and returns the summed kernel milliseconds and the number of timed launches.        */
ff_status fixedfanin_profile_begin(ff_layer* layer, int32_t max_launches);
ff_status fixedfanin_profile_end(ff_layer* layer, double* kernel_ms_host, int32_t* launches_host);
/* paused != 0: launches are not timed until resumed (host flag, no synchronisation), so a
 * benchmark can time a sample of its steps and keep event recording out of the others.   */
ff_status fixedfanin_profile_pause(ff_layer* layer, int32_t paused);

/* Number of kernel launches the last API call enqueued (host counter, for benchmarks). */
int32_t fixedfanin_last_launch_count(void);

/* Thread-local message of the last non-OK status ("" if none). */
const char* fixedfanin_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* FIXEDFANIN_H */
