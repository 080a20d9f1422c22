/*
 * fedsim_b200 C-ABI — the drop-in boundary of the FL round loop.
 *
 * The reference's plugin API for this path is the backend module selected
 * in pkg/src/fedsim/backends/__init__.py:1-63 (NAME, forward,
 * loss_and_grad, sign_align_count) plus the round-level callers that loop
 * over it: client.train_local (client.py:98-172), selection
 * calculate_relevance/filter_update (selection.py:53-85) and
 * server.aggregate (server.py:72-86), evaluated per round by
 * FederationEngine._evaluate_global (server.py:321-328).  Each entry point
 * below names the reference interface it replaces.
 *
 * Conventions
 *  - every pointer argument is DEVICE memory unless its name ends in _host;
 *  - every call is stream-ordered and non-blocking on `stream` (a
 *    cudaStream_t passed as void*); no call allocates device memory — the
 *    caller passes workspaces sized by the matching *_workspace_bytes query;
 *  - return 0 on success or a negative FS_E* code; fs_last_error() returns a
 *    thread-local message for the last failure on the calling thread;
 *  - parameter vectors use the reference's flat float64 layout
 *    (numpy_backend.py:3-14): per layer W[fan_in x fan_out] row-major, then b.
 */
#ifndef FEDSIM_B200_H
#define FEDSIM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FS_ABI_VERSION 1
#define FS_MAX_LAYERS 8 /* weight layers, hidden + head */

enum fs_status {
  FS_OK = 0,
  FS_EINVAL = -1,   /* maps to ValueError (layout/length mismatch) */
  FS_ECUDA = -2,    /* CUDA runtime failure */
  FS_ENCCL = -3,    /* collective failure */
  FS_EDIVERGED = -4 /* non-finite loss: TrainingDivergedError, model.py:207-211 */
};

enum fs_mask_mode { FS_MASK_NONE = 0, FS_MASK_BITS = 1, FS_MASK_DENSE = 2 };

enum fs_align_mode { FS_ALIGN_WEIGHT_SIGN = 0, FS_ALIGN_DELTA_SIGN = 1 };

const char* fs_last_error(void);
/* Layout check for bindings: sizes of the ABI structs in this build, in the
 * order fs_train_desc, fs_client_done, fs_async_world, fs_async_yield,
 * fs_async_logview, fs_async_device. Writes min(n, 6) entries, returns 6.  */
int32_t fs_struct_sizes(size_t* out, int32_t n);
int fs_abi_version(void);
/* dst[0..n) = value (device, stream-ordered): per-request launch arguments
 * that are one value for a whole round (start model pointer, step size bits) */
int fs_fill_u64(uint64_t* dst, uint64_t value, int64_t n, void* stream);
/* flag[0] = value after all work queued before it on `stream` (release store):
 * publishes a chunk of an upload to kernels polling on other streams     */
int fs_publish_flag(int32_t* flag, int32_t value, void* stream);
/* chunked host -> device upload of two row-aligned arrays (page-locked host
 * memory): for chunk c = rows [bounds[2c], bounds[2c+1]) the rows of a
 * (a_row_bytes each) and of b (b_row_bytes each) are copied, then
 * flags[c] = tag is published as by fs_publish_flag; one call per upload
 * instead of three per chunk (the re-upload of DeviceWorld.refill)        */
int fs_upload_chunks(void* dst_a, const void* src_a, int64_t a_row_bytes, void* dst_b, const void* src_b,
                     int64_t b_row_bytes, const int64_t* bounds, int32_t n_chunks, int32_t* flags, int32_t tag,
                     void* stream);
/* stream-ordered device-to-device copy (engine-owned model versions -> caller tensors) */
int fs_memcpy_d2d(void* dst, const void* src, size_t bytes, void* stream);

/* ---------------------------------------------------------------- K1 seeds
 * derive_seed(master, *path) with integer label words (rng.py:42-44).
 * Host-side helper used by tests and the host control plane.            */
int fs_derive_seed_host(uint64_t master, const uint32_t* path_host, int32_t n_path,
                        uint64_t* out_host);

/* Host-side batch of train seeds (all pointers host memory).            */
int fs_train_seeds_host(uint64_t master, const int32_t* client_ids_host, const int32_t* cycles_host,
                        int32_t n, uint64_t* seeds_out_host);

/* seeds[i] = derive_seed(master, "train", client_ids[i], cycles[i])
 * (server.py:207).                                                       */
int fs_train_seeds(uint64_t master, const int32_t* client_ids, const int32_t* cycles, int32_t n,
                   uint64_t* seeds_out, void* stream);

/* ---------------------------------------------------------------- K2 shuffles
 * perm_out[perm_off[r] + e*n_rows[r] + i] =
 *   derive_rng(seeds[r], "shuffle", e).permutation(n_rows[r])[i]
 * for e in [0, epochs)  (client.py:136).                                  */
int fs_shuffle_perms(const uint64_t* seeds, const int32_t* n_rows, const int64_t* perm_off,
                     int32_t n_req, int32_t epochs, int32_t max_rows, int32_t* perm_out,
                     void* stream);

/* ---------------------------------------------------------------- K3 masks
 * Dropout keep-bits of every (request, epoch, step) of a training batch
 * (model.py:153-166 with the seed of client.py:150). Step (e, s) of request
 * r occupies ceil(batch[r]*sum_hidden/32) words at
 *   mask_off[r] + (e*steps_per_epoch_r + s) * slot_words_r;
 * bit j of a slot is draw j of the step's stream (layer-major, then row,
 * then unit): keep iff random() < keep.                                   */
int fs_dropout_bits(const uint64_t* seeds, const int32_t* n_rows, const int32_t* batch,
                    const int64_t* mask_off, int32_t n_req, int32_t epochs, int32_t sum_hidden,
                    double keep, uint32_t* bits_out, void* stream);

/* Keep-bits of one stream: default_rng(SeedSequence(mask_seed)) drawing
 * n_draws doubles (model.dropout_masks).                                  */
/* K3 overlapped with its own round's trainer: one CTA per (request, step),
 * step-major in `order`, each step published by a release store of `tag`
 * (non-zero, fresh per launch) into flags[r * max_steps + step].         */
int fs_dropout_bits_flagged(const uint64_t* seeds, const int32_t* n_rows, const int32_t* batch,
                            const int64_t* mask_off, const int32_t* order, int32_t n_req, int32_t epochs,
                            int32_t max_steps, int32_t sum_hidden, double keep, uint32_t* bits_out, int32_t* flags,
                            int32_t tag, void* stream);
int fs_dropout_bits_seed(uint64_t mask_seed, int64_t n_draws, double keep, uint32_t* bits_out,
                         void* stream);

/* ---------------------------------------------------------------- K5 trainer
 * Batched local SGD (client.train_local, client.py:98-172): request r trains
 * from w_start[r] over steps [start_step[r], end_step[r]) of its shard and
 * leaves its parameters in w_out + r*ldw.                                  */
typedef struct fs_train_desc {
  int32_t n_dims;
  int32_t dims[FS_MAX_LAYERS + 1];
  int32_t n_req;
  int32_t epochs;
  int32_t max_batch;           /* max over requests of batch[r]                 */
  int32_t mask_mode;           /* FS_MASK_NONE or FS_MASK_BITS                  */
  double scale;                /* 1/(1-p): value of a kept unit                 */
  const double* features;      /* [rows x dims[0]] packed shards                */
  const double* labels;        /* [rows] 0.0 / 1.0                              */
  const int64_t* row_off;      /* [n_req] first shard row                       */
  const int32_t* n_rows;       /* [n_req]                                       */
  const int32_t* batch;        /* [n_req]                                       */
  const double* lr;            /* [n_req x epochs] step size of each epoch      */
  const uint64_t* w_start;     /* [n_req] device pointers (const double*)       */
  double* w_out;               /* [n_req x ldw]                                 */
  int64_t ldw;
  const int32_t* perm;         /* K2 output                                     */
  const int64_t* perm_off;
  const uint32_t* mask_bits;   /* K3 output (FS_MASK_BITS)                      */
  const int64_t* mask_off;
  const int32_t* start_step;   /* [n_req]                                       */
  const int32_t* end_step;     /* [n_req]                                       */
  const int32_t* order;        /* [n_req] processing order (longest first)      */
  int32_t* status;             /* [n_req] out: 1 = non-finite logit (diverged)  */
  void* workspace;
  size_t workspace_bytes;
  int32_t grid;                /* CTAs; 0 = auto                                */
  /* bf16 unit-major trainer only: keep bits still being produced by
   * fs_dropout_bits_flagged on another stream; step s of request r is read
   * after mask_flags[r * max_steps + s] == mask_tag (NULL: bits complete)  */
  const int32_t* mask_flags;
  int32_t mask_tag;
  int32_t max_steps;
  /* bf16 unit-major trainer only: per-client completion records. When
   * done != NULL, each client's CTA counts the sign alignment of its trained
   * row against (w_start[r], w_prev[r]) (align_mode FS_ALIGN_*, -1 = none)
   * and then publishes {aligned, status, tag = done_tag} to the
   * fs_client_done record at done[r] (typically mapped host memory), so a
   * host can consume clients as they finish instead of the whole launch.  */
  const uint64_t* done;
  const uint64_t* w_prev;
  int32_t align_mode;
  int32_t done_tag;
  /* bf16 unit-major trainer only: the shards are still being uploaded in
   * chunks; request r reads its rows after data_flags[data_chunk[r]] ==
   * data_tag (NULL: resident)                                             */
  const int32_t* data_flags;
  const int32_t* data_chunk;
  int32_t data_tag;
  /* bf16 unit-major trainer only: when align_counts != NULL (and done ==
   * NULL) each client's CTA writes the K6 count of its trained row against
   * (w_start[r], w_prev[r]) under align_mode to align_counts[r] — the sync
   * round's alignment fused into the trainer instead of a second pass over
   * the rows (fs_sign_align_rows)                                          */
  int64_t* align_counts;
  /* bf16 unit-major trainer only: w_start == NULL and w_start_all != NULL
   * starts every request from the one model w_start_all (a sync round);
   * counter_zeroed = 1 promises the workspace's work counter is already 0
   * (prepared ahead on another stream), so no memset precedes the launch   */
  const void* w_start_all;
  int32_t counter_zeroed;
  /* opt-in local optimizer (an extension; the reference is plain SGD,
   * model.py:215-221): FS_OPT_SGD, or FS_OPT_ADAM with moments m, v in
   * opt_state [n_req x 2 x ldw] of the parameter dtype (m at r*2*ldw, v at
   * r*2*ldw + ldw), zeroed at each request's start; step t = global step + 1,
   * p -= lr * m_hat / (sqrt(v_hat) + eps). fp64 trainer and the wide bf16
   * trainer (fs_train_bf16 routes Adam requests there).                     */
  int32_t optimizer;
  double adam_beta1, adam_beta2, adam_eps;
  void* opt_state;
  /* max over requests of n_rows[r], or 0 (unknown). The wide bf16 trainer
   * sizes its factored (low-rank history) mode from it: with SGD and
   * epochs * max_rows history rows well under the layer width, a client's
   * weights are kept as its start model plus its own step rows, and the
   * trained row is written once (fs_train_wide.cu). 0 = dense lockstep.   */
  int32_t max_rows;
} fs_train_desc;

#define FS_OPT_SGD 0
#define FS_OPT_ADAM 1

typedef struct {
  int64_t aligned;
  int32_t status;
  volatile int32_t tag;
} fs_client_done;

size_t fs_train_workspace_bytes(const fs_train_desc* desc);
int fs_train_f64(const fs_train_desc* desc, void* stream);

/* bf16 mixed-precision trainer (tcgen05/TMEM): same descriptor, but
 * w_start[r] points to float32 parameters and w_out is a float32 [n_req x
 * ldw] buffer (fp32 master weights, bf16 GEMM operands, fp32 accumulate).
 * Features/labels come pre-converted by fs_prep_features_bf16 (desc->features
 * and desc->labels are ignored). Hidden widths must be multiples of 32 (<=256),
 * input width <= 64, at most 4 hidden layers.                              */
int fs_bf16_supported(const int32_t* dims, int32_t n_dims);
/* Diagnostic: accumulate per-phase SM cycles of the bf16 trainer into 32
 * device counters (nullptr disables).                                     */
void fs_bf16_set_profile(unsigned long long* counters);
/* Diagnostic: 1 = always run the generic bf16 kernel (optimizer state in
 * HBM) instead of the on-chip-state kernel for 3-hidden-layer MLPs.       */
void fs_bf16_force_generic(int mode); /* 0 auto, 1 generic, 2 row-major V2 */
int fs_prep_features_bf16(const double* x, const double* y, int64_t rows, int32_t d, int32_t dp,
                          void* xb_out, float* y_out, void* stream);
size_t fs_train_bf16_workspace_bytes(const fs_train_desc* desc);
/* K8 forward in bf16 mode (_core.pyx:109-137 with bf16 GEMM operands, fp32
 * accumulation): probs_out[rows] (float64) of fs_prep_features_bf16 rows under
 * fp32 parameters w. Layer shapes of the unit-major trainer only (3 hidden
 * layers, f1 in {128, 256}, f2 = 128, f3 = 64, f0 <= 64); else FS_EINVAL. */
int fs_forward_bf16(const int32_t* dims, int32_t n_dims, const float* w, const void* x_bf16, int32_t rows,
                    double* probs_out, void* stream);
int fs_train_bf16(const fs_train_desc* desc, const void* features_bf16, const float* labels_f32,
                  void* stream);
/* K8 forward in bf16 mode for shapes beyond the on-chip kernels (the wide
 * MLP): cuBLAS bf16 GEMMs, fp32 accumulation, fused relu/bias epilogues,
 * fp32 head; probs_out[rows] (float64) of fs_prep_features_bf16 rows.     */
size_t fs_forward_wide_workspace_bytes(const int32_t* dims, int32_t n_dims, int32_t rows);
int fs_forward_wide(const int32_t* dims, int32_t n_dims, const float* w, const void* x_bf16, int32_t rows,
                    double* probs_out, void* workspace, size_t workspace_bytes, void* stream);

/* backend.loss_and_grad (_core.pyx:140-219 / numpy_backend.py:60-104):
 * one batch x[rows x dims[0]], labels y[rows], optional dense pre-scaled masks
 * (layer-major [rows x h_l] blocks) -> loss_out[1], grad_out[M]. Shares the
 * trainer's step code, so train_local == fold(loss_and_grad + sgd_step)
 * bitwise.                                                                 */
size_t fs_step_workspace_bytes(const int32_t* dims, int32_t n_dims, int32_t rows);
int fs_loss_and_grad_f64(const int32_t* dims, int32_t n_dims, const double* w, const double* x,
                         const double* y, int32_t rows, const double* dense_masks,
                         double* loss_out, double* grad_out, int32_t* status, void* workspace,
                         size_t workspace_bytes, void* stream);

/* backend.forward (_core.pyx:109-137): class-1 probabilities of x rows.   */
size_t fs_forward_workspace_bytes(const int32_t* dims, int32_t n_dims, int32_t rows);
int fs_forward_f64(const int32_t* dims, int32_t n_dims, const double* w, const double* x,
                   int32_t rows, const double* dense_masks, double* probs_out, void* workspace,
                   size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------- K6 alignment
 * aligned_out[r] = #{j : sgn(a_j) == sgn(b_j)}, sgn in {-1,0,+1}
 * (_core.pyx:222-236) with a = wc[r], b = wg[r] (weight_sign) or
 * a = wc[r]-wg[r], b = wg[r]-wg_prev[r] (delta_sign), selection.py:53-74.
 * wc/wg/wg_prev are [n_req] arrays of device pointers to float64 [M].      */
int fs_sign_align_f64(const uint64_t* wc, const uint64_t* wg, const uint64_t* wg_prev,
                      int32_t n_req, int64_t M, int32_t mode, int64_t* aligned_out,
                      void* stream);

/* float32 variant (bf16 mixed-precision mode: fp32 parameter vectors).   */
int fs_sign_align_f32(const uint64_t* wc, const uint64_t* wg, const uint64_t* wg_prev,
                      int32_t n_req, int64_t M, int32_t mode, int64_t* aligned_out,
                      void* stream);

/* Synchronous-round form: every request compares against the same wg (and
 * wg_prev) vectors, given directly as device pointers (16-byte aligned);
 * rows in wc must be 16-byte aligned. dtype_bytes = 8 (fp64) or 4 (fp32).  */
int fs_sign_align_shared(const uint64_t* wc, const void* wg, const void* wg_prev, int32_t n_req,
                         int64_t M, int32_t mode, int32_t dtype_bytes, int64_t* aligned_out,
                         void* stream);

/* ---------------------------------------------------------------- K7/K9 FedAvg
 * keys_out[i*n_keys + t] = bswap64(bits(rows[i][t])) — the leading bytes
 * of values.tobytes() as big-endian integers (server.py:84 sort key).     */
int fs_gather_sort_keys_f64(const uint64_t* rows, int32_t k, int32_t n_keys, uint64_t* keys_out,
                            void* stream);
/* Device-side K9: sorted_rows = rows ordered by values.tobytes() (k <= 1024),
 * no host round trip; feeds fs_aggregate_* / fs_sum_rows directly.        */
int fs_canonical_order(const uint64_t* rows, int32_t k, int64_t M, int32_t dtype_bytes,
                       uint64_t* sorted_rows, void* stream);
/* out[j] = (sum_{i=0..k-1} rows[i][j]) / k, summed sequentially in the given
 * row order (server.py:84-86: stack in sorted order, mean(axis=0)).        */
int fs_aggregate_f64(const uint64_t* rows, int32_t k, int64_t M, double* out, void* stream);

/* float32 variants (bf16 mode): keys are bswap32 of the leading floats;
 * the mean is accumulated in float64 and rounded once to float32.         */
int fs_gather_sort_keys_f32(const uint64_t* rows, int32_t k, int32_t n_keys, uint64_t* keys_out,
                            void* stream);
int fs_aggregate_f32(const uint64_t* rows, int32_t k, int64_t M, float* out, void* stream);

/* Client-sharded rounds (one GPU per rank): each rank sums its accepted
 * updates (float64 accumulation, rows of float32 or float64 given by
 * dtype_bytes), the ranks all-reduce [sum | counts] over NCCL, and every
 * rank finishes out[j] = sum[j] / k in the parameter dtype, so the global
 * model stays replicated without a broadcast.                            */
/* K6 for rows at base + i * stride_bytes, i < n_req (a trainer launch's
 * output block), against one shared (w_g, w_g_prev): no pointer array.     */
int fs_sign_align_rows(uint64_t base, int64_t stride_bytes, const void* wg, const void* wg_prev, int32_t n_req,
                       int64_t M, int32_t mode, int32_t dtype_bytes, int64_t* aligned_out, void* stream);

/* Many FedAvg means in one launch pair (an async run's aggregations between
 * two training flushes): job j = mean of rows[job_off[j]..job_off[j+1]) in
 * canonical byte order -> job_out[j] (device pointers; 1 <= rows per job <=
 * max_k <= 1024; sorted_scratch holds job_off[n_jobs] pointers).         */
int fs_aggregate_jobs(const uint64_t* rows, const int64_t* job_off, int32_t n_jobs, int32_t max_k, int64_t M,
                      int32_t dtype_bytes, uint64_t* sorted_scratch, const uint64_t* job_out, void* stream);
/* Weighted jobs (opt-in staleness-weighted FedAvg, an extension; the
 * reference's mean is unweighted, server.py:587-593): job j's output is
 * sum_i w_i x_i / sum_i w_i over its rows in canonical byte order; weights
 * [job_off[n_jobs]] float64 in job order, sorted_w the same size scratch.   */
int fs_aggregate_jobs_weighted(const uint64_t* rows, const double* weights, const int64_t* job_off, int32_t n_jobs,
                               int32_t max_k, int64_t M, int32_t dtype_bytes, uint64_t* sorted_scratch,
                               double* sorted_w, const uint64_t* job_out, void* stream);

/* filter_update on the device for a synchronous round (selection.py:77-85):
 * accepted rows (aligned[i] / den >= theta, den = M for the sign counts or
 * FS_COSINE_SCALE for cosine scores; all rows when scored == 0) in client
 * order -> rows_out, job_off = {0, k}, job_out[0] = out: the single job of
 * fs_aggregate_jobs, so FedAvg follows K6 with no host round trip. Rows are
 * base + i * stride_bytes. top_k > 0 (opt-in extension, n <= 16384) keeps
 * only the top_k highest-scoring accepted rows (ties: lower index first).  */
int fs_select_rows(const int64_t* aligned, int32_t n, int64_t den, double theta, int32_t scored, int32_t top_k,
                   uint64_t base, int64_t stride_bytes, uint64_t* rows_out, int64_t* job_off, uint64_t* job_out,
                   uint64_t out, void* stream);

/* K6c, opt-in `delta_cosine` relevance (an extension; the reference counts
 * matching signs, selection.py:53-74): score_out[r] = llrint(cos * 2^40),
 * cos = <w_c - w_g, w_g - w_prev> / (|w_c - w_g| |w_g - w_prev|) (0 when a
 * norm is 0), float64 with a fixed summation order. Rows are wc[r] (device
 * pointer array) or, when wc == NULL, base + r * stride_bytes.              */
#define FS_COSINE_SCALE 1099511627776LL /* 2^40 */
size_t fs_cosine_align_workspace_bytes(int32_t n_req);
int fs_cosine_align(const uint64_t* wc, uint64_t base, int64_t stride_bytes, const void* wg, const void* wg_prev,
                    int32_t n_req, int64_t M, int32_t dtype_bytes, int64_t* score_out, void* workspace,
                    size_t workspace_bytes, void* stream);

/* bf16-mode FedAvg of one fs_select_rows job of float32 rows: the rows
 * (client order) cut into 16 groups summed in parallel (float64 partials,
 * groups added in order): deterministic, tolerance-matched (the canonical
 * numpy order is the fp64 parity mode's contract, fs_aggregate_jobs).
 * sorted_scratch is unused.                                                 */
size_t fs_aggregate_rowsplit_workspace_bytes(int64_t M);
int fs_aggregate_rowsplit_f32(const uint64_t* rows, const int64_t* job_off, int32_t max_k, int64_t M,
                              uint64_t* sorted_scratch, const uint64_t* job_out, void* workspace,
                              size_t workspace_bytes, void* stream);

int fs_sum_rows(const uint64_t* rows, int32_t k, int64_t M, int32_t dtype_bytes, double* out,
                void* stream);

/* Client-sharded synchronous round on the device (parallel.py): no host
 * round trip before the all-reduce.
 *   fs_sum_job          canonical-order float64 sum of one fs_select_rows job
 *                       (k read on the device) -> *job_out[0] (double [M]);
 *   fs_pack_exchange    tail[0..2N] = {counts scattered to own_idx | k |
 *                       status scattered to own_idx} (zeros elsewhere);
 *   fs_mean_finish_dev  out = sum / k (k = *k_dev, after the all-reduce), or
 *                       keep (the previous model) when k == 0.               */
int fs_sum_job(const uint64_t* rows, const int64_t* job_off, int32_t max_k, int64_t M, int32_t dtype_bytes,
               uint64_t* sorted_scratch, const uint64_t* job_out, void* stream);
int fs_pack_exchange(const int64_t* counts, const int32_t* status, const int32_t* own_idx, int32_t k, int32_t N,
                     const int64_t* job_off, double* tail, void* stream);
int fs_mean_finish_dev(const double* sum, const double* k_dev, int64_t M, int32_t dtype_bytes, const void* keep,
                       void* out, void* stream);
int fs_mean_finish(const double* sum, int64_t k, int64_t M, int32_t dtype_bytes, void* out, void* stream);

/* ---------------------------------------------------------------- K8 metrics
 * accuracy at `threshold` and rank AUC with midrank ties
 * (metrics.py:118-165): counts_out[0] = #correct, counts_out[1] = 2*U_pos
 * (exact), counts_out[2] = n_pos.                                          */
size_t fs_eval_workspace_bytes(int32_t n);
int fs_eval_metrics(const double* scores, const int8_t* labels, int32_t n, double threshold,
                    int64_t* counts_out, void* workspace, size_t workspace_bytes, void* stream);
/* Same counts when every score is a widened float (the bf16 evaluation,
 * fs_forward_bf16): ranks on float keys, half the radix-sort passes.      */
int fs_eval_metrics_f32(const double* scores, const int8_t* labels, int32_t n, double threshold,
                        int64_t* counts_out, void* workspace, size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------- f2 async event engine
 * Host-side (all pointers HOST memory; no CUDA): the event loop of
 * FederationEngine.run_async (server.py:485-637; simnet.py:18-103 clock).
 * It never touches parameters. fs_async_run processes events until a
 * train_done needs the outcome of a not-yet-trained cycle, then returns
 * FS_ASYNC_NEED_EVAL with every pending cycle listed (eval_*: deferred id,
 * client index, cycle, fetched model version); the caller trains + scores
 * them and calls fs_async_provide, then fs_async_run again. Aggregations are
 * returned as jobs (new version <- mean of the member cycles' updates, in
 * server.aggregate's canonical order), to be launched before the next
 * training batch; window reports likewise. The yield's arrays stay valid
 * until the next fs_async_run. The processed-event log is read with
 * fs_async_log (columnar; kind codes as in paper_2503_15448_b200/server.py). */
#define FS_ASYNC_NEED_EVAL 1
#define FS_ASYNC_REPORT 2   /* device mode: window reports ready (rep_w = versions to evaluate) */

typedef struct fs_async_engine fs_async_engine;

typedef struct {
  int32_t n_clients, max_cycles, rounds, k_min;
  int64_t budget;                /* rounds * n_clients accepted updates */
  double buffer_timeout_s, agg_cost_per_update_s;
  double horizon_s;              /* < 0: none */
  double recovery_s, transfer_s0;
  const int32_t* cid;            /* [n_clients] client ids */
  const int32_t* steps;          /* [n_clients] SGD steps per training */
  const double *down, *up;       /* [n_clients] latencies */
  int32_t plan_per_cycle;        /* 1: plan arrays are [n_clients x max_cycles]; 0: [n_clients] */
  const uint8_t *trains, *failed, *recovered;
  const double *fail_off, *span;
  const int32_t* n_captures;     /* checkpoint events per cycle (leading capture offsets) */
  const int32_t* cap_ptr;        /* [n_clients + 1] CSR into cap_off */
  const double* cap_off;
  int64_t w_counts0[4];          /* open window at start: accepted, rejected, failures, steps */
} fs_async_world;

typedef struct {
  int32_t n_eval;
  const int32_t *eval_id, *eval_ci, *eval_cycle, *eval_version;
  int32_t n_jobs;
  const int32_t* job_version;    /* version created by job j */
  const int64_t* job_off;        /* [n_jobs + 1] CSR into job_member (deferred ids) */
  const int32_t* job_member;
  int32_t n_reports;
  const int64_t* rep_i;          /* [n_reports x 9]: window, version, updates, aggregations,
                                    accepted, rejected, failures, steps, 0 */
  const double* rep_d;           /* [n_reports x 2]: t_s, cumulative transfer_s */
  const int64_t* rep_off;        /* [n_reports + 1] CSR into rep_stale */
  const int32_t* rep_stale;
  double now_s;
  int64_t seq;
  int32_t agg_count;
  int64_t trainings;
  int32_t stopped;
  double transfer_s;
  int64_t w_counts[4];           /* open window: accepted, rejected, failures, steps */
  /* device mode (fs_async_attach_device) */
  const uint64_t* rep_w;         /* [n_reports] device pointers of the report versions */
  uint64_t w_g, w_g_prev;        /* current / previous global model (device; 0 = none) */
  int64_t flushes, launches;     /* training flushes and kernel-launching calls so far */
  int32_t diverged_client, diverged_cycle;  /* set with FS_EDIVERGED */
  double host_s[3];              /* diagnostics: host seconds preparing flushes, waiting on them, after them */
} fs_async_yield;

typedef struct {
  int64_t n;
  const int8_t* kind;
  const double* t;
  const int32_t *ci, *cycle;
  const int64_t *a, *b;
  const double* x;
  const int64_t* l;              /* aggregate records: offset into list_cid / list_stale */
  int64_t n_list;
  const int32_t *list_cid, *list_stale;
} fs_async_logview;

/* Device mode: the engine does the parameter work itself on `stream` --
 * per deferred flush one staged metadata copy, K2 + K3 + K5 + K6 and one
 * device->host read of the counts; aggregation jobs go to fs_aggregate_jobs.
 * fs_async_run then returns only FS_ASYNC_REPORT (evaluate rep_w, call
 * again), FS_EDIVERGED or 0 (done). Model versions and trained rows are
 * stream-ordered allocations owned by the engine (freed by destroy). */
typedef struct {
  int32_t n_dims;
  int32_t dims[FS_MAX_LAYERS + 1];
  int32_t epochs;
  int32_t bf16;                  /* 1: tcgen05 trainer (float32 rows); 0: fp64 parity trainer */
  double dropout_rate;
  int32_t align_mode;            /* FS_ALIGN_* */
  double theta;
  uint64_t master_seed;
  double base_lr, lr_decay;
  int32_t grid;                  /* trainer CTAs (0 = auto) */
  const void *features, *labels; /* fp64 shards (fp64) or fs_prep_features_bf16 rows + float32 labels */
  const int64_t* row_off_host;   /* [n_clients] */
  const int32_t* n_rows_host;    /* [n_clients] */
  const int32_t* batch_host;     /* [n_clients] */
  const void* w0;                /* version 0 (caller-owned, device) */
  const void* w0_prev;           /* w_g_prev at start (caller-owned; NULL = none) */
  void* stream;
  /* opt-in extension (< 0 = off, the reference's unweighted mean): flush
   * means weighted by (1 + staleness) ** -staleness_alpha                  */
  double staleness_alpha;
  /* client sharding over the ranks of a node (world_size > 1; parallel.py
   * ownership, server.py:409-417 call sites): every rank runs the same event
   * loop; a flush trains only the cycles of clients with owner_host[ci] ==
   * rank, and `exchange` sums a device float64 buffer over the ranks in
   * place (an all-reduce; called after `stream` is synchronised, must
   * return with the sum written): once per flush for [aligned | status] of
   * every pending cycle and once for the float64 partial sums of the
   * aggregation jobs (each rank sums its own members in canonical order).
   * world_size <= 1: unsharded, the other fields are ignored.              */
  int32_t rank;
  int32_t world_size;
  const int32_t* owner_host;     /* [n_clients] */
  int (*exchange)(void* ctx, double* buf, int64_t n, void* stream);
  void* exchange_ctx;
} fs_async_device;

fs_async_engine* fs_async_create(const fs_async_world* world);
int fs_async_attach_device(fs_async_engine* engine, const fs_async_device* dev);
void fs_async_destroy(fs_async_engine* engine);
int fs_async_run(fs_async_engine* engine, fs_async_yield* out);
int fs_async_provide(fs_async_engine* engine, int32_t n, const uint8_t* accepted_host,
                     const double* relevance_host);
int fs_async_log(const fs_async_engine* engine, fs_async_logview* out);

#ifdef __cplusplus
}
#endif
#endif /* FEDSIM_B200_H */
