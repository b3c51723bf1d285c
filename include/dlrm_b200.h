/*
 * dlrm_b200.h — C ABI of libdlrmb200.so, the sm_100a kernels behind the
 * DLRM training step (arXiv 1906.00091).
 *
 * The reference (dlrmkit) is pure Python/numpy and has no FFI; its operator
 * API *is* the set of Python functions re-exported by
 * /root/reference/pkg/src/dlrmkit/__init__.py:10-80.  Each entry point below
 * replaces the numerical core of one of those functions and cites it.  The
 * Python package paper_1906_00091_b200 binds these with ctypes (see
 * INTEGRATION.md) and keeps the reference's names, argument meanings and
 * exceptions.
 *
 * Conventions
 *   - Every pointer is a DEVICE pointer unless documented otherwise; the
 *     caller owns every buffer; the library never allocates caller-visible
 *     memory (workspaces are sized by *_workspace_size and passed in).
 *   - Every call is asynchronous on the given stream and never synchronises
 *     the host, so a whole training step can be captured in a CUDA graph.
 *   - Return codes: 0 ok, 1 invalid argument, 2 CUDA error; the message is
 *     available from dlrm_last_error() (thread-local).
 *   - All floating-point work is fp32; index work is int64/uint32 and
 *     bit-exact with the reference.
 */
#ifndef DLRM_B200_H
#define DLRM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* dlrm_stream_t; /* a cudaStream_t */

#define DLRM_MAX_TABLES 128
#define DLRM_MAX_FEATURES 129

/* One table's bags for a multi-table call (host struct, passed by value to
 * the kernels).  Mirrors SparseBatch (ref embedding.py:74-124) plus where the
 * table lives in the rank's concatenated weight buffer and where its pooled
 * rows go.  All tables of one call have the same num_bags (the batch). */
typedef struct {
  const int64_t* offsets;  /* [num_bags+1], offsets[0]==0, terminal == nnz   */
  const int64_t* indices;  /* [capacity] (first offsets[num_bags] are live) */
  const float* weights;    /* [capacity] per-index weights or NULL          */
  int64_t row_base;        /* first row of this table in W_all              */
  int64_t num_rows;        /* m                                            */
  int64_t out_offset;      /* element offset of bag 0's row in out / grad   */
  int64_t capacity;        /* index slots reserved (>= nnz); sort size      */
  int64_t table_id;        /* reported in LookupIndexError                  */
} dlrm_table_desc;

/* Parameter update rule applied by the fused *_upd / *_apply entry points
 * (ref optim.py).  For every updated fp32 parameter p with gradient g:
 *   DLRM_UPD_SGD      p -= fl(lr*g)                                (31-46)
 *   DLRM_UPD_ADAGRAD  G += fl(g*g);  p -= fl(fl(lr*g) / fl(sqrt(G) + eps))
 *                                                                 (49-73)
 * with G the accumulator at address &p + accum_delta (floats): the caller
 * keeps one accumulator buffer with the SAME layout as each parameter buffer
 * (the tables' W_all, the flat MLP buffer) and passes the pointer distance.
 * Products / quotients are rounded before the subtraction exactly like numpy
 * (no FMA contraction). */
#define DLRM_UPD_SGD 0
#define DLRM_UPD_ADAGRAD 1
typedef struct {
  int32_t kind;        /* DLRM_UPD_SGD or DLRM_UPD_ADAGRAD */
  float lr;
  float eps;           /* Adagrad only */
  int64_t accum_delta; /* Adagrad only: accumulator = parameter + delta */
} dlrm_update;

/* ---- embedding bags (north_star subsystem 1) --------------------------- */

/* Reset the error records: err_pos[0..nt) = INT64_MAX, *err_flag = 0. */
int dlrm_err_reset(int64_t* err_pos, int32_t nt, int32_t* err_flag,
                   dlrm_stream_t stream);

/* err_val[t] = tables[t].indices[err_pos[t]] when *err_flag is set and
 * table t has a recorded position, else 0: the offending index VALUE for
 * LookupIndexError (ref embedding.py:117-124), read on the device from the
 * batch that ran.  Launch it after the kernels that record errors. */
int dlrm_err_resolve(const dlrm_table_desc* tables, int32_t nt, const int64_t* err_pos,
                     const int32_t* err_flag, int64_t* err_val, dlrm_stream_t stream);

/* Pooled lookup S = A^T W for nt tables (ref lookup_batch,
 * embedding.py:155-179): out[out_offset_t + j*out_stride + c] =
 * strict ascending-position fold over bag j of W[row_base+idx]*a.  Empty bags
 * give zero rows.  Out-of-range indices are skipped and recorded as
 * atomicMin(err_pos[t], position) + *err_flag = 1 (ref check_bounds,
 * embedding.py:117-124). */
int dlrm_emb_fwd(const float* W_all, int64_t dim, const dlrm_table_desc* tables,
                 int32_t nt, int64_t num_bags, float* out, int64_t out_stride,
                 int64_t* err_pos, int32_t* err_flag, dlrm_stream_t stream);

/* Bytes of scratch needed by dlrm_emb_bwd_sgd / dlrm_emb_bwd_coalesce for
 * total_capacity index slots over total_rows rows of dim floats. */
size_t dlrm_emb_bwd_workspace_size(int64_t total_capacity, int64_t total_rows,
                                   int64_t dim);

/* Sparse backward fused with the SGD row update (ref lookup_backward,
 * embedding.py:182-210, then sgd_step_rows, optim.py:38-46):
 *   for every touched row r:  W[r] -= lr * fold_{k: idx_k = r, ascending k}
 *                                        grad[bag(k)] * a_k
 * via a stable radix sort of (row, position) pairs and a deterministic
 * segmented fold — no float atomics.  grad rows are read at
 * grad[out_offset_t + j*grad_stride].  If *err_flag is set no row is
 * written (the reference raises before mutating). */
int dlrm_emb_bwd_sgd(float* W_all, int64_t dim, const dlrm_table_desc* tables,
                     int32_t nt, int64_t num_bags, const float* grad,
                     int64_t grad_stride, float lr, const int32_t* err_flag,
                     int64_t total_rows, void* workspace, size_t ws_bytes,
                     dlrm_stream_t stream);

/* dlrm_emb_bwd_sgd in two phases so the index-only work can run off the
 * critical path (e.g. on a side stream during the forward pass):
 *   prepare    keys + stable radix sort of (row, position) pairs; reads only
 *              offsets / indices, writes the workspace;
 *   apply_sgd  segmented fold of grad + row update from that workspace (same
 *              arguments and semantics as dlrm_emb_bwd_sgd).
 * apply_sgd must be ordered after prepare on the same workspace and tables.
 * dlrm_emb_bwd_sgd == prepare; apply_sgd. */
int dlrm_emb_bwd_prepare(int64_t dim, const dlrm_table_desc* tables, int32_t nt,
                         int64_t num_bags, int64_t total_rows, void* workspace,
                         size_t ws_bytes, dlrm_stream_t stream);
int dlrm_emb_bwd_apply_sgd(float* W_all, int64_t dim, const dlrm_table_desc* tables,
                           int32_t nt, int64_t num_bags, const float* grad,
                           int64_t grad_stride, float lr, const int32_t* err_flag,
                           int64_t total_rows, void* workspace, size_t ws_bytes,
                           dlrm_stream_t stream);
/* apply with any update rule (SGD or Adagrad; ref adagrad_step_rows,
 * optim.py:62-73): the rule is applied once per touched row to its folded
 * gradient; the row accumulators live at W_all + upd->accum_delta. */
int dlrm_emb_bwd_apply(float* W_all, int64_t dim, const dlrm_table_desc* tables,
                       int32_t nt, int64_t num_bags, const float* grad,
                       int64_t grad_stride, const dlrm_update* upd,
                       const int32_t* err_flag, int64_t total_rows, void* workspace,
                       size_t ws_bytes, dlrm_stream_t stream);

/* lookup_backward parity path for ONE table: coalesced SparseRowGrad.
 * rows_out[u] ascending unique local rows, values_out[u*dim..] their folded
 * gradients, *num_unique = u (device int64).  Buffers sized for nnz rows.
 * Out-of-range indices are recorded in err_pos[0] / *err_flag like
 * dlrm_emb_fwd (the caller raises LookupIndexError). */
int dlrm_emb_bwd_coalesce(int64_t dim, const dlrm_table_desc* table,
                          int64_t num_bags, const float* grad,
                          int64_t grad_stride, int64_t* rows_out,
                          float* values_out, int64_t* num_unique,
                          int64_t* err_pos, int32_t* err_flag,
                          void* workspace, size_t ws_bytes,
                          dlrm_stream_t stream);

/* W[rows[i]] -= lr * values[i]  (ref sgd_step_rows, optim.py:38-46). */
int dlrm_sgd_rows(float* W, int64_t dim, const int64_t* rows,
                  const float* values, int64_t n, float lr,
                  dlrm_stream_t stream);
/* rows update with any rule (ref sgd_step_rows / adagrad_step_rows). */
int dlrm_update_rows(float* W, int64_t dim, const int64_t* rows, const float* values,
                     int64_t n, const dlrm_update* upd, dlrm_stream_t stream);

/* ---- dot interaction (north_star subsystem 2) -------------------------- */

/* Feature f of sample b lives at feat[f] + b*feat_stride[f] (d floats);
 * f = 0 is the bottom-MLP output, f = 1+t table t.  (host arrays) */
typedef struct {
  const float* feat[DLRM_MAX_FEATURES];
  int64_t feat_stride[DLRM_MAX_FEATURES];
} dlrm_features;

/* out[b*ld_out + :] = [z0 | z_i.z_j for i<j row-major] (ref interact,
 * model.py:218-242); columns [d+P, pad_to) are written as zeros. */
int dlrm_interact_fwd(const dlrm_features* feats, int32_t nf, int64_t dim,
                      int64_t batch, float* out, int64_t ld_out,
                      int64_t pad_to, dlrm_stream_t stream);

/* grad_feat[f] + b*grad_stride[f] = [f==0] gout[b,:d] + sum_{j!=f} g_fj z_j
 * (ref interact_backward, model.py:245-268).  grad_feat / grad_stride are
 * HOST arrays of nf entries (device pointers / element strides). */
int dlrm_interact_bwd(const dlrm_features* feats, int32_t nf, int64_t dim,
                      int64_t batch, const float* gout, int64_t ld_gout,
                      float* const* grad_feat, const int64_t* grad_stride,
                      int32_t relu_mask_f0, dlrm_stream_t stream);
/* relu_mask_f0 != 0 multiplies feature 0's gradient by (z0 > 0): the
 * bottom MLP's last ReLU folded into the interaction backward (training
 * step only; the API-level interact_backward passes 0). */

/* ---- MLP layers (north_star subsystem 2) ------------------------------- */

enum { DLRM_ACT_IDENTITY = 0, DLRM_ACT_RELU = 1 };

/* Y[m, n] = act((X W^T)[m, n] + b[n]) for m < M, n < N (ref mlp_forward,
 * model.py:142-156 with matmul dense.py:62-78).  X: M x K (ldx), W: N x K
 * (ldw).  Columns [N, pad_n) of Y are zeroed. */
int dlrm_linear_fwd(const float* X, int64_t ldx, const float* W, int64_t ldw,
                    const float* b, float* Y, int64_t ldy, int64_t M,
                    int64_t N, int64_t K, int64_t pad_n, int32_t act,
                    dlrm_stream_t stream);

/* dX[m, k] = (gZ W)[m, k] * (mask ? (mask[m, k] > 0) : 1)
 * (ref mlp_backward_trace, model.py:173-179; mask = the previous layer's
 * ReLU output, whose positivity equals act'(z) > 0). */
int dlrm_linear_bwd_data(const float* gZ, int64_t ldg, const float* W,
                         int64_t ldw, const float* mask, int64_t ldm,
                         float* dX, int64_t ldx, int64_t M, int64_t N,
                         int64_t K, dlrm_stream_t stream);

/* The same two GEMMs with the weights' TF32 low parts precomputed:
 * W_lo = dlrm_tf32_split_lo(W) in W's layout (the engine refreshes it once
 * per step for all layers).  The tensor-core kernels then load B_lo by TMA
 * instead of converting it per output tile; results are bitwise those of
 * dlrm_linear_fwd / dlrm_linear_bwd_data.  W_lo = NULL: the plain calls. */
int dlrm_linear_fwd_wlo(const float* X, int64_t ldx, const float* W,
                        const float* W_lo, int64_t ldw, const float* b, float* Y,
                        int64_t ldy, int64_t M, int64_t N, int64_t K,
                        int64_t pad_n, int32_t act, dlrm_stream_t stream);
int dlrm_linear_bwd_data_wlo(const float* gZ, int64_t ldg, const float* W,
                             const float* W_lo, int64_t ldw, const float* mask,
                             int64_t ldm, float* dX, int64_t ldx, int64_t M,
                             int64_t N, int64_t K, dlrm_stream_t stream);
/* lo[i] = tf32(x[i] - x[i] with its low 13 mantissa bits cleared), n a
 * multiple of 4, 16-byte aligned buffers. */
int dlrm_tf32_split_lo(const float* x, float* lo, int64_t n, dlrm_stream_t stream);

/* Input staging: on `stream`, wait for wait_ev (if any), copy `bytes` from
 * pinned host memory to the device, then record ev1 / ev2 (if any; CUDA
 * event handles).  The Python packer calls it right after packing a batch,
 * without the interpreter lock. */
int dlrm_h2d_async(void* dst, const void* src, size_t bytes, void* wait_ev, void* ev1,
                   void* ev2, dlrm_stream_t stream);

/* Device-to-device copy on `stream` after wait_ev, then ev recorded (the
 * staged input block handed to the step engine in one call). */
int dlrm_d2d_async(void* dst, const void* src, size_t bytes, void* wait_ev, void* ev,
                   dlrm_stream_t stream);

/* A step's result read-back on `stream` in one call: the result block to
 * pinned host memory, the probabilities device to device, then `ev`
 * recorded (the engine's asynchronous results; one call instead of three
 * runtime calls from the training thread). */
int dlrm_step_result_copy(void* host_dst, const void* res, size_t res_bytes, void* prob_dst,
                          const void* prob, size_t prob_bytes, void* ev,
                          dlrm_stream_t stream);

size_t dlrm_linear_bwd_weight_workspace_size(int64_t M, int64_t N, int64_t K);

/* dW = gZ^T X (N x K), db = column sums of gZ (ref mlp_backward,
 * model.py:191-208, as a plain fp32 reduction over the batch with a fixed
 * split order — deterministic).  If dW/db are NULL they are not stored.
 * If W_upd/b_upd are non-NULL the SGD step W -= lr*dW, b -= lr*db
 * (ref sgd_step, optim.py:31-35) is fused in, skipped when *err_flag != 0. */
int dlrm_linear_bwd_weight(const float* gZ, int64_t ldg, const float* X,
                           int64_t ldx, int64_t M, int64_t N, int64_t K,
                           float* dW, int64_t lddw, float* db,
                           float* W_upd, int64_t ldw, float* b_upd, float lr,
                           const int32_t* err_flag, void* workspace,
                           size_t ws_bytes, dlrm_stream_t stream);
/* the same with any update rule for W_upd / b_upd (accumulators at
 * parameter + upd->accum_delta). */
int dlrm_linear_bwd_weight_upd(const float* gZ, int64_t ldg, const float* X,
                               int64_t ldx, int64_t M, int64_t N, int64_t K,
                               float* dW, int64_t lddw, float* db, float* W_upd,
                               int64_t ldw, float* b_upd, const dlrm_update* upd,
                               const int32_t* err_flag, void* workspace,
                               size_t ws_bytes, dlrm_stream_t stream);

/* ---- loss head (last top layer, N = 1) --------------------------------- */

/* z[m] = A[m,:K] . w + b;  prob = sigmoid(z);  per-sample BCE from logits;
 * g[m] = (sigmoid(z) - y) / n_total;  stats[0] += sum(per) (fp32, fixed
 * order), stats[1] += #((p > 0.5) == (y > 0.5))   (ref bce_from_logits,
 * model.py:448-461; accuracy parallel.py:286).  logits/prob may be NULL. */
size_t dlrm_bce_head_workspace_size(int64_t M);
int dlrm_bce_head(const float* A, int64_t lda, const float* w, const float* b,
                  int64_t M, int64_t K, const float* y, float n_total,
                  float* logits, float* prob, float* grad_z, float* per_sample,
                  float* stats, void* workspace, size_t ws_bytes,
                  dlrm_stream_t stream);

/* The whole loss head in two launches (forward of the N = 1 layer, BCE,
 * logit gradient, and its backward + update; one pass over A): what
 * dlrm_bce_head followed by dlrm_head_bwd_upd compute, with dw / db / the
 * loss statistics reduced in a fixed CTA order.  Needs K % 4 == 0,
 * K <= 1024, 16-byte aligned A / w / dA rows.  Optional outputs may be NULL:
 * prob, grad_z, dA, dw, db, w_upd, b_upd. */
size_t dlrm_head_step_workspace_size(int64_t M, int64_t K);
int dlrm_head_step(const float* A, int64_t lda, const float* w, const float* b,
                   int64_t M, int64_t K, const float* y, float n_total, float* prob,
                   float* grad_z, float* stats, float* dA, int64_t ldda,
                   int32_t relu_mask, float* dw, float* db, float* w_upd, float* b_upd,
                   const dlrm_update* upd, const int32_t* err_flag, void* workspace,
                   size_t ws_bytes, dlrm_stream_t stream);
/* dlrm_head_step as its two launches: _partials (prob, grad_z, dA and the
 * per-CTA partial dw / db / loss / correct sums in the workspace) and _reduce
 * (fixed-order reduction into dw / db / stats + the fused update).  Only the
 * workspace links them, so _reduce may run on another stream, ordered after
 * _partials (the step engine takes it off the critical path: the data
 * gradients below the head need only dA). */
int dlrm_head_step_partials(const float* A, int64_t lda, const float* w, const float* b,
                            int64_t M, int64_t K, const float* y, float n_total, float* prob,
                            float* grad_z, float* dA, int64_t ldda, int32_t relu_mask,
                            void* workspace, size_t ws_bytes, dlrm_stream_t stream);
int dlrm_head_step_reduce(int64_t M, int64_t K, float* stats, float* dw, float* db,
                          float* w_upd, float* b_upd, const dlrm_update* upd,
                          const int32_t* err_flag, void* workspace, size_t ws_bytes,
                          dlrm_stream_t stream);

/* Backward through the N = 1 head: dA[m,k] = g[m]*w[k] (* (A[m,k] > 0) when
 * relu_mask, i.e. A is a ReLU output); dw[k] = sum_m g[m]*A[m,k];
 * db = sum_m g[m]; optional fused SGD (w -= lr*dw, b -= lr*db). */
size_t dlrm_head_bwd_workspace_size(int64_t M, int64_t K);
int dlrm_head_bwd(const float* A, int64_t lda, const float* w, const float* g,
                  int64_t M, int64_t K, float* dA, int64_t ldda,
                  int32_t relu_mask, float* dw, float* db, float* w_upd,
                  float* b_upd, float lr,
                  const int32_t* err_flag, void* workspace, size_t ws_bytes,
                  dlrm_stream_t stream);
int dlrm_head_bwd_upd(const float* A, int64_t lda, const float* w, const float* g,
                      int64_t M, int64_t K, float* dA, int64_t ldda,
                      int32_t relu_mask, float* dw, float* db, float* w_upd,
                      float* b_upd, const dlrm_update* upd,
                      const int32_t* err_flag, void* workspace, size_t ws_bytes,
                      dlrm_stream_t stream);

/* out[m, n] = g[m, n] * (act[m, n] > 0)   (ref activation_grad relu,
 * dense.py:110-120, applied as in model.py:177). */
int dlrm_relu_grad(const float* g, int64_t ldg, const float* act, int64_t lda,
                   float* out, int64_t ldo, int64_t M, int64_t N,
                   dlrm_stream_t stream);

/* ---- dense SGD ---------------------------------------------------------- */

/* p[i] -= lr * g[i], product rounded first (ref sgd_step, optim.py:31-35);
 * skipped when err_flag != NULL and *err_flag != 0. */
int dlrm_sgd_dense(float* p, const float* g, int64_t n, float lr,
                   const int32_t* err_flag, dlrm_stream_t stream);
/* dense update with any rule (ref sgd_step / adagrad_step, optim.py:31-59);
 * skipped when *err_flag. */
int dlrm_update_dense(float* p, const float* g, int64_t n, const dlrm_update* upd,
                      const int32_t* err_flag, dlrm_stream_t stream);

/* ---- misc --------------------------------------------------------------- */

/* Kernel selection (tests / A-B measurements): 0 = default (tcgen05 3xTF32
 * GEMMs wherever the shape and strides allow; the dot interaction on the
 * tensor cores where that is measured faster), 1 = SIMT fp32
 * only (MLP GEMMs and the dot interaction), 2 = tensor cores wherever legal
 * (the interaction at every size too). */
int dlrm_gemm_mode(int32_t mode);
/* the current kernel selection (dlrm_gemm_mode) */
int dlrm_gemm_mode_get(void);

/* ---- input pipeline: Criteo TSV ingestion (host code, multithreaded) ----
 * Replaces dlrmkit.datagen.parse_criteo / read_criteo (datagen.py:318-371)
 * for whole blocks of text.  Parses up to max_records non-blank lines of
 * text[0, nbytes) (whitespace-only lines skipped but counted)
 * into labels[r] (0 / 1), dense[r * ld_dense + i] = fp32(log1p(max(x, 0)))
 * (13 fields, empty -> 0) and cat[i * ld_cat + r] = blake2b64(token) %
 * vocab_sizes[i] (26 fields, empty -> 0).  *consumed = bytes used.  Returns
 * the record count; -1 bad arguments; -2 a malformed record, whose message
 * ("line k: ...", k counted from first_lineno, the reference's
 * CriteoFormatError text) is in dlrm_last_error().  flags: bit 0 = universal
 * newlines ('\n', '\r', "\r\n" end a line, as Python text-mode files do for
 * read_criteo; otherwise only '\n'); bits 8.. = threads (0: all cores).
 * Pointers are HOST pointers (pinned buffers of the next batch). */
int64_t dlrm_criteo_parse(const char* text, int64_t nbytes, const int64_t* vocab_sizes,
                          int64_t max_records, float* labels, float* dense, int64_t ld_dense,
                          int64_t* cat, int64_t ld_cat, int64_t first_lineno, int64_t* consumed,
                          int32_t flags);
/* The 64-bit token hash (ref datagen.py _hash_token): BLAKE2b, 8-byte digest,
 * no key, digest bytes read little-endian. */
uint64_t dlrm_blake2b64(const void* data, int64_t nbytes);

/* ---- input pipeline: the reference's random source (host code) ---------
 * Variable-length bags of the reference's random batches (dlrmkit
 * datagen.py:79-96 through cli.py:294-314), bit-identical to numpy:
 * per table t and sample j a length uniform in [1, k] then that many row
 * indices uniform in [0, rows[t]), drawn from numpy's Philox stream whose
 * state (Generator.bit_generator.state: counter[4], key[2], buffer[4],
 * buffer_pos, has_uint32, uinteger) is passed in `state` and advanced in
 * place.  offsets_out: [nt][batch + 1] (CSR, terminal entry included);
 * indices_out: [nt][batch * k] (the first nnz_out[t] of each row live).
 * rows[t] < 2^32.  Host pointers.  Returns 0, or 1 for bad arguments. */
int dlrm_random_bags(uint64_t* state, const int64_t* rows, int32_t nt, int64_t batch, int64_t k,
                     int64_t* offsets_out, int64_t* indices_out, int64_t* nnz_out);

/* One batch of the reference's host arrays packed into a step's input block
 * (the layout of paper_1906_00091_b200.pipeline.InputLayout; sec[] = byte
 * offsets of the x, labels, offsets, indices and per-index-weight sections,
 * the last -1 when unweighted): dense float64 rows -> fp32 (pitch ldx
 * floats), labels float64 -> fp32, offsets / indices int64 copied (table t's
 * indices at slot cap_base[t]), weights float64 -> fp32 (NULL table entry:
 * ones).  Runs on nthreads native threads.  Host pointers; 0 ok, 1 bad
 * arguments (an index count above its capacity included). */
int dlrm_pack_batch(uint8_t* dst, const int64_t* sec, int64_t batch, int64_t k0, int64_t ldx,
                    int32_t nt, const int64_t* cap_base, const double* dense, int64_t ld_dense,
                    const double* labels, const int64_t* const* offsets,
                    const int64_t* const* indices, const int64_t* nnz,
                    const double* const* weights, int32_t nthreads);

/* Count of this library's kernel launches since load (for bench.py). */
int64_t dlrm_launch_count(void);
const char* dlrm_last_error(void);
const char* dlrm_build_info(void);

#ifdef __cplusplus
}
#endif
#endif /* DLRM_B200_H */
