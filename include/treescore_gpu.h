/*
 * treescore_gpu.h -- C ABI of the B200 tree-ensemble scoring engine.
 *
 * Drop-in boundary for the reference package `treescore` (pure Python; its
 * only native crossing is the ctypes-loaded CodeGen unit, codegen.py:150-167).
 * Every entry point is plain C: pointers, sizes and status codes, no torch
 * types.  Errors return a nonzero ts_status and set a thread-local message
 * (ts_last_error); no entry point aborts the process.
 *
 *   reference interface                        replaced by
 *   ----------------------------------------   ------------------------------
 *   VPredicatedEvaluator.__init__               ts_pack
 *     (evaluators.py:490-512; expand_to_complete model.py:315-349)
 *   VPredicatedEvaluator._predict_into          ts_score  (device buffers,
 *     (evaluators.py:520-546; batch kernel        stream-ordered)
 *      evaluators.py:90-99)
 *   GeneratedUnit score_batch(const float *x,   ts_score_host (host buffers,
 *     int64_t n, int64_t f, double *out)          same argument meaning)
 *     (codegen.py:115-121, :173-179)
 *   GeneratedUnit score_ensemble(const float*)  ts_score_host with n = 1
 *     (codegen.py:108-113)
 *   leaf_index_predicated / batch_kernel        ts_score with ord_out != NULL
 *     ordinals (evaluators.py:122-134, :90-99)
 *   Evaluator.stored_node_count                 ts_model_info.table_entries
 *     (evaluators.py:197-200, :548-550)
 *   DepthLimitError (model.py:70-71, :324-327)  TS_ERR_DEPTH
 *   ValueError dataset shape (evaluators.py:212-220)  TS_ERR_SHAPE
 *   Dataset non-finite ValueError (data.py:50-51)     TS_ERR_NONFINITE
 *
 * Semantics (identical to the reference predicated kinds): a node sends x
 * right iff x[fid] >= threshold (ties go right); dummy padding nodes
 * (fid 0, theta +inf) always go left for finite x; the per-tree leaf ordinal
 * is the predicated ordinal of the tree's complete expansion to its own
 * depth; scores are acc = +0.0; acc = acc + weight * (double)leaf in tree
 * order, f64, multiply then add (no FMA) -- bit-identical to the reference.
 */
#ifndef TREESCORE_GPU_H
#define TREESCORE_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    TS_OK = 0,
    TS_ERR_INVALID = 1,      /* malformed model description or argument   */
    TS_ERR_DEPTH = 2,        /* tree deeper than TS_MAX_DEPTH              */
    TS_ERR_SHAPE = 3,        /* f != model num_features, bad ld / sizes    */
    TS_ERR_NONFINITE = 4,    /* instance matrix holds NaN or +-inf         */
    TS_ERR_CUDA = 5,         /* CUDA runtime failure (message has details) */
    TS_ERR_NOMEM = 6,
    TS_ERR_UNSUPPORTED = 7,
    TS_ERR_SYNTAX = 8        /* malformed model document (line/col set)    */
} ts_status;

#define TS_MAX_DEPTH 16

/* Flat logical model (the text model format's shape, SPEC "External
 * Interfaces" / model.py:356-387): trees in evaluation order; the nodes of
 * tree t are [tree_node_offset[t], tree_node_offset[t+1]) with tree-local
 * ids, id 0 the root.  node_fid[i] == -1 marks a leaf.  node_value is the
 * fp32 threshold (internal) or fp32 leaf value (leaf).  node_left/right are
 * tree-local child ids (ignored for leaves). */
typedef struct {
    int32_t num_features;
    int32_t num_trees;
    const int64_t *tree_node_offset;   /* [num_trees + 1] */
    const double *tree_weight;         /* [num_trees], finite */
    const int32_t *node_fid;
    const float *node_value;
    const int32_t *node_left;
    const int32_t *node_right;
} ts_model_desc;

typedef struct ts_model ts_model;

typedef struct {
    int32_t num_features;
    int32_t num_trees;
    int32_t max_depth;
    int32_t num_segments;          /* kernel launches per ts_score call     */
    int64_t sum_depth;             /* sum over trees of d_t (visits/instance) */
    int64_t table_entries;         /* sum 2^(d_t+1)-1: ref stored_node_count */
    int64_t device_bytes;          /* packed tables resident on the device  */
    int32_t complete_trees;        /* trees packed in the implicit heap form */
    int32_t compact_trees;         /* trees packed in the child-index form   */
    int32_t device;
    int32_t unit_weights;          /* all weights == 1.0 */
    int32_t rank_trees;            /* complete trees in the rank layout      */
    int32_t reserved;
} ts_model_info;

/* Validate, pack and upload a model to `device`.  The description is only
 * read during the call.  Returns TS_ERR_INVALID / TS_ERR_DEPTH on bad
 * models with a message naming the tree. */
int ts_pack(const ts_model_desc *desc, int device, ts_model **out);

/* ts_pack with options: TS_PACK_TRACE also uploads the logical trees for
 * ts_trace (16 bytes per node).  TS_PACK_ANY_DEPTH accepts trees deeper than
 * TS_MAX_DEPTH (up to TS_MAX_LINKED_DEPTH levels, <= 65535 nodes each), as the
 * reference's linked strategies do (ref evaluators.py: heap/compact linked,
 * contiguous): they are walked from their own child-index records; such a
 * model scores normally but refuses predicated ordinals (ord_out) with
 * TS_ERR_DEPTH, since no complete table exists for them. */
#define TS_PACK_TRACE 1
#define TS_PACK_ANY_DEPTH 2
/* TS_PACK_NO_RANK keeps complete trees in the fp32-threshold layout instead
 * of the rank layout deep trees otherwise get (thresholds replaced by their
 * rank among the ensemble's distinct thresholds of the feature, instances
 * ranked by a pre-pass; same results bit for bit).  ts_score_pipe needs it. */
#define TS_PACK_NO_RANK 4
#define TS_MAX_LINKED_DEPTH 31
int ts_pack_ex(const ts_model_desc *desc, int device, int flags, ts_model **out);

int ts_model_get_info(const ts_model *model, ts_model_info *info);

/* Score n instances already resident on the model's device.
 *   x        fp32 [n, f] row-major, row stride ld >= f (elements)
 *   out      f64 [n]
 *   ord_out  nullable; uint16 [num_trees, ld_ord] predicated leaf ordinals
 *            (tree-major so that rows are contiguous), ld_ord >= n
 *   status   nullable; int32 device word, OR-ed with 1 if any x is NaN/inf
 *   stream   cudaStream_t (NULL = legacy default stream)
 * Stream-ordered; returns after enqueueing.  Allocates nothing from the
 * caller's heaps: small batches with long walks (the two-pass tree split)
 * and rank-layout segments (deep complete trees: the instance ranks, 2 bytes
 * per value, in chunks of <= 2M rows) take per-call scratch from the
 * library's own stream-ordered memory pool (cudaMallocFromPoolAsync /
 * cudaFreeAsync on `stream`, so it stays CUDA-graph capturable). */
int ts_score(const ts_model *model, const float *x, int64_t n, int64_t f, int64_t ld,
             double *out, uint16_t *ord_out, int64_t ld_ord, int32_t *status,
             void *stream);

/* ts_score with an incoming partial sum: when accumulate != 0, out[i] holds
 * the f64 sum of the trees that precede this model's trees in evaluation
 * order and scoring continues from it (acc = out[i]; acc = acc + w*leaf ...),
 * so a tree-sharded ensemble scored shard after shard -- on one GPU or
 * pipelined across GPUs -- reproduces the single-model sum bit for bit. */
int ts_score_ex(const ts_model *model, const float *x, int64_t n, int64_t f, int64_t ld,
                double *out, uint16_t *ord_out, int64_t ld_ord, int32_t *status,
                int accumulate, void *stream);

/* Traced prediction (ref predict_ensemble_traced, evaluators.py:599-620, and
 * measure_feature_coverage, bench.py:412-427) for a device batch: scores
 * (nullable), LOGICAL left-to-right leaf ordinals [T][ld_ord] (nullable) and
 * per-instance visited-feature bitsets visited[n][words] (nullable; bit fid
 * of word fid/32), walking the logical trees (left iff x < theta).  Needs a
 * model packed with TS_PACK_TRACE.  Stream-ordered. */
int ts_trace(const ts_model *model, const float *x, int64_t n, int64_t f, int64_t ld,
             double *out, uint16_t *leaf_ord, int64_t ld_ord, uint32_t *visited,
             int32_t words, void *stream);

/* Fused cross-GPU running-sum pipeline for TREE-SHARDED scoring (BASELINE
 * config 4b), bit-exact: rank r holds trees [t_r, t_{r+1}) and scores all n
 * rows; inside the kernel each 32-row block waits until flags_in[block] ==
 * epoch (set by rank r-1 over NVLink, system-scope acquire), continues the f64
 * sums from sums_in, and when its walk over rank r's trees is done stores the
 * running sums straight into rank r+1's sums_in (a peer pointer from
 * ts_ipc_open) and releases flags_out[block] = epoch.  Transfers overlap the
 * walks block by block; every addition happens in global tree order, so the
 * last rank's `out` equals single-GPU scoring bit for bit.
 *   sums_in / flags_in   NULL on the first rank (start at +0.0)
 *   sums_out / flags_out NULL on the last rank (write `out`)
 *   epoch                increases by one per call (flags are never reset)
 * Needs a model packed as one streaming segment of complete trees
 * (TS_ERR_UNSUPPORTED otherwise).  Calls must be separated by a host barrier
 * across ranks (a rank may not overwrite sums it has not seen consumed). */
typedef struct {
    const double *sums_in;
    const uint32_t *flags_in;
    double *sums_out;
    uint32_t *flags_out;
    uint32_t epoch;
} ts_pipe;

int ts_score_pipe(const ts_model *model, const float *x, int64_t n, int64_t f, int64_t ld,
                  double *out, const ts_pipe *pipe, void *stream);

/* Pipeline receive buffers: f64 sums[n] and u32 flags[ceil(n/32)] (zeroed),
 * as their own cudaMalloc allocations on `device`, with CUDA IPC handles
 * (64 bytes each) for the previous rank to open with ts_ipc_open. */
int ts_pipe_alloc(int device, int64_t n, double **sums, uint32_t **flags,
                  void *sums_handle64, void *flags_handle64);
void ts_pipe_free(double *sums, uint32_t *flags);
int ts_ipc_open(const void *handle64, void **dev_ptr);
void ts_ipc_close(void *dev_ptr);

/* Tree-shard partial scores combined by ONE NCCL f64 sum-reduce to `root`
 * over NVLink / NVSwitch (SURVEY 8(b) ts_reduce_partials; the NCCL
 * equivalent of the reference's sequential sum is exact to ~1e-16 relative,
 * not bit-exact -- ts_score_pipe is the bit-exact alternative).  NCCL is
 * resolved at run time (libnccl.so.2); TS_ERR_UNSUPPORTED without it.
 *   ts_nccl_get_unique_id: on one rank; broadcast the 128 bytes to the others
 *   ts_nccl_comm_init:     every rank, device = its GPU
 *   ts_reduce_partials:    out (valid on root) = sum over ranks of partial[n]
 * A communicator created by the caller's own NCCL (ncclComm_t) may be
 * passed as `comm` as well. */
int ts_nccl_get_unique_id(void *id128);
int ts_nccl_comm_init(const void *id128, int nranks, int rank, int device, void **comm);
int ts_reduce_partials(void *comm, const double *partial, double *out, int64_t n, int root,
                       void *stream);
int ts_nccl_comm_destroy(void *comm);
/* Wait for the collectives enqueued on `stream`, polling
 * ncclCommGetAsyncError meanwhile (SURVEY 5 failure detection): a peer or
 * network failure aborts the communicator (ncclCommAbort, so the stream is
 * released) and returns TS_ERR_CUDA with NCCL's message; so does a wait
 * longer than timeout_ms (< 0: no limit).  ts_reduce_partials also checks
 * the communicator's async state before and after enqueueing. */
int ts_nccl_wait(void *comm, void *stream, int64_t timeout_ms);

/* Host-buffer scoring: same argument meaning as the reference's generated
 * score_batch(x, n, f, out).  Copies x to the device in chunks on two
 * streams (H2D of chunk i+1 overlaps scoring of chunk i), copies the scores
 * back, synchronises.  Pinned host memory gives full PCIe bandwidth; any
 * host memory is accepted.  Returns TS_ERR_NONFINITE (out still written)
 * if x held NaN/inf. */
int ts_score_host(const ts_model *model, const float *x, int64_t n, int64_t f,
                  double *out);

void ts_free(ts_model *model);

/* Thread-local message for the last failing call on this thread. */
const char *ts_last_error(void);

/* Number of scoring-kernel launches issued by this process so far. */
int64_t ts_launch_count(void);

/* Native parser for the text model format (ref model.py:416-602, grammar in
 * the reference SPEC "External Interfaces").  On success *out holds the flat
 * model (nodes in file-id order); on failure it still holds err_line /
 * err_col for TS_ERR_SYNTAX.  Free with ts_flat_free in both cases.
 * Semantic errors return TS_ERR_INVALID with the reference's messages. */
typedef struct {
    int32_t num_features;
    int32_t num_trees;
    int64_t num_nodes;
    int64_t *tree_node_offset;   /* [num_trees + 1] */
    double *tree_weight;         /* [num_trees] */
    int32_t *node_fid;           /* [num_nodes], -1 = leaf */
    float *node_value;
    int32_t *node_left;
    int32_t *node_right;
    int32_t err_line;
    int32_t err_col;
} ts_flat_model;

int ts_parse_model(const char *text, int64_t len, ts_flat_model **out);
void ts_flat_free(ts_flat_model *model);

/* Synthetic instances (BASELINE configs 3/4): fills rows [row0, row0+n) of a
 * counter-based uniform [0,1) matrix in place on the current device, with
 * entries zeroed with probability zero_prob.  Element e = row*f + col takes
 * u = splitmix64(seed + (e+1)*0x9E3779B97F4A7C15) >> 40, scaled by 2^-24
 * (reproducible on the host).  Not part of the reference interface. */
int ts_synth_uniform(float *x, int64_t n, int64_t f, int64_t ld, uint64_t seed,
                     int64_t row0, double zero_prob, void *stream);

/* Kernel-path selector for parity tests and A/B timing: 0 = automatic
 * (shared-memory streaming kernel when the tables fit, else the L1 path),
 * 1 = always the L1 (global-read) kernels.  Process-wide; takes effect for
 * models packed after the call (the choice fixes the table layout). */
int ts_set_kernel_path(int path);

/* Library version string, e.g. "0.1.0 sm_100a". */
const char *ts_version(void);

#ifdef __cplusplus
}
#endif

#endif /* TREESCORE_GPU_H */
