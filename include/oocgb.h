/*
 * oocgb.h — C ABI of the B200 (sm_100a) hot path of "Out-of-Core GPU Gradient Boosting"
 * (R. Ou, arXiv 2005.09148).  Library: paper_2005_09148_b200/liboocgb.so.
 *
 * Calls follow the paper's statement of the problem (BASELINE.json north_star):
 *   quantise(X, max_bin) -> ELLPACK pages      Alg. 2-5
 *   set_gradients(g, h)                        Eq. 4-5
 *   sample(ratio, mode)                        Alg. 7; SGB L212-220; MVS Eq. 9
 *   build_tree(depth, lambda, gamma)           Alg. 1; Eq. 6; Eq. 8
 *   predict                                    Eq. 1
 * Readings of the paper where it is silent are numbered R1..R24 in DESIGN.md §3.
 *
 * Conventions (all calls):
 *  - Every call returns an oocgb_status.  On failure oocgb_last_error() returns a
 *    thread-local, human-readable message; no handle is modified except as documented.
 *  - Pointers to caller data (X, g, h, margin, labels) may be HOST or DEVICE pointers
 *    (distinguished with cudaPointerGetAttributes); they are borrowed for the duration of the
 *    call only.  Anything the library keeps, it copies.  Host output buffers are caller-
 *    allocated with the sizes stated per call.
 *  - All device work is ordered on the context's stream.  A call that reads or writes HOST
 *    buffers returns when they may be reused / read; a call whose caller buffers are all DEVICE
 *    pointers is stream-ordered (it may return before the device work finishes; the next call,
 *    or any work the caller enqueues on the same stream, sees its results).  oocgb_build_tree
 *    and oocgb_sample with a non-NULL info always synchronise (their outputs live on the host).
 *  - Handles are library-owned; free them with the matching *_destroy.
 *  - One owner thread per context (not thread-safe); exported trees are immutable.
 */
#ifndef OOCGB_H
#define OOCGB_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  OOCGB_OK = 0,
  OOCGB_ERR_ARG = 2,     /* bad argument: sizes, ranges, non-finite X, call-order misuse of args */
  OOCGB_ERR_NOMEM = 3,   /* device or pinned-host allocation failed (lower `ratio`)     */
  OOCGB_ERR_DEVICE = 4,  /* CUDA or NCCL failure; message carries the error string             */
  OOCGB_ERR_STATE = 5    /* call-order violation (e.g. build_tree before sample)               */
} oocgb_status;

typedef struct oocgb_ctx_s *oocgb_ctx;   /* one per process == one GPU                        */
typedef struct oocgb_data_s *oocgb_data; /* cuts + ELLPACK pages + per-round row state         */
typedef struct oocgb_tree_s *oocgb_tree; /* one regression tree f_k (Eq. 1) + debug dumps      */

enum { OOCGB_PLACE_DEVICE = 0, OOCGB_PLACE_PINNED_HOST = 1 };
enum { OOCGB_SAMPLE_NONE = 0, OOCGB_SAMPLE_UNIFORM = 1, OOCGB_SAMPLE_MVS = 2, OOCGB_SAMPLE_GOSS = 3 };

/* Exported tree node, heap order: children of i are 2i+1 (left: bin <= split_bin, i.e.
 * x <= split_value) and 2i+2.  feature = -1 leaf, -2 absent slot below a leaf.
 * default_left (R27): a row MISSING the split feature goes left (1) or right (0); always 0 for
 * data without missing values.
 * leaf_value = (float)(eta * -G/(H+lambda)) (Eq. 6, R15) is set for every present node.
 * sum_g/sum_h are the node's dequantised gradient sums over the SAMPLED rows (scaled by
 * 1/p); n_rows the number of sampled rows in the node, summed over all ranks.           */
typedef struct {
  int32_t feature;
  int32_t split_bin;
  float split_value;
  float leaf_value;
  double gain;
  double sum_g;
  double sum_h;
  int64_t n_rows;
  int32_t default_left;
  int32_t pad;
} oocgb_node;

typedef struct {
  int64_t n_rows_local;   /* rows held by this rank                                           */
  int64_t n_rows_global;  /* rows over all ranks                                             */
  int64_t row0_global;    /* global id of this rank's first row                              */
  int32_t n_features;     /* m                                                               */
  int32_t row_stride;     /* bytes per ELLPACK row = 32 ceil(m / 32) (R5; tiled pages)        */
  int32_t max_bin;
  int32_t placement;      /* OOCGB_PLACE_*                                                   */
  int64_t n_pages;        /* ELLPACK pages (1 for a single device page)                      */
  int64_t rows_per_page;  /* floor(page_bytes / row_stride), last page holds the remainder   */
  int64_t total_cuts;     /* sum_j B_j                                                       */
  int32_t has_missing;    /* R27: some value is missing (NaN / absent CSR entry), symbol 255  */
  int32_t pad;
} oocgb_info;

typedef struct {
  int64_t n_selected_local;
  int64_t n_selected_global;
  int64_t k_star;         /* MVS: rows forced to p = 1 (-1 when every non-zero row has p = 1) */
  double mu;              /* MVS threshold (R9), 0 when unused                               */
  int32_t e_g, e_h;       /* fixed-point exponents (R12): q = rint(x 2^e)                     */
  int32_t e_prime;        /* MVS: g_hat quantisation exponent                                */
  int32_t fallback_uniform; /* MVS with all g_hat == 0 fell back to uniform        */
} oocgb_sample_info;

/* ---- context ------------------------------------------------------------------------------
 * oocgb_nccl_unique_id: rank 0 creates the NCCL id; the caller broadcasts the 128 bytes
 * (e.g. with torch.distributed) and passes them to oocgb_ctx_create on every rank.
 * oocgb_ctx_create: binds `device`; rank/world describe the row sharding (the
 * histograms are "summed across all GPUs"; here a reduce-scatter by feature slice, each rank
 * evaluates its slice and the candidates are all-gathered).  nccl_id may be NULL iff
 * world == 1; world == 1 WITH an nccl_id runs the multi-GPU code path (every exchange step
 * through NCCL) on a 1-rank communicator, results identical to the plain context (tests).  cuda_stream: a cudaStream_t cast to uint64 to order work on, 0 = library
 * creates its own non-blocking stream.  ERR_ARG on rank/world mismatch; ERR_DEVICE on
 * CUDA/NCCL init failure.  oocgb_ctx_destroy returns ERR_STATE while data handles are alive. */
int oocgb_nccl_unique_id(uint8_t out[128]);
int oocgb_ctx_create(int32_t device, int32_t rank, int32_t world, const uint8_t *nccl_id,
                     uint64_t cuda_stream, oocgb_ctx *out);
int oocgb_ctx_destroy(oocgb_ctx ctx);

/* Test-only transport for the exchange steps (several ranks sharing one GPU, or no NCCL):
 * every collective is run as: synchronise the ctx stream, copy the device buffer to host,
 * call fn, copy back (a reduce-scatter is an all-reduce sum of every block, then the rank keeps
 * its own).  op: 0 all-reduce sum, 1 all-reduce max, 2 all-gather (buf holds
 * world * count elements, this rank's block at rank * count); dtype: 0 int64, 1 uint64,
 * 2 uint32.  fn returns 0 on success.  The compute path is unchanged (all kernels on the GPU);
 * build_tree is not graph-captured in this mode.  ERR_ARG if fn is NULL or world < 1.       */
typedef int (*oocgb_collective_fn)(int32_t op, int32_t dtype, void *buf, int64_t count, void *user);
int oocgb_ctx_create_hostcomm(int32_t device, int32_t rank, int32_t world, oocgb_collective_fn fn,
                              void *user, uint64_t cuda_stream, oocgb_ctx *out);

/* ---- quantise: Alg. 2 (in-core sketch) + Alg. 4 (ELLPACK page), PAPER.md L256-318 ---------
 * X: float32 row-major [n_rows][n_features], this rank's rows, global ids
 * row0_global .. row0_global+n_rows-1 of n_rows_global in total.  max_bin in [2, 256]
 * (P:L157-158 default 256).  Cuts (R1-R4): exact rank cuts over a global-row-keyed Philox
 * sketch sample of <= 2^20 rows (all rows when n_rows_global <= 2^20), seed = `seed`.
 * page_bytes: ELLPACK page size (P:L326 uses 32 MiB); 0 = one page.  placement DEVICE keeps
 * the pages in HBM; PINNED_HOST keeps them in pinned host memory (out-of-core, Alg. 5 with
 * disk replaced by host RAM).  Missing values (R27; the paper's pages are CSR):
 * NaN marks a missing value; the cuts skip it, its symbol is 255 (so data with missing values
 * needs max_bin <= 255) and every split learns a default direction for it.  Errors: ERR_ARG
 * (sizes, max_bin, +-inf in X, missing values with max_bin 256), ERR_NOMEM.                */
int oocgb_quantise(oocgb_ctx ctx, const float *X, int64_t n_rows, int64_t row0_global,
                   int64_t n_rows_global, int32_t n_features, int32_t max_bin,
                   int64_t page_bytes, int32_t placement, uint64_t seed, oocgb_data *out);

/* Sparse CSR input (R27; "the training data is already parsed and written to disk
 * in CSR pages"): row i of this rank holds values[indptr[i] .. indptr[i+1]) at feature indices
 * indices[...] (each < n_features, no repeats within a row); absent entries are MISSING.
 * indptr int64 [n_rows + 1] (indptr[0] may be non-zero: it is subtracted), indices int32 and
 * values float32 [nnz]; host or device pointers.  Same cuts, pages and errors as
 * oocgb_quantise on the dense matrix with NaN at the absent entries (bit-identical).       */
int oocgb_quantise_csr(oocgb_ctx ctx, const int64_t *indptr, const int32_t *indices, const float *values,
                       int64_t n_rows, int64_t row0_global, int64_t n_rows_global, int32_t n_features,
                       int32_t max_bin, int64_t page_bytes, int32_t placement, uint64_t seed,
                       oocgb_data *out);

/* Streamed quantise (Alg. 3 + Alg. 5): sketch_begin, any number of sketch_push (pass 1, rows
 * in any order, each row pushed once), cuts_finalize, then pages_push with the rows in
 * ascending global order (pass 2).  X batches may be host or device pointers.             */
int oocgb_sketch_begin(oocgb_ctx ctx, int32_t n_features, int32_t max_bin, int64_t n_rows,
                       int64_t row0_global, int64_t n_rows_global, int64_t page_bytes,
                       int32_t placement, uint64_t seed, oocgb_data *out);
int oocgb_sketch_push(oocgb_data data, const float *X, int64_t row0_global, int64_t n);
int oocgb_cuts_finalize(oocgb_data data);
int oocgb_pages_push(oocgb_data data, const float *X, int64_t row0_global, int64_t n);

/* Bin held-out rows with the cuts of `ref` (no sketch), e.g. for predict + AUC.          */
int oocgb_quantise_like(oocgb_data ref, const float *X, int64_t n_rows, int32_t placement,
                        oocgb_data *out);
int oocgb_data_info(oocgb_data data, oocgb_info *out);
int oocgb_data_destroy(oocgb_data data);

/* ---- per-round calls ------------------------------------------------------------------------
 * set_gradients (Eq. 5): g, h float32 [n_local] (host or device), copied in.  Invalidates
 * any previous sample.  ERR_ARG on a length mismatch.                                      */
int oocgb_set_gradients(oocgb_data data, const float *g, const float *h, int64_t n_local);

/* Harness helper (binary:logistic, Eq. 5): g = sigmoid(m) - y, h = sigmoid(m)(1 - sigmoid(m))
 * computed on the device from margin/labels [n_local] and stored as the gradients, exactly
 * like set_gradients(g, h).  margin/labels host or device.                                  */
int oocgb_set_logistic_gradients(oocgb_data data, const float *margin, const float *labels,
                                 int64_t n_local);

/* sample (Alg. 7, R9-R12): mode NONE (all rows), UNIFORM (SGB, Bernoulli(f), scale 1),
 * MVS (Eq. 9, capped PPS with an exact integer threshold, g' = g/p, h' = h/p).  Random draws
 * are Philox4x64-10 keyed (seed, round) with counter (global_row, 0, 0, 0) (R24), so the
 * sample is independent of world size and page size.  Then fixed point (R12):
 * q = rint(x 2^e), e = quant_bits - k with frexp(max|x|) = (., k); quant_bits in [8, 20] (R12: non-returning s32 shared atomics need chunk_rows * 2^quant_bits < 2^31).
 * For PINNED_HOST data this also compacts the selected rows of every page into one device
 * page (Alg. 7).  ERR_ARG: ratio not in (0, 1], bad mode/quant_bits; ERR_STATE:
 * no gradients; ERR_NOMEM: sampled page does not fit (lower ratio).  info may be NULL: then
 * the f = 1 in-core path runs without any host synchronisation.                           */
int oocgb_sample(oocgb_data data, int32_t mode, double ratio, double mvs_lambda, uint64_t seed,
                 uint64_t round, int32_t quant_bits, oocgb_sample_info *info);

/* GOSS (R25): the round(a n) rows with the largest |g| (quantised like MVS's g_hat;
 * ties at the threshold all included) are kept with p = 1; every other row is drawn
 * Bernoulli(p_rest), p_rest = rint(b 2^32) / (2^32 - rint(a 2^32)), and scaled by 1 / p_rest
 * (= (1-a)/b, "to make the gradient statistics unbiased").  Same Philox draws, fixed point and
 * compaction as oocgb_sample.  ERR_ARG unless 0 <= a, 0 < b, a + b <= 1.  info->k_star = the top
 * count round(a n), info->mu = p_rest.                                                        */
int oocgb_sample_goss(oocgb_data data, double a, double b, uint64_t seed, uint64_t round,
                      int32_t quant_bits, oocgb_sample_info *info);

/* Alg. 6: with enable != 0, an f = 1 sample (mode NONE)
 * of PINNED_HOST data is NOT copied to the device; build_tree then streams the pinned pages once
 * per level (batches of ~1 GB, copy/compute overlapped) and builds every node's histogram
 * directly (no sibling subtraction).  The tree is identical to the in-core one.
 * Samples with f < 1 keep using Alg. 7 (compaction).  ERR_ARG unless PINNED_HOST; one GPU.   */
int oocgb_set_streaming(oocgb_data data, int32_t enable);

/* build_tree (Alg. 1, depth-wise R16): histograms (fixed-point int, bit-exact), sibling
 * subtraction (R17), split evaluation (Eq. 8, R13-R14), partition (set semantics, R26), leaf values
 * (Eq. 6, eta applied at creation R15).  max_depth in [0, 16]; lambda >= 0; the tree is
 * written to *out.  keep_debug != 0 keeps per-node histograms and the final partition for
 * oocgb_get_histogram / oocgb_get_partition (memory: 2^D * m * 4 KB).  ERR_STATE before
 * oocgb_sample; ERR_ARG if H + lambda <= 0 at a node.                                      */
int oocgb_build_tree(oocgb_data data, int32_t max_depth, double lambda, double gamma,
                     double min_child_weight, double eta, int32_t keep_debug, oocgb_tree *out);
int oocgb_tree_export(oocgb_tree tree, oocgb_node *nodes, int32_t capacity, int32_t *n_nodes);
int oocgb_tree_destroy(oocgb_tree tree);

/* predict (Eq. 1): margin_inout[i] (float32) += leaf(tree_k, bins_i) for each of the
 * n_trees trees, this rank's rows, traversing the binned rows (bin <= split_bin -> left).
 * margin_inout: host or device float32 [n_local].  Works on DEVICE and PINNED_HOST data
 * (pages streamed).                                                                        */
int oocgb_predict(oocgb_data data, const oocgb_tree *trees, int32_t n_trees, float *margin_inout);

/* Fast margin update for the tree just built from THIS data's current sample (in-core,
 * f = 1): margin[row] += leaf via the final partition (12 B/row instead of a traversal).
 * ERR_STATE if the sample did not select every row or the tree is not the latest.       */
int oocgb_update_margin(oocgb_data data, oocgb_tree tree, float *margin_inout);

/* ---- parity dumps (caller-allocated HOST buffers) --------------------------------------- */
int oocgb_get_cuts(oocgb_data data, float *values /*total_cuts*/, int32_t *offsets /*m+1*/);
int oocgb_get_bins(oocgb_data data, int64_t row0_local, int64_t n, uint8_t *out /*n*stride*/);
/* selected rows (global ids, ascending) and their fixed-point (q_g, q_h)                   */
int oocgb_get_sample(oocgb_data data, int64_t *gid, int64_t *q_g, int64_t *q_h);
/* node's histogram, int64 [m][256][2] (g, h), summed over ranks; needs keep_debug         */
int oocgb_get_histogram(oocgb_tree tree, int32_t node, int64_t *gh);
/* leaf_of_row[n_selected_local]: heap index of the final node of each selected row, in the
 * order of oocgb_get_sample; needs keep_debug                                              */
int oocgb_get_partition(oocgb_tree tree, int32_t *leaf_of_row);
/* row_order[n_selected_local]: the final partition as positions -> selected-row index (order of
 * oocgb_get_sample).  RepartitionInstances (Alg. 1) lays every split's left child before
 * its right child, so the rows of each leaf form one contiguous block and the blocks come in
 * left-first depth-first order; the order inside a block is unspecified (R26).  In-core
 * builds only (ERR_STATE for an Alg. 6 streamed tree); needs keep_debug.                       */
int oocgb_get_row_order(oocgb_tree tree, int32_t *row_order);

/* Per-phase device timings of the last call (CUDA events on the ctx stream), milliseconds:
 * [0] histogram kernels, [1] split evaluation, [2] partition, [3] sample+quantise,
 * [4] predict, [5] page streaming (H2D), [6] whole build_tree, [7] histogram kernel launches,
 * [8] algorithmic histogram bytes of the last build_tree.  n = capacity.                */
int oocgb_get_timings(oocgb_ctx ctx, double *out, int32_t n);
int oocgb_set_profiling(oocgb_ctx ctx, int32_t enable);

const char *oocgb_last_error(void);
int32_t oocgb_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* OOCGB_H */
