// Internal declarations of liboocgb (B200 / sm_100a).  Not part of the ABI (include/oocgb.h).
// Citations: "P:Lx" = PAPER.md line, "Rk" = reading k in DESIGN.md §3.
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>
#include <stdint.h>

#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/oocgb.h"

namespace oocgb {

// ---------------------------------------------------------------------------------------------
// Errors: thrown inside the library, turned into a status code + thread-local message at the
// C-ABI boundary (api.cu).
struct Error : std::runtime_error {
  int status;
  Error(int s, const std::string &m) : std::runtime_error(m), status(s) {}
};

#define OOCGB_CK(call)                                                                       \
  do {                                                                                       \
    cudaError_t e_ = (call);                                                                 \
    if (e_ != cudaSuccess) {                                                                 \
      int st_ = (e_ == cudaErrorMemoryAllocation) ? OOCGB_ERR_NOMEM : OOCGB_ERR_DEVICE;      \
      throw ::oocgb::Error(st_, std::string(#call) + ": " + cudaGetErrorString(e_) + " @" + \
                                    __FILE__ + ":" + std::to_string(__LINE__));             \
    }                                                                                        \
  } while (0)

// NCCL is loaded lazily with dlopen("libnccl.so.2") (nccl_api() in api.cu) so that a process
// that never goes multi-GPU never loads it, and a process that imported torch first binds to
// torch's NCCL instead of a second copy.
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId *);
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t);
  ncclResult_t (*ReduceScatter)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
  const char *(*GetErrorString)(ncclResult_t);
};
const NcclApi &nccl_api();

#define OOCGB_NCCL(call)                                                                     \
  do {                                                                                       \
    ncclResult_t r_ = (call);                                                                \
    if (r_ != ncclSuccess)                                                                   \
      throw ::oocgb::Error(OOCGB_ERR_DEVICE, std::string(#call) + ": " + ::oocgb::nccl_api().GetErrorString(r_)); \
  } while (0)

#define OOCGB_REQUIRE(cond, status, msg)                                                     \
  do {                                                                                       \
    if (!(cond)) throw ::oocgb::Error((status), (msg));                                      \
  } while (0)

// ---------------------------------------------------------------------------------------------
// Tuning constants.
constexpr int kFG = 32;              // features per histogram feature-group (one 32 B sector)
constexpr int kBins = 256;           // uint8 symbols (R5, R7)
#ifndef OOCGB_HIST_THREADS
#define OOCGB_HIST_THREADS 512
#define OOCGB_HIST_CTAS 2
#define OOCGB_HIST_DEPTH 3
#endif
constexpr int kHistThreads = OOCGB_HIST_THREADS;  // histogram CTA (512 x 2 per SM: 32 warps, measured best)
constexpr int kHistCtasPerSm = OOCGB_HIST_CTAS;
constexpr int kHistDepth = OOCGB_HIST_DEPTH;      // k_hist's register pipeline depth (rows in flight per lane)
constexpr int kHistSmem = 2 * kBins * kFG * 4;  // s32 [bin][g: 32 features | h: 32 features]
constexpr int kPartTile = 2048;      // positions per partition tile
constexpr int kPartThreads = 256;

// Device node record (heap order).  G/H keep the exact fixed-point sums.
struct DNode {
  int32_t feature;     // -2 absent, -1 leaf, >= 0 split feature
  int32_t split_bin;
  float split_value;
  float leaf_value;
  double gain;
  double sum_g, sum_h;
  long long n_rows;    // global sampled rows
  long long Gq, Hq;    // fixed-point sums (global)
  int32_t default_left;  // R27: missing values (symbol 255) go left
  int32_t seg;           // the node's segment index at its level (set by the plan that creates it)
  double tP;             // G^2 / (H + lambda) of the node (Eq. 8's parent term), set with the sums
};

// Row segment of the partition at one depth (pass-through segments carry leaves).
struct Seg {
  int32_t begin, count;  // local positions
  int32_t node;          // heap index
  int32_t dec;           // the node's split at this level, written by k_finalize: -1 none, else
                         // feature << 10 | default_left << 9 | split_bin (the partition's one read)
};
__host__ __device__ __forceinline__ int seg_dec(int feature, int default_left, int split_bin) {
  return (feature << 10) | (default_left << 9) | split_bin;
}

// Sibling pair built at a level: `built` gets a histogram from rows, `derived` = parent - built.
struct Pair {
  int32_t parent;      // heap id (-1 at the root level)
  int32_t built;       // heap id
  int32_t derived;     // heap id (-1 at the root level)
  int32_t begin;       // local positions of the built child's rows
  int32_t count;
  int32_t chunk_base;  // first global chunk of this pair
  int32_t n_chunks;
  int32_t chunk_rows;
  int32_t compact;     // bit 0: parent, bit 1: built, bit 2: derived histogram kept as s32 pairs
  int32_t pad[3];
};

// Best split candidate of one (node, feature).
struct Cand {
  double gain;
  int32_t bin;         // candidate key 2 b + dir (dir 1: missing values left, R27)
  int32_t valid;
  long long GL, HL;
};

// Device-resident result of oocgb_sample (R12): fixed-point exponents, root sums, counts.
// Written by the sample kernels, read by build_tree's first kernel — no host round trip.
struct SampleState {
  unsigned long long maxbits[2];  // max |g'|, max |h'| as double bit patterns (all ranks)
  long long G, H;                 // fixed-point root sums (all ranks)
  long long n_sel_local, n_sel_global;
  int e_g, e_h, quant_bits, pad;
};

struct LevelCtl {       // device-resident control block of one build
  int n_pairs;
  int n_items;
  int n_segs;
  int n_splits;         // splits decided at the current level
  int error;            // 1: H + lambda <= 0 at a node
  int part_done;        // partition tiles finished (last-block ticket), reset by the last block
  int hist_next;        // k_hist dynamic item counter, zeroed by whoever writes the level's chunk plan
  int n_ew, n_en;       // eval work lists: (pair, side) entries of nodes with > kmax / <= kmax rows
  unsigned bar_count;   // k_partition's grid barrier: arrivals of the current generation
  unsigned bar_gen;     // and its generation counter
};

// Histogram chunk size (rows) for a level with tot_rows built rows in n_pairs pairs, k_hist run
// by `grid` persistent CTAs over (chunk, feature group) items: the smallest number of waves w
// such that C = floor(w grid / n_fg) >= 2 n_pairs - 1 chunks of at most kmax rows (the s32 bound) hold every pair
// (sum_p ceil(count_p / cr) <= tot/cr + n_pairs - n_pairs/cr < C + 1 with cr = ceil(tot / (C -
// n_pairs + 1))), so the items fill w whole waves (config 2 root: 37 equal chunks = 2 x 296 items
// instead of 31 chunks = 1.68 waves).
__host__ __device__ __forceinline__ long long hist_chunk_rows(long long tot, int n_pairs, int n_fg, int grid,
                                                               long long kmax) {
  const long long lo = kmax < 1024 ? kmax : 1024;
  if (tot <= 0) return lo;
  for (long long w = 1;; ++w) {
    const long long C = w * grid / n_fg;
    // C >= 2 n_pairs - 1 keeps the largest chunk within ~2x the mean (cr <= tot / (C / 2)): a
    // level with one big pair among many small ones (config 2 level 5: 39k rows + 15 pairs of
    // < 5k) would otherwise get few huge chunks and a one-item straggler wave
    if (C < 2LL * n_pairs - 1 || C < 1) continue;
    const long long cr = (tot + (C - n_pairs + 1) - 1) / (C - n_pairs + 1);
    if (cr <= kmax) return cr < lo ? lo : cr;
  }
}

// byte offset of symbol (row, f) in a tiled ELLPACK buffer of pages of rpp rows, planes of gw
// bytes (gw = 64: features 64 P .. 64 P + 63 of a row are one 64-B DRAM burst, R5)
__host__ __device__ __forceinline__ size_t ell_off(int64_t row, int f, int64_t rpp, int gw, int stride) {
  const int64_t p = row / rpp, r = row - p * rpp;
  return (size_t)p * (size_t)rpp * stride + (size_t)(f / gw) * (size_t)rpp * gw + (size_t)r * gw + (size_t)(f % gw);
}
// plane width of a data set.  64-B planes (features 64 P .. 64 P + 63 of a row = one DRAM burst)
// halve k_hist's DRAM bytes below the root (1.22x -> 0.99x the algorithmic bytes per round) but
// were measured slower on B200: every 16-row warp load of a 32-feature item touches
// 8 instead of 4 L1 lines (root +13 us, L1-pipe bound), and the partition's 1-byte gathers fetch a
// burst of one row instead of two useful rows' sectors (+2.5 us per level).  OOCGB_PLANE_64 = 1
// selects them (every kernel is layout-generic).
#ifndef OOCGB_PLANE_64
#define OOCGB_PLANE_64 0
#endif
__host__ __device__ __forceinline__ int plane_width(int n_fg) { return (OOCGB_PLANE_64 && n_fg >= 2) ? 64 : 32; }

struct PNode {          // compact node for predict
  int32_t feature;
  int32_t split_bin;
  float leaf;
  int32_t default_left;  // R27
};

// RepartitionInstances / predict rule (R27): symbol 255 of data with missing values follows the
// node's default direction; every other symbol goes left iff bin <= split_bin (for data without
// missing values default_left is 0, so the rule reduces to bin <= split_bin)
__host__ __device__ __forceinline__ bool goes_left(int b, int split_bin, int default_left) {
  return b <= split_bin || (b == 255 && default_left);
}

}  // namespace oocgb

// ---------------------------------------------------------------------------------------------
// Opaque handle structs.
struct oocgb_ctx_s {
  int device = 0, rank = 0, world = 1;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  cudaStream_t copy_stream = nullptr;
  ncclComm_t comm = nullptr;
  bool coll = false;  // collectives on: world > 1, or a 1-rank NCCL communicator (nccl_id given)
  oocgb_collective_fn host_coll = nullptr;  // test transport (oocgb_ctx_create_hostcomm)
  void *host_coll_user = nullptr;
  int live_data = 0;
  int live_trees = 0;
  bool mvs_attr = false;  // k_mvs_decide's dynamic shared memory attribute set on this device
  // page-pipeline events (stream.cuh), created with the ctx on its device
  cudaEvent_t pipe_copy_done[3] = {}, pipe_consumed[3] = {};
  int num_sms = 148;
  bool profiling = false;
  double timings[16] = {0};
  std::vector<cudaEvent_t> ev_pool;          // recycled events
  std::vector<int> pending_slot;             // (slot, event a, event b) recorded, not yet read
  std::vector<cudaEvent_t> pending_a, pending_b;
  std::vector<std::pair<size_t, void *>> node_pool;  // recycled tree node buffers (no cudaFree sync)
  // scratch for small host<->device exchanges
  void *d_small = nullptr;   // 1 MB device scratch
  void *h_small = nullptr;   // 1 MB pinned scratch
};

struct oocgb_data_s {
  oocgb_ctx ctx = nullptr;
  int64_t n_local = 0, n_global = 0, row0 = 0;
  int32_t m = 0, stride = 0, max_bin = 256, placement = OOCGB_PLACE_DEVICE;
  int32_t n_fg = 0;                // feature groups of 32 (the histogram's items)
  int32_t gw = 32;                 // tiled plane width in bytes (32 or 64), stride = gw * planes
  int64_t rows_per_page = 0, n_pages = 1;
  uint64_t seed = 0;
  // cuts (R1-R4)
  float *d_cut_values = nullptr;
  int32_t *d_cut_ptrs = nullptr;
  std::vector<float> h_cut_values;
  std::vector<int32_t> h_cut_ptrs;
  bool cuts_ready = false;
  bool has_missing = false;     // R27: some value was missing (NaN / absent CSR entry)
  int *d_missing = nullptr;     // device flag set by the binning kernel
  // ELLPACK (R5-R6)
  // Tiled ELLPACK (R5): pages of rows_per_page rows; inside a page the symbols of
  // feature group g (features 32g..32g+31) of all the page's rows are contiguous:
  //   offset(row, f) = page * (rpp * stride) + (f / gw) * (rpp * gw) + (row % rpp) * gw + f % gw
  uint8_t *d_bins = nullptr;    // DEVICE placement: one tiled page, rpp = n_local
  // PINNED_HOST placement: ROW-MAJOR [n_local][stride] (a row is one contiguous block, so pages
  // stream as plain row ranges and selected rows can be gathered zero-copy over PCIe); the
  // device-side sampled page built from it is tiled.
  uint8_t *h_pages = nullptr;
  int64_t rows_written = 0;     // streamed pages_push progress
  // streamed sketch state
  uint32_t *d_sketch = nullptr; // column-major ordered keys [m][cap]
  int64_t sketch_cap = 0;
  unsigned long long *d_sketch_count = nullptr;
  bool sketch_all_rows = true;
  // gradients
  float *d_g = nullptr, *d_h = nullptr;
  bool has_grad = false;
  // sample
  bool has_sample = false;
  bool all_selected = false;
  int64_t n_sel = 0, n_sel_global = 0;
  int32_t *d_sel_rows = nullptr;   // local row ids, ascending
  int2 *d_q = nullptr;             // (q_g, q_h), |q| <= 2^quant_bits
  int32_t e_g = 0, e_h = 0, quant_bits = 16;
  long long G_root = 0, H_root = 0;   // host mirrors, valid after a synchronising sample
  oocgb::SampleState *d_ss = nullptr; // device sample state (always valid after sample)
  oocgb::SampleState *h_ss = nullptr; // pinned mirror
  uint8_t *d_sampled_page = nullptr;  // PINNED_HOST: compacted selected rows (Alg. 7)
  int64_t sampled_cap = 0;
  int64_t sel_cap = 0;
  double *d_gs = nullptr, *d_hs = nullptr;  // scaled g', h' of the selected rows
  long long *d_tmp64 = nullptr;             // MVS g_hat / q64 [n_local]
  float *d_absparts = nullptr;              // f = 1, one rank: per-block max |g|, |h| (k_absmax2)
  void *d_mvs = nullptr;                    // MVS device threshold state (sample.cu MvsDev)
  unsigned long long *d_mvs_stats = nullptr;  // its per-bucket (count, sum, max) [3][2048]
  int64_t tmp_cap = 0;
  // tree workspace (lazy, sized for (n_sel cap, depth))
  struct Work *work = nullptr;
  uint64_t tree_serial = 0;
  uint64_t sample_serial = 0;   // bumped by every sample / set_streaming: trees remember theirs
  // Alg. 6 streamed build (f = 1, PINNED_HOST): trees are built by level-batched passes over the
  // pinned pages instead of copying every page into HBM
  bool streamed = false;
  int64_t stream_batch_rows = 0;
  int32_t *streamed_row_node = nullptr;  // final leaf of every row after a streamed build
  uint8_t *d_bstage[3] = {nullptr, nullptr, nullptr};
  // persistent device staging for host-pointer arguments (margin, labels): no per-call malloc
  void *d_arg[2] = {nullptr, nullptr};
  size_t arg_bytes[2] = {0, 0};
  // staging for streamed pages
  uint8_t *d_stage[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t stage_ev[3] = {};
  int64_t stage_rows = 0;
};

struct oocgb_tree_s {
  oocgb_data owner = nullptr;
  oocgb_ctx ctx = nullptr;
  size_t pnodes_bytes = 0;
  uint64_t serial = 0;
  uint64_t sample_serial = 0;        // the data's sample this tree was built from
  int32_t max_depth = 0;
  std::vector<oocgb_node> nodes;
  oocgb::PNode *d_pnodes = nullptr;  // device copy for predict
  bool debug = false;
  std::vector<long long> hist;       // [2^D - 1][m][256][2]
  std::vector<int32_t> leaf_of_row;  // selected order
  std::vector<int32_t> row_order;    // final partition: position -> selected-order index
  bool has_row_order = false;
};

namespace oocgb {

// ---------------------------------------------------------------------------------------------
// Host-side launchers, one per kernel family (quantise.cu, sample.cu, tree.cu).
void set_last_error(const std::string &msg);
void *dmalloc(size_t bytes);
void *pool_get(oocgb_ctx c, size_t bytes);   // device buffer from the ctx pool (or cudaMalloc)
void pool_put(oocgb_ctx c, size_t bytes, void *p);
void dfree(void *p);
bool is_device_ptr(const void *p);

// quantise.cu
void sketch_append(oocgb_data d, const float *dX, int64_t row0_global, int64_t n);
void cuts_finalize(oocgb_data d);
void bin_rows(oocgb_data d, const float *dX, int64_t n, int64_t row_local0, uint8_t *out_base, int *d_err);
void csr_to_dense(oocgb_ctx c, const int64_t *d_indptr, const int32_t *d_indices, const float *d_values,
                  int64_t base, int64_t r0, int64_t nr, int m, float *d_out, int *d_err);

// sample.cu
void logistic_gradients(oocgb_data d, const float *d_margin, const float *d_labels);
void sample_rows(oocgb_data d, int mode, double ratio, double mvs_lambda, uint64_t seed,
                 uint64_t round, int quant_bits, oocgb_sample_info *info, double goss_b = 0.0);

// tree.cu
oocgb_tree build_tree(oocgb_data d, int max_depth, double lambda, double gamma, double mcw,
                      double eta, bool keep_debug);
oocgb_tree build_tree_streamed(oocgb_data d, int max_depth, double lambda, double gamma, double mcw,
                               double eta, bool keep_debug);
void predict_device(oocgb_data d, const uint8_t *d_bins, size_t row_step, size_t pitch, int lgw, int64_t n_rows,
                    int64_t row_offset,
                    const oocgb_tree *trees, int n_trees, float *d_margin);
void update_margin(oocgb_data d, oocgb_tree t, float *d_margin);
void free_work(oocgb_data d);


// NCCL helpers (no-ops when world == 1)
void allreduce_sum_i64(oocgb_ctx c, long long *d_buf, size_t count);
void allreduce_max_u64(oocgb_ctx c, unsigned long long *d_buf, size_t count);
void allgather_u32(oocgb_ctx c, const uint32_t *d_send, uint32_t *d_recv, size_t count);
// in place: buf holds world blocks of `count` int64, this rank's block filled (P:L188-190 exchange)
void allgather_i64_inplace(oocgb_ctx c, long long *d_buf, size_t count);
// send holds world blocks of `count` int64; recv gets the sum over ranks of this rank's block
void reduce_scatter_i64(oocgb_ctx c, const long long *d_send, long long *d_recv, size_t count);

// profiling: when ctx->profiling, records an event pair around a phase on the ctx stream
// (no synchronisation); oocgb_get_timings() later sums the elapsed times into timings[slot].
struct PhaseTimer {
  oocgb_ctx c;
  int slot;
  cudaEvent_t a = nullptr;
  PhaseTimer(oocgb_ctx c_, int s);
  ~PhaseTimer();
};
void drain_timers(oocgb_ctx c);

}  // namespace oocgb
