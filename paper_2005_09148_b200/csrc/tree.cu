// Tree construction (Alg. 1) for sm_100a, depth-wise (R16):
//   per level d:  k_hist (BuildHistograms, L174-175)      -> s32 partial histograms
//                 [multi-GPU: k_reduce_partials + ncclAllReduce(int64), P:L188-190]
//                 k_eval, k_eval_narrow (EvaluateSplit, L176-178; Eq. 8) -> per-(node, feature)
//                          best split over the plan's int64 / int32 work lists, sibling =
//                          parent - built (R17), parents kept for the next level
//                 k_finalize (node decision: argmax over features,
//                          Eq. 6 leaf values, R13-R15)
//                 k_part_fused / k_part_plan (RepartitionInstances, L172-173):
//                          one pass: per-(tile, node) atomic reservations, left rows forward,
//                          right rows backward; gradient pairs travel with rows
// Everything stays on the device: one host sync per tree (the export).
//
// Histogram kernel design (measured in tools/microbench):
//  * s32 shared accumulators in a bin-major layout [bin][32 features] (g plane, h plane), so
//    the bank of (bin, f) is f.  Each lane owns one row and visits its 32 features rotated by
//    its lane id (feature (lane + s) & 31 at step s): the 32 lanes of every atomic hit 32
//    distinct banks -> conflict-free ATOMS at 1 warp-instruction/clk/SM (microbench: 4.57 T
//    symbols/s on B200, vs 0.15 T with bin-driven random banks).
//  * non-returning atomics: a chunk holds <= (2^31-1) >> quant_bits rows, so no s32 sum can
//    overflow (|q| <= 2^quant_bits) and no carry handling is needed.
//  * each (chunk, feature-group) item writes its s32 partial once (no zero-fill, no global
//    atomics, deterministic); k_eval sums the partials of a node in int64.
#include "internal.cuh"
#include "stream.cuh"

#include <climits>
#include <cmath>

#ifndef OOCGB_EVAL_FOLD
#define OOCGB_EVAL_FOLD 1
#endif
#ifndef OOCGB_NARROW_CU
#define OOCGB_NARROW_CU 2  // chunk partials per load batch in k_eval_narrow
#endif
#ifndef OOCGB_HIST_LOAD
#define OOCGB_HIST_LOAD 1  // measured: -4% at the levels below the root (profiles/r01_microbench_hist_levels.txt)
#endif
#ifndef OOCGB_FLUSH256
#define OOCGB_FLUSH256 1  // k_hist flush with 256-bit stores (STG.E.ENL2.256)
#endif
#ifndef OOCGB_HIST_EXPERIMENT
#define OOCGB_HIST_EXPERIMENT 0  // tools/microbench/hist_levels.cu only
#endif

// Per-call scalars read by the captured kernels (so one CUDA graph serves every round).
struct RoundParams {
  long long G, H, n_rows_global;
  double sg_inv, sh_inv;
  long long h_min;   // candidate valid iff H_L >= h_min and H_R >= h_min (exact form of R13)
  float sg_inv_f, sh_inv_f;
  float fold_c, fold_lq;  // the float pre-filter's folded scales c = sg^2 / sh, lambda / sh (per round)
  int prefilter;     // 0: scales outside float's safe range -> every candidate evaluated exactly
};

struct GraphKey {
  int n, D, m, ridx_mode, keep_debug, profiling, world, has_missing, root_list;
  double lambda, gamma, mcw, eta;
  const void *bins;
  size_t pitch;
  int quant_bits;
  bool operator==(const GraphKey &o) const {
    return n == o.n && D == o.D && m == o.m && ridx_mode == o.ridx_mode && keep_debug == o.keep_debug &&
           has_missing == o.has_missing && root_list == o.root_list &&
           profiling == o.profiling && world == o.world && lambda == o.lambda && gamma == o.gamma &&
           mcw == o.mcw && eta == o.eta && bins == o.bins && pitch == o.pitch && quant_bits == o.quant_bits;
  }
};

// buffers of the Alg. 6 streamed build (build_tree_streamed), owned by the data's Work
struct StreamWork {
  int64_t cap_n = 0, cap_b = 0;
  int max_slots = 0;
  int32_t *row_node = nullptr;   // [n] current node of each row
  int32_t *b_slot = nullptr;     // [batch] slot of each batch row at this level (-1: leaf)
  int32_t *b_ridx = nullptr;     // [batch] batch rows grouped by slot
  int2 *b_q = nullptr;           // [batch] their gradient pairs
  int *slot_cnt = nullptr;       // [2^(D-1)] rows per slot in the batch
  int *slot_cur = nullptr;       // scatter cursors
};

struct Work {
  int64_t cap_rows = 0;
  int max_depth = -1, m = 0, n_fg = 0;
  int64_t items_cap = 0;
  int32_t *ridx[2] = {nullptr, nullptr};
  int2 *q[2] = {nullptr, nullptr};
  oocgb::Seg *segs[2] = {nullptr, nullptr};
  int *seg_cur[2] = {nullptr, nullptr};  // per-segment (left, right) cursors, ping-pong by level
  int *tile_seg = nullptr;               // partition tile -> first segment
  int2 *chunk_rng = nullptr;            // histogram chunk -> its position range [r0, r1)
  long long *seg_cnt = nullptr;
  oocgb::Pair *pairs = nullptr;
  int *partial = nullptr;
  long long *phist[2] = {nullptr, nullptr};
  long long *built64 = nullptr;
  long long *rs_send = nullptr;  // world > 1: reduce-scatter send buffer [rank][pair][msl][256][2]
  int msl = 0, max_slots = 0;    // features per rank slice; candidate slots per level
  oocgb::Cand *cand = nullptr;
  int4 *ent = nullptr;  // eval work lists [2][ent_cap] of (pair, side, node, 0)
  int ent_cap = 0;
  oocgb::DNode *dnodes = nullptr;
  oocgb::LevelCtl *ctl = nullptr;
  long long *dbg = nullptr;
  size_t dbg_bytes = 0;
  int final_cur = 0;  // which ridx / segs buffer holds the final partition
  int root_list = 0;  // level 0's evaluation list when known (1 general, 2 narrow; 0 both)
  int hist_grid = 0;
  RoundParams *d_rp = nullptr;     // device copy of the per-call scalars
  RoundParams *h_rp = nullptr;     // pinned staging
  oocgb::DNode *h_dn = nullptr;    // pinned export staging (node records, control block, predict nodes):
  oocgb::LevelCtl *h_ctl = nullptr;  // the tree's predict nodes go up asynchronously, so build_tree
  oocgb::PNode *h_pn = nullptr;    // synchronises the host once per tree
  cudaGraphExec_t graph = nullptr; // captured level loop of the last key
  GraphKey key{};
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> graph_events;  // profiling
  StreamWork sw;                   // streamed build only
};

namespace oocgb {

__host__ __device__ __forceinline__ int level_first(int d) { return (1 << d) - 1; }

// Leaf weight (Eq. 6) and dequantised sums of a node from its exact fixed-point sums (R15).
__device__ void node_fill(DNode &nd, long long Gq, long long Hq, double sg_inv, double sh_inv,
                          double lambda, double eta, int *err) {
  double g = __dmul_rn((double)Gq, sg_inv), h = __dmul_rn((double)Hq, sh_inv);
  nd.Gq = Gq;
  nd.Hq = Hq;
  nd.sum_g = g;
  nd.sum_h = h;
  double den = __dadd_rn(h, lambda);
  if (!(den > 0.0)) atomicExch(err, 1);
  nd.tP = __ddiv_rn(__dmul_rn(g, g), den);  // the split evaluation's parent term (R14 order)
  double w = __ddiv_rn(-g, den);
  nd.leaf_value = __double2float_rn(__dmul_rn(eta, w));
}

// Derives the per-call scalars from the device sample state (exactly the host formulas they
// replace: dequantisation scales 2^-e, the integer form of R13, the pre-filter guard).
__device__ __forceinline__ long long clamp_ll(double x) {
  if (!(x > -9.0e18)) return LLONG_MIN / 2;
  if (!(x < 9.0e18)) return LLONG_MAX / 2;
  return (long long)x;
}

__global__ void k_init_build(DNode *dn, int n_nodes, const SampleState *__restrict__ ss, RoundParams *rp,
                             double lambda, double mcw, double eta, Seg *segs,
                             Pair *pairs, LevelCtl *ctl, int n_sel_arg, int n_fg, int target_items,
                             int kmax, int max_depth, const int32_t *sel_rows, int32_t *ridx,
                             const int2 *q_in, int2 *q_out, int ridx_mode, int2 *chunk_rng, int4 *ent,
                             int ent_cap, int *tile_seg, int n_tiles, int *seg_cur0) {
  int tid = blockIdx.x * blockDim.x + threadIdx.x;
  int nth = gridDim.x * blockDim.x;
  // (the former memsets of the build's graph) one root segment for every partition tile
  if (tile_seg)
    for (int t = tid; t < n_tiles; t += nth) tile_seg[t] = 0;
  // n_sel_arg < 0: the sample's row count from the device sample state (graph independent of it)
  const int n_sel = n_sel_arg >= 0 ? n_sel_arg : (int)ss->n_sel_local;
  {
    const long long cr = hist_chunk_rows(n_sel, 1, n_fg, target_items, kmax);
    const int nch = (int)((n_sel + cr - 1) / cr);
    const int crq = nch > 0 ? (int)((n_sel + nch - 1) / nch) : (int)cr;  // equal chunks of the root
    for (int c = tid; c < nch; c += nth) chunk_rng[c] = make_int2(c * crq, min(n_sel, (c + 1) * crq));
  }
  for (int v = tid; v < n_nodes; v += nth) {
    DNode nd{};
    nd.feature = -2;
    dn[v] = nd;
  }
  // the level loop reads the sample's own buffers at level 0 (identity rows / the selected rows,
  // the sample's q) and the partition writes buffer 1 first; only a depth-0 build (no level)
  // needs buffer 0 filled for its exports
  if (max_depth == 0)
    for (int i = tid; i < n_sel; i += nth) {
      ridx[i] = (ridx_mode == 1) ? sel_rows[i] : i;  // 1: in-core sampled (bins of the full page)
      q_out[i] = q_in[i];
    }
  if (tid == 0) {
    *ctl = LevelCtl{};  // the control block and the root segment's cursors start at zero
    if (seg_cur0) { seg_cur0[0] = 0; seg_cur0[1] = 0; }
    RoundParams P;
    P.G = ss->G;
    P.H = ss->H;
    P.n_rows_global = ss->n_sel_global;
    P.sg_inv = ldexp(1.0, -ss->e_g);
    P.sh_inv = ldexp(1.0, -ss->e_h);
    P.sg_inv_f = ldexpf(1.0f, -ss->e_g);
    P.sh_inv_f = ldexpf(1.0f, -ss->e_h);
    P.fold_c = P.sg_inv_f * P.sg_inv_f / P.sh_inv_f;
    P.fold_lq = (float)lambda / P.sh_inv_f;
    // R13 exactly, in integers: hl = HL 2^-e_h is exact, so hl >= mcw <=> HL >= ceil(mcw 2^e_h)
    // and hl + lambda > 0 <=> HL >= floor(-lambda 2^e_h) + 1 (clamped to the int64 range)
    const long long t1 = clamp_ll(ceil(ldexp(mcw, ss->e_h)));
    const long long t2 = clamp_ll(floor(ldexp(-lambda, ss->e_h))) + 1;
    P.h_min = t1 > t2 ? t1 : t2;
    // float pre-filter only where every scale is a normal float: 2^-e_g, 2^-e_h, and the folded
    // c = 2^(e_h - 2 e_g), lambda 2^e_h
    P.prefilter = (abs(ss->e_g) <= 60 && abs(ss->e_h) <= 60 && abs(ss->e_h - 2 * ss->e_g) <= 100) ? 1 : 0;
    *rp = P;
    DNode r{};
    r.feature = -1;
    r.n_rows = P.n_rows_global;
    node_fill(r, P.G, P.H, P.sg_inv, P.sh_inv, lambda, eta, &ctl->error);
    dn[0] = r;
    segs[0] = Seg{0, n_sel, 0, -1};
    const long long cr = hist_chunk_rows(n_sel, 1, n_fg, target_items, kmax);
    const int nch = (int)((n_sel + cr - 1) / cr);
    const int crq = nch > 0 ? (int)((n_sel + nch - 1) / nch) : (int)cr;  // equal chunks
    pairs[0] = Pair{-1, 0, -1, 0, n_sel, 0, nch, crq, (P.n_rows_global <= kmax) ? 2 : 0, {0, 0, 0}};
    ctl->hist_next = 0;
    ctl->n_pairs = max_depth > 0 ? 1 : 0;
    ctl->n_items = max_depth > 0 ? nch * n_fg : 0;
    ctl->n_segs = 1;
    ctl->n_splits = 0;
    const bool narrow = P.n_rows_global <= kmax;  // eval work list of the root (pair 0, side 0)
    ent[narrow ? ent_cap : 0] = make_int4(0, 0, 0, 0);
    ctl->n_ew = (max_depth > 0 && !narrow) ? 1 : 0;
    ctl->n_en = (max_depth > 0 && narrow) ? 1 : 0;
  }
}

// ---------------------------------------------------------------------------------------------
// BuildHistograms.  Persistent CTAs over items = (global chunk, feature group).
// Shared accumulators: s32 words [bin][g: 32 features | h: 32 features] -> word(bin, f) =
// 64 bin + f for g and + 32 for h, so the bank of every accumulator is its feature f.
// Lane l of a warp works on row slot r = l >> 1 and half h = l & 1 of the 32-feature group
// (features 16h .. 16h + 15): its 16 symbols are one 16-B load from the group plane (the two
// lanes of a row read one 32-B sector; a warp's 16 consecutive rows are 512 contiguous bytes).
// At step s the lane adds into feature 16h + ((r + s) & 15): for a fixed s the 32 lanes hit 32
// distinct banks (h picks the bank half, the rotation a bank inside it) -> conflict-free ATOMS.
// Per symbol: one PRMT (bin * 256 straight from the packed word), one IADD3 (+ the lane's
// precomputed feature offset and the shared base), two ATOMS.
__global__ void __launch_bounds__(kHistThreads, kHistCtasPerSm)
k_hist(const uint8_t *__restrict__ bins, size_t pitch, int m, int n_fg, const int32_t *__restrict__ ridx,
       const int2 *__restrict__ q, const Pair *__restrict__ pairs, LevelCtl *ctl,
       const int2 *__restrict__ chunk_rng, int *__restrict__ partial, int identity, int row_step, int gshift) {
  extern __shared__ int4 smem4[];
  int *S = reinterpret_cast<int *>(smem4);
  char *Sb = reinterpret_cast<char *>(smem4);
  const int n_items = ctl->n_items;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int half = lane & 1, rslot = lane >> 1;
  const int wq = rslot >> 2, bq = (rslot & 3) * 8;
  // 32-bit shared address of feature 16h + ((rslot + s) & 15) in bin 0 (the shared base is folded
  // in here once, so the inner loop never rematerialises it)
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem4);
  uint32_t f4[16];
#pragma unroll
  for (int s = 0; s < 16; ++s) f4[s] = sbase + 4u * (uint32_t)(16 * half + ((rslot + s) & 15));
  constexpr int RT = kHistThreads / 2;  // rows per CTA step
  // symbol (row, f) of group fg = f / 32 at bins + (fg >> gshift) * pitch + row * row_step + (fg &
  // (2^gshift - 1)) * 32 + f % 32: row_step = gw (32 or 64-B planes, gshift 0 or 1) for the tiled
  // device pages, the row stride for a row-major (streamed) page with pitch 32, gshift 0
  // items: the first from blockIdx, then dynamically from ctl->hist_next (chunks are numbered
  // largest first by the plan, so this is longest-processing-time-first list scheduling); the
  // next item is fetched while the current one runs (double-buffered slot, read after the
  // item's closing barrier)
  __shared__ int s_next[2];
  int par = 0;
  for (int item = blockIdx.x; item < n_items; par ^= 1) {
    if (threadIdx.x == 0) s_next[par] = (int)gridDim.x + atomicAdd(&ctl->hist_next, 1);
    const int fg = item % n_fg, cg = item / n_fg;
    const int2 rg = chunk_rng[cg];  // the chunk's positions (written by the plan: one load)
    const int r0 = rg.x, r1 = rg.y;
#if !(OOCGB_HIST_EXPERIMENT & 4)  // microbenchmark: no zero fill
    for (int i = threadIdx.x; i < 2 * kBins * kFG / 4; i += kHistThreads) smem4[i] = make_int4(0, 0, 0, 0);
#endif
    __syncthreads();
    // 32-feature group fg lives in plane fg >> gshift at byte (fg & ((1 << gshift) - 1)) * 32
    const uint8_t *base = bins + (size_t)(fg >> gshift) * pitch + (fg & ((1 << gshift) - 1)) * 32 + half * 16;
    auto row_of = [&](int kk) -> int { return identity ? kk : __ldg(ridx + kk); };
    auto load_row = [&](int kk, int row, uint4 &x, int2 &qv) {
      if (kk < r1) {
#if OOCGB_HIST_LOAD == 1  // streaming symbols: no L1 allocation
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w) : "l"(base + (size_t)row * row_step));
#elif OOCGB_HIST_LOAD == 2  // + a 256-B L2 prefetch hint
        asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w) : "l"(base + (size_t)row * row_step));
#else
        x = __ldg(reinterpret_cast<const uint4 *>(base + (size_t)row * row_step));
#endif
        qv = __ldg(q + kk);
      }
    };
    // one row: rotate the lane's 16 symbols right by `rslot` bytes (byte s = feature
    // 16h + ((rslot + s) & 15)), then 16 x 2 conflict-free shared reductions.  PRMT moves byte
    // (s & 3) of a word to bits 8..15 with zeros elsewhere = bin * 256 (the bin's 256-B line).
#if OOCGB_HIST_EXPERIMENT & 1
    uint32_t xacc = 0;
#endif
    auto accumulate = [&](const uint4 &x, const int2 qq) {
      uint32_t w[4] = {x.x, x.y, x.z, x.w};
      uint32_t t[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) t[i] = (wq & 1) ? w[(i + 1) & 3] : w[i];
#pragma unroll
      for (int i = 0; i < 4; ++i) w[i] = (wq & 2) ? t[(i + 2) & 3] : t[i];
#pragma unroll
      for (int i = 0; i < 4; ++i) t[i] = __funnelshift_r(w[i], w[(i + 1) & 3], bq);
#pragma unroll
      for (int s = 0; s < 16; ++s) {
        const uint32_t a = __byte_perm(t[s >> 2], 0u, 0x4404u | ((uint32_t)(s & 3) << 4)) + f4[s];
#if OOCGB_HIST_EXPERIMENT & 1  // microbenchmark: no shared atomics (one register XOR keeps the data live)
        xacc ^= a + (uint32_t)qq.x;
#else
        asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(a), "r"(qq.x));
        asm volatile("red.shared.add.s32 [%0+128], %1;" ::"r"(a), "r"(qq.y));
#endif
      }
    };
    // Software pipeline over rows k, k + RT, k + 2RT, ...: kDepth register sets rotate (the loop
    // is unrolled by kDepth); a set is consumed (rotation + reductions) and only then refilled
    // with the row kDepth steps ahead, so no in-flight register is ever copied; the row id for
    // a refill is loaded one round earlier still.
    constexpr int kDepth = kHistDepth;
    int k = r0 + (threadIdx.x >> 1);
    uint4 xs[kDepth];
    int2 qs[kDepth];
    int rs[kDepth];
#pragma unroll
    for (int i = 0; i < kDepth; ++i) {
      xs[i] = make_uint4(0, 0, 0, 0);
      qs[i] = make_int2(0, 0);
      rs[i] = 0;
      if (k + i * RT < r1) load_row(k + i * RT, row_of(k + i * RT), xs[i], qs[i]);
    }
#pragma unroll
    for (int i = 0; i < kDepth; ++i)
      if (k + (kDepth + i) * RT < r1) rs[i] = row_of(k + (kDepth + i) * RT);
    while (k < r1) {
      bool done = false;
#pragma unroll
      for (int i = 0; i < kDepth; ++i) {
        if (!done) {
          const int kk = k + i * RT;
          if (kk >= r1) {
            done = true;
          } else {
            accumulate(xs[i], qs[i]);
            load_row(kk + kDepth * RT, rs[i], xs[i], qs[i]);
            if (kk + 2 * kDepth * RT < r1) rs[i] = row_of(kk + 2 * kDepth * RT);
          }
        }
      }
      k += kDepth * RT;
    }
#if OOCGB_HIST_EXPERIMENT & 1
    if (xacc == 0x9e3779b9u) S[threadIdx.x] = (int)xacc;  // keep the experiment's data live
#endif
    __syncthreads();
    // flush: warp w owns bins [32w, 32w+32); lane l = feature l -> conflict-free reads; each lane
    // writes its feature's 32 (g, h) pairs = 256 contiguous bytes of the [32][256][2] partial.
    // Each store is one 256-bit STG of 4 bins (g, h): a lane-strided store touches one line per
    // lane whatever its width, so 32-B stores halve the flush's L1 wavefronts against 16-B ones.
    const int f = fg * kFG + lane;
    for (int bb = warp; bb < kBins / 32; bb += kHistThreads / 32) {
      int *dst = partial + (((size_t)item * kFG + lane) * kBins + bb * 32) * 2;
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        const int i0 = (bb * 32 + i) * 64 + lane;
        const int a0 = S[i0], a1 = S[i0 + 32], a2 = S[i0 + 64], a3 = S[i0 + 96];
        const int a4 = S[i0 + 128], a5 = S[i0 + 160], a6 = S[i0 + 192], a7 = S[i0 + 224];
#if OOCGB_HIST_EXPERIMENT & 2  // microbenchmark: no partial stores
        if (f < m && a0 == 0x7fffffff)
#else
        if (f < m)
#endif
        {
#if OOCGB_FLUSH256
          asm volatile("st.global.v8.u32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst + 2 * i), "r"(a0),
                       "r"(a1), "r"(a2), "r"(a3), "r"(a4), "r"(a5), "r"(a6), "r"(a7)
                       : "memory");
#else
          reinterpret_cast<int4 *>(dst + 2 * i)[0] = make_int4(a0, a1, a2, a3);
          reinterpret_cast<int4 *>(dst + 2 * i)[1] = make_int4(a4, a5, a6, a7);
#endif
        }
      }
    }
    __syncthreads();
    item = s_next[par];
  }
}

// ---------------------------------------------------------------------------------------------
// BuildHistograms at an identity level (the root of an in-core build: position = row, and the
// gradient pairs in position order) with a bulk-asynchronous feed: the rows of an item are a
// contiguous 32-B-per-row run of the group plane (and a contiguous run of q), so one thread
// streams them into a shared-memory ring with cp.async.bulk (TMA engine, no per-thread load
// instructions, no registers held by loads in flight) and the 16 warps only read shared memory
// and issue the shared reductions.  Ring: kTmaStages stages of kTmaRows rows (one CTA step:
// 16 warps x 16 rows); stage s is complete when its mbarrier full[s] has seen the bytes, and free
// again when the 16 warps have arrived on empty[s].  Same accumulators, lane mapping, rotation
// and flush as k_hist (identical partials).
// Measured on B200 (config 2 root, r02): 219 us against k_hist's 181 us.  The kernel stays
// L1-pipe bound (80% busy) and the bulk writes into shared memory take bank cycles from the
// reductions (ncu: 41.1 M atomic wavefronts for 32 M ideal, 9.1 M of them bank conflicts; k_hist
// has none), so it is built only with -DOOCGB_HIST_TMA=1 (tools/gpu_ab.sh) and off by default.
#ifndef OOCGB_HIST_TMA
#define OOCGB_HIST_TMA 0
#endif
#if OOCGB_HIST_TMA
constexpr int kTmaRows = kHistThreads / 2;                 // rows per stage = rows per CTA step
constexpr int kTmaStages = 4;
constexpr int kTmaSymBytes = kTmaRows * 32;                 // 8 KB
constexpr int kTmaQBytes = ((kTmaRows + 2) * 8 + 15) / 16 * 16;  // even-aligned q run (+ 1 row each end)
constexpr int kTmaSmem = kHistSmem + kTmaStages * (kTmaSymBytes + kTmaQBytes) + 2 * kTmaStages * 8;

__device__ __forceinline__ void mbar_init(uint32_t a, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t a, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, unsigned bytes, uint32_t mbar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(mbar)
               : "memory");
}

__global__ void __launch_bounds__(kHistThreads, kHistCtasPerSm)
k_hist_tma(const uint8_t *__restrict__ bins, size_t pitch, int m, int n_fg, const int2 *__restrict__ q,
           const Pair *__restrict__ pairs, LevelCtl *ctl, const int2 *__restrict__ chunk_rng,
           int *__restrict__ partial) {
  extern __shared__ int4 smem4[];
  int *S = reinterpret_cast<int *>(smem4);
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem4);
  const uint32_t s_sym = sbase + kHistSmem;
  const uint32_t s_q = s_sym + kTmaStages * kTmaSymBytes;
  const uint32_t s_full = s_q + kTmaStages * kTmaQBytes, s_empty = s_full + 8 * kTmaStages;
  const int n_items = ctl->n_items;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int half = lane & 1, rslot = lane >> 1;
  const int wq = rslot >> 2, bq = (rslot & 3) * 8;
  uint32_t f4[16];
#pragma unroll
  for (int s = 0; s < 16; ++s) f4[s] = sbase + 4u * (uint32_t)(16 * half + ((rslot + s) & 15));
  if (threadIdx.x == 0) {
    for (int s = 0; s < kTmaStages; ++s) {
      mbar_init(s_full + 8 * s, 1);
      mbar_init(s_empty + 8 * s, kHistThreads / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // ring position: batches issued / consumed so far by this CTA (stage = n % S, phase = n / S)
  unsigned n_issued = 0, n_used = 0;
  __shared__ int s_next[2];
  int par = 0;
  for (int item = blockIdx.x; item < n_items; par ^= 1) {
    if (threadIdx.x == 0) s_next[par] = (int)gridDim.x + atomicAdd(&ctl->hist_next, 1);
    const int fg = item % n_fg, cg = item / n_fg;
    const Pair P = pairs[chunk_rng[cg]];
    const int c = cg - P.chunk_base;
    const int r0 = P.begin + c * P.chunk_rows;
    const int r1 = min(P.begin + P.count, r0 + P.chunk_rows);
    const int nb = r1 > r0 ? (r1 - r0 + kTmaRows - 1) / kTmaRows : 0;
    const uint8_t *plane = bins + (size_t)fg * pitch;
    // producer: batch b of this item into the next ring slot (thread 0 only)
    auto issue = [&](int b) {
      const unsigned st = n_issued % kTmaStages;
      if (n_issued >= kTmaStages) mbar_wait(s_empty + 8 * st, ((n_issued / kTmaStages) - 1) & 1);
      const int rb = r0 + b * kTmaRows, re = min(r1, rb + kTmaRows);
      const int qa = rb & ~1, qe = (re + 1) & ~1;
      const unsigned sb = (unsigned)(re - rb) * 32u, qb = (unsigned)(qe - qa) * 8u;
      mbar_expect_tx(s_full + 8 * st, sb + qb);
      bulk_g2s(s_sym + st * kTmaSymBytes, plane + (size_t)rb * 32, sb, s_full + 8 * st);
      bulk_g2s(s_q + st * kTmaQBytes, q + qa, qb, s_full + 8 * st);
      ++n_issued;
    };
    int b_next = 0;  // next batch of this item to issue (thread 0's view)
    if (threadIdx.x == 0)
      for (; b_next < nb && b_next < kTmaStages; ++b_next) issue(b_next);
    for (int i = threadIdx.x; i < 2 * kBins * kFG / 4; i += kHistThreads) smem4[i] = make_int4(0, 0, 0, 0);
    __syncthreads();
    for (int b = 0; b < nb; ++b) {
      const unsigned st = n_used % kTmaStages;
      mbar_wait(s_full + 8 * st, (n_used / kTmaStages) & 1);
      const int rb = r0 + b * kTmaRows;
      const int ib = warp * 16 + rslot;  // this lane's row in the batch
      if (rb + ib < r1) {
        uint4 x;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(x.x), "=r"(x.y), "=r"(x.z), "=r"(x.w)
                     : "r"(s_sym + st * kTmaSymBytes + ib * 32 + half * 16));
        int2 qq;
        asm volatile("ld.shared.v2.s32 {%0, %1}, [%2];"
                     : "=r"(qq.x), "=r"(qq.y)
                     : "r"(s_q + st * kTmaQBytes + (rb + ib - (rb & ~1)) * 8));
        uint32_t w[4] = {x.x, x.y, x.z, x.w};
        uint32_t t[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) t[i] = (wq & 1) ? w[(i + 1) & 3] : w[i];
#pragma unroll
        for (int i = 0; i < 4; ++i) w[i] = (wq & 2) ? t[(i + 2) & 3] : t[i];
#pragma unroll
        for (int i = 0; i < 4; ++i) t[i] = __funnelshift_r(w[i], w[(i + 1) & 3], bq);
#pragma unroll
        for (int s = 0; s < 16; ++s) {
          const uint32_t a = __byte_perm(t[s >> 2], 0u, 0x4404u | ((uint32_t)(s & 3) << 4)) + f4[s];
          asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(a), "r"(qq.x));
          asm volatile("red.shared.add.s32 [%0+128], %1;" ::"r"(a), "r"(qq.y));
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(s_empty + 8 * st);
      ++n_used;
      if (threadIdx.x == 0 && b_next < nb) issue(b_next++);
    }
    __syncthreads();
    const int f = fg * kFG + lane;
    for (int bb = warp; bb < kBins / 32; bb += kHistThreads / 32) {
      int4 *dst = reinterpret_cast<int4 *>(partial + (((size_t)item * kFG + lane) * kBins + bb * 32) * 2);
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        const int i0 = (bb * 32 + i) * 64 + lane, i1 = i0 + 64;
        const int4 v = make_int4(S[i0], S[i0 + 32], S[i1], S[i1 + 32]);
        if (f < m) dst[i >> 1] = v;
      }
    }
    __syncthreads();
    item = s_next[par];
  }
}
#endif  // OOCGB_HIST_TMA

// Multi-GPU: sum a pair's s32 chunk partials into int64 histograms that are then reduce-scattered
// over the ranks ("summed across all GPUs"; each rank receives the sums of its feature
// slice and evaluates only those features).  Thread per (pair, feature, bin).
// Multi-GPU (world > 1): the send buffer of the reduce-scatter is sliced by feature owner: rank r
// owns features [r msl, (r + 1) msl) and receives block r = [pair][feature - r msl][256][2].
__global__ void k_reduce_partials(const int *__restrict__ partial, const Pair *__restrict__ pairs,
                                  const LevelCtl *__restrict__ ctl, int m, int n_fg, int msl, int lvl_pairs,
                                  long long *__restrict__ out) {
  const int n_pairs = ctl->n_pairs;
  int64_t total = (int64_t)n_pairs * m * kBins;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int b = (int)(t % kBins);
    int j = (int)((t / kBins) % m);
    int p = (int)(t / ((int64_t)kBins * m));
    const Pair P = pairs[p];
    long long g = 0, h = 0;
    for (int c = 0; c < P.n_chunks; ++c) {
      size_t item = (size_t)(P.chunk_base + c) * n_fg + j / kFG;
      const int2 v = reinterpret_cast<const int2 *>(partial)[(item * kFG + (j % kFG)) * kBins + b];
      g += v.x;
      h += v.y;
    }
    const int r = j / msl;
    const size_t o = (((size_t)r * lvl_pairs + p) * msl + (j - r * msl)) * kBins + b;
    out[o * 2] = g;
    out[o * 2 + 1] = h;
  }
}

// ---------------------------------------------------------------------------------------------
// EvaluateSplit: one warp per (pair, feature j); lane owns bins [8 lane, 8 lane + 8).
struct EvalArgs {
  int d, D, m, n_fg;
  const Pair *pairs;
  LevelCtl *ctl;
  const int *partial;
  const long long *built64;   // non-null: multi-GPU all-reduced built histograms
  const long long *phist_prev;
  long long *phist_next;
  long long *dbg;
  const int *cut_ptrs;
  DNode *dn;
  Cand *cand;
  double lambda, gamma, mcw;
  const RoundParams *rp;
  long long kmax;  // nodes with <= kmax rows keep their parent histogram as exact s32 pairs
  int streamed;    // Alg. 6 mode: every node built directly, no parent histograms kept
  const float *cut_values;
  double eta;
  const int4 *ent;  // per-level work lists of (pair, side, node, 0): general [0, n_ew), narrow [ent_cap, + n_en)
  int ent_cap;
  int has_missing;  // R27: bin 255 holds missing values; candidates in both default directions
  // feature slice (world > 1: this rank evaluates features [f0, f0 + mf) from reduce-scattered
  // histograms whose rows hold hm = msl features; world == 1: f0 = 0, mf = hm = msl = m)
  int f0, mf, hm, msl, max_slots;
  int crank;  // candidate block of this rank's slice: f0 / msl
  int root_list;  // level 0 only: 1 the root is on the general list, 2 narrow, 0 unknown
  Seg *segs;      // this level's segments (k_finalize records each split in its node's segment)
};

// candidates [owner rank][slot][msl]: rank r writes features [r msl, (r + 1) msl) into block r,
// the blocks are all-gathered, and every rank's k_finalize reads all m features
__host__ __device__ __forceinline__ size_t cand_index(int msl, int max_slots, int slot, int j) {
  const int r = j / msl;
  return ((size_t)r * max_slots + slot) * msl + (j - r * msl);
}
// the same for a feature of this rank's slice (j in [r msl, (r + 1) msl), r = the slice's owner):
// no integer division on the evaluation's per-item path
__device__ __forceinline__ size_t cand_index_own(int msl, int max_slots, int r, int slot, int j) {
  return ((size_t)r * max_slots + slot) * msl + (j - r * msl);
}

__device__ __forceinline__ int warp_excl_scan_i(int v, int lane, int &total) {
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  total = __shfl_sync(0xffffffffu, incl, 31);
  return incl - v;
}

__device__ __forceinline__ long long warp_excl_scan_ll(long long v, int lane, long long &total) {
  long long incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    long long u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  total = __shfl_sync(0xffffffffu, incl, 31);
  return incl - v;
}

// 1 / x to <= 1 ulp with no denormal range handling (a denormal x flushes to 0 -> +inf).
__device__ __forceinline__ float frcp_ftz(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// Exact Eq. 8 gain in double, the oracle's operation order (R14).
__device__ __forceinline__ double gain_exact(long long GL, long long HL, long long G, long long H, double tP,
                                             double sg_inv, double sh_inv, double lambda, double gamma) {
  const double gl = __dmul_rn((double)GL, sg_inv), hl = __dmul_rn((double)HL, sh_inv);
  const double gr = __dmul_rn((double)(G - GL), sg_inv), hr = __dmul_rn((double)(H - HL), sh_inv);
  const double tL = __ddiv_rn(__dmul_rn(gl, gl), __dadd_rn(hl, lambda));
  const double tR = __ddiv_rn(__dmul_rn(gr, gr), __dadd_rn(hr, lambda));
  return __dsub_rn(__dmul_rn(0.5, __dsub_rn(__dadd_rn(tL, tR), tP)), gamma);
}

// EvaluateSplit of one node for feature j: lane owns bins [8 lane, 8 lane + 8).
// 1) validity (R13) as an exact integer test: hl >= mcw and hl + lambda > 0 with hl = HL 2^-e_h
//    exactly (power-of-two scaling) is HL >= h_min (host-derived integer threshold);
// 2) float32 pre-filter: every candidate's gain in float with a rigorous bound tol
//    (|gain_f - gain| <= tol, all terms non-negative); L = max(gain_f - tol) over the warp;
// 3) exact double gains only for candidates with gain_f + tol >= L.  The exact argmax and all
//    its exact ties always pass (gain_f + tol >= gain >= gain(c') >= gain_f(c') - tol(c')), so
//    the result is identical to evaluating every candidate in double.
// I = int for nodes with <= kmax rows (every partial sum is then exact in int32), else long long.
// Returns the lane that owns the winning bin (it wrote the candidate), or 0.
template <typename I, bool MISS>
__device__ int eval_node_impl(const EvalArgs &A, int node, int j, int lane, const I (&g)[8], const I (&h)[8],
                              const RoundParams &rp, const long long G_, const long long H_, const double tP,
                              const I Gm, const I Hm) {
  const int B = A.cut_ptrs[j + 1] - A.cut_ptrs[j];
  const I G = (I)G_, H = (I)H_;
  I lg = 0, lh = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) { lg += g[i]; lh += h[i]; }
  I tg, th, eg, eh;
  if constexpr (sizeof(I) == 4) {
    eg = warp_excl_scan_i(lg, lane, tg);
    eh = warp_excl_scan_i(lh, lane, th);
  } else {
    eg = warp_excl_scan_ll(lg, lane, tg);
    eh = warp_excl_scan_ll(lh, lane, th);
  }
  // integer validity (R13) in the node's width: hmin <= HL and H - HL >= h_min <=> HL <= hmax,
  // the thresholds clamped to I (|HL| <= H < 2^31 when I = int, so clamping never flips a test)
  auto clampI = [](long long x) -> I {
    if (sizeof(I) == 4) return (I)(x > INT_MAX ? INT_MAX : (x < INT_MIN ? INT_MIN : x));
    return (I)x;
  };
  const I hmin = clampI(rp.h_min);
  const I hmax = clampI((long long)H_ - rp.h_min);
  // Float pre-filter on T = GL^2 / (HL + lq) + GR^2 / (HR + lq) (folded scales: with sg = 2^-e_g,
  // sh = 2^-e_h exact powers of two, tL + tR = c T with c = sg^2 / sh, lq = lambda / sh; the
  // pre-filter is on only while c and lq are normal floats, see k_init_build).  For one node the
  // gain 0.5 (c T - tP) - gamma is increasing in T, so the exact argmax (and every exact tie) has
  // the largest exact T.  With u = 2^-24, each float T carries <= 10 u relative error (int ->
  // float u each, the square 3 u, the lambda add 2 u, rcp.approx.ftz <= 1 ulp = 2 u, the product
  // u, the sum u) and the double evaluation of the gain rounds at ~2^-50 of c T + tP, so keeping
  // every candidate with T_f >= (1 - 2^-18) max T_f (2^-18 = 64 u > 2 x 10 u) keeps the true
  // argmax and its ties; only those are evaluated in double.  A denominator below FLT_MIN flushes
  // to 0 in the ftz reciprocal -> T_f = inf or NaN -> "not finite" -> always evaluated exactly.
  const float lq = rp.fold_lq;
  // candidate key 2 b + dir: dir 0 = missing rows right (left sums = the prefix), dir 1 = missing
  // rows left (prefix + the missing bin's sums; MISS only, R27)
  // tv: T_f of a valid candidate (+inf when not finite: always re-evaluated), NaN when invalid
  // (fails every >= test).  Tmax = fmaxf over the valid T_f (fmaxf ignores NaN); a valid +inf
  // makes Tmax = +inf, and then every valid candidate is evaluated exactly (thr = -inf below): a
  // superset of the survivors, so the same argmax.
  float tv[MISS ? 2 : 1][8];
  float Tmax = -INFINITY;
  auto pre = [&](I GLx, I HLx, bool vb, float &u, int) {
    const bool v = vb && HLx >= hmin && HLx <= hmax;
    const float GLf = (float)GLx, HLf = (float)HLx, GRf = (float)(G - GLx), HRf = (float)(H - HLx);
    const float T = GLf * GLf * frcp_ftz(HLf + lq) + GRf * GRf * frcp_ftz(HRf + lq);
    u = v ? (T < INFINITY ? T : INFINITY) : __int_as_float(0x7fc00000);
    Tmax = fmaxf(Tmax, v ? T : -INFINITY);
  };
  // pass 1: float T of every candidate
  I GL = eg, HL = eh;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    GL += g[i];
    HL += h[i];
    const int b = lane * 8 + i;
    // an empty bin repeats the previous candidate exactly, which wins the tie (lower bin)
    const bool vb = b <= B - 2 && ((g[i] | h[i]) != 0 || b == 0);
    pre(GL, HL, vb, tv[0][i], 2 * i);
    if constexpr (MISS) pre(GL + Gm, HL + Hm, vb, tv[MISS ? 1 : 0][i], 2 * i + 1);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) Tmax = fmaxf(Tmax, __shfl_xor_sync(0xffffffffu, Tmax, o));
  const float thr = (rp.prefilter && Tmax < INFINITY) ? Tmax * (1.0f - 0x1p-18f) : -INFINITY;
  // pass 2: exact double gains of the survivors, in key order (strict > keeps the lower key)
  double best = 0.0;
  int bkey = 0x7fffffff, have = 0;
  long long bGL = 0, bHL = 0;
  GL = eg;
  HL = eh;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    GL += g[i];
    HL += h[i];
#pragma unroll
    for (int dir = 0; dir < (MISS ? 2 : 1); ++dir) {
      if (tv[dir][i] >= thr) {  // NaN (invalid) fails
        const I GLx = dir ? GL + Gm : GL, HLx = dir ? HL + Hm : HL;
        const double gain = gain_exact(GLx, HLx, G, H, tP, rp.sg_inv, rp.sh_inv, A.lambda, A.gamma);
        if (!have || gain > best) {
          have = 1; best = gain; bkey = 2 * (lane * 8 + i) + dir; bGL = (long long)GLx; bHL = (long long)HLx;
        }
      }
    }
  }
  // warp argmax over (gain, key): larger gain, then lower key; invalid = -inf.  Usually one lane
  // holds every survivor of the pre-filter: its best is the warp's.  Otherwise only the pair is
  // shuffled; the lane that owns the winning key writes its own G_L, H_L.
  double bg = have ? best : -INFINITY;
  int bb = have ? bkey : 0x7fffffff;
  const unsigned hv = __ballot_sync(0xffffffffu, have);
  if (hv & (hv - 1)) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double og = __shfl_xor_sync(0xffffffffu, bg, o);
      const int ob = __shfl_xor_sync(0xffffffffu, bb, o);
      if (og > bg || (og == bg && ob < bb)) { bg = og; bb = ob; }
    }
  }
  const bool any = hv != 0;
  const int owner = any ? ((hv & (hv - 1)) ? (bb >> 4) : __ffs(hv) - 1) : 0;  // 16 keys per lane
  if (lane == owner) {
    const int slot = node - level_first(A.d);
    Cand cd;
    cd.gain = any ? bg : 0.0;
    cd.bin = bb;
    cd.valid = any ? 1 : 0;
    cd.GL = any ? bGL : 0;
    cd.HL = any ? bHL : 0;
    A.cand[cand_index_own(A.msl, A.max_slots, A.crank, slot, j)] = cd;
  }
  return owner;
}

// EvaluateSplit of one node for feature j (see eval_node_impl).  With missing values (R27) the
// missing bin 255 (lane 31's last element) holds the rows missing feature j; a feature with
// missing rows in this node also tries every candidate with those rows on the left.
template <typename I, bool HAS_MISSING>
__device__ int eval_node(const EvalArgs &A, int node, int j, int lane, const I (&g)[8],
                                         const I (&h)[8], const RoundParams &rp, const long long G_,
                                         const long long H_, const double tP) {
  if constexpr (HAS_MISSING) {  // a separate kernel instantiation: dense data keeps its registers
    const I Gm = __shfl_sync(0xffffffffu, g[7], 31), Hm = __shfl_sync(0xffffffffu, h[7], 31);
    if (Gm != 0 || Hm != 0) return eval_node_impl<I, true>(A, node, j, lane, g, h, rp, G_, H_, tP, Gm, Hm);
  }
  return eval_node_impl<I, false>(A, node, j, lane, g, h, rp, G_, H_, tP, (I)0, (I)0);
}

__device__ __forceinline__ void store_hist8(long long *dst, const long long (&g)[8], const long long (&h)[8]) {
  longlong2 *d2 = reinterpret_cast<longlong2 *>(dst);
#pragma unroll
  for (int i = 0; i < 8; ++i) d2[i] = make_longlong2(g[i], h[i]);
}

// One warp per (pair, feature j, side): side 0 evaluates the built child (sum of its s32 chunk
// partials, or the all-reduced int64 buffer), side 1 the derived sibling = parent - built (R17).
// Loads, the subtraction and the parent store use the coalesced bin order bin = 32 i + lane;
// a padded per-warp shared tile (conflict-free for both orders) then hands each lane its 8
// consecutive bins 8 lane .. 8 lane + 7 for the scan and the evaluation.
constexpr int kEvalWarps = 4;  // 4-warp blocks: measured best of 1, 2, 4, 8
constexpr int kEvalBlocksWide = 4, kEvalBlocksNarrow = 6;  // resident blocks per SM (registers)
template <bool HAS_MISSING>
__device__ __forceinline__ void eval_item_wide(const EvalArgs &A, int p, int side, int node, int j, int lane,
                                               longlong2 *tl) {
  const Pair P = A.pairs[p];  // (the node comes with the entry: its record loads alongside)
  if (node < 0) return;
  if (A.streamed && A.dn[node].feature == -2) return;  // streamed levels list every slot
  const long long nodeG = A.dn[node].Gq, nodeH = A.dn[node].Hq;  // prefetched for eval_node
  const double nodeTP = A.dn[node].tP;
  const long long nodeRows = A.dn[node].n_rows;
  long long g[8], h[8];  // strided: element i is bin 32 i + lane
  const size_t hsz = (size_t)A.hm * kBins * 2;  // built64 / parent rows: this rank's feature slice
  const int jl = j - A.f0;
  const size_t dsz = (size_t)A.m * kBins * 2;    // debug dumps: every feature
  longlong2 par[8];
  if (side) {  // parent loads first so they overlap the chunk loads
    const int ps = P.parent - level_first(A.d - 1);
    if (P.compact & 1) {  // compact s32 parent (exact: |sum| < 2^31)
      const int2 *src = reinterpret_cast<const int2 *>(A.phist_prev + (size_t)ps * hsz) + (size_t)jl * kBins;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int2 v = __ldg(src + 32 * i + lane);
        par[i] = make_longlong2(v.x, v.y);
      }
    } else {
      const longlong2 *src = reinterpret_cast<const longlong2 *>(A.phist_prev + (size_t)ps * hsz + (size_t)jl * kBins * 2);
#pragma unroll
      for (int i = 0; i < 8; ++i) par[i] = __ldg(src + 32 * i + lane);
    }
  }
  if (A.built64) {
    const longlong2 *src = reinterpret_cast<const longlong2 *>(A.built64 + (size_t)p * hsz + (size_t)jl * kBins * 2);
#pragma unroll
    for (int i = 0; i < 8; ++i) { longlong2 v = src[32 * i + lane]; g[i] = v.x; h[i] = v.y; }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) { g[i] = 0; h[i] = 0; }
    const size_t cstride = (size_t)A.n_fg * kFG * kBins;  // int2 elements between chunks
    const int2 *src0 = reinterpret_cast<const int2 *>(A.partial) +
                       (((size_t)P.chunk_base * A.n_fg + j / kFG) * kFG + (j % kFG)) * kBins + lane;
    int c = 0;
    for (; c + 2 <= P.n_chunks; c += 2) {
      int2 v[2][8];
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int i = 0; i < 8; ++i) v[u][i] = __ldg(src0 + (c + u) * cstride + 32 * i);
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int i = 0; i < 8; ++i) { g[i] += v[u][i].x; h[i] += v[u][i].y; }
    }
    if (c < P.n_chunks) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        int2 v = __ldg(src0 + c * cstride + 32 * i);
        g[i] += v.x; h[i] += v.y;
      }
    }
  }
  if (side) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { g[i] = par[i].x - g[i]; h[i] = par[i].y - h[i]; }
  }
  const int f_d = level_first(A.d);
  if (A.d <= A.D - 2 && !A.streamed) {
    if (P.compact & (side ? 4 : 2)) {
      int2 *dst = reinterpret_cast<int2 *>(A.phist_next + (size_t)(node - f_d) * hsz) + (size_t)jl * kBins;
#pragma unroll
      for (int i = 0; i < 8; ++i) dst[32 * i + lane] = make_int2((int)g[i], (int)h[i]);
    } else {
      longlong2 *dst = reinterpret_cast<longlong2 *>(A.phist_next + (size_t)(node - f_d) * hsz + (size_t)jl * kBins * 2);
#pragma unroll
      for (int i = 0; i < 8; ++i) dst[32 * i + lane] = make_longlong2(g[i], h[i]);
    }
  }
  if (A.dbg) {
    longlong2 *dst = reinterpret_cast<longlong2 *>(A.dbg + (size_t)node * dsz + (size_t)j * kBins * 2);
#pragma unroll
    for (int i = 0; i < 8; ++i) dst[32 * i + lane] = make_longlong2(g[i], h[i]);
  }
  // transpose through the padded tile: element e lives in slot e + e / 8 (16-B slots), which
  // is conflict-free per quarter-warp both for e = 32 i + lane and for e = 8 lane + i
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int e = 32 * i + lane;
    tl[e + (e >> 3)] = make_longlong2(g[i], h[i]);
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int e = 8 * lane + i;
    const longlong2 v = tl[e + (e >> 3)];
    g[i] = v.x;
    h[i] = v.y;
  }
  __syncwarp();  // the tile is reused by the warp's next item
  const RoundParams rp = *A.rp;
  if (nodeRows <= A.kmax) {  // every partial sum of the node is exact in int32
    int g32[8], h32[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { g32[i] = (int)g[i]; h32[i] = (int)h[i]; }
    eval_node<int, HAS_MISSING>(A, node, j, lane, g32, h32, rp, nodeG, nodeH, nodeTP);
  } else {
    eval_node<long long, HAS_MISSING>(A, node, j, lane, g, h, rp, nodeG, nodeH, nodeTP);
  }
}

// Persistent warps over the level's work list: item t = (entry t / m, feature t % m), entry =
// (pair, side) written by the plan (general list: nodes with > kmax rows, streamed levels).
template <bool HAS_MISSING>
__global__ void __launch_bounds__(kEvalWarps * 32, kEvalBlocksWide) k_eval(EvalArgs A) {
  __shared__ longlong2 tile[kEvalWarps][256 + 32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int n_items = A.ctl->n_ew * A.mf;
  if (n_items <= 0) return;  // (also mf = 0: a rank with no features)
  const int nw = (int)(gridDim.x * blockDim.x) >> 5;
  int t = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  int e = t / A.mf, jj = t - e * A.mf;  // item t = (entry e, feature f0 + jj), advanced by nw
  const int de = nw / A.mf, dj = nw - de * A.mf;
  for (; t < n_items; t += nw) {
    const int4 en = A.ent[e];
    eval_item_wide<HAS_MISSING>(A, en.x, en.y, en.z, A.f0 + jj, lane, tile[wib]);
    e += de;
    jj += dj;
    if (jj >= A.mf) { jj -= A.mf; ++e; }
  }
}

// k_eval for nodes with <= kmax rows (most nodes below the first levels): every histogram sum of
// such a node, and every prefix sum, is exact in int32, so the whole warp works in 32-bit
// (a wider parent or all-reduced sum is read through its low word: parent - built is exact
// modulo 2^32 and fits).  Fewer registers than k_eval -> twice the resident warps.
#ifndef OOCGB_EVAL_NARROW_MINB
#define OOCGB_EVAL_NARROW_MINB 6  // 80 registers, no spills (= kEvalBlocksNarrow)
#endif
template <bool HAS_MISSING>
__device__ __forceinline__ void eval_item_narrow(const EvalArgs &A, int p, int side, int node, int j, int lane,
                                                 int2 *tl) {
  const Pair P = A.pairs[p];  // (the node comes with the entry: its record loads alongside)
  if (node < 0) return;
  if (A.streamed && A.dn[node].feature == -2) return;
  const long long nodeG = A.dn[node].Gq, nodeH = A.dn[node].Hq;
  const double nodeTP = A.dn[node].tP;
  int g[8], h[8];  // strided: element i is bin 32 i + lane
  const size_t hsz = (size_t)A.hm * kBins * 2;  // built64 / parent rows: this rank's feature slice
  const int jl = j - A.f0;
  const size_t dsz = (size_t)A.m * kBins * 2;    // debug dumps: every feature
  int2 par[8];
  if (side) {
    const int ps = P.parent - level_first(A.d - 1);
    if (P.compact & 1) {
      const int2 *src = reinterpret_cast<const int2 *>(A.phist_prev + (size_t)ps * hsz) + (size_t)jl * kBins;
#pragma unroll
      for (int i = 0; i < 8; ++i) par[i] = __ldg(src + 32 * i + lane);
    } else {  // low words of the int64 pairs
      const int4 *src = reinterpret_cast<const int4 *>(A.phist_prev + (size_t)ps * hsz + (size_t)jl * kBins * 2);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int4 v = __ldg(src + 32 * i + lane);
        par[i] = make_int2(v.x, v.z);
      }
    }
  }
  if (A.built64) {
    const int4 *src = reinterpret_cast<const int4 *>(A.built64 + (size_t)p * hsz + (size_t)jl * kBins * 2);
#pragma unroll
    for (int i = 0; i < 8; ++i) { const int4 v = src[32 * i + lane]; g[i] = v.x; h[i] = v.z; }
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) { g[i] = 0; h[i] = 0; }
    const size_t cstride = (size_t)A.n_fg * kFG * kBins;
    const int2 *src0 = reinterpret_cast<const int2 *>(A.partial) +
                       (((size_t)P.chunk_base * A.n_fg + j / kFG) * kFG + (j % kFG)) * kBins + lane;
    // chunk partials NARROW_CU at a time (their loads in flight together: a multi-chunk node is
    // one L2 round trip per NARROW_CU chunks, not per chunk)
    int c = 0;
#if OOCGB_NARROW_CU > 1
    for (; c + OOCGB_NARROW_CU <= P.n_chunks; c += OOCGB_NARROW_CU) {
      int2 v[OOCGB_NARROW_CU][8];
#pragma unroll
      for (int u = 0; u < OOCGB_NARROW_CU; ++u)
#pragma unroll
        for (int i = 0; i < 8; ++i) v[u][i] = __ldg(src0 + (c + u) * cstride + 32 * i);
#pragma unroll
      for (int u = 0; u < OOCGB_NARROW_CU; ++u)
#pragma unroll
        for (int i = 0; i < 8; ++i) { g[i] += v[u][i].x; h[i] += v[u][i].y; }
    }
#endif
    for (; c < P.n_chunks; ++c) {
      int2 v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = __ldg(src0 + c * cstride + 32 * i);
#pragma unroll
      for (int i = 0; i < 8; ++i) { g[i] += v[i].x; h[i] += v[i].y; }
    }
  }
  if (side) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { g[i] = par[i].x - g[i]; h[i] = par[i].y - h[i]; }
  }
  const int f_d = level_first(A.d);
  if (A.d <= A.D - 2 && !A.streamed) {
    if (P.compact & (side ? 4 : 2)) {
      int2 *dst = reinterpret_cast<int2 *>(A.phist_next + (size_t)(node - f_d) * hsz) + (size_t)jl * kBins;
#pragma unroll
      for (int i = 0; i < 8; ++i) dst[32 * i + lane] = make_int2(g[i], h[i]);
    } else {
      longlong2 *dst = reinterpret_cast<longlong2 *>(A.phist_next + (size_t)(node - f_d) * hsz + (size_t)jl * kBins * 2);
#pragma unroll
      for (int i = 0; i < 8; ++i) dst[32 * i + lane] = make_longlong2(g[i], h[i]);
    }
  }
  if (A.dbg) {
    longlong2 *dst = reinterpret_cast<longlong2 *>(A.dbg + (size_t)node * dsz + (size_t)j * kBins * 2);
#pragma unroll
    for (int i = 0; i < 8; ++i) dst[32 * i + lane] = make_longlong2(g[i], h[i]);
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int e = 32 * i + lane;
    tl[e + (e >> 3)] = make_int2(g[i], h[i]);
  }
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int e = 8 * lane + i;
    const int2 v = tl[e + (e >> 3)];
    g[i] = v.x;
    h[i] = v.y;
  }
  __syncwarp();  // the tile is reused by the warp's next item
  const RoundParams rp = *A.rp;
  eval_node<int, HAS_MISSING>(A, node, j, lane, g, h, rp, nodeG, nodeH, nodeTP);
}

// Persistent warps over the level's narrow list (nodes with <= kmax global rows, from the plan).
template <bool HAS_MISSING>
__global__ void __launch_bounds__(kEvalWarps * 32, OOCGB_EVAL_NARROW_MINB) k_eval_narrow(EvalArgs A) {
  __shared__ int2 tile2[kEvalWarps][256 + 32];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int n_items = A.ctl->n_en * A.mf;
  if (n_items <= 0) return;  // (also mf = 0: a rank with no features)
  const int nw = (int)(gridDim.x * blockDim.x) >> 5;
  int t = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  int e = t / A.mf, jj = t - e * A.mf;  // item t = (entry e, feature f0 + jj), advanced by nw
  const int de = nw / A.mf, dj = nw - de * A.mf;
  for (; t < n_items; t += nw) {
    const int4 en = A.ent[A.ent_cap + e];
    eval_item_narrow<HAS_MISSING>(A, en.x, en.y, en.z, A.f0 + jj, lane, tile2[wib]);
    e += de;
    jj += dj;
    if (jj >= A.mf) { jj -= A.mf; ++e; }
  }
}

// ---------------------------------------------------------------------------------------------
// General list (nodes with > kmax rows, and every node of a streamed level): these items are few
// (config 2: the root's m, then the one or two large nodes of a level) and each is a latency
// chain (chunk sums, int64 scans, exact double gains), so one 128-thread block works on one
// (pair, feature j, side) item: thread t owns the consecutive bins 2t, 2t + 1 (coalesced 16-B
// partial loads and 32-B int64 loads/stores, no transpose), block scans in int64, the same float
// pre-filter and exact double pass as eval_node_impl, and a block argmax with the same order
// (larger gain, then lower key 2 b + dir).  The results are those of the warp version: every
// sum is the same exact integer, every float and double operation the same.
// Measured (config 2, cold-cache launch list): root 19.9 -> 12.5 us, level 1 15.4 -> 14.9 us, but
// slower where a level has several large nodes (level 5: 14.8 -> 20.5 us: a block per item has
// less throughput than four warps on four items), so it runs where every item gets its own
// block: levels whose general list fits one wave (the root; OOCGB_EVAL_WIDE_BLOCK=0: never).
#ifndef OOCGB_EVAL_WIDE_BLOCK
#define OOCGB_EVAL_WIDE_BLOCK 1
#endif
constexpr int kBlkThreads = 128, kBlkPerSm = 4, kBlkChunkUnroll = 4;
struct BlkShared {
  long long wg[kBlkThreads / 32], wh[kBlkThreads / 32];  // warp totals for the block scan
  float wT[kBlkThreads / 32];                            // warp max of T_f
  double bg[kBlkThreads / 32];                           // warp best (gain, key)
  int bk[kBlkThreads / 32];
  long long Gm, Hm;                                      // the missing bin's sums (R27)
  int win;                                               // the block's winning key
};

__device__ __forceinline__ long long warp_incl_scan_ll(long long v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long u = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

template <bool HAS_MISSING>
__device__ __forceinline__ void eval_item_blk(const EvalArgs &A, int p, int side, int node, int j, BlkShared &S) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const Pair P = A.pairs[p];  // (the node comes with the entry)
  if (node < 0) return;                                // uniform over the block
  if (A.streamed && A.dn[node].feature == -2) return;  // streamed levels list every slot
  const long long G = A.dn[node].Gq, H = A.dn[node].Hq;
  const double tP = A.dn[node].tP;
  const size_t hsz = (size_t)A.hm * kBins * 2;
  const int jl = j - A.f0;
  const size_t dsz = (size_t)A.m * kBins * 2;
  long long g[2], h[2];
  long long pg[2] = {0, 0}, ph[2] = {0, 0};
  if (side) {  // parent first so its loads overlap the chunk loads
    const int ps = P.parent - level_first(A.d - 1);
    if (P.compact & 1) {
      const int4 v = __ldg(reinterpret_cast<const int4 *>(A.phist_prev + (size_t)ps * hsz) + (size_t)jl * (kBins / 2) + tid);
      pg[0] = v.x; ph[0] = v.y; pg[1] = v.z; ph[1] = v.w;
    } else {
      const longlong2 *src = reinterpret_cast<const longlong2 *>(A.phist_prev + (size_t)ps * hsz + (size_t)jl * kBins * 2) + 2 * tid;
      const longlong2 a = __ldg(src), b = __ldg(src + 1);
      pg[0] = a.x; ph[0] = a.y; pg[1] = b.x; ph[1] = b.y;
    }
  }
  if (A.built64) {
    const longlong2 *src = reinterpret_cast<const longlong2 *>(A.built64 + (size_t)p * hsz + (size_t)jl * kBins * 2) + 2 * tid;
    const longlong2 a = src[0], b = src[1];
    g[0] = a.x; h[0] = a.y; g[1] = b.x; h[1] = b.y;
  } else {
    g[0] = g[1] = h[0] = h[1] = 0;
    const size_t cstride = (size_t)A.n_fg * kFG * kBins / 2;  // int4 (= 2 bins) between chunks
    const int4 *src0 = reinterpret_cast<const int4 *>(A.partial) +
                       (((size_t)P.chunk_base * A.n_fg + j / kFG) * kFG + (j % kFG)) * (kBins / 2) + tid;
    int c = 0;
    for (; c + kBlkChunkUnroll <= P.n_chunks; c += kBlkChunkUnroll) {
      int4 v[kBlkChunkUnroll];
#pragma unroll
      for (int u = 0; u < kBlkChunkUnroll; ++u) v[u] = __ldg(src0 + (c + u) * cstride);
#pragma unroll
      for (int u = 0; u < kBlkChunkUnroll; ++u) { g[0] += v[u].x; h[0] += v[u].y; g[1] += v[u].z; h[1] += v[u].w; }
    }
    for (; c < P.n_chunks; ++c) {
      const int4 v = __ldg(src0 + c * cstride);
      g[0] += v.x; h[0] += v.y; g[1] += v.z; h[1] += v.w;
    }
  }
  if (side) {
#pragma unroll
    for (int i = 0; i < 2; ++i) { g[i] = pg[i] - g[i]; h[i] = ph[i] - h[i]; }
  }
  const int f_d = level_first(A.d);
  if (A.d <= A.D - 2 && !A.streamed) {
    if (P.compact & (side ? 4 : 2)) {
      int4 *dst = reinterpret_cast<int4 *>(A.phist_next + (size_t)(node - f_d) * hsz) + (size_t)jl * (kBins / 2) + tid;
      *dst = make_int4((int)g[0], (int)h[0], (int)g[1], (int)h[1]);
    } else {
      longlong2 *dst = reinterpret_cast<longlong2 *>(A.phist_next + (size_t)(node - f_d) * hsz + (size_t)jl * kBins * 2) + 2 * tid;
      dst[0] = make_longlong2(g[0], h[0]);
      dst[1] = make_longlong2(g[1], h[1]);
    }
  }
  if (A.dbg) {
    longlong2 *dst = reinterpret_cast<longlong2 *>(A.dbg + (size_t)node * dsz + (size_t)j * kBins * 2) + 2 * tid;
    dst[0] = make_longlong2(g[0], h[0]);
    dst[1] = make_longlong2(g[1], h[1]);
  }
  // block exclusive scan of the thread's (g, h) pair sums
  const long long ig = warp_incl_scan_ll(g[0] + g[1], lane), ih = warp_incl_scan_ll(h[0] + h[1], lane);
  if (lane == 31) { S.wg[w] = ig; S.wh[w] = ih; }
  if (HAS_MISSING && tid == kBlkThreads - 1) { S.Gm = g[1]; S.Hm = h[1]; }  // bin 255
  __syncthreads();
  long long eg = ig - (g[0] + g[1]), eh = ih - (h[0] + h[1]);
#pragma unroll
  for (int u = 0; u < kBlkThreads / 32; ++u)
    if (u < w) { eg += S.wg[u]; eh += S.wh[u]; }
  long long Gm = 0, Hm = 0;
  if (HAS_MISSING) { Gm = S.Gm; Hm = S.Hm; }
  const bool miss = HAS_MISSING && (Gm != 0 || Hm != 0);  // uniform over the block
  const RoundParams &rp = *A.rp;
  const int B = A.cut_ptrs[j + 1] - A.cut_ptrs[j];
  const long long hmin = rp.h_min, hmax = H - rp.h_min;
  const float lq = rp.fold_lq;
  // pass 1: float T of the thread's candidates (see eval_node_impl for the bound and the rules)
  float tv[2][2];
  unsigned vmask = 0;
  float Tmax = -INFINITY;
  long long GL = eg, HL = eh;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    GL += g[i];
    HL += h[i];
    const int b = 2 * tid + i;
    const bool vb = b <= B - 2 && ((g[i] | h[i]) != 0 || b == 0);
#pragma unroll
    for (int dir = 0; dir < 2; ++dir) {
      if (dir == 1 && !miss) { tv[i][1] = -INFINITY; continue; }
      const long long GLx = dir ? GL + Gm : GL, HLx = dir ? HL + Hm : HL;
      const bool v = vb && HLx >= hmin && HLx <= hmax;
      const float GLf = (float)GLx, HLf = (float)HLx, GRf = (float)(G - GLx), HRf = (float)(H - HLx);
      const float T = GLf * GLf * frcp_ftz(HLf + lq) + GRf * GRf * frcp_ftz(HRf + lq);
      const bool fin = T < INFINITY;
      vmask |= v ? 1u << (2 * i + dir) : 0u;
      tv[i][dir] = v ? (fin ? T : INFINITY) : -INFINITY;
      Tmax = fmaxf(Tmax, (v && fin) ? T : -INFINITY);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) Tmax = fmaxf(Tmax, __shfl_xor_sync(0xffffffffu, Tmax, o));
  if (lane == 0) S.wT[w] = Tmax;
  __syncthreads();
#pragma unroll
  for (int u = 0; u < kBlkThreads / 32; ++u) Tmax = fmaxf(Tmax, S.wT[u]);
  const float thr = rp.prefilter ? Tmax * (1.0f - 0x1p-18f) : -INFINITY;
  // pass 2: exact double gains of the survivors, in key order
  double best = 0.0;
  int bkey = 0x7fffffff, have = 0;
  long long bGL = 0, bHL = 0;
  GL = eg;
  HL = eh;
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    GL += g[i];
    HL += h[i];
#pragma unroll
    for (int dir = 0; dir < 2; ++dir) {
      if (((vmask >> (2 * i + dir)) & 1u) && tv[i][dir] >= thr) {
        const long long GLx = dir ? GL + Gm : GL, HLx = dir ? HL + Hm : HL;
        const double gain = gain_exact(GLx, HLx, G, H, tP, rp.sg_inv, rp.sh_inv, A.lambda, A.gamma);
        if (!have || gain > best) {
          have = 1; best = gain; bkey = 2 * (2 * tid + i) + dir; bGL = GLx; bHL = HLx;
        }
      }
    }
  }
  // block argmax over (gain, key): warp shuffles only where a warp has more than one survivor
  double bg = have ? best : -INFINITY;
  int bb = have ? bkey : 0x7fffffff;
  const unsigned hv = __ballot_sync(0xffffffffu, have);
  if (hv & (hv - 1)) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double og = __shfl_xor_sync(0xffffffffu, bg, o);
      const int ob = __shfl_xor_sync(0xffffffffu, bb, o);
      if (og > bg || (og == bg && ob < bb)) { bg = og; bb = ob; }
    }
  } else if (hv) {
    const int src = __ffs(hv) - 1;
    bg = __shfl_sync(0xffffffffu, bg, src);
    bb = __shfl_sync(0xffffffffu, bb, src);
  }
  if (lane == 0) { S.bg[w] = bg; S.bk[w] = bb; }
  __syncthreads();
  double wg = S.bg[0];
  int wk = S.bk[0];
#pragma unroll
  for (int u = 1; u < kBlkThreads / 32; ++u)
    if (S.bg[u] > wg || (S.bg[u] == wg && S.bk[u] < wk)) { wg = S.bg[u]; wk = S.bk[u]; }
  const bool any = wk != 0x7fffffff;
  const int owner = any ? (wk >> 2) : 0;  // 4 keys (2 bins x 2 directions) per thread
  if (tid == owner) {
    const int slot = node - level_first(A.d);
    Cand cd;
    cd.gain = any ? wg : 0.0;
    cd.bin = wk;
    cd.valid = any ? 1 : 0;
    cd.GL = any ? bGL : 0;
    cd.HL = any ? bHL : 0;
    A.cand[cand_index_own(A.msl, A.max_slots, A.crank, slot, j)] = cd;
  }
  __syncthreads();  // the shared block is reused by the next item
}

// Persistent blocks over the general list: item t = (entry t / mf, feature t mod mf).
template <bool HAS_MISSING>
__global__ void __launch_bounds__(kBlkThreads, kBlkPerSm) k_eval_blk(EvalArgs A) {
  __shared__ BlkShared S;
  const int n_items = A.ctl->n_ew * A.mf;
  if (n_items <= 0) return;
  int t = blockIdx.x;
  int e = t / A.mf, jj = t - e * A.mf;
  const int de = (int)gridDim.x / A.mf, dj = (int)gridDim.x - de * A.mf;
  for (; t < n_items; t += gridDim.x) {
    const int4 en = A.ent[e];
    eval_item_blk<HAS_MISSING>(A, en.x, en.y, en.z, A.f0 + jj, S);
    e += de;
    jj += dj;
    if (jj >= A.mf) { jj -= A.mf; ++e; }
  }
}

// Split decision per node at depth d: argmax over features (ties: lowest feature, R13),
// split iff gain > 0; children get their exact sums and Eq. 6 leaf values.  One 256-thread
// block per node (blockIdx.x = 2 pair + side).
struct BestSplit {
  double gain;
  int have, j, bin;
  long long GL, HL;
  int cp;  // k_finalize: cut_ptrs[j] (loaded with the candidate)
};
__device__ __forceinline__ bool better(const BestSplit &a, const BestSplit &b) {  // a beats b
  return a.have && (!b.have || a.gain > b.gain || (a.gain == b.gain && a.j < b.j));
}
__device__ __forceinline__ BestSplit shfl_best(const BestSplit &x, int o) {
  BestSplit y;
  y.gain = __shfl_down_sync(0xffffffffu, x.gain, o);
  y.have = __shfl_down_sync(0xffffffffu, x.have, o);
  y.j = __shfl_down_sync(0xffffffffu, x.j, o);
  y.bin = __shfl_down_sync(0xffffffffu, x.bin, o);
  y.GL = __shfl_down_sync(0xffffffffu, x.GL, o);
  y.HL = __shfl_down_sync(0xffffffffu, x.HL, o);
  y.cp = __shfl_down_sync(0xffffffffu, x.cp, o);
  return y;
}

__global__ void __launch_bounds__(256)
k_finalize(int d, int m, int msl, int max_slots, const Pair *__restrict__ pairs, LevelCtl *ctl,
           const Cand *__restrict__ cand, DNode *dn, const float *__restrict__ cut_values,
           const int *__restrict__ cut_ptrs, const RoundParams *__restrict__ rp, double lambda, double eta,
           Seg *segs) {
  // block b decides slot b of the level: the node index needs no pair record, so the candidate
  // loads start at once; a slot whose node is not an unsplit node of this level (feature -2:
  // absent) is dropped after them
  (void)pairs;
  const int slot = blockIdx.x;
  const int node = level_first(d) + slot;
  const int feat0 = dn[node].feature;
  const long long Gq0 = dn[node].Gq, Hq0 = dn[node].Hq, seg0 = dn[node].seg;  // early: used at the end
  BestSplit best{0.0, 0, 0x7fffffff, 0, 0, 0, 0};
  // candidate (slot, j) at cand_index(msl, max_slots, slot, j), the owner block r = j / msl
  // carried along instead of divided per candidate
  int r = (int)threadIdx.x / msl, jr = (int)threadIdx.x - r * msl;
  for (int j = threadIdx.x; j < m; j += blockDim.x) {
    const Cand cd = cand[((size_t)r * max_slots + slot) * msl + jr];
    BestSplit x{cd.gain, cd.valid, j, cd.bin, cd.GL, cd.HL, __ldg(cut_ptrs + j)};
    if (better(x, best)) best = x;
    jr += blockDim.x;
    while (jr >= msl) { jr -= msl; ++r; }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    BestSplit y = shfl_best(best, o);
    if (better(y, best)) best = y;
  }
  __shared__ BestSplit s_best[8];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) s_best[w] = best;
  __syncthreads();
  if (feat0 != -1) return;  // absent slot (uniform over the block)
  if (threadIdx.x == 0) {
    for (int u = 1; u < (int)(blockDim.x >> 5); ++u)
      if (better(s_best[u], best)) best = s_best[u];
    if (best.have && best.gain > 0.0) {
      DNode &nd = dn[node];
      nd.feature = best.j;
      nd.split_bin = best.bin >> 1;      // candidate key 2 b + dir (R27)
      nd.default_left = best.bin & 1;
      nd.split_value = cut_values[best.cp + (best.bin >> 1)];
      nd.gain = best.gain;
      if (segs) segs[seg0].dec = seg_dec(best.j, best.bin & 1, best.bin >> 1);  // for the partition
      DNode L{}, R{};
      L.feature = -1;
      R.feature = -1;
      node_fill(L, best.GL, best.HL, rp->sg_inv, rp->sh_inv, lambda, eta, &ctl->error);
      node_fill(R, Gq0 - best.GL, Hq0 - best.HL, rp->sg_inv, rp->sh_inv, lambda, eta, &ctl->error);
      dn[2 * node + 1] = L;
      dn[2 * node + 2] = R;
      atomicAdd(&ctl->n_splits, 1);
    }
  }
}

static void launch_eval(const EvalArgs &A, int max_pairs, oocgb_ctx c, cudaStream_t st) {
  const int num_sms = c->num_sms;
  const int64_t blocks = ((int64_t)max_pairs * std::max(1, A.mf) * 2 + kEvalWarps - 1) / kEvalWarps;
  const unsigned gw = (unsigned)std::min<int64_t>(blocks, (int64_t)num_sms * kEvalBlocksWide);
  const unsigned gn = (unsigned)std::min<int64_t>(blocks, (int64_t)num_sms * OOCGB_EVAL_NARROW_MINB);
  // the general list fits one wave of blocks (the root level: one built node, no sibling)
  const bool blk = OOCGB_EVAL_WIDE_BLOCK && !A.streamed && A.d == 0 && A.mf <= num_sms * kBlkPerSm;
  if (blk) {
    const unsigned gb = (unsigned)std::max(1, A.mf);
    // the root is on exactly one list; root_list (host-known when every row is selected): 1
    // general, 2 narrow, 0 unknown (a sampled graph serves every row count: both launched)
    if (A.has_missing) {  // R27: candidates in both default directions
      if (A.root_list != 2) k_eval_blk<true><<<gb, kBlkThreads, 0, st>>>(A);
      if (A.root_list != 1) k_eval_narrow<true><<<gn, kEvalWarps * 32, 0, st>>>(A);
    } else {
      if (A.root_list != 2) k_eval_blk<false><<<gb, kBlkThreads, 0, st>>>(A);
      if (A.root_list != 1) k_eval_narrow<false><<<gn, kEvalWarps * 32, 0, st>>>(A);
    }
  } else if (A.has_missing) {  // R27: candidates in both default directions
    k_eval<true><<<gw, kEvalWarps * 32, 0, st>>>(A);
    k_eval_narrow<true><<<gn, kEvalWarps * 32, 0, st>>>(A);
  } else {
    k_eval<false><<<gw, kEvalWarps * 32, 0, st>>>(A);
    k_eval_narrow<false><<<gn, kEvalWarps * 32, 0, st>>>(A);
  }
  OOCGB_CK(cudaGetLastError());
  // world > 1: every rank evaluated its feature slice; gather the candidates of all features
  if (c->coll && !A.streamed)
    allgather_i64_inplace(c, reinterpret_cast<long long *>(A.cand),
                          (size_t)A.max_slots * A.msl * (sizeof(Cand) / sizeof(long long)));
  k_finalize<<<(unsigned)(max_pairs * 2), 256, 0, st>>>(A.d, A.m, A.msl, A.max_slots, A.pairs, A.ctl, A.cand, A.dn,
                                                         A.cut_values, A.cut_ptrs, A.rp, A.lambda, A.eta, A.segs);
  OOCGB_CK(cudaGetLastError());
}

// ---------------------------------------------------------------------------------------------
// RepartitionInstances (Alg. 1) in one pass per level.  Rows of a split segment s go
// left (bin <= split_bin) or right; the order of rows inside a child is irrelevant to every
// result (histograms are exact integer sums, the exports are per row), so no global scan is
// needed: each tile reserves, with one atomic per (tile, segment) on the segment's cursors, a
// block of its left rows growing forward from begin_s and a block of its right rows growing
// backward from end_s; inside its blocks a tile keeps ascending position order (locality for the
// next level's gathers).  At the end cur[2s], cur[2s+1] hold the segment's (left, right) counts.
// Rows of unsplit segments stay in place.
__device__ __forceinline__ int seg_of(const Seg *segs, int n_segs, int i) {
  int lo = 0, hi = n_segs - 1;  // last segment with begin <= i (non-empty one containing i)
  while (lo < hi) {
    int mid = (lo + hi + 1) >> 1;
    if (segs[mid].begin <= i) lo = mid; else hi = mid - 1;
  }
  while (lo < n_segs - 1 && segs[lo].begin + segs[lo].count <= i) ++lo;
  return lo;
}

// Segments overlapping one partition tile, staged in shared memory (at most kTileSegs; a tile
// that overlaps more takes the per-thread fallback).
constexpr int kTileSegs = 256;
struct TileSegs {
  int first, count;  // segment range overlapping the tile
  int begin[kTileSegs], end[kTileSegs];
  int feat[kTileSegs], sbin[kTileSegs];
  int l0[kTileSegs], r0[kTileSegs];    // tile-prefix (left, right) at the segment's first position in the tile
  int bl[kTileSegs], br[kTileSegs];    // reserved: left base, right base + count
};

// tile_seg[t] = the non-empty segment containing position t kPartTile (written by the previous
// level's plan); the range may also include empty segments and the one starting at the next
// tile, which no position maps to.
__device__ __forceinline__ void load_tile_segs(TileSegs &T, const Seg *__restrict__ segs, int n_segs,
                                               const DNode *__restrict__ dn, const int *__restrict__ tile_seg,
                                               int tile, int n_tiles) {
  if (threadIdx.x == 0) {
    const int f = tile_seg[tile];
    const int l = tile + 1 < n_tiles ? tile_seg[tile + 1] : n_segs - 1;
    T.first = f;
    T.count = l - f + 1;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < T.count && k < kTileSegs; k += blockDim.x) {
    const Seg S = segs[T.first + k];
    T.begin[k] = S.begin;
    T.end[k] = S.begin + S.count;
    T.feat[k] = S.dec >= 0 ? S.dec >> 10 : -1;     // the decision rides in the segment (one read)
    T.sbin[k] = S.dec >= 0 ? (S.dec & 0x3ff) : 0;   // split_bin | default_left << 9 (R27); bit 8 clear
  }
  __syncthreads();
}

// Block-wide exclusive scan.  Returns the exclusive prefix of v and writes the block total to
// *total.  Contains __syncthreads(); call from all threads.
__device__ int block_excl_scan(int v, int *total) {
  __shared__ int s_w[32];
  __shared__ int s_tot;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) s_w[w] = incl;
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    int x = lane < nw ? s_w[lane] : 0, xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int u = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) xi += u;
    }
    if (lane < nw) s_w[lane] = xi - x;
    if (lane == 31) s_tot = xi;
  }
  __syncthreads();
  const int r = s_w[w] + incl - v;
  *total = s_tot;
  __syncthreads();
  return r;
}

// The same with two alternating buffers and no trailing barrier: call sites pass buf = 0, 1, 0,
// 1, ... so a buffer is rewritten only after the next call's two barriers (plan_level's scans).
__device__ int block_excl_scan2(int v, int *total, int buf) {
  __shared__ int s_w2[2][32];
  __shared__ int s_tot2[2];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  if (lane == 31) s_w2[buf][w] = incl;
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    int x = lane < nw ? s_w2[buf][lane] : 0, xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int u = __shfl_up_sync(0xffffffffu, xi, o);
      if (lane >= o) xi += u;
    }
    if (lane < nw) s_w2[buf][lane] = xi - x;
    if (lane == 31) s_tot2[buf] = xi;
  }
  __syncthreads();
  *total = s_tot2[buf];
  return s_w2[buf][w] + incl - v;
}

struct PlanArgs {
  const Seg *segs;
  Seg *segs_next;
  LevelCtl *ctl;
  DNode *dn;
  const int *cur;
  const long long *seg_cnt;  // global (left, right) counts when world > 1, else null
  int *cur_next;
  Pair *pairs;
  int *tile_seg;
  int2 *chunk_rng;  // histogram chunk -> its position range (k_hist's item lookup)
  const long long *n_dev;  // the sample's rows (device sample state)
  int n_fg, target_items, kmax;
  int4 *ent;        // eval work lists (EvalArgs::ent)
  int ent_cap;
  int last;         // the tree's last level: only segments, children counts and the tile table
};
__device__ void plan_level(const PlanArgs &A, int n_segs);
#ifdef OOCGB_PLAN_TRACE
__device__ unsigned long long g_part_t0 = ~0ull;  // trace build only: first partition block's start
#endif

// One 2048-position tile per block; thread t handles positions t0 + 256 u + t (u < 8), so every
// warp-wide load, gather and store touches consecutive positions (coalesced ridx / q, adjacent
// 32-B rows for the bin gathers, consecutive destinations).  (u, thread) order is position order:
// left/right ranks come from warp ballots plus a 64-entry (u, warp) scan.
__global__ void __launch_bounds__(kPartThreads, 4)
k_part_fused(const long long *__restrict__ n_dev, const Seg *__restrict__ segs, const LevelCtl *__restrict__ ctl,
             const DNode *__restrict__ dn, const uint8_t *__restrict__ bins, size_t pitch, int lgw,
             const int32_t *__restrict__ ridx, const int2 *__restrict__ q, int32_t *__restrict__ ridx_out,
             int2 *__restrict__ q_out, int *__restrict__ cur, const int *__restrict__ tile_seg, int plan_inline,
             PlanArgs PA, int cap) {
  static_assert(kPartTile == 8 * kPartThreads, "8 positions per thread");
#ifdef OOCGB_PLAN_TRACE
  if (threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    atomicMin(&g_part_t0, t);
  }
#endif
  __shared__ TileSegs T;
  __shared__ int s_pre[8][kPartThreads / 32];  // (left | right << 16) per (u, warp), then exclusive prefix
  __shared__ int s_tot;
  const int t0 = blockIdx.x * kPartTile;
  // row ids and gradient pairs first, bounded by the buffers' capacity (not the sample's row
  // count, which is itself a load): both round trips overlap
  int rows[8], sg[8];
  int2 qs[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int p = t0 + u * kPartThreads + threadIdx.x;
    if (p < cap) { rows[u] = ridx ? ridx[p] : p; qs[u] = q[p]; }  // ridx null: identity (level 0)
  }
  const int n_segs = ctl->n_segs;
  const int n = (int)*n_dev;  // the sample's rows (the grid covers the capacity)
  const int n_tiles = (n + kPartTile - 1) / kPartTile;
  const int t1 = min(n, t0 + kPartTile);
  if (t0 < n) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  load_tile_segs(T, segs, n_segs, dn, tile_seg, blockIdx.x, n_tiles);
  const bool staged = T.count <= kTileSegs;
  uint32_t rbits = 0, lbits = 0;  // right / left (of a split segment) per u
  {
    int k = staged ? 0 : -1;
    uint8_t b[8];
    int sb[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int p = t0 + u * kPartThreads + threadIdx.x;
      int f = -1;
      sb[u] = 0;
      sg[u] = 0;
      if (p < t1) {
        if (staged) {
          while (T.end[k] <= p) ++k;
          f = T.feat[k];
          sb[u] = T.sbin[k];
        } else {
          k = k < 0 ? seg_of(segs, n_segs, p) : k;
          while (segs[k].begin + segs[k].count <= p) ++k;
          const int dec = segs[k].dec;
          f = dec >= 0 ? dec >> 10 : -1;
          sb[u] = dec >= 0 ? (dec & 0x3ff) : 0;
        }
        sg[u] = k;
      }
      b[u] = f >= 0 ? bins[(size_t)(f >> lgw) * pitch + ((size_t)rows[u] << lgw) + (f & ((1 << lgw) - 1))] : 0;
      if (f >= 0) sb[u] |= 0x100;  // split marker
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (sb[u] & 0x100) {
        if (goes_left(b[u], sb[u] & 0xff, (sb[u] >> 9) & 1)) lbits |= 1u << u; else rbits |= 1u << u;
      }
  }
  const uint32_t lt = (1u << lane) - 1u;
  if (staged) {
    uint32_t balL[8], balR[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      balL[u] = __ballot_sync(0xffffffffu, (lbits >> u) & 1);
      balR[u] = __ballot_sync(0xffffffffu, (rbits >> u) & 1);
    }
    if (lane == 0) {
#pragma unroll
      for (int u = 0; u < 8; ++u) s_pre[u][wid] = __popc(balL[u]) | (__popc(balR[u]) << 16);
    }
    __syncthreads();
    if (wid == 0) {  // exclusive scan of the 64 (u, warp) counts in position order
      const int v0 = (&s_pre[0][0])[2 * lane], v1 = (&s_pre[0][0])[2 * lane + 1];
      int incl = v0 + v1;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int ex = incl - v0 - v1;
      (&s_pre[0][0])[2 * lane] = ex;
      (&s_pre[0][0])[2 * lane + 1] = ex + v0;
      if (lane == 31) s_tot = incl;
    }
    __syncthreads();
    int exL[8], exR[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int pre = s_pre[u][wid];
      exL[u] = (pre & 0xffff) + __popc(balL[u] & lt);
      exR[u] = (pre >> 16) + __popc(balR[u] & lt);
      const int p = t0 + u * kPartThreads + threadIdx.x;
      if (p < t1 && p == max(T.begin[sg[u]], t0)) {  // first position of the segment in this tile
        T.l0[sg[u]] = exL[u];
        T.r0[sg[u]] = exR[u];
      }
    }
    __syncthreads();
    // per segment: the tile's (left, right) rows = prefix difference to the next non-empty one
    for (int k = threadIdx.x; k < T.count; k += blockDim.x) {
      const int f0 = max(T.begin[k], t0);
      if (T.feat[k] < 0 || f0 >= min(T.end[k], t1)) continue;
      int k2 = k + 1;
      while (k2 < T.count && max(T.begin[k2], t0) >= min(T.end[k2], t1)) ++k2;
      const int nxt = k2 < T.count ? (T.l0[k2] | (T.r0[k2] << 16)) : s_tot;
      const int cl = (nxt & 0xffff) - T.l0[k], cr = (nxt >> 16) - T.r0[k];
      const int s = T.first + k;
      T.bl[k] = cl ? atomicAdd(&cur[2 * s], cl) : 0;
      T.br[k] = (cr ? atomicAdd(&cur[2 * s + 1], cr) : 0) + cr;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int p = t0 + u * kPartThreads + threadIdx.x;
      if (p >= t1) break;
      const int k = sg[u];
      int pos = p;
      if ((lbits >> u) & 1) pos = T.begin[k] + T.bl[k] + (exL[u] - T.l0[k]);
      else if ((rbits >> u) & 1) pos = T.end[k] - T.br[k] + (exR[u] - T.r0[k]);
      ridx_out[pos] = rows[u];
      q_out[pos] = qs[u];
    }
  } else {
    // many segments in the tile (deep trees, tiny nodes): one global reservation per row
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int p = t0 + u * kPartThreads + threadIdx.x;
      if (p >= t1) break;
      int pos = p;
      if ((lbits >> u) & 1) pos = segs[sg[u]].begin + atomicAdd(&cur[2 * sg[u]], 1);
      else if ((rbits >> u) & 1)
        pos = segs[sg[u]].begin + segs[sg[u]].count - 1 - atomicAdd(&cur[2 * sg[u] + 1], 1);
      ridx_out[pos] = rows[u];
      q_out[pos] = qs[u];
    }
  }
  }  // t0 < n
  if (!plan_inline) return;
  // world == 1: the last tile to finish plans the next level (its cursors are final).  The plan
  // reads only the cursors (atomics, at L2); the barrier + one thread's fence order this block's
  // cursor atomics before its ticket (fences are cumulative over the barrier).
  __shared__ int s_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&PA.ctl->part_done, 1) == (int)gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
#ifdef OOCGB_PLAN_TRACE
  unsigned long long tp0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tp0));
#endif
  plan_level(PA, n_segs);
  if (threadIdx.x == 0) PA.ctl->part_done = 0;
#ifdef OOCGB_PLAN_TRACE
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long tp1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tp1));
    printf("PLANTRACE segs %d plan_ns %llu since_first_block_ns %llu\n", n_segs, tp1 - tp0, tp1 - g_part_t0);
    g_part_t0 = ~0ull;
  }
#endif
}

// world > 1: the local (left, right) counts of the level's segments, widened for the all-reduce
// (entries past n_segs are zero on every rank).
__global__ void k_part_counts(const int *__restrict__ cur, const LevelCtl *__restrict__ ctl, int len,
                              long long *__restrict__ seg_cnt) {
  const int n2 = 2 * ctl->n_segs;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < len; i += gridDim.x * blockDim.x)
    seg_cnt[i] = i < n2 ? cur[i] : 0;
}

// Single block, after the partition: children n_rows (global counts: seg_cnt when world > 1,
// else the local cursors), next level's segments (split -> 2, leaf -> pass-through 1) and sibling
// pairs (built = child with fewer global rows, ties left, R17), histogram chunking; zeroes the
// next level's cursors.
// General plan (any number of segments): block-strided loops; reads back what it wrote.
__device__ void plan_level_loop(const PlanArgs &A) {
  const Seg *__restrict__ segs = A.segs;
  Seg *__restrict__ segs_next = A.segs_next;
  LevelCtl *ctl = A.ctl;
  DNode *dn = A.dn;
  const long long *__restrict__ seg_cnt = A.seg_cnt;
  Pair *__restrict__ pairs = A.pairs;
  const int n_fg = A.n_fg, target_items = A.target_items, kmax = A.kmax;
  const int T = blockDim.x;
  const int n_segs = ctl->n_segs;
  int nseg_carry = 0, npair_carry = 0;
  long long rows_local = 0;
  for (int base = 0; base < n_segs; base += T) {
    const int s = base + threadIdx.x;
    int split = 0;
    if (s < n_segs) split = segs[s].dec >= 0;
    int tot_s, tot_p;
    const int es = block_excl_scan(s < n_segs ? 1 + split : 0, &tot_s);
    const int ep = block_excl_scan(split, &tot_p);
    if (s < n_segs) {
      const Seg S = segs[s];
      const int ns = nseg_carry + es, np = npair_carry + ep;
      if (split) {
        const int nl = __ldcg(A.cur + 2 * s), nr = __ldcg(A.cur + 2 * s + 1);  // final atomics (L2)
        const long long gl = seg_cnt ? seg_cnt[2 * s] : nl, gr = seg_cnt ? seg_cnt[2 * s + 1] : nr;
        dn[2 * S.node + 1].n_rows = gl;
        dn[2 * S.node + 2].n_rows = gr;
        segs_next[ns] = Seg{S.begin, nl, 2 * S.node + 1, -1};
        segs_next[ns + 1] = Seg{S.begin + nl, nr, 2 * S.node + 2, -1};
        dn[2 * S.node + 1].seg = ns;
        dn[2 * S.node + 2].seg = ns + 1;
        Pair pr;
        pr.parent = S.node;
        long long gb, gd;
        if (gl <= gr) { pr.built = 2 * S.node + 1; pr.derived = 2 * S.node + 2; pr.begin = S.begin; pr.count = nl; gb = gl; gd = gr; }
        else { pr.built = 2 * S.node + 2; pr.derived = 2 * S.node + 1; pr.begin = S.begin + nl; pr.count = nr; gb = gr; gd = gl; }
        pr.chunk_base = 0; pr.n_chunks = 0; pr.chunk_rows = 0;
        // s32 histograms are exact for nodes with <= kmax rows (|q| <= 2^quant_bits)
        pr.compact = ((gl + gr) <= kmax ? 1 : 0) | (gb <= kmax ? 2 : 0) | (gd <= kmax ? 4 : 0);
        pairs[np] = pr;
        rows_local += pr.count;
      } else {
        segs_next[ns] = S;
      }
    }
    nseg_carry += tot_s;
    npair_carry += tot_p;
  }
  for (int i = threadIdx.x; i < 2 * nseg_carry; i += T) A.cur_next[i] = 0;
  // tile -> first segment table of the next level (segs_next written above by this block)
  __syncthreads();
  const int n_tiles = (int)((*A.n_dev + kPartTile - 1) / kPartTile);
  for (int sn = threadIdx.x; sn < nseg_carry; sn += T) {
    const Seg S = segs_next[sn];
    if (S.count == 0) continue;
    for (int t = (S.begin + kPartTile - 1) / kPartTile; t < n_tiles && t * kPartTile < S.begin + S.count; ++t)
      A.tile_seg[t] = sn;
  }
  // chunk size: whole waves of k_hist items, within [1024, kmax] rows (s32 bound)
  __shared__ unsigned long long s_rows;
  if (threadIdx.x == 0) s_rows = 0;
  __syncthreads();
  atomicAdd(&s_rows, (unsigned long long)rows_local);
  __syncthreads();
  const int n_pairs = npair_carry;
  // eval work lists: (pair, side) of nodes with <= kmax global rows -> narrow, else general
  {
    int ew_carry = 0, en_carry = 0;
    for (int base = 0; base < n_pairs; base += T) {
      const int p = base + threadIdx.x;
      int nn = 0;
      long long rb = 0, rd = 0;
      if (p < n_pairs) {
        rb = dn[pairs[p].built].n_rows;
        rd = dn[pairs[p].derived].n_rows;
        nn = (rb <= kmax) + (rd <= kmax);
      }
      int tw, tn;
      const int ew = block_excl_scan(p < n_pairs ? 2 - nn : 0, &tw);
      const int en = block_excl_scan(nn, &tn);
      if (p < n_pairs) {
        int iw = ew_carry + ew, in = en_carry + en;
        const int4 eb = make_int4(p, 0, pairs[p].built, 0), ed = make_int4(p, 1, pairs[p].derived, 0);
        if (rb <= kmax) A.ent[A.ent_cap + in++] = eb; else A.ent[iw++] = eb;
        if (rd <= kmax) A.ent[A.ent_cap + in] = ed; else A.ent[iw] = ed;
      }
      ew_carry += tw;
      en_carry += tn;
    }
    if (threadIdx.x == 0) { ctl->n_ew = ew_carry; ctl->n_en = en_carry; }
  }
  const long long cr = hist_chunk_rows((long long)s_rows, n_pairs, n_fg, target_items, kmax);
  int chunk_carry = 0;
  for (int base = 0; base < n_pairs; base += T) {
    const int p = base + threadIdx.x;
    const int cnt = p < n_pairs ? pairs[p].count : 0;
    const int nch = (int)((cnt + cr - 1) / cr);
    int tot;
    const int e = block_excl_scan(nch, &tot);
    if (p < n_pairs) {
      pairs[p].chunk_base = chunk_carry + e;
      pairs[p].n_chunks = nch;
      pairs[p].chunk_rows = nch > 0 ? (cnt + nch - 1) / nch : (int)cr;  // equal chunks
      const int b0 = pairs[p].begin, crp = nch > 0 ? (cnt + nch - 1) / nch : 0;
      for (int c = 0; c < nch; ++c) A.chunk_rng[chunk_carry + e + c] = make_int2(b0 + c * crp, min(b0 + cnt, b0 + (c + 1) * crp));
    }
    chunk_carry += tot;
  }
  if (threadIdx.x == 0) {
    ctl->n_pairs = n_pairs;
    ctl->n_items = chunk_carry * n_fg;
    ctl->n_segs = nseg_carry;
    ctl->n_splits = 0;
    ctl->hist_next = 0;
  }
}


// Plan with one thread per segment (n_segs <= blockDim.x, every level of a depth <= 9 tree at
// the last-block size of 256): each thread loads its segment, cursors and node decision once and
// writes what derives from them (children segments and cursors, its pair with chunking) without
// reading back global memory: three dependent round trips; then the tile -> segment and chunk ->
// pair tables are filled block-wide (a single thread filling a shallow level's ~250 tiles per
// segment serially was ~19 us of tail on one SM).
__device__ void plan_level(const PlanArgs &A, int n_segs) {
  if (n_segs > (int)blockDim.x) {
    plan_level_loop(A);
    return;
  }
  const int s = threadIdx.x;
  Seg S{};
  int split = 0, nl = 0, nr = 0;
  long long gl = 0, gr = 0;
  if (s < n_segs) {
    S = A.segs[s];
    nl = __ldcg(A.cur + 2 * s);  // final cursor atomics (L2)
    nr = __ldcg(A.cur + 2 * s + 1);
    if (A.seg_cnt) { gl = A.seg_cnt[2 * s]; gr = A.seg_cnt[2 * s + 1]; }
    split = S.dec >= 0;
  }
  if (!A.seg_cnt) { gl = nl; gr = nr; }
  int tot_s, tot_p;
  // one scan of two packed 16-bit counts (next segments | pairs << 16; totals <= 512)
  int tot_sp;
  const int nsp = block_excl_scan2((s < n_segs ? 1 + split : 0) | (split << 16), &tot_sp, 0);
  const int ns = nsp & 0xffff, np = nsp >> 16;
  tot_s = tot_sp & 0xffff;
  tot_p = tot_sp >> 16;
  Pair pr{};
  const int n_tiles = (int)((*A.n_dev + kPartTile - 1) / kPartTile);
  // next-level segment starts staged in shared memory for the tile table (filled block-wide below)
  __shared__ int s_begin[2 * 1024];
  auto emit = [&](int idx, const Seg &C) {
    A.segs_next[idx] = C;
    A.cur_next[2 * idx] = 0;
    A.cur_next[2 * idx + 1] = 0;
    s_begin[idx] = C.begin;
  };
  if (s < n_segs) {
    if (split) {
      A.dn[2 * S.node + 1].n_rows = gl;
      A.dn[2 * S.node + 2].n_rows = gr;
      emit(ns, Seg{S.begin, nl, 2 * S.node + 1, -1});
      emit(ns + 1, Seg{S.begin + nl, nr, 2 * S.node + 2, -1});
      A.dn[2 * S.node + 1].seg = ns;
      A.dn[2 * S.node + 2].seg = ns + 1;
      pr.parent = S.node;
      long long gb, gd;
      if (gl <= gr) { pr.built = 2 * S.node + 1; pr.derived = 2 * S.node + 2; pr.begin = S.begin; pr.count = nl; gb = gl; gd = gr; }
      else { pr.built = 2 * S.node + 2; pr.derived = 2 * S.node + 1; pr.begin = S.begin + nl; pr.count = nr; gb = gr; gd = gl; }
      // s32 histograms are exact for nodes with <= kmax rows (|q| <= 2^quant_bits)
      pr.compact = ((gl + gr) <= A.kmax ? 1 : 0) | (gb <= A.kmax ? 2 : 0) | (gd <= A.kmax ? 4 : 0);
    } else {
      emit(ns, S);
    }
  }
  if (A.last) {  // no next level: its pairs, work lists and chunking are never read
    __syncthreads();
    for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) {
      int lo = 0, hi = tot_s - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (s_begin[mid] <= t * kPartTile) lo = mid; else hi = mid - 1;
      }
      A.tile_seg[t] = lo;
    }
    if (threadIdx.x == 0) {
      A.ctl->n_pairs = 0;
      A.ctl->n_items = 0;
      A.ctl->n_segs = tot_s;
      A.ctl->n_splits = 0;
      A.ctl->hist_next = 0;
      A.ctl->n_ew = 0;
      A.ctl->n_en = 0;
    }
    return;
  }
  // eval work lists: (pair, side) of nodes with <= kmax global rows -> narrow, else general
  {
    long long gb = 0, gd = 0;
    if (split) { gb = pr.built == 2 * S.node + 1 ? gl : gr; gd = pr.built == 2 * S.node + 1 ? gr : gl; }
    const int nn = split ? (gb <= A.kmax) + (gd <= A.kmax) : 0;
    int tw, tn;
    int twn;  // one scan of (general | narrow << 16) entry counts (totals <= 512)
    const int ewn = block_excl_scan2((split ? 2 - nn : 0) | (nn << 16), &twn, 1);
    const int ew = ewn & 0xffff, en = ewn >> 16;
    tw = twn & 0xffff;
    tn = twn >> 16;
    if (split) {
      int iw = ew, in = en;
      const int4 eb = make_int4(np, 0, pr.built, 0), ed = make_int4(np, 1, pr.derived, 0);
      if (gb <= A.kmax) A.ent[A.ent_cap + in++] = eb; else A.ent[iw++] = eb;
      if (gd <= A.kmax) A.ent[A.ent_cap + in] = ed; else A.ent[iw] = ed;
    }
    if (threadIdx.x == 0) { A.ctl->n_ew = tw; A.ctl->n_en = tn; }
  }
  // chunk size from the level's built rows (whole waves of k_hist items), equal chunks per pair;
  // chunks are numbered in decreasing chunk size (longest-processing-time-first order for
  // k_hist's dynamic item fetch; ties: pair order)
  int tot_rows;
  block_excl_scan2(split ? pr.count : 0, &tot_rows, 0);
  const long long cr = hist_chunk_rows(tot_rows, tot_p, A.n_fg, A.target_items, A.kmax);
  const int nch = split ? (int)((pr.count + cr - 1) / cr) : 0;
  const int crp = nch > 0 ? (pr.count + nch - 1) / nch : 0;
  __shared__ int s_cbase[1024];  // by LPT rank: first chunk
  __shared__ int s_key[1024];    // by pair: chunk rows; then by LPT rank: pair
  if (split) s_key[np] = crp;
  __syncthreads();
  int rank = 0;
  if (split) {
    for (int q = 0; q < tot_p; ++q) {
      const int kq = s_key[q];
      rank += (kq > crp || (kq == crp && q < np)) ? 1 : 0;
    }
  }
  __syncthreads();
  __shared__ int s_pb[1024], s_pe[1024], s_pr[1024];  // by LPT rank: pair begin, end, chunk rows
  if (split) { s_key[rank] = np; s_cbase[rank] = nch; s_pb[rank] = pr.begin; s_pe[rank] = pr.begin + pr.count; s_pr[rank] = crp; }
  __syncthreads();
  int tot_c;
  const int cb = block_excl_scan2(s < tot_p ? s_cbase[s] : 0, &tot_c, 1);  // scan in rank order
  if (s < tot_p) s_cbase[s] = cb;
  __syncthreads();
  if (split) {
    pr.chunk_base = s_cbase[rank];
    pr.n_chunks = nch;
    pr.chunk_rows = nch > 0 ? crp : (int)cr;
    A.pairs[np] = pr;
  }
  __syncthreads();
  // tile -> segment containing the tile's first position: the last segment starting at or
  // before it (that one is non-empty); chunk -> pair: the last pair whose chunks start at or
  // before it.  Block-wide binary searches in shared memory.
  for (int t = threadIdx.x; t < n_tiles; t += blockDim.x) {
    int lo = 0, hi = tot_s - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_begin[mid] <= t * kPartTile) lo = mid; else hi = mid - 1;
    }
    A.tile_seg[t] = lo;
  }
  for (int c = threadIdx.x; c < tot_c; c += blockDim.x) {
    int lo = 0, hi = tot_p - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (s_cbase[mid] <= c) lo = mid; else hi = mid - 1;
    }
    const int b0 = s_pb[lo] + (c - s_cbase[lo]) * s_pr[lo];
    A.chunk_rng[c] = make_int2(b0, min(s_pe[lo], b0 + s_pr[lo]));
  }
  if (threadIdx.x == 0) {
    A.ctl->n_pairs = tot_p;
    A.ctl->n_items = tot_c * A.n_fg;
    A.ctl->n_segs = tot_s;
    A.ctl->n_splits = 0;
    A.ctl->hist_next = 0;
  }
}

__global__ void __launch_bounds__(1024) k_part_plan(PlanArgs A) { plan_level(A, A.ctl->n_segs); }

// ---------------------------------------------------------------------------------------------
// Prediction (Eq. 1): margin[row] += leaf(tree, bins_row), binned traversal, per tree in order.
// Layout-generic addressing: symbol (row i, f) at bins + i * row_step + (f >> lgw) * pitch +
// (f & (2^lgw - 1)) (tiled device page: row_step = gw, pitch rpp * gw, lgw = log2 gw; row-major
// pinned page: row_step = stride, pitch 32, lgw 5).
__global__ void k_predict(const uint8_t *__restrict__ bins, size_t row_step, size_t pitch, int lgw, int64_t n,
                          const PNode *const *__restrict__ trees, int n_trees, float *__restrict__ margin) {
  const int gmask = (1 << lgw) - 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    float mg = margin[i];
    const uint8_t *row = bins + i * row_step;
    for (int t = 0; t < n_trees; ++t) {
      const PNode *nd = trees[t];
      int v = 0;
      while (nd[v].feature >= 0) {
        const int f = nd[v].feature;
        v = goes_left(row[(size_t)(f >> lgw) * pitch + (f & gmask)], nd[v].split_bin, nd[v].default_left) ? 2 * v + 1
                                                                                                         : 2 * v + 2;
      }
      mg = mg + nd[v].leaf;
    }
    margin[i] = mg;
  }
}

// margin[row] += leaf of the row's final segment (in-core, all rows selected).
// margin[row] += leaf value of the row's final segment (Eq. 1).  The segment comes from the last
// plan's tile -> segment table (the segment holding the tile's first position) and a short
// forward scan, instead of a binary search over every segment per position.
__global__ void k_update_margin(int n, const Seg *__restrict__ segs, const LevelCtl *__restrict__ ctl,
                                const DNode *__restrict__ dn, const int32_t *__restrict__ ridx,
                                const int *__restrict__ tile_seg, float *__restrict__ margin) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int s;
  if (tile_seg) {
    s = tile_seg[i / kPartTile];
    while (segs[s].begin + segs[s].count <= i) ++s;
  } else {
    s = seg_of(segs, ctl->n_segs, i);
  }
  const int r = ridx[i];
  margin[r] = margin[r] + dn[segs[s].node].leaf_value;
}

__global__ void k_leaf_of_pos(int n, const Seg *__restrict__ segs, int n_segs, const int32_t *__restrict__ ridx,
                              int32_t *__restrict__ out_row, int32_t *__restrict__ out_leaf) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int s = seg_of(segs, n_segs, i);
  out_row[i] = ridx[i];
  out_leaf[i] = segs[s].node;
}

// ---------------------------------------------------------------------------------------------
static int kmax_of(oocgb_data d) { return (int)((0x7fffffffLL) >> d->quant_bits); }

static void ensure_work(oocgb_data d, int D) {
  oocgb_ctx c = d->ctx;
  Work *&w = d->work;
  const int m = d->m;
  const int n_fg = (m + kFG - 1) / kFG;
  // capacity: the build's CUDA graph depends on it, not on the sample's row count (which the kernels
  // read from the device sample state), so a sampled round (n_sel varies) reuses the graph; a
  // sample keeps 1/8 headroom up to the data's row count
  const int64_t need = std::max<int64_t>(1, d->n_sel);
  const int64_t n = d->all_selected ? need : std::min<int64_t>(std::max<int64_t>(need, d->n_local),
                                                               need + need / 8 + 4096);
  const int kmax = (int)((0x7fffffffLL) >> d->quant_bits);
  const int hist_grid = c->num_sms * kHistCtasPerSm;
  const int target = hist_grid;
  const int64_t max_pairs = D > 0 ? (1LL << (D - 1)) : 1;
  // bound of hist_chunk_rows' item count: C <= 2 n_pairs - 1 + ceil(rows / kmax) + ceil(grid / n_fg)
  auto items_for = [&](int64_t rows) { return target + (int64_t)n_fg * (((rows + kmax - 1) / kmax) + 2 * max_pairs + 2) + n_fg; };
  const int64_t items = items_for(n);
  const bool need64 = c->coll || d->streamed;  // all-reduced / streamed int64 node histograms
  if (w && w->cap_rows >= need && w->max_depth >= D && w->m == m && w->items_cap >= items_for(need) &&
      (!need64 || w->built64))
    return;
  free_work(d);
  w = new Work();
  w->cap_rows = n;
  w->max_depth = D;
  w->m = m;
  w->n_fg = n_fg;
  w->items_cap = items;
  w->hist_grid = hist_grid;
  const int64_t tiles = (n + kPartTile - 1) / kPartTile;
  const int64_t max_segs = 1LL << std::max(D, 1);
  for (int i = 0; i < 2; ++i) {
    w->ridx[i] = (int32_t *)dmalloc(sizeof(int32_t) * n);
    w->q[i] = (int2 *)dmalloc(sizeof(int2) * (n + 2));  // k_hist_tma reads q in even-aligned runs
    w->segs[i] = (Seg *)dmalloc(sizeof(Seg) * max_segs);
  }
  for (int i = 0; i < 2; ++i) w->seg_cur[i] = (int *)dmalloc(sizeof(int) * 2 * max_segs);
  w->tile_seg = (int *)dmalloc(sizeof(int) * std::max<int64_t>(1, tiles));
  w->chunk_rng = (int2 *)dmalloc(sizeof(int2) * items);  // chunks <= items
  w->seg_cnt = (long long *)dmalloc(sizeof(long long) * 2 * max_segs);
  w->pairs = (Pair *)dmalloc(sizeof(Pair) * max_pairs);
  OOCGB_CK(cudaMemset(w->pairs, 0, sizeof(Pair) * max_pairs));  // k_finalize reads past the count
  w->partial = (int *)dmalloc((size_t)items * kFG * kBins * 2 * sizeof(int));
  // world > 1: each rank evaluates a slice of msl = ceil(m / W) features (reduce-scattered
  // histograms), so parent histograms and the received sums hold msl features per row
  const int W = c->coll ? c->world : 1;
  w->msl = (m + W - 1) / W;
  w->max_slots = (int)(2 * max_pairs);
  const size_t hsz = (size_t)m * kBins * 2, hsl = (size_t)w->msl * kBins * 2;
  const int64_t pslots = D >= 2 ? (1LL << (D - 2)) : 1;
  for (int i = 0; i < 2; ++i) w->phist[i] = (long long *)dmalloc(sizeof(long long) * hsl * pslots);
  if (need64) w->built64 = (long long *)dmalloc(sizeof(long long) * hsz * 2 * max_pairs);
  if (c->coll) w->rs_send = (long long *)dmalloc(sizeof(long long) * hsl * (size_t)W * max_pairs);
  w->cand = (Cand *)dmalloc(sizeof(Cand) * (size_t)W * w->max_slots * w->msl);
  w->ent_cap = (int)(2 * max_pairs);
  w->ent = (int4 *)dmalloc(sizeof(int4) * 2 * w->ent_cap);
  w->dnodes = (DNode *)dmalloc(sizeof(DNode) * ((1LL << (D + 1)) - 1));
  w->ctl = (LevelCtl *)dmalloc(sizeof(LevelCtl));
  w->d_rp = (RoundParams *)dmalloc(sizeof(RoundParams));
  OOCGB_CK(cudaMallocHost(&w->h_rp, sizeof(RoundParams)));
  OOCGB_CK(cudaMallocHost(&w->h_dn, sizeof(DNode) * ((1LL << (D + 1)) - 1)));
  OOCGB_CK(cudaMallocHost(&w->h_ctl, sizeof(LevelCtl)));
  OOCGB_CK(cudaMallocHost(&w->h_pn, sizeof(PNode) * ((1LL << (D + 1)) - 1)));
  OOCGB_CK(cudaFuncSetAttribute(k_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, kHistSmem));
#if OOCGB_HIST_TMA
  OOCGB_CK(cudaFuncSetAttribute(k_hist_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, kTmaSmem));
#endif
}

static void drop_graph(Work *w);

void free_work(oocgb_data d) {
  Work *w = d->work;
  if (!w) return;
  for (int i = 0; i < 2; ++i) { dfree(w->ridx[i]); dfree(w->q[i]); dfree(w->segs[i]); dfree(w->phist[i]); }
  dfree(w->seg_cur[0]); dfree(w->seg_cur[1]); dfree(w->tile_seg); dfree(w->chunk_rng); dfree(w->seg_cnt); dfree(w->pairs); dfree(w->partial); dfree(w->built64); dfree(w->rs_send);
  dfree(w->cand); dfree(w->ent); dfree(w->dnodes); dfree(w->ctl); dfree(w->dbg); dfree(w->d_rp);
  dfree(w->sw.row_node); dfree(w->sw.b_slot); dfree(w->sw.b_ridx); dfree(w->sw.b_q); dfree(w->sw.slot_cnt);
  dfree(w->sw.slot_cur);
  d->streamed_row_node = nullptr;
  if (w->h_rp) cudaFreeHost(w->h_rp);
  if (w->h_dn) cudaFreeHost(w->h_dn);
  if (w->h_ctl) cudaFreeHost(w->h_ctl);
  if (w->h_pn) cudaFreeHost(w->h_pn);
  drop_graph(w);
  delete w;
  d->work = nullptr;
}

// Records the whole device side of one build_tree on the ctx stream (captured into a graph).
// `tev` collects (slot, event pair) for profiling; events are recorded only if non-null.
static void record_build(oocgb_data d, int D, double lambda, double gamma, double mcw, double eta,
                         bool keep_debug, const uint8_t *bins, size_t pitch, int ridx_mode,
                         std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> *tev) {
  oocgb_ctx c = d->ctx;
  Work *w = d->work;
  const int m = d->m, n_fg = w->n_fg;
  // geometry from the capacity; the kernels read the sample's row count from the device
  const int n = (int)w->cap_rows;
  const long long *n_dev = &d->d_ss->n_sel_local;
  const int n_nodes = (1 << (D + 1)) - 1;
  const int kmax = (int)((0x7fffffffLL) >> d->quant_bits);
  const int target = w->hist_grid;  // one wave of items per level
  const size_t hsz = (size_t)m * kBins * 2;
  auto mark = [&](int slot, bool begin) {
    if (!tev) return;
    if (begin) {
      cudaEvent_t a, b;
      OOCGB_CK(cudaEventCreate(&a));
      OOCGB_CK(cudaEventCreate(&b));
      tev->push_back({slot, {a, b}});
      // external event nodes behave like ordinary stream records (timable) when replayed
      OOCGB_CK(cudaEventRecordWithFlags(a, c->stream, cudaEventRecordExternal));
    } else {
      OOCGB_CK(cudaEventRecordWithFlags(tev->back().second.second, c->stream, cudaEventRecordExternal));
    }
  };
  if (keep_debug) OOCGB_CK(cudaMemsetAsync(w->dbg, 0, sizeof(long long) * hsz * (size_t)std::max(1, (1 << D) - 1), c->stream));
  int cur = 0;
  const int tiles = (n + kPartTile - 1) / kPartTile;
  k_init_build<<<c->num_sms * 4, 256, 0, c->stream>>>(
      w->dnodes, n_nodes, d->d_ss, w->d_rp, lambda, mcw, eta, w->segs[0], w->pairs, w->ctl, -1, n_fg, target, kmax,
      D, d->d_sel_rows, w->ridx[0], d->d_q, w->q[0], ridx_mode, w->chunk_rng, w->ent, w->ent_cap, w->tile_seg, tiles,
      w->seg_cur[0]);
  OOCGB_CK(cudaGetLastError());
  for (int lv = 0; lv < D; ++lv) {
    const int max_pairs = lv == 0 ? 1 : (1 << (lv - 1));
    // this level's positions: level 0 reads the sample's buffers directly (identity rows or the
    // selected rows, the sample's q), later levels the previous partition's output
    const int32_t *lv_ridx = lv > 0 ? w->ridx[cur] : (ridx_mode == 1 ? d->d_sel_rows : nullptr);
    const int2 *lv_q = lv > 0 ? w->q[cur] : d->d_q;
    mark(0, true);
#if OOCGB_HIST_TMA
    if (lv == 0 && ridx_mode == 0 && d->gw == 32)  // identity level: bulk feed
      k_hist_tma<<<w->hist_grid, kHistThreads, kTmaSmem, c->stream>>>(bins, pitch, m, n_fg, lv_q, w->pairs,
                                                                      w->ctl, w->chunk_rng, w->partial);
    else
#endif
      k_hist<<<w->hist_grid, kHistThreads, kHistSmem, c->stream>>>(bins, pitch, m, n_fg, lv_ridx, lv_q,
                                                                   w->pairs, w->ctl, w->chunk_rng, w->partial,
                                                                   (lv == 0 && ridx_mode == 0) ? 1 : 0, d->gw,
                                                                   d->gw == 64 ? 1 : 0);
    OOCGB_CK(cudaGetLastError());
    mark(0, false);
    if (c->coll) {  // every rank receives the global sums of its feature slice
      int64_t tot = (int64_t)max_pairs * m * kBins;
      k_reduce_partials<<<(int)std::min<int64_t>((tot + 255) / 256, c->num_sms * 16), 256, 0, c->stream>>>(
          w->partial, w->pairs, w->ctl, m, n_fg, w->msl, max_pairs, w->rs_send);
      reduce_scatter_i64(c, w->rs_send, w->built64, (size_t)max_pairs * w->msl * kBins * 2);
    }
    mark(1, true);
    EvalArgs A;
    A.d = lv; A.D = D; A.m = m; A.n_fg = n_fg;
    A.pairs = w->pairs; A.ctl = w->ctl; A.partial = w->partial;
    A.built64 = c->coll ? w->built64 : nullptr;
    A.phist_prev = w->phist[(lv + 1) & 1];
    A.phist_next = w->phist[lv & 1];
    A.dbg = keep_debug ? w->dbg : nullptr;
    A.cut_ptrs = d->d_cut_ptrs; A.dn = w->dnodes; A.cand = w->cand;
    A.lambda = lambda; A.gamma = gamma; A.mcw = mcw; A.rp = w->d_rp; A.kmax = kmax; A.streamed = 0;
    A.cut_values = d->d_cut_values; A.eta = eta;
    A.ent = w->ent; A.ent_cap = w->ent_cap; A.has_missing = d->has_missing ? 1 : 0;
    A.msl = w->msl; A.max_slots = 2 * max_pairs; A.hm = w->msl;  // candidate blocks sized for this level
    A.f0 = c->coll ? std::min(m, c->rank * w->msl) : 0;
    A.mf = std::max(0, std::min(m, A.f0 + w->msl) - A.f0);
    A.crank = c->coll ? c->rank : 0;
    // f = 1: the root's global row count is fixed, so its list is known when capturing
    A.root_list = lv == 0 ? w->root_list : 0;
    A.segs = w->segs[cur];
    launch_eval(A, max_pairs, c, c->stream);
    mark(1, false);
    mark(2, true);
    PlanArgs PA;
    PA.segs = w->segs[cur]; PA.segs_next = w->segs[cur ^ 1]; PA.ctl = w->ctl; PA.dn = w->dnodes;
    PA.cur = w->seg_cur[lv & 1]; PA.seg_cnt = c->coll ? w->seg_cnt : nullptr;
    PA.cur_next = w->seg_cur[(lv + 1) & 1]; PA.pairs = w->pairs; PA.tile_seg = w->tile_seg;
    PA.chunk_rng = w->chunk_rng;
    PA.n_dev = n_dev; PA.n_fg = n_fg; PA.target_items = target; PA.kmax = kmax;
    PA.ent = w->ent; PA.ent_cap = w->ent_cap;
    PA.last = lv == D - 1 ? 1 : 0;
    const bool inline_plan = !c->coll && n > 0;
    if (n > 0) {
      k_part_fused<<<tiles, kPartThreads, 0, c->stream>>>(n_dev, w->segs[cur], w->ctl, w->dnodes, bins, pitch,
                                                          d->gw == 64 ? 6 : 5,
                                                          lv_ridx, lv_q, w->ridx[cur ^ 1], w->q[cur ^ 1],
                                                          w->seg_cur[lv & 1], w->tile_seg, inline_plan ? 1 : 0, PA,
                                                          lv > 0 ? n : (int)std::min<int64_t>(n, d->sel_cap));
      OOCGB_CK(cudaGetLastError());
    }
    if (c->coll) {
      const int len = 2 * (1 << lv);
      k_part_counts<<<(len + 255) / 256, 256, 0, c->stream>>>(w->seg_cur[lv & 1], w->ctl, len, w->seg_cnt);
      allreduce_sum_i64(c, w->seg_cnt, (size_t)len);
    }
    if (!inline_plan) {
      k_part_plan<<<1, 1024, 0, c->stream>>>(PA);
      OOCGB_CK(cudaGetLastError());
    }
    mark(2, false);
    cur ^= 1;
  }
  // world > 1: each rank dumped its feature slice of every node histogram (debug builds only)
  if (keep_debug && c->coll) allreduce_sum_i64(c, w->dbg, hsz * (size_t)std::max(1, (1 << D) - 1));
  w->final_cur = cur;
}

static void add_graph_timings(oocgb_ctx c, Work *w) {
  for (auto &e : w->graph_events) {
    float ms = 0.f;
    OOCGB_CK(cudaEventElapsedTime(&ms, e.second.first, e.second.second));
    c->timings[e.first] += ms;
    if (e.first == 0) c->timings[7] += 1.0;
  }
}

static void drop_graph(Work *w) {
  if (w->graph) cudaGraphExecDestroy(w->graph);
  w->graph = nullptr;
  for (auto &e : w->graph_events) {
    cudaEventDestroy(e.second.first);
    cudaEventDestroy(e.second.second);
  }
  w->graph_events.clear();
}

oocgb_tree build_tree(oocgb_data d, int D, double lambda, double gamma, double mcw, double eta,
                      bool keep_debug) {
  oocgb_ctx c = d->ctx;
  PhaseTimer whole(c, 6);
  ensure_work(d, D);
  Work *w = d->work;
  const int m = d->m;
  const int n = (int)d->n_sel;
  const int n_nodes = (1 << (D + 1)) - 1;
  const size_t hsz = (size_t)m * kBins * 2;
  const uint8_t *bins;
  int ridx_mode;
  size_t pitch;  // bytes of one feature-group plane of the tiled page the tree reads
  if (d->placement == OOCGB_PLACE_PINNED_HOST) {
    bins = d->d_sampled_page; ridx_mode = 0; pitch = (size_t)d->sampled_cap * d->gw;
  } else {
    bins = d->d_bins; ridx_mode = d->all_selected ? 0 : 1; pitch = (size_t)d->rows_per_page * d->gw;
  }
  if (keep_debug) {
    size_t need = sizeof(long long) * hsz * (size_t)std::max(1, (1 << D) - 1);
    if (w->dbg_bytes < need) { drop_graph(w); dfree(w->dbg); w->dbg = (long long *)dmalloc(need); w->dbg_bytes = need; }
  }
  // keyed by the capacity, not the sample's row count: sampled rounds replay one graph
  // f = 1: every row is selected, so the root's list (general iff > kmax global rows) is known
  // here and the other list's level-0 launch is left out of the graph
  w->root_list = d->all_selected ? (d->n_global > kmax_of(d) ? 1 : 2) : 0;
  GraphKey key{(int)w->cap_rows, D, m, ridx_mode, keep_debug ? 1 : 0, c->profiling ? 1 : 0, c->world,
               d->has_missing ? 1 : 0, w->root_list, lambda, gamma, mcw, eta, bins, pitch, d->quant_bits};
  if (c->host_coll) {
    // host-callback collectives synchronise the stream: run the level loop directly
    drop_graph(w);
    record_build(d, D, lambda, gamma, mcw, eta, keep_debug, bins, pitch, ridx_mode,
                 c->profiling ? &w->graph_events : nullptr);
  } else if (!w->graph || !(w->key == key)) {
    drop_graph(w);
    cudaGraph_t g;
    OOCGB_CK(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    try {
      record_build(d, D, lambda, gamma, mcw, eta, keep_debug, bins, pitch, ridx_mode,
                   c->profiling ? &w->graph_events : nullptr);
    } catch (...) {
      cudaStreamEndCapture(c->stream, &g);
      throw;
    }
    OOCGB_CK(cudaStreamEndCapture(c->stream, &g));
    OOCGB_CK(cudaGraphInstantiate(&w->graph, g, 0));
    cudaGraphDestroy(g);
    w->key = key;
    c->timings[9] += 1.0;  // graph captures (diagnostic)
  }
  if (!c->host_coll) OOCGB_CK(cudaGraphLaunch(w->graph, c->stream));
  const int cur = w->final_cur;
  // export
  const DNode *hn = w->h_dn;
  OOCGB_CK(cudaMemcpyAsync(w->h_dn, w->dnodes, sizeof(DNode) * n_nodes, cudaMemcpyDeviceToHost, c->stream));
  OOCGB_CK(cudaMemcpyAsync(w->h_ctl, w->ctl, sizeof(LevelCtl), cudaMemcpyDeviceToHost, c->stream));
  OOCGB_CK(cudaStreamSynchronize(c->stream));
  const LevelCtl hctl = *w->h_ctl;
  OOCGB_REQUIRE(hctl.error == 0, OOCGB_ERR_ARG, "build_tree: H + lambda <= 0 at a node (S:L406)");
  if (c->profiling) add_graph_timings(c, w);
  oocgb_tree t = new oocgb_tree_s();
  t->owner = d;
  t->serial = ++d->tree_serial;
  t->sample_serial = d->sample_serial;
  c->live_trees++;
  t->max_depth = D;
  t->nodes.resize(n_nodes);
  PNode *pn = w->h_pn;  // pinned: the H2D below is asynchronous (reused only after the next sync)
  for (int v = 0; v < n_nodes; ++v) {
    oocgb_node &o = t->nodes[v];
    o.feature = hn[v].feature;
    o.split_bin = hn[v].split_bin;
    o.split_value = hn[v].split_value;
    o.leaf_value = hn[v].leaf_value;
    o.gain = hn[v].gain;
    o.sum_g = hn[v].sum_g;
    o.sum_h = hn[v].sum_h;
    o.n_rows = hn[v].n_rows;
    o.default_left = hn[v].feature >= 0 ? hn[v].default_left : 0;
    o.pad = 0;
    if (o.feature == -2) { o.split_bin = 0; o.split_value = 0; o.leaf_value = 0; o.gain = 0; o.sum_g = 0; o.sum_h = 0; o.n_rows = 0; }
    if (o.feature == -1) { o.split_bin = 0; o.split_value = 0; o.gain = 0; }
    pn[v] = PNode{o.feature, o.split_bin, o.leaf_value, o.default_left};
  }
  t->ctx = c;
  t->pnodes_bytes = sizeof(PNode) * n_nodes;
  t->d_pnodes = (PNode *)pool_get(c, t->pnodes_bytes);
  OOCGB_CK(cudaMemcpyAsync(t->d_pnodes, pn, sizeof(PNode) * n_nodes, cudaMemcpyHostToDevice, c->stream));
  if (keep_debug) {
    t->debug = true;
    size_t cnt = hsz * (size_t)std::max(0, (1 << D) - 1);
    t->hist.resize(cnt);
    if (cnt) OOCGB_CK(cudaMemcpyAsync(t->hist.data(), w->dbg, sizeof(long long) * cnt, cudaMemcpyDeviceToHost, c->stream));
    // final partition: position -> (row index, leaf)
    LevelCtl h2;
    OOCGB_CK(cudaMemcpyAsync(&h2, w->ctl, sizeof(LevelCtl), cudaMemcpyDeviceToHost, c->stream));
    OOCGB_CK(cudaStreamSynchronize(c->stream));
    int32_t *d_rows = (int32_t *)dmalloc(sizeof(int32_t) * std::max(1, n));
    int32_t *d_leaf = (int32_t *)dmalloc(sizeof(int32_t) * std::max(1, n));
    if (n > 0)
      k_leaf_of_pos<<<(n + 255) / 256, 256, 0, c->stream>>>(n, w->segs[cur], D > 0 ? h2.n_segs : 1, w->ridx[cur],
                                                             d_rows, d_leaf);
    std::vector<int32_t> rows(n), leaf(n);
    if (n > 0) {
      OOCGB_CK(cudaMemcpyAsync(rows.data(), d_rows, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, c->stream));
      OOCGB_CK(cudaMemcpyAsync(leaf.data(), d_leaf, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, c->stream));
    }
    OOCGB_CK(cudaStreamSynchronize(c->stream));
    dfree(d_rows);
    dfree(d_leaf);
    // row index -> selected order
    t->leaf_of_row.assign(n, -1);
    t->row_order.assign(n, -1);
    t->has_row_order = true;
    if (ridx_mode == 1) {
      std::vector<int32_t> sel(n);
      if (n) OOCGB_CK(cudaMemcpy(sel.data(), d->d_sel_rows, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
      for (int i = 0; i < n; ++i) {
        int k = (int)(std::lower_bound(sel.begin(), sel.end(), rows[i]) - sel.begin());
        t->leaf_of_row[k] = leaf[i];
        t->row_order[i] = k;
      }
    } else {
      for (int i = 0; i < n; ++i) {
        t->leaf_of_row[rows[i]] = leaf[i];
        t->row_order[i] = rows[i];
      }
    }
  }
  return t;  // one host synchronisation per tree (the export); predict nodes follow on the stream
}

// ---------------------------------------------------------------------------------------------
// Alg. 6, level-batched (NEXT #1): f = 1 data that stays in pinned host memory.
// Each level is one streamed pass over batches of pages: every row moves to its child under the
// previous level's split (the per-row node id replaces the device-wide partition), the batch's
// rows are grouped by node (counting sort), k_hist runs on the staged row-major batch, and the
// batch's s32 partials are added into int64 per-node histograms; then every node of the level is
// evaluated directly (no sibling subtraction: the children's sizes are only known after the pass).
__global__ void k_stream_init(int32_t *row_node, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    row_node[i] = 0;
}

// rows of one batch: move to the child under the previous level's split (update != 0), count
// the rows per child (n_rows, exact integer atomics), and tag rows of depth-d nodes with their
// slot (node - first(d)); rows in earlier leaves get -1.
__global__ void k_stream_assign(const uint8_t *__restrict__ batch, int stride, int64_t r0, int64_t nr,
                                int32_t *__restrict__ row_node, DNode *dn, int first_d, int update, int hist,
                                int32_t *__restrict__ b_slot, int *__restrict__ slot_cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nr; i += (int64_t)gridDim.x * blockDim.x) {
    int v = row_node[r0 + i];
    if (update) {
      const int f = dn[v].feature;
      if (f >= 0) {
        v = goes_left(batch[(size_t)i * stride + f], dn[v].split_bin, dn[v].default_left) ? 2 * v + 1 : 2 * v + 2;
        row_node[r0 + i] = v;
        atomicAdd((unsigned long long *)&dn[v].n_rows, 1ull);
      }
    }
    if (hist) {
      const int sl = (v >= first_d && dn[v].feature == -1) ? v - first_d : -1;
      b_slot[i] = sl;
      if (sl >= 0) atomicAdd(&slot_cnt[sl], 1);
    }
  }
}

// single block: slot offsets, the batch's pair table (one "pair" per slot: built = node, no
// derived) with chunking, and the item count (batch_rows = 0: the pair list alone).
__global__ void __launch_bounds__(1024)
k_stream_plan(int n_slots, int first_d, const int *__restrict__ slot_cnt, int *__restrict__ slot_cur,
              Pair *__restrict__ pairs, LevelCtl *ctl, int n_fg, int target_items, int kmax, int64_t batch_rows,
              int2 *__restrict__ chunk_rng, int4 *__restrict__ ent) {
  const long long cr = hist_chunk_rows(batch_rows, n_slots, n_fg, target_items, kmax);
  int carry_rows = 0, carry_chunks = 0;
  for (int base = 0; base < n_slots; base += blockDim.x) {
    const int sl = base + threadIdx.x;
    const int cnt = sl < n_slots ? slot_cnt[sl] : 0;
    const int nch = batch_rows > 0 ? (int)((cnt + cr - 1) / cr) : 0;  // 0: pair list only (evaluation)
    int tr, tc;
    const int er = block_excl_scan(cnt, &tr);
    const int ec = block_excl_scan(nch, &tc);
    if (sl < n_slots) {
      slot_cur[sl] = carry_rows + er;
      Pair pr;
      pr.parent = -1; pr.built = first_d + sl; pr.derived = -1;
      pr.begin = carry_rows + er; pr.count = cnt;
      pr.chunk_base = carry_chunks + ec; pr.n_chunks = nch;
      pr.chunk_rows = nch > 0 ? (cnt + nch - 1) / nch : (int)cr;  // equal chunks
      pr.compact = 0;
      pairs[sl] = pr;
      for (int c = 0; c < nch; ++c)
        chunk_rng[carry_chunks + ec + c] = make_int2(pr.begin + c * pr.chunk_rows, min(pr.begin + cnt, pr.begin + (c + 1) * pr.chunk_rows));
      ent[sl] = make_int4(sl, 0, first_d + sl, 0);  // streamed evaluation: every slot in the general list
    }
    carry_rows += tr;
    carry_chunks += tc;
  }
  if (threadIdx.x == 0) {
    ctl->n_pairs = n_slots;
    ctl->n_items = carry_chunks * n_fg;
    ctl->hist_next = 0;
    ctl->n_ew = n_slots;
    ctl->n_en = 0;
  }
}

__global__ void k_stream_scatter(int64_t r0, int64_t nr, const int32_t *__restrict__ b_slot,
                                 int *__restrict__ slot_cur, const int2 *__restrict__ q,
                                 int32_t *__restrict__ b_ridx, int2 *__restrict__ b_q) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nr; i += (int64_t)gridDim.x * blockDim.x) {
    const int sl = b_slot[i];
    if (sl < 0) continue;
    const int pos = atomicAdd(&slot_cur[sl], 1);  // order inside a slot is irrelevant: integer sums
    b_ridx[pos] = (int32_t)i;
    b_q[pos] = q[r0 + i];
  }
}

// built64[slot][j][b] += sum of the batch's chunk partials of that slot (thread per (slot, j, b)).
__global__ void k_accum_partials(const int *__restrict__ partial, const Pair *__restrict__ pairs, int n_slots,
                                 int m, int n_fg, long long *__restrict__ out) {
  const int64_t total = (int64_t)n_slots * m * kBins;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int b = (int)(t % kBins);
    const int j = (int)((t / kBins) % m);
    const int p = (int)(t / ((int64_t)kBins * m));
    const Pair P = pairs[p];
    if (P.n_chunks == 0) continue;
    long long g = 0, h = 0;
    for (int c = 0; c < P.n_chunks; ++c) {
      const size_t item = (size_t)(P.chunk_base + c) * n_fg + j / kFG;
      const int2 v = reinterpret_cast<const int2 *>(partial)[(item * kFG + (j % kFG)) * kBins + b];
      g += v.x;
      h += v.y;
    }
    out[t * 2] += g;
    out[t * 2 + 1] += h;
  }
}

__global__ void k_stream_leaf_margin(const int32_t *__restrict__ row_node, int64_t n, const DNode *__restrict__ dn,
                                     float *__restrict__ margin) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    margin[i] = margin[i] + dn[row_node[i]].leaf_value;
}

oocgb_tree build_tree_streamed(oocgb_data d, int D, double lambda, double gamma, double mcw, double eta,
                               bool keep_debug) {
  oocgb_ctx c = d->ctx;
  OOCGB_REQUIRE(!c->coll, OOCGB_ERR_ARG, "streamed build (Alg. 6) runs on one GPU in this version");
  OOCGB_REQUIRE(d->all_selected, OOCGB_ERR_STATE, "streamed build needs sample(NONE) (f = 1)");
  PhaseTimer whole(c, 6);
  ensure_work(d, D);
  Work *w = d->work;
  const int m = d->m, n_fg = w->n_fg;
  const int64_t n = d->n_local;
  const int n_nodes = (1 << (D + 1)) - 1;
  const int kmax = (int)((0x7fffffffLL) >> d->quant_bits);
  const size_t hsz = (size_t)m * kBins * 2;
  const int64_t brows = std::min<int64_t>(std::max<int64_t>(1, n),
                                          std::max<int64_t>(d->rows_per_page, (1LL << 30) / d->stride));
  StreamWork &sw = w->sw;
  if (sw.cap_n < n || sw.cap_b < brows || sw.max_slots < (1 << std::max(0, D - 1))) {
    dfree(sw.row_node); dfree(sw.b_slot); dfree(sw.b_ridx); dfree(sw.b_q); dfree(sw.slot_cnt); dfree(sw.slot_cur);
    sw.cap_n = std::max<int64_t>(1, n);
    sw.cap_b = brows;
    sw.max_slots = 1 << std::max(0, D - 1);
    sw.row_node = (int32_t *)dmalloc(sizeof(int32_t) * sw.cap_n);
    sw.b_slot = (int32_t *)dmalloc(sizeof(int32_t) * brows);
    sw.b_ridx = (int32_t *)dmalloc(sizeof(int32_t) * brows);
    sw.b_q = (int2 *)dmalloc(sizeof(int2) * brows);
    sw.slot_cnt = (int *)dmalloc(sizeof(int) * sw.max_slots);
    sw.slot_cur = (int *)dmalloc(sizeof(int) * sw.max_slots);
  }
  if (keep_debug) {
    size_t need = sizeof(long long) * hsz * (size_t)std::max(1, (1 << D) - 1);
    if (w->dbg_bytes < need) { dfree(w->dbg); w->dbg = (long long *)dmalloc(need); w->dbg_bytes = need; }
    OOCGB_CK(cudaMemsetAsync(w->dbg, 0, need, c->stream));
  }
  OOCGB_CK(cudaMemsetAsync(w->ctl, 0, sizeof(LevelCtl), c->stream));
  const int target = w->hist_grid;
  k_init_build<<<c->num_sms * 4, 256, 0, c->stream>>>(w->dnodes, n_nodes, d->d_ss, w->d_rp, lambda, mcw, eta,
                                                       w->segs[0], w->pairs, w->ctl, 0, n_fg, target, kmax, D,
                                                       d->d_sel_rows, w->ridx[0], d->d_q, w->q[0], 0, w->chunk_rng, w->ent,
                                                       w->ent_cap, nullptr, 0, nullptr);
  k_stream_init<<<c->num_sms * 4, 256, 0, c->stream>>>(sw.row_node, n);
  OOCGB_CK(cudaGetLastError());
  const int grid = c->num_sms * 8;
  for (int lv = 0; lv <= D; ++lv) {
    const bool hist = lv < D;  // the last pass only moves rows to their leaves
    const int n_slots = 1 << lv;
    const int first = level_first(lv);
    if (hist) OOCGB_CK(cudaMemsetAsync(w->built64, 0, sizeof(long long) * hsz * n_slots, c->stream));
    for_each_batch(d, brows, [&](const uint8_t *batch, int64_t r0, int64_t nr) {
      if (hist) OOCGB_CK(cudaMemsetAsync(sw.slot_cnt, 0, sizeof(int) * n_slots, c->stream));
      k_stream_assign<<<grid, 256, 0, c->stream>>>(batch, d->stride, r0, nr, sw.row_node, w->dnodes, first,
                                                   lv > 0 ? 1 : 0, hist ? 1 : 0, sw.b_slot, sw.slot_cnt);
      OOCGB_CK(cudaGetLastError());
      if (!hist) return;
      k_stream_plan<<<1, 1024, 0, c->stream>>>(n_slots, first, sw.slot_cnt, sw.slot_cur, w->pairs, w->ctl, n_fg,
                                               target, kmax, nr, w->chunk_rng, w->ent);
      k_stream_scatter<<<grid, 256, 0, c->stream>>>(r0, nr, sw.b_slot, sw.slot_cur, d->d_q, sw.b_ridx, sw.b_q);
      {
        PhaseTimer t(c, 0);
        k_hist<<<w->hist_grid, kHistThreads, kHistSmem, c->stream>>>(batch, 32, m, n_fg, sw.b_ridx, sw.b_q, w->pairs,
                                                                     w->ctl, w->chunk_rng, w->partial, 0, d->stride, 0);
      }
      const int64_t tot = (int64_t)n_slots * m * kBins;
      k_accum_partials<<<(int)std::min<int64_t>((tot + 255) / 256, c->num_sms * 16), 256, 0, c->stream>>>(
          w->partial, w->pairs, n_slots, m, n_fg, w->built64);
      OOCGB_CK(cudaGetLastError());
    });
    if (!hist) break;
    // every node of the level: pairs[s] = {built = first + s} over the whole data
    k_stream_plan<<<1, 1024, 0, c->stream>>>(n_slots, first, sw.slot_cnt, sw.slot_cur, w->pairs, w->ctl, n_fg,
                                             target, kmax, 0, w->chunk_rng, w->ent);
    PhaseTimer t(c, 1);
    EvalArgs A;
    A.d = lv; A.D = D; A.m = m; A.n_fg = n_fg;
    A.pairs = w->pairs; A.ctl = w->ctl; A.partial = w->partial;
    A.built64 = w->built64;
    A.phist_prev = w->phist[0];
    A.phist_next = w->phist[1];
    A.dbg = keep_debug ? w->dbg : nullptr;
    A.cut_ptrs = d->d_cut_ptrs; A.dn = w->dnodes; A.cand = w->cand;
    A.lambda = lambda; A.gamma = gamma; A.mcw = mcw; A.rp = w->d_rp; A.kmax = kmax; A.streamed = 1;
    A.cut_values = d->d_cut_values; A.eta = eta;
    A.ent = w->ent; A.ent_cap = w->ent_cap; A.has_missing = d->has_missing ? 1 : 0;
    A.msl = w->msl; A.max_slots = n_slots; A.hm = w->msl;
    A.f0 = c->coll ? std::min(m, c->rank * w->msl) : 0;
    A.mf = std::max(0, std::min(m, A.f0 + w->msl) - A.f0);
    A.crank = c->coll ? c->rank : 0;
    A.root_list = 0;
    A.segs = nullptr;  // no partition in the streamed build
    launch_eval(A, n_slots, c, c->stream);
  }
  // export (same as the in-core path)
  const DNode *hn = w->h_dn;
  OOCGB_CK(cudaMemcpyAsync(w->h_dn, w->dnodes, sizeof(DNode) * n_nodes, cudaMemcpyDeviceToHost, c->stream));
  OOCGB_CK(cudaMemcpyAsync(w->h_ctl, w->ctl, sizeof(LevelCtl), cudaMemcpyDeviceToHost, c->stream));
  OOCGB_CK(cudaStreamSynchronize(c->stream));
  const LevelCtl hctl = *w->h_ctl;
  OOCGB_REQUIRE(hctl.error == 0, OOCGB_ERR_ARG, "build_tree: H + lambda <= 0 at a node (S:L406)");
  oocgb_tree t = new oocgb_tree_s();
  t->owner = d;
  t->serial = ++d->tree_serial;
  t->sample_serial = d->sample_serial;
  c->live_trees++;
  t->max_depth = D;
  t->nodes.resize(n_nodes);
  PNode *pn = w->h_pn;  // pinned: the H2D below is asynchronous (reused only after the next sync)
  for (int v = 0; v < n_nodes; ++v) {
    oocgb_node &o = t->nodes[v];
    o.feature = hn[v].feature; o.split_bin = hn[v].split_bin; o.split_value = hn[v].split_value;
    o.leaf_value = hn[v].leaf_value; o.gain = hn[v].gain; o.sum_g = hn[v].sum_g; o.sum_h = hn[v].sum_h;
    o.n_rows = hn[v].n_rows;
    o.default_left = hn[v].feature >= 0 ? hn[v].default_left : 0;
    o.pad = 0;
    if (o.feature == -2) { o.split_bin = 0; o.split_value = 0; o.leaf_value = 0; o.gain = 0; o.sum_g = 0; o.sum_h = 0; o.n_rows = 0; }
    if (o.feature == -1) { o.split_bin = 0; o.split_value = 0; o.gain = 0; }
    pn[v] = PNode{o.feature, o.split_bin, o.leaf_value, o.default_left};
  }
  t->ctx = c;
  t->pnodes_bytes = sizeof(PNode) * n_nodes;
  t->d_pnodes = (PNode *)pool_get(c, t->pnodes_bytes);
  OOCGB_CK(cudaMemcpyAsync(t->d_pnodes, pn, sizeof(PNode) * n_nodes, cudaMemcpyHostToDevice, c->stream));
  if (keep_debug) {
    t->debug = true;
    size_t cnt = hsz * (size_t)std::max(0, (1 << D) - 1);
    t->hist.resize(cnt);
    if (cnt) OOCGB_CK(cudaMemcpyAsync(t->hist.data(), w->dbg, sizeof(long long) * cnt, cudaMemcpyDeviceToHost, c->stream));
    t->leaf_of_row.assign(n, -1);
    if (n) OOCGB_CK(cudaMemcpyAsync(t->leaf_of_row.data(), sw.row_node, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, c->stream));
  }
  OOCGB_CK(cudaStreamSynchronize(c->stream));
  d->streamed_row_node = sw.row_node;
  return t;
}

void predict_device(oocgb_data d, const uint8_t *d_bins, size_t row_step, size_t pitch, int lgw, int64_t n_rows,
                    int64_t row_offset,
                    const oocgb_tree *trees, int n_trees, float *d_margin) {
  oocgb_ctx c = d->ctx;
  if (n_rows <= 0 || n_trees <= 0) return;
  std::vector<const PNode *> ptrs(n_trees);
  for (int t = 0; t < n_trees; ++t) ptrs[t] = trees[t]->d_pnodes;
  const PNode **d_ptrs = (const PNode **)((char *)c->d_small + (768 << 10));
  OOCGB_REQUIRE(n_trees <= 4096, OOCGB_ERR_ARG, "predict: at most 4096 trees per call");
  OOCGB_CK(cudaMemcpyAsync(d_ptrs, ptrs.data(), sizeof(void *) * n_trees, cudaMemcpyHostToDevice, c->stream));
  int blocks = (int)std::min<int64_t>((n_rows + 255) / 256, (int64_t)c->num_sms * 16);
  k_predict<<<blocks, 256, 0, c->stream>>>(d_bins, row_step, pitch, lgw, n_rows, d_ptrs, n_trees, d_margin + row_offset);
  OOCGB_CK(cudaGetLastError());
}

void update_margin(oocgb_data d, oocgb_tree t, float *d_margin) {
  oocgb_ctx c = d->ctx;
  Work *w = d->work;
  if (d->streamed && d->placement == OOCGB_PLACE_PINNED_HOST) {
    OOCGB_REQUIRE(w && t->serial == d->tree_serial && t->sample_serial == d->sample_serial && d->all_selected &&
                      d->streamed_row_node,
                  OOCGB_ERR_STATE,
                  "update_margin: needs the latest tree of an f = 1 sample");
    k_stream_leaf_margin<<<c->num_sms * 8, 256, 0, c->stream>>>(d->streamed_row_node, d->n_local, w->dnodes, d_margin);
    OOCGB_CK(cudaGetLastError());
    return;
  }
  OOCGB_REQUIRE(w && t->serial == d->tree_serial && t->sample_serial == d->sample_serial && d->all_selected &&
                    !d->streamed && d->placement == OOCGB_PLACE_DEVICE,
                OOCGB_ERR_STATE, "update_margin: needs the latest tree of an in-core, f = 1 sample");
  const int n = (int)d->n_sel;
  if (n > 0)
    k_update_margin<<<(n + 255) / 256, 256, 0, c->stream>>>(n, w->segs[w->final_cur], w->ctl, w->dnodes,
                                                            w->ridx[w->final_cur],
                                                            w->tile_seg, d_margin);
  OOCGB_CK(cudaGetLastError());
}

}  // namespace oocgb
