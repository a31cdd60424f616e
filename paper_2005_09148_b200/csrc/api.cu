// C-ABI of liboocgb (include/oocgb.h): argument checking, handle lifetime, host<->device
// marshalling, NCCL plumbing and the page streamer.  The arithmetic of the method lives in
// quantise.cu, sample.cu and tree.cu.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>

#include "internal.cuh"
#include "stream.cuh"

namespace oocgb {

static thread_local std::string g_last_error;
void set_last_error(const std::string &m) { g_last_error = m; }

void *dmalloc(size_t bytes) {
  void *p = nullptr;
  cudaError_t e = cudaMalloc(&p, std::max<size_t>(bytes, 16));
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw Error(OOCGB_ERR_NOMEM, "device allocation of " + std::to_string(bytes) +
                                     " bytes failed (" + cudaGetErrorString(e) +
                                     "); lower the sampling ratio or use PINNED_HOST pages");
  }
  return p;
}
void dfree(void *p) {
  if (p) cudaFree(p);
}
void *pool_get(oocgb_ctx c, size_t bytes) {
  for (size_t i = 0; i < c->node_pool.size(); ++i)
    if (c->node_pool[i].first == bytes) {
      void *p = c->node_pool[i].second;
      c->node_pool.erase(c->node_pool.begin() + (long)i);
      return p;
    }
  return dmalloc(bytes);
}
void pool_put(oocgb_ctx c, size_t bytes, void *p) {
  if (!p) return;
  if (c->node_pool.size() >= 4096) { dfree(p); return; }
  c->node_pool.push_back({bytes, p});
}
bool is_device_ptr(const void *p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

const NcclApi &nccl_api() {
  static NcclApi api{};
  static bool loaded = false;
  if (loaded) return api;
  void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) throw Error(OOCGB_ERR_DEVICE, std::string("cannot load NCCL: ") + dlerror());
  auto sym = [&](const char *n) {
    void *p = dlsym(h, n);
    if (!p) throw Error(OOCGB_ERR_DEVICE, std::string("NCCL symbol missing: ") + n);
    return p;
  };
  api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
  api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
  api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
  api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
  api.AllGather = (decltype(api.AllGather))sym("ncclAllGather");
  api.ReduceScatter = (decltype(api.ReduceScatter))sym("ncclReduceScatter");
  api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
  loaded = true;
  return api;
}

void allreduce_sum_i64(oocgb_ctx c, long long *d_buf, size_t count) {
  if (!c->coll || count == 0) return;
  if (c->host_coll) {
    std::vector<long long> h(count);
    OOCGB_CK(cudaMemcpyAsync(h.data(), d_buf, 8 * count, cudaMemcpyDeviceToHost, c->stream));
    OOCGB_CK(cudaStreamSynchronize(c->stream));
    OOCGB_REQUIRE(c->host_coll(0, 0, h.data(), (int64_t)count, c->host_coll_user) == 0, OOCGB_ERR_DEVICE,
                  "host collective (all-reduce sum) failed");
    OOCGB_CK(cudaMemcpyAsync(d_buf, h.data(), 8 * count, cudaMemcpyHostToDevice, c->stream));
    OOCGB_CK(cudaStreamSynchronize(c->stream));
    return;
  }
  OOCGB_NCCL(nccl_api().AllReduce(d_buf, d_buf, count, ncclInt64, ncclSum, c->comm, c->stream));
}
void allreduce_max_u64(oocgb_ctx c, unsigned long long *d_buf, size_t count) {
  if (!c->coll || count == 0) return;
  if (c->host_coll) {
    std::vector<unsigned long long> h(count);
    OOCGB_CK(cudaMemcpyAsync(h.data(), d_buf, 8 * count, cudaMemcpyDeviceToHost, c->stream));
    OOCGB_CK(cudaStreamSynchronize(c->stream));
    OOCGB_REQUIRE(c->host_coll(1, 1, h.data(), (int64_t)count, c->host_coll_user) == 0, OOCGB_ERR_DEVICE,
                  "host collective (all-reduce max) failed");
    OOCGB_CK(cudaMemcpyAsync(d_buf, h.data(), 8 * count, cudaMemcpyHostToDevice, c->stream));
    OOCGB_CK(cudaStreamSynchronize(c->stream));
    return;
  }
  OOCGB_NCCL(nccl_api().AllReduce(d_buf, d_buf, count, ncclUint64, ncclMax, c->comm, c->stream));
}
void allgather_u32(oocgb_ctx c, const uint32_t *d_send, uint32_t *d_recv, size_t count) {
  if (c->host_coll) {
    std::vector<uint32_t> h(count * c->world);
    OOCGB_CK(cudaMemcpyAsync(h.data() + (size_t)c->rank * count, d_send, 4 * count, cudaMemcpyDeviceToHost, c->stream));
    OOCGB_CK(cudaStreamSynchronize(c->stream));
    OOCGB_REQUIRE(c->host_coll(2, 2, h.data(), (int64_t)count, c->host_coll_user) == 0, OOCGB_ERR_DEVICE,
                  "host collective (all-gather) failed");
    OOCGB_CK(cudaMemcpyAsync(d_recv, h.data(), 4 * count * c->world, cudaMemcpyHostToDevice, c->stream));
    OOCGB_CK(cudaStreamSynchronize(c->stream));
    return;
  }
  OOCGB_NCCL(nccl_api().AllGather(d_send, d_recv, count, ncclUint32, c->comm, c->stream));
}

void allgather_i64_inplace(oocgb_ctx c, long long *d_buf, size_t count) {
  if (!c->coll || count == 0) return;
  if (c->host_coll) {  // the transport gathers by summing blocks that are zero outside their owner
    std::vector<long long> h(count * c->world, 0);
    OOCGB_CK(cudaMemcpyAsync(h.data() + (size_t)c->rank * count, d_buf + (size_t)c->rank * count, 8 * count,
                             cudaMemcpyDeviceToHost, c->stream));
    OOCGB_CK(cudaStreamSynchronize(c->stream));
    OOCGB_REQUIRE(c->host_coll(2, 0, h.data(), (int64_t)count, c->host_coll_user) == 0, OOCGB_ERR_DEVICE,
                  "host collective (all-gather) failed");
    OOCGB_CK(cudaMemcpyAsync(d_buf, h.data(), 8 * count * c->world, cudaMemcpyHostToDevice, c->stream));
    OOCGB_CK(cudaStreamSynchronize(c->stream));
    return;
  }
  OOCGB_NCCL(nccl_api().AllGather(d_buf + (size_t)c->rank * count, d_buf, count, ncclInt64, c->comm, c->stream));
}
void reduce_scatter_i64(oocgb_ctx c, const long long *d_send, long long *d_recv, size_t count) {
  if (!c->coll || count == 0) return;
  if (c->host_coll) {  // all-reduce of every block, then keep this rank's
    std::vector<long long> h(count * c->world);
    OOCGB_CK(cudaMemcpyAsync(h.data(), d_send, 8 * count * c->world, cudaMemcpyDeviceToHost, c->stream));
    OOCGB_CK(cudaStreamSynchronize(c->stream));
    OOCGB_REQUIRE(c->host_coll(0, 0, h.data(), (int64_t)(count * c->world), c->host_coll_user) == 0,
                  OOCGB_ERR_DEVICE, "host collective (reduce-scatter) failed");
    OOCGB_CK(cudaMemcpyAsync(d_recv, h.data() + (size_t)c->rank * count, 8 * count, cudaMemcpyHostToDevice,
                             c->stream));
    OOCGB_CK(cudaStreamSynchronize(c->stream));
    return;
  }
  OOCGB_NCCL(nccl_api().ReduceScatter(d_send, d_recv, count, ncclInt64, ncclSum, c->comm, c->stream));
}

cudaEvent_t pool_event(oocgb_ctx c) {
  if (c->ev_pool.empty()) {
    cudaEvent_t e;
    OOCGB_CK(cudaEventCreate(&e));
    return e;
  }
  cudaEvent_t e = c->ev_pool.back();
  c->ev_pool.pop_back();
  return e;
}
PhaseTimer::PhaseTimer(oocgb_ctx c_, int s) : c(c_), slot(s) {
  if (c->profiling) {
    a = pool_event(c);
    OOCGB_CK(cudaEventRecord(a, c->stream));
  }
}
PhaseTimer::~PhaseTimer() {
  if (!a) return;
  cudaEvent_t b = pool_event(c);
  cudaEventRecord(b, c->stream);
  c->pending_slot.push_back(slot);
  c->pending_a.push_back(a);
  c->pending_b.push_back(b);
}
void record_copy_timing(oocgb_ctx c, cudaEvent_t a, cudaEvent_t b) {
  c->pending_slot.push_back(5);
  c->pending_a.push_back(a);
  c->pending_b.push_back(b);
}
void drain_timers(oocgb_ctx c) {
  for (size_t i = 0; i < c->pending_slot.size(); ++i) {
    OOCGB_CK(cudaEventSynchronize(c->pending_b[i]));
    float ms = 0.f;
    OOCGB_CK(cudaEventElapsedTime(&ms, c->pending_a[i], c->pending_b[i]));
    c->timings[c->pending_slot[i]] += ms;
    if (c->pending_slot[i] == 0) c->timings[7] += 1.0;  // histogram launches
    c->ev_pool.push_back(c->pending_a[i]);
    c->ev_pool.push_back(c->pending_b[i]);
  }
  c->pending_slot.clear();
  c->pending_a.clear();
  c->pending_b.clear();
}

void ensure_staging(oocgb_data d) {
  if (d->d_stage[0]) return;
  d->stage_rows = d->rows_per_page;
  for (int i = 0; i < kStages; ++i)
    d->d_stage[i] = (uint8_t *)dmalloc((size_t)std::max<int64_t>(1, d->stage_rows) * d->stride);
}

}  // namespace oocgb

using namespace oocgb;

#define API_BEGIN try {
#define API_END                                  \
  return OOCGB_OK;                               \
  }                                              \
  catch (const oocgb::Error &e) {                \
    set_last_error(e.what());                    \
    return e.status;                             \
  }                                              \
  catch (const std::bad_alloc &) {               \
    set_last_error("host allocation failed");    \
    return OOCGB_ERR_NOMEM;                      \
  }                                              \
  catch (const std::exception &e) {              \
    set_last_error(e.what());                    \
    return OOCGB_ERR_DEVICE;                     \
  }

static void bind(oocgb_ctx c) { OOCGB_CK(cudaSetDevice(c->device)); }

// Device view of a caller array: the pointer itself if it is device memory, else a copy in
// the data handle's persistent staging slot (no per-call allocation).
struct DevView {
  const void *ptr = nullptr;
  bool staged = false;
};
static void *arg_slot(oocgb_data d, int slot, size_t bytes) {
  if (d->arg_bytes[slot] < bytes) {
    dfree(d->d_arg[slot]);
    d->d_arg[slot] = dmalloc(bytes);
    d->arg_bytes[slot] = bytes;
  }
  return d->d_arg[slot];
}
static void view_on_device(oocgb_data d, int slot, const void *src, size_t bytes, DevView &v) {
  if (is_device_ptr(src)) { v.ptr = src; return; }
  void *dst = arg_slot(d, slot, bytes);
  OOCGB_CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, d->ctx->stream));
  v.ptr = dst;
  v.staged = true;
}

static oocgb_data new_data(oocgb_ctx c, int64_t n_local, int64_t row0, int64_t n_global, int m,
                           int max_bin, int64_t page_bytes, int placement, uint64_t seed) {
  OOCGB_REQUIRE(m >= 1, OOCGB_ERR_ARG, "n_features must be >= 1");
  OOCGB_REQUIRE(max_bin >= 2 && max_bin <= 256, OOCGB_ERR_ARG, "max_bin must be in [2, 256] (uint8 symbols)");
  OOCGB_REQUIRE(n_local >= 0 && row0 >= 0 && n_global >= n_local && row0 + n_local <= n_global,
                OOCGB_ERR_ARG, "row counts: need 0 <= row0, row0 + n_rows <= n_rows_global");
  OOCGB_REQUIRE(n_local < (1LL << 31) - kPartTile, OOCGB_ERR_ARG, "at most 2^31 - 2048 rows per GPU");
  OOCGB_REQUIRE(placement == OOCGB_PLACE_DEVICE || placement == OOCGB_PLACE_PINNED_HOST, OOCGB_ERR_ARG,
                "placement must be DEVICE or PINNED_HOST");
  OOCGB_REQUIRE(page_bytes >= 0, OOCGB_ERR_ARG, "page_bytes must be >= 0");
  oocgb_data d = new oocgb_data_s();
  d->ctx = c;
  d->n_local = n_local;
  d->row0 = row0;
  d->n_global = n_global;
  d->m = m;
  d->n_fg = (m + 31) / 32;
  d->gw = plane_width(d->n_fg);
  d->stride = d->gw * ((m + d->gw - 1) / d->gw);  // bytes per row summed over the planes (R5)
  d->max_bin = max_bin;
  d->placement = placement;
  d->seed = seed;
  // DEVICE placement keeps one page (the device-resident ELLPACK matrix, Alg. 4); PINNED_HOST
  // pages hold floor(page_bytes / stride) rows (R6)
  d->rows_per_page = (page_bytes > 0 && placement == OOCGB_PLACE_PINNED_HOST)
                         ? std::max<int64_t>(1, page_bytes / d->stride)
                         : std::max<int64_t>(1, n_local);
  d->n_pages = std::max<int64_t>(1, (n_local + d->rows_per_page - 1) / d->rows_per_page);
  c->live_data++;
  return d;
}

static void free_data(oocgb_data d) {
  free_work(d);
  dfree(d->d_cut_values); dfree(d->d_cut_ptrs); dfree(d->d_bins); dfree(d->d_sketch);
  dfree(d->d_sketch_count); dfree(d->d_g); dfree(d->d_h); dfree(d->d_sel_rows); dfree(d->d_q);
  dfree(d->d_sampled_page); dfree(d->d_gs); dfree(d->d_hs); dfree(d->d_tmp64); dfree(d->d_mvs); dfree(d->d_mvs_stats);
  dfree(d->d_absparts);
  dfree(d->d_missing);
  for (int i = 0; i < 3; ++i) dfree(d->d_stage[i]);
  for (int i = 0; i < 2; ++i) dfree(d->d_arg[i]);
  for (int i = 0; i < 3; ++i) dfree(d->d_bstage[i]);
  if (d->d_ss) cudaFree(d->d_ss);
  if (d->h_ss) cudaFreeHost(d->h_ss);
  if (d->h_pages) cudaFreeHost(d->h_pages);
  d->ctx->live_data--;
  delete d;
}

static void alloc_pages(oocgb_data d) {
  const size_t bytes = (size_t)d->n_pages * (size_t)d->rows_per_page * d->stride;
  if (d->placement == OOCGB_PLACE_DEVICE) {
    d->d_bins = (uint8_t *)dmalloc(bytes);
  } else {
    cudaError_t e = cudaHostAlloc((void **)&d->h_pages, bytes, cudaHostAllocDefault);
    if (e != cudaSuccess) {
      cudaGetLastError();
      throw Error(OOCGB_ERR_NOMEM, "pinned host allocation of " + std::to_string(bytes) + " bytes failed");
    }
  }
}

// Bin rows [row_local0, row_local0 + n) of X (device) straight into the tiled pages: device
// memory, or pinned host memory written zero-copy (mapped, UVA) by the binning kernel.
static void write_pages(oocgb_data d, const float *dX, int64_t row_local0, int64_t n) {
  oocgb_ctx c = d->ctx;
  int *d_err = (int *)((char *)c->d_small + 4096);
  if (!d->d_missing) {
    d->d_missing = (int *)dmalloc(sizeof(int));
    OOCGB_CK(cudaMemsetAsync(d->d_missing, 0, sizeof(int), c->stream));
  }
  OOCGB_CK(cudaMemsetAsync(d_err, 0, sizeof(int), c->stream));
  uint8_t *base = d->placement == OOCGB_PLACE_DEVICE ? d->d_bins : d->h_pages;
  bin_rows(d, dX, n, row_local0, base, d_err);
  int herr = 0, hmiss = 0;
  OOCGB_CK(cudaMemcpyAsync(&herr, d_err, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  OOCGB_CK(cudaMemcpyAsync(&hmiss, d->d_missing, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  OOCGB_CK(cudaStreamSynchronize(c->stream));
  OOCGB_REQUIRE(herr != 2, OOCGB_ERR_ARG, "quantise: +-inf in X (R4; NaN marks a missing value)");
  OOCGB_REQUIRE(herr != 5, OOCGB_ERR_ARG,
                "quantise: missing values need max_bin <= 255 (symbol 255 marks a missing value, R27)");
  OOCGB_REQUIRE(herr == 0, OOCGB_ERR_ARG, "quantise: bad value in X");
  if (hmiss) d->has_missing = true;
}

// After the last page: every rank agrees on has_missing (it changes the split candidates, R27).
static void finish_missing(oocgb_data d) {
  oocgb_ctx c = d->ctx;
  if (!c->coll) return;
  unsigned long long *buf = (unsigned long long *)((char *)c->d_small + 8192);
  unsigned long long v = d->has_missing ? 1 : 0;
  OOCGB_CK(cudaMemcpyAsync(buf, &v, 8, cudaMemcpyHostToDevice, c->stream));
  allreduce_max_u64(c, buf, 1);
  OOCGB_CK(cudaMemcpyAsync(&v, buf, 8, cudaMemcpyDeviceToHost, c->stream));
  OOCGB_CK(cudaStreamSynchronize(c->stream));
  d->has_missing = v != 0;
}

// Run fn(dX_batch, row_offset, n_batch) over X (host or device) in device batches.
template <class F>
static void over_batches(oocgb_ctx c, const float *X, int64_t n, int m, F fn) {
  if (n <= 0) return;
  if (is_device_ptr(X)) { fn(X, 0, n); return; }
  const int64_t batch = std::max<int64_t>(1, (256LL << 20) / ((int64_t)m * 4));
  float *buf = (float *)dmalloc(sizeof(float) * (size_t)std::min(batch, n) * m);
  try {
    for (int64_t r = 0; r < n; r += batch) {
      int64_t nr = std::min(batch, n - r);
      OOCGB_CK(cudaMemcpyAsync(buf, X + r * m, sizeof(float) * (size_t)nr * m, cudaMemcpyHostToDevice, c->stream));
      fn(buf, r, nr);
      OOCGB_CK(cudaStreamSynchronize(c->stream));
    }
  } catch (...) {
    dfree(buf);
    throw;
  }
  dfree(buf);
}

extern "C" {

const char *oocgb_last_error(void) { return g_last_error.c_str(); }
int32_t oocgb_abi_version(void) { return 2; }  // 2: oocgb_node.default_left, oocgb_info.has_missing, CSR input

int oocgb_nccl_unique_id(uint8_t out[128]) {
  API_BEGIN
  OOCGB_REQUIRE(out, OOCGB_ERR_ARG, "out is NULL");
  ncclUniqueId id;
  OOCGB_NCCL(nccl_api().GetUniqueId(&id));
  static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
  memcpy(out, &id, 128);
  API_END
}

int oocgb_ctx_create(int32_t device, int32_t rank, int32_t world, const uint8_t *nccl_id,
                     uint64_t cuda_stream, oocgb_ctx *out) {
  API_BEGIN
  OOCGB_REQUIRE(out, OOCGB_ERR_ARG, "out is NULL");
  OOCGB_REQUIRE(world >= 1 && rank >= 0 && rank < world, OOCGB_ERR_ARG, "need 0 <= rank < world");
  OOCGB_REQUIRE(world == 1 || nccl_id, OOCGB_ERR_ARG, "nccl_id required when world > 1");
  int ndev = 0;
  OOCGB_CK(cudaGetDeviceCount(&ndev));
  OOCGB_REQUIRE(device >= 0 && device < ndev, OOCGB_ERR_ARG, "device out of range");
  OOCGB_CK(cudaSetDevice(device));
  oocgb_ctx c = new oocgb_ctx_s();
  c->device = device;
  c->rank = rank;
  c->world = world;
  try {
    cudaDeviceProp p;
    OOCGB_CK(cudaGetDeviceProperties(&p, device));
    c->num_sms = p.multiProcessorCount;
    if (cuda_stream) {
      c->stream = (cudaStream_t)cuda_stream;
    } else {
      OOCGB_CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
      c->own_stream = true;
    }
    OOCGB_CK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    for (int i = 0; i < 3; ++i) {
      OOCGB_CK(cudaEventCreateWithFlags(&c->pipe_copy_done[i], cudaEventDisableTiming));
      OOCGB_CK(cudaEventCreateWithFlags(&c->pipe_consumed[i], cudaEventDisableTiming));
    }
    OOCGB_CK(cudaMalloc(&c->d_small, 1 << 20));
    OOCGB_CK(cudaMallocHost(&c->h_small, 1 << 20));
    if (world > 1 || nccl_id) {  // world == 1 with an id: the multi-GPU path on a 1-rank communicator
      ncclUniqueId id;
      memcpy(&id, nccl_id, 128);
      OOCGB_NCCL(nccl_api().CommInitRank(&c->comm, world, id, rank));
      c->coll = true;
    }
  } catch (...) {
    if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    for (int i = 0; i < 3; ++i) {
      if (c->pipe_copy_done[i]) cudaEventDestroy(c->pipe_copy_done[i]);
      if (c->pipe_consumed[i]) cudaEventDestroy(c->pipe_consumed[i]);
    }
    if (c->d_small) cudaFree(c->d_small);
    if (c->h_small) cudaFreeHost(c->h_small);
    delete c;
    throw;
  }
  *out = c;
  API_END
}

int oocgb_ctx_create_hostcomm(int32_t device, int32_t rank, int32_t world, oocgb_collective_fn fn, void *user,
                              uint64_t cuda_stream, oocgb_ctx *out) {
  API_BEGIN
  OOCGB_REQUIRE(fn && out, OOCGB_ERR_ARG, "collective callback / out is NULL");
  OOCGB_REQUIRE(world >= 1 && rank >= 0 && rank < world, OOCGB_ERR_ARG, "need 0 <= rank < world");
  oocgb_ctx c = nullptr;
  const int rc = oocgb_ctx_create(device, 0, 1, nullptr, cuda_stream, &c);
  if (rc != OOCGB_OK) return rc;
  c->rank = rank;
  c->world = world;
  c->host_coll = fn;
  c->host_coll_user = user;
  c->coll = world > 1;
  *out = c;
  API_END
}

int oocgb_ctx_destroy(oocgb_ctx c) {
  API_BEGIN
  OOCGB_REQUIRE(c, OOCGB_ERR_ARG, "ctx is NULL");
  OOCGB_REQUIRE(c->live_data == 0, OOCGB_ERR_STATE, "ctx_destroy: data handles are still alive");
  OOCGB_REQUIRE(c->live_trees == 0, OOCGB_ERR_STATE, "ctx_destroy: tree handles are still alive");
  bind(c);
  for (int i = 0; i < 3; ++i) {
    if (c->pipe_copy_done[i]) cudaEventDestroy(c->pipe_copy_done[i]);
    if (c->pipe_consumed[i]) cudaEventDestroy(c->pipe_consumed[i]);
  }
  cudaStreamSynchronize(c->stream);
  if (c->comm) nccl_api().CommDestroy(c->comm);
  for (auto e : c->ev_pool) cudaEventDestroy(e);
  for (auto e : c->pending_a) cudaEventDestroy(e);
  for (auto e : c->pending_b) cudaEventDestroy(e);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  cudaStreamDestroy(c->copy_stream);
  for (auto &p : c->node_pool) cudaFree(p.second);
  cudaFree(c->d_small);
  cudaFreeHost(c->h_small);
  delete c;
  API_END
}

int oocgb_quantise(oocgb_ctx c, const float *X, int64_t n_rows, int64_t row0_global, int64_t n_rows_global,
                   int32_t n_features, int32_t max_bin, int64_t page_bytes, int32_t placement, uint64_t seed,
                   oocgb_data *out) {
  API_BEGIN
  OOCGB_REQUIRE(c && out, OOCGB_ERR_ARG, "ctx/out is NULL");
  OOCGB_REQUIRE(X || n_rows == 0, OOCGB_ERR_ARG, "X is NULL");
  bind(c);
  oocgb_data d = new_data(c, n_rows, row0_global, n_rows_global, n_features, max_bin, page_bytes, placement, seed);
  try {
    // Alg. 2 (sketch) then Alg. 4/5 (ELLPACK pages)
    over_batches(c, X, n_rows, n_features, [&](const float *dX, int64_t r, int64_t nr) {
      sketch_append(d, dX, row0_global + r, nr);
    });
    cuts_finalize(d);
    alloc_pages(d);
    over_batches(c, X, n_rows, n_features, [&](const float *dX, int64_t r, int64_t nr) {
      write_pages(d, dX, r, nr);
    });
    d->rows_written = n_rows;
    finish_missing(d);
  } catch (...) {
    free_data(d);
    throw;
  }
  *out = d;
  API_END
}

// Sparse CSR input (R27): the rows are expanded batch by batch to dense float32 with NaN at the
// absent entries (csr_to_dense, on the device) and go through exactly the dense path's two passes,
// so cuts and pages equal oocgb_quantise on the NaN-filled matrix.
int oocgb_quantise_csr(oocgb_ctx c, const int64_t *indptr, const int32_t *indices, const float *values,
                       int64_t n_rows, int64_t row0_global, int64_t n_rows_global, int32_t n_features,
                       int32_t max_bin, int64_t page_bytes, int32_t placement, uint64_t seed, oocgb_data *out) {
  API_BEGIN
  OOCGB_REQUIRE(c && out && (indptr || n_rows == 0), OOCGB_ERR_ARG, "NULL argument");
  OOCGB_REQUIRE(n_rows >= 0 && n_features > 0, OOCGB_ERR_ARG, "quantise_csr: bad sizes");
  bind(c);
  // row pointers on the host (sizes) and on the device (the scatter kernel)
  std::vector<int64_t> hptr(n_rows + 1, 0);
  if (n_rows >= 0 && indptr) {
    if (is_device_ptr(indptr))
      OOCGB_CK(cudaMemcpy(hptr.data(), indptr, sizeof(int64_t) * (n_rows + 1), cudaMemcpyDeviceToHost));
    else
      memcpy(hptr.data(), indptr, sizeof(int64_t) * (n_rows + 1));
  }
  const int64_t base = hptr[0], nnz = hptr[n_rows] - base;
  OOCGB_REQUIRE(nnz >= 0 && (nnz == 0 || (indices && values)), OOCGB_ERR_ARG, "quantise_csr: bad indptr / arrays");
  for (int64_t i = 0; i < n_rows; ++i)
    OOCGB_REQUIRE(hptr[i + 1] >= hptr[i] && hptr[i + 1] - hptr[i] <= n_features, OOCGB_ERR_ARG,
                  "quantise_csr: indptr must be non-decreasing with <= n_features entries per row");
  int64_t *d_ptr = (int64_t *)dmalloc(sizeof(int64_t) * (n_rows + 1));
  int32_t *d_idx = (int32_t *)dmalloc(sizeof(int32_t) * std::max<int64_t>(1, nnz));
  float *d_val = (float *)dmalloc(sizeof(float) * std::max<int64_t>(1, nnz));
  const int64_t batch = std::max<int64_t>(1, (256LL << 20) / ((int64_t)n_features * 4));
  float *buf = (float *)dmalloc(sizeof(float) * (size_t)std::max<int64_t>(1, std::min(batch, n_rows)) * n_features);
  oocgb_data d = nullptr;
  try {
    OOCGB_CK(cudaMemcpyAsync(d_ptr, hptr.data(), sizeof(int64_t) * (n_rows + 1), cudaMemcpyHostToDevice, c->stream));
    if (nnz > 0) {
      OOCGB_CK(cudaMemcpyAsync(d_idx, indices + base, sizeof(int32_t) * nnz, cudaMemcpyDefault, c->stream));
      OOCGB_CK(cudaMemcpyAsync(d_val, values + base, sizeof(float) * nnz, cudaMemcpyDefault, c->stream));
    }
    int *d_err = (int *)((char *)c->d_small + 12288);
    OOCGB_CK(cudaMemsetAsync(d_err, 0, sizeof(int), c->stream));
    d = new_data(c, n_rows, row0_global, n_rows_global, n_features, max_bin, page_bytes, placement, seed);
    auto each_batch = [&](auto fn) {
      for (int64_t r = 0; r < n_rows; r += batch) {
        const int64_t nr = std::min(batch, n_rows - r);
        csr_to_dense(c, d_ptr, d_idx, d_val, base, r, nr, n_features, buf, d_err);
        fn(buf, r, nr);
        OOCGB_CK(cudaStreamSynchronize(c->stream));
      }
      int herr = 0;
      OOCGB_CK(cudaMemcpy(&herr, d_err, sizeof(int), cudaMemcpyDeviceToHost));
      OOCGB_REQUIRE(herr == 0, OOCGB_ERR_ARG, "quantise_csr: a column index outside [0, n_features)");
    };
    each_batch([&](const float *dX, int64_t r, int64_t nr) { sketch_append(d, dX, row0_global + r, nr); });
    cuts_finalize(d);
    alloc_pages(d);
    each_batch([&](const float *dX, int64_t r, int64_t nr) { write_pages(d, dX, r, nr); });
    d->rows_written = n_rows;
    finish_missing(d);
  } catch (...) {
    if (d) free_data(d);
    dfree(d_ptr); dfree(d_idx); dfree(d_val); dfree(buf);
    throw;
  }
  dfree(d_ptr); dfree(d_idx); dfree(d_val); dfree(buf);
  *out = d;
  API_END
}

int oocgb_sketch_begin(oocgb_ctx c, int32_t n_features, int32_t max_bin, int64_t n_rows, int64_t row0_global,
                       int64_t n_rows_global, int64_t page_bytes, int32_t placement, uint64_t seed,
                       oocgb_data *out) {
  API_BEGIN
  OOCGB_REQUIRE(c && out, OOCGB_ERR_ARG, "ctx/out is NULL");
  bind(c);
  oocgb_data d = new_data(c, n_rows, row0_global, n_rows_global, n_features, max_bin, page_bytes, placement, seed);
  *out = d;
  API_END
}

int oocgb_sketch_push(oocgb_data d, const float *X, int64_t row0_global, int64_t n) {
  API_BEGIN
  OOCGB_REQUIRE(d && (X || n == 0), OOCGB_ERR_ARG, "data/X is NULL");
  OOCGB_REQUIRE(!d->cuts_ready, OOCGB_ERR_STATE, "sketch_push after cuts_finalize");
  OOCGB_REQUIRE(row0_global >= d->row0 && row0_global + n <= d->row0 + d->n_local, OOCGB_ERR_ARG,
                "sketch_push: rows outside this rank's range");
  bind(d->ctx);
  over_batches(d->ctx, X, n, d->m, [&](const float *dX, int64_t r, int64_t nr) {
    sketch_append(d, dX, row0_global + r, nr);
  });
  API_END
}

int oocgb_cuts_finalize(oocgb_data d) {
  API_BEGIN
  OOCGB_REQUIRE(d, OOCGB_ERR_ARG, "data is NULL");
  OOCGB_REQUIRE(!d->cuts_ready, OOCGB_ERR_STATE, "cuts already finalized");
  bind(d->ctx);
  cuts_finalize(d);
  alloc_pages(d);
  API_END
}

int oocgb_pages_push(oocgb_data d, const float *X, int64_t row0_global, int64_t n) {
  API_BEGIN
  OOCGB_REQUIRE(d && (X || n == 0), OOCGB_ERR_ARG, "data/X is NULL");
  OOCGB_REQUIRE(d->cuts_ready, OOCGB_ERR_STATE, "pages_push before cuts_finalize");
  OOCGB_REQUIRE(row0_global == d->row0 + d->rows_written && d->rows_written + n <= d->n_local, OOCGB_ERR_ARG,
                "pages_push: rows must arrive in ascending global order, each once");
  bind(d->ctx);
  const int64_t base = d->rows_written;
  over_batches(d->ctx, X, n, d->m, [&](const float *dX, int64_t r, int64_t nr) {
    write_pages(d, dX, base + r, nr);
  });
  d->rows_written += n;
  if (d->rows_written == d->n_local) finish_missing(d);
  API_END
}

int oocgb_quantise_like(oocgb_data ref, const float *X, int64_t n_rows, int32_t placement, oocgb_data *out) {
  API_BEGIN
  OOCGB_REQUIRE(ref && out && (X || n_rows == 0), OOCGB_ERR_ARG, "NULL argument");
  OOCGB_REQUIRE(ref->cuts_ready, OOCGB_ERR_STATE, "reference data has no cuts");
  oocgb_ctx c = ref->ctx;
  bind(c);
  oocgb_data d = new_data(c, n_rows, 0, n_rows, ref->m, ref->max_bin,
                          ref->rows_per_page * (int64_t)ref->stride, placement, ref->seed);
  try {
    d->h_cut_values = ref->h_cut_values;
    d->h_cut_ptrs = ref->h_cut_ptrs;
    d->d_cut_values = (float *)dmalloc(sizeof(float) * std::max<size_t>(1, d->h_cut_values.size()));
    d->d_cut_ptrs = (int32_t *)dmalloc(sizeof(int32_t) * (d->m + 1));
    OOCGB_CK(cudaMemcpyAsync(d->d_cut_values, d->h_cut_values.data(), sizeof(float) * d->h_cut_values.size(),
                             cudaMemcpyHostToDevice, c->stream));
    OOCGB_CK(cudaMemcpyAsync(d->d_cut_ptrs, d->h_cut_ptrs.data(), sizeof(int32_t) * (d->m + 1),
                             cudaMemcpyHostToDevice, c->stream));
    d->cuts_ready = true;
    alloc_pages(d);
    over_batches(c, X, n_rows, d->m, [&](const float *dX, int64_t r, int64_t nr) { write_pages(d, dX, r, nr); });
    d->rows_written = n_rows;
    d->has_missing = d->has_missing || ref->has_missing;
  } catch (...) {
    free_data(d);
    throw;
  }
  *out = d;
  API_END
}

int oocgb_data_info(oocgb_data d, oocgb_info *out) {
  API_BEGIN
  OOCGB_REQUIRE(d && out, OOCGB_ERR_ARG, "NULL argument");
  out->n_rows_local = d->n_local;
  out->n_rows_global = d->n_global;
  out->row0_global = d->row0;
  out->n_features = d->m;
  out->row_stride = d->stride;
  out->max_bin = d->max_bin;
  out->placement = d->placement;
  out->n_pages = d->n_pages;
  out->rows_per_page = d->rows_per_page;
  out->total_cuts = (int64_t)d->h_cut_values.size();
  out->has_missing = d->has_missing ? 1 : 0;
  out->pad = 0;
  API_END
}

int oocgb_data_destroy(oocgb_data d) {
  API_BEGIN
  OOCGB_REQUIRE(d, OOCGB_ERR_ARG, "data is NULL");
  bind(d->ctx);
  cudaStreamSynchronize(d->ctx->stream);
  free_data(d);
  API_END
}

static void ensure_grad(oocgb_data d) {
  if (!d->d_g) {
    d->d_g = (float *)dmalloc(sizeof(float) * std::max<int64_t>(1, d->n_local));
    d->d_h = (float *)dmalloc(sizeof(float) * std::max<int64_t>(1, d->n_local));
  }
}

int oocgb_set_gradients(oocgb_data d, const float *g, const float *h, int64_t n_local) {
  API_BEGIN
  OOCGB_REQUIRE(d && ((g && h) || n_local == 0), OOCGB_ERR_ARG, "NULL argument");
  OOCGB_REQUIRE(n_local == d->n_local, OOCGB_ERR_ARG, "set_gradients: length != n_rows_local");
  oocgb_ctx c = d->ctx;
  bind(c);
  ensure_grad(d);
  if (n_local > 0) {
    OOCGB_CK(cudaMemcpyAsync(d->d_g, g, sizeof(float) * n_local, cudaMemcpyDefault, c->stream));
    OOCGB_CK(cudaMemcpyAsync(d->d_h, h, sizeof(float) * n_local, cudaMemcpyDefault, c->stream));
    if (!is_device_ptr(g) || !is_device_ptr(h)) OOCGB_CK(cudaStreamSynchronize(c->stream));
  }
  d->has_grad = true;
  d->has_sample = false;
  API_END
}

int oocgb_set_logistic_gradients(oocgb_data d, const float *margin, const float *labels, int64_t n_local) {
  API_BEGIN
  OOCGB_REQUIRE(d && ((margin && labels) || n_local == 0), OOCGB_ERR_ARG, "NULL argument");
  OOCGB_REQUIRE(n_local == d->n_local, OOCGB_ERR_ARG, "set_logistic_gradients: length != n_rows_local");
  oocgb_ctx c = d->ctx;
  bind(c);
  ensure_grad(d);
  DevView vm, vy;
  if (n_local > 0) {
    view_on_device(d, 0, margin, sizeof(float) * n_local, vm);
    view_on_device(d, 1, labels, sizeof(float) * n_local, vy);
    logistic_gradients(d, (const float *)vm.ptr, (const float *)vy.ptr);
    if (vm.staged || vy.staged) OOCGB_CK(cudaStreamSynchronize(c->stream));
  }
  d->has_grad = true;
  d->has_sample = false;
  API_END
}

int oocgb_sample(oocgb_data d, int32_t mode, double ratio, double mvs_lambda, uint64_t seed, uint64_t round,
                 int32_t quant_bits, oocgb_sample_info *info) {
  API_BEGIN
  OOCGB_REQUIRE(d, OOCGB_ERR_ARG, "data is NULL");
  OOCGB_REQUIRE(mode >= 0 && mode <= 2, OOCGB_ERR_ARG, "mode must be NONE, UNIFORM or MVS");
  OOCGB_REQUIRE(ratio > 0.0 && ratio <= 1.0, OOCGB_ERR_ARG, "ratio must be in (0, 1] (S:L302)");
  OOCGB_REQUIRE(mvs_lambda >= 0.0 && std::isfinite(mvs_lambda), OOCGB_ERR_ARG, "mvs_lambda must be >= 0");
  OOCGB_REQUIRE(quant_bits >= 8 && quant_bits <= 20, OOCGB_ERR_ARG, "quant_bits must be in [8, 20] (R12)");
  OOCGB_REQUIRE(d->cuts_ready && d->rows_written == d->n_local, OOCGB_ERR_STATE, "sample: pages not complete");
  OOCGB_REQUIRE(d->has_grad, OOCGB_ERR_STATE, "sample before set_gradients");
  bind(d->ctx);
  d->sample_serial++;
  sample_rows(d, mode, ratio, mvs_lambda, seed, round, quant_bits, info);
  API_END
}

int oocgb_sample_goss(oocgb_data d, double a, double b, uint64_t seed, uint64_t round, int32_t quant_bits,
                      oocgb_sample_info *info) {
  API_BEGIN
  OOCGB_REQUIRE(d, OOCGB_ERR_ARG, "data is NULL");
  OOCGB_REQUIRE(a >= 0.0 && b > 0.0 && a + b <= 1.0 && std::isfinite(a) && std::isfinite(b), OOCGB_ERR_ARG,
                "GOSS needs 0 <= a, 0 < b, a + b <= 1 (S:L309)");
  OOCGB_REQUIRE(nearbyint(a * 4294967296.0) < 4294967296.0, OOCGB_ERR_ARG, "GOSS needs a < 1");
  OOCGB_REQUIRE(quant_bits >= 8 && quant_bits <= 20, OOCGB_ERR_ARG, "quant_bits must be in [8, 20] (R12)");
  OOCGB_REQUIRE(d->cuts_ready && d->rows_written == d->n_local, OOCGB_ERR_STATE, "sample: pages not complete");
  OOCGB_REQUIRE(d->has_grad, OOCGB_ERR_STATE, "sample before set_gradients");
  bind(d->ctx);
  d->sample_serial++;
  sample_rows(d, OOCGB_SAMPLE_GOSS, a, 0.0, seed, round, quant_bits, info, b);
  API_END
}

int oocgb_set_streaming(oocgb_data d, int32_t enable) {
  API_BEGIN
  OOCGB_REQUIRE(d, OOCGB_ERR_ARG, "data is NULL");
  OOCGB_REQUIRE(!enable || d->placement == OOCGB_PLACE_PINNED_HOST, OOCGB_ERR_ARG,
                "streamed build needs PINNED_HOST pages");
  d->streamed = enable != 0;
  d->has_sample = false;
  d->sample_serial++;
  API_END
}

int oocgb_build_tree(oocgb_data d, int32_t max_depth, double lambda, double gamma, double min_child_weight,
                     double eta, int32_t keep_debug, oocgb_tree *out) {
  API_BEGIN
  OOCGB_REQUIRE(d && out, OOCGB_ERR_ARG, "NULL argument");
  OOCGB_REQUIRE(max_depth >= 0 && max_depth <= 16, OOCGB_ERR_ARG, "max_depth must be in [0, 16]");
  OOCGB_REQUIRE(lambda >= 0.0 && std::isfinite(lambda) && std::isfinite(gamma) && std::isfinite(eta) &&
                    std::isfinite(min_child_weight),
                OOCGB_ERR_ARG, "lambda >= 0 and finite gamma / eta / min_child_weight required");
  OOCGB_REQUIRE(d->has_sample, OOCGB_ERR_STATE, "build_tree before sample");
  bind(d->ctx);
  if (d->streamed && d->placement == OOCGB_PLACE_PINNED_HOST && d->all_selected)
    *out = build_tree_streamed(d, max_depth, lambda, gamma, min_child_weight, eta, keep_debug != 0);
  else
    *out = build_tree(d, max_depth, lambda, gamma, min_child_weight, eta, keep_debug != 0);
  API_END
}

int oocgb_tree_export(oocgb_tree t, oocgb_node *nodes, int32_t capacity, int32_t *n_nodes) {
  API_BEGIN
  OOCGB_REQUIRE(t && n_nodes, OOCGB_ERR_ARG, "NULL argument");
  *n_nodes = (int32_t)t->nodes.size();
  if (nodes) {
    OOCGB_REQUIRE(capacity >= (int32_t)t->nodes.size(), OOCGB_ERR_ARG, "tree_export: capacity too small");
    memcpy(nodes, t->nodes.data(), sizeof(oocgb_node) * t->nodes.size());
  }
  API_END
}

int oocgb_tree_destroy(oocgb_tree t) {
  API_BEGIN
  OOCGB_REQUIRE(t, OOCGB_ERR_ARG, "tree is NULL");
  // stream-ordered reuse: later users of the buffer run after every kernel already enqueued
  pool_put(t->ctx, t->pnodes_bytes, t->d_pnodes);
  t->ctx->live_trees--;
  delete t;
  API_END
}

int oocgb_predict(oocgb_data d, const oocgb_tree *trees, int32_t n_trees, float *margin) {
  API_BEGIN
  OOCGB_REQUIRE(d && (trees || n_trees == 0) && (margin || d->n_local == 0), OOCGB_ERR_ARG, "NULL argument");
  OOCGB_REQUIRE(d->cuts_ready && d->rows_written == d->n_local, OOCGB_ERR_STATE, "predict: pages not complete");
  for (int t = 0; t < n_trees; ++t) OOCGB_REQUIRE(trees[t], OOCGB_ERR_ARG, "NULL tree");
  oocgb_ctx c = d->ctx;
  bind(c);
  PhaseTimer timer(c, 4);
  if (d->n_local == 0 || n_trees == 0) return OOCGB_OK;
  const bool dev = is_device_ptr(margin);
  float *dm = margin;
  if (!dev) {
    dm = (float *)arg_slot(d, 0, sizeof(float) * d->n_local);
    OOCGB_CK(cudaMemcpyAsync(dm, margin, sizeof(float) * d->n_local, cudaMemcpyHostToDevice, c->stream));
  }
  {
    for (int t0 = 0; t0 < n_trees; t0 += 4096) {
      int nt = std::min(4096, n_trees - t0);
      if (d->placement == OOCGB_PLACE_DEVICE) {
        predict_device(d, d->d_bins, d->gw, (size_t)d->rows_per_page * d->gw, d->gw == 64 ? 6 : 5, d->n_local, 0,
                       trees + t0, nt, dm);
      } else {
        for_each_page(d, [&](const uint8_t *page, int64_t r0, int64_t nr) {
          predict_device(d, page, (size_t)d->stride, 32, 5, nr, r0, trees + t0, nt, dm);  // row-major page
        });
      }
    }
    if (!dev) {
      OOCGB_CK(cudaMemcpyAsync(margin, dm, sizeof(float) * d->n_local, cudaMemcpyDeviceToHost, c->stream));
      OOCGB_CK(cudaStreamSynchronize(c->stream));
    }
  }
  if (d->placement == OOCGB_PLACE_PINNED_HOST) OOCGB_CK(cudaStreamSynchronize(c->stream));  // staging reuse
  API_END
}

int oocgb_update_margin(oocgb_data d, oocgb_tree t, float *margin) {
  API_BEGIN
  OOCGB_REQUIRE(d && t && (margin || d->n_local == 0), OOCGB_ERR_ARG, "NULL argument");
  OOCGB_REQUIRE(t->owner == d, OOCGB_ERR_STATE, "update_margin: tree built from another data handle");
  oocgb_ctx c = d->ctx;
  bind(c);
  PhaseTimer timer(c, 4);
  if (d->n_local == 0) return OOCGB_OK;
  const bool dev = is_device_ptr(margin);
  float *dm = margin;
  if (!dev) {
    dm = (float *)arg_slot(d, 0, sizeof(float) * d->n_local);
    OOCGB_CK(cudaMemcpyAsync(dm, margin, sizeof(float) * d->n_local, cudaMemcpyHostToDevice, c->stream));
  }
  update_margin(d, t, dm);
  if (!dev) {
    OOCGB_CK(cudaMemcpyAsync(margin, dm, sizeof(float) * d->n_local, cudaMemcpyDeviceToHost, c->stream));
    OOCGB_CK(cudaStreamSynchronize(c->stream));
  }
  API_END
}

int oocgb_get_cuts(oocgb_data d, float *values, int32_t *offsets) {
  API_BEGIN
  OOCGB_REQUIRE(d && values && offsets, OOCGB_ERR_ARG, "NULL argument");
  OOCGB_REQUIRE(d->cuts_ready, OOCGB_ERR_STATE, "no cuts yet");
  memcpy(values, d->h_cut_values.data(), sizeof(float) * d->h_cut_values.size());
  memcpy(offsets, d->h_cut_ptrs.data(), sizeof(int32_t) * d->h_cut_ptrs.size());
  API_END
}

int oocgb_get_bins(oocgb_data d, int64_t row0_local, int64_t n, uint8_t *out) {
  API_BEGIN
  OOCGB_REQUIRE(d && (out || n == 0), OOCGB_ERR_ARG, "NULL argument");
  OOCGB_REQUIRE(row0_local >= 0 && n >= 0 && row0_local + n <= d->rows_written, OOCGB_ERR_ARG,
                "get_bins: row range outside the written pages");
  bind(d->ctx);
  if (n == 0) return OOCGB_OK;
  if (d->placement == OOCGB_PLACE_PINNED_HOST) {  // pinned pages are already row-major
    memcpy(out, d->h_pages + (size_t)row0_local * d->stride, (size_t)n * d->stride);
    return OOCGB_OK;
  }
  // tiled pages -> row-major [n][stride] (ABI order: row i, feature j at out[i * stride + j])
  const int64_t rpp = d->rows_per_page;
  std::vector<uint8_t> page_buf;
  for (int64_t r = row0_local; r < row0_local + n;) {
    const int64_t p = r / rpp, r_in = r - p * rpp;
    const int64_t cnt = std::min<int64_t>(rpp - r_in, row0_local + n - r);
    const int gw = d->gw;
    for (int g = 0; g < d->stride / gw; ++g) {
      const size_t off = ell_off(r, gw * g, rpp, gw, d->stride);
      const uint8_t *src;
      if (d->placement == OOCGB_PLACE_DEVICE) {
        page_buf.resize((size_t)cnt * gw);
        OOCGB_CK(cudaMemcpy(page_buf.data(), d->d_bins + off, (size_t)cnt * gw, cudaMemcpyDeviceToHost));
        src = page_buf.data();
      } else {
        src = d->h_pages + off;
      }
      for (int64_t i = 0; i < cnt; ++i)
        memcpy(out + (size_t)(r - row0_local + i) * d->stride + gw * g, src + (size_t)i * gw, gw);
    }
    r += cnt;
  }
  API_END
}

int oocgb_get_sample(oocgb_data d, int64_t *gid, int64_t *q_g, int64_t *q_h) {
  API_BEGIN
  OOCGB_REQUIRE(d, OOCGB_ERR_ARG, "NULL argument");
  OOCGB_REQUIRE(d->has_sample, OOCGB_ERR_STATE, "get_sample before sample");
  bind(d->ctx);
  const int64_t n = d->n_sel;
  std::vector<int2> q(n);
  std::vector<int32_t> rows(n);
  if (n) {
    OOCGB_CK(cudaMemcpy(q.data(), d->d_q, sizeof(int2) * n, cudaMemcpyDeviceToHost));
    if (!d->all_selected) OOCGB_CK(cudaMemcpy(rows.data(), d->d_sel_rows, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
  }
  for (int64_t i = 0; i < n; ++i) {
    if (gid) gid[i] = d->row0 + (d->all_selected ? i : rows[i]);
    if (q_g) q_g[i] = q[i].x;
    if (q_h) q_h[i] = q[i].y;
  }
  API_END
}

int oocgb_get_histogram(oocgb_tree t, int32_t node, int64_t *gh) {
  API_BEGIN
  OOCGB_REQUIRE(t && gh, OOCGB_ERR_ARG, "NULL argument");
  OOCGB_REQUIRE(t->debug, OOCGB_ERR_STATE, "get_histogram needs build_tree(keep_debug=1)");
  OOCGB_REQUIRE(node >= 0 && node < (1 << t->max_depth) - 1, OOCGB_ERR_ARG, "node must have depth < max_depth");
  const size_t hsz = (size_t)t->owner->m * kBins * 2;
  memcpy(gh, t->hist.data() + hsz * node, sizeof(int64_t) * hsz);
  API_END
}

int oocgb_get_partition(oocgb_tree t, int32_t *leaf_of_row) {
  API_BEGIN
  OOCGB_REQUIRE(t && leaf_of_row, OOCGB_ERR_ARG, "NULL argument");
  OOCGB_REQUIRE(t->debug, OOCGB_ERR_STATE, "get_partition needs build_tree(keep_debug=1)");
  memcpy(leaf_of_row, t->leaf_of_row.data(), sizeof(int32_t) * t->leaf_of_row.size());
  API_END
}

int oocgb_get_row_order(oocgb_tree t, int32_t *row_order) {
  API_BEGIN
  OOCGB_REQUIRE(t && row_order, OOCGB_ERR_ARG, "NULL argument");
  OOCGB_REQUIRE(t->debug && t->has_row_order, OOCGB_ERR_STATE,
                "get_row_order needs an in-core build_tree(keep_debug=1)");
  memcpy(row_order, t->row_order.data(), sizeof(int32_t) * t->row_order.size());
  API_END
}

int oocgb_get_timings(oocgb_ctx c, double *out, int32_t n) {
  API_BEGIN
  OOCGB_REQUIRE(c && out, OOCGB_ERR_ARG, "NULL argument");
  bind(c);
  drain_timers(c);
  for (int i = 0; i < n && i < 16; ++i) out[i] = c->timings[i];
  for (int i = 0; i < 16; ++i) c->timings[i] = 0.0;
  API_END
}

int oocgb_set_profiling(oocgb_ctx c, int32_t enable) {
  API_BEGIN
  OOCGB_REQUIRE(c, OOCGB_ERR_ARG, "NULL argument");
  bind(c);
  drain_timers(c);
  c->profiling = enable != 0;
  for (int i = 0; i < 16; ++i) c->timings[i] = 0.0;
  API_END
}

}  // extern "C"
