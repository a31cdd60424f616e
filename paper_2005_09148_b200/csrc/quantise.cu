// Quantile sketch (Alg. 2-3) and ELLPACK page writer (Alg. 4-5)
// for sm_100a.  One-time preprocessing ("should only be done once at the beginning of
// training") — not in sec/round.
//
// Cuts (R1-R4): a global-row-keyed Philox Bernoulli sample of <= 2^20 rows (all rows when
// n_global <= 2^20) is gathered as order-preserving uint32 keys, sorted per feature with a
// segmented radix sort (CUB, a library sort primitive), and the cut of rank ceil(b N / B) is
// read for b = 1..B (or every distinct value when there are <= B of them).
// Bins (R3, R5): bin = lower_bound(cuts_j, x) clamped to B_j - 1, one byte per (row, feature).
#include <cub/device/device_segmented_radix_sort.cuh>

#include "internal.cuh"
#include "philox.cuh"

namespace oocgb {

// Order-preserving float -> uint32 key, -0.0 canonicalised to +0.0 (R4).  A missing value (NaN,
// R27) gets the largest key 0xFFFFFFFF, above every finite key (<= 0xFF7FFFFF): it sorts last and
// the cut extraction stops before it (like the all-gather's padding rows).
constexpr uint32_t kMissingKey = 0xFFFFFFFFu;
__device__ __forceinline__ uint32_t float_key(float x) {
  if (isnan(x)) return kMissingKey;
  if (x == 0.0f) x = 0.0f;
  uint32_t u = __float_as_uint(x);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key_float(uint32_t k) {
  uint32_t u = (k & 0x80000000u) ? (k ^ 0x80000000u) : ~k;
  return __uint_as_float(u);
}

// One warp per row: Philox selection (stream 1, round 2^64-1, R2), then the row's m keys are
// appended row-major at an atomically claimed slot (slot order is irrelevant: keys are sorted).
__global__ void k_sketch_append(const float *__restrict__ X, int64_t n, int m, int64_t row0_global,
                                int64_t n_global, uint64_t seed, bool all_rows, uint32_t *sample,
                                int64_t cap, unsigned long long *count, int *err) {
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  int nwarps = (gridDim.x * blockDim.x) >> 5;
  const double p = (double)(1 << 20) / (double)n_global;
  for (int64_t r = warp; r < n; r += nwarps) {
    bool sel = true;
    if (!all_rows) sel = philox_uniform(seed, ~0ull, (uint64_t)(row0_global + r), 1) < p;
    if (!sel) continue;
    unsigned long long slot = 0;
    if (lane == 0) slot = atomicAdd(count, 1ull);
    slot = __shfl_sync(0xffffffffu, slot, 0);
    if ((int64_t)slot >= cap) {
      if (lane == 0) atomicExch(err, 3);
      continue;
    }
    const float *xr = X + r * (int64_t)m;
    uint32_t *out = sample + (int64_t)slot * m;
    for (int j = lane; j < m; j += 32) {
      float x = xr[j];
      if (isinf(x)) atomicExch(err, 2);  // R4; NaN = missing (R27)
      out[j] = float_key(x);
    }
  }
}

// Row-major [N][m] -> column-major [m][N] through a padded 32x32 shared tile.
__global__ void k_transpose_keys(const uint32_t *__restrict__ in, int64_t N, int m,
                                 uint32_t *__restrict__ out) {
  __shared__ uint32_t t[32][33];
  int64_t r0 = (int64_t)blockIdx.x * 32;
  int c0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    int64_t r = r0 + i;
    int c = c0 + threadIdx.x;
    if (r < N && c < m) t[i][threadIdx.x] = in[r * m + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    int c = c0 + i;
    int64_t r = r0 + threadIdx.x;
    if (r < N && c < m) out[(int64_t)c * N + r] = t[threadIdx.x][i];
  }
}

// One block per feature over its sorted keys s[0..N): O1 steps 3-5 on the feature's present
// values, s[0..N_j) with N_j = the first missing / padding key (R27).
__global__ void k_extract_cuts(const uint32_t *__restrict__ sorted, int64_t N_all, int B,
                               float *cuts_out /*[m][256]*/, int *cnt_out /*[m]*/) {
  int j = blockIdx.x;
  const uint32_t *s = sorted + (int64_t)j * N_all;
  int64_t N;
  {  // lower_bound(s, kMissingKey): every thread runs the same binary search
    int64_t lo = 0, hi = N_all;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (s[mid] < kMissingKey) lo = mid + 1; else hi = mid;
    }
    N = lo;
  }
  __shared__ unsigned long long distinct;
  __shared__ uint32_t vals[256];
  __shared__ int nvals;
  __shared__ int keep[257];
  if (threadIdx.x == 0) { distinct = 0; nvals = 0; }
  __syncthreads();
  if (N == 0) {  // step 5: no observed values -> one cut 0.0
    if (threadIdx.x == 0) { cuts_out[j * 256] = 0.0f; cnt_out[j] = 1; }
    return;
  }
  unsigned long long dl = 0;
  for (int64_t i = threadIdx.x; i < N; i += blockDim.x) dl += (i == 0 || s[i] != s[i - 1]);
  for (int o = 16; o; o >>= 1) dl += __shfl_down_sync(0xffffffffu, dl, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(&distinct, dl);
  __syncthreads();
  if (distinct <= (unsigned long long)B) {
    // step 3: every distinct value is a cut (collected, then ordered by rank)
    for (int64_t i = threadIdx.x; i < N; i += blockDim.x)
      if (i == 0 || s[i] != s[i - 1]) vals[atomicAdd(&nvals, 1)] = s[i];
    __syncthreads();
    int D = nvals;
    if (threadIdx.x < D) {
      uint32_t v = vals[threadIdx.x];
      int rank = 0;
      for (int u = 0; u < D; ++u) rank += vals[u] < v;
      cuts_out[j * 256 + rank] = key_float(v);
    }
    if (threadIdx.x == 0) cnt_out[j] = D;
  } else {
    // step 4: c_b = v[ceil(b N / B)] (1-based), repeats dropped
    int b = threadIdx.x + 1;
    uint32_t v = 0;
    if (b <= B) {
      int64_t idx = ((int64_t)b * N + B - 1) / B;
      v = s[idx - 1];
      vals[threadIdx.x] = v;
    }
    __syncthreads();
    int k = (b <= B) && (b == 1 || v > vals[threadIdx.x - 1]);
    keep[threadIdx.x] = k;
    __syncthreads();
    if (threadIdx.x == 0) {  // B <= 256: a sequential scan is fine
      int acc = 0;
      for (int t = 0; t < B; ++t) { int kk = keep[t]; keep[t] = acc; acc += kk; }
      keep[256] = acc;
    }
    __syncthreads();
    if (k) cuts_out[j * 256 + keep[threadIdx.x]] = key_float(v);
    if (threadIdx.x == 0) cnt_out[j] = keep[256];
  }
}

// LookupBin + Write (Alg. 4) into the tiled page layout.  Thread per (feature group g,
// row r, quad u): consecutive threads write consecutive 32-bit words of a group plane, so the
// output is fully coalesced (device pages, or pinned host pages written zero-copy over PCIe).
__global__ void k_bin_rows(const float *__restrict__ X, int64_t n, int m, int n_fg, int gw, int stride,
                           int64_t row_local0, int64_t rpp, const float *__restrict__ cuts,
                           const int *__restrict__ ptrs, uint8_t *__restrict__ out, int *err, int rowmajor,
                           int *missing) {
  const int64_t total = (int64_t)n_fg * n * 8;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int u = (int)(t & 7);
    const int64_t gr = t >> 3;
    const int g = (int)(gr / n);
    const int64_t r = gr - (int64_t)g * n;
    uint32_t word = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int j = g * 32 + u * 4 + c;
      if (j >= m) break;
      const float x = X[r * m + j];
      const int lo = __ldg(ptrs + j), hi = __ldg(ptrs + j + 1);
      const int B = hi - lo;
      if (isnan(x)) {  // missing (R27): symbol 255; a feature with 256 bins cannot hold it
        word |= 255u << (8 * c);
        if (B > 255) atomicExch(err, 5);
        if (*missing == 0) atomicExch(missing, 1);
        continue;
      }
      if (isinf(x)) { atomicExch(err, 2); continue; }
      int a = 0, bnd = B;  // lower_bound: smallest b with x <= c_b
      while (a < bnd) {
        const int mid = (a + bnd) >> 1;
        if (x <= __ldg(cuts + lo + mid)) bnd = mid; else a = mid + 1;
      }
      if (a > B - 1) a = B - 1;  // clamp above the last cut (R3)
      word |= (uint32_t)a << (8 * c);
    }
    const size_t off = rowmajor ? (size_t)(row_local0 + r) * stride + g * 32 + u * 4
                                : ell_off(row_local0 + r, g * 32 + u * 4, rpp, gw, stride);
    *reinterpret_cast<uint32_t *>(out + off) = word;
  }
}

// ---------------------------------------------------------------------------------------------
static int64_t sketch_capacity(oocgb_data d) {
  if (d->n_global <= (1 << 20)) return d->n_local;
  double mu = (double)d->n_local * ((double)(1 << 20) / (double)d->n_global);
  return (int64_t)(mu + 8.0 * sqrt(mu) + 1024.0);
}

void sketch_append(oocgb_data d, const float *dX, int64_t row0_global, int64_t n) {
  oocgb_ctx c = d->ctx;
  if (!d->d_sketch) {
    d->sketch_cap = sketch_capacity(d);
    d->d_sketch = (uint32_t *)dmalloc(sizeof(uint32_t) * (size_t)std::max<int64_t>(1, d->sketch_cap) * d->m);
    d->d_sketch_count = (unsigned long long *)dmalloc(sizeof(unsigned long long));
    OOCGB_CK(cudaMemsetAsync(d->d_sketch_count, 0, sizeof(unsigned long long), c->stream));
    d->sketch_all_rows = d->n_global <= (1 << 20);
  }
  if (n <= 0) return;
  int *d_err = (int *)c->d_small;
  OOCGB_CK(cudaMemsetAsync(d_err, 0, sizeof(int), c->stream));
  int blocks = (int)std::min<int64_t>((n + 7) / 8, (int64_t)c->num_sms * 16);
  k_sketch_append<<<blocks, 256, 0, c->stream>>>(dX, n, d->m, row0_global, d->n_global, d->seed,
                                                 d->sketch_all_rows, d->d_sketch, d->sketch_cap,
                                                 d->d_sketch_count, d_err);
  OOCGB_CK(cudaGetLastError());
  int herr = 0;
  OOCGB_CK(cudaMemcpyAsync(&herr, d_err, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  OOCGB_CK(cudaStreamSynchronize(c->stream));
  OOCGB_REQUIRE(herr != 2, OOCGB_ERR_ARG, "quantise: +-inf in X (R4; NaN marks a missing value)");
  OOCGB_REQUIRE(herr != 3, OOCGB_ERR_NOMEM, "quantise: sketch sample exceeded its capacity");
}

// Per-feature sort of column-major keys [m][N] (CUB segmented radix sort).  CUB takes 32-bit
// item counts and segment offsets, so the features go in batches of at most (2^31 - 1) / N
// columns (offsets relative to the batch), which keeps N * m >= 2^31 inputs exact.
static void sort_columns(oocgb_ctx c, const uint32_t *colmajor, uint32_t *sorted, int64_t N, int m) {
  if (N <= 0 || m <= 0) return;
  OOCGB_REQUIRE(N <= 0x7fffffffLL, OOCGB_ERR_ARG, "cuts: sketch sample above 2^31 rows");
  const int fb = (int)std::max<int64_t>(1, std::min<int64_t>(m, 0x7fffffffLL / N));
  std::vector<int> offs(fb + 1);
  for (int j = 0; j <= fb; ++j) offs[j] = (int)(j * N);
  int *d_offs = (int *)dmalloc(sizeof(int) * (fb + 1));
  OOCGB_CK(cudaMemcpyAsync(d_offs, offs.data(), sizeof(int) * (fb + 1), cudaMemcpyHostToDevice, c->stream));
  size_t tmp = 0;
  OOCGB_CK(cub::DeviceSegmentedRadixSort::SortKeys(nullptr, tmp, colmajor, sorted, (int)(N * fb), fb, d_offs,
                                                   d_offs + 1, 0, 32, c->stream));
  void *d_tmp = dmalloc(std::max<size_t>(tmp, 16));
  for (int j0 = 0; j0 < m; j0 += fb) {
    const int nf = std::min(fb, m - j0);
    OOCGB_CK(cub::DeviceSegmentedRadixSort::SortKeys(d_tmp, tmp, colmajor + (size_t)j0 * N, sorted + (size_t)j0 * N,
                                                     (int)(N * nf), nf, d_offs, d_offs + 1, 0, 32, c->stream));
  }
  OOCGB_CK(cudaStreamSynchronize(c->stream));
  dfree(d_tmp);
  dfree(d_offs);
}

void cuts_finalize(oocgb_data d) {
  oocgb_ctx c = d->ctx;
  if (!d->d_sketch) sketch_append(d, nullptr, 0, 0);
  unsigned long long n_local_sample = 0;
  OOCGB_CK(cudaMemcpyAsync(&n_local_sample, d->d_sketch_count, sizeof(n_local_sample),
                           cudaMemcpyDeviceToHost, c->stream));
  OOCGB_CK(cudaStreamSynchronize(c->stream));
  const int m = d->m;
  uint32_t *rowmajor = d->d_sketch;
  int64_t N = (int64_t)n_local_sample;
  uint32_t *gathered = nullptr;
  if (c->coll) {
    // allgather the sketch sample: pad every rank to the max count with
    // 0xFFFFFFFF keys (sort after every finite key) and drop them after sorting.
    unsigned long long *d_cnt = (unsigned long long *)c->d_small;
    OOCGB_CK(cudaMemcpyAsync(d_cnt, &n_local_sample, 8, cudaMemcpyHostToDevice, c->stream));
    allreduce_max_u64(c, d_cnt, 1);
    unsigned long long maxc = 0;
    OOCGB_CK(cudaMemcpyAsync(&maxc, d_cnt, 8, cudaMemcpyDeviceToHost, c->stream));
    long long tot = (long long)n_local_sample;
    long long *d_tot = (long long *)((char *)c->d_small + 64);
    OOCGB_CK(cudaMemcpyAsync(d_tot, &tot, 8, cudaMemcpyHostToDevice, c->stream));
    allreduce_sum_i64(c, d_tot, 1);
    OOCGB_CK(cudaMemcpyAsync(&tot, d_tot, 8, cudaMemcpyDeviceToHost, c->stream));
    OOCGB_CK(cudaStreamSynchronize(c->stream));
    uint32_t *padded = (uint32_t *)dmalloc(sizeof(uint32_t) * (size_t)std::max<unsigned long long>(1, maxc) * m);
    OOCGB_CK(cudaMemsetAsync(padded, 0xFF, sizeof(uint32_t) * (size_t)maxc * m, c->stream));
    OOCGB_CK(cudaMemcpyAsync(padded, rowmajor, sizeof(uint32_t) * (size_t)n_local_sample * m,
                             cudaMemcpyDeviceToDevice, c->stream));
    gathered = (uint32_t *)dmalloc(sizeof(uint32_t) * (size_t)std::max<unsigned long long>(1, maxc) * m * c->world);
    allgather_u32(c, padded, gathered, (size_t)maxc * m);
    OOCGB_CK(cudaStreamSynchronize(c->stream));
    dfree(padded);
    rowmajor = gathered;
    N = (int64_t)maxc * c->world;  // includes padding rows; trimmed per feature below
    d->n_global = d->n_global;     // unchanged
    // padding rows sort last; the true count per feature is `tot`
    int64_t Ntrue = tot;
    uint32_t *colmajor = (uint32_t *)dmalloc(sizeof(uint32_t) * (size_t)std::max<int64_t>(1, N) * m);
    dim3 tb(32, 8), tg((unsigned)((N + 31) / 32), (unsigned)((m + 31) / 32));
    if (N > 0) k_transpose_keys<<<tg, tb, 0, c->stream>>>(rowmajor, N, m, colmajor);
    OOCGB_CK(cudaGetLastError());
    dfree(gathered);
    // sort per feature, then extract with the true count (padding keys sit at the end)
    uint32_t *sorted = (uint32_t *)dmalloc(sizeof(uint32_t) * (size_t)std::max<int64_t>(1, N) * m);
    sort_columns(c, colmajor, sorted, N, m);
    dfree(colmajor);
    // compact each feature's first Ntrue keys into [m][Ntrue]
    uint32_t *trimmed = (uint32_t *)dmalloc(sizeof(uint32_t) * (size_t)std::max<int64_t>(1, Ntrue) * m);
    for (int j = 0; j < m; ++j)
      OOCGB_CK(cudaMemcpyAsync(trimmed + (int64_t)j * Ntrue, sorted + (int64_t)j * N,
                               sizeof(uint32_t) * (size_t)Ntrue, cudaMemcpyDeviceToDevice, c->stream));
    dfree(sorted);
    rowmajor = nullptr;
    N = Ntrue;
    // fall through to extraction with `trimmed` as the sorted column-major keys
    float *d_cuts = (float *)dmalloc(sizeof(float) * (size_t)m * 256);
    int *d_cnt2 = (int *)dmalloc(sizeof(int) * m);
    k_extract_cuts<<<m, 256, 0, c->stream>>>(trimmed, N, d->max_bin, d_cuts, d_cnt2);
    OOCGB_CK(cudaGetLastError());
    std::vector<float> hc((size_t)m * 256);
    std::vector<int> hn(m);
    OOCGB_CK(cudaMemcpyAsync(hc.data(), d_cuts, sizeof(float) * hc.size(), cudaMemcpyDeviceToHost, c->stream));
    OOCGB_CK(cudaMemcpyAsync(hn.data(), d_cnt2, sizeof(int) * m, cudaMemcpyDeviceToHost, c->stream));
    OOCGB_CK(cudaStreamSynchronize(c->stream));
    dfree(trimmed); dfree(d_cuts); dfree(d_cnt2);
    d->h_cut_ptrs.assign(m + 1, 0);
    d->h_cut_values.clear();
    for (int j = 0; j < m; ++j) {
      for (int k = 0; k < hn[j]; ++k) d->h_cut_values.push_back(hc[(size_t)j * 256 + k]);
      d->h_cut_ptrs[j + 1] = (int)d->h_cut_values.size();
    }
  } else {
    uint32_t *colmajor = (uint32_t *)dmalloc(sizeof(uint32_t) * (size_t)std::max<int64_t>(1, N) * m);
    dim3 tb(32, 8), tg((unsigned)((N + 31) / 32), (unsigned)((m + 31) / 32));
    if (N > 0) k_transpose_keys<<<tg, tb, 0, c->stream>>>(rowmajor, N, m, colmajor);
    OOCGB_CK(cudaGetLastError());
    uint32_t *sorted = (uint32_t *)dmalloc(sizeof(uint32_t) * (size_t)std::max<int64_t>(1, N) * m);
    sort_columns(c, colmajor, sorted, N, m);
    dfree(colmajor);
    float *d_cuts = (float *)dmalloc(sizeof(float) * (size_t)m * 256);
    int *d_cnt2 = (int *)dmalloc(sizeof(int) * m);
    k_extract_cuts<<<m, 256, 0, c->stream>>>(sorted, N, d->max_bin, d_cuts, d_cnt2);
    OOCGB_CK(cudaGetLastError());
    std::vector<float> hc((size_t)m * 256);
    std::vector<int> hn(m);
    OOCGB_CK(cudaMemcpyAsync(hc.data(), d_cuts, sizeof(float) * hc.size(), cudaMemcpyDeviceToHost, c->stream));
    OOCGB_CK(cudaMemcpyAsync(hn.data(), d_cnt2, sizeof(int) * m, cudaMemcpyDeviceToHost, c->stream));
    OOCGB_CK(cudaStreamSynchronize(c->stream));
    dfree(sorted); dfree(d_cuts); dfree(d_cnt2);
    d->h_cut_ptrs.assign(m + 1, 0);
    d->h_cut_values.clear();
    for (int j = 0; j < m; ++j) {
      for (int k = 0; k < hn[j]; ++k) d->h_cut_values.push_back(hc[(size_t)j * 256 + k]);
      d->h_cut_ptrs[j + 1] = (int)d->h_cut_values.size();
    }
  }
  dfree(d->d_sketch);
  d->d_sketch = nullptr;
  dfree(d->d_sketch_count);
  d->d_sketch_count = nullptr;
  d->d_cut_values = (float *)dmalloc(sizeof(float) * std::max<size_t>(1, d->h_cut_values.size()));
  d->d_cut_ptrs = (int32_t *)dmalloc(sizeof(int32_t) * (m + 1));
  OOCGB_CK(cudaMemcpyAsync(d->d_cut_values, d->h_cut_values.data(), sizeof(float) * d->h_cut_values.size(),
                           cudaMemcpyHostToDevice, c->stream));
  OOCGB_CK(cudaMemcpyAsync(d->d_cut_ptrs, d->h_cut_ptrs.data(), sizeof(int32_t) * (m + 1),
                           cudaMemcpyHostToDevice, c->stream));
  OOCGB_CK(cudaStreamSynchronize(c->stream));
  d->cuts_ready = true;
}

// CSR rows [r0, r0 + nr) -> dense float32 [nr][m] with NaN (missing, R27) at the absent entries:
// the buffer is pre-filled with 0xFF bytes (a NaN), then one warp per row scatters its entries.
__global__ void k_csr_scatter(const int64_t *__restrict__ indptr, const int32_t *__restrict__ indices,
                              const float *__restrict__ values, int64_t base, int64_t r0, int64_t nr, int m,
                              float *__restrict__ out, int *err) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < nr;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t b = indptr[r0 + r] - base, e = indptr[r0 + r + 1] - base;
    for (int64_t k = b + lane; k < e; k += 32) {
      const int j = indices[k];
      if (j < 0 || j >= m) { atomicExch(err, 6); continue; }
      out[r * m + j] = values[k];
    }
  }
}

void csr_to_dense(oocgb_ctx c, const int64_t *d_indptr, const int32_t *d_indices, const float *d_values,
                  int64_t base, int64_t r0, int64_t nr, int m, float *d_out, int *d_err) {
  if (nr <= 0) return;
  OOCGB_CK(cudaMemsetAsync(d_out, 0xFF, sizeof(float) * (size_t)nr * m, c->stream));
  const int blocks = (int)std::min<int64_t>((nr + 7) / 8, (int64_t)c->num_sms * 16);
  k_csr_scatter<<<blocks, 256, 0, c->stream>>>(d_indptr, d_indices, d_values, base, r0, nr, m, d_out, d_err);
  OOCGB_CK(cudaGetLastError());
}

void bin_rows(oocgb_data d, const float *dX, int64_t n, int64_t row_local0, uint8_t *out_base, int *d_err) {
  oocgb_ctx c = d->ctx;
  if (n <= 0) return;
  const int64_t total = (int64_t)d->n_fg * n * 8;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, (int64_t)c->num_sms * 32);
  k_bin_rows<<<blocks, 256, 0, c->stream>>>(dX, n, d->m, d->n_fg, d->gw, d->stride, row_local0, d->rows_per_page,
                                            d->d_cut_values,
                                            d->d_cut_ptrs, out_base, d_err,
                                            d->placement == OOCGB_PLACE_PINNED_HOST ? 1 : 0, d->d_missing);
  OOCGB_CK(cudaGetLastError());
}

}  // namespace oocgb
