// Sample(g) and Compact (Alg. 7) for sm_100a, plus the fixed-point
// quantisation of the sampled gradient pairs (R12).
//
//  NONE    all rows, p = 1.
//  UNIFORM SGB: Bernoulli(f) with f_q = rint(f 2^32), scale 1 (R11).
//  MVS     Eq. 9: g_hat = sqrt(g^2 + lambda h^2); capped PPS with the exact
//          integer threshold of R9: k* = min{k : D(k) < 0},
//          D(k) = a_{k+1} (F - k 2^32) - 2^32 R_k over the descending g_hat_q.  D is monotone
//          on the distinct values, so instead of a sort we run a radix descent over the value
//          space with per-bucket (count, sum, max) — exactly what multi-GPU needs (the stats
//          are all-reduced).  p = 1 above the threshold, g_hat_q / mu below.
//  Selection u < p with u from Philox(seed, round; global_row, stream 0) (R24); g' = g/p.
//  Fixed point: q = rint(x 2^e), e = quant_bits - k, frexp(max|x|) = (., k) (R12).
#include "internal.cuh"
#include "philox.cuh"
#include "stream.cuh"

#include <algorithm>
#include <cstring>

namespace oocgb {

constexpr int kSelThreads = 256;
constexpr int kSelPerThread = 8;
constexpr int kSelTile = kSelThreads * kSelPerThread;
constexpr int kRadixBuckets = 2048;

__device__ __forceinline__ void atomic_max_abs(unsigned long long *dst, double x) {
  atomicMax(dst, (unsigned long long)__double_as_longlong(fabs(x)));
}

// binary:logistic gradients (Eq. 5; harness helper): double arithmetic, float32 results.
__global__ void k_logistic(const float *__restrict__ margin, const float *__restrict__ y, int64_t n,
                           float *__restrict__ g, float *__restrict__ h) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double p = 1.0 / (1.0 + exp(-(double)margin[i]));
    g[i] = (float)(p - (double)y[i]);
    h[i] = (float)(p * (1.0 - p));
  }
}

// Eq. 9: g_hat = sqrt(g*g + lambda*(h*h)), no contraction (explicit _rn intrinsics).
__global__ void k_ghat(const float *__restrict__ g, const float *__restrict__ h, int64_t n,
                       double lam, double *__restrict__ ghat, unsigned long long *maxbits) {
  double mx = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double gi = (double)g[i], hi = (double)h[i];
    double v = __dsqrt_rn(__dadd_rn(__dmul_rn(gi, gi), __dmul_rn(lam, __dmul_rn(hi, hi))));
    ghat[i] = v;
    mx = fmax(mx, v);
  }
  for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_down_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) atomicMax(maxbits, (unsigned long long)__double_as_longlong(mx));
}

// g_hat_q = rint(g_hat 2^e'), in place (double -> int64).
__global__ void k_ghat_q(long long *__restrict__ buf, int64_t n, double scale) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = __longlong_as_double(buf[i]);
    buf[i] = __double2ll_rn(__dmul_rn(v, scale));
  }
}

// Per-bucket (count, sum, max) of the values in [lo, lo + NB << shift).
__global__ void k_radix_stats(const long long *__restrict__ q, int64_t n, unsigned long long lo,
                              int shift, int nb, unsigned long long *cnt, unsigned long long *sum,
                              unsigned long long *mx) {
  __shared__ unsigned int s_cnt[kRadixBuckets];
  __shared__ unsigned long long s_sum[kRadixBuckets];
  __shared__ unsigned long long s_max[kRadixBuckets];
  for (int b = threadIdx.x; b < nb; b += blockDim.x) { s_cnt[b] = 0; s_sum[b] = 0; s_max[b] = 0; }
  __syncthreads();
  const unsigned long long span = (unsigned long long)nb << shift;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long v = (unsigned long long)q[i];
    if (v < lo || v - lo >= span) continue;
    int b = (int)((v - lo) >> shift);
    atomicAdd(&s_cnt[b], 1u);
    atomicAdd(&s_sum[b], v);
    atomicMax(&s_max[b], v);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    if (s_cnt[b]) {
      atomicAdd(&cnt[b], (unsigned long long)s_cnt[b]);
      atomicAdd(&sum[b], s_sum[b]);
      atomicMax(&mx[b], s_max[b]);
    }
  }
}

// count(q > t), sum(q <= t)
__global__ void k_threshold_totals(const long long *__restrict__ q, int64_t n, long long t,
                                   unsigned long long *out /*[2]*/) {
  unsigned long long c = 0, s = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    long long v = q[i];
    if (v > t) ++c; else s += (unsigned long long)v;
  }
  for (int o = 16; o; o >>= 1) {
    c += __shfl_down_sync(0xffffffffu, c, o);
    s += __shfl_down_sync(0xffffffffu, s, o);
  }
  if ((threadIdx.x & 31) == 0) { atomicAdd(&out[0], c); atomicAdd(&out[1], s); }
}

struct SelParams {
  int mode;          // 1 uniform, 2 mvs, 3 goss (p_uniform = p_rest, t = top threshold)
  double p_uniform;  // f_q 2^-32
  int has_t;         // MVS: threshold exists
  long long t;       // MVS t* = a_{k*+1}
  double mu;
  uint64_t seed, round;
  int64_t row0;
};

__device__ __forceinline__ double sel_prob(const SelParams &P, const long long *q64, int64_t i) {
  if (P.mode == 1) return P.p_uniform;
  if (P.mode == 3) return (P.has_t && q64[i] >= P.t) ? 1.0 : P.p_uniform;
  long long v = q64[i];
  if (v == 0) return 0.0;
  if (!P.has_t) return 1.0;
  if (v > P.t) return 1.0;
  return __ddiv_rn((double)v, P.mu);
}

// pass 1: selection flags (bytes) + per-tile counts
__global__ void k_select_flags(SelParams P, const long long *__restrict__ q64, int64_t n,
                               uint8_t *__restrict__ flags, int *__restrict__ tile_cnt) {
  int64_t base = (int64_t)blockIdx.x * kSelTile;
  int c = 0;
#pragma unroll
  for (int k = 0; k < kSelPerThread; ++k) {
    int64_t i = base + k * kSelThreads + threadIdx.x;
    if (i < n) {
      double p = sel_prob(P, q64, i);
      double u = philox_uniform(P.seed, P.round, (uint64_t)(P.row0 + i), 0);
      uint8_t s = u < p;
      flags[i] = s;
      c += s;
    }
  }
  for (int o = 16; o; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
  __shared__ int ws[kSelThreads / 32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < kSelThreads / 32; ++w) t += ws[w];
    tile_cnt[blockIdx.x] = t;
  }
}

// single-block exclusive scan of n ints -> out (int64 total at *total)
__global__ void k_scan_exclusive(const int *__restrict__ in, int64_t n, long long *__restrict__ out,
                                 long long *total) {
  __shared__ long long part[1024];
  int64_t per = (n + blockDim.x - 1) / blockDim.x;
  int64_t b = threadIdx.x * per, e = min(n, b + per);
  long long s = 0;
  for (int64_t i = b; i < e; ++i) s += in[i];
  part[threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long acc = 0;
    for (int t = 0; t < (int)blockDim.x; ++t) { long long v = part[t]; part[t] = acc; acc += v; }
    *total = acc;
  }
  __syncthreads();
  long long acc = part[threadIdx.x];
  for (int64_t i = b; i < e; ++i) { out[i] = acc; acc += in[i]; }
}

// pass 2: ordered scatter of the selected rows; g' = g/p (MVS) in double; max |g'|, |h'|.
__global__ void k_select_scatter(SelParams P, const long long *__restrict__ q64,
                                 const uint8_t *__restrict__ flags, const long long *__restrict__ tile_off,
                                 const float *__restrict__ g, const float *__restrict__ h, int64_t n,
                                 int32_t *__restrict__ sel_rows, double *__restrict__ gs,
                                 double *__restrict__ hs, unsigned long long *maxbits /*[2]*/) {
  __shared__ int s_flags[kSelTile];
  __shared__ int s_warp[kSelThreads / 32];
  int64_t base = (int64_t)blockIdx.x * kSelTile;
  // each thread owns kSelPerThread consecutive positions
  int local[kSelPerThread];
  int cnt = 0;
#pragma unroll
  for (int k = 0; k < kSelPerThread; ++k) {
    int64_t i = base + threadIdx.x * kSelPerThread + k;
    local[k] = (i < n) ? flags[i] : 0;
    cnt += local[k];
  }
  // block exclusive scan of cnt
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int incl = cnt;
  for (int o = 1; o < 32; o <<= 1) {
    int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) s_warp[w] = incl;
  __syncthreads();
  int woff = 0;
  for (int k = 0; k < w; ++k) woff += s_warp[k];
  long long pos = tile_off[blockIdx.x] + woff + incl - cnt;
  double mg = 0.0, mh = 0.0;
#pragma unroll
  for (int k = 0; k < kSelPerThread; ++k) {
    int64_t i = base + threadIdx.x * kSelPerThread + k;
    if (local[k]) {
      sel_rows[pos] = (int32_t)i;
      double gi = (double)g[i], hi = (double)h[i];
      if (P.mode >= 2) {
        double p = sel_prob(P, q64, i);
        gi = __ddiv_rn(gi, p);
        hi = __ddiv_rn(hi, p);
      }
      gs[pos] = gi;
      hs[pos] = hi;
      mg = fmax(mg, fabs(gi));
      mh = fmax(mh, fabs(hi));
      ++pos;
    }
  }
  (void)s_flags;
  for (int o = 16; o; o >>= 1) {
    mg = fmax(mg, __shfl_down_sync(0xffffffffu, mg, o));
    mh = fmax(mh, __shfl_down_sync(0xffffffffu, mh, o));
  }
  if (lane == 0) { atomic_max_abs(&maxbits[0], mg); atomic_max_abs(&maxbits[1], mh); }
}

// max |g|, |h| over all rows (NONE mode)
__global__ void k_absmax2(const float *__restrict__ g, const float *__restrict__ h, int64_t n,
                          unsigned long long *maxbits) {
  double mg = 0.0, mh = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    mg = fmax(mg, fabs((double)g[i]));
    mh = fmax(mh, fabs((double)h[i]));
  }
  for (int o = 16; o; o >>= 1) {
    mg = fmax(mg, __shfl_down_sync(0xffffffffu, mg, o));
    mh = fmax(mh, __shfl_down_sync(0xffffffffu, mh, o));
  }
  if ((threadIdx.x & 31) == 0) { atomic_max_abs(&maxbits[0], mg); atomic_max_abs(&maxbits[1], mh); }
}

// e = P - k with frexp(max |x|) = (., k); 0 when max = 0 (R12).  Device copy of the host rule.
__device__ __forceinline__ int quant_exponent(unsigned long long maxbits, int P) {
  const double M = __longlong_as_double((long long)maxbits);
  if (!(M > 0.0)) return 0;
  int k;
  frexp(M, &k);
  return P - k;
}

__global__ void k_sstate_init(SampleState *ss, long long n_sel_local, int quant_bits) {
  ss->maxbits[0] = 0;
  ss->maxbits[1] = 0;
  ss->G = 0;
  ss->H = 0;
  ss->n_sel_local = n_sel_local;  // < 0: written later by the selection scan
  ss->n_sel_global = 0;
  ss->quant_bits = quant_bits;
}

__global__ void k_sstate_globalise(SampleState *ss) {
  ss->n_sel_global = ss->n_sel_local;  // summed over ranks by an all-reduce when world > 1
}

// q = rint(x 2^e) (half to even), plus exact int64 sums for the root node; the exponents come
// from the (all-reduced) maxima in the sample state, the row count from the selection scan.
template <typename T>
__global__ void k_quantise(const T *__restrict__ gs, const T *__restrict__ hs, SampleState *ss,
                           int2 *__restrict__ q) {
  const int eg = quant_exponent(ss->maxbits[0], ss->quant_bits);
  const int eh = quant_exponent(ss->maxbits[1], ss->quant_bits);
  if (blockIdx.x == 0 && threadIdx.x == 0) { ss->e_g = eg; ss->e_h = eh; }
  const double sg = ldexp(1.0, eg), sh = ldexp(1.0, eh);
  const int64_t n = ss->n_sel_local;
  long long *sums = &ss->G;
  long long G = 0, H = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int qg = (int)__double2ll_rn(__dmul_rn((double)gs[i], sg));
    int qh = (int)__double2ll_rn(__dmul_rn((double)hs[i], sh));
    q[i] = make_int2(qg, qh);
    G += qg;
    H += qh;
  }
  for (int o = 16; o; o >>= 1) {
    G += __shfl_down_sync(0xffffffffu, G, o);
    H += __shfl_down_sync(0xffffffffu, H, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd((unsigned long long *)&sums[0], (unsigned long long)G);
    atomicAdd((unsigned long long *)&sums[1], (unsigned long long)H);
  }
}

// all-reduce helpers need contiguous arrays: sums (G, H) and counts live next to each other

// Compact (Alg. 7): row-major rows -> the tiled device sampled page.  One warp per row:
// lane l moves 16-B chunk l (features 16l .. 16l + 15 -> plane l / (gw / 16)).  The source is
// either a staged page in HBM (f = 1: src_rows = nullptr, row k of the output is row r0 + k of
// the page) or the pinned host pages read zero-copy over PCIe (f < 1: only the selected rows
// cross the link, 512 contiguous bytes per row).
__global__ void k_rows_to_tiled(const uint8_t *__restrict__ src, int stride, int gw,
                                const int32_t *__restrict__ src_rows, int64_t src_row0, int64_t k0, int64_t k1,
                                int64_t cap, uint8_t *__restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int chunks = stride / 16;
  const int cpp = gw / 16;  // 16-B chunks per plane row
  for (int64_t k = k0 + (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5); k < k1;
       k += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int64_t r = (src_rows ? (int64_t)src_rows[k] : k) - src_row0;
    const uint8_t *srow = src + (size_t)r * stride;
    for (int ch = lane; ch < chunks; ch += 32) {
      const uint4 v = *reinterpret_cast<const uint4 *>(srow + ch * 16);
      *reinterpret_cast<uint4 *>(out + ((size_t)(ch / cpp) * cap + k) * gw + (ch % cpp) * 16) = v;
    }
  }
}

// ---------------------------------------------------------------------------------------------
static int grid_for(oocgb_ctx c, int64_t n, int threads = 256) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, (int64_t)c->num_sms * 8));
}

static int ceil_log2(int64_t n) {
  int k = 0;
  while (((int64_t)1 << k) < n) ++k;
  return k;
}

void logistic_gradients(oocgb_data d, const float *d_margin, const float *d_labels) {
  oocgb_ctx c = d->ctx;
  if (d->n_local > 0)
    k_logistic<<<grid_for(c, d->n_local), 256, 0, c->stream>>>(d_margin, d_labels, d->n_local, d->d_g, d->d_h);
  OOCGB_CK(cudaGetLastError());
}

static void ensure_sample_buffers(oocgb_data d) {
  if (d->sel_cap < d->n_local) {
    dfree(d->d_sel_rows); dfree(d->d_q); dfree(d->d_gs); dfree(d->d_hs); dfree(d->d_tmp64);
    int64_t cap = std::max<int64_t>(1, d->n_local);
    d->d_sel_rows = (int32_t *)dmalloc(sizeof(int32_t) * cap);
    d->d_q = (int2 *)dmalloc(sizeof(int2) * cap);
    d->d_gs = (double *)dmalloc(sizeof(double) * cap);
    d->d_hs = (double *)dmalloc(sizeof(double) * cap);
    d->d_tmp64 = (long long *)dmalloc(sizeof(long long) * cap);
    d->sel_cap = cap;
  }
}

void sample_rows(oocgb_data d, int mode, double ratio, double mvs_lambda, uint64_t seed,
                 uint64_t round, int quant_bits, oocgb_sample_info *info, double goss_b) {
  oocgb_ctx c = d->ctx;
  PhaseTimer timer(c, 3);
  const int64_t n = d->n_local;
  ensure_sample_buffers(d);
  d->has_sample = false;
  oocgb_sample_info si{};
  si.k_star = -1;
  unsigned long long *d_u = (unsigned long long *)c->d_small;  // small scratch
  unsigned long long *h_u = (unsigned long long *)c->h_small;
  const uint64_t f_q = (uint64_t)nearbyint(ratio * 4294967296.0);
  const __int128 two32 = (__int128)1 << 32;
  const __int128 F = (__int128)f_q * (__int128)d->n_global;

  SelParams P{};
  P.seed = seed;
  P.round = round;
  P.row0 = d->row0;
  P.p_uniform = (double)f_q * 0x1.0p-32;
  int eff_mode = mode;

  if (mode == OOCGB_SAMPLE_MVS) {
    // Eq. 9 + global max
    OOCGB_CK(cudaMemsetAsync(d_u, 0, 8, c->stream));
    if (n > 0)
      k_ghat<<<grid_for(c, n), 256, 0, c->stream>>>(d->d_g, d->d_h, n, mvs_lambda,
                                                    (double *)d->d_tmp64, d_u);
    allreduce_max_u64(c, d_u, 1);
    OOCGB_CK(cudaMemcpyAsync(h_u, d_u, 8, cudaMemcpyDeviceToHost, c->stream));
    OOCGB_CK(cudaStreamSynchronize(c->stream));
    double gmax;
    memcpy(&gmax, h_u, 8);
    if (gmax == 0.0) {
      eff_mode = OOCGB_SAMPLE_UNIFORM;  // S:L320 fallback
      si.fallback_uniform = 1;
    } else {
      int kM;
      frexp(gmax, &kM);
      int e = (62 - ceil_log2(d->n_global)) - kM;
      si.e_prime = e;
      if (n > 0) k_ghat_q<<<grid_for(c, n), 256, 0, c->stream>>>(d->d_tmp64, n, ldexp(1.0, e));
      // radix descent over [0, 2^qbits), qbits = bit width of the largest g_hat_q (known from
      // the global max), in passes of <= 11 bits: starting at the top set bit keeps the first
      // pass's buckets spread (no all-in-bucket-0 contention at large n)
      const unsigned long long qmax = (unsigned long long)nearbyint(ldexp(gmax, e));
      const int qbits = qmax ? 64 - __builtin_clzll(qmax) : 1;
      unsigned long long lo = 0, above = 0, below_sum = 0;
      long long below_max = -1, fallback = -1;
      bool have_fb = false, found = false;
      long long tstar = -1;
      unsigned long long *d_stats = d_u + 16;
      unsigned long long *h_stats = h_u + 16;
      for (int bits_left = qbits; bits_left > 0 && !found;) {
        const int wdt = std::min(11, bits_left);
        const int sh = bits_left - wdt;
        bits_left -= wdt;
        int nb = 1 << wdt;
        OOCGB_CK(cudaMemsetAsync(d_stats, 0, sizeof(unsigned long long) * 3 * nb, c->stream));
        if (n > 0)
          k_radix_stats<<<grid_for(c, n), 256, 0, c->stream>>>(d->d_tmp64, n, lo, sh, nb, d_stats,
                                                               d_stats + nb, d_stats + 2 * nb);
        OOCGB_CK(cudaGetLastError());
        allreduce_sum_i64(c, (long long *)d_stats, 2 * (size_t)nb);
        allreduce_max_u64(c, d_stats + 2 * nb, nb);
        OOCGB_CK(cudaMemcpyAsync(h_stats, d_stats, sizeof(unsigned long long) * 3 * nb,
                                 cudaMemcpyDeviceToHost, c->stream));
        OOCGB_CK(cudaStreamSynchronize(c->stream));
        const unsigned long long *cnt = h_stats, *sum = h_stats + nb, *mx = h_stats + 2 * nb;
        // evaluate P at every edge j = 0..nb (edge value lo + j << sh)
        std::vector<unsigned long long> suf_cnt(nb + 1, 0);
        for (int j = nb - 1; j >= 0; --j) suf_cnt[j] = suf_cnt[j + 1] + cnt[j];
        int jstar = -1;
        long long A_at_jstar = -1;
        unsigned long long Rj = below_sum;
        long long Aj = below_max;
        for (int j = 0; j <= nb; ++j) {
          if (j > 0) {
            Rj += sum[j - 1];
            if (cnt[j - 1]) Aj = std::max<long long>(Aj, (long long)mx[j - 1]);
          }
          unsigned long long kj = above + suf_cnt[j];
          bool Pj = false;
          if (Aj >= 0 && Rj > 0) {
            __int128 lhs = (__int128)Aj * (F - (__int128)kj * two32);
            __int128 rhs = two32 * (__int128)Rj;
            Pj = lhs < rhs;
          }
          if (Pj) { jstar = j; A_at_jstar = Aj; }
        }
        if (jstar < 0) {
          if (have_fb) { tstar = fallback; found = true; break; }
          // No edge is true and nothing lies below lo: the bottom edge is degenerate (no
          // A below it), so t* — if it exists — is inside bucket 0.  Descend without a fallback.
          if (sh == 0) { found = true; break; }  // no threshold: every non-zero row gets p = 1
          above += suf_cnt[1];
          continue;
        }
        if (sh == 0 || jstar == nb) { tstar = A_at_jstar; found = true; break; }
        fallback = A_at_jstar;
        have_fb = true;
        for (int j = 0; j < jstar; ++j) {
          below_sum += sum[j];
          if (cnt[j]) below_max = std::max<long long>(below_max, (long long)mx[j]);
        }
        above += suf_cnt[jstar + 1];
        lo += (unsigned long long)jstar << sh;
      }
      if (tstar >= 0) {
        OOCGB_CK(cudaMemsetAsync(d_u, 0, 16, c->stream));
        if (n > 0) k_threshold_totals<<<grid_for(c, n), 256, 0, c->stream>>>(d->d_tmp64, n, tstar, d_u);
        allreduce_sum_i64(c, (long long *)d_u, 2);
        OOCGB_CK(cudaMemcpyAsync(h_u, d_u, 16, cudaMemcpyDeviceToHost, c->stream));
        OOCGB_CK(cudaStreamSynchronize(c->stream));
        unsigned long long kstar = h_u[0], R = h_u[1];
        double mu = ((double)(long long)R * 4294967296.0) / (double)(F - (__int128)kstar * two32);
        P.has_t = 1;
        P.t = tstar;
        P.mu = mu;
        si.k_star = (int64_t)kstar;
        si.mu = mu;
      } else {
        P.has_t = 0;
        si.k_star = -1;
      }
    }
  }
  if (mode == OOCGB_SAMPLE_GOSS) {
    // R25: |g| quantised like g_hat (lambda = 0: sqrt(g^2) = |g| exactly), the k_a-th largest
    // by a radix select over the counts, then Bernoulli(p_rest) for the rest, scale 1/p
    const uint64_t a_q = (uint64_t)nearbyint(ratio * 4294967296.0);
    const uint64_t b_q = (uint64_t)nearbyint(goss_b * 4294967296.0);
    double p_rest = (double)b_q / (double)(4294967296ULL - a_q);
    if (p_rest > 1.0) p_rest = 1.0;
    const long long k_a = (long long)(((unsigned __int128)a_q * (unsigned __int128)d->n_global + (1ULL << 31)) >> 32);
    P.p_uniform = p_rest;
    P.has_t = 0;
    OOCGB_CK(cudaMemsetAsync(d_u, 0, 8, c->stream));
    if (n > 0)
      k_ghat<<<grid_for(c, n), 256, 0, c->stream>>>(d->d_g, d->d_h, n, 0.0, (double *)d->d_tmp64, d_u);
    allreduce_max_u64(c, d_u, 1);
    OOCGB_CK(cudaMemcpyAsync(h_u, d_u, 8, cudaMemcpyDeviceToHost, c->stream));
    OOCGB_CK(cudaStreamSynchronize(c->stream));
    double gmax;
    memcpy(&gmax, h_u, 8);
    int e = 0;
    if (gmax > 0.0) {
      int kM;
      frexp(gmax, &kM);
      e = (62 - ceil_log2(d->n_global)) - kM;
    }
    si.e_prime = e;
    if (n > 0) k_ghat_q<<<grid_for(c, n), 256, 0, c->stream>>>(d->d_tmp64, n, ldexp(1.0, e));
    if (k_a > 0 && gmax > 0.0) {
      // radix select of the k_a-th largest value over [0, 2^qbits), passes of <= 11 bits
      const unsigned long long qmax = (unsigned long long)nearbyint(ldexp(gmax, e));
      const int qbits = qmax ? 64 - __builtin_clzll(qmax) : 1;
      unsigned long long lo = 0, above = 0;
      unsigned long long *d_stats = d_u + 16;
      unsigned long long *h_stats = h_u + 16;
      for (int bits_left = qbits; bits_left > 0;) {
        const int wdt = std::min(11, bits_left);
        const int sh = bits_left - wdt;
        bits_left -= wdt;
        const int nb = 1 << wdt;
        OOCGB_CK(cudaMemsetAsync(d_stats, 0, sizeof(unsigned long long) * 3 * nb, c->stream));
        if (n > 0)
          k_radix_stats<<<grid_for(c, n), 256, 0, c->stream>>>(d->d_tmp64, n, lo, sh, nb, d_stats,
                                                               d_stats + nb, d_stats + 2 * nb);
        OOCGB_CK(cudaGetLastError());
        allreduce_sum_i64(c, (long long *)d_stats, (size_t)nb);
        OOCGB_CK(cudaMemcpyAsync(h_stats, d_stats, sizeof(unsigned long long) * nb, cudaMemcpyDeviceToHost, c->stream));
        OOCGB_CK(cudaStreamSynchronize(c->stream));
        int j = nb - 1;
        for (; j > 0; --j) {
          if (above + h_stats[j] >= (unsigned long long)k_a) break;
          above += h_stats[j];
        }
        lo += (unsigned long long)j << sh;
      }
      if (lo > 0) { P.has_t = 1; P.t = (long long)lo; }
    }
    si.k_star = k_a;
    si.mu = p_rest;
    eff_mode = OOCGB_SAMPLE_GOSS;
  }
  P.mode = eff_mode == OOCGB_SAMPLE_MVS ? 2 : (eff_mode == OOCGB_SAMPLE_GOSS ? 3 : 1);

  if (!d->d_ss) {
    d->d_ss = (SampleState *)dmalloc(sizeof(SampleState));
    OOCGB_CK(cudaMallocHost(&d->h_ss, sizeof(SampleState)));
  }
  SampleState *ss = d->d_ss;
  d->quant_bits = quant_bits;
  bool need_sync = (info != nullptr);
  if (eff_mode == OOCGB_SAMPLE_NONE) {
    d->all_selected = true;
    d->n_sel = n;
    k_sstate_init<<<1, 1, 0, c->stream>>>(ss, n, quant_bits);
    if (n > 0) k_absmax2<<<grid_for(c, n), 256, 0, c->stream>>>(d->d_g, d->d_h, n, ss->maxbits);
  } else {
    d->all_selected = false;
    need_sync = true;  // the host needs n_sel (grids, graph key, compaction)
    k_sstate_init<<<1, 1, 0, c->stream>>>(ss, 0, quant_bits);
    int64_t tiles = (n + kSelTile - 1) / kSelTile;
    uint8_t *flags = reinterpret_cast<uint8_t *>(d->d_q);  // consumed before q is written
    int *tile_cnt = (int *)((char *)c->d_small + (256 << 10));
    long long *tile_off = (long long *)((char *)c->d_small + (512 << 10));
    int *tcnt = tile_cnt;
    long long *toff = tile_off;
    std::vector<void *> tmp_alloc;
    if (tiles > (32 << 10)) {  // large inputs: dedicated tile tables
      tcnt = (int *)dmalloc(sizeof(int) * tiles);
      toff = (long long *)dmalloc(sizeof(long long) * tiles);
      tmp_alloc.push_back(tcnt);
      tmp_alloc.push_back(toff);
    }
    if (n > 0) {
      k_select_flags<<<(unsigned)tiles, kSelThreads, 0, c->stream>>>(P, d->d_tmp64, n, flags, tcnt);
      k_scan_exclusive<<<1, 1024, 0, c->stream>>>(tcnt, tiles, toff, &ss->n_sel_local);
      k_select_scatter<<<(unsigned)tiles, kSelThreads, 0, c->stream>>>(
          P, d->d_tmp64, flags, toff, d->d_g, d->d_h, n, d->d_sel_rows, d->d_gs, d->d_hs, ss->maxbits);
      OOCGB_CK(cudaGetLastError());
    }
    OOCGB_CK(cudaMemcpyAsync(d->h_ss, ss, sizeof(SampleState), cudaMemcpyDeviceToHost, c->stream));
    OOCGB_CK(cudaStreamSynchronize(c->stream));
    for (void *p : tmp_alloc) dfree(p);
    d->n_sel = d->h_ss->n_sel_local;
  }
  allreduce_max_u64(c, ss->maxbits, 2);
  k_sstate_globalise<<<1, 1, 0, c->stream>>>(ss);
  allreduce_sum_i64(c, &ss->n_sel_global, 1);
  const int qgrid = grid_for(c, std::max<int64_t>(1, d->n_sel));
  if (d->all_selected)
    k_quantise<float><<<qgrid, 256, 0, c->stream>>>(d->d_g, d->d_h, ss, d->d_q);
  else
    k_quantise<double><<<qgrid, 256, 0, c->stream>>>(d->d_gs, d->d_hs, ss, d->d_q);
  OOCGB_CK(cudaGetLastError());
  allreduce_sum_i64(c, &ss->G, 2);
  if (need_sync || d->placement == OOCGB_PLACE_PINNED_HOST) {
    OOCGB_CK(cudaMemcpyAsync(d->h_ss, ss, sizeof(SampleState), cudaMemcpyDeviceToHost, c->stream));
    OOCGB_CK(cudaStreamSynchronize(c->stream));
    d->n_sel_global = d->h_ss->n_sel_global;
    d->e_g = d->h_ss->e_g;
    d->e_h = d->h_ss->e_h;
    d->G_root = d->h_ss->G;
    d->H_root = d->h_ss->H;
  }

  // Compact (Alg. 7): pinned pages -> one device page of the selected rows (an f = 1 sample of
  // data in streamed mode skips it: Alg. 6 builds the tree from the pinned pages directly)
  if (d->placement == OOCGB_PLACE_PINNED_HOST && !(d->streamed && d->all_selected)) {
    if (d->sampled_cap < d->n_sel) {
      dfree(d->d_sampled_page);
      d->d_sampled_page = nullptr;
      d->sampled_cap = 0;
      d->d_sampled_page = (uint8_t *)dmalloc((size_t)std::max<int64_t>(1, d->n_sel) * d->stride);  // tiled, cap rows
      d->sampled_cap = std::max<int64_t>(1, d->n_sel);
    }
    if (d->all_selected) {
      // f = 1: every page streams (H2D) and is re-laid out tiled on the device
      for_each_page(d, [&](const uint8_t *page, int64_t r0, int64_t nr) {
        const int blocks = (int)std::min<int64_t>((nr + 7) / 8, (int64_t)c->num_sms * 16);
        k_rows_to_tiled<<<blocks, 256, 0, c->stream>>>(page, d->stride, d->gw, nullptr, r0, r0, r0 + nr,
                                                       d->sampled_cap, d->d_sampled_page);
        OOCGB_CK(cudaGetLastError());
      });
    } else if (d->n_sel > 0) {
      // f < 1: gather only the selected rows, zero-copy from the pinned pages (NEXT #2: the link
      // carries n_sel rows instead of a second full pass)
      PhaseTimer link(c, 5);
      const int blocks = (int)std::min<int64_t>((d->n_sel + 7) / 8, (int64_t)c->num_sms * 32);
      k_rows_to_tiled<<<blocks, 256, 0, c->stream>>>(d->h_pages, d->stride, d->gw, d->d_sel_rows, 0, 0, d->n_sel,
                                                     d->sampled_cap, d->d_sampled_page);
      OOCGB_CK(cudaGetLastError());
    }
  }
  d->has_sample = true;
  if (!info) return;
  si.n_selected_local = d->n_sel;
  si.n_selected_global = d->n_sel_global;
  si.e_g = d->e_g;
  si.e_h = d->e_h;
  if (info) *info = si;
}

}  // namespace oocgb
