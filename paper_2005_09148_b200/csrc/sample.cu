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
//          The descent runs entirely on the device (k_mvs_*: no host round trip); GOSS's
//          k-th-largest select reuses its passes (k_goss_decide).
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

__device__ __forceinline__ void atomic_max_abs(unsigned long long *dst, double x) {
  atomicMax(dst, (unsigned long long)__double_as_longlong(fabs(x)));
}
// The same from one thread per block after a block reduction, and only when the value can raise
// the current maximum (a plain read filters the rest: same-address atomics serialise at L2).
__device__ __forceinline__ void atomic_max_bits_filtered(unsigned long long *dst, unsigned long long bits) {
  if (bits > *(volatile unsigned long long *)dst) atomicMax(dst, bits);
}
__device__ __forceinline__ double block_max_d(double v, double *s_w) {
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) s_w[w] = v;
  __syncthreads();
  v = lane < (int)(blockDim.x >> 5) ? s_w[lane] : 0.0;
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  return v;
}

// binary:logistic gradients (Eq. 5; harness helper): double arithmetic, float32 results.
// 4 rows per thread and step (16-B loads and stores), the same per-row arithmetic.
__device__ __forceinline__ void logistic_one(float m, float yv, float &g, float &h) {
  double p = 1.0 / (1.0 + exp(-(double)m));
  g = (float)(p - (double)yv);
  h = (float)(p * (1.0 - p));
}
__global__ void k_logistic(const float *__restrict__ margin, const float *__restrict__ y, int64_t n,
                           float *__restrict__ g, float *__restrict__ h) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
  const int64_t n4 = ((reinterpret_cast<uintptr_t>(margin) | reinterpret_cast<uintptr_t>(y) |
                       reinterpret_cast<uintptr_t>(g) | reinterpret_cast<uintptr_t>(h)) & 15) ? 0 : n >> 2;
  for (int64_t i = tid; i < n4; i += nth) {
    const float4 m = __ldg(reinterpret_cast<const float4 *>(margin) + i);
    const float4 yv = __ldg(reinterpret_cast<const float4 *>(y) + i);
    float4 a, b;
    logistic_one(m.x, yv.x, a.x, b.x);
    logistic_one(m.y, yv.y, a.y, b.y);
    logistic_one(m.z, yv.z, a.z, b.z);
    logistic_one(m.w, yv.w, a.w, b.w);
    reinterpret_cast<float4 *>(g)[i] = a;
    reinterpret_cast<float4 *>(h)[i] = b;
  }
  for (int64_t i = 4 * n4 + tid; i < n; i += nth) logistic_one(margin[i], y[i], g[i], h[i]);
}

// ---------------------------------------------------------------------------------------------
// MVS threshold on the device (R9): the radix descent of the exact integer
// threshold runs as a fixed sequence of kernels on the ctx stream -- no host round trip.
//   k_mvs_ghat_max   max g_hat (all ranks: all-reduce max)
//   k_mvs_init       e', the bit width of the largest g_hat_q, the first pass's buckets
//   k_mvs_pass<1>    g_hat_q = rint(g_hat 2^e') stored + (count, sum, max) per bucket of the
//                    top <= 11 bits (one pass over g, h)
//   k_mvs_decide     D(k) at every bucket edge in exact int128 (the host loop it replaces,
//                    DESIGN.md §5): found / descend into one bucket
//   k_mvs_pass<2+>   statistics of the next <= 11 bits over the values still in range; pass 2 reads
//                    every g_hat_q and compacts the in-range ones, later passes read only those
//   k_mvs_totals     k* = #{q > t*}, R = sum{q <= t*}; k_mvs_finish: mu (R9)
// Per-bucket counts use native 32-bit shared atomics; the 64-bit sums are two 32-bit words with
// an explicit carry (returning ATOMS on the low word); the bucket maximum takes a 64-bit CAS
// only when a value exceeds the current maximum (a plain read filters the rest).
struct MvsDev {
  unsigned long long maxbits;            // max g_hat, double bits (all ranks)
  int e, fallback_uniform, qbits, npass_used;
  unsigned long long lo, above, below_sum;
  long long below_max, fallback, tstar;
  int have_fb, found, bits_left, sh, nb, pass;
  unsigned long long compact_n[2];       // compacted in-range values per ping-pong buffer
  unsigned long long tot[2];             // k_mvs_totals: count(q > t*), sum(q <= t*)
  long long kstar;
  double mu;
  int has_t, pad;
};
constexpr int kMvsBuckets = 2048;
constexpr int kMvsDecideSmem = 3 * (kMvsBuckets + 1) * 8;

__global__ void k_mvs_ghat_max(const float *__restrict__ g, const float *__restrict__ h, int64_t n, double lam,
                               unsigned long long *maxbits) {
  double mx = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double gi = (double)g[i], hi = (double)h[i];
    mx = fmax(mx, __dsqrt_rn(__dadd_rn(__dmul_rn(gi, gi), __dmul_rn(lam, __dmul_rn(hi, hi)))));
  }
  __shared__ double s_w[32];
  mx = block_max_d(mx, s_w);
  if (threadIdx.x == 0) atomic_max_bits_filtered(maxbits, (unsigned long long)__double_as_longlong(mx));
}

__device__ __forceinline__ void mvs_geometry(MvsDev *mv) {
  const int wdt = mv->bits_left < 11 ? mv->bits_left : 11;
  mv->sh = mv->bits_left - wdt;
  mv->bits_left -= wdt;
  mv->nb = 1 << wdt;
}

__global__ void k_mvs_init(MvsDev *mv, int log2n, unsigned long long *stats) {
  const double gmax = __longlong_as_double((long long)mv->maxbits);
  MvsDev m = *mv;
  m.found = 0; m.have_fb = 0; m.lo = 0; m.above = 0; m.below_sum = 0; m.below_max = -1; m.fallback = -1;
  m.tstar = -1; m.pass = 0; m.compact_n[0] = m.compact_n[1] = 0; m.tot[0] = m.tot[1] = 0; m.has_t = 0;
  m.kstar = -1; m.mu = 0.0; m.fallback_uniform = 0; m.e = 0; m.npass_used = 0;
  if (!(gmax > 0.0)) {
    m.fallback_uniform = 1;  // every g_hat is 0 -> uniform sampling
    m.found = 1;
  } else {
    int kM;
    frexp(gmax, &kM);
    m.e = (62 - log2n) - kM;
    const unsigned long long qmax = (unsigned long long)__double2ll_rn(ldexp(gmax, m.e));
    m.qbits = qmax ? 64 - __clzll((long long)qmax) : 1;
    m.bits_left = m.qbits;
    mvs_geometry(&m);
  }
  *mv = m;
  for (int i = threadIdx.x; i < 3 * kMvsBuckets; i += blockDim.x) stats[i] = 0;
}

// statistics of one pass: values v in [lo, lo + nb << sh) -> bucket (v - lo) >> sh
struct MvsSmem {
  unsigned cnt[kMvsBuckets];
  unsigned slo[kMvsBuckets], shi[kMvsBuckets];
  unsigned long long mx[kMvsBuckets];
};
// Warp-aggregated update: lanes whose values fall in the same bucket (__match_any) combine their
// count, sum and maximum with shuffles first, and one leader per bucket issues the shared atomics
// (early rounds put nearly every g_hat in one bucket: p ~ 0.5 gives g_hat ~ 0.559 on every row, a
// 32-way conflict per warp without the aggregation).  A group's sum cannot overflow: every
// g_hat_q <= 2^(62 - ceil_log2 n) and a group holds at most min(32, n) of them.
__device__ __forceinline__ void mvs_add(MvsSmem &S, bool in, int b, unsigned long long v) {
  const unsigned inmask = __ballot_sync(__activemask(), in);
  if (!in) return;
  const unsigned peers = __match_any_sync(inmask, b);
  unsigned long long sum = 0, mx = 0;
  for (unsigned m = peers; m; m &= m - 1) {
    const unsigned long long x = __shfl_sync(peers, v, __ffs(m) - 1);
    sum += x;
    mx = x > mx ? x : mx;
  }
  if ((int)(threadIdx.x & 31) != __ffs(peers) - 1) return;
  atomicAdd(&S.cnt[b], (unsigned)__popc(peers));
  const unsigned vl = (unsigned)sum, vh = (unsigned)(sum >> 32);
  const unsigned old = atomicAdd(&S.slo[b], vl);
  const unsigned carry = (old + vl < old) ? 1u : 0u;
  if (vh + carry) atomicAdd(&S.shi[b], vh + carry);
  if (mx > *(volatile unsigned long long *)&S.mx[b]) atomicMax(&S.mx[b], mx);
}

// PASS == 1: g_hat_q from (g, h) (stored to q64); PASS == 2: every q64, in-range values compacted
// to dst; PASS == 3: the compacted values of the previous pass (src, count compact_n[src_slot])
template <int PASS>
__global__ void __launch_bounds__(256) k_mvs_pass(const float *__restrict__ g, const float *__restrict__ h,
                                                  double lam, long long *__restrict__ q64, int64_t n,
                                                  long long *buf0, long long *buf1, MvsDev *mv,
                                                  unsigned long long *stats) {
  __shared__ MvsSmem S;
  if (mv->found) return;
  const unsigned long long lo = mv->lo;
  const int sh = mv->sh, nb = mv->nb;
  const unsigned long long span = (unsigned long long)nb << sh;
  const int slot = mv->pass & 1;
  long long *dst = slot ? buf1 : buf0;
  const long long *src = slot ? buf0 : buf1;
  int64_t cnt_n = n;
  if (PASS == 3) cnt_n = (int64_t)mv->compact_n[slot ^ 1];
  for (int b = threadIdx.x; b < nb; b += blockDim.x) { S.cnt[b] = 0; S.slo[b] = 0; S.shi[b] = 0; S.mx[b] = 0; }
  __syncthreads();
  const double scale = PASS == 1 ? ldexp(1.0, mv->e) : 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt_n; i += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long v;
    if (PASS == 1) {
      const double gi = (double)g[i], hi = (double)h[i];
      const double gh = __dsqrt_rn(__dadd_rn(__dmul_rn(gi, gi), __dmul_rn(lam, __dmul_rn(hi, hi))));
      const long long q = __double2ll_rn(__dmul_rn(gh, scale));
      q64[i] = q;
      v = (unsigned long long)q;
    } else {
      v = (unsigned long long)(PASS == 2 ? q64[i] : src[i]);
    }
    const bool in = v >= lo && v - lo < span;
    mvs_add(S, in, in ? (int)((v - lo) >> sh) : -1, v);
    if (PASS >= 2) {  // compaction for the next pass (order irrelevant: statistics only)
      const unsigned m = __ballot_sync(__activemask(), in);
      if (in) {
        const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
        unsigned long long base = 0;
        if (lane == leader) base = atomicAdd(&mv->compact_n[slot], (unsigned long long)__popc(m));
        base = __shfl_sync(m, base, leader);
        dst[base + __popc(m & ((1u << lane) - 1u))] = (long long)v;
      }
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    if (S.cnt[b]) {
      atomicAdd(&stats[b], (unsigned long long)S.cnt[b]);
      atomicAdd(&stats[kMvsBuckets + b], ((unsigned long long)S.shi[b] << 32) | S.slo[b]);
      atomicMax(&stats[2 * kMvsBuckets + b], S.mx[b]);
    }
  }
}

// One descent step (the former host loop, same operation order): D at every edge j = 0..nb,
// j* = the largest j with P_j; then found / descend.  Single block of 1024 threads.
__global__ void __launch_bounds__(1024) k_mvs_decide(MvsDev *mv, unsigned long long *stats, unsigned long long f_q,
                                                      long long n_global) {
  if (mv->found) return;
  extern __shared__ unsigned long long s_dyn[];  // 3 x (kMvsBuckets + 1) words (> 48 KB: dynamic)
  unsigned long long *s_cnt = s_dyn, *s_sum = s_dyn + (kMvsBuckets + 1);
  long long *s_max = reinterpret_cast<long long *>(s_dyn + 2 * (kMvsBuckets + 1));
  __shared__ int s_jstar;
  const int nb = mv->nb;
  const unsigned long long *cnt = stats, *sum = stats + kMvsBuckets, *mx = stats + 2 * kMvsBuckets;
  // suffix counts suf[j] = sum_{b >= j} cnt[b]; prefix sums pre[j] = sum_{b < j} sum[b];
  // prefix maxima A[j] = max over non-empty b < j of mx[b] (-1 if none)
  for (int j = threadIdx.x; j <= nb; j += blockDim.x) {
    s_cnt[j] = j < nb ? cnt[j] : 0;
    s_sum[j] = j > 0 ? sum[j - 1] : 0;
    s_max[j] = (j > 0 && cnt[j - 1]) ? (long long)mx[j - 1] : -1;
  }
  if (threadIdx.x == 0) s_jstar = -1;
  __syncthreads();
  for (int o = 1; o <= nb; o <<= 1) {  // Hillis-Steele scans (suffix for counts)
    unsigned long long c[3], su[3];
    long long m[3];
    int k = 0;
    for (int j = threadIdx.x; j <= nb; j += blockDim.x, ++k) {
      c[k] = (j + o <= nb) ? s_cnt[j + o] : 0;
      su[k] = j >= o ? s_sum[j - o] : 0;
      m[k] = j >= o ? s_max[j - o] : -1;
    }
    __syncthreads();
    k = 0;
    for (int j = threadIdx.x; j <= nb; j += blockDim.x, ++k) {
      s_cnt[j] += c[k];
      s_sum[j] += su[k];
      if (m[k] > s_max[j]) s_max[j] = m[k];
    }
    __syncthreads();
  }
  const __int128 two32 = (__int128)1 << 32;
  const __int128 F = (__int128)f_q * (__int128)n_global;
  for (int j = threadIdx.x; j <= nb; j += blockDim.x) {
    const unsigned long long Rj = mv->below_sum + s_sum[j];
    const long long Aj = s_max[j] > mv->below_max ? s_max[j] : mv->below_max;
    const unsigned long long kj = mv->above + s_cnt[j];
    if (Aj >= 0 && Rj > 0) {
      const __int128 lhs = (__int128)Aj * (F - (__int128)kj * two32);
      const __int128 rhs = two32 * (__int128)Rj;
      if (lhs < rhs) atomicMax(&s_jstar, j);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int jstar = s_jstar;
    const int sh = mv->sh;
    mv->npass_used = mv->pass + 1;
    if (jstar < 0) {
      if (mv->have_fb) { mv->tstar = mv->fallback; mv->found = 1; }
      else if (sh == 0) { mv->found = 1; }                 // no threshold: every non-zero row p = 1
      else { mv->above += nb >= 1 ? s_cnt[1] : 0; }        // descend into bucket 0
    } else {
      const long long A_at = s_max[jstar] > mv->below_max ? s_max[jstar] : mv->below_max;
      if (sh == 0 || jstar == nb) { mv->tstar = A_at; mv->found = 1; }
      else {
        mv->fallback = A_at;
        mv->have_fb = 1;
        mv->below_sum += s_sum[jstar];
        const long long bm = s_max[jstar];
        if (bm > mv->below_max) mv->below_max = bm;
        mv->above += s_cnt[jstar + 1];
        mv->lo += (unsigned long long)jstar << sh;
      }
    }
    if (!mv->found) {
      mv->pass += 1;
      if (mv->bits_left <= 0) mv->found = 1;  // defensive: no bits left (cannot happen for sh > 0)
      else mvs_geometry(mv);
      mv->compact_n[mv->pass & 1] = 0;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 3 * kMvsBuckets; i += blockDim.x) stats[i] = 0;
}

// k* = #{q > t*}, R = sum{q <= t*}
__global__ void k_mvs_totals(const long long *__restrict__ q, int64_t n, MvsDev *mv) {
  if (mv->tstar < 0) return;
  const long long t = mv->tstar;
  unsigned long long c = 0, s = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const long long v = q[i];
    if (v > t) ++c; else s += (unsigned long long)v;
  }
  for (int o = 16; o; o >>= 1) {
    c += __shfl_down_sync(0xffffffffu, c, o);
    s += __shfl_down_sync(0xffffffffu, s, o);
  }
  __shared__ unsigned long long s_c[32], s_s[32];  // block sums: one atomic per block and value
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) { s_c[w] = c; s_s[w] = s; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) { c += s_c[k]; s += s_s[k]; }
    atomicAdd(&mv->tot[0], c);
    atomicAdd(&mv->tot[1], s);
  }
}

__global__ void k_mvs_finish(MvsDev *mv, unsigned long long f_q, long long n_global) {
  if (mv->tstar >= 0) {
    const __int128 two32 = (__int128)1 << 32;
    const __int128 F = (__int128)f_q * (__int128)n_global;
    const unsigned long long kstar = mv->tot[0], R = mv->tot[1];
    mv->kstar = (long long)kstar;
    mv->mu = ((double)(long long)R * 4294967296.0) / (double)(F - (__int128)kstar * two32);
    mv->has_t = 1;
  } else {
    mv->kstar = -1;
    mv->has_t = 0;
  }
}

// GOSS (R25): one step of the radix select of the k_a-th largest value: the largest bucket j whose
// count from the top (above + suffix count) reaches k_a (the host loop it replaces)
__global__ void __launch_bounds__(1024) k_goss_decide(MvsDev *mv, unsigned long long *stats, unsigned long long k_a) {
  if (mv->found) return;
  extern __shared__ unsigned long long s_dyn[];
  unsigned long long *s_cnt = s_dyn;
  __shared__ int s_j;
  const int nb = mv->nb;
  for (int j = threadIdx.x; j <= nb; j += blockDim.x) s_cnt[j] = j < nb ? stats[j] : 0;
  if (threadIdx.x == 0) s_j = 0;
  __syncthreads();
  for (int o = 1; o <= nb; o <<= 1) {  // suffix sums
    unsigned long long c[3];
    int k = 0;
    for (int j = threadIdx.x; j <= nb; j += blockDim.x, ++k) c[k] = (j + o <= nb) ? s_cnt[j + o] : 0;
    __syncthreads();
    k = 0;
    for (int j = threadIdx.x; j <= nb; j += blockDim.x, ++k) s_cnt[j] += c[k];
    __syncthreads();
  }
  for (int j = threadIdx.x + 1; j < nb; j += blockDim.x)
    if (mv->above + s_cnt[j] >= k_a) atomicMax(&s_j, j);
  __syncthreads();
  if (threadIdx.x == 0) {
    const int j = s_j;
    mv->npass_used = mv->pass + 1;
    mv->above += s_cnt[j + 1];
    mv->lo += (unsigned long long)j << mv->sh;
    if (mv->sh == 0 || mv->bits_left <= 0) {
      mv->found = 1;
    } else {
      mv->pass += 1;
      mvs_geometry(mv);
      mv->compact_n[mv->pass & 1] = 0;
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 3 * kMvsBuckets; i += blockDim.x) stats[i] = 0;
}

__global__ void k_goss_finish(MvsDev *mv, long long k_a) {
  mv->tstar = (long long)mv->lo;
  mv->has_t = (k_a > 0 && !mv->fallback_uniform && mv->lo > 0) ? 1 : 0;
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
// MVS (mode 2): the threshold, mu and the all-zero fallback come from the device state
__device__ __forceinline__ SelParams sel_params(const SelParams &P0, const MvsDev *mv) {
  SelParams P = P0;
  if (mv && P.mode == 2) {
    if (mv->fallback_uniform) {
      P.mode = 1;
    } else {
      P.has_t = mv->has_t;
      P.t = mv->tstar;
      P.mu = mv->mu;
    }
  } else if (mv && P.mode == 3) {  // GOSS: the top set threshold (p_rest stays the host's)
    P.has_t = mv->has_t;
    P.t = mv->tstar;
  }
  return P;
}

__global__ void k_select_flags(SelParams P0, const MvsDev *mv, const long long *__restrict__ q64, int64_t n,
                               uint8_t *__restrict__ flags, int *__restrict__ tile_cnt) {
  const SelParams P = sel_params(P0, mv);
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
__global__ void k_select_scatter(SelParams P0, const MvsDev *mv, const long long *__restrict__ q64,
                                 const uint8_t *__restrict__ flags, const long long *__restrict__ tile_off,
                                 const float *__restrict__ g, const float *__restrict__ h, int64_t n,
                                 int32_t *__restrict__ sel_rows, double *__restrict__ gs,
                                 double *__restrict__ hs, unsigned long long *maxbits /*[2]*/) {
  const SelParams P = sel_params(P0, mv);
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
  __shared__ double s_m[32];
  mg = block_max_d(mg, s_m);  // (|g'|, |h'| >= 0)
  mh = block_max_d(mh, s_m);
  if (threadIdx.x == 0) {
    atomic_max_bits_filtered(&maxbits[0], (unsigned long long)__double_as_longlong(mg));
    atomic_max_bits_filtered(&maxbits[1], (unsigned long long)__double_as_longlong(mh));
  }
}

// max |g|, |h| over all rows (NONE mode): 16-B loads (4 rows per thread and step), the maxima
// reduced per block and one 64-bit atomic max per block and value (r01: one per warp, ~9.5k
// same-address atomics serialised at L2).  |x| maxima in float are exact; the bits are those
// of the same value as a double.
__device__ __forceinline__ float block_max_f(float v, float *s_w) {
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) s_w[w] = v;
  __syncthreads();
  v = lane < (int)(blockDim.x >> 5) ? s_w[lane] : 0.0f;
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  __syncthreads();
  return v;
}
// One rank (parts != nullptr): each block writes its (max |g|, max |h|) to parts[2 b .. 2 b + 1]
// (no atomics, so nothing to zero first) and block 0 also initialises the sample state for f = 1
// (k_sstate_init + k_sstate_globalise folded in); k_quantise reduces the parts.
__global__ void __launch_bounds__(256) k_absmax2(const float *__restrict__ g, const float *__restrict__ h, int64_t n,
                                                 unsigned long long *maxbits, float *parts, SampleState *ss,
                                                 int quant_bits) {
  __shared__ float s_w[32];
  float mg = 0.0f, mh = 0.0f;
  const int64_t n4 = n >> 2;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
  const float4 *g4 = reinterpret_cast<const float4 *>(g), *h4 = reinterpret_cast<const float4 *>(h);
  for (int64_t i = tid; i < n4; i += nth) {
    const float4 a = __ldg(g4 + i), b = __ldg(h4 + i);
    mg = fmaxf(mg, fmaxf(fmaxf(fabsf(a.x), fabsf(a.y)), fmaxf(fabsf(a.z), fabsf(a.w))));
    mh = fmaxf(mh, fmaxf(fmaxf(fabsf(b.x), fabsf(b.y)), fmaxf(fabsf(b.z), fabsf(b.w))));
  }
  for (int64_t i = 4 * n4 + tid; i < n; i += nth) {
    mg = fmaxf(mg, fabsf(g[i]));
    mh = fmaxf(mh, fabsf(h[i]));
  }
  mg = block_max_f(mg, s_w);
  mh = block_max_f(mh, s_w);
  if (threadIdx.x == 0) {
    if (parts) {
      parts[2 * blockIdx.x] = mg;
      parts[2 * blockIdx.x + 1] = mh;
      if (blockIdx.x == 0) {
        ss->G = 0;
        ss->H = 0;
        ss->n_sel_local = n;
        ss->n_sel_global = n;
        ss->quant_bits = quant_bits;
      }
    } else {
      atomic_max_abs(&maxbits[0], (double)mg);
      atomic_max_abs(&maxbits[1], (double)mh);
    }
  }
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
// 4 rows per thread and step (16-B loads of float rows, 2 x 16-B stores of q), the sums reduced
// per block with one 64-bit atomic per block and value (r01: one per warp).
__device__ __forceinline__ long long block_sum_ll(long long v, long long *s_w) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) s_w[w] = v;
  __syncthreads();
  v = lane < (int)(blockDim.x >> 5) ? s_w[lane] : 0;
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  return v;
}
template <typename T>
__global__ void __launch_bounds__(256) k_quantise(const T *__restrict__ gs, const T *__restrict__ hs, SampleState *ss,
                                                  int2 *__restrict__ q, const float *__restrict__ parts, int n_parts) {
  __shared__ long long s_w[32];
  __shared__ unsigned long long s_mb[2];
  if (parts) {  // one rank, f = 1: the maxima from k_absmax2's per-block parts
    __shared__ float s_f[32];
    float mg = 0.0f, mh = 0.0f;
    for (int i = threadIdx.x; i < n_parts; i += blockDim.x) {
      mg = fmaxf(mg, parts[2 * i]);
      mh = fmaxf(mh, parts[2 * i + 1]);
    }
    mg = block_max_f(mg, s_f);
    mh = block_max_f(mh, s_f);
    if (threadIdx.x == 0) {
      s_mb[0] = (unsigned long long)__double_as_longlong((double)mg);
      s_mb[1] = (unsigned long long)__double_as_longlong((double)mh);
      if (blockIdx.x == 0) { ss->maxbits[0] = s_mb[0]; ss->maxbits[1] = s_mb[1]; }
    }
  } else if (threadIdx.x == 0) {
    s_mb[0] = ss->maxbits[0];
    s_mb[1] = ss->maxbits[1];
  }
  __syncthreads();
  const int eg = quant_exponent(s_mb[0], ss->quant_bits);
  const int eh = quant_exponent(s_mb[1], ss->quant_bits);
  if (blockIdx.x == 0 && threadIdx.x == 0) { ss->e_g = eg; ss->e_h = eh; }
  const double sg = ldexp(1.0, eg), sh = ldexp(1.0, eh);
  const int64_t n = ss->n_sel_local;
  long long *sums = &ss->G;
  long long G = 0, H = 0;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nth = (int64_t)gridDim.x * blockDim.x;
  auto one = [&](T x, T y) -> int2 {
    const int qg = (int)__double2ll_rn(__dmul_rn((double)x, sg));
    const int qh = (int)__double2ll_rn(__dmul_rn((double)y, sh));
    G += qg;
    H += qh;
    return make_int2(qg, qh);
  };
  int64_t i0 = 0;
  if constexpr (sizeof(T) == 4) {  // float rows: vectorised
    const int64_t n4 = n >> 2;
    const float4 *g4 = reinterpret_cast<const float4 *>(gs), *h4 = reinterpret_cast<const float4 *>(hs);
    int4 *q4 = reinterpret_cast<int4 *>(q);
    for (int64_t i = tid; i < n4; i += nth) {
      const float4 a = __ldg(g4 + i), b = __ldg(h4 + i);
      const int2 r0 = one(a.x, b.x), r1 = one(a.y, b.y), r2 = one(a.z, b.z), r3 = one(a.w, b.w);
      q4[2 * i] = make_int4(r0.x, r0.y, r1.x, r1.y);
      q4[2 * i + 1] = make_int4(r2.x, r2.y, r3.x, r3.y);
    }
    i0 = 4 * n4;
  }
  for (int64_t i = i0 + tid; i < n; i += nth) q[i] = one(gs[i], hs[i]);
  G = block_sum_ll(G, s_w);
  H = block_sum_ll(H, s_w);
  if (threadIdx.x == 0) {
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
static int grid_for(oocgb_ctx c, int64_t n, int threads = 256, int per_sm = 8) {
  return (int)std::max<int64_t>(1, std::min<int64_t>((n + threads - 1) / threads, (int64_t)c->num_sms * per_sm));
}

static int ceil_log2(int64_t n) {
  int k = 0;
  while (((int64_t)1 << k) < n) ++k;
  return k;
}

void logistic_gradients(oocgb_data d, const float *d_margin, const float *d_labels) {
  oocgb_ctx c = d->ctx;
  if (d->n_local > 0)
    k_logistic<<<grid_for(c, (d->n_local + 3) / 4), 256, 0, c->stream>>>(d_margin, d_labels, d->n_local, d->d_g, d->d_h);
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

static MvsDev *mvs_state(oocgb_data d) {
  oocgb_ctx c = d->ctx;
  if (!d->d_mvs) {
    d->d_mvs = dmalloc(sizeof(MvsDev));
    d->d_mvs_stats = (unsigned long long *)dmalloc(sizeof(unsigned long long) * 3 * kMvsBuckets);
    OOCGB_CK(cudaMemsetAsync(d->d_mvs, 0, sizeof(MvsDev), c->stream));  // every field defined
  }
  if (!c->mvs_attr) {  // per ctx (= per device)
    OOCGB_CK(cudaFuncSetAttribute(k_mvs_decide, cudaFuncAttributeMaxDynamicSharedMemorySize, kMvsDecideSmem));
    OOCGB_CK(cudaFuncSetAttribute(k_goss_decide, cudaFuncAttributeMaxDynamicSharedMemorySize, kMvsDecideSmem));
    c->mvs_attr = true;
  }
  return (MvsDev *)d->d_mvs;
}

// the radix passes over g_hat_q (<= ceil((63 - ceil_log2 n) / 11), each followed by `decide`)
template <class Decide>
static void mvs_passes(oocgb_data d, MvsDev *mv, unsigned long long *stats, double lam, int log2n, Decide decide) {
  oocgb_ctx c = d->ctx;
  const int64_t n = d->n_local;
  long long *buf0 = reinterpret_cast<long long *>(d->d_gs), *buf1 = reinterpret_cast<long long *>(d->d_hs);
  const int npass = std::max(1, (63 - log2n + 10) / 11);
  for (int p = 0; p < npass; ++p) {
    if (p == 0)
      k_mvs_pass<1><<<grid_for(c, n), 256, 0, c->stream>>>(d->d_g, d->d_h, lam, d->d_tmp64, n, buf0, buf1, mv, stats);
    else if (p == 1)
      k_mvs_pass<2><<<grid_for(c, n), 256, 0, c->stream>>>(d->d_g, d->d_h, lam, d->d_tmp64, n, buf0, buf1, mv, stats);
    else
      k_mvs_pass<3><<<c->num_sms * 8, 256, 0, c->stream>>>(d->d_g, d->d_h, lam, d->d_tmp64, n, buf0, buf1, mv,
                                                            stats);
    OOCGB_CK(cudaGetLastError());
    decide();
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
  const uint64_t f_q = (uint64_t)nearbyint(ratio * 4294967296.0);
  const __int128 two32 = (__int128)1 << 32;
  const __int128 F = (__int128)f_q * (__int128)d->n_global;

  SelParams P{};
  P.seed = seed;
  P.round = round;
  P.row0 = d->row0;
  P.p_uniform = (double)f_q * 0x1.0p-32;
  int eff_mode = mode;

  const MvsDev *mvp = nullptr;
  if (mode == OOCGB_SAMPLE_MVS) {
    // R9 on the device (no host round trip): max g_hat, then the radix descent of the exact
    // threshold over g_hat_q (<= ceil((63 - ceil_log2 n) / 11) passes), then k*, R, mu
    MvsDev *mv = mvs_state(d);
    unsigned long long *stats = d->d_mvs_stats;
    const int log2n = ceil_log2(d->n_global);
    OOCGB_CK(cudaMemsetAsync(&mv->maxbits, 0, 8, c->stream));
    if (n > 0)
      k_mvs_ghat_max<<<grid_for(c, n), 256, 0, c->stream>>>(d->d_g, d->d_h, n, mvs_lambda, &mv->maxbits);
    allreduce_max_u64(c, &mv->maxbits, 1);
    k_mvs_init<<<1, 256, 0, c->stream>>>(mv, log2n, stats);
    mvs_passes(d, mv, stats, mvs_lambda, log2n, [&]() {
      allreduce_sum_i64(c, (long long *)stats, 2 * (size_t)kMvsBuckets);
      allreduce_max_u64(c, stats + 2 * kMvsBuckets, kMvsBuckets);
      k_mvs_decide<<<1, 1024, kMvsDecideSmem, c->stream>>>(mv, stats, f_q, d->n_global);
    });
    if (n > 0) k_mvs_totals<<<grid_for(c, n), 256, 0, c->stream>>>(d->d_tmp64, n, mv);
    allreduce_sum_i64(c, (long long *)mv->tot, 2);
    k_mvs_finish<<<1, 1, 0, c->stream>>>(mv, f_q, d->n_global);
    OOCGB_CK(cudaGetLastError());
    mvp = mv;
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
    // the k_a-th largest |g|_q by the device radix select (the MVS passes with lambda = 0:
    // sqrt(g^2) = |g| exactly), no host round trip
    MvsDev *mv = mvs_state(d);
    unsigned long long *stats = d->d_mvs_stats;
    const int log2n = ceil_log2(d->n_global);
    OOCGB_CK(cudaMemsetAsync(&mv->maxbits, 0, 8, c->stream));
    if (n > 0) k_mvs_ghat_max<<<grid_for(c, n), 256, 0, c->stream>>>(d->d_g, d->d_h, n, 0.0, &mv->maxbits);
    allreduce_max_u64(c, &mv->maxbits, 1);
    k_mvs_init<<<1, 256, 0, c->stream>>>(mv, log2n, stats);
    if (k_a > 0) mvs_passes(d, mv, stats, 0.0, log2n, [&]() {
      allreduce_sum_i64(c, (long long *)stats, (size_t)kMvsBuckets);
      k_goss_decide<<<1, 1024, kMvsDecideSmem, c->stream>>>(mv, stats, (unsigned long long)k_a);
    });
    k_goss_finish<<<1, 1, 0, c->stream>>>(mv, k_a);
    OOCGB_CK(cudaGetLastError());
    mvp = mv;
    si.k_star = k_a;
    si.mu = p_rest;
    eff_mode = OOCGB_SAMPLE_GOSS;
  }
  P.mode = eff_mode == OOCGB_SAMPLE_MVS ? 2 : (eff_mode == OOCGB_SAMPLE_GOSS ? 3 : 1);

  if (!d->d_ss) {
    d->d_ss = (SampleState *)dmalloc(sizeof(SampleState));
    OOCGB_CK(cudaMemsetAsync(d->d_ss, 0, sizeof(SampleState), c->stream));  // every field defined
    OOCGB_CK(cudaMallocHost(&d->h_ss, sizeof(SampleState)));
  }
  SampleState *ss = d->d_ss;
  d->quant_bits = quant_bits;
  bool need_sync = (info != nullptr);
  // one rank, f = 1, rows present: 2 launches (k_absmax2 with the state init, k_quantise with the
  // maxima reduction) instead of 4
  const bool fuse1 = eff_mode == OOCGB_SAMPLE_NONE && !c->coll && n > 0;
  int abs_parts = 0;
  if (fuse1 && !d->d_absparts) d->d_absparts = (float *)dmalloc(sizeof(float) * 2 * (size_t)c->num_sms * 2);
  if (eff_mode == OOCGB_SAMPLE_NONE) {
    d->all_selected = true;
    d->n_sel = n;
    if (fuse1) {  // one rank: state init folded into k_absmax2, maxima reduced by k_quantise
      abs_parts = grid_for(c, (n + 3) / 4, 256, 2);
      k_absmax2<<<abs_parts, 256, 0, c->stream>>>(d->d_g, d->d_h, n, nullptr, d->d_absparts, ss, quant_bits);
    } else {
      k_sstate_init<<<1, 1, 0, c->stream>>>(ss, n, quant_bits);
      if (n > 0)
        k_absmax2<<<grid_for(c, (n + 3) / 4, 256, 2), 256, 0, c->stream>>>(d->d_g, d->d_h, n, ss->maxbits, nullptr,
                                                                          nullptr, 0);
    }
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
      k_select_flags<<<(unsigned)tiles, kSelThreads, 0, c->stream>>>(P, mvp, d->d_tmp64, n, flags, tcnt);
      k_scan_exclusive<<<1, 1024, 0, c->stream>>>(tcnt, tiles, toff, &ss->n_sel_local);
      k_select_scatter<<<(unsigned)tiles, kSelThreads, 0, c->stream>>>(
          P, mvp, d->d_tmp64, flags, toff, d->d_g, d->d_h, n, d->d_sel_rows, d->d_gs, d->d_hs, ss->maxbits);
      OOCGB_CK(cudaGetLastError());
    }
    OOCGB_CK(cudaMemcpyAsync(d->h_ss, ss, sizeof(SampleState), cudaMemcpyDeviceToHost, c->stream));
    MvsDev *hmv = reinterpret_cast<MvsDev *>((char *)c->h_small + (900 << 10));
    if (mvp) OOCGB_CK(cudaMemcpyAsync(hmv, mvp, sizeof(MvsDev), cudaMemcpyDeviceToHost, c->stream));
    OOCGB_CK(cudaStreamSynchronize(c->stream));
    for (void *p : tmp_alloc) dfree(p);
    d->n_sel = d->h_ss->n_sel_local;
    if (mvp && mode == OOCGB_SAMPLE_MVS) {  // R9 results for the info record
      si.e_prime = hmv->e;
      si.fallback_uniform = hmv->fallback_uniform;
      si.k_star = hmv->has_t ? hmv->kstar : -1;
      si.mu = hmv->has_t ? hmv->mu : 0.0;
    } else if (mvp) {
      si.e_prime = hmv->e;
    }
  }
  if (!fuse1) {
    allreduce_max_u64(c, ss->maxbits, 2);
    k_sstate_globalise<<<1, 1, 0, c->stream>>>(ss);
    allreduce_sum_i64(c, &ss->n_sel_global, 1);
  }
  const int qgrid = grid_for(c, std::max<int64_t>(1, (d->n_sel + 3) / 4), 256, 2);
  if (d->all_selected)
    k_quantise<float><<<qgrid, 256, 0, c->stream>>>(d->d_g, d->d_h, ss, d->d_q, fuse1 ? d->d_absparts : nullptr,
                                                    abs_parts);
  else
    k_quantise<double><<<qgrid, 256, 0, c->stream>>>(d->d_gs, d->d_hs, ss, d->d_q, nullptr, 0);
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
      // tiled, cap rows; 1/8 headroom (the page pitch is part of the build graph's key)
      const int64_t cap = std::max<int64_t>(1, std::min<int64_t>(std::max<int64_t>(d->n_sel, d->n_local),
                                                                 d->n_sel + d->n_sel / 8 + 4096));
      d->d_sampled_page = (uint8_t *)dmalloc((size_t)cap * d->stride);
      d->sampled_cap = cap;
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
