/*
 * oocgb ORACLE — plain, slow, obviously-correct CPU reference for the hot path of
 * "Out-of-Core GPU Gradient Boosting" (arXiv 2005.09148, PAPER.md).
 *
 * THIS IS TEST INFRASTRUCTURE, NOT PRODUCT CODE.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  It shares no code, header,
 * table or constant generator with the CUDA library under paper_2005_09148_b200/; the two
 * meet only through the seeded input generators (synth/) and the tests.
 *
 * Citations: "P:Lx" = PAPER.md line x; "S:Lx" = SPEC.md line x (interface/test ideas only);
 * "Ox" = the reading numbered in DESIGN.md §3 (restated from SURVEY.md §8(c)).
 *
 * Arithmetic discipline: IEEE double, round-to-nearest, compiled with
 * -O2 -ffp-contract=off and no fast-math, so every expression below is evaluated exactly in
 * the written order.  Integer sums are int64 (fixed point, O5); the MVS threshold is int128.
 *
 * Parity status per function (pins live in tests/test_oracle_*.py):
 *   orc_philox4x64_10  pinned: Random123 known answer + numpy.random.Philox
 *   orc_cuts           pinned: SPEC worked examples, np.sort/np.unique re-derivation, rank bound
 *   orc_bins           pinned: SPEC examples, np.searchsorted, brute-force linear scan
 *   orc_sample         pinned: closed forms, Fraction brute force, Monte-Carlo
 *                      unbiasedness, sum p = f n, monotone inclusion
 *   orc_sample_goss    pinned: SPEC S:L313 example, top-set = np.argsort definition, Monte-Carlo
 *                      unbiasedness, scale (1-a)/b
 *   orc_quantise       pinned: closed-form round trip, |q| <= 2^P, exact dequantisation
 *   orc_histogram      pinned: brute-force masks, conservation, additivity
 *   orc_build_tree     pinned: exhaustive greedy enumeration from raw rows (n <= 256),
 *                      Eq.6/Eq.8 closed forms, separable-feature tree, depth-0 leaf
 *   orc_predict        pinned: raw-value traversal == binned traversal, partition leaf map
 *   orc_logistic_grad  pinned: S:L486 closed form and finite differences
 *
 * Missing values (R27): NaN (dense input) = missing.  The cuts
 * skip missing values, a missing value's symbol is 255 (data with missing values has at most
 * 255 bins per feature), and every split candidate is tried with the missing rows on either side
 * (the learned "default direction"); ties keep the lower bin, then missing-right.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef __int128 i128;

/* ------------------------------------------------------------------------------------------
 * O3. Counter-based RNG: Philox4x64-10 (Salmon et al. 2011).  key = (seed, round),
 * counter = (global_row, stream, 0, 0).  u = (out[0] >> 11) * 2^-53 in [0, 1).
 * Streams: 0 = sampling (Alg. 7), 1 = sketch row sample (O1), 2 = data generator.
 * ---------------------------------------------------------------------------------------- */
static void mulhilo64(uint64_t a, uint64_t b, uint64_t *hi, uint64_t *lo) {
  unsigned __int128 p = (unsigned __int128)a * (unsigned __int128)b;
  *hi = (uint64_t)(p >> 64);
  *lo = (uint64_t)p;
}

void orc_philox4x64_10(const uint64_t ctr_in[4], const uint64_t key_in[2], uint64_t out[4]) {
  uint64_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint64_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; ++r) {
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo64(0xD2E7470EE14C6C93ULL, c0, &hi0, &lo0);
    mulhilo64(0xCA5A826395121157ULL, c2, &hi1, &lo1);
    uint64_t n0 = hi1 ^ c1 ^ k0;
    uint64_t n1 = lo1;
    uint64_t n2 = hi0 ^ c3 ^ k1;
    uint64_t n3 = lo0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B97F4A7C15ULL;
    k1 += 0xBB67AE8584CAA73BULL;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

double orc_uniform(uint64_t seed, uint64_t round, uint64_t row, uint64_t stream) {
  uint64_t ctr[4] = {row, stream, 0, 0}, key[2] = {seed, round}, out[4];
  orc_philox4x64_10(ctr, key, out);
  return (double)(out[0] >> 11) * 0x1.0p-53;
}

/* ------------------------------------------------------------------------------------------
 * O1. Cut points: Alg. 2-3 "FindColumnCuts"; "cut points dividing the range of
 * each feature into continuous intervals (i.e. bins) with equal probabilities";
 * max_bin.  Readings 1-2: exact rank cuts on a sorted column of a
 * global-row-keyed sample of <= 2^20 rows (all rows when n_global <= 2^20).
 * ---------------------------------------------------------------------------------------- */
static int cmp_double(const void *a, const void *b) {
  double x = *(const double *)a, y = *(const double *)b;
  return (x < y) ? -1 : (x > y) ? 1 : 0;
}

int orc_sketch_row_selected(int64_t n_global, uint64_t seed, int64_t row) {
  if (n_global <= (1LL << 20)) return 1;
  double p = (double)(1LL << 20) / (double)n_global;
  return orc_uniform(seed, UINT64_MAX, (uint64_t)row, 1) < p;
}

/* X: row-major n x m float32 holding global rows row0 .. row0+n-1 (the whole dataset for the
 * oracle).  Output cut_values capacity m*max_bin, cut_ptrs[m+1].  Returns 0, or 2 on a
 * non-finite value (reading 4). */
int orc_cuts(const float *X, int64_t n, int32_t m, int32_t max_bin, int64_t row0,
             int64_t n_global, uint64_t seed, float *cut_values, int32_t *cut_ptrs) {
  double *col = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
  int32_t out = 0;
  cut_ptrs[0] = 0;
  for (int32_t j = 0; j < m; ++j) {
    /* step 1: the sketch sample (all rows when n_global <= 2^20) */
    int64_t N = 0;
    for (int64_t i = 0; i < n; ++i) {
      if (!orc_sketch_row_selected(n_global, seed, row0 + i)) continue;
      float x = X[i * m + j];
      if (isnan(x)) continue;                  /* missing (R27): not part of the column */
      if (isinf(x)) { free(col); return 2; }   /* reading 4 */
      double v = (double)x;
      if (v == 0.0) v = 0.0; /* canonicalise -0.0 (reading 4) */
      col[N++] = v;
    }
    /* step 2: sort ascending */
    qsort(col, (size_t)N, sizeof(double), cmp_double);
    if (N == 0) { /* step 5: no observed values -> one cut 0.0, never split */
      cut_values[out++] = 0.0f;
      cut_ptrs[j + 1] = out;
      continue;
    }
    int64_t distinct = 1;
    for (int64_t i = 1; i < N; ++i) if (col[i] != col[i - 1]) ++distinct;
    if (distinct <= max_bin) { /* step 3: every distinct value is a cut */
      cut_values[out++] = (float)col[0];
      for (int64_t i = 1; i < N; ++i) if (col[i] != col[i - 1]) cut_values[out++] = (float)col[i];
    } else { /* step 4: c_b = v[ceil(b N / B)] (1-based), b = 1..B, repeats dropped */
      int32_t start = out;
      for (int64_t b = 1; b <= max_bin; ++b) {
        int64_t idx = (b * N + max_bin - 1) / max_bin; /* ceil(b*N/B), 1-based */
        float c = (float)col[idx - 1];
        if (out == start || c > cut_values[out - 1]) cut_values[out++] = c;
      }
    }
    cut_ptrs[j + 1] = out;
  }
  free(col);
  return 0;
}

/* ------------------------------------------------------------------------------------------
 * O2. LookupBin + Write (Alg. 4): bin(i,j) = smallest b with x_ij <= c_{j,b}
 * (right-inclusive, reading 3), clamped to B_j - 1 above the last cut; one byte per
 * (row, feature) in a row-major ELLPACK row of `stride` bytes (reading 5), pad bytes 0.
 * Linear scan on purpose: it is the definition.
 * ---------------------------------------------------------------------------------------- */
int orc_bins(const float *X, int64_t n, int32_t m, const float *cut_values,
             const int32_t *cut_ptrs, int32_t stride, uint8_t *bins) {
  for (int64_t i = 0; i < n; ++i) {
    for (int32_t j = 0; j < stride; ++j) bins[i * stride + j] = 0;
    for (int32_t j = 0; j < m; ++j) {
      float x = X[i * m + j];
      int32_t B = cut_ptrs[j + 1] - cut_ptrs[j];
      if (isnan(x)) {                     /* missing (R27): symbol 255, needs B_j <= 255 */
        if (B > 255) return 2;
        bins[i * stride + j] = 255;
        continue;
      }
      if (isinf(x)) return 2;
      int32_t b = B - 1;
      for (int32_t k = 0; k < B; ++k) {
        if (x <= cut_values[cut_ptrs[j] + k]) { b = k; break; }
      }
      bins[i * stride + j] = (uint8_t)b;
    }
  }
  return 0;
}

/* ------------------------------------------------------------------------------------------
 * O4. Sample(g) (Alg. 7; SGB P:L212-220; MVS Eq. 9).
 * mode 0 NONE: all rows, p = 1.  mode 1 UNIFORM: p = f_q / 2^32, f_q = rint(f 2^32), scale 1
 * (reading 11).  mode 2 MVS: capped probability-proportional-to-size with an exact integer
 * threshold (reading 9), 1/p scaling of g and h.
 * Outputs: selected[i] in {0,1}; p[i]; gs/hs = scaled g', h' (double) for every row (0 when
 * not selected).  info: [0]=n_selected [1]=k_star [2]=mu [3]=e_prime (MVS), as doubles.
 * Returns 0, or 2 on bad arguments.
 * ---------------------------------------------------------------------------------------- */
static int cmp_i64_desc(const void *a, const void *b) {
  int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
  return (x > y) ? -1 : (x < y) ? 1 : 0;
}

static int ceil_log2_i64(int64_t n) {
  int k = 0;
  while (((int64_t)1 << k) < n) ++k;
  return k;
}

int orc_sample(const float *g, const float *h, int64_t n, int32_t mode, double ratio,
               double mvs_lambda, uint64_t seed, uint64_t round, uint8_t *selected, double *p,
               double *gs, double *hs, double *info) {
  if (!(ratio > 0.0 && ratio <= 1.0)) return 2;
  if (mode < 0 || mode > 2) return 2;
  uint64_t f_q = (uint64_t)nearbyint(ratio * 4294967296.0); /* rint(f * 2^32) */
  for (int64_t i = 0; i < n; ++i) p[i] = 0.0;
  info[1] = -1.0; info[2] = 0.0; info[3] = 0.0;
  int fallback_uniform = 0;

  if (mode == 2) {
    /* step 1: g_hat = sqrt(g^2 + lambda h^2), Eq. 9 */
    double *ghat = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double gmax = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      double gi = (double)g[i], hi = (double)h[i];
      double gg = gi * gi;
      double hh = hi * hi;
      double lh = mvs_lambda * hh;
      ghat[i] = sqrt(gg + lh);
      if (ghat[i] > gmax) gmax = ghat[i];
    }
    if (gmax == 0.0) {
      fallback_uniform = 1; /* all g_hat = 0 -> uniform */
    } else {
      /* step 2: ghat_q = rint(ghat 2^e'), e' = (62 - ceil(log2 n)) - k_M */
      int kM;
      frexp(gmax, &kM);
      int e = (62 - ceil_log2_i64(n)) - kM;
      int64_t *q = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
      int64_t *sorted = (int64_t *)malloc(sizeof(int64_t) * (size_t)n);
      for (int64_t i = 0; i < n; ++i) {
        q[i] = (int64_t)nearbyint(ldexp(ghat[i], e));
        sorted[i] = q[i];
      }
      /* step 3: descending order, R_k = sum_{j>k} a_j */
      qsort(sorted, (size_t)n, sizeof(int64_t), cmp_i64_desc);
      int64_t *R = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n + 1));
      R[n] = 0;
      for (int64_t k = n - 1; k >= 0; --k) R[k] = R[k + 1] + sorted[k]; /* R[k] = sum a_{k+1..n} */
      /* steps 4-5: D(k) = a_{k+1} (F - k 2^32) - 2^32 R_k, k* = min{k : D(k) < 0} */
      i128 F = (i128)f_q * (i128)n;
      i128 two32 = (i128)1 << 32;
      int64_t kstar = -1;
      for (int64_t k = 0; k < n; ++k) {
        i128 D = (i128)sorted[k] * (F - (i128)k * two32) - two32 * (i128)R[k];
        if (D < 0) { kstar = k; break; }
      }
      info[3] = (double)e;
      if (kstar < 0) {
        /* no k: every row with g_hat > 0 gets p = 1 */
        for (int64_t i = 0; i < n; ++i) p[i] = (q[i] > 0) ? 1.0 : 0.0;
        info[1] = -1.0;
        info[2] = 0.0;
      } else {
        /* step 6: mu = R_{k*} 2^32 / (F - k* 2^32) */
        double mu = ((double)R[kstar] * 4294967296.0) / (double)(F - (i128)kstar * two32);
        info[1] = (double)kstar;
        info[2] = mu;
        int64_t top = (kstar > 0) ? sorted[kstar - 1] : INT64_MAX;
        /* step 7: top-k* rows p = 1, others p = q/mu, zero rows p = 0 */
        for (int64_t i = 0; i < n; ++i) {
          if (q[i] == 0) p[i] = 0.0;
          else if (kstar > 0 && q[i] >= top) p[i] = 1.0;
          else p[i] = (double)q[i] / mu;
        }
      }
      free(q); free(sorted); free(R);
    }
    free(ghat);
  }
  if (mode == 0) {
    for (int64_t i = 0; i < n; ++i) p[i] = 1.0;
  }
  if (mode == 1 || fallback_uniform) {
    double pu = (double)f_q * 0x1.0p-32;
    for (int64_t i = 0; i < n; ++i) p[i] = pu;
  }
  /* step 8: select iff u_i < p_i; step 9: g' = g / p, h' = h / p (MVS only; SGB scale 1) */
  int64_t ns = 0;
  for (int64_t i = 0; i < n; ++i) {
    int sel;
    if (mode == 0) sel = 1;
    else sel = orc_uniform(seed, round, (uint64_t)i, 0) < p[i];
    selected[i] = (uint8_t)sel;
    if (sel) {
      ++ns;
      if (mode == 2 && !fallback_uniform) {
        gs[i] = (double)g[i] / p[i];
        hs[i] = (double)h[i] / p[i];
      } else {
        gs[i] = (double)g[i];
        hs[i] = (double)h[i];
      }
    } else {
      gs[i] = 0.0;
      hs[i] = 0.0;
    }
  }
  info[0] = (double)ns;
  return 0;
}

/* ------------------------------------------------------------------------------------------
 * O4b. GOSS: "the top a x 100% of training instances with
 * the largest gradients are selected, then from the rest of the data a random sample of
 * b x 100% instances is drawn.  The samples are scaled by (1-a)/b".  Reading R25:
 * |g| is quantised like MVS's g_hat (e' from frexp(max |g|)); k_a = round(a_q n / 2^32) (half
 * up) with a_q = rint(a 2^32); t = the k_a-th largest |g|_q (no top set when k_a = 0, or when t = 0);
 * top rows (|g|_q >= t) have p = 1; every other row is drawn Bernoulli(p_rest) with
 * p_rest = b_q / (2^32 - a_q) (expected b n rows) and scaled g' = g / p_rest, h' = h / p_rest
 * (= (1-a)/b).  info: [0] n_selected, [1] k_a, [2] t (as double), [3] e'.
 * ---------------------------------------------------------------------------------------- */
int orc_sample_goss(const float *g, const float *h, int64_t n, double a, double b, uint64_t seed,
                    uint64_t round, uint8_t *selected, double *p, double *gs, double *hs,
                    double *info) {
  if (!(a >= 0.0 && b > 0.0 && a + b <= 1.0)) return 2;
  uint64_t a_q = (uint64_t)nearbyint(a * 4294967296.0);
  uint64_t b_q = (uint64_t)nearbyint(b * 4294967296.0);
  if (a_q >= 4294967296ULL) return 2;
  double p_rest = (double)b_q / (double)(4294967296ULL - a_q);
  if (p_rest > 1.0) p_rest = 1.0;
  double gmax = 0.0;
  for (int64_t i = 0; i < n; ++i) if (fabs((double)g[i]) > gmax) gmax = fabs((double)g[i]);
  int64_t *q = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  int64_t *sorted = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  int e = 0;
  if (gmax > 0.0) {
    int kM;
    frexp(gmax, &kM);
    e = (62 - ceil_log2_i64(n)) - kM;
  }
  for (int64_t i = 0; i < n; ++i) {
    q[i] = gmax > 0.0 ? (int64_t)nearbyint(ldexp(fabs((double)g[i]), e)) : 0;
    sorted[i] = q[i];
  }
  qsort(sorted, (size_t)n, sizeof(int64_t), cmp_i64_desc);
  int64_t k_a = (int64_t)(((unsigned __int128)a_q * (unsigned __int128)n + (1ULL << 31)) >> 32);
  int64_t t = INT64_MAX;  /* no top set */
  if (k_a > 0 && sorted[k_a - 1] > 0) t = sorted[k_a - 1];
  int64_t ns = 0;
  for (int64_t i = 0; i < n; ++i) {
    int top = q[i] >= t;
    p[i] = top ? 1.0 : p_rest;
    int sel = top || orc_uniform(seed, round, (uint64_t)i, 0) < p_rest;
    selected[i] = (uint8_t)sel;
    gs[i] = sel ? (double)g[i] / p[i] : 0.0;
    hs[i] = sel ? (double)h[i] / p[i] : 0.0;
    ns += sel;
  }
  info[0] = (double)ns;
  info[1] = (double)k_a;
  info[2] = (double)t;
  info[3] = (double)e;
  free(q);
  free(sorted);
  return 0;
}

/* ------------------------------------------------------------------------------------------
 * O5. Fixed point (reading 12; north_star "deterministic fixed-point integer accumulation"):
 * e = P - k where frexp(max |x|) = (mant, k); q = rint(x 2^e), half to even; M = 0 -> e = 0.
 * x: values of the n selected rows (double).  Writes q[n], returns e.
 * ---------------------------------------------------------------------------------------- */
int orc_quantise(const double *x, int64_t n, int32_t P, int64_t *q) {
  double M = 0.0;
  for (int64_t i = 0; i < n; ++i) if (fabs(x[i]) > M) M = fabs(x[i]);
  int e = 0;
  if (M > 0.0) {
    int k;
    frexp(M, &k);
    e = P - k;
  }
  for (int64_t i = 0; i < n; ++i) q[i] = (int64_t)nearbyint(ldexp(x[i], e));
  return e;
}

/* ------------------------------------------------------------------------------------------
 * O6. BuildHistograms (Alg. 1): H[j][b] = (sum q_g, sum q_h) over the listed rows
 * with bin(row, j) = b.  hist layout [m][256][2] int64, zero-filled here.
 * rows[] index into bins / q arrays (local indices of the selected set).
 * ---------------------------------------------------------------------------------------- */
void orc_histogram(const uint8_t *bins, int32_t stride, int32_t m, const int64_t *rows,
                   int64_t n_rows, const int64_t *qg, const int64_t *qh, int64_t *hist) {
  memset(hist, 0, sizeof(int64_t) * (size_t)m * 256 * 2);
  for (int64_t k = 0; k < n_rows; ++k) {
    int64_t r = rows[k];
    for (int32_t j = 0; j < m; ++j) {
      int b = bins[r * stride + j];
      hist[((int64_t)j * 256 + b) * 2 + 0] += qg[r];
      hist[((int64_t)j * 256 + b) * 2 + 1] += qh[r];
    }
  }
}

/* ------------------------------------------------------------------------------------------
 * Tree node as exported (heap order: children of i are 2i+1, 2i+2).  feature = -1 leaf,
 * -2 absent slot (below a leaf).  Same field meaning as the library's oocgb_node, declared
 * independently here.
 * ---------------------------------------------------------------------------------------- */
typedef struct {
  int32_t feature;
  int32_t split_bin;
  float split_value;
  float leaf_value;
  double gain;
  double sum_g;
  double sum_h;
  int64_t n_rows;
  int32_t default_left;  /* R27: rows missing the split feature go left */
  int32_t pad;
} orc_node;

/* O7. EvaluateSplit (Eq. 8) by exhaustive enumeration over (j, b <= B_j - 2),
 * left = bins <= b.  t = (G*G)/(H+lambda); gain = 0.5*((tL + tR) - tP) - gamma.
 * Valid iff hL >= mcw, hR >= mcw and both H + lambda > 0 (R13).  Max gain, ties -> lowest j then lowest b (strict >
 * in ascending scan).  Returns 1 and fills (*bj, *bb, *bgain) when a split with gain > 0
 * exists (reading 13). */
/* R27 (has_missing): every candidate is tried twice, missing rows right (dir 0: the left sums are
 * the prefix) and left (dir 1: prefix + the missing bin 255's sums); scan order (j, b, dir). */
static int orc_best_split(const int64_t *hist, int32_t m, const int32_t *cut_ptrs, int64_t G,
                          int64_t H, int e_g, int e_h, double lambda, double gamma, double mcw,
                          int has_missing, int32_t *bj, int32_t *bb, int32_t *bdir, double *bgain) {
  double gP = ldexp((double)G, -e_g), hP = ldexp((double)H, -e_h);
  double tP = (gP * gP) / (hP + lambda);
  int found = 0;
  double best = 0.0;
  for (int32_t j = 0; j < m; ++j) {
    int32_t B = cut_ptrs[j + 1] - cut_ptrs[j];
    int64_t Gm = has_missing ? hist[((int64_t)j * 256 + 255) * 2 + 0] : 0;
    int64_t Hm = has_missing ? hist[((int64_t)j * 256 + 255) * 2 + 1] : 0;
    int64_t GP = 0, HP = 0; /* prefix over the present bins 0..b */
    for (int32_t b = 0; b <= B - 2; ++b) {
      GP += hist[((int64_t)j * 256 + b) * 2 + 0];
      HP += hist[((int64_t)j * 256 + b) * 2 + 1];
      for (int32_t dir = 0; dir <= (has_missing ? 1 : 0); ++dir) {
        int64_t GL = GP + (dir ? Gm : 0), HL = HP + (dir ? Hm : 0);
        int64_t GR = G - GL, HR = H - HL;
        double gl = ldexp((double)GL, -e_g), hl = ldexp((double)HL, -e_h);
        double gr = ldexp((double)GR, -e_g), hr = ldexp((double)HR, -e_h);
        if (!(hl >= mcw && hr >= mcw && hl + lambda > 0.0 && hr + lambda > 0.0)) continue;
        double tL = (gl * gl) / (hl + lambda);
        double tR = (gr * gr) / (hr + lambda);
        double gain = 0.5 * ((tL + tR) - tP) - gamma;
        if (!found || gain > best) {
          found = 1; best = gain; *bj = j; *bb = b; *bdir = dir;
        }
      }
    }
  }
  *bgain = best;
  return found && best > 0.0;
}

/* O10. leaf = (float)(eta * (-G/(H+lambda))), Eq. 6, eta at creation (reading 15). */
static float orc_leaf(int64_t G, int64_t H, int e_g, int e_h, double lambda, double eta) {
  double g = ldexp((double)G, -e_g), h = ldexp((double)H, -e_h);
  double w = -g / (h + lambda);
  return (float)(eta * w);
}

/* O9. Depth-wise growth (Alg. 1, reading 16): each node's decision depends only on its own
 * rows, so the level order computes what Alg. 1's queue computes.  Histograms are built
 * directly for every node (no sibling subtraction, reading 17 is the GPU's business).
 * n_sel selected rows with local index 0..n_sel-1 into bins/qg/qh.
 * Outputs: nodes[2^(D+1)-1]; leaf_of_row[n_sel] = heap index of the final node of each row;
 * hist_out (optional, may be NULL): [2^D - 1 + ... ] per heap node with depth < D, each
 * m*256*2 int64, zero for absent nodes. */
int orc_build_tree(const uint8_t *bins, int32_t stride, int32_t m, const int32_t *cut_ptrs,
                   const float *cut_values, int64_t n_sel, const int64_t *qg, const int64_t *qh,
                   int32_t e_g, int32_t e_h, int32_t max_depth, double lambda, double gamma,
                   double mcw, double eta, int32_t has_missing, orc_node *nodes, int32_t *leaf_of_row,
                   int64_t *hist_out) {
  if (max_depth < 0 || max_depth > 20) return 2;
  int64_t n_nodes = ((int64_t)1 << (max_depth + 1)) - 1;
  int64_t hsz = (int64_t)m * 256 * 2;
  int64_t *hist = (int64_t *)malloc(sizeof(int64_t) * (size_t)hsz);
  /* node row lists, per heap slot */
  int64_t **rows = (int64_t **)calloc((size_t)n_nodes, sizeof(int64_t *));
  int64_t *cnt = (int64_t *)calloc((size_t)n_nodes, sizeof(int64_t));
  for (int64_t v = 0; v < n_nodes; ++v) {
    nodes[v].feature = -2; nodes[v].split_bin = 0; nodes[v].split_value = 0.0f;
    nodes[v].leaf_value = 0.0f; nodes[v].gain = 0.0; nodes[v].sum_g = 0.0;
    nodes[v].sum_h = 0.0; nodes[v].n_rows = 0; nodes[v].default_left = 0; nodes[v].pad = 0;
  }
  rows[0] = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n_sel > 0 ? n_sel : 1));
  for (int64_t i = 0; i < n_sel; ++i) rows[0][i] = i;
  cnt[0] = n_sel;
  nodes[0].feature = -1;
  if (hist_out) memset(hist_out, 0, sizeof(int64_t) * (size_t)hsz * (size_t)(((int64_t)1 << max_depth) - 1));
  for (int32_t d = 0; d <= max_depth; ++d) {
    int64_t first = ((int64_t)1 << d) - 1, last = ((int64_t)1 << (d + 1)) - 1;
    for (int64_t v = first; v < last; ++v) {
      if (nodes[v].feature == -2) continue; /* absent slot */
      int64_t G = 0, H = 0;
      for (int64_t k = 0; k < cnt[v]; ++k) { G += qg[rows[v][k]]; H += qh[rows[v][k]]; }
      double hd = ldexp((double)H, -e_h);
      if (!(hd + lambda > 0.0)) { /* H + lambda <= 0 */
        for (int64_t u = 0; u < n_nodes; ++u) free(rows[u]);
        free(rows); free(cnt); free(hist);
        return 2;
      }
      nodes[v].sum_g = ldexp((double)G, -e_g);
      nodes[v].sum_h = hd;
      nodes[v].n_rows = cnt[v];
      nodes[v].leaf_value = orc_leaf(G, H, e_g, e_h, lambda, eta);
      nodes[v].feature = -1;
      if (d == max_depth) continue; /* depth-D nodes are leaves */
      orc_histogram(bins, stride, m, rows[v], cnt[v], qg, qh, hist);
      if (hist_out) memcpy(hist_out + v * hsz, hist, sizeof(int64_t) * (size_t)hsz);
      int32_t bj = -1, bb = -1, bdir = 0;
      double bgain = 0.0;
      if (!orc_best_split(hist, m, cut_ptrs, G, H, e_g, e_h, lambda, gamma, mcw, has_missing, &bj, &bb,
                          &bdir, &bgain))
        continue;
      nodes[v].feature = bj;
      nodes[v].split_bin = bb;
      nodes[v].split_value = cut_values[cut_ptrs[bj] + bb];
      nodes[v].gain = bgain;
      nodes[v].default_left = bdir;
      /* O8. RepartitionInstances (Alg. 1): stable, bin <= b goes left; a missing
       * value (symbol 255, R27) goes the default direction */
      int64_t L = 2 * v + 1, R = 2 * v + 2;
      rows[L] = (int64_t *)malloc(sizeof(int64_t) * (size_t)(cnt[v] > 0 ? cnt[v] : 1));
      rows[R] = (int64_t *)malloc(sizeof(int64_t) * (size_t)(cnt[v] > 0 ? cnt[v] : 1));
      for (int64_t k = 0; k < cnt[v]; ++k) {
        int64_t r = rows[v][k];
        int b = bins[r * stride + bj];
        int left = has_missing && b == 255 ? bdir : (b <= bb);
        if (left) rows[L][cnt[L]++] = r;
        else rows[R][cnt[R]++] = r;
      }
      nodes[L].feature = -1;
      nodes[R].feature = -1;
    }
  }
  for (int64_t v = 0; v < n_nodes; ++v) {
    if (nodes[v].feature == -1)
      for (int64_t k = 0; k < cnt[v]; ++k) leaf_of_row[rows[v][k]] = (int32_t)v;
    free(rows[v]);
  }
  free(rows); free(cnt); free(hist);
  return 0;
}

/* O11. Eq. 1: margin_i (float32) += leaf(tree, bins_i); bin <= split_bin -> left;
 * has_missing: symbol 255 (missing, R27) -> the node's default direction. */
void orc_predict(const uint8_t *bins, int32_t stride, int64_t n, const orc_node *nodes,
                 int32_t has_missing, float *margin) {
  for (int64_t i = 0; i < n; ++i) {
    int64_t v = 0;
    while (nodes[v].feature >= 0) {
      int b = bins[i * stride + nodes[v].feature];
      int left = has_missing && b == 255 ? nodes[v].default_left : (b <= nodes[v].split_bin);
      v = left ? 2 * v + 1 : 2 * v + 2;
    }
    margin[i] = margin[i] + nodes[v].leaf_value;
  }
}

/* O12 (harness, Eq. 5 P:L123-128 for binary:logistic): p = 1/(1+exp(-m)); g = p - y;
 * h = p (1 - p); double arithmetic, stored float32. */
void orc_logistic_grad(const float *margin, const float *y, int64_t n, float *g, float *h) {
  for (int64_t i = 0; i < n; ++i) {
    double pr = 1.0 / (1.0 + exp(-(double)margin[i]));
    g[i] = (float)(pr - (double)y[i]);
    h[i] = (float)(pr * (1.0 - pr));
  }
}

/* AUC (O12): rank statistic, ties count 1/2.  O(n^2) on purpose for tiny n; tests pin it to
 * sklearn.metrics.roc_auc_score. */
double orc_auc_bruteforce(const float *score, const float *y, int64_t n) {
  double num = 0.0, pos = 0.0, neg = 0.0;
  for (int64_t i = 0; i < n; ++i) { if (y[i] > 0.5f) pos += 1.0; else neg += 1.0; }
  for (int64_t i = 0; i < n; ++i) {
    if (!(y[i] > 0.5f)) continue;
    for (int64_t k = 0; k < n; ++k) {
      if (y[k] > 0.5f) continue;
      if (score[i] > score[k]) num += 1.0;
      else if (score[i] == score[k]) num += 0.5;
    }
  }
  return num / (pos * neg);
}
