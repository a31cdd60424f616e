// Microbenchmark: k_hist (the library's kernel, included from tree.cu) on synthetic levels shaped
// like config 2's tree (oracle tree shapes): the root (1M contiguous rows), one
// large scattered node, and deep levels of many small scattered nodes.  Build variants with
// -DOOCGB_HIST_EXPERIMENT=1 (no atomics), 2 (no partial stores), 4 (no zero fill) to split the
// per-item costs.  Build (from the repo root):
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false -I. \
//        -o hist_levels tools/microbench/hist_levels.cu paper_2005_09148_b200/csrc/{api,quantise,sample}.cu -ldl
#include "../../paper_2005_09148_b200/csrc/tree.cu"

#include <algorithm>
#include <cstdio>
#include <random>
#include <vector>

using namespace oocgb;

// reference: plain streaming read of the whole page (grid-stride 16-B loads)
__global__ void stream_read(const uint4 *__restrict__ p, size_t n, unsigned *out) {
  unsigned acc = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const uint4 v = __ldg(p + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) out[0] = acc;
}
// the k_hist access pattern without any compute: CTA b streams rows of plane fg in 8-KB steps
__global__ void plane_read(const uint8_t *__restrict__ bins, size_t pitch, int rows_per_item, int n_items,
                           int n_fg, unsigned *out) {
  unsigned acc = 0;
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int fg = item % n_fg, c = item / n_fg;
    const uint8_t *base = bins + (size_t)fg * pitch + (threadIdx.x & 1) * 16;
    const int rend = min((c + 1) * rows_per_item, 1 << 20);
    for (int r = c * rows_per_item + (threadIdx.x >> 1); r < rend; r += blockDim.x / 2) {
      const uint4 v = __ldg(reinterpret_cast<const uint4 *>(base + (size_t)r * 32));
      acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main(int argc, char **argv) {
  const int N = 1 << 20, m = 500, n_fg = 16;
  const size_t pad = argc > 1 ? (size_t)atoll(argv[1]) : 0;  // bytes added to the plane pitch
#ifndef MB_GW
#define MB_GW 64  // tiled plane width (the library: 64 once m > 32)
#endif
  const int n_planes = n_fg * 32 / MB_GW;
  const size_t pitch = (size_t)N * MB_GW + pad;
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  const int grid = prop.multiProcessorCount * kHistCtasPerSm;
  const int kmax = 0x7fffffff >> 16;
  uint8_t *bins;
  cudaMalloc(&bins, pitch * n_planes);
  {
    std::vector<uint8_t> h(pitch * n_planes);
    std::mt19937 g(1);
    for (auto &x : h) x = (uint8_t)g();
    cudaMemcpy(bins, h.data(), h.size(), cudaMemcpyHostToDevice);
  }
  int32_t *ridx; int2 *q; Pair *pairs; LevelCtl *ctl; int2 *chunk_rng; int *partial;
  cudaMalloc(&ridx, 4 * N); cudaMalloc(&q, 8 * N); cudaMalloc(&pairs, sizeof(Pair) * 1024);
  cudaMalloc(&ctl, sizeof(LevelCtl)); cudaMalloc(&chunk_rng, 8 * 65536);
  cudaMalloc(&partial, (size_t)65536 * 2 * kFG * kBins * 4 / 4);  // 64k items x 16 KB... sized below
  cudaFree(partial);
  cudaMalloc(&partial, (size_t)8192 * kFG * kBins * 2 * 4);  // up to 8192 items
  cudaMemset(q, 1, 8 * N);
  cudaFuncSetAttribute(k_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, kHistSmem);
  struct Level { const char *name; std::vector<int> counts; bool identity; };
  std::vector<Level> levels = {
      {"root: 1 x 1M contiguous", {N}, true},
      {"level-1 like: 1 x 496k scattered", {496094}, false},
      {"level-2 like: 2 x ~17k", {15625, 19531}, false},
      {"level-5 like: 82k + 27k + 14 small", {82032, 27344, 4583, 1785, 1444, 1400, 1300, 1200, 1100, 1000, 900, 800, 700, 600, 500, 400}, false},
      {"level-7 like: 48 x 350", std::vector<int>(48, 350), false},
      {"level-7 like: 48 x 2000", std::vector<int>(48, 2000), false},
  };
  {
    unsigned *o; cudaMalloc(&o, 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const size_t bytes = (size_t)N * 32 * n_fg;
    for (int g : {148 * 4, 148 * 8, 148 * 16}) {
      float best = 1e30f;
      for (int it = 0; it < 10; ++it) {
        cudaEventRecord(a); stream_read<<<g, 512>>>(reinterpret_cast<const uint4 *>(bins), bytes / 16, o); cudaEventRecord(b);
        cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); best = std::min(best, ms);
      }
      printf("stream_read grid %5d: %.1f us  %.2f TB/s\n", g, best * 1e3, bytes / (best * 1e-3) / 1e12);
    }
    for (int thr : {512, 1024}) {
      if (MB_GW != 32) break;  // the plane_read pattern models 32-B planes
      float best = 1e30f;
      for (int it = 0; it < 10; ++it) {
        cudaEventRecord(a); plane_read<<<grid, thr>>>(bins, pitch, 28340, 592, n_fg, o); cudaEventRecord(b);
        cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); best = std::min(best, ms);
      }
      printf("plane_read (k_hist root pattern, %d thr): %.1f us  %.2f TB/s\n", thr, best * 1e3, bytes / (best * 1e-3) / 1e12);
    }
  }
  std::mt19937_64 rng(7);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (auto &L : levels) {
    // rows: disjoint random subsets, ascending inside each node (as the partition leaves them)
    std::vector<int> perm(N);
    for (int i = 0; i < N; ++i) perm[i] = i;
    if (!L.identity) std::shuffle(perm.begin(), perm.end(), rng);
    std::vector<int32_t> hr;
    std::vector<Pair> hp;
    long long tot = 0;
    int off = 0;
    for (int c : L.counts) {
      std::vector<int> r(perm.begin() + off, perm.begin() + off + c);
      std::sort(r.begin(), r.end());
      Pair P{};
      P.begin = (int)hr.size(); P.count = c; P.parent = 0; P.built = 1; P.derived = 2;
      hr.insert(hr.end(), r.begin(), r.end());
      hp.push_back(P);
      off += c; tot += c;
    }
    const long long cr = hist_chunk_rows(tot, (int)hp.size(), n_fg, grid, kmax);
    std::vector<int> cp;
    for (int p = 0; p < (int)hp.size(); ++p) {
      const int nch = (int)((hp[p].count + cr - 1) / cr);
      hp[p].chunk_base = (int)cp.size(); hp[p].n_chunks = nch;
      hp[p].chunk_rows = (hp[p].count + nch - 1) / nch;
      for (int c = 0; c < nch; ++c) cp.push_back(p);
    }
    // LPT order: chunks sorted by chunk size, largest first (as the plan numbers them)
    std::vector<int> order(hp.size());
    for (int i = 0; i < (int)order.size(); ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return hp[a].chunk_rows > hp[b].chunk_rows; });
    cp.clear();
    for (int p : order) { hp[p].chunk_base = (int)cp.size(); for (int c = 0; c < hp[p].n_chunks; ++c) cp.push_back(p); }
    LevelCtl hc{};
    hc.n_items = (int)cp.size() * n_fg;
    hc.n_pairs = (int)hp.size();
    cudaMemcpy(ridx, hr.data(), 4 * hr.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(pairs, hp.data(), sizeof(Pair) * hp.size(), cudaMemcpyHostToDevice);
    std::vector<int2> rg;  // chunk -> position range (what the plan writes)
    for (size_t k = 0; k < cp.size(); ++k) {
      const Pair &P = hp[cp[k]];
      const int b0 = P.begin + ((int)k - P.chunk_base) * P.chunk_rows;
      rg.push_back(make_int2(b0, std::min(P.begin + P.count, b0 + P.chunk_rows)));
    }
    cudaMemcpy(chunk_rng, rg.data(), 8 * rg.size(), cudaMemcpyHostToDevice);
    float best = 1e30f;
    for (int it = 0; it < 20; ++it) {
      cudaMemcpy(ctl, &hc, sizeof(hc), cudaMemcpyHostToDevice);
      // flush L2 between launches (the real level reads cold data)
      cudaMemset(partial, it, (size_t)8192 * kFG * kBins * 2 * 4 / 2);
      cudaEventRecord(e0);
      k_hist<<<grid, kHistThreads, kHistSmem>>>(bins, pitch, m, n_fg, ridx, q, pairs, ctl, chunk_rng,
                                               partial, L.identity ? 1 : 0, MB_GW, MB_GW == 64 ? 1 : 0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      if (cudaGetLastError() != cudaSuccess) { printf("launch failed: %s\n", L.name); return 1; }
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (it >= 3) best = std::min(best, ms);
    }
    const double sym = (double)tot * m;
    printf("%-40s rows %8lld items %5d chunk %6lld  %8.1f us  %6.2f T symbols/s  %.1f us/item-wave\n", L.name, tot,
           hc.n_items, cr, best * 1e3, sym / (best * 1e-3) / 1e12, best * 1e3 / ((double)hc.n_items / grid));
  }
  printf("err: %s (experiment %d, pitch pad %zu, plane width %d)\n", cudaGetErrorString(cudaGetLastError()),
         OOCGB_HIST_EXPERIMENT, pad, MB_GW);
  return 0;
}
