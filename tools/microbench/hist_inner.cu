// Microbenchmark: k_hist's inner loop in isolation (same lane mapping, rotation, PRMT addressing,
// two non-returning shared atomics per symbol, kDepth-deep register pipeline) over an L2-resident
// buffer of random symbols, no items / zeroing / flush.  Prints warp-atomics per clock per SM.
// Variants: V=0 the k_hist loop; V=1 same without the global loads (symbols from registers);
// V=2 loads only (no atomics).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hist_inner hist_inner.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kBins = 256, kFG = 32;

// g at [a + 4S], h-grad at [a + 128 + 4S]: the step index is an immediate
template <int S>
__device__ __forceinline__ void red2(uint32_t t, uint32_t lbase, int x, int y) {
  const uint32_t a = __byte_perm(t, lbase, 0x7604u | ((uint32_t)(S & 3) << 4));
  asm volatile("red.shared.add.s32 [%0+%3], %1;\n\tred.shared.add.s32 [%0+%4], %2;" ::"r"(a), "r"(x), "r"(y),
               "n"(4 * S), "n"(128 + 4 * S));
}

template <int V, int kDepth>
__global__ void __launch_bounds__(V >= 3 ? 1024 : 512, V >= 3 ? 1 : 2) hist_inner(const uint8_t *__restrict__ bins, int n_rows, const int2 *__restrict__ q,
                                                      int iters, int *out) {
  extern __shared__ int4 smem4[];
  const int lane = threadIdx.x & 31;
  const int half = lane & 1, rslot = lane >> 1;
  const int wq = rslot >> 2, bq = (rslot & 3) * 8;
  const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem4);
  uint32_t f4[16];
#pragma unroll
  for (int s = 0; s < 16; ++s) f4[s] = sbase + 4u * (uint32_t)(16 * half + ((rslot + s) & 15));
  // V >= 3: plane h at byte offset h * (64 KB + 64 B); word (bin, slot) at bin * 256 + 4 slot,
  // g at slot r + s, h-grad at slot 32 + r + s; lane base = plane offset + 4 r
  const uint32_t lbase = sbase + (uint32_t)half * (65536u + 64u) + 4u * (uint32_t)rslot;
  const int zwords = V >= 3 ? (2 * 65536 + 128) / 16 : 2 * kBins * kFG / 4;
  for (int i = threadIdx.x; i < zwords; i += blockDim.x) smem4[i] = make_int4(0, 0, 0, 0);
  __syncthreads();
  const int RT = blockDim.x / 2;
  const uint8_t *base = bins + half * 16;
  auto accumulate = [&](const uint4 &x, const int2 qq) {
    uint32_t w[4] = {x.x, x.y, x.z, x.w};
    uint32_t t[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) t[i] = (wq & 1) ? w[(i + 1) & 3] : w[i];
#pragma unroll
    for (int i = 0; i < 4; ++i) w[i] = (wq & 2) ? t[(i + 2) & 3] : t[i];
#pragma unroll
    for (int i = 0; i < 4; ++i) t[i] = __funnelshift_r(w[i], w[(i + 1) & 3], bq);
    if (V >= 3) {
      // one PRMT: bytes 0, 2, 3 from the lane base, byte 1 = the symbol (= bin * 256)
      red2<0>(t[0], lbase, qq.x, qq.y); red2<1>(t[0], lbase, qq.x, qq.y);
      red2<2>(t[0], lbase, qq.x, qq.y); red2<3>(t[0], lbase, qq.x, qq.y);
      red2<4>(t[1], lbase, qq.x, qq.y); red2<5>(t[1], lbase, qq.x, qq.y);
      red2<6>(t[1], lbase, qq.x, qq.y); red2<7>(t[1], lbase, qq.x, qq.y);
      red2<8>(t[2], lbase, qq.x, qq.y); red2<9>(t[2], lbase, qq.x, qq.y);
      red2<10>(t[2], lbase, qq.x, qq.y); red2<11>(t[2], lbase, qq.x, qq.y);
      red2<12>(t[3], lbase, qq.x, qq.y); red2<13>(t[3], lbase, qq.x, qq.y);
      red2<14>(t[3], lbase, qq.x, qq.y); red2<15>(t[3], lbase, qq.x, qq.y);
    } else {
#pragma unroll
    for (int s = 0; s < 16; ++s) {
      const uint32_t a = __byte_perm(t[s >> 2], 0u, 0x4404u | ((uint32_t)(s & 3) << 4)) + f4[s];
      if (V != 2) {
        asm volatile("red.shared.add.s32 [%0], %1;" ::"r"(a), "r"(qq.x));
        asm volatile("red.shared.add.s32 [%0+128], %1;" ::"r"(a), "r"(qq.y));
      }
    }
    }
  };
  uint32_t sink = 0;
  const int rows_per_cta = n_rows / gridDim.x;
  const int r0 = blockIdx.x * rows_per_cta, r1 = r0 + rows_per_cta;
  for (int it = 0; it < iters; ++it) {
    int k = r0 + (threadIdx.x >> 1);
    uint4 xs[kDepth];
    int2 qs[kDepth];
#pragma unroll
    for (int i = 0; i < kDepth; ++i) {
      if (V == 1 || V == 4) { xs[i] = make_uint4(k * 2654435761u, k * 40503u + i, k ^ 0x9e3779b9u, k + i); qs[i] = make_int2(k, i); }
      else { xs[i] = __ldg(reinterpret_cast<const uint4 *>(base + (size_t)(k + i * RT) * 32)); qs[i] = __ldg(q + k + i * RT); }
    }
    while (k < r1) {
#pragma unroll
      for (int i = 0; i < kDepth; ++i) {
        const int kk = k + i * RT;
        if (kk < r1) {
          accumulate(xs[i], qs[i]);
          if (V == 2) sink += xs[i].x ^ xs[i].w ^ qs[i].x;
          const int nk = kk + kDepth * RT;
          if (nk < r1) {
            if (V == 1 || V == 4) { xs[i].x = xs[i].x * 1664525u + 1013904223u; xs[i].y ^= xs[i].x; xs[i].z += xs[i].y; xs[i].w ^= xs[i].z; }
            else { xs[i] = __ldg(reinterpret_cast<const uint4 *>(base + (size_t)nk * 32)); qs[i] = __ldg(q + nk); }
          }
        }
      }
      k += kDepth * RT;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = reinterpret_cast<int *>(smem4)[blockIdx.x & 8191] + (int)sink;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  const int n_rows = 1 << 19;  // 512k rows x 32 B = 16 MB (L2-resident)
  uint8_t *bins;
  int2 *q;
  int *out;
  cudaMalloc(&bins, (size_t)n_rows * 32 + 64);
  cudaMalloc(&q, (size_t)n_rows * 8 + 64);
  cudaMalloc(&out, 1 << 20);
  {
    uint8_t *h = new uint8_t[(size_t)n_rows * 32];
    uint32_t s = 12345;
    for (size_t i = 0; i < (size_t)n_rows * 32; ++i) { s = s * 1664525u + 1013904223u; h[i] = s >> 24; }
    cudaMemcpy(bins, h, (size_t)n_rows * 32, cudaMemcpyHostToDevice);
    delete[] h;
  }
  cudaMemset(q, 1, (size_t)n_rows * 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](auto kern, const char *name, int big = 0) {
    const int smem = big ? 2 * 65536 + 128 : 2 * kBins * kFG * 4;
    const int thr = big ? 1024 : 512, per_sm = big ? 1 : 2;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int grid = p.multiProcessorCount * per_sm, iters = 200;
    kern<<<grid, thr, smem>>>(bins, n_rows, q, 2, out);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    kern<<<grid, thr, smem>>>(bins, n_rows, q, iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double symbols = (double)n_rows * 32 * iters;
    const double watoms = symbols * 2 / 32;
    printf("%-34s %.3f ms  %.2f T symbols/s  %.3f warp-atomics/clk/SM (at %d MHz)\n", name, ms, symbols / ms / 1e9,
           watoms / (ms * 1e-3) / p.multiProcessorCount / (p.clockRate * 1e3), p.clockRate / 1000);
  };
  run(hist_inner<0, 3>, "k_hist loop, depth 3");
  run(hist_inner<0, 5>, "k_hist loop, depth 5");
  run(hist_inner<1, 3>, "no global loads (register symbols)");
  run(hist_inner<2, 3>, "loads only (no atomics)");
  run(hist_inner<3, 3>, "PRMT-only addressing, depth 3", 1);
  run(hist_inner<3, 4>, "PRMT-only addressing, depth 4", 1);
  run(hist_inner<4, 3>, "PRMT-only, no global loads", 1);
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
