// Microbenchmark: shared-memory integer atomic throughput on sm_100a, plus HBM copy and
// pinned host->device bandwidth.  Decides the histogram kernel design.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atoms_bench atoms_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// mode 0: random addresses in [0, nwords), returned value unused
// mode 1: random addresses, returned value used (carry detection like the histogram)
// mode 2: conflict-free (bank = lane)
// mode 3: all lanes same address
// mode 4: random 8-bit bins, 16 features per thread-row, two atomics per symbol (g lo, h lo)
//         with carry check -> the exact inner loop shape of the histogram kernel
// mode 5: same as 4 but lanes of a warp rotate features so a warp's 32 lanes touch 16 features
__global__ void atoms_kernel(int mode, int iters, int nwords, uint32_t *out) {
  extern __shared__ uint32_t sm[];
  for (int i = threadIdx.x; i < nwords; i += blockDim.x) sm[i] = 0;
  __syncthreads();
  uint32_t lane = threadIdx.x & 31;
  uint32_t seed = hash32(blockIdx.x * 1024 + threadIdx.x);
  uint32_t acc = 0;
  if (mode == 0) {
    for (int it = 0; it < iters; ++it) {
      seed = hash32(seed + it);
      atomicAdd(&sm[seed % nwords], 1u);
    }
  } else if (mode == 1) {
    for (int it = 0; it < iters; ++it) {
      seed = hash32(seed + it);
      uint32_t old = atomicAdd(&sm[seed % nwords], 12345u);
      acc += (old + 12345u < old);
    }
  } else if (mode == 2) {
    for (int it = 0; it < iters; ++it) {
      seed = hash32(seed + it);
      atomicAdd(&sm[((seed & 255) * 32 + lane) % nwords], 1u);
    }
  } else if (mode == 3) {
    for (int it = 0; it < iters; ++it) atomicAdd(&sm[0], 1u);
  } else if (mode == 4 || mode == 5) {
    // 16 features x 256 bins x {g_lo, h_lo} = 32 KB
    for (int it = 0; it < iters / 32; ++it) {
      seed = hash32(seed + it);
      uint32_t s0 = hash32(seed), s1 = hash32(s0), s2 = hash32(s1), s3 = hash32(s2);
      uint32_t w[4] = {s0, s1, s2, s3};
      uint32_t qg = seed & 0xffffff, qh = (seed >> 8) & 0xffffff;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        int f = (mode == 5) ? ((k + lane) & 15) : k;
        uint32_t bin = (w[f >> 2] >> ((f & 3) * 8)) & 255;
        uint32_t a = (f * 256 + bin) * 2;
        uint32_t o1 = atomicAdd(&sm[a], qg);
        uint32_t o2 = atomicAdd(&sm[a + 1], qh);
        acc += (o1 + qg < o1) + (o2 + qh < o2);
      }
    }
  } else if (mode == 6) {
    // SoA variant of mode 4: g_lo plane then h_lo plane (bank = bin % 32 for both)
    for (int it = 0; it < iters / 32; ++it) {
      seed = hash32(seed + it);
      uint32_t s0 = hash32(seed), s1 = hash32(s0), s2 = hash32(s1), s3 = hash32(s2);
      uint32_t w[4] = {s0, s1, s2, s3};
      uint32_t qg = seed & 0xffffff, qh = (seed >> 8) & 0xffffff;
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        uint32_t bin = (w[k >> 2] >> ((k & 3) * 8)) & 255;
        uint32_t a = k * 256 + bin;
        uint32_t o1 = atomicAdd(&sm[a], qg);
        uint32_t o2 = atomicAdd(&sm[4096 + a], qh);
        acc += (o1 + qg < o1) + (o2 + qh < o2);
      }
    }
  }
  __syncthreads();
  if (acc == 0xdeadbeef) out[0] = acc;
  if (threadIdx.x == 0) out[blockIdx.x + 1] = sm[blockIdx.x % nwords];
}

__global__ void copy_kernel(const int4 *__restrict__ a, int4 *__restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, s = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += s) b[i] = a[i];
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("device %s SMs %d smemPerBlockOptin %zu smemPerSM %zu L2 %d MB clock %d kHz mem %zu MB\n",
         p.name, p.multiProcessorCount, p.sharedMemPerBlockOptin, p.sharedMemPerMultiprocessor,
         p.l2CacheSize >> 20, p.clockRate, p.totalGlobalMem >> 20);
  uint32_t *out; CK(cudaMalloc(&out, 1 << 20));
  CK(cudaFuncSetAttribute(atoms_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char *names[] = {"random", "random+ret", "conflict-free", "same-addr", "hist AoS 2x16", "hist AoS rot", "hist SoA 2x16"};
  for (int mode = 0; mode < 7; ++mode) {
    for (int threads : {256, 512, 1024}) {
      int nwords = (mode >= 4) ? 8192 : 8192;
      int iters = 4096;
      int blocks = p.multiProcessorCount * (2048 / threads);
      atoms_kernel<<<blocks, threads, nwords * 4>>>(mode, iters, nwords, out);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      atoms_kernel<<<blocks, threads, nwords * 4>>>(mode, iters, nwords, out);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double atoms = (double)blocks * threads * iters;
      double persm_per_ns = atoms / (ms * 1e6) / p.multiProcessorCount;
      printf("mode %-16s thr %4d: %.3f ms  %.1f G lane-atomics/s  %.2f lane-atomics/ns/SM\n",
             names[mode], threads, ms, atoms / (ms * 1e6), persm_per_ns);
    }
  }
  // HBM copy
  size_t bytes = 4ull << 30;
  int4 *a, *b; CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
  cudaMemset(a, 1, bytes);
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    copy_kernel<<<p.multiProcessorCount * 8, 512>>>(a, b, bytes / 16);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("hbm copy kernel: %.1f GB/s (r+w)\n", 2.0 * bytes / (ms * 1e6));
  }
  // pinned H2D
  size_t hb = 1ull << 30; void *h; CK(cudaMallocHost(&h, hb)); memset(h, 1, hb);
  float best = 1e9;
  for (int r = 0; r < 6; ++r) {
    cudaEventRecord(e0); cudaMemcpyAsync(a, h, hb, cudaMemcpyHostToDevice); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  printf("pinned H2D 1 GiB best: %.1f GB/s\n", hb / (best * 1e6));
  best = 1e9;
  for (int r = 0; r < 6; ++r) {
    cudaEventRecord(e0); cudaMemcpyAsync(h, a, hb, cudaMemcpyDeviceToHost); cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1)); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  printf("pinned D2H 1 GiB best: %.1f GB/s\n", hb / (best * 1e6));
  return 0;
}
