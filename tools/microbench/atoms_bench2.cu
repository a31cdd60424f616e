// Microbench v2: ATOMS throughput with addresses precomputed in registers (no ALU noise).
// pattern 0: histogram layout [bin][32 features], lane l at step s touches feature (l+s)&31
//            -> bank = feature, conflict-free; 2 planes (g, h); non-returning.
// pattern 1: same but feature = s for all lanes -> random banks (bin-driven).
// pattern 2: pattern 0 with returned values consumed (carry check).
// pattern 3: pattern 0 but with s32 atomics replaced by plain LDS+STS (not atomic, wrong result) as
//            an upper bound of the LSU pipe.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x; }
template <int PAT>
__global__ void k(int iters, uint32_t *out) {
  extern __shared__ uint32_t sm[];
  for (int i = threadIdx.x; i < 2 * 256 * 32; i += blockDim.x) sm[i] = 0;
  __syncthreads();
  uint32_t lane = threadIdx.x & 31;
  uint32_t w[8];
  uint32_t s = hash32(blockIdx.x * 4096 + threadIdx.x);
#pragma unroll
  for (int i = 0; i < 8; ++i) { s = hash32(s); w[i] = s; }
  uint32_t qg = s & 0xffff, qh = (s >> 16) & 0xffff, acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int st = 0; st < 32; ++st) {
      uint32_t bin = (w[st >> 2] >> ((st & 3) * 8)) & 255;
      uint32_t f = (PAT == 1) ? st : ((lane + st) & 31);
      uint32_t a = bin * 32 + f;
      if (PAT == 0 || PAT == 1) { atomicAdd(&sm[a], qg); atomicAdd(&sm[8192 + a], qh); }
      else if (PAT == 2) { uint32_t o1 = atomicAdd(&sm[a], qg), o2 = atomicAdd(&sm[8192 + a], qh);
                           acc += (o1 + qg < o1) | (o2 + qh < o2); }
      else { sm[a] += qg; sm[8192 + a] += qh; }
    }
    w[it & 7] ^= it * 0x9e3779b9u;
  }
  __syncthreads();
  if (acc == 12345) out[0] = acc;
  if (threadIdx.x == 0) out[blockIdx.x + 1] = sm[blockIdx.x & 8191];
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  uint32_t *out; cudaMalloc(&out, 1 << 20);
  cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);cudaFuncSetAttribute(k<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);cudaFuncSetAttribute(k<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const char *nm[] = {"conflict-free rotated", "random-bank", "conflict-free +ret", "plain LDS/STS"};
  for (int pat = 0; pat < 4; ++pat) for (int thr : {256, 512, 1024}) {
    int blocks = p.multiProcessorCount * (2048 / thr) / 1;  // 64 KB smem -> 3 CTAs/SM max anyway
    int iters = 2048;
    auto launch = [&]() {
      if (pat == 0) k<0><<<blocks, thr, 65536>>>(iters, out);
      if (pat == 1) k<1><<<blocks, thr, 65536>>>(iters, out);
      if (pat == 2) k<2><<<blocks, thr, 65536>>>(iters, out);
      if (pat == 3) k<3><<<blocks, thr, 65536>>>(iters, out);
    };
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * thr * iters * 64;
    printf("%-24s thr %4d: %.3f ms %.1f G lane-ops/s = %.2f lane-ops/ns/SM  (symbols/s %.1f G)\n", nm[pat], thr, ms,
           ops / ms / 1e6, ops / ms / 1e6 / p.multiProcessorCount, ops / 2 / ms / 1e6);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
