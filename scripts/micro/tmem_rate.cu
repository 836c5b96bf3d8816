// Microbenchmark: tcgen05.ld (32x32b.x32) aggregate TMEM read bandwidth per SM vs warp count.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2605_08524_b200/csrc/sm100_ptx.cuh"
using namespace fcpb;
__global__ void tmem_loop(int iters, unsigned long long* cyc, float* out) {
  __shared__ uint32_t tbase;
  if (threadIdx.x < 32) tmem_alloc<512>(&tbase);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tbase;
  const uint32_t w = threadIdx.x >> 5;
  const uint32_t addr = tmem + (((w & 3) * 32) << 16) + (w >> 2) * 32;
  uint32_t acc = 0;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t v[32];
    tmem_ld32(addr + ((i & 3) * 64 & 255), v);
    tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < 32; ++j) acc += v[j];
  }
  unsigned long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}
int main() {
  unsigned long long* cyc; float* out; cudaMalloc(&cyc, 148 * 8); cudaMalloc(&out, 148 * 1024 * 4);
  const int iters = 4096;
  for (int warps : {4, 8, 16, 32}) {
    tmem_loop<<<148, warps * 32>>>(iters, cyc, out); cudaDeviceSynchronize();
    unsigned long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    double bytes = (double)warps * 32 * 32 * 4 * iters;
    printf("warps=%2d  TMEM ld bytes/clk/SM = %.1f  (%s)\n", warps, bytes / h, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
