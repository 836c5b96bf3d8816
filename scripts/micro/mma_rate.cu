// Microbenchmark: tcgen05.mma issue rate per SM for SS / TS operands at M=128, N in {64,128,256}.
// One CTA per SM; an elected thread issues `iters` MMAs of K=16 on resident smem/TMEM data.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2605_08524_b200/csrc/sm100_ptx.cuh"
using namespace fcpb;

template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) mma_loop(int iters, unsigned long long* cycles) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tbase;
  __shared__ uint64_t bar;
  if (threadIdx.x < 32) tmem_alloc<512>(&tbase);
  if (threadIdx.x == 32) { mbar_init(&bar, 1); fence_barrier_init(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tbase;
  if (threadIdx.x < 32) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 65536);
    const uint32_t id = idesc_bf16_f32(128, N, false, false);
    unsigned long long t0 = clock64();
    if (elect_one()) {
      for (int i = 0; i < iters; ++i) {
        const uint32_t off = (i & 3) * 32;
        if (TS) mma_ts(tmem + 256, tmem + (i & 7) * 8, smem_desc_sw128(b + off, 16, 1024), id, 1);
        else mma_ss(tmem + 256, smem_desc_sw128(a + off, 16, 1024), smem_desc_sw128(b + off, 16, 1024), id, 1);
      }
      mma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  }
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

template <int N, bool TS>
void run(const char* name) {
  const int iters = 20000, sms = 148;
  unsigned long long* d; cudaMalloc(&d, sms * 8);
  size_t smem = 160 * 1024;
  cudaFuncSetAttribute(mma_loop<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  mma_loop<N, TS><<<sms, 128, smem>>>(iters, d);
  cudaEvent_t s, e; cudaEventCreate(&s); cudaEventCreate(&e);
  cudaEventRecord(s);
  mma_loop<N, TS><<<sms, 128, smem>>>(iters, d);
  cudaEventRecord(e); cudaEventSynchronize(e);
  float ms; cudaEventElapsedTime(&ms, s, e);
  unsigned long long h[148]; cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  double flops = 2.0 * 128 * N * 16 * (double)iters * sms;
  printf("%-14s N=%3d cycles/mma=%6.1f  ideal=%5.1f  TFLOP/s=%7.1f  err=%s\n", name, N, (double)h[0] / iters,
         128.0 * N / 256, flops / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<64, false>("SS");  run<128, false>("SS");  run<256, false>("SS");
  run<64, true>("TS");   run<128, true>("TS");   run<256, true>("TS");
  return 0;
}
