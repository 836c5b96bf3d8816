// Microbenchmark: MUFU.EX2 (ex2.approx.ftz.f32) and FFMA2 throughput per SM per clock.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void ex2_loop(int iters, float* out, unsigned long long* cyc) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
  }
  unsigned long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void fma2_loop(int iters, float* out, unsigned long long* cyc) {
  float2 a[8]; const float2 b = make_float2(1.0001f, 0.9999f), c = make_float2(1e-7f, 2e-7f);
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = make_float2(threadIdx.x * 1e-3f, i * 1e-4f);
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __ffma2_rn(a[i], b, c);
  }
  unsigned long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
__global__ void cvt_loop(int iters, float* out, unsigned long long* cyc) {
  float a[16];
  uint32_t acc = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; i += 2) {
      uint32_t r;
      asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a[i]), "f"(a[i + 1]));
      acc ^= r;
      a[i] += 1e-7f;
    }
  }
  unsigned long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* out; unsigned long long* cyc; cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
  const int iters = 4096;
  for (int threads : {128, 256, 512, 1024}) {
    ex2_loop<<<148, threads>>>(iters, out, cyc); cudaDeviceSynchronize();
    unsigned long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    double ops = (double)threads * iters * 8;
    printf("ex2  threads/SM=%4d  ex2/clk/SM=%.2f\n", threads, ops / h);
    fma2_loop<<<148, threads>>>(iters, out, cyc); cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("fma2 threads/SM=%4d  ffma2 instr/clk/SM=%.2f (x2 flops-lanes)\n", threads, ops / h);
    cvt_loop<<<148, threads>>>(iters, out, cyc); cudaDeviceSynchronize();
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("cvt  threads/SM=%4d  cvt.bf16x2 /clk/SM=%.2f\n", threads, ops / h);
  }
  return 0;
}
