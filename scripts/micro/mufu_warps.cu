// Microbenchmark: how many warps per SMSP it takes to saturate MUFU.EX2 on sm_100, for
// (a) pure ex2 with K independent values per thread and (b) the forward softmax's exp phase
// (FFMA2 scale, ex2, bf16 pack, FADD2 row sum) over C columns per thread -- i.e. a 128-column
// row done by one warp (C=128) versus split over two warps of the same SMSP (C=64 each).
// Reports elements per clock per SM (ceiling 16 on B200).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 mufu_warps.cu -o mufu_warps
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

template <int K>
__global__ void pure_ex2(int iters, unsigned long long* cyc, float* out) {
  float a[K];
#pragma unroll
  for (int i = 0; i < K; ++i) a[i] = -1e-3f * threadIdx.x - 1e-4f * i;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < K; ++i) a[i] = ex2f(a[i]) - 1.5f;
  }
  const unsigned long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < K; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// The forward's per-row exp phase over C columns (values regenerated cheaply each pass).
template <int C>
__global__ void softmax_exp(int iters, unsigned long long* cyc, float* out) {
  float s[C];
#pragma unroll
  for (int i = 0; i < C; ++i) s[i] = 0.01f * (threadIdx.x & 31) + 0.02f * i;
  uint32_t sink = 0;
  float l = 0.f;
  __syncthreads();
  const unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const float neg = -1.0f - 1e-6f * it;
    float2 sp[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
    for (int i = 0; i < C; i += 2) {
      const float2 x = __ffma2_rn(make_float2(s[i], s[i + 1]), make_float2(0.18f, 0.18f), make_float2(neg, neg));
      const float2 e = make_float2(ex2f(x.x), ex2f(x.y));
      sp[(i >> 1) & 1] = __fadd2_rn(sp[(i >> 1) & 1], e);
      __nv_bfloat162 b = __floats2bfloat162_rn(e.x, e.y);
      sink ^= *reinterpret_cast<uint32_t*>(&b);
    }
    l += sp[0].x + sp[0].y + sp[1].x + sp[1].y;
  }
  const unsigned long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = l + sink;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <typename F>
void run(const char* name, F kern, int warps, int elems_per_thread_iter, int iters) {
  unsigned long long* cyc;
  float* out;
  cudaMalloc(&cyc, 148 * 8);
  cudaMalloc(&out, 148 * 1024 * 4);
  kern<<<148, warps * 32>>>(iters, cyc, out);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h = 0;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-22s warps/SM=%2d  elem/clk/SM=%6.2f  %s\n", name, warps,
         (double)warps * 32 * elems_per_thread_iter * iters / h, cudaGetErrorString(e));
  cudaFree(cyc);
  cudaFree(out);
}

int main() {
  const int it = 2048;
  for (int w : {4, 8, 12, 16}) {
    run("pure ex2 K=8", pure_ex2<8>, w, 8, it);
    run("pure ex2 K=32", pure_ex2<32>, w, 32, it);
  }
  for (int w : {4, 8, 16}) {
    run("softmax C=128", softmax_exp<128>, w, 128, it / 4);
    run("softmax C=64", softmax_exp<64>, w, 64, it / 2);
  }
  return 0;
}
