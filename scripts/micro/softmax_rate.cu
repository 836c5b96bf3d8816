// Microbenchmark: the dQ kernel's per-row dS math (ds_cols<false>, 32 columns/thread) in
// isolation, with TMEM stores, 16 warps/SM; reports elements/clk/SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2605_08524_b200/csrc/attn_dq_sm100.cuh"
using namespace fcpb;
__global__ void __launch_bounds__(544, 1) sm_loop(int iters, unsigned long long* cyc, float* out, int do_st, int mma) {
  __shared__ uint32_t tbase;
  if (threadIdx.x < 32) tmem_alloc<512>(&tbase);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tbase;
  const uint32_t w = threadIdx.x >> 5;
  const uint32_t lane_bits = ((w & 3) * 32) << 16;
  (void)lane_bits;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int nsm = (blockDim.x - 32) / 32;   // softmax warps; the last warp issues MMAs
  if (w == nsm) {
    if (mma && elect_one()) {
      const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
      const uint32_t id = idesc_bf16_f32(128, 128, false, false);
      unsigned long long t0 = clock64();
      // keep the tensor pipe busy for roughly the softmax duration (S/dP-sized MMAs into cols 0-255)
      for (int i = 0; i < iters * 4; ++i)
        mma_ss(tmem + (i & 1) * 128, smem_desc_sw128(a + (i & 3) * 32, 16, 1024),
               smem_desc_sw128(b + (i & 3) * 32, 16, 1024), id, 1);
      (void)t0;
    }
    __syncwarp();
  } else {
  uint32_t s[32], dp[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) { s[i] = __float_as_uint(0.01f * (threadIdx.x + i)); dp[i] = __float_as_uint(0.02f * i); }
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint32_t t_ds = tmem + lane_bits + 384 + (w >> 2) * 16 + (it & 1) * 64;
    if (do_st) dq::ds_cols<false>(s, dp, 0.127f, -1.0f, -0.5f, t_ds, 0, 128, 128);
    else {
      // same math, no TMEM store
      const float2 c2 = make_float2(0.127f, 0.127f), nl = make_float2(-1.f, -1.f), nd = make_float2(-.5f, -.5f);
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const float2 x = __ffma2_rn(make_float2(__uint_as_float(s[2*u]), __uint_as_float(s[2*u+1])), c2, nl);
        float p0 = ex2(x.x), p1 = ex2(x.y);
        const float2 d = __fmul2_rn(make_float2(p0, p1), __fadd2_rn(make_float2(__uint_as_float(dp[2*u]), __uint_as_float(dp[2*u+1])), nd));
        s[2*u] = pack_bf16(d.x, d.y);
      }
    }
    tmem_wait_st();
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  float acc = 0; for (int i = 0; i < 32; ++i) acc += __uint_as_float(s[i]);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  }
  __syncthreads();
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}
int main() {
  unsigned long long* cyc; float* out; cudaMalloc(&cyc, 148 * 8); cudaMalloc(&out, 148 * 1024 * 4);
  const int iters = 2048;
  cudaFuncSetAttribute(sm_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  for (int mma : {1}) for (int st : {0, 1}) for (int warps : {16}) {
    sm_loop<<<148, warps * 32 + 32, 70 * 1024>>>(iters, cyc, out, st, mma); cudaDeviceSynchronize();
    unsigned long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    double el = (double)warps * 32 * 32 * iters;
    printf("mma=%d tmem_st=%d warps=%2d  elements/clk/SM = %.2f  (%s)\n", mma, st, warps, el / h, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
