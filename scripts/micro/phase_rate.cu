// Microbenchmark: the dK/dV kernel's phase-1 chunk (bwd::p_chunk, 32 columns per thread:
// lse loads from smem, FFMA2 scale, ex2 (half MUFU, half polynomial), bf16 pack, TMEM store)
// in isolation, W softmax warps per SM, optionally preceded by the tcgen05.ld of S and
// optionally with an MMA warp keeping the tensor pipe busy on other TMEM columns.
// Reports cycles per chunk per warp and elements/clk/SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 phase_rate.cu -o phase_rate
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2605_08524_b200/csrc/attn_bwd_sm100.cuh"
using namespace fcpb;

__global__ void __launch_bounds__(544, 1)
phase_loop(int iters, int nsm_warps, int do_ld, int mma, int kind, unsigned long long* cyc, float* out) {
  __shared__ uint32_t tbase;
  __shared__ __align__(16) float lse[128];
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  if (threadIdx.x < 32) tmem_alloc<512>(&tbase);
  if (threadIdx.x < 128) lse[threadIdx.x] = -3.f - 0.001f * threadIdx.x;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  const uint32_t w = threadIdx.x >> 5;
  const uint32_t lane_bits = ((w & 3) * 32) << 16;
  if (w == (uint32_t)nsm_warps) {
    // MMA warp: TS MMAs, A = TMEM cols [256,320), accumulate into cols [384,512)
    if (mma && elect_one()) {
      const uint32_t b = smem_u32(smem);
      const uint32_t id = idesc_bf16_f32(128, 128, false, true);
      for (int i = 0; i < iters * 3; ++i)
        mma_ts(tmem + 384, tmem + 256 + (i & 7) * 8, smem_desc_sw128(b + (i & 7) * 2048, 16384, 1024),
               id, 1);
      mma_commit(reinterpret_cast<uint64_t*>(smem + 65536));
    }
    __syncwarp();
  } else if (w < (uint32_t)nsm_warps) {
    const int wg = w >> 2;                                   // 32-column slice of S [0,128)
    const uint32_t t_s = tmem + lane_bits + wg * 32;
    uint32_t sv[32];
    float pr[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) sv[i] = __float_as_uint(0.01f * (threadIdx.x & 31) + 0.02f * i);
    float acc = 0.f;
    const uint32_t l2 = smem_u32(&lse[wg * 32]);
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      if (do_ld) {
        tmem_ld32(t_s, sv);
        tmem_wait_ld();
      }
      if (kind == 0) {
        bwd::p_chunk<false>(sv, l2, 1.2f, pr, t_s + 16 * (it & 1), true, 0, 0, 0);
        tmem_wait_st();
      } else if (kind == 1) {          // same math, no TMEM store
        const float2 c2 = make_float2(1.2f, 1.2f);
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const float2 x = __ffma2_rn(make_float2(__uint_as_float(sv[2 * u]), __uint_as_float(sv[2 * u + 1])),
                                      c2, make_float2(-3.f, -3.1f));
          float2 e;
          if (u & 1) e = ex2_poly2(x); else e = make_float2(ex2(x.x), ex2(x.y));
          pr[2 * u] = e.x; pr[2 * u + 1] = e.y;
          sv[2 * u] = pack_bf16(e.x, e.y);
        }
      } else if (kind == 3) {          // ex2.approx.ftz.bf16x2: 2 results per MUFU instruction
        const float2 c2 = make_float2(1.2f, 1.2f);
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const float2 x = __ffma2_rn(make_float2(__uint_as_float(sv[2 * u]), __uint_as_float(sv[2 * u + 1])),
                                      c2, make_float2(-3.f, -3.1f));
          uint32_t xb = pack_bf16(x.x, x.y), eb;
          asm("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(eb) : "r"(xb));
          pr[2 * u] = __uint_as_float(eb << 16);
          pr[2 * u + 1] = __uint_as_float(eb & 0xffff0000u);
          sv[2 * u] = eb;
        }
      } else {                         // MUFU only, no store
        const float2 c2 = make_float2(1.2f, 1.2f);
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const float2 x = __ffma2_rn(make_float2(__uint_as_float(sv[2 * u]), __uint_as_float(sv[2 * u + 1])),
                                      c2, make_float2(-3.f, -3.1f));
          const float2 e = make_float2(ex2(x.x), ex2(x.y));
          pr[2 * u] = e.x; pr[2 * u + 1] = e.y;
          sv[2 * u] = pack_bf16(e.x, e.y);
        }
      }
#pragma unroll
      for (int i = 0; i < 32; i += 8) acc += pr[i];
    }
    const unsigned long long t1 = clock64();
    if ((threadIdx.x & 31) == 0 && w == 0) cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

int main() {
  unsigned long long* cyc;
  float* out;
  cudaMalloc(&cyc, 148 * 8);
  cudaMalloc(&out, 148 * 1024 * 4);
  const int iters = 4096;
  cudaFuncSetAttribute(phase_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  const char* kinds[] = {"p_chunk+st", "math only ", "mufu only ", "bf16x2 ex2"};
  for (int kind : {2, 3})
    for (int warps : {4, 8, 16})
      for (int ld : {0})
        for (int mma : {1}) {
          phase_loop<<<148, warps * 32 + 32, 80 * 1024>>>(iters, warps, ld, mma, kind, cyc, out);
          cudaError_t e = cudaDeviceSynchronize();
          unsigned long long h = 0;
          cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
          printf("%s warps=%2d ld=%d mma=%d  cycles/chunk/warp=%7.1f  elem/clk/SM=%6.2f  %s\n", kinds[kind],
                 warps, ld, mma, (double)h / iters, (double)warps * 32 * 32 * iters / h,
                 cudaGetErrorString(e));
        }
  return 0;
}
