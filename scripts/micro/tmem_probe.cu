// Microbenchmarks for the softmax phases' TMEM traffic, one CTA per SM (148 CTAs):
//  (1) tcgen05.ld 32x32b.x32 aggregate read rate per SM vs warps, with 1 or 4 loads in
//      flight per wait (K1/K2 issue four 32-column loads before one wait);
//  (2) tcgen05.st 32x32b.x16 aggregate write rate;
//  (3) kind::f16 MMA with bf16 operands and an f16 accumulator (c_format = 0): legal on
//      sm_100a?  Result layout and accuracy vs an fp32-accumulated reference.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tmem_probe tmem_probe.cu
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include "../../paper_2605_08524_b200/csrc/sm100_ptx.cuh"
using namespace fcpb;

template <int INFLIGHT>
__global__ void ld_loop(int iters, unsigned long long* cyc, uint32_t* out) {
  __shared__ uint32_t tbase;
  if (threadIdx.x < 32) tmem_alloc<512>(&tbase);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tbase;
  const uint32_t w = threadIdx.x >> 5;
  const uint32_t addr = tmem + (((w & 3) * 32) << 16) + ((w >> 2) & 3) * 128;
  uint32_t acc = 0;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; i += INFLIGHT) {
    uint32_t v[INFLIGHT][32];
#pragma unroll
    for (int f = 0; f < INFLIGHT; ++f) tmem_ld32(addr + f * 32, v[f]);
    tmem_wait_ld();
#pragma unroll
    for (int f = 0; f < INFLIGHT; ++f)
#pragma unroll
      for (int j = 0; j < 32; ++j) acc ^= v[f][j];
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

__global__ void st_loop(int iters, unsigned long long* cyc) {
  __shared__ uint32_t tbase;
  if (threadIdx.x < 32) tmem_alloc<512>(&tbase);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tbase;
  const uint32_t w = threadIdx.x >> 5;
  const uint32_t addr = tmem + (((w & 3) * 32) << 16) + ((w >> 2) & 3) * 128;
  uint32_t v[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) v[j] = threadIdx.x * 16 + j;
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    tmem_st16(addr + (i & 7) * 16, v);
    v[0] += 1;
  }
  tmem_wait_st();
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

// (3) D[128 x 128] = A[128 x 128] * B[128 x 128]^T, both K-major bf16 in SW128 panels, with
// c_format 0 (f16) -- read back 128 columns of 32-bit cells per row.
__global__ void f16acc(const __nv_bfloat16* a, const __nv_bfloat16* b, uint32_t* out, int f16) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint32_t tbase;
  __shared__ uint64_t bar;
  // stage A and B as two 64-column SW128 panels each (row r, 16-byte chunk c -> c ^ (r & 7))
  for (int idx = threadIdx.x; idx < 128 * 16; idx += blockDim.x) {
    const int r = idx / 16, c = idx % 16, panel = c / 8, cc = c % 8;
    const uint4 va = reinterpret_cast<const uint4*>(a + r * 128)[c];
    const uint4 vb = reinterpret_cast<const uint4*>(b + r * 128)[c];
    const int off = panel * 16384 + r * 128 + ((cc ^ (r & 7)) * 16);
    *reinterpret_cast<uint4*>(smem + off) = va;
    *reinterpret_cast<uint4*>(smem + 32768 + off) = vb;
  }
  fence_proxy_async_smem();
  if (threadIdx.x < 32) tmem_alloc<512>(&tbase);
  if (threadIdx.x == 32) { mbar_init(&bar, 1); fence_barrier_init(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = tbase;
  if (threadIdx.x < 32) {
    uint32_t id = idesc_bf16_f32(128, 128, false, false);
    if (f16) id &= ~(3u << 4);            // c_format = F16
    if (elect_one()) {
      const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 32768);
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
        mma_ss(tmem, smem_desc_sw128(sa + off, 16, 1024), smem_desc_sw128(sb + off, 16, 1024), id, kk > 0);
      }
      mma_commit(&bar);
    }
    __syncwarp();
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  const uint32_t w = threadIdx.x >> 5;
  if (w < 4) {
    const int row = w * 32 + (threadIdx.x & 31);
    for (int c = 0; c < 4; ++c) {
      uint32_t v[32];
      tmem_ld32(tmem + ((w * 32) << 16) + c * 32, v);
      tmem_wait_ld();
      for (int j = 0; j < 32; ++j) out[row * 128 + c * 32 + j] = v[j];
    }
  }
  tc_fence_before(); __syncthreads();
  if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc<512>(tmem); }
}

int main() {
  unsigned long long* cyc; uint32_t* out;
  cudaMalloc(&cyc, 148 * 8); cudaMalloc(&out, 148 * 1024 * 4);
  const int iters = 4096;
  for (int warps : {4, 8, 16}) {
    for (int inflight : {1, 4}) {
      if (inflight == 1) ld_loop<1><<<148, warps * 32>>>(iters, cyc, out);
      else ld_loop<4><<<148, warps * 32>>>(iters, cyc, out);
      cudaDeviceSynchronize();
      unsigned long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      const double bytes = (double)warps * 32 * 32 * 4 * iters;
      printf("ld x32 warps=%2d inflight=%d: %.1f B/clk/SM (%s)\n", warps, inflight, bytes / h,
             cudaGetErrorString(cudaGetLastError()));
    }
    st_loop<<<148, warps * 32>>>(iters, cyc);
    cudaDeviceSynchronize();
    unsigned long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    const double bytes = (double)warps * 32 * 16 * 4 * iters;
    printf("st x16 warps=%2d: %.1f B/clk/SM (%s)\n", warps, bytes / h, cudaGetErrorString(cudaGetLastError()));
  }
  // (3) f16 accumulation with bf16 operands
  std::vector<__nv_bfloat16> ha(128 * 128), hb(128 * 128);
  std::vector<float> fa(128 * 128), fb(128 * 128);
  uint32_t seed = 12345;
  auto rnd = [&]() { seed = seed * 1664525u + 1013904223u; return ((seed >> 8) & 0xffff) / 65536.f * 4.f - 2.f; };
  for (int i = 0; i < 128 * 128; ++i) {
    ha[i] = __float2bfloat16(rnd()); fa[i] = __bfloat162float(ha[i]);
    hb[i] = __float2bfloat16(rnd()); fb[i] = __bfloat162float(hb[i]);
  }
  __nv_bfloat16 *da, *db; uint32_t* dout;
  cudaMalloc(&da, 32768); cudaMalloc(&db, 32768); cudaMalloc(&dout, 128 * 128 * 4);
  cudaMemcpy(da, ha.data(), 32768, cudaMemcpyHostToDevice);
  cudaMemcpy(db, hb.data(), 32768, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(f16acc, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  for (int f16 : {0, 1}) {
    cudaMemset(dout, 0, 128 * 128 * 4);
    f16acc<<<1, 128, 70000>>>(da, db, dout, f16);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<uint32_t> h(128 * 128);
    cudaMemcpy(h.data(), dout, h.size() * 4, cudaMemcpyDeviceToHost);
    double max_err_lo = 0, max_err_packed = 0, max_ref = 0;
    for (int r = 0; r < 128; ++r)
      for (int c = 0; c < 128; ++c) {
        double ref = 0;
        for (int k = 0; k < 128; ++k) ref += (double)fa[r * 128 + k] * fb[c * 128 + k];
        max_ref = fmax(max_ref, fabs(ref));
        if (!f16) {
          float g; memcpy(&g, &h[r * 128 + c], 4);
          max_err_lo = fmax(max_err_lo, fabs(g - ref));
        } else {
          // hypothesis A: one f16 per 32-bit cell (low half); B: two per cell (column c/2)
          __half lo; uint16_t bits = h[r * 128 + c] & 0xffff; memcpy(&lo, &bits, 2);
          max_err_lo = fmax(max_err_lo, fabs(__half2float(lo) - ref));
          uint32_t cell = h[r * 128 + c / 2];
          uint16_t pb = (c & 1) ? (cell >> 16) : (cell & 0xffff);
          __half pk; memcpy(&pk, &pb, 2);
          max_err_packed = fmax(max_err_packed, fabs(__half2float(pk) - ref));
        }
      }
    printf("f16acc=%d (%s): max|ref| %.2f  max err (one per cell) %.4g  (packed pairs) %.4g\n", f16,
           cudaGetErrorString(e), max_ref, max_err_lo, max_err_packed);
  }
  return 0;
}
