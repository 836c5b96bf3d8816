// K5 pull kernel: the forward KV exchange as SM loads from peer memory over NVLink.
//
// When a rank's forward runs as one wave after the exchange (executor fuse_remote="all"),
// nothing overlaps the pulls, so they are done by every SM instead of by copy engines: each
// copy-engine transfer of a 2-10 MB run reached 370-500 GB/s (profiles/r02_exchange_*),
// while 148 SMs keep enough 16-byte loads in flight over NVLink to approach the link rate.
// Each segment is a contiguous byte range (one plane of one merged run, split by the host
// into pieces of at most kSegBytes) from a peer's IPC region into the receive arena.
#pragma once
#include <cstdint>

namespace fcpb {
namespace p2p {

struct Seg {
  uint64_t dst;      // local receive-arena address (16-byte aligned)
  uint64_t src;      // peer-mapped source address (16-byte aligned)
  int64_t bytes;     // multiple of 16, <= kSegBytes
};

constexpr int kThreads = 512;
constexpr int kVec = 8;                                   // 16-byte loads in flight per thread
constexpr int64_t kSegBytes = int64_t(kThreads) * kVec * 16;   // 64 KB: one pass of a CTA

// One CTA per segment at a time (grid-stride over the segment list): all kVec loads of a
// thread are issued before its first store, so a CTA has 64 KB of peer reads in flight.
// Loads bypass L1 (.cg: the bytes are used once, by this copy); stores are plain so the
// arena stays in L2 for the forward kernel that reads it next.
__device__ __forceinline__ void copy_segment(uint4* dst, const uint4* src, int64_t bytes) {
  const int nv = static_cast<int>(bytes >> 4);
  uint4 r[kVec];
#pragma unroll
  for (int i = 0; i < kVec; ++i) {
    const int j = i * kThreads + threadIdx.x;
    if (j < nv) r[i] = __ldcg(src + j);
  }
#pragma unroll
  for (int i = 0; i < kVec; ++i) {
    const int j = i * kThreads + threadIdx.x;
    if (j < nv) dst[j] = r[i];
  }
}

__global__ void __launch_bounds__(kThreads) gather_kernel(const Seg* __restrict__ segs, int n) {
  for (int s = blockIdx.x; s < n; s += gridDim.x) {
    const Seg sg = segs[s];
    copy_segment(reinterpret_cast<uint4*>(sg.dst), reinterpret_cast<const uint4*>(sg.src), sg.bytes);
  }
}

// Base-relative segments: address = bases[a >> 56] + (a & (2^56 - 1)).
constexpr int kMaxBases = 32;
struct Bases { uint64_t p[kMaxBases]; };
__global__ void __launch_bounds__(kThreads) gather_based_kernel(const Seg* __restrict__ segs, int n,
                                                                const __grid_constant__ Bases b) {
  constexpr uint64_t kOff = (uint64_t{1} << 56) - 1;
  for (int s = blockIdx.x; s < n; s += gridDim.x) {
    const Seg sg = segs[s];
    copy_segment(reinterpret_cast<uint4*>(b.p[sg.dst >> 56] + (sg.dst & kOff)),
                 reinterpret_cast<const uint4*>(b.p[sg.src >> 56] + (sg.src & kOff)), sg.bytes);
  }
}

}  // namespace p2p
}  // namespace fcpb
