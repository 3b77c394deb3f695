// scan.cuh -- pack_start of pecr_convert (src/pecr.cpp:83-131): the exclusive
// prefix sum of the per-pack entry totals, where a pack's total is the sum of
// its pool_w*pool_h window counts.  Reduce-then-scan in three launches, any
// number of packs, 64-bit offsets, deterministic (integer sums):
//
//   1. pack_scan_partial: each CTA reduces a chunk of kScanChunk packs to one
//      partial sum (a thread sums kScanItems consecutive packs, then the CTA
//      reduces by warp shuffles);
//   2. pack_scan_partials: one CTA turns the partials into exclusive chunk
//      offsets (1024-wide tiles with a running carry);
//   3. pack_scan_final: each CTA rescans its chunk -- thread-local prefix over
//      its packs, block-wide exclusive scan of the thread sums, plus the
//      chunk offset -- and writes start[i + 1]; start[0] = 0.
#pragma once

#include <stdint.h>

#include "common.cuh"

namespace sconv_cu {

constexpr int kScanThreads = 256;
constexpr int kScanItems = 8;
constexpr int kScanChunk = kScanThreads * kScanItems;

__device__ __forceinline__ int64_t pack_total(const int32_t* count, int wpp, int64_t p) {
  int64_t t = 0;
  for (int n = 0; n < wpp; ++n) t += count[p * wpp + n];
  return t;
}

// Block-wide exclusive scan of one value per thread (kScanThreads threads);
// also returns the block total.
__device__ __forceinline__ int64_t block_exclusive_scan(int64_t v, int64_t* total) {
  __shared__ int64_t warp_sums[kScanThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int64_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) warp_sums[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    int64_t s = lane < kScanThreads / 32 ? warp_sums[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(kFull, s, o);
      if (lane >= o) s += y;
    }
    if (lane < kScanThreads / 32) warp_sums[lane] = s;  // inclusive over warps
  }
  __syncthreads();
  const int64_t warp_off = wid ? warp_sums[wid - 1] : 0;
  *total = warp_sums[kScanThreads / 32 - 1];
  __syncthreads();  // warp_sums is reused by the next call
  return warp_off + incl - v;
}

__global__ void __launch_bounds__(kScanThreads) pack_scan_partial(const int32_t* count, int wpp,
                                                                  int64_t npacks, int64_t* partial) {
  const int64_t p0 = static_cast<int64_t>(blockIdx.x) * kScanChunk + threadIdx.x * kScanItems;
  int64_t s = 0;
  for (int i = 0; i < kScanItems; ++i)
    if (p0 + i < npacks) s += pack_total(count, wpp, p0 + i);
  int64_t total;
  block_exclusive_scan(s, &total);
  if (threadIdx.x == 0) partial[blockIdx.x] = total;
}

__global__ void __launch_bounds__(1024) pack_scan_partials(int64_t* partial, int64_t nparts) {
  __shared__ int64_t carry_s;
  __shared__ int64_t warp_sums[32];
  if (threadIdx.x == 0) carry_s = 0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int64_t base = 0; base < nparts; base += 1024) {
    __syncthreads();
    const int64_t i = base + threadIdx.x;
    const int64_t v = i < nparts ? partial[i] : 0;
    int64_t incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) warp_sums[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      int64_t s = warp_sums[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t y = __shfl_up_sync(kFull, s, o);
        if (lane >= o) s += y;
      }
      warp_sums[lane] = s;
    }
    __syncthreads();
    const int64_t carry = carry_s;
    if (i < nparts) partial[i] = carry + (wid ? warp_sums[wid - 1] : 0) + incl - v;  // exclusive
    __syncthreads();
    if (threadIdx.x == 0) carry_s = carry + warp_sums[31];
  }
}

__global__ void __launch_bounds__(kScanThreads) pack_scan_final(const int32_t* count, int wpp,
                                                                int64_t npacks,
                                                                const int64_t* offsets,
                                                                int64_t* start) {
  const int64_t p0 = static_cast<int64_t>(blockIdx.x) * kScanChunk + threadIdx.x * kScanItems;
  int64_t t[kScanItems];
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    t[i] = p0 + i < npacks ? pack_total(count, wpp, p0 + i) : 0;
    s += t[i];
  }
  int64_t total;
  int64_t run = offsets[blockIdx.x] + block_exclusive_scan(s, &total);
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    run += t[i];
    if (p0 + i < npacks) start[p0 + i + 1] = run;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) start[0] = 0;
}

}  // namespace sconv_cu
