// ingest.cuh -- device side of the compressed ingest (host/pack.cpp): expand
// a batch of maps shipped as nonzero bitmap + packed values back to dense
// [n][C][H][W] in HBM, right before the convolution reads it.
//
// One warp per 1024-element block: lane l holds word l of the block, a warp
// prefix sum of the word popcounts gives every word's first value, and the
// block is written word by word with lanes over the 32 elements of a word
// (128-byte coalesced stores); a set bit's value is values[first + popc(bits
// below it)].  Zeros are written as +0.0.
#pragma once

#include "common.cuh"

namespace sconv_cu {

struct ExpandArgs {
  const uint32_t* bits;   // [n][words]
  const int64_t* base;    // [n][blocks + 1], absolute offsets into the caller's values
  const float* values;    // values[0] holds the nonzero at absolute offset value0
  int64_t value0;
  int n;
  int64_t elems, words, blocks;  // per image
  float* x;               // [n][elems]
};

__global__ void expand_packed_kernel(const ExpandArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t total = static_cast<int64_t>(a.n) * a.blocks;
  const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  for (int64_t g = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; g < total;
       g += warps) {
    const int64_t img = g / a.blocks, b = g - img * a.blocks;
    const int64_t wi = b * 32 + lane;
    const uint32_t word = wi < a.words ? __ldg(a.bits + img * a.words + wi) : 0u;
    // exclusive prefix of the popcounts over the block's words
    const int cnt = __popc(word);
    int incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += t;
    }
    const int64_t first = __ldg(a.base + img * (a.blocks + 1) + b) - a.value0 + (incl - cnt);
    const float* vals = a.values;
    float* out = a.x + img * a.elems + b * 1024;
    const int64_t left = a.elems - b * 1024;  // elements of this block inside the image
    const unsigned below = (1u << lane) - 1u;
#pragma unroll 4
    for (int w = 0; w < 32; ++w) {
      if (w * 32 >= left) break;  // warp-uniform: past the image's last word
      const uint32_t m = __shfl_sync(kFull, word, w);
      const int64_t f = __shfl_sync(kFull, first, w);
      const int e = w * 32 + lane;
      const float v = (m >> lane) & 1u ? __ldg(vals + f + __popc(m & below)) : 0.0f;
      if (e < left) out[e] = v;
    }
  }
}

}  // namespace sconv_cu
