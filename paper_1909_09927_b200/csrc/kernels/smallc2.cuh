// smallc2.cuh -- ECR for maps with few input channels, lanes over pixels
// (VGG conv1_1: C = 3 -> K = 64 at 224x224, the one VGG-19 layer whose roof
// is HBM: 861 MB moved for 3.3 GFLOP).
//
// Every other kernel puts the 32 lanes of a warp on output channels, so that
// a window's nonzero mask is warp-uniform and zero cells are skipped by a
// branch.  That pays when the reduction is long (C >= 64).  With C = 3 a
// window holds 27 terms; ecr_smallc_kernel (smallc.cuh) spends ~1360
// instructions per 4x4 x 64 tile, of which the FFMA2 are a quarter and, with
// R = 2 blocks that ptxas if-converts, already 82% of the dense count (ncu,
// profiles/r01): the layer ran at 74% of issue slots and 30% of HBM.
//
// Here lane l owns output pixel x0 + l of 4 consecutive output rows, and a
// pass covers KG = 8 filters (32 accumulators).  For each term (c, i, j) in
// the reference's order the lane reads its 4 cells from shared memory
// (consecutive lanes, consecutive words); the term's 8 weights are the same
// for every lane and come from the constant bank straight into uniform
// registers (LDCU), each weight pair feeding one FFMA2 per row.  Zero cells
// are multiplied: with finite weights that adds +-0 to an accumulator that
// is never -0, which leaves it unchanged, so every output is exactly the
// reference's sum of its window's nonzero terms in (c, i, j) order
// (ecr_convert + ecr_spmv_conv, src/ecr.cpp:79-91,117-120; EXACT = rounded
// mul + rounded add, bit-identical); any Inf / NaN weight switches the CTA
// to a path that predicates zero cells off per lane.  The FMA pipe is the
// limit (ncu: 75% busy; 27 FFMA2 per output pixel and filter pair).
//
// Outputs leave by TMA: each pass stages its 8 x 4 x 32 box in shared
// memory and one elected lane issues a bulk tensor store (rows, columns and
// filters past the map are clipped by the unit); without a 16-byte row
// pitch (OW % 4 != 0) lanes store directly, one 128-byte row segment per
// instruction.
//
// Persistent CTAs: the 8 warps of a CTA take the 8 items (image, band of 4
// output rows, 32 columns) of an octet and walk the filter groups in
// lockstep; each CTA owns a contiguous, equal share of the (octet, group)
// units, and the next octet's 6 x 34 x C input windows are prefetched with
// cp.async into the other half of a per-warp double buffer.
//
// The filters of a launch live in one of kSc2Slots constant-memory slots
// (host: launch_smallc2_c, sconv_cuda.cu), copied on the launch's stream and
// released by an event, so concurrent launches never share a slot.
#pragma once

#include <cuda.h>

#include "common.cuh"

namespace sconv_cu {

struct SmallC2Args {
  const float* x;   // [N][C][H][W]
  const float* wt;  // [C][9][Kp]  (transposed filters, Kp a multiple of 64)
  float* y;         // [N][K][OH][OW]
  int N, C, H, W, K, Kp, OH, OW;
  int bands, strips, total_items;  // items = N * bands * strips
  int relu;
  int slot;         // c_sc2_w slot holding this launch's K-block of filters
  int k0;           // first filter of the block
};

#ifndef SCONV_SC2_MINB  // resident CTAs per SM the register budget is cut for
#define SCONV_SC2_MINB 4
#endif
#ifndef SCONV_SC2_KG  // filters per lane pass (accumulators = 4 rows x KG)
#define SCONV_SC2_KG 8
#endif

constexpr int kSc2Warps = 8;
constexpr int kSc2Slots = 4;                      // constant-memory filter slots
constexpr int kSc2SlotFloats = 4 * 9 * 64;        // C <= 4 channels x 9 taps x 64 filters

// The filters of one launch ([C][9][64], one K-block), read by every lane at
// the same address: from the constant bank they feed FFMA2 as uniform
// registers (one LDCU.64 per weight pair, 8 bytes per warp), where a
// shared-memory broadcast would return 512 bytes per warp through the LSU.
__constant__ float4 c_sc2_w[kSc2Slots][kSc2SlotFloats / 4];
#ifndef SCONV_SC2_ROWS  // output rows per work item (and per lane)
#define SCONV_SC2_ROWS 4
#endif
constexpr int kSc2Rows = SCONV_SC2_ROWS;
constexpr int kSc2KG = SCONV_SC2_KG;              // filters per pass of a lane
constexpr int kSc2WinRows = kSc2Rows + 2;         // input rows of its window
#ifndef SCONV_SC2_SPLIT  // TMA store boxes per filter group (1: one KG-filter box; 2: two halves)
#define SCONV_SC2_SPLIT 2
#endif
constexpr int kSc2Pitch = 34;                     // window row pitch (floats)
constexpr int kSc2Chan = kSc2WinRows * kSc2Pitch; // one channel of a window

constexpr int kSc2Split = SCONV_SC2_SPLIT;
constexpr int kSc2BoxK = kSc2KG / kSc2Split;      // filters per TMA store box
constexpr int kSc2Out = kSc2BoxK * kSc2Rows * 32; // one warp's staging slot (floats)

__host__ __device__ constexpr int sc2_smem_bytes(int C, int Kp) {
  return (2 * kSc2Warps * C * kSc2Chan + kSc2Warps * kSc2Out) * 4;
}

// {a0, a1} += {w0, w1} * v   (FAST: one FFMA2; EXACT: rounded product, rounded sum)
template <bool FAST>
__device__ __forceinline__ void mac2(float& a0, float& a1, float w0, float w1, float v) {
  if constexpr (FAST) {
    ffma2(a0, a1, w0, w1, v);
  } else {
    exact2_mul(a0, a1, w0, w1, v);  // FMA-pipe-bound here: see common.cuh
  }
}

// The 9C terms of 4 output rows x KG filters of one lane, in (c, i, j)
// order: lane l's cell of term (c, i, j) for output row r is
// win[c][r + i][l + j]; the KG weights of the term (filters KG*g ..
// KG*g + KG-1) come from the constant bank as uniform registers, each pair
// feeding one FFMA2 per output row.  A zero cell contributes nothing: with finite weights
// its products are +-0 and acc + (+-0) == acc (acc is never -0: it starts at
// +0 and a round-to-nearest sum is -0 only when both addends are), so the
// FFMA2 run unconditionally; SKIP = true (some weight is Inf / NaN, whose
// product with 0 would not vanish) predicates them off per lane, as
// ecr_convert drops the cell (src/ecr.cpp:84).
template <int C, bool FAST, bool SKIP>
__device__ __forceinline__ void sc2_terms(float (&acc)[kSc2Rows][kSc2KG], const float* wn, const float4* wk) {
#pragma unroll 1
  for (int c = 0; c < C; ++c)
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        float v[kSc2Rows];
#pragma unroll
        for (int r = 0; r < kSc2Rows; ++r) v[r] = wn[c * kSc2Chan + (r + i) * kSc2Pitch + j];
        const float4* wq = wk + (c * 9 + i * 3 + j) * 16;
#pragma unroll
        for (int q = 0; q < kSc2KG / 4; ++q) {
          const float4 w4 = wq[q];
#pragma unroll
          for (int r = 0; r < kSc2Rows; ++r) {
            if (!SKIP || v[r] != 0.0f) {
              mac2<FAST>(acc[r][4 * q], acc[r][4 * q + 1], w4.x, w4.y, v[r]);
              mac2<FAST>(acc[r][4 * q + 2], acc[r][4 * q + 3], w4.z, w4.w, v[r]);
            }
          }
        }
      }
}

template <int C, bool FAST, bool RELU, bool TMA>
__global__ void __launch_bounds__(256, SCONV_SC2_MINB)
    ecr_smallc2_kernel(const SmallC2Args a, const __grid_constant__ CUtensorMap ymap) {
  extern __shared__ float4 sc2_smem[];
  float* win = reinterpret_cast<float*>(sc2_smem);   // [2][8 warps][C][6][36]
  float* ost = win + 2 * kSc2Warps * C * kSc2Chan;   // [8 warps][KG][4][32] TMA store boxes

  const int tid = threadIdx.x;
  const int warp = __shfl_sync(kFull, tid >> 5, 0), lane = tid & 31;
  const float4* wk = c_sc2_w[a.slot];

  int bad = 0;  // any non-finite weight (see sc2_terms)
  for (int i = tid; i < C * 9 * 16; i += 256) {
    const float4 v = wk[i];
    bad |= !isfinite(v.x) | !isfinite(v.y) | !isfinite(v.z) | !isfinite(v.w);
  }

  const size_t plane = static_cast<size_t>(a.H) * a.W;
  const int items = a.total_items;
  // work item w -> (n, band, strip), strips fastest; warps of a CTA take
  // consecutive items
  auto coords = [&](int w, int& n, int& y0, int& x0) {
    const int sx = w % a.strips, r = w / a.strips;
    x0 = sx * 32;
    y0 = (r % a.bands) * kSc2Rows;
    n = r / a.bands;
  };
  // cp.async the 6 x 34 x C input window of item w into buffer b
  auto stage = [&](int w, int b) {
    int n, y0, x0;
    coords(w, n, y0, x0);
    float* dst = win + (b * kSc2Warps + warp) * C * kSc2Chan + lane;
    const float* src = a.x + (static_cast<size_t>(n) * C * plane + static_cast<size_t>(y0) * a.W + x0 + lane);
    const bool col_a = x0 + lane < a.W, col_b = lane < 2 && x0 + 32 + lane < a.W;
#pragma unroll
    for (int c = 0; c < C; ++c) {
#pragma unroll
      for (int r = 0; r < kSc2WinRows; ++r) {
        const bool row = y0 + r < a.H;
        const float* s = src + (static_cast<size_t>(c) * plane + r * a.W);
        cp_async4(dst + c * kSc2Chan + r * kSc2Pitch, row && col_a ? s : a.x, row && col_a);
        if (lane < 2) cp_async4(dst + c * kSc2Chan + r * kSc2Pitch + 32, row && col_b ? s + 32 : a.x, row && col_b);
      }
    }
  };

  // Work units are (octet of items, filter group): the 8 warps of a CTA run
  // the 8 items of an octet side by side, in lockstep over the same filter
  // groups (their constant-bank reads hit the same lines), and CTA b takes
  // the contiguous range [u0, u1) of an even split of the units, so every
  // CTA has the same work to within one group (a whole-item split leaves up
  // to one item -- 1/7 of a warp's work at conv1_1's size -- as a tail).
  // Consecutive units of one octet reuse its staged windows.
  const int kn = min(64, a.K - a.k0);
  const int ng = (kn + kSc2KG - 1) / kSc2KG;
  const int octets = (items + kSc2Warps - 1) / kSc2Warps;
  const int units = octets * ng;  // host: < 2^31
  const int nb = gridDim.x, b = blockIdx.x;
  const int q = units / nb, rem = units - q * nb;
  const int u0 = b * q + min(b, rem), u1 = u0 + q + (b < rem ? 1 : 0);
  const int first = u0 / ng;
  const int last = u1 > u0 ? (u1 - 1) / ng : first - 1;
  auto item_of = [&](int o) { return o * kSc2Warps + warp; };
  int buf = 0;
  if (first <= last && item_of(first) < items) stage(item_of(first), 0);
  cp_async_commit();
  const bool nonfinite = __syncthreads_or(bad);

  const size_t oplane = static_cast<size_t>(a.OH) * a.OW;
  for (int o = first; o <= last; ++o) {
    if (o < last && item_of(o + 1) < items) stage(item_of(o + 1), buf ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncwarp();
    const int w = item_of(o);
    const int g_lo = o == first ? u0 - o * ng : 0;
    const int g_hi = o == last ? u1 - o * ng : ng;
    if (w >= items) {  // the last octet may be partial: keep this warp's slot in step
      buf ^= 1;
      continue;
    }
    int n, y0, x0;
    coords(w, n, y0, x0);
    const float* wn = win + (buf * kSc2Warps + warp) * C * kSc2Chan + lane;
    const bool col_ok = x0 + lane < a.OW;
    float* yk = a.y + ((static_cast<size_t>(n) * a.K + a.k0) * a.OH + y0) * a.OW + x0 + lane;
    // groups of KG filters; the window stays in shared memory across them
#pragma unroll 1
    for (int g = g_lo; g < g_hi; ++g) {
      float acc[kSc2Rows][kSc2KG];
#pragma unroll
      for (int r = 0; r < kSc2Rows; ++r)
#pragma unroll
        for (int k = 0; k < kSc2KG; ++k) acc[r][k] = 0.0f;
      if (!nonfinite) {
        sc2_terms<C, FAST, false>(acc, wn, wk + (kSc2KG / 4) * g);
      } else {
        sc2_terms<C, FAST, true>(acc, wn, wk + (kSc2KG / 4) * g);
      }
      if constexpr (TMA) {
        // the warp's KG x 4 x 32 outputs go out as kSc2Split TMA stores of
        // BoxK filters (rows past OH, columns past OW and filters past K are
        // clipped by the unit); the staging slot is refilled once the
        // previous store has read it (2 KB slots: 4 CTAs fit an SM)
        float* ob = ost + warp * kSc2Out + lane;
        const unsigned slot = static_cast<unsigned>(__cvta_generic_to_shared(ost + warp * kSc2Out));
#pragma unroll
        for (int hbox = 0; hbox < kSc2Split; ++hbox) {
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          __syncwarp();
#pragma unroll
          for (int k = 0; k < kSc2BoxK; ++k)
#pragma unroll
            for (int r = 0; r < kSc2Rows; ++r) {
              const float v = acc[r][hbox * kSc2BoxK + k];
              ob[(k * kSc2Rows + r) * 32] = RELU ? relu_f(v) : v;
            }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            asm volatile(
                "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];"
                ::"l"(reinterpret_cast<uint64_t>(&ymap)), "r"(x0), "r"(y0),
                  "r"(a.k0 + kSc2KG * g + hbox * kSc2BoxK), "r"(n), "r"(slot)
                : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
      } else if (col_ok) {
        // plain stores: each writes one 128-byte segment of one channel row
        const int kv = kn - kSc2KG * g;
#pragma unroll
        for (int r = 0; r < kSc2Rows; ++r) {
          if (y0 + r >= a.OH) break;
          float* yo = yk + r * a.OW + kSc2KG * g * oplane;
#pragma unroll
          for (int k = 0; k < kSc2KG; ++k) {
            if (k < kv) __stcs(yo, RELU ? relu_f(acc[r][k]) : acc[r][k]);
            yo += oplane;
          }
        }
      }
    }
    __syncwarp();  // every lane has read buffer `buf` before it is restaged
    buf ^= 1;
  }
  cp_async_wait<0>();
  if (TMA && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

}  // namespace sconv_cu
