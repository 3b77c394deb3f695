// ecr_body.cuh -- the per-channel ECR step shared by the v2 (ecr_tiled.cuh)
// and v3 (ecr_ws.cuh) kernels.
//
// One warp, one input channel c, one TH x TW output tile: `is` points at the
// warp's (TH-1)S+KH x (TW-1)S+KW input window of channel c in shared memory
// (row pitch SPITCH floats, rows 16B aligned), and (m0, m1) is the window's
// nonzero mask from two ballots, bit Y*BPITCH + X for window cell (Y, X).
// That mask is the ECR compaction of the window (ecr_convert keeps exactly the
// v != 0 cells, src/ecr.cpp:79-91); it is computed once per channel and
// shared by all 32*R output channels of the warp.
//
// For every set bit, in window raster order, the cell value v is broadcast
// and multiplied into each output whose 3x3 (KH x KW) window covers the cell,
// against register-resident weights wr[i*KW+j][r]: for every output the
// terms of channel c arrive in (i, j) order, so with EXACT arithmetic (rounded
// mul, rounded add) the sum is bit-identical to ecr_spmv_conv (:117-120).
// FAST uses packed FFMA2 (same order, fused rounding).
//
// The branch per cell is warp-uniform (the mask came from a ballot); its cost
// (~4 SMSP cycles on B200, tools/micro/branch_cost.cu) is what bounds this
// kernel.  ROWSKIP adds one test per window row and skips rows without a
// nonzero: a win once fewer than ~1/4 of the cells are nonzero, so the
// kernels select it per channel from the mask's popcount.
#pragma once

#include "common.cuh"

// EXACT arithmetic with packed f32x2 mul + add (1) or scalar FMUL + FADD (0)
#ifndef SCONV_EXACT2
#define SCONV_EXACT2 1
#endif

// 0: let ptxas if-convert small blocks; 2: keep every block behind its branch
#ifndef SCONV_BODY_GUARD
#define SCONV_BODY_GUARD 0
#endif

// Blocks of at most LOW FFMA2 (1-2-tap cells at R = 4) are if-converted by
// ptxas with or without the guard, which then only adds a predicated NOP:
// guarding only the blocks in (LOW, MIN) measured -1.1% (WsA) / -2.6% (conv1_2)
// at s = 0.7 against guarding every block under MIN.
#ifndef SCONV_GUARD_LOW_FFMA2
#define SCONV_GUARD_LOW_FFMA2 4
#endif
#ifndef SCONV_GUARD_MIN_FFMA2
#define SCONV_GUARD_MIN_FFMA2 8
#endif

namespace sconv_cu {

// One window row (WPW cells, 16B-aligned) from shared memory by volatile
// loads, so ptxas keeps them where they are issued (row prefetch below).
template <int WPW>
__device__ __forceinline__ void lds_row_pinned(float (&dst)[4 * ((WPW + 3) / 4)], const float* src) {
  const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(src));
#pragma unroll
  for (int q = 0; q < (WPW + 3) / 4; ++q) {
    if (4 * q + 2 >= WPW) {
      asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(dst[4 * q]), "=f"(dst[4 * q + 1]) : "r"(a + 16 * q));
      dst[4 * q + 2] = dst[4 * q + 3] = 0.0f;
    } else {
      asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                   : "=f"(dst[4 * q]), "=f"(dst[4 * q + 1]), "=f"(dst[4 * q + 2]), "=f"(dst[4 * q + 3])
                   : "r"(a + 16 * q));
    }
  }
}

// Number of (i, j) taps through which window cell (Y, X) reaches the tile.
template <int KH, int KW, int S, int TH, int TW>
__host__ __device__ constexpr int cell_taps(int Y, int X) {
  int n = 0;
  for (int i = 0; i < KH; ++i)
    for (int j = 0; j < KW; ++j) {
      const int dy = Y - i, dx = X - j;
      if (dy >= 0 && dy % S == 0 && dy / S < TH && dx >= 0 && dx % S == 0 && dx / S < TW) ++n;
    }
  return n;
}

template <int KH, int KW, int S, int TH, int TW, int R, int WPH, int WPW, int BPITCH, int SPITCH,
          bool FAST, bool ROWSKIP, bool NOSKIP = false, bool RP = false>
__device__ __forceinline__ void ecr_channel(float (&acc)[TH][TW][R], const float (&wr)[KH * KW][R],
                                            const float* is, unsigned m0, unsigned m1) {
  static_assert(WPH * BPITCH <= 64, "window mask must fit 64 bits");
  constexpr int W4 = (WPW + 3) / 4;
  const unsigned long long mm = (static_cast<unsigned long long>(m1) << 32) | m0;
  // RP: row Y+1 is read while row Y runs (its load latency leaves the row
  // start), at the price of one wasted read per empty row
  float nrow[4 * W4];
  if constexpr (RP) lds_row_pinned<WPW>(nrow, is);
#pragma unroll
  for (int Y = 0; Y < WPH; ++Y) {
    float row[4 * W4];
    if constexpr (RP) {
#pragma unroll
      for (int q = 0; q < 4 * W4; ++q) row[q] = nrow[q];
      if (Y + 1 < WPH) lds_row_pinned<WPW>(nrow, is + (Y + 1) * SPITCH);
    }
    if constexpr (ROWSKIP) {
      if (((mm >> (Y * BPITCH)) & ((1ull << WPW) - 1ull)) == 0ull) continue;  // empty row
    }
    if constexpr (!RP) {
#pragma unroll
      for (int q = 0; q < W4; ++q) {
        const float4 v4 = *reinterpret_cast<const float4*>(is + Y * SPITCH + 4 * q);
        row[4 * q + 0] = v4.x;
        row[4 * q + 1] = v4.y;
        row[4 * q + 2] = v4.z;
        row[4 * q + 3] = v4.w;
      }
    }
#pragma unroll
    for (int X = 0; X < WPW; ++X) {
      const int b = Y * BPITCH + X;
      const bool nz = b < 32 ? ((m0 >> b) & 1u) : ((m1 >> (b - 32)) & 1u);
      if (NOSKIP || nz) {  // warp-uniform
#if SCONV_BODY_GUARD == 1
        if constexpr (!NOSKIP) SCONV_KEEP_BRANCH();
#elif SCONV_BODY_GUARD == 2
        if constexpr (!NOSKIP) __syncwarp();
#else
        // Sparse channels (the ROWSKIP variant) keep every cell behind its
        // branch: ptxas would otherwise if-convert the 1-3-tap border cells,
        // whose predicated FFMA2 cost their pipe cycles even when the cell is
        // zero -- most of a channel's time once density falls below ~0.2.
        // (Only small blocks need it: SCONV_GUARD_MIN_FFMA2 = the block size,
        // in FFMA2, from which ptxas keeps a block branched by itself.)
        if constexpr (ROWSKIP && !NOSKIP) {
          if (cell_taps<KH, KW, S, TH, TW>(Y, X) * R / 2 < SCONV_GUARD_MIN_FFMA2 &&
              cell_taps<KH, KW, S, TH, TW>(Y, X) * R / 2 > SCONV_GUARD_LOW_FFMA2)
            __syncwarp();
        }
#endif
        const float v = row[X];
#pragma unroll
        for (int i = 0; i < KH; ++i) {
          const int dy = Y - i;
          if (dy < 0 || dy % S != 0 || dy / S >= TH) continue;
#pragma unroll
          for (int j = 0; j < KW; ++j) {
            const int dx = X - j;
            if (dx < 0 || dx % S != 0 || dx / S >= TW) continue;
            if constexpr (R % 2 == 0 && (FAST || SCONV_EXACT2)) {
#pragma unroll
              for (int r = 0; r < R; r += 2) {
                if constexpr (FAST)
                  ffma2(acc[dy / S][dx / S][r], acc[dy / S][dx / S][r + 1], wr[i * KW + j][r],
                        wr[i * KW + j][r + 1], v);
                else
                  exact2(acc[dy / S][dx / S][r], acc[dy / S][dx / S][r + 1], wr[i * KW + j][r],
                         wr[i * KW + j][r + 1], v);
              }
            } else {
#pragma unroll
              for (int r = 0; r < R; ++r)
                acc[dy / S][dx / S][r] = mac<FAST>(acc[dy / S][dx / S][r], v, wr[i * KW + j][r]);
            }
          }
        }
      }
    }
  }
}

}  // namespace sconv_cu
