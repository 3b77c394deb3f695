// ecr_isc.cuh -- the hot path, v4: fused ECR compaction + sparse convolution
// (+ the PECR ReLU/pooling epilogue) as a row-input-stationary column walk,
// FAST arithmetic only (3x3, stride 1).
//
// Why a new loop nest.  In v3 (ecr_ws.cuh) a warp owns a TH x TW output tile
// and visits every cell of its (TH+2) x (TW+2) input window once per channel;
// the zero skip is one warp-uniform branch per cell, and on B200 a branch
// costs ~4 SMSP issue cycles whether or not it is taken
// (tools/micro/branch_cost.cu, ubranch_cost.cu).  Border cells of the window
// feed only 1-3 of their 9 taps, so a 4x4 tile pays 36 branches for 144
// (cell, tap) pairs and the branch cost caps the kernel near 55% of FFMA issue.
//
// v4 makes the walk input-stationary along y: a warp owns a column of TW
// outputs and walks DOWN the image in steps of 4 input rows.  In a step it
// visits the 4 x (TW+2) cells of rows 4r..4r+3 and adds each into every
// output row it touches (rows 4r-2..4r+3 -> acc rows 0..5), so every cell
// feeds all 3 of its vertical taps: 24 branches for the same 144 (cell, tap)
// pairs.  After the C channels of a step, acc rows 0..3 (outputs 4r-2..4r+1)
// are complete and are stored (or pooled); rows 4,5 still miss the next
// step's cells and are carried in registers into rows 0,1.  The pre-pool
// output still never reaches HBM.
//
// The column is cut into segments of S steps so the grid fills the GPU; a
// segment other than the first starts with one warm-up step whose complete
// rows belong to the previous segment (they are not stored) and whose carried
// rows become the segment's first rows.  Every segment runs L = S + 1 steps
// (steps past the map read zero-filled cells: they cost the mask test only),
// so all warps of a CTA stay in lockstep with the producer warp.
//
// Arithmetic: FFMA2, and per output the terms of one step arrive channel by
// channel, so an output's sum is (carry from the step above) + (this step) --
// a fixed order, independent of the segmentation and of the grid, hence
// deterministic, but not the reference's (c, i, j) order: FAST tolerance
// (|d| <= 1e-5 + 1e-5|ref|).  EXACT calls stay on v3.
#pragma once

#include <cuda.h>

#include "common.cuh"
#include "ecr_ws.cuh"  // mbarrier / TMA helpers, ws_lds_w, ws_lane_chan

namespace sconv_cu {

template <int TW_, int R_, int WPC_, int CC_, int NS_, int P_>
struct IscCfg {
  static constexpr int TW = TW_, R = R_, WPC = WPC_, CC = CC_, NS = NS_, P = P_;
  static constexpr int KK = 9;
  static constexpr int SR = 4;                       // input rows per step
  static constexpr int KT = 32 * R;                  // output channels per CTA
  static constexpr int WPW = TW + 2;                 // cells per warp row
  static constexpr int PITCH = WPW <= 8 ? 8 : 16;    // sub-patch row pitch (floats)
  static constexpr int PATCH = SR * PITCH;           // floats per (warp, channel)
  static constexpr int NCELL = SR * WPW;
  static constexpr int IN_STAGE = (WPC * CC * PATCH + 31) / 32 * 32;
  static constexpr int W_STAGE = CC * KK * KT;
  static constexpr int STAGE = IN_STAGE + W_STAGE;
  static constexpr int NT = 32 * (WPC + 1);
  static constexpr int SMEM_BYTES = NS * STAGE * 4 + 2 * NS * 8;
  static constexpr int CELLS = WPC * NCELL;
  static constexpr int CELLS_PER_LANE = (CELLS + 31) / 32;
  static constexpr bool TWO = PATCH > 32;            // two ballots per channel
  static_assert(PATCH <= 64, "mask must fit 64 bits");
  static_assert(R == 2 || R == 4, "R");
  static_assert(TW % 4 == 0, "TW");
  static_assert(P == 0 || P == 2, "pool");
  static_assert((IN_STAGE * 4) % 128 == 0 && (STAGE * 4) % 128 == 0, "TMA alignment");
  static constexpr unsigned W_BYTES = W_STAGE * 4;
};

struct IscArgs {
  const float* x;   // [N][C][H][W]
  float* y;         // [N][K][OH][OW] or pooled [N][K][OH/2][OW/2]
  int N, C, H, W, K, OH, OW;
  int tiles_x;      // column tiles per image
  int segs;         // segments per column
  int S;            // owned steps per segment (segment 0 owns S + 1)
  int total;        // N * segs * tiles_x work items
  int mode;         // pool mode (P > 0)
};

// One channel: every nonzero cell (Y, X) of the warp's 4 x (TW+2) patch is
// multiplied into acc[Y-i+2][X-j] for the taps (i, j) with 0 <= X-j < TW.
// VL selects how the cell value reaches the lanes: 0 = the patch row is read
// once per row with LDS.128 (registers), 1 = one broadcast LDS per nonzero
// cell, 2 = a shuffle from the lane that tested the cell for the ballot.
#ifndef SCONV_ISC_GUARD
#define SCONV_ISC_GUARD 1
#endif
#ifndef SCONV_ISC_VL
#define SCONV_ISC_VL 0
#endif
template <class Cfg>
__device__ __forceinline__ void isc_channel(float (&acc)[6][Cfg::TW][Cfg::R],
                                            const float (&wr)[9][Cfg::R], const float* is,
                                            unsigned m0, unsigned m1, float c0v, float c1v) {
  constexpr int TW = Cfg::TW, R = Cfg::R, WPW = Cfg::WPW, PITCH = Cfg::PITCH;
  constexpr int W4 = (WPW + 3) / 4;
  constexpr int VL = SCONV_ISC_VL;
#pragma unroll
  for (int Y = 0; Y < Cfg::SR; ++Y) {
    float row[4 * W4];
    if constexpr (VL == 0) {
#pragma unroll
      for (int q = 0; q < W4; ++q) {
        const float4 v4 = *reinterpret_cast<const float4*>(is + Y * PITCH + 4 * q);
        row[4 * q + 0] = v4.x;
        row[4 * q + 1] = v4.y;
        row[4 * q + 2] = v4.z;
        row[4 * q + 3] = v4.w;
      }
    }
#pragma unroll
    for (int X = 0; X < WPW; ++X) {
      const int b = Y * PITCH + X;
      const bool nz = b < 32 ? ((m0 >> b) & 1u) : ((m1 >> (b - 32)) & 1u);
      if (nz) {  // warp-uniform
#if SCONV_ISC_GUARD
        __syncwarp();  // keeps the block behind its branch (no if-conversion)
#endif
        float v;
        if constexpr (VL == 0) v = row[X];
        else if constexpr (VL == 1) v = is[b];
        else v = __shfl_sync(kFull, b < 32 ? c0v : c1v, b & 31);
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          const int u = Y - i + 2;
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            const int ox = X - j;
            if (ox < 0 || ox >= TW) continue;
#pragma unroll
            for (int r = 0; r < R; r += 2)
              ffma2(acc[u][ox][r], acc[u][ox][r + 1], wr[i * 3 + j][r], wr[i * 3 + j][r + 1], v);
          }
        }
      }
    }
  }
}

template <class Cfg>
__global__ void __launch_bounds__(Cfg::NT, 1)
    ecr_isc_kernel(const IscArgs a, const __grid_constant__ CUtensorMap wmap) {
  constexpr int TW = Cfg::TW, R = Cfg::R, KT = Cfg::KT, CC = Cfg::CC, NS = Cfg::NS, P = Cfg::P;
  constexpr int WPC = Cfg::WPC, WPW = Cfg::WPW, PITCH = Cfg::PITCH, PATCH = Cfg::PATCH;
  constexpr int SR = Cfg::SR, KK = Cfg::KK;

  extern __shared__ float4 smem_raw[];
  float* smem = reinterpret_cast<float*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NS * Cfg::STAGE);
  uint64_t* empty = full + NS;

  const int tid = threadIdx.x;
  const int warp = __shfl_sync(kFull, tid >> 5, 0), lane = tid & 31;
  // K-blocks vary fastest over the linear grid: CTAs sharing a patch run together
  const int kblocks = (a.K + KT - 1) / KT;
  const int cta = blockIdx.x / kblocks;
  const int k0 = (blockIdx.x - cta * kblocks) * KT;
  const int C = a.C, H = a.H, W = a.W, K = a.K;
  const int nchunks = (C + CC - 1) / CC;
  const int L = a.S + 1;           // steps per warp
  const int total_chunks = L * nchunks;

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 33);  // 32 cp.async lane arrivals + the TMA expect_tx arrival
      mbar_init(&empty[s], WPC);
    }
  }
  __syncthreads();

  if (warp == WPC) {
    // ------------------------------ producer ------------------------------
    const size_t plane = static_cast<size_t>(H) * W;
    int src_off[Cfg::CELLS_PER_LANE];  // offset of the cell in step 0 (channel 0)
    int row0[Cfg::CELLS_PER_LANE];     // its input row in step 0
    int dst_off[Cfg::CELLS_PER_LANE];
    bool ok[Cfg::CELLS_PER_LANE];
#pragma unroll
    for (int e = 0; e < Cfg::CELLS_PER_LANE; ++e) {
      const int q = lane + 32 * e;
      const int wi = q / Cfg::NCELL, pos = q - wi * Cfg::NCELL;
      const int Y = pos / WPW, X = pos - (pos / WPW) * WPW;
      const int t = cta * WPC + wi;
      const int tx = t % a.tiles_x, rest = t / a.tiles_x;
      const int sg = rest % a.segs, n = rest / a.segs;
      const int first = sg == 0 ? 0 : sg * a.S;  // first step of the segment
      const int iy = first * SR + Y, ix = tx * TW + X;
      ok[e] = q < Cfg::CELLS && t < a.total && ix < W;
      row0[e] = iy;
      src_off[e] = ok[e] ? static_cast<int>((static_cast<size_t>(n) * C * H) * W + ix) : 0;
      dst_off[e] = (wi * CC) * PATCH + Y * PITCH + X;
    }
    if (lane == 0)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&wmap)) : "memory");
    for (int g = 0; g < total_chunks; ++g) {
      const int s = g % NS;
      const int l = g / nchunks, k = g - l * nchunks;
      if (g >= NS) mbar_wait_sleep(&empty[s], ((g / NS) + 1) & 1);
      float* in_s = smem + s * Cfg::STAGE;
      float* w_s = in_s + Cfg::IN_STAGE;
      const int c0 = k * CC;
#pragma unroll
      for (int e = 0; e < Cfg::CELLS_PER_LANE; ++e) {
        if (lane + 32 * e < Cfg::CELLS) {
          const int iy = row0[e] + l * SR;
          const bool rv = ok[e] && iy < H;
#pragma unroll
          for (int ch = 0; ch < CC; ++ch) {
            const bool v = rv && c0 + ch < C;
            const float* src = v ? a.x + src_off[e] + (static_cast<size_t>(c0 + ch) * H + iy) * W : a.x;
            cp_async4(in_s + dst_off[e] + ch * PATCH, src, v);
          }
        }
      }
      if (lane == 0) {
        mbar_arrive_expect_tx(&full[s], Cfg::W_BYTES);
        tma_load_3d(w_s, &wmap, k0, 0, c0, &full[s]);
      }
      mbar_arrive_cp_async(&full[s]);
    }
    cp_async_wait<0>();
    return;
  }

  // ------------------------------- consumers -------------------------------
  const int t = cta * WPC + warp;
  const bool active = t < a.total;
  const int tx = t % a.tiles_x, rest = t / a.tiles_x;
  const int sg = rest % a.segs, n = active ? rest / a.segs : 0;
  const int first = sg == 0 ? 0 : sg * a.S;
  const int ox0 = tx * TW;

  float acc[6][TW][R];
#pragma unroll
  for (int u = 0; u < 6; ++u)
#pragma unroll
    for (int j = 0; j < TW; ++j)
#pragma unroll
      for (int r = 0; r < R; ++r) acc[u][j][r] = 0.0f;

  const bool t0 = (lane % PITCH) < WPW && (lane / PITCH) < SR;
  const bool t1 = ((lane + 32) % PITCH) < WPW && ((lane + 32) / PITCH) < SR;

  int g = 0;
  for (int l = 0; l < L; ++l) {
    for (int k = 0; k < nchunks; ++k, ++g) {
      const int s = g % NS;
      mbar_wait(&full[s], (g / NS) & 1);
      if (active) {
        const float* ic = smem + s * Cfg::STAGE + warp * CC * PATCH;
        const float* wsrc = smem + s * Cfg::STAGE + Cfg::IN_STAGE;
        const int cn = min(CC, C - k * CC);
#pragma unroll 1
        for (int c = 0; c < cn; ++c, ic += PATCH, wsrc += KK * KT) {
          const float c0v = ic[lane];
          const float c1v = Cfg::TWO ? ic[lane + 32] : 0.0f;
          const unsigned m0 = __ballot_sync(kFull, t0 && c0v != 0.0f);
          const unsigned m1 = Cfg::TWO ? __ballot_sync(kFull, t1 && c1v != 0.0f) : 0u;
          float wr[KK][R];
#pragma unroll
          for (int ij = 0; ij < KK; ++ij) ws_lds_w<R>(wr[ij], wsrc + ij * KT, lane);
          isc_channel<Cfg>(acc, wr, ic, m0, m1, c0v, c1v);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (!active) continue;

    // ---- step epilogue: acc rows 0..3 = output rows oy0..oy0+3 complete ----
    const int step = first + l;
    const int oy0 = step * SR - 2;
    const bool store = !(sg > 0 && l == 0);  // warm-up rows belong to the segment above
    if (store) {
      if constexpr (P == 0) {
        const bool vec = a.OW % 4 == 0;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int kk = k0 + ws_lane_chan<R>(lane, r);
          if (kk >= K) continue;
          float* dst = a.y + ((static_cast<size_t>(n) * K + kk) * a.OH) * a.OW + ox0;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int oy = oy0 + u;
            if (oy < 0 || oy >= a.OH) continue;
            if (vec) {
#pragma unroll
              for (int q = 0; q < TW / 4; ++q)
                if (ox0 + 4 * q < a.OW)
                  *reinterpret_cast<float4*>(dst + static_cast<size_t>(oy) * a.OW + 4 * q) =
                      make_float4(acc[u][4 * q][r], acc[u][4 * q + 1][r], acc[u][4 * q + 2][r],
                                  acc[u][4 * q + 3][r]);
            } else {
#pragma unroll
              for (int ox = 0; ox < TW; ++ox)
                if (ox0 + ox < a.OW) dst[static_cast<size_t>(oy) * a.OW + ox] = acc[u][ox][r];
            }
          }
        }
      } else {
        const int PHo = a.OH / 2, PWo = a.OW / 2;
        const int px0 = ox0 / 2;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int kk = k0 + ws_lane_chan<R>(lane, r);
          if (kk >= K) continue;
          float* dst = a.y + ((static_cast<size_t>(n) * K + kk) * PHo) * PWo + px0;
#pragma unroll
          for (int pu = 0; pu < 2; ++pu) {
            const int py = (oy0 >> 1) + pu;  // oy0 is even
            if (py < 0 || py >= PHo) continue;
#pragma unroll
            for (int px = 0; px < TW / 2; ++px) {
              if (px0 + px >= PWo) continue;
              PoolFold f;
#pragma unroll
              for (int du = 0; du < 2; ++du)
#pragma unroll
                for (int dv = 0; dv < 2; ++dv) f.add(acc[2 * pu + du][2 * px + dv][r], a.mode);
              dst[static_cast<size_t>(py) * PWo + px] = f.result(a.mode, 4);
            }
          }
        }
      }
    }
    // carry rows 4,5 (outputs oy0+4, oy0+5) into rows 0,1
#pragma unroll
    for (int j = 0; j < TW; ++j)
#pragma unroll
      for (int r = 0; r < R; ++r) {
        acc[0][j][r] = acc[4][j][r];
        acc[1][j][r] = acc[5][j][r];
        acc[2][j][r] = 0.0f;
        acc[3][j][r] = 0.0f;
        acc[4][j][r] = 0.0f;
        acc[5][j][r] = 0.0f;
      }
  }
}

}  // namespace sconv_cu
