// smallc.cuh -- ECR / PECR for maps with few input channels (VGG conv1_1:
// C = 3 -> K = 64 at 224x224), the one VGG-19 layer bound by HBM rather than
// FP32 issue (861 MB moved for 3.3 GFLOP).
//
// With C = 3 a CTA has almost no reduction to pipeline, so the v2/v3 staging
// machinery (CTA-wide shared-memory chunks, producer warp, barriers) is pure
// latency, and their 128-180-register tiles leave 2 warps per scheduler.
// Here every warp is independent: it owns one 4x4 output tile x 64 output
// channels (R = 2), reads its 6x6 input window of each channel straight from
// global memory (L1/L2; neighbouring tiles share halos), parks it in a
// private 48-float shared-memory slot, and runs the same per-channel body as
// v2/v3 (ecr_body.cuh: ballot compaction + warp-uniform zero skip, terms of
// each output in (c, i, j) order, so EXACT stays bit-identical).  No
// __syncthreads in the channel loop.  ECR: 64 registers (16-20 B of spills), 4 CTAs =
// 8 warps per scheduler: conv1_1 345 -> 333 us vs 3 CTAs at <= 80 registers;
// PECR keeps 3 CTAs (its pool epilogue spills ~100 B at 64).
#pragma once

#include "common.cuh"
#include "ecr_body.cuh"

namespace sconv_cu {

struct SmallCArgs {
  const float* x;   // [N][C][H][W]
  const float* wt;  // [C][9][Kp]  (transposed filters)
  float* y;         // [N][K][OH][OW] or pooled [N][K][OH/2][OW/2]
  int N, C, H, W, K, Kp, OH, OW;
  int tiles_x, tiles_per_img, total_tiles;
  int mode;         // P != 0: pool mode; P == 0: fused ReLU flag
  // P == -1 (any pool): pool geometry, pooled map, conv-output tile strides
  // (see WsArgs in ecr_ws.cuh); P >= 0: tsy = tsx = 4
  int pw = 0, ph = 0, ps = 1, PHo = 0, PWo = 0, tsy = 4, tsx = 4;
};

template <int P, bool FAST>
__global__ void __launch_bounds__(256, P == 0 ? 4 : 3) ecr_smallc_kernel(const SmallCArgs a) {
  constexpr int TH = 4, TW = 4, R = 2, KT = 64, WPH = 6, WPW = 6, PITCH = 8;
  __shared__ __align__(16) float win[8][WPH * PITCH];
  const int warp = __shfl_sync(kFull, threadIdx.x >> 5, 0), lane = threadIdx.x & 31;
  const int t = blockIdx.x * 8 + warp;
  if (t >= a.total_tiles) return;  // whole warp exits together
  const int k0 = blockIdx.y * KT;
  const int n = t / a.tiles_per_img, tt = t - n * a.tiles_per_img;
  const int ty = tt / a.tiles_x, tx = tt - ty * a.tiles_x;
  const int oy0 = ty * a.tsy, ox0 = tx * a.tsx;

  // lane l stages window cells l and l + 32 (cell q -> (q / 6, q % 6))
  const int q1 = lane + 32;
  const int y_a = oy0 + lane / WPW, x_a = ox0 + lane % WPW;
  const int y_b = oy0 + q1 / WPW, x_b = ox0 + q1 % WPW;
  const bool in_a = lane < WPH * WPW && y_a < a.H && x_a < a.W;
  const bool in_b = q1 < WPH * WPW && y_b < a.H && x_b < a.W;
  const size_t plane = static_cast<size_t>(a.H) * a.W;
  const float* xn = a.x + static_cast<size_t>(n) * a.C * plane;
  const size_t off_a = static_cast<size_t>(y_a) * a.W + x_a, off_b = static_cast<size_t>(y_b) * a.W + x_b;
  float* w_s = win[warp];
  const int s_a = (lane / WPW) * PITCH + lane % WPW, s_b = (q1 / WPW) * PITCH + q1 % WPW;
  // ballot bit of a cell: Y * PITCH + X (the layout ecr_channel expects)
  const bool t0 = (lane % PITCH) < WPW && (lane / PITCH) < WPH;
  const bool t1 = ((lane + 32) % PITCH) < WPW && ((lane + 32) / PITCH) < WPH;

  float acc[TH][TW][R];
#pragma unroll
  for (int i = 0; i < TH; ++i)
#pragma unroll
    for (int j = 0; j < TW; ++j)
#pragma unroll
      for (int r = 0; r < R; ++r) acc[i][j][r] = 0.0f;

#pragma unroll 1
  for (int c = 0; c < a.C; ++c) {
    const float va = in_a ? __ldg(xn + c * plane + off_a) : 0.0f;
    const float vb = in_b ? __ldg(xn + c * plane + off_b) : 0.0f;
    if (lane < WPH * WPW) w_s[s_a] = va;
    if (q1 < WPH * WPW) w_s[s_b] = vb;
    float wr[9][R];
    const float* wc = a.wt + static_cast<size_t>(c) * 9 * a.Kp + k0 + lane * R;
#pragma unroll
    for (int ij = 0; ij < 9; ++ij) {
      const float2 p = __ldg(reinterpret_cast<const float2*>(wc + ij * a.Kp));
      wr[ij][0] = p.x;
      wr[ij][1] = p.y;
    }
    __syncwarp();
    const unsigned m0 = __ballot_sync(kFull, t0 && w_s[lane] != 0.0f);
    const unsigned m1 = __ballot_sync(kFull, t1 && w_s[lane + 32] != 0.0f);
    ecr_channel<3, 3, 1, TH, TW, R, WPH, WPW, PITCH, PITCH, FAST, false>(acc, wr, w_s, m0, m1);
    __syncwarp();  // the slot is rewritten by the next channel
  }

  if constexpr (P < 0) {
    // any pool geometry: the conv tile goes through the warp's slice of shared
    // memory and each lane folds the pool windows of its channels in window
    // raster order (pecr_conv_pool, src/pecr.cpp:147-167)
    __shared__ float ptile[8][TH * TW * KT];
    float* eb = ptile[warp];
#pragma unroll
    for (int u = 0; u < TH; ++u)
#pragma unroll
      for (int v = 0; v < TW; ++v)
#pragma unroll
        for (int r = 0; r < R; ++r) eb[(u * TW + v) * KT + lane * R + r] = acc[u][v][r];
    __syncwarp();
    const int PTH = (TH - a.ph) / a.ps + 1, PTW = (TW - a.pw) / a.ps + 1;
    const int py0 = ty * PTH, px0 = tx * PTW;
    for (int r = 0; r < R; ++r) {
      const int ch = lane * R + r, kk = k0 + ch;
      if (kk >= a.K) continue;
      float* dst = a.y + (static_cast<size_t>(n) * a.K + kk) * a.PHo * a.PWo;
      for (int py = 0; py < PTH && py0 + py < a.PHo; ++py)
        for (int px = 0; px < PTW && px0 + px < a.PWo; ++px) {
          PoolFold f;
          const float* wb = eb + (py * a.ps * TW + px * a.ps) * KT + ch;
          for (int du = 0; du < a.ph; ++du)
            for (int dv = 0; dv < a.pw; ++dv) f.add(wb[(du * TW + dv) * KT], a.mode);
          dst[(py0 + py) * a.PWo + px0 + px] = f.result(a.mode, a.ph * a.pw);
        }
    }
  } else if constexpr (P == 0) {
    if (a.mode) relu_tile(acc);  // fused Activation::kRelu (forward)
    // When the CTA's 8 tiles are one 32-wide strip of a row band, the tile is
    // transposed through shared memory so every warp store writes whole
    // 128-byte lines of one channel row (lanes over channels would write 32
    // scattered 16-byte pieces per instruction: ncu, conv1_1, L1/L2 at 64%
    // throughput with DRAM at 20%).
    if (a.tiles_x % 8 == 0 && a.OW % 4 == 0 && k0 + KT <= a.K) {
      constexpr int CP = 4 * 32 + 4;  // channel pitch (floats): odd in float4 units
      __shared__ __align__(16) float otile[KT * CP];
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int oy = 0; oy < TH; ++oy)
          *reinterpret_cast<float4*>(&otile[(r * 32 + lane) * CP + oy * 32 + warp * 4]) =
              make_float4(acc[oy][0][r], acc[oy][1][r], acc[oy][2][r], acc[oy][3][r]);
      __syncthreads();
      const int strip_x = ox0 - warp * 4;  // first column of the CTA strip
      const int p = lane >> 3, q = lane & 7;
#pragma unroll 2
      for (int it = 0; it < KT * TH / (4 * 8); ++it) {
        const int item = (it * 8 + warp) * 4 + p;  // (channel, row) pair
        const int kk = item >> 2, oy = item & 3;
        if (oy0 + oy >= a.OH) continue;
        const int sl = (kk & 1) * 32 + (kk >> 1);   // smem slot of channel kk
        const float4 v = *reinterpret_cast<const float4*>(&otile[sl * CP + oy * 32 + q * 4]);
        *reinterpret_cast<float4*>(a.y + ((static_cast<size_t>(n) * a.K + k0 + kk) * a.OH + oy0 + oy) *
                                             a.OW + strip_x + q * 4) = v;
      }
      return;
    }
    const bool vec = a.OW % 4 == 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int kk = k0 + lane * R + r;
      if (kk >= a.K) continue;
      float* dst = a.y + ((static_cast<size_t>(n) * a.K + kk) * a.OH + oy0) * a.OW + ox0;
#pragma unroll
      for (int oy = 0; oy < TH; ++oy) {
        if (oy0 + oy >= a.OH) continue;
        if (vec && ox0 + 4 <= a.OW) {
          *reinterpret_cast<float4*>(dst + oy * a.OW) =
              make_float4(acc[oy][0][r], acc[oy][1][r], acc[oy][2][r], acc[oy][3][r]);
        } else {
#pragma unroll
          for (int ox = 0; ox < TW; ++ox)
            if (ox0 + ox < a.OW) dst[oy * a.OW + ox] = acc[oy][ox][r];
        }
      }
    }
  } else {
    const int PHo = a.OH / 2, PWo = a.OW / 2, py0 = oy0 / 2, px0 = ox0 / 2;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int kk = k0 + lane * R + r;
      if (kk >= a.K) continue;
      float* dst = a.y + ((static_cast<size_t>(n) * a.K + kk) * PHo + py0) * PWo + px0;
#pragma unroll
      for (int py = 0; py < 2; ++py) {
        if (py0 + py >= PHo) continue;
#pragma unroll
        for (int px = 0; px < 2; ++px) {
          if (px0 + px >= PWo) continue;
          PoolFold f;
#pragma unroll
          for (int u = 0; u < 2; ++u)
#pragma unroll
            for (int v = 0; v < 2; ++v) f.add(acc[2 * py + u][2 * px + v][r], a.mode);
          dst[py * PWo + px] = f.result(a.mode, 4);
        }
      }
    }
  }
}

}  // namespace sconv_cu
