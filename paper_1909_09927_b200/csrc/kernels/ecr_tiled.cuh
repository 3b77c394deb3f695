// ecr_tiled.cuh -- the hot path: fused ECR compaction + sparse convolution
// (+ the PECR ReLU/pooling epilogue) for sm_100a CUDA cores.
//
// What the reference does per (image, filter) -- ecr_convert then
// ecr_spmv_conv (src/ecr.cpp:51-128), or pecr_convert then pecr_conv_pool
// (src/pecr.cpp:83-172) -- is done here for N images x K filters in one
// launch, and the compressed format never leaves the SM:
//
// * Input-stationary, lanes over output channels.  A CTA owns one image, an
//   (OTH x OTW) output tile and KT = 32*R*WK output channels.  Each warp owns
//   TH x TW outputs x 32*R channels; lane l owns channels l*R .. l*R+R-1 of
//   its warp's slice and keeps TH*TW*R fp32 accumulators in registers.
// * The input is streamed channel by channel (c ascending).  For channel c
//   the warp walks its (TH-1)*S+KH x (TW-1)*S+KW input patch in raster order;
//   every input value is the same for all 32 lanes (a broadcast LDS.128), so
//   the ECR zero test `v != 0` (ecr.cpp:84, -0.0 counts as zero) is a
//   warp-uniform branch: a zero costs one compare+branch for the whole warp,
//   a nonzero feeds up to KH*KW*R multiply-adds per lane against filter
//   weights held in registers.  This is the compaction of Alg. 1 done at
//   warp granularity on the filter-independent operand, shared by every
//   output channel instead of re-done per filter.
// * For any one output the terms arrive in (c, i, j) order -- the order in
//   which ecr_convert lays out f_data/k_data -- so with EXACT arithmetic
//   (rounded mul, rounded add) the result is bit-identical to
//   ecr_spmv_conv.  FAST uses FFMA in the same order.
// * Input patches and weight slabs for CC channels are staged into shared
//   memory with cp.async, double-buffered against compute.
// * P > 0 selects the PECR epilogue: P x P pooling with stride P folded over
//   the register tile in window raster order (ReLU folded into the max
//   initialised at +0.0, pecr.cpp:149), so only the pooled map is stored.
#pragma once

#include "common.cuh"

namespace sconv_cu {

template <int KH_, int KW_, int S_, int TH_, int TW_, int R_, int WK_, int WSY_, int WSX_, int CC_,
          int P_>
struct TiledCfg {
  static constexpr int KH = KH_, KW = KW_, S = S_, TH = TH_, TW = TW_, R = R_;
  static constexpr int WK = WK_, WSY = WSY_, WSX = WSX_, CC = CC_, P = P_;
  static constexpr int KK = KH * KW;
  static constexpr int NWARPS = WK * WSY * WSX;
  static constexpr int NT = 32 * NWARPS;
  static constexpr int KT = 32 * R * WK;        // output channels per CTA
  static constexpr int OTH = TH * WSY;          // output rows per CTA
  static constexpr int OTW = TW * WSX;          // output cols per CTA
  static constexpr int PH = (OTH - 1) * S + KH; // CTA input patch rows
  static constexpr int PW = (OTW - 1) * S + KW; // CTA input patch cols
  static constexpr int WPH = (TH - 1) * S + KH; // warp patch rows
  static constexpr int WPW = (TW - 1) * S + KW; // warp patch cols
  static constexpr int WPW4 = (WPW + 3) / 4 * 4;
  static constexpr int PWS_A = (PW + 3) / 4 * 4;
  static constexpr int PWS_B = (WSX - 1) * TW * S + WPW4;
  static constexpr int PWS = PWS_A > PWS_B ? PWS_A : PWS_B;  // smem row pitch
  static constexpr int IN_STAGE = CC * PH * PWS;  // floats
  static constexpr int W_STAGE = CC * KK * KT;    // floats
  static constexpr int STAGE = IN_STAGE + W_STAGE;
  static constexpr int SMEM_BYTES = 2 * STAGE * 4;
  static_assert((TW * S) % 4 == 0, "warp patch columns must stay 16B aligned");
  static_assert(R == 1 || R == 2 || R == 4 || R == 8, "R");
  static_assert(P == 0 || (TH % (P ? P : 1) == 0 && TW % (P ? P : 1) == 0), "pool tile");
};

struct TiledArgs {
  const float* x;   // [N][C][H][W]
  const float* wt;  // [C][KH*KW][K]  (filters transposed once per call)
  float* y;         // [N][K][OH][OW] or pooled [N][K][OH/P][OW/P]
  int C, H, W, K, OH, OW;
  int tiles_x;      // output tiles along x
  int mode;         // pool mode (P > 0)
};

template <int R>
__device__ __forceinline__ void lds_r(float (&dst)[R], const float* src) {
  if constexpr (R == 8) {
    const float4 a = *reinterpret_cast<const float4*>(src);
    const float4 b = *reinterpret_cast<const float4*>(src + 4);
    dst[0] = a.x; dst[1] = a.y; dst[2] = a.z; dst[3] = a.w;
    dst[4] = b.x; dst[5] = b.y; dst[6] = b.z; dst[7] = b.w;
  } else if constexpr (R == 4) {
    const float4 a = *reinterpret_cast<const float4*>(src);
    dst[0] = a.x; dst[1] = a.y; dst[2] = a.z; dst[3] = a.w;
  } else if constexpr (R == 2) {
    const float2 a = *reinterpret_cast<const float2*>(src);
    dst[0] = a.x; dst[1] = a.y;
  } else {
    dst[0] = src[0];
  }
}

template <class Cfg, bool FAST, int MINB>
__global__ void __launch_bounds__(Cfg::NT, MINB) ecr_tiled_kernel(const TiledArgs a) {
  constexpr int KH = Cfg::KH, KW = Cfg::KW, S = Cfg::S, TH = Cfg::TH, TW = Cfg::TW, R = Cfg::R;
  constexpr int KK = Cfg::KK, KT = Cfg::KT, CC = Cfg::CC, P = Cfg::P;
  constexpr int PH = Cfg::PH, PW = Cfg::PW, PWS = Cfg::PWS;
  constexpr int WPH = Cfg::WPH, WPW = Cfg::WPW, WPW4 = Cfg::WPW4;

  extern __shared__ float4 smem_raw[];
  float* smem = reinterpret_cast<float*>(smem_raw);

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wsx = warp % Cfg::WSX;
  const int wsy = (warp / Cfg::WSX) % Cfg::WSY;
  const int wk = warp / (Cfg::WSX * Cfg::WSY);

  const int n = blockIdx.z;
  const int k0 = blockIdx.y * KT;
  const int ty = blockIdx.x / a.tiles_x, tx = blockIdx.x % a.tiles_x;
  const int oy0 = ty * Cfg::OTH, ox0 = tx * Cfg::OTW;
  const int iy0 = oy0 * S, ix0 = ox0 * S;
  const int C = a.C, H = a.H, W = a.W, K = a.K;
  const float* xn = a.x + static_cast<size_t>(n) * C * H * W;

  // ---- cp.async staging of one CC-channel chunk -------------------------
  auto stage = [&](int c0, int buf) {
    float* in_s = smem + buf * Cfg::STAGE;
    float* w_s = in_s + Cfg::IN_STAGE;
    for (int idx = tid; idx < CC * PH * PW; idx += Cfg::NT) {
      const int c = idx / (PH * PW);
      const int rem = idx - c * (PH * PW);
      const int yy = rem / PW, xx = rem - (rem / PW) * PW;
      const int gc = c0 + c, gy = iy0 + yy, gx = ix0 + xx;
      const bool ok = gc < C && gy < H && gx < W;
      const float* src = ok ? xn + (static_cast<size_t>(gc) * H + gy) * W + gx : xn;
      cp_async4(in_s + (c * PH + yy) * PWS + xx, src, ok);
    }
    if ((K & 3) == 0) {
      for (int idx = tid; idx < CC * KK * (KT / 4); idx += Cfg::NT) {
        const int row = idx / (KT / 4), q = idx - row * (KT / 4);
        const int c = row / KK, ij = row - c * KK;
        const int gc = c0 + c, k = k0 + 4 * q;
        const bool ok = gc < C && k < K;
        const float* src = ok ? a.wt + (static_cast<size_t>(gc) * KK + ij) * K + k : a.wt;
        cp_async16(w_s + row * KT + 4 * q, src, ok);
      }
    } else {
      for (int idx = tid; idx < CC * KK * KT; idx += Cfg::NT) {
        const int row = idx / KT, q = idx - row * KT;
        const int c = row / KK, ij = row - c * KK;
        const int gc = c0 + c, k = k0 + q;
        const bool ok = gc < C && k < K;
        const float* src = ok ? a.wt + (static_cast<size_t>(gc) * KK + ij) * K + k : a.wt;
        cp_async4(w_s + row * KT + q, src, ok);
      }
    }
  };

  float acc[TH][TW][R];
#pragma unroll
  for (int i = 0; i < TH; ++i)
#pragma unroll
    for (int j = 0; j < TW; ++j)
#pragma unroll
      for (int r = 0; r < R; ++r) acc[i][j][r] = 0.0f;

  const int nchunks = (C + CC - 1) / CC;
  stage(0, 0);
  cp_async_commit();
  for (int ch = 0; ch < nchunks; ++ch) {
    if (ch + 1 < nchunks) stage((ch + 1) * CC, (ch + 1) & 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();

    const float* in_s = smem + (ch & 1) * Cfg::STAGE;
    const float* w_s = in_s + Cfg::IN_STAGE;
    const int cn = min(CC, C - ch * CC);
#pragma unroll 1
    for (int c = 0; c < cn; ++c) {
      float wr[KK][R];
      const float* wsrc = w_s + c * KK * KT + wk * 32 * R + lane * R;
#pragma unroll
      for (int ij = 0; ij < KK; ++ij) lds_r<R>(wr[ij], wsrc + ij * KT);

      const float* is = in_s + c * PH * PWS + (wsy * TH * S) * PWS + wsx * TW * S;
#pragma unroll
      for (int Y = 0; Y < WPH; ++Y) {
        float row[WPW4];
#pragma unroll
        for (int q = 0; q < WPW4 / 4; ++q) {
          const float4 v4 = *reinterpret_cast<const float4*>(is + Y * PWS + 4 * q);
          row[4 * q + 0] = v4.x;
          row[4 * q + 1] = v4.y;
          row[4 * q + 2] = v4.z;
          row[4 * q + 3] = v4.w;
        }
#pragma unroll
        for (int X = 0; X < WPW; ++X) {
          const float v = row[X];
          if (v != 0.0f) {  // warp-uniform: every lane holds the same v
#pragma unroll
            for (int i = 0; i < KH; ++i) {
              const int dy = Y - i;
              if (dy < 0 || dy % S != 0 || dy / S >= TH) continue;
#pragma unroll
              for (int j = 0; j < KW; ++j) {
                const int dx = X - j;
                if (dx < 0 || dx % S != 0 || dx / S >= TW) continue;
#pragma unroll
                for (int r = 0; r < R; ++r)
                  acc[dy / S][dx / S][r] = mac<FAST>(acc[dy / S][dx / S][r], v, wr[i * KW + j][r]);
              }
            }
          }
        }
      }
    }
    __syncthreads();
  }

  // ---- epilogue ----------------------------------------------------------
  const int kl = k0 + wk * 32 * R + lane * R;
  if constexpr (P == 0) {
    const int gx0 = ox0 + wsx * TW;
    const bool vec = (a.OW % 4 == 0) && (TW % 4 == 0);
#pragma unroll
    for (int oy = 0; oy < TH; ++oy) {
      const int gy = oy0 + wsy * TH + oy;
      if (gy >= a.OH) continue;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int k = kl + r;
        if (k >= K) continue;
        float* dst = a.y + ((static_cast<size_t>(n) * K + k) * a.OH + gy) * a.OW + gx0;
        if (vec) {
#pragma unroll
          for (int q = 0; q < TW / 4; ++q) {
            if (gx0 + 4 * q < a.OW) {
              *reinterpret_cast<float4*>(dst + 4 * q) =
                  make_float4(acc[oy][4 * q][r], acc[oy][4 * q + 1][r], acc[oy][4 * q + 2][r],
                              acc[oy][4 * q + 3][r]);
            }
          }
        } else {
#pragma unroll
          for (int ox = 0; ox < TW; ++ox)
            if (gx0 + ox < a.OW) dst[ox] = acc[oy][ox][r];
        }
      }
    }
  } else {
    const int PHo = a.OH / P, PWo = a.OW / P;
    const int py0 = (oy0 + wsy * TH) / P, px0 = (ox0 + wsx * TW) / P;
#pragma unroll
    for (int py = 0; py < TH / P; ++py) {
      if (py0 + py >= PHo) continue;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int k = kl + r;
        if (k >= K) continue;
        float* dst = a.y + ((static_cast<size_t>(n) * K + k) * PHo + py0 + py) * PWo + px0;
#pragma unroll
        for (int px = 0; px < TW / P; ++px) {
          if (px0 + px >= PWo) continue;
          PoolFold f;
#pragma unroll
          for (int u = 0; u < P; ++u)
#pragma unroll
            for (int v = 0; v < P; ++v) f.add(acc[py * P + u][px * P + v][r], a.mode);
          dst[px] = f.result(a.mode, P * P);
        }
      }
    }
  }
}

}  // namespace sconv_cu
