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
#include "ecr_body.cuh"

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

// Lane <-> channel map.  Lane l of a warp owns R output channels; for R >= 4
// they are {g*128 + 4l + q : g < R/4, q < 4} so each group of four is one
// conflict-free LDS.128 of a 512-byte weight row; for R < 4 they are
// {R*l + q}.
template <int R>
__device__ __forceinline__ int lane_chan(int lane, int r) {
  if constexpr (R >= 4) {
    return (r / 4) * 128 + lane * 4 + (r % 4);
  } else {
    return lane * R + r;
  }
}

template <int R>
__device__ __forceinline__ void lds_w(float (&dst)[R], const float* row, int lane) {
  if constexpr (R >= 4) {
#pragma unroll
    for (int g = 0; g < R / 4; ++g) {
      const float4 a = *reinterpret_cast<const float4*>(row + g * 128 + lane * 4);
      dst[4 * g + 0] = a.x;
      dst[4 * g + 1] = a.y;
      dst[4 * g + 2] = a.z;
      dst[4 * g + 3] = a.w;
    }
  } else if constexpr (R == 2) {
    const float2 a = *reinterpret_cast<const float2*>(row + lane * 2);
    dst[0] = a.x;
    dst[1] = a.y;
  } else {
    dst[0] = row[lane];
  }
}

// NOSKIP (calibration only) multiplies zeros too: identical results, dense work.
template <class Cfg, bool FAST, int MINB, bool NOSKIP = false>
__global__ void __launch_bounds__(Cfg::NT, MINB) ecr_tiled_kernel(const TiledArgs a) {
  constexpr int KH = Cfg::KH, KW = Cfg::KW, S = Cfg::S, TH = Cfg::TH, TW = Cfg::TW, R = Cfg::R;
  constexpr int KK = Cfg::KK, KT = Cfg::KT, CC = Cfg::CC, P = Cfg::P;
  constexpr int PH = Cfg::PH, PW = Cfg::PW, PWS = Cfg::PWS;
  constexpr int WPH = Cfg::WPH, WPW = Cfg::WPW, WPW4 = Cfg::WPW4;
  constexpr int NPOS = WPH * WPW;  // input positions a warp visits per channel
  static_assert(NPOS <= 64, "warp patch must fit two ballots");

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
  // Input patch: thread t owns patch elements t, t+NT, ... (fixed across
  // chunks), so the per-copy work is one address increment of H*W.
  constexpr int PE = PH * PW;
  constexpr int EPT = (PE + Cfg::NT - 1) / Cfg::NT;  // patch elements per thread
  const size_t plane = static_cast<size_t>(H) * W;
  const float* in_src[EPT];
  int in_dst[EPT];
  bool in_ok[EPT];
#pragma unroll
  for (int e = 0; e < EPT; ++e) {
    const int idx = tid + e * Cfg::NT;
    const int yy = idx / PW, xx = idx - (idx / PW) * PW;
    const int gy = iy0 + yy, gx = ix0 + xx;
    in_ok[e] = idx < PE && gy < H && gx < W;
    in_src[e] = in_ok[e] ? xn + static_cast<size_t>(gy) * W + gx : xn;
    in_dst[e] = yy * PWS + xx;
  }
  // Weights: rows (c, ij) of KT floats, contiguous per row in wt.
  constexpr int QW = KT / 4;                 // float4 per weight row
  constexpr int RSTEP = Cfg::NT / QW;        // rows covered per pass
  static_assert(Cfg::NT % QW == 0, "thread count must cover whole weight rows");
  const int wq = tid % QW, wrow0 = tid / QW;
  const bool wk_ok = k0 + 4 * wq < K;

  auto stage = [&](int c0, int buf) {
    float* in_s = smem + buf * Cfg::STAGE;
    float* w_s = in_s + Cfg::IN_STAGE;
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      if (tid + e * Cfg::NT < PE) {
        const float* src = in_src[e] + c0 * plane;
        float* dst = in_s + in_dst[e];
#pragma unroll
        for (int c = 0; c < CC; ++c) {
          const bool ok = in_ok[e] && c0 + c < C;
          cp_async4(dst + c * PH * PWS, ok ? src + c * plane : xn, ok);
        }
      }
    }
    const int rows_left = (C - c0) * KK;  // valid weight rows from c0
    if ((K & 3) == 0) {
      const float* wsrc = a.wt + static_cast<size_t>(c0) * KK * K + k0 + 4 * wq;
      float* wdst = w_s + 4 * wq;
#pragma unroll 4
      for (int row = wrow0; row < CC * KK; row += RSTEP) {
        const bool ok = wk_ok && row < rows_left;
        cp_async16(wdst + row * KT, ok ? wsrc + static_cast<size_t>(row) * K : a.wt, ok);
      }
    } else {
      for (int idx = tid; idx < CC * KK * KT; idx += Cfg::NT) {
        const int row = idx / KT, q = idx - row * KT;
        const bool ok = row < rows_left && k0 + q < K;
        const float* src = ok ? a.wt + (static_cast<size_t>(c0) * KK + row) * K + k0 + q : a.wt;
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

  // Lane l tests positions l and l+32 of the warp patch; the two ballots are
  // the ECR nonzero index of this (channel, patch), uniform across the warp.
  const int wbase = (wsy * TH * S) * PWS + wsx * TW * S;
  const int q0 = lane, q1 = lane + 32;
  const int off0 = wbase + (q0 / WPW) * PWS + q0 % WPW;
  const int off1 = q1 < NPOS ? wbase + (q1 / WPW) * PWS + q1 % WPW : wbase;

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
    const float* ic = in_s;
    const float* wsrc = w_s + wk * 32 * R;
#pragma unroll 1
    for (int c = 0; c < cn; ++c, ic += PH * PWS, wsrc += KK * KT) {
      const unsigned m0 = __ballot_sync(kFull, ic[off0] != 0.0f);
      const unsigned m1 = NPOS > 32 ? __ballot_sync(kFull, q1 < NPOS && ic[off1] != 0.0f) : 0u;

      float wr[KK][R];
#pragma unroll
      for (int ij = 0; ij < KK; ++ij) lds_w<R>(wr[ij], wsrc + ij * KT, lane);

      const float* is = ic + wbase;
      if (!NOSKIP && (__popc(m0) + __popc(m1)) * 4 <= NPOS)
        ecr_channel<KH, KW, S, TH, TW, R, WPH, WPW, WPW, PWS, FAST, true>(acc, wr, is, m0, m1);
      else
        ecr_channel<KH, KW, S, TH, TW, R, WPH, WPW, WPW, PWS, FAST, false, NOSKIP>(acc, wr, is, m0,
                                                                                 m1);
    }
    __syncthreads();
  }

  // ---- epilogue ----------------------------------------------------------
  const int kw0 = k0 + wk * 32 * R;
  if constexpr (P == 0) {
    if (a.mode) relu_tile(acc);  // fused Activation::kRelu (forward)
    const int gx0 = ox0 + wsx * TW;
    const bool vec = (a.OW % 4 == 0) && (TW % 4 == 0);
#pragma unroll
    for (int oy = 0; oy < TH; ++oy) {
      const int gy = oy0 + wsy * TH + oy;
      if (gy >= a.OH) continue;
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int k = kw0 + lane_chan<R>(lane, r);
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
        const int k = kw0 + lane_chan<R>(lane, r);
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
