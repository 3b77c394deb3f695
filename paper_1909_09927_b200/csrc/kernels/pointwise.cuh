// pointwise.cuh -- 1x1 stride-1 ECR conv as a dense, ordered SIMT GEMM.
//
// For a 1x1 window every window is a single cell per channel, so the
// zero-skipping kernels pay a ballot, a mask test and a branch for at most
// one tap per (cell, channel) -- on the GoogLeNet 1x1 branches (BASELINE
// config 2) that chain, not the arithmetic, set the time.  Here the layer is
// Y[n] (K x P) = W (K x C) * X[n] (C x P), P = H*W, computed densely:
//
// * order: every output accumulates its terms over c = 0 .. C-1, one after
//   the other, exactly like ecr_spmv_conv's per-window loop
//   (src/ecr.cpp:117-120) -- no split of the reduction;
// * zero cells: the reference skips them (src/ecr.cpp:84, v != 0 incl. -0);
//   here they are multiplied.  With a finite weight w the product w * (+-0)
//   is +-0 and acc + (+-0) == acc, because acc is never -0 (it starts at +0,
//   and a round-to-nearest sum is -0 only when both addends are), so the
//   result is bit-identical.  A stage whose weights hold an Inf / NaN (whose
//   product with 0 is NaN) runs with the zero cells predicated off instead;
// * EXACT: rounded product then rounded sum (exact2: FFMA2 with a -0 addend + FADD2);
//   FAST: FFMA2.
//
// Tiling: CTA BM output channels x BN output columns (columns = the N*P
// (image, pixel) pairs), BK = 8 channels per stage in a 4-stage cp.async
// ring (these layers are short and the channel chain is serial, so the
// copies must run well ahead); each thread holds TM x TN accumulators (rows
// ty*4.. and, for TM = 8, BM/2 + ty*4.. (TM = 2: ty*2..); columns tx*4..
// and, for TN = 8, BN/2 + tx*4..: conflict-free float4 shared reads).
// Smaller thread tiles put more warps on the grids too small to fill the
// GPU (pw_tile in sconv_cuda.cu).
#pragma once

#include "common.cuh"

namespace sconv_cu {

struct PwArgs {
  const float* x;   // [N][C][P]
  const float* wt;  // [C][Kp]  (the transposed filters of the tiled kernels, KK = 1)
  float* y;         // [N][K][P]
  int N, C, P, K, Kp;
  long long cols;   // N * P
  int relu;         // fused ReLU (forward)
};

template <int BM, int BN, int TM, int TN>
struct PwCfg {
  static constexpr int BK = 8, NS = 4;
  static constexpr int TX = BN / TN, TY = BM / TM, NT = TX * TY;
  static constexpr int XPER = BK * BN / NT;  // X elements a thread copies per stage
  static constexpr int WCH = BK * BM / 4;                 // 16-byte weight chunks per stage
  static constexpr int WPER = (WCH + NT - 1) / NT;        // ... a thread copies (or checks)
  static_assert(WCH % NT == 0 || WCH < NT, "weight chunks");
  static_assert(NT % BN == 0, "column loader: one column per thread");
};

template <int BM, int BN, int TM, int TN, bool FAST>
__global__ void __launch_bounds__(PwCfg<BM, BN, TM, TN>::NT)
    pw_gemm_kernel(const PwArgs a) {
  using Cfg = PwCfg<BM, BN, TM, TN>;
  constexpr int BK = Cfg::BK, TX = Cfg::TX, NT = Cfg::NT, NS = Cfg::NS;
  __shared__ __align__(16) float Ws[NS][BK][BM];
  __shared__ __align__(16) float Xs[NS][BK][BN];
  // row of accumulator i (< TM) and column of accumulator j (< 8)
  auto row = [&](int ty, int i) {
    return TM == 2 ? ty * 2 + i : TM == 8 && i >= 4 ? BM / 2 + ty * 4 + i - 4 : ty * 4 + i;
  };
  auto col = [&](int tx, int j) { return TN == 8 && j >= 4 ? BN / 2 + tx * 4 + j - 4 : tx * 4 + j; };

  const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
  const int k0 = blockIdx.y * BM;
  const long long j0 = static_cast<long long>(blockIdx.x) * BN;

  // X loader: element e = tid + NT * i of the BK x BN stage tile ->
  // (channel e / BN, column e % BN); NT is a multiple of BN, so a thread's
  // column is fixed and its channels step by NT / BN
  constexpr int XSTEP = NT / BN;
  const int xcl = tid % BN, xch0 = tid / BN;
  const long long jx = j0 + xcl;
  const bool xok = jx < a.cols;
  const float* xcol = a.x;
  if (xok) {
    const long long n = jx / a.P, p = jx - n * a.P;
    xcol = a.x + n * a.C * a.P + p;
  }
  auto load = [&](int st, int c0) {
#pragma unroll
    for (int i = 0; i < Cfg::WPER; ++i) {
      const int e = tid + NT * i, wc = e / (BM / 4), wq = e % (BM / 4);
      if (Cfg::WCH < NT && e >= Cfg::WCH) break;
      const int c = c0 + wc, kk = k0 + 4 * wq;
      const bool v = c < a.C && kk < a.Kp;  // Kp % 4 == 0: a chunk is all in or all out
      cp_async16(&Ws[st][wc][4 * wq], v ? a.wt + static_cast<size_t>(c) * a.Kp + kk : a.wt, v);
    }
    const float* src = xcol + static_cast<size_t>(c0 + xch0) * a.P;
#pragma unroll
    for (int i = 0; i < Cfg::XPER; ++i, src += static_cast<size_t>(XSTEP) * a.P) {
      const int ch = xch0 + XSTEP * i;
      const bool v = xok && c0 + ch < a.C;
      cp_async4(&Xs[st][ch][xcl], v ? src : a.x, v);
    }
  };

  float acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0f;

  const int stages = (a.C + BK - 1) / BK;
#pragma unroll
  for (int p = 0; p < NS - 1; ++p) {
    if (p < stages) load(p, p * BK);
    cp_async_commit();
  }
  for (int s = 0; s < stages; ++s) {
    const int b = s % NS;
    cp_async_wait<NS - 2>();  // this thread's copies of stage s have landed
    // this thread's weight chunks of the stage: any Inf / NaN? (past C and
    // Kp they are zero-filled, so finite)
    int bad = 0;
#pragma unroll
    for (int i = 0; i < Cfg::WPER; ++i) {
      const int e = tid + NT * i, wc = e / (BM / 4), wq = e % (BM / 4);
      if (Cfg::WCH < NT && e >= Cfg::WCH) break;
      const float4 w4 = *reinterpret_cast<const float4*>(&Ws[b][wc][4 * wq]);
      bad |= !isfinite(w4.x) | !isfinite(w4.y) | !isfinite(w4.z) | !isfinite(w4.w);
    }
    // publishes every thread's copies of stage s, and every thread is past
    // stage s - 1, whose buffer the next copy refills
    const bool skip = __syncthreads_or(bad);
    if (s + NS - 1 < stages) load((s + NS - 1) % NS, (s + NS - 1) * BK);
    cp_async_commit();
    if (!skip) {
#pragma unroll
      for (int c = 0; c < BK; ++c) {
        float av[TM], bv[TN];
        if constexpr (TM == 2) {
          const float2 a0 = *reinterpret_cast<const float2*>(&Ws[b][c][ty * 2]);
          av[0] = a0.x, av[1 % TM] = a0.y;
        } else {
          const float4 a0 = *reinterpret_cast<const float4*>(&Ws[b][c][ty * 4]);
          av[0] = a0.x, av[1] = a0.y, av[2 % TM] = a0.z, av[3 % TM] = a0.w;
          if constexpr (TM == 8) {
            const float4 a1 = *reinterpret_cast<const float4*>(&Ws[b][c][BM / 2 + ty * 4]);
            av[4 % TM] = a1.x, av[5 % TM] = a1.y, av[6 % TM] = a1.z, av[7 % TM] = a1.w;
          }
        }
        const float4 b0 = *reinterpret_cast<const float4*>(&Xs[b][c][tx * 4]);
        bv[0] = b0.x, bv[1] = b0.y, bv[2] = b0.z, bv[3] = b0.w;
        if constexpr (TN == 8) {
          const float4 b1 = *reinterpret_cast<const float4*>(&Xs[b][c][BN / 2 + tx * 4]);
          bv[4 % TN] = b1.x, bv[5 % TN] = b1.y, bv[6 % TN] = b1.z, bv[7 % TN] = b1.w;
        }
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int q = 0; q < TN / 2; ++q) {
            if constexpr (FAST)
              ffma2(acc[i][2 * q], acc[i][2 * q + 1], bv[2 * q], bv[2 * q + 1], av[i]);
            else
              exact2(acc[i][2 * q], acc[i][2 * q + 1], bv[2 * q], bv[2 * q + 1], av[i]);
          }
      }
    } else {
      // an Inf / NaN weight in the stage: zero cells skipped as the
      // reference does (v != 0; -0 counts as zero)
#pragma unroll 1
      for (int c = 0; c < BK; ++c) {
#pragma unroll
        for (int i = 0; i < TM; ++i) {
          const float w = Ws[b][c][row(ty, i)];
#pragma unroll
          for (int j = 0; j < TN; ++j) {
            const float v = Xs[b][c][col(tx, j)];
            if (v != 0.0f) acc[i][j] = mac<FAST>(acc[i][j], v, w);
          }
        }
      }
    }
  }
  cp_async_wait<0>();

  // epilogue: y[n][k][p] for the thread's TM x TN (k, column) outputs
#pragma unroll
  for (int j = 0; j < TN; ++j) {
    const long long jj = j0 + col(tx, j);
    if (jj >= a.cols) continue;
    const long long n = jj / a.P, p = jj - n * a.P;
    float* yc = a.y + n * a.K * a.P + p;
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int k = k0 + row(ty, i);
      if (k < a.K) yc[static_cast<size_t>(k) * a.P] = a.relu ? relu_f(acc[i][j]) : acc[i][j];
    }
  }
}

}  // namespace sconv_cu
