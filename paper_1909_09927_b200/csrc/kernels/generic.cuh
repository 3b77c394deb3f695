// generic.cuh -- shape-generic ECR / PECR kernels (any kernel size, stride,
// pooling window and pooling stride).  One thread per output; used for the
// configurations the tiled kernel is not specialised for.  Same term order
// and arithmetic modes as the tiled path, so EXACT stays bit-identical.
#pragma once

#include "common.cuh"

namespace sconv_cu {

struct GenericArgs {
  const float* x;  // [N][C][H][W]
  const float* w;  // [K][C][kh][kw]
  float* y;
  int N, C, H, W, K, kh, kw, S, OH, OW;
  int pw, ph, ps, mode;  // PECR pool geometry; mode = pool mode (PECR) / fused ReLU (ECR)
  int PH, PW;            // PECR pack grid
};

template <bool FAST>
__device__ __forceinline__ float window_dot(const float* xn, const float* wk, int C, int H, int W,
                                            int kh, int kw, int y0, int x0) {
  float acc = 0.0f;
  for (int c = 0; c < C; ++c) {
    const float* xc = xn + (static_cast<size_t>(c) * H + y0) * W + x0;
    const float* wc = wk + c * kh * kw;
    for (int i = 0; i < kh; ++i)
      for (int j = 0; j < kw; ++j) {
        const float v = __ldg(xc + i * W + j);
        if (v != 0.0f) acc = mac<FAST>(acc, v, __ldg(wc + i * kw + j));
      }
  }
  return acc;
}

// ECR: ecr_convert + ecr_spmv_conv per (image, filter, window).
template <bool FAST>
__global__ void ecr_generic_kernel(const GenericArgs a) {
  const size_t total = static_cast<size_t>(a.N) * a.K * a.OH * a.OW;
  for (size_t idx = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int ox = static_cast<int>(idx % a.OW);
    const int oy = static_cast<int>((idx / a.OW) % a.OH);
    const int k = static_cast<int>((idx / (static_cast<size_t>(a.OW) * a.OH)) % a.K);
    const int n = static_cast<int>(idx / (static_cast<size_t>(a.OW) * a.OH * a.K));
    const float* xn = a.x + static_cast<size_t>(n) * a.C * a.H * a.W;
    const float* wk = a.w + static_cast<size_t>(k) * a.C * a.kh * a.kw;
    const float v = window_dot<FAST>(xn, wk, a.C, a.H, a.W, a.kh, a.kw, oy * a.S, ox * a.S);
    a.y[idx] = a.mode ? relu_f(v) : v;  // mode = fused ReLU for ECR launches
  }
}

// PECR: pack (b, t) folds windows n = 0 .. pw*ph-1 in raster order, window n
// at (b*cs*ps + (n/pw)*cs, t*cs*ps + (n%pw)*cs) -- src/pecr.cpp:106-112.
template <bool FAST>
__global__ void pecr_generic_kernel(const GenericArgs a) {
  const size_t total = static_cast<size_t>(a.N) * a.K * a.PH * a.PW;
  const int wpp = a.pw * a.ph;
  for (size_t idx = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int t = static_cast<int>(idx % a.PW);
    const int b = static_cast<int>((idx / a.PW) % a.PH);
    const int k = static_cast<int>((idx / (static_cast<size_t>(a.PW) * a.PH)) % a.K);
    const int n = static_cast<int>(idx / (static_cast<size_t>(a.PW) * a.PH * a.K));
    const float* xn = a.x + static_cast<size_t>(n) * a.C * a.H * a.W;
    const float* wk = a.w + static_cast<size_t>(k) * a.C * a.kh * a.kw;
    PoolFold f;
    for (int q = 0; q < wpp; ++q) {
      const int wy = b * a.S * a.ps + (q / a.pw) * a.S;
      const int wx = t * a.S * a.ps + (q % a.pw) * a.S;
      f.add(window_dot<FAST>(xn, wk, a.C, a.H, a.W, a.kh, a.kw, wy, wx), a.mode);
    }
    a.y[idx] = f.result(a.mode, wpp);
  }
}

// Filter re-layout for the tiled kernels: wt[c][i*kw+j][k] = w[k][c][i][j],
// rows padded to Kp >= K output channels with zeros (16B-aligned rows).  A
// transpose of the K x M matrix (M = C*kh*kw) through 32 x 33 shared tiles:
// both the reads (along m) and the writes (along k) are coalesced.
// grid = (ceil(Kp / 32), ceil(M / 32)), block = 32 x 8.
__global__ void __launch_bounds__(256) transpose_filters_kernel(const float* __restrict__ w,
                                                                float* __restrict__ wt, int K,
                                                                int Kp, int C, int KK) {
  __shared__ float tile[32][33];
  const long long M = static_cast<long long>(C) * KK;
  const int k0 = blockIdx.x * 32;
  const long long m0 = static_cast<long long>(blockIdx.y) * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
#pragma unroll
  for (int r = ty; r < 32; r += 8) {  // tile[k][m] = w[k0 + r][m0 + tx]
    const int k = k0 + r;
    const long long m = m0 + tx;
    tile[r][tx] = (k < K && m < M) ? __ldg(w + static_cast<long long>(k) * M + m) : 0.0f;
  }
  __syncthreads();
#pragma unroll
  for (int r = ty; r < 32; r += 8) {  // wt[m0 + r][k0 + tx] = tile[tx][r]
    const long long m = m0 + r;
    const int k = k0 + tx;
    if (m < M && k < Kp) wt[m * Kp + k] = tile[tx][r];
  }
}

// PECR pooling of a conv output already in memory (pecr_conv_pool's fold,
// src/pecr.cpp:147-167: windows n = 0 .. pw*ph-1 in raster order, max from
// +0.0 -> ReLU folded, or mean of max(acc, 0)).  Used for pool shapes the
// fused epilogue does not cover (anything but 2x2/2): conv by a tiled kernel,
// then this -- bit-identical to the fused / generic PECR in EXACT mode.
__global__ void pecr_pool_fold_kernel(const float* __restrict__ conv, float* __restrict__ y,
                                      size_t planes, int OH, int OW, int pw, int ph, int ps,
                                      int mode, int PH, int PW) {
  const size_t total = planes * PH * PW;
  const int wpp = pw * ph;
  for (size_t idx = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int t = static_cast<int>(idx % PW);
    const int b = static_cast<int>((idx / PW) % PH);
    const size_t pl = idx / (static_cast<size_t>(PW) * PH);
    const float* cp = conv + pl * OH * OW;
    PoolFold f;
    for (int q = 0; q < wpp; ++q)
      f.add(cp[static_cast<size_t>(b * ps + q / pw) * OW + t * ps + q % pw], mode);
    y[idx] = f.result(mode, wpp);
  }
}

// ReLU in place (Activation::kRelu after an unfused conv).
__global__ void relu_kernel(float* __restrict__ v, size_t n) {
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<size_t>(gridDim.x) * blockDim.x)
    v[i] = relu_f(v[i]);
}

// pool() of src/tensor.cpp:97-129 over [N*C] planes of H x W: max starts from
// the window's first element and keeps `v > best`; mean sums in raster order
// and divides by the window count.  Output dims use conv_output_dims (floor).
__global__ void pool_kernel(const float* __restrict__ x, float* __restrict__ y, size_t planes,
                            int H, int W, int pw, int ph, int ps, int mode, int OH, int OW) {
  const size_t total = planes * OH * OW;
  const float count = static_cast<float>(pw * ph);
  for (size_t idx = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const int ox = static_cast<int>(idx % OW);
    const int oy = static_cast<int>((idx / OW) % OH);
    const size_t pl = idx / (static_cast<size_t>(OW) * OH);
    const float* xp = x + pl * H * W + static_cast<size_t>(oy * ps) * W + ox * ps;
    if (mode == 0) {
      float best = xp[0];
      for (int i = 0; i < ph; ++i)
        for (int j = 0; j < pw; ++j) {
          const float v = xp[i * W + j];
          if (v > best) best = v;
        }
      y[idx] = best;
    } else {
      float sum = 0.0f;
      for (int i = 0; i < ph; ++i)
        for (int j = 0; j < pw; ++j) sum = __fadd_rn(sum, xp[i * W + j]);
      y[idx] = __fdiv_rn(sum, count);
    }
  }
}

}  // namespace sconv_cu
