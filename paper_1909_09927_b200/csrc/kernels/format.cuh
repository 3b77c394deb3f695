// format.cuh -- ECR / PECR format kernels (the reference's two-phase API) and
// the integer op counters.
//
// Compaction is warp-ballot + popc prefix: a warp walks one window's
// C*kh*kw slot in (c, i, j) order 32 entries at a time; lane e tests its
// entry, __ballot_sync gives the nonzero mask, and popc(mask & lanes_below)
// is the entry's position among the window's nonzeros.  That reproduces the
// sequential `filled++` of ecr_convert (src/ecr.cpp:79-91) and the push_back
// order of pecr_convert (src/pecr.cpp:114-125) exactly.
#pragma once

#include "common.cuh"

namespace sconv_cu {

__device__ __forceinline__ unsigned lanes_below() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---- ECR export: ecr_convert (src/ecr.cpp:51-97) -------------------------
struct EcrExportArgs {
  const float* x;       // [C][H][W]
  const float* filter;  // [C][kh][kw]
  int C, H, W, kh, kw, S, OH, OW;
  int32_t* ptr;         // [OH*OW]
  int32_t* offsets;     // [OH*OW*slot]
  float* f_data;
  float* k_data;
};

__global__ void ecr_export_kernel(const EcrExportArgs a) {
  const int lane = threadIdx.x & 31;
  const size_t win = (blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x) >> 5;
  if (win >= static_cast<size_t>(a.OH) * a.OW) return;
  const int b = static_cast<int>(win / a.OW), t = static_cast<int>(win % a.OW);
  const int kk = a.kh * a.kw, slot = a.C * kk;
  const size_t base = win * slot;
  const unsigned below = lanes_below();
  int filled = 0;
  for (int e0 = 0; e0 < slot; e0 += 32) {
    const int e = e0 + lane;
    float v = 0.0f;
    if (e < slot) {
      const int c = e / kk, r = e - c * kk, i = r / a.kw, j = r - i * a.kw;
      v = __ldg(a.x + (static_cast<size_t>(c) * a.H + b * a.S + i) * a.W + t * a.S + j);
    }
    const bool nz = v != 0.0f;  // -0.0 is zero (ecr.cpp:84)
    const unsigned m = __ballot_sync(kFull, nz);
    if (nz) {
      const size_t p = base + filled + __popc(m & below);
      a.f_data[p] = v;
      a.k_data[p] = __ldg(a.filter + e);
      a.offsets[p] = e;  // (c*kh + i)*kw + j == e
    }
    filled += __popc(m);
  }
  for (int p = filled + lane; p < slot; p += 32) {  // filler (ecr.cpp:64-70)
    a.f_data[base + p] = 0.0f;
    a.k_data[base + p] = 0.0f;
    a.offsets[base + p] = -1;
  }
  if (lane == 0) a.ptr[win] = filled ? filled : -1;  // sentinel (ecr.cpp:93)
}

// ---- ECR SpMV: ecr_spmv_conv (src/ecr.cpp:99-128) -------------------------
struct EcrSpmvArgs {
  const int32_t* ptr;
  const float* f_data;
  const float* k_data;
  int nwin, slot;
  float* y;
  unsigned long long* ops;  // [0] muls, [1] adds  (nullable)
  int* bad;                 // set when a ptr is outside [-1, slot]
};

// EXACT: one thread per window, sequential acc += f*k (ecr.cpp:117-120).
__global__ void ecr_spmv_exact_kernel(const EcrSpmvArgs a) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long muls = 0, adds = 0;
  if (w < a.nwin) {
    const int nnz = a.ptr[w];
    if (nnz < -1 || nnz > a.slot) {
      atomicOr(a.bad, 1);
    } else if (nnz == -1) {
      a.y[w] = 0.0f;
    } else {
      const size_t base = static_cast<size_t>(w) * a.slot;
      float acc = 0.0f;
      for (int p = 0; p < nnz; ++p) acc = mac<false>(acc, a.f_data[base + p], a.k_data[base + p]);
      a.y[w] = acc;
      muls = nnz;
      adds = nnz > 0 ? nnz - 1 : 0;
    }
  }
  if (a.ops) {
    block_add_u64(muls, a.ops);
    block_add_u64(adds, a.ops + 1);
  }
}

// FAST: one warp per window, lane-strided FFMA partial sums, then a
// warp-shuffle tree reduction.
__global__ void ecr_spmv_fast_kernel(const EcrSpmvArgs a) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  unsigned long long muls = 0, adds = 0;
  if (w < a.nwin) {
    const int nnz = a.ptr[w];
    if (nnz < -1 || nnz > a.slot) {
      if (lane == 0) atomicOr(a.bad, 1);
    } else {
      const size_t base = static_cast<size_t>(w) * a.slot;
      float acc = 0.0f;
      for (int p = lane; p < nnz; p += 32) acc = __fmaf_rn(a.f_data[base + p], a.k_data[base + p], acc);
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
      if (lane == 0) {
        a.y[w] = nnz == -1 ? 0.0f : acc;
        muls = nnz > 0 ? nnz : 0;
        adds = nnz > 0 ? nnz - 1 : 0;
      }
    }
  }
  if (a.ops) {
    block_add_u64(muls, a.ops);
    block_add_u64(adds, a.ops + 1);
  }
}

// ---- PECR export: pecr_convert (src/pecr.cpp:83-131) ----------------------
struct PecrFmtArgs {
  const float* x;  // [C][H][W]
  int C, H, W, kh, kw, S, pw, ph, ps, PH, PW;
  int32_t* count;            // [PH*PW*pw*ph]
  const int64_t* pack_start; // fill phase
  float* data;
  int32_t* index;
};

// one warp per (pack, window n); phase 0 counts, phase 1 fills.
template <int PHASE>
__global__ void pecr_export_kernel(const PecrFmtArgs a) {
  const int lane = threadIdx.x & 31;
  const int wpp = a.pw * a.ph;
  const size_t item = (blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x) >> 5;
  if (item >= static_cast<size_t>(a.PH) * a.PW * wpp) return;
  const size_t pack = item / wpp;
  const int n = static_cast<int>(item % wpp);
  const int b = static_cast<int>(pack / a.PW), t = static_cast<int>(pack % a.PW);
  const int wy = b * a.S * a.ps + (n / a.pw) * a.S;
  const int wx = t * a.S * a.ps + (n % a.pw) * a.S;
  const int kk = a.kh * a.kw, slot = a.C * kk;
  int64_t pos = 0;
  if (PHASE == 1) {
    pos = a.pack_start[pack];
    for (int m = 0; m < n; ++m) pos += a.count[pack * wpp + m];
  }
  const unsigned below = lanes_below();
  int filled = 0;
  for (int e0 = 0; e0 < slot; e0 += 32) {
    const int e = e0 + lane;
    float v = 0.0f;
    if (e < slot) {
      const int c = e / kk, r = e - c * kk, i = r / a.kw, j = r - i * a.kw;
      v = __ldg(a.x + (static_cast<size_t>(c) * a.H + wy + i) * a.W + wx + j);
    }
    const bool nz = v != 0.0f;
    const unsigned m = __ballot_sync(kFull, nz);
    if (PHASE == 1 && nz) {
      const int64_t p = pos + filled + __popc(m & below);
      a.data[p] = v;
      a.index[p] = e;  // (c*kh + i)*kw + j
    }
    filled += __popc(m);
  }
  if (PHASE == 0 && lane == 0) a.count[item] = filled;
}

// ---- PECR pooling over a format: pecr_conv_pool (src/pecr.cpp:133-172) ----
struct PecrPoolArgs {
  const int32_t* count;
  const int64_t* pack_start;
  const float* data;
  const int32_t* index;
  const float* kernel;  // [C*kh*kw]
  int npacks, wpp, cap, mode;
  float* y;
  unsigned long long* ops;
  int* bad;
};

// check_pecr (src/pecr.cpp:40-55) on device
__global__ void pecr_check_kernel(const PecrPoolArgs a, int64_t total) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= a.npacks) return;
  int64_t s = 0;
  for (int n = 0; n < a.wpp; ++n) {
    const int c = a.count[static_cast<size_t>(p) * a.wpp + n];
    if (c < 0 || c > a.cap) atomicOr(a.bad, 1);
    s += c;
  }
  const int64_t b = a.pack_start[p], e = a.pack_start[p + 1];
  if (e - b != s || b < 0 || e > total) {
    atomicOr(a.bad, 1);
    return;
  }
  for (int64_t q = b; q < e; ++q)
    if (a.index[q] < 0 || a.index[q] >= a.cap) atomicOr(a.bad, 1);
}

// Both pool kernels run after pecr_check_kernel on device formats: a format
// it flagged is never read (the reference throws FormatError before any
// computation, src/pecr.cpp:24-58), so a bad index cannot fault the context.
__global__ void pecr_pool_exact_kernel(const PecrPoolArgs a) {
  if (*a.bad) return;  // uniform across the grid
  const int pk = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long muls = 0, adds = 0;
  if (pk < a.npacks) {
    int64_t p = a.pack_start[pk];
    PoolFold f;
    for (int n = 0; n < a.wpp; ++n) {
      const int cn = a.count[static_cast<size_t>(pk) * a.wpp + n];
      float acc = 0.0f;
      for (int q = 0; q < cn; ++q, ++p) acc = mac<false>(acc, a.data[p], __ldg(a.kernel + a.index[p]));
      f.add(acc, a.mode);
      muls += cn;
      adds += cn > 0 ? cn - 1 : 0;
    }
    a.y[pk] = f.result(a.mode, a.wpp);
  }
  if (a.ops) {
    block_add_u64(muls, a.ops);
    block_add_u64(adds, a.ops + 1);
  }
}

__global__ void pecr_pool_fast_kernel(const PecrPoolArgs a) {
  if (*a.bad) return;
  const int lane = threadIdx.x & 31;
  const int pk = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  unsigned long long muls = 0, adds = 0;
  if (pk < a.npacks) {
    int64_t p = a.pack_start[pk];
    PoolFold f;
    for (int n = 0; n < a.wpp; ++n) {
      const int cn = a.count[static_cast<size_t>(pk) * a.wpp + n];
      float acc = 0.0f;
      for (int q = lane; q < cn; q += 32) acc = __fmaf_rn(a.data[p + q], __ldg(a.kernel + a.index[p + q]), acc);
      for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(kFull, acc, o);
      f.add(acc, a.mode);
      p += cn;
      if (lane == 0) {
        muls += cn;
        adds += cn > 0 ? cn - 1 : 0;
      }
    }
    if (lane == 0) a.y[pk] = f.result(a.mode, a.wpp);
  }
  if (a.ops) {
    block_add_u64(muls, a.ops);
    block_add_u64(adds, a.ops + 1);
  }
}

// ---- OpCount for the fused path (integer, deterministic) ------------------
// pix[n][y][x] = number of channels with a nonzero at (y, x).
__global__ void pixel_nnz_kernel(const float* __restrict__ x, int N, int C, int H, int W,
                                 int32_t* __restrict__ pix) {
  const size_t plane = static_cast<size_t>(H) * W;
  const size_t total = static_cast<size_t>(N) * plane;
  for (size_t idx = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t n = idx / plane, yx = idx % plane;
    const float* p = x + n * C * plane + yx;
    int cnt = 0;
    for (int c = 0; c < C; ++c) cnt += __ldg(p + c * plane) != 0.0f;
    pix[idx] = cnt;
  }
}

// Window nnz of conv window (cy, cx) = box sum of pix.  ECR: every window
// once; PECR: every window of every pack (packs may overlap, and the
// reference counts each pack's windows, pecr.cpp:162-163).
struct OpsArgs {
  const int32_t* pix;
  int N, H, W, kh, kw, S;
  int OH, OW;            // ECR window grid
  int PH, PW, pw, ph, ps; // PECR packs (pw == 0 -> ECR)
  unsigned long long* ops;
};

__device__ __forceinline__ int window_nnz_at(const OpsArgs& a, const int32_t* pn, int cy, int cx) {
  int s = 0;
  for (int i = 0; i < a.kh; ++i)
    for (int j = 0; j < a.kw; ++j) s += pn[(cy * a.S + i) * a.W + cx * a.S + j];
  return s;
}

// window_nnz_counts (src/dataset.cpp:249-268) for a batch: counts[n][oy][ox]
// = nonzeros of window (oy, ox) over all channels, and per image the sum of
// them and of the raw nonzeros (sparsity_profile, dataset.cpp:270-286).
__global__ void window_nnz_kernel(const OpsArgs a, int32_t* __restrict__ counts,
                                  unsigned long long* __restrict__ win_sum) {
  const size_t per_img = static_cast<size_t>(a.OH) * a.OW;
  const size_t total = static_cast<size_t>(a.N) * per_img;
  for (size_t idx = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t n = idx / per_img, r = idx % per_img;
    const int nnz = window_nnz_at(a, a.pix + n * a.H * a.W, static_cast<int>(r / a.OW),
                                  static_cast<int>(r % a.OW));
    if (counts) counts[idx] = nnz;
    if (win_sum && nnz) atomicAdd(win_sum + n, static_cast<unsigned long long>(nnz));  // integer: order-free
  }
}

__global__ void pixel_sum_kernel(const int32_t* __restrict__ pix, int N, size_t plane,
                                 unsigned long long* __restrict__ raw_sum) {
  const size_t total = static_cast<size_t>(N) * plane;
  for (size_t idx = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<size_t>(gridDim.x) * blockDim.x)
    if (pix[idx]) atomicAdd(raw_sum + idx / plane, static_cast<unsigned long long>(pix[idx]));
}

__global__ void ops_kernel(const OpsArgs a) {
  unsigned long long muls = 0, adds = 0;
  const bool pecr = a.pw > 0;
  const size_t per_img = pecr ? static_cast<size_t>(a.PH) * a.PW : static_cast<size_t>(a.OH) * a.OW;
  const size_t total = static_cast<size_t>(a.N) * per_img;
  for (size_t idx = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const size_t n = idx / per_img, r = idx % per_img;
    const int32_t* pn = a.pix + n * a.H * a.W;
    if (!pecr) {
      const int nnz = window_nnz_at(a, pn, static_cast<int>(r / a.OW), static_cast<int>(r % a.OW));
      muls += nnz;
      adds += nnz > 0 ? nnz - 1 : 0;
    } else {
      const int b = static_cast<int>(r / a.PW), t = static_cast<int>(r % a.PW);
      for (int q = 0; q < a.pw * a.ph; ++q) {
        const int nnz = window_nnz_at(a, pn, b * a.ps + q / a.pw, t * a.ps + q % a.pw);
        muls += nnz;
        adds += nnz > 0 ? nnz - 1 : 0;
      }
    }
  }
  block_add_u64(muls, a.ops);
  block_add_u64(adds, a.ops + 1);
}

}  // namespace sconv_cu
