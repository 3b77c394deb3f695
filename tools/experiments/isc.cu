// isc.cu -- launch layer of the v4 row-input-stationary ECR/PECR kernel
// (kernels/ecr_isc.cuh).  A separate translation unit so the registry builds
// in parallel with sconv_cuda.cu; called from fused_conv() there.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "host/tma.h"
#include "kernels/ecr_isc.cuh"

namespace sconv_cu {
namespace {

// IscCfg<TW, R, WPC, CC, NS, P>
template <int P> using IscA = IscCfg<4, 4, 11, 4, 4, P>;  // K % 128 == 0, 12 warps, 1 CTA/SM
template <int P> using IscB = IscCfg<8, 2, 11, 4, 4, P>;  // K = 64, 8-wide columns
template <int P> using IscC = IscCfg<4, 2, 15, 4, 4, P>;  // K = 64, 4-wide columns, 16 warps
template <int P> using IscD = IscCfg<4, 4, 7, 4, 4, P>;   // K % 128 == 0, 8 warps

constexpr int kSR = 4;

template <class Cfg>
int resident_ctas(int num_sms) {
  static int per_sm = [] {
    int b = 0;
    auto kern = ecr_isc_kernel<Cfg>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, Cfg::NT, Cfg::SMEM_BYTES) != cudaSuccess)
      b = 1;
    return std::max(b, 1);
  }();
  return per_sm * num_sms;
}

// Segment length: minimise waves x steps-per-wave (a segment of S owned steps
// runs S + 1 steps; the extra one is the warm-up of every segment but the first).
void choose_segments(int nsteps, long items_per_seg, int wpc, int kblocks, int slots, int* S_out,
                     int* segs_out) {
  long best = -1;
  int bestS = nsteps - 1 > 0 ? nsteps - 1 : 1, bestSegs = 1;
  for (int S = std::max(1, nsteps - 1); S >= 1; --S) {
    const int segs = 1 + std::max(0, (nsteps - (S + 1) + S - 1) / S);
    const long ctas = (items_per_seg * segs + wpc - 1) / wpc * kblocks;
    const long waves = (ctas + slots - 1) / slots;
    const long cost = waves * (S + 1);
    if (best < 0 || cost < best) {
      best = cost;
      bestS = S;
      bestSegs = segs;
    }
  }
  *S_out = bestS;
  *segs_out = bestSegs;
}

template <class Cfg>
IscArgs geometry(const IscRequest& rq) {
  IscArgs a{};
  a.x = rq.x;
  a.y = rq.y;
  a.N = rq.N;
  a.C = rq.C;
  a.H = rq.H;
  a.W = rq.W;
  a.K = rq.K;
  a.OH = rq.OH;
  a.OW = rq.OW;
  a.mode = rq.mode;
  a.tiles_x = (rq.OW + Cfg::TW - 1) / Cfg::TW;
  const int nsteps = (rq.OH + 2 + kSR - 1) / kSR;  // step r completes output rows 4r-2 .. 4r+1
  const int kblocks = (rq.K + Cfg::KT - 1) / Cfg::KT;
  choose_segments(nsteps, long(rq.N) * a.tiles_x, Cfg::WPC, kblocks, resident_ctas<Cfg>(rq.num_sms),
                  &a.S, &a.segs);
  a.total = rq.N * a.segs * a.tiles_x;
  return a;
}

template <class Cfg>
IscShape shape_of(const IscRequest& rq) {
  const IscArgs a = geometry<Cfg>(rq);
  return IscShape{(rq.K + Cfg::KT - 1) / Cfg::KT * ((a.total + Cfg::WPC - 1) / Cfg::WPC), 1, Cfg::NT,
                  Cfg::SMEM_BYTES, kSR * a.S, Cfg::TW, Cfg::KT};
}

template <class Cfg>
cudaError_t launch_cfg(const IscRequest& rq, cudaStream_t st, const char** what) {
  auto kern = ecr_isc_kernel<Cfg>;
  static bool attr_done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (!attr_done[dev & 63]) {
    *what = "cudaFuncSetAttribute(ecr_isc_kernel)";
    const cudaError_t e =
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_done[dev & 63] = true;
  }
  const IscArgs a = geometry<Cfg>(rq);
  const int kblocks = (rq.K + Cfg::KT - 1) / Cfg::KT;
  CUtensorMap wmap;
  *what = "cuTensorMapEncodeTiled";
  if (encode_weight_map(rq.wt, rq.C, Cfg::KK, rq.Kp, Cfg::KT, Cfg::CC, &wmap) != CUDA_SUCCESS)
    return cudaErrorInvalidValue;
  dim3 grid(kblocks * ((a.total + Cfg::WPC - 1) / Cfg::WPC));
  *what = "ecr_isc_kernel";
  kern<<<grid, Cfg::NT, Cfg::SMEM_BYTES, st>>>(a, wmap);
  return cudaGetLastError();
}

template <template <int> class CfgT>
cudaError_t launch_p(const IscRequest& rq, cudaStream_t st, const char** what) {
  return rq.P == 2 ? launch_cfg<CfgT<2>>(rq, st, what) : launch_cfg<CfgT<0>>(rq, st, what);
}

}  // namespace

int isc_pick(int K, int C, int H, int W, int kh, int kw, int stride, int P, bool fast, int forced) {
  if (!fast || kh != 3 || kw != 3 || stride != 1 || !(P == 0 || P == 2) || K < 64) return 0;
  if (P == 2 && (((H - 2) % 2) != 0 || ((W - 2) % 2) != 0)) return 0;
  // producer cell offsets are 32-bit
  if (double(C) * H * W * 64.0 >= 2147483647.0) return 0;
  const char* e = std::getenv("SCONV_KERNEL");
  if (e && e[0] == 'i' && e[1] >= '1' && e[1] <= '4') forced = e[1] - '0';
  if (e && e[0] != 'i') return 0;  // another kernel family forced
  if (forced >= 1 && forced <= 4) {
    if ((forced == 1 || forced == 4) && K % 128 != 0) return 0;
    return forced;
  }
  return 0;  // not selected by default (measured slower than v3)
}

IscShape isc_shape(int which, int N, int K, int OH, int OW, int num_sms) {
  IscRequest rq{};
  rq.N = N;
  rq.K = K;
  rq.OH = OH;
  rq.OW = OW;
  rq.num_sms = num_sms;
  switch (which) {
    case 1: return shape_of<IscA<0>>(rq);
    case 2: return shape_of<IscB<0>>(rq);
    case 3: return shape_of<IscC<0>>(rq);
    default: return shape_of<IscD<0>>(rq);
  }
}

cudaError_t isc_launch(int which, const IscRequest& rq, cudaStream_t st, const char** what) {
  switch (which) {
    case 1: return launch_p<IscA>(rq, st, what);
    case 2: return launch_p<IscB>(rq, st, what);
    case 3: return launch_p<IscC>(rq, st, what);
    case 4: return launch_p<IscD>(rq, st, what);
    default: *what = "isc_launch"; return cudaErrorInvalidValue;
  }
}

}  // namespace sconv_cu
