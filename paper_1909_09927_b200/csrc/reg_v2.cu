// reg_v2.cu -- registry of the v2 tiled ECR/PECR kernels (kernels/ecr_tiled.cuh):
// configurations, selection and launch.  Its own translation unit so the
// template instantiations compile in parallel with the rest of the library.
#include <cstdlib>
#include <mutex>

#include "host/internal.h"

namespace sconv_cu {
namespace host {
namespace {

// ---------------------------------------------------------------------------
// Tiled kernel registry.  Specialisations exist for the VGG / AlexNet /
// GoogLeNet 3x3 stride-1 shapes; every other shape takes the generic kernel.
// ---------------------------------------------------------------------------
// TiledCfg<KH, KW, S, TH, TW, R, WK, WSY, WSX, CC, P> -- warp tile TH x TW
// outputs x 32R channels, CTA = WSY x WSX warps (x WK along channels).
template <int P> using Cfg1 = TiledCfg<3, 3, 1, 4, 4, 8, 1, 2, 4, 8, P>;  // 8x16 x 256ch
template <int P> using Cfg2 = TiledCfg<3, 3, 1, 4, 4, 4, 1, 2, 4, 8, P>;  // 8x16 x 128ch
template <int P> using Cfg3 = TiledCfg<3, 3, 1, 4, 8, 4, 1, 2, 2, 8, P>;  // 8x16 x 128ch
template <int P> using Cfg4 = TiledCfg<3, 3, 1, 4, 8, 2, 1, 2, 2, 8, P>;  // 8x16 x 64ch
template <int P> using Cfg5 = TiledCfg<3, 3, 1, 2, 8, 8, 1, 4, 2, 8, P>;  // 8x16 x 256ch
template <int P> using Cfg6 = TiledCfg<3, 3, 1, 4, 4, 2, 1, 2, 4, 8, P>;  // 8x16 x 64ch
template <int P> using Cfg7 = TiledCfg<3, 3, 1, 2, 4, 4, 1, 4, 2, 8, P>;  // 8x8 x 128ch

template <class Cfg>
constexpr int min_blocks() {
  return Cfg::R >= 8 ? 1 : 2;
}

template <class Cfg, bool FAST, bool NOSKIP = false>
int launch_tiled_cfg(sconv_cu_ctx* ctx, const TiledArgs& a, int N) {
  auto kern = ecr_tiled_kernel<Cfg, FAST, min_blocks<Cfg>(), NOSKIP>;
  static std::once_flag attr_once[64];  // per (instantiation, device), thread-safe
  cudaError_t attr_err = cudaSuccess;
  std::call_once(attr_once[ctx->device & 63], [&] {
    attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
  });
  CK(attr_err);
  const int tiles_y = (a.OH + Cfg::OTH - 1) / Cfg::OTH;
  const int tiles_x = (a.OW + Cfg::OTW - 1) / Cfg::OTW;
  TiledArgs b = a;
  b.tiles_x = tiles_x;
  dim3 grid(tiles_y * tiles_x, (a.K + Cfg::KT - 1) / Cfg::KT, N);
  kern<<<grid, Cfg::NT, Cfg::SMEM_BYTES, ctx->stream>>>(b);
  return finish_launch(ctx, "ecr_tiled_kernel");
}

int forced_cfg() {
  static const int v = [] {
    const char* e = std::getenv("SCONV_TILED_CFG");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}

}  // namespace

// which tiled config (0 = none -> generic)
int pick_tiled(int K, int kh, int kw, int S, int P) {
  if (!(kh == 3 && kw == 3 && S == 1 && (P == 0 || P == 2) && K >= 32)) return 0;
  const int f = forced_cfg();
  if ((f >= 1 && f <= kNumCfgs) || (f >= 11 && f <= 17 && P == 0)) return f;
  if (K % 128 == 0) return 2;  // measured best on VGG K=128..512 (tools/tune.py)
  return 4;
}

namespace {

template <template <int> class CfgT, bool FAST>
int launch_p(sconv_cu_ctx* ctx, int P, const TiledArgs& a, int N) {
  return P == 0 ? launch_tiled_cfg<CfgT<0>, FAST>(ctx, a, N)
                : launch_tiled_cfg<CfgT<2>, FAST>(ctx, a, N);
}

template <bool FAST>
int launch_tiled_t(sconv_cu_ctx* ctx, int which, int P, const TiledArgs& a, int N) {
  switch (which) {
    case 1: return launch_p<Cfg1, FAST>(ctx, P, a, N);
    case 2: return launch_p<Cfg2, FAST>(ctx, P, a, N);
    case 3: return launch_p<Cfg3, FAST>(ctx, P, a, N);
    case 4: return launch_p<Cfg4, FAST>(ctx, P, a, N);
    case 5: return launch_p<Cfg5, FAST>(ctx, P, a, N);
    case 6: return launch_p<Cfg6, FAST>(ctx, P, a, N);
    case 17: return launch_tiled_cfg<Cfg7<0>, FAST, true>(ctx, a, N);  // calibration
    case 11: return launch_tiled_cfg<Cfg1<0>, FAST, true>(ctx, a, N);  // calibration
    case 12: return launch_tiled_cfg<Cfg2<0>, FAST, true>(ctx, a, N);  // calibration
    default: return launch_p<Cfg7, FAST>(ctx, P, a, N);
  }
}

}  // namespace

template <class Cfg>
static void fill_plan(sconv_launch_plan* p, int which, int N, int K, int OH, int OW) {
  p->kernel = which;
  p->grid_x = ((OH + Cfg::OTH - 1) / Cfg::OTH) * ((OW + Cfg::OTW - 1) / Cfg::OTW);
  p->grid_y = (K + Cfg::KT - 1) / Cfg::KT;
  p->grid_z = N;
  p->block_threads = Cfg::NT;
  p->smem_bytes = Cfg::SMEM_BYTES;
  p->tile_h = Cfg::OTH;
  p->tile_w = Cfg::OTW;
  p->tile_k = Cfg::KT;
}

void plan_for(sconv_launch_plan* p, int which, int N, int K, int OH, int OW) {
  switch (which) {
    case 1: return fill_plan<Cfg1<0>>(p, which, N, K, OH, OW);
    case 2: return fill_plan<Cfg2<0>>(p, which, N, K, OH, OW);
    case 3: return fill_plan<Cfg3<0>>(p, which, N, K, OH, OW);
    case 4: return fill_plan<Cfg4<0>>(p, which, N, K, OH, OW);
    case 5: return fill_plan<Cfg5<0>>(p, which, N, K, OH, OW);
    case 11: return fill_plan<Cfg1<0>>(p, which, N, K, OH, OW);
    case 12: return fill_plan<Cfg2<0>>(p, which, N, K, OH, OW);
    case 6: return fill_plan<Cfg6<0>>(p, which, N, K, OH, OW);
    case 17: return fill_plan<Cfg7<0>>(p, which, N, K, OH, OW);
    default: return fill_plan<Cfg7<0>>(p, which, N, K, OH, OW);
  }
}

int launch_tiled(sconv_cu_ctx* ctx, bool fast, int which, int P, const TiledArgs& a, int N) {
  return fast ? launch_tiled_t<true>(ctx, which, P, a, N) : launch_tiled_t<false>(ctx, which, P, a, N);
}

}  // namespace host
}  // namespace sconv_cu
