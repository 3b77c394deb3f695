// reg_v3.cu -- v3 selection and launch plans (no kernel instantiations).
#include "reg_v3.inc"

namespace sconv_cu {
namespace host {

// which ws config (0 = none); P is 0 (ECR) or 2 (PECR 2x2/2)
bool ws_applies(int id, int K, int kh, int kw, int S, int P) {
  if (K < 32) return false;
  if (id >= 18 && id <= 20) {  // general-pool configs (P == -1 only)
    if (P != -1 || S != 1) return false;
    return id == 18 ? (kh == 3 && kw == 3) : id == 19 ? (kh == 5 && kw == 5) : (kh == 1 && kw == 1);
  }
  if (!(P == 0 || P == 2)) return false;
  if (id == 21 || id == 22) return kh == 3 && kw == 3 && S == 1 && P == 0;
  if (id == 23) return kh == 3 && kw == 3 && S == 1;
  if (id == 11) return kh == 3 && kw == 3 && S == 2;
  if (id == 12) return kh == 3 && kw == 3 && S == 3;
  if (S != 1) return false;
  if (id >= 1 && id <= 7) return kh == 3 && kw == 3 && !(id == 2 && P != 0);
  if (id == 8 || id == 9 || id == 14 || id == 15) return kh == 1 && kw == 1;
  if (id == 10 || id == 17) return kh == 5 && kw == 5;
  if (id == 16) return kh == 3 && kw == 3;
  return false;
}

int pick_ws(int K, int C, int OW, int kh, int kw, int S, int P, long tiles4, long tiles2) {
  if (!((P == 0 || P == 2) && K >= 32)) return 0;
  // strided 3x3 (the paper's stride-2/3 experiments):
  // 2x2 output tiles whose 5x5 / 6x6 input windows fit the 64-bit mask
  if (kh == 3 && kw == 3 && (S == 2 || S == 3)) return S == 2 ? 11 : 12;
  if (S != 1) return 0;
  // 1x1 / 5x5 (GoogLeNet / LeNet layers, BASELINE config 2): the same
  // warp-specialised kernel instantiated for that window (tools/config2.py)
  //
  // Maps too small to fill the GPU with 4x4 tiles take 2x2 tiles (WsN-WsQ)
  // when those still fit in one wave of 7-consumer CTAs at 2 per SM: on every
  // config-2 layer (tools/config2.py, profiles/r01/config2_layers.jsonl) this
  // picks the faster of the two (AlexNet conv3 114 -> 71 us, inception 5a 1x1
  // 138 -> 101 us, 5b 5x5 34 -> 26 us; 4a's 12x12 3x3 stays on 4x4 tiles:
  // 62 vs 104 us).  tiles2 = images x 2x2 output tiles.
  const long wave = 148L * 2 * 7;
  const long kb128 = (K + 127) / 128, kb64 = (K + 63) / 64;
  if (kh == 1 && kw == 1) {
    if (K >= 128) return tiles2 * kb128 <= wave ? 14 : 8;
    return tiles2 * kb64 <= wave ? 15 : 9;
  }
  if (kh == 5 && kw == 5) return tiles2 * kb64 <= wave ? 17 : 10;
  if (!(kh == 3 && kw == 3)) return 0;
  const char* e = std::getenv("SCONV_KERNEL");
  if (e && std::strcmp(e, "v2") == 0) return 0;
  if (e && e[0] == 'w' && e[1] >= 'A' && e[1] <= 'W' && ws_applies(e[1] - 'A' + 1, K, kh, kw, S, P))
    return e[1] - 'A' + 1;
  if (e && std::strcmp(e, "v3") == 0) {
    if (K <= 64) return 3;
    if (OW % 4 != 0 && OW % 7 == 0 && P == 0) return 2;
    return 1;
  }
  // Measured on B200 (tools/tune.py, tools/ksweep.py, profiles/r01): with the
  // filters staged by TMA, v3 beats v2 on every K >= 128 VGG layer (17-20%);
  // for K = 64 PECR the 6x6-tile WsG wins (its pooled 3x3 stores are small),
  // for K = 64 ECR the 4x4-tile WsD (float4 stores, 3 CTAs/SM: conv1_2 3588
  // -> 3320 us); small C goes to the small-C kernel before this is asked.
  if (K >= 128 && tiles2 * kb128 <= wave) return 16;
  // K = 64 PECR on a big grid (tiles4 >= ~15 6x6 tiles per SM): the 6x6 tiles
  // in one persistent CTA of 15 consumers per SM (WsW) -- conv1_2 2901 -> 2783
  // us at s = 0.7, -5% / -6% at 0.9 / 0.95 (tools/gpu_runs/gpu_r2_abgen.sh);
  // ECR stays on WsD (+7% with WsW).
  if (K < 128 && C >= 16 && P == 2 && tiles4 >= 148L * 15 * 36 / 16) return 23;
  if (K < 128) return C >= 16 ? (P == 2 ? 7 : 4) : 0;
  // One CTA of 15 consumer warps per SM (WsA) beats two CTAs of 7 (WsE) once
  // there are enough channel chunks to amortise a CTA's pipeline fill and
  // drain (C >= 128): one producer per SM instead of two, and finer last
  // waves (conv4_2 2638 -> 2451 us, conv4_1 -6%, conv3_2 / conv2_2 -2%);
  // with C = 64 (16 chunks) the overlap of two CTAs wins (conv2_1 1302 vs
  // 1366).  Below one wave WsA leaves SMs idle that WsE's smaller CTAs still
  // reach; tools/smallgrid.py over batches 2-32 of the C >= 128 VGG layers
  // puts the crossover between 1024 (WsE 311 vs 414 us) and 1568 (WsA 418 vs
  // 450 us) warp tiles.  With the 15-consumer CTA the 4x4 tiles also beat the
  // waste-free 2x7 tiles (WsB) on 14x14 maps at every batch measured (conv5_1
  // at 64: 797 vs 819 us; at 16: WsE 311 vs WsB 319 us), so WsB is forced-only.
  // tiles4 = 4x4 output tiles x K-blocks of 128.  Round 2: with the
  // persistent grid WsA runs for C <= 128 (reg_v3.inc), its ring no longer
  // refills per CTA and it also wins at C = 64 (conv2_1 1254 vs WsE 1355 us,
  // tools/gpu_runs/gpu_r2_c12.sh).
  // 14-wide maps (VGG conv5) in ECR: 7x2 tiles in the same 15-consumer CTA
  // (WsV: 14 tiles per image instead of sixteen 4x4 tiles, no overhang) once
  // the lean producer and the row prefetch were in: conv5_1 -1.2 / -3.4 /
  // -3.6 / -2.4% at s = 0.5 / 0.7 / 0.8 / 0.9 (tools/gpu_runs/gpu_r2_v_rp.sh;
  // it lost 3-11% at s >= 0.9 before them).
  if (C >= 128 && P == 0 && OW % 7 == 0 && OW % 4 != 0 && tiles4 >= 148L * 10) return 22;
  return (C >= 64 && tiles4 >= 148L * 10) ? 1 : 5;
}

// The general-pool config for a window / pool geometry (0 = none: the pool
// then runs as conv + pecr_pool_fold_kernel): the conv tile must hold at
// least one whole pool window.
int pick_ws_pool(int K, int kh, int kw, int S, int pw, int ph) {
  if (K < 32 || S != 1) return 0;
  if (kh == 3 && kw == 3) return (pw <= WsR::TW && ph <= WsR::TH) ? 18 : 0;
  if (kh == 5 && kw == 5) return (pw <= WsS::TW && ph <= WsS::TH) ? 19 : 0;
  if (kh == 1 && kw == 1) return (pw <= WsT::TW && ph <= WsT::TH) ? 20 : 0;
  return 0;
}

// Plan of a v3 launch: kernel id 100 + registry index; grid_x counts CTAs of
// WPC warp tiles over the flat (image, tile) list, grid_z is 1.
namespace {
template <class Cfg>
void plan_ws_t(sconv_launch_plan* p, int which, int N, int K, int OH, int OW, int pw, int ph,
               int ps) {
  long tiles = long((OH + Cfg::TH - 1) / Cfg::TH) * ((OW + Cfg::TW - 1) / Cfg::TW) * N;
  if (Cfg::P < 0 && pw > 0) {  // tiles of whole pool windows over the pooled map
    const int pth = (Cfg::TH - ph) / ps + 1, ptw = (Cfg::TW - pw) / ps + 1;
    const int PHo = (OH - ph) / ps + 1, PWo = (OW - pw) / ps + 1;
    tiles = long((PHo + pth - 1) / pth) * ((PWo + ptw - 1) / ptw) * N;
  }
  p->kernel = 100 + which;
  p->grid_x = static_cast<int>((tiles + Cfg::WPC - 1) / Cfg::WPC) * ((K + Cfg::KT - 1) / Cfg::KT);
  p->grid_y = 1;
  p->grid_z = 1;
  p->block_threads = Cfg::NT;
  p->smem_bytes = Cfg::SMEM_BYTES;
  p->tile_h = Cfg::TH;
  p->tile_w = Cfg::TW;
  p->tile_k = Cfg::KT;
}

}  // namespace

void plan_ws(sconv_launch_plan* out, int ws, int n, int k, int OH, int OW, int pw, int ph, int ps) {
  switch (ws) {
    case 18: plan_ws_t<WsR>(out, ws, n, k, OH, OW, pw, ph, ps); return;
    case 19: plan_ws_t<WsS>(out, ws, n, k, OH, OW, pw, ph, ps); return;
    case 20: plan_ws_t<WsT>(out, ws, n, k, OH, OW, pw, ph, ps); return;
    case 21: plan_ws_t<WsU>(out, ws, n, k, OH, OW, 0, 0, 1); return;
    case 22: plan_ws_t<WsV>(out, ws, n, k, OH, OW, 0, 0, 1); return;
    case 23: plan_ws_t<WsW<0>>(out, ws, n, k, OH, OW, 0, 0, 1); return;
    case 1: plan_ws_t<WsA<0>>(out, ws, n, k, OH, OW, 0, 0, 1); break;
    case 2: plan_ws_t<WsB<0>>(out, ws, n, k, OH, OW, 0, 0, 1); break;
    case 4: plan_ws_t<WsD<0>>(out, ws, n, k, OH, OW, 0, 0, 1); break;
    case 5: plan_ws_t<WsE<0>>(out, ws, n, k, OH, OW, 0, 0, 1); break;
    case 6: plan_ws_t<WsF<0>>(out, ws, n, k, OH, OW, 0, 0, 1); break;
    case 7: plan_ws_t<WsG<0>>(out, ws, n, k, OH, OW, 0, 0, 1); break;
    case 8: plan_ws_t<WsH<0>>(out, ws, n, k, OH, OW, 0, 0, 1); break;
    case 9: plan_ws_t<WsI<0>>(out, ws, n, k, OH, OW, 0, 0, 1); break;
    case 10: plan_ws_t<WsJ<0>>(out, ws, n, k, OH, OW, 0, 0, 1); break;
    case 11: plan_ws_t<WsK<0>>(out, ws, n, k, OH, OW, 0, 0, 1); break;
    case 12: plan_ws_t<WsL<0>>(out, ws, n, k, OH, OW, 0, 0, 1); break;
    case 14: plan_ws_t<WsN<0>>(out, ws, n, k, OH, OW, 0, 0, 1); break;
    case 15: plan_ws_t<WsO<0>>(out, ws, n, k, OH, OW, 0, 0, 1); break;
    case 16: plan_ws_t<WsP<0>>(out, ws, n, k, OH, OW, 0, 0, 1); break;
    case 17: plan_ws_t<WsQ<0>>(out, ws, n, k, OH, OW, 0, 0, 1); break;
    default: plan_ws_t<WsC<0>>(out, ws, n, k, OH, OW, 0, 0, 1); break;
  }
}

}  // namespace host
}  // namespace sconv_cu
