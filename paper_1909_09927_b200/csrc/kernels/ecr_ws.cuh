// ecr_ws.cuh -- the hot path, v3: warp-specialised fused ECR compaction +
// sparse convolution (+ the PECR ReLU/pooling epilogue) for sm_100a.
//
// Same arithmetic as ecr_tiled.cuh (input-stationary, lanes over output
// channels, warp-uniform zero skip, terms in (c, i, j) order per output), but
// the CTA is organised around what the B200 profile of v2 showed:
//
// * One producer warp stages CC-channel chunks into an NS-deep ring of
//   shared-memory stages with cp.async and signals a `full` mbarrier
//   (cp.async.mbarrier.arrive.noinc); consumer warps release a stage through
//   an `empty` mbarrier.  There is no __syncthreads in the main loop, so a
//   warp whose tiles happen to be denser than its neighbours' no longer
//   stalls the CTA at every chunk (v2: ~13-17% of stall samples were
//   barrier), and the consumers execute no staging address arithmetic.
// * Each consumer warp owns one TH x TW output tile of any image; the
//   producer copies that warp's (TH-1)S+KH x (TW-1)S+KW input window into a
//   private, 16B-aligned sub-patch (halo columns duplicated).  Tiles are a
//   flat list over (image, tile) so any tile shape covers any map size with
//   no partial-tile waste (v2 computed 32x32 for the 28x28 layers).
// * FAST mode multiplies with packed FFMA2 (fma.rn.f32x2, the input value
//   broadcast to both halves): half the FMA instructions of v2 and no
//   even/odd register-bank conflicts between weight and accumulator.
//
// Bit-exactness in EXACT mode is unchanged: per output, terms arrive in
// channel order (chunks ascend, channels inside a chunk ascend) and within a
// channel in window raster order, i.e. the order of ecr_convert's f_data /
// k_data (src/ecr.cpp:79-91) summed as in ecr_spmv_conv (:117-120).
#pragma once

#include <cuda.h>

#include "common.cuh"
#include "ecr_body.cuh"

namespace sconv_cu {

#ifndef SCONV_EMPTY_ALL_LANES  // 1: every consumer lane arrives on `empty` (sanitizer build)
#define SCONV_EMPTY_ALL_LANES 0
#endif

#ifndef SCONV_WS_OPAQUE_LANE
#define SCONV_WS_OPAQUE_LANE 1
#endif
// Window-row prefetch: 0 never, 1 always, 2 per launch from the sampled
// input density (at least SCONV_WS_RP_DENSITY_PCT percent nonzero)
#ifndef SCONV_WS_RP
#define SCONV_WS_RP 2
#endif
#ifndef SCONV_WS_RP_DENSITY_PCT
#define SCONV_WS_RP_DENSITY_PCT 15
#endif
#ifndef SCONV_SPARSE_PCT_WIDE  // see WsCfg::SPARSE_PCT
#define SCONV_SPARSE_PCT_WIDE 100
#endif

template <int KH_, int KW_, int S_, int TH_, int TW_, int R_, int WPC_, int CC_, int NS_, int P_,
          int NP_ = 1>
struct WsCfg {
  static constexpr int KH = KH_, KW = KW_, S = S_, TH = TH_, TW = TW_, R = R_;
  static constexpr int WPC = WPC_, CC = CC_, NS = NS_, P = P_;
  static constexpr int NP = NP_;                     // producer warps (cells split between them)
  static constexpr int KK = KH * KW;
  static constexpr int KT = 32 * R;                  // output channels per CTA
  static constexpr int WPH = (TH - 1) * S + KH;      // warp input window rows
  static constexpr int WPW = (TW - 1) * S + KW;      // warp input window cols
  // sub-patch row pitch (floats): 8 or 16; 4 for tall 4-column windows
  // (7x2 tiles: 9 rows x 4) whose 8-float rows would overflow the 64-bit mask
  static constexpr int PITCH = WPW <= 8 ? ((WPW <= 4 && WPH * 8 > 64) ? 4 : 8) : 16;
  static constexpr int PATCH = WPH * PITCH;          // floats per (warp, channel)
  static constexpr int NPOS = WPH * WPW;
  static constexpr int IN_STAGE = (WPC * CC * PATCH + 31) / 32 * 32;  // floats, 128B aligned
  static constexpr int W_STAGE = CC * KK * KT;       // floats
  static constexpr int STAGE = IN_STAGE + W_STAGE;
  static constexpr int NT = 32 * (WPC + NP);         // + producer warps
  static constexpr int MINB =  // CTAs/SM (register budget: accumulators + weight registers)
      (NT > 256 || R >= 8) ? 1 : ((TH * TW * R <= 32 && KH * KW * R <= 36) ? 3 : 2);
  // P == -1 (any pool geometry): the epilogue stages each warp's conv tile in
  // shared memory, aliased onto the ring once every consumer has left it
  static constexpr int EPI = P < 0 ? WPC * TH * TW * KT : 0;
  static constexpr int RING = NS * STAGE > EPI ? NS * STAGE : EPI;  // floats before the barriers
  static constexpr int SMEM_BYTES = RING * 4 + 2 * NS * 8;
  static constexpr int CELLS = WPC * NPOS;           // input cells per channel
  static constexpr int CELLS_PER_LANE = (CELLS + 32 * NP - 1) / (32 * NP);
  // Producer copies cells in 8-byte pairs when every window row starts on an
  // even column (even row width, even tile stride and map width): half the
  // cp.async instructions and requests.
  static constexpr bool PAIR = (WPW % 2 == 0) && ((TW * S) % 2 == 0);
  // Channels whose window density is at most SPARSE_PCT percent take the
  // row-skipping, fully branched body; denser ones the body whose 1-3-tap
  // border cells ptxas predicates (their FFMA2 run even for zero cells).
  // Measured (A/B, tools/gpu_ab2.sh): with R = 2 or 2-row tiles the border
  // cells carry so little work that branching always wins (conv5 2x7 -3.5%,
  // conv1_2 ECR -2.3%).  4x4 R = 4 tiles preferred predication above 25% in
  // round 1; re-measured on the round-2 build (tools/gpu_runs/gpu_r2_pct.sh)
  // the fully branched body everywhere is 0.3-0.8% faster at s = 0.7 and
  // equal at 0.9 (threshold 0: 1-4% slower at 0.7, 20-26% at 0.9), so WIDE
  // is now 100 -- one body per channel, half the hot code.  (The dense body
  // with every cell branched and no row tests: 0-2.5% slower at 0.7, 29% at
  // 0.9.)
  // 2x2 tiles and 1x1 windows are the opposite case: a cell feeds at most
  // four outputs (one for 1x1), so its one to eight FFMA2 cost less than the
  // branch that would skip it, and only all-zero windows branch.  Measured:
  // inception 5a 1x1 on 2x2 tiles 101.6 -> 81.0 us, 4a.7 55.4 -> 44.0 us;
  // 3x3 on 2x2 tiles: VGG conv4_2 at batch 1 164.6 -> 140.5 us, AlexNet conv4
  // 102.5 -> 91.3 us, stride 3 conv4_2 1006 -> 913 us, stride 2 -3...-4%
  // (the 4x4 R = 4 1x1 config loses 4% that way and keeps the threshold).
  static constexpr int SPARSE_PCT =
      (TH == 2 && TW == 2) ? 0 : (R <= 2 || TH <= 2) ? (KH == 1 && KW == 1 ? 0 : 100) : SCONV_SPARSE_PCT_WIDE;
  // Channel-loop unroll: small bodies (2x2 tiles) are latency-bound per
  // channel (cell load -> ballot -> branch -> FFMA2), so two channels in
  // flight let the next channel's loads issue under this one's FFMA2.
#ifndef SCONV_WS_SMALL_UNROLL
#define SCONV_WS_SMALL_UNROLL 2
#endif
#ifndef SCONV_WS_BIG_UNROLL
#define SCONV_WS_BIG_UNROLL 1
#endif
  // (measured on the config-2 layers, tools/gpu_runs/gpu_r2_c2ab.sh: 2 for the
  // 2x2 tiles and the 1x1 windows -- inception 4a 1x1 on 4x4 tiles -3.6% --;
  // 3 costs the 3x3 2x2-tile AlexNet layers 10%; the 4x4 3x3 bodies lose 5%
  // with 2)
  static constexpr int CU = (TH * TW <= 4 || KH * KW == 1) ? SCONV_WS_SMALL_UNROLL : SCONV_WS_BIG_UNROLL;
  // the window-row prefetch (ecr_channel RP) is measured, and instantiated,
  // for the 3x3 stride-1 one-body configs
  static constexpr bool RPOK = SPARSE_PCT >= 100 && KH == 3 && KW == 3 && S == 1 && P >= 0;
  static constexpr int PAIRS = WPC * NPOS / 2;
  static constexpr int PAIRS_PER_LANE = (PAIRS + 32 * NP - 1) / (32 * NP);
  static_assert(PATCH <= 64, "sub-patch must fit the two 32-bit ballots");
  static_assert(R == 2 || R == 4 || R == 8, "R");
  static_assert(P <= 0 || (TH % P == 0 && TW % P == 0), "pool tile");
  static_assert((IN_STAGE * 4) % 128 == 0 && (STAGE * 4) % 128 == 0, "TMA destination alignment");
  static constexpr unsigned W_BYTES = W_STAGE * 4;   // one TMA box (CC x KK x KT floats)
};

struct WsArgs {
  const float* x;   // [N][C][H][W]
  const float* wt;  // [C][KH*KW][Kp]  (filters transposed once per call)
  float* y;         // [N][K][OH][OW] or pooled [N][K][PHo][PWo]
  int N, C, H, W, K, Kp, OH, OW;
  int tiles_x, tiles_per_img, total_tiles;
  int mode;  // pool mode (P != 0); P == 0: fused ReLU flag
  // P == -1: the pool window / stride and the pooled map; a warp tile then
  // holds PTH x PTW whole pool windows ((PTH-1)*ps + ph <= TH conv rows) and
  // consecutive tiles start tsy / tsx conv outputs apart (= PTH*ps, PTW*ps;
  // = TH, TW for P >= 0): overlapping pools recompute the shared conv rows
  // instead of sending the pre-pool map through HBM.
  int pw = 0, ph = 0, ps = 1, PHo = 0, PWo = 0, tsy = 0, tsx = 0;
  // Row-prefetch gate (RPOK configs): the plain and the row-prefetching
  // instantiation are both launched and every CTA of the one not chosen by
  // ws_density_gate_kernel (*gate = 1: prefetch) exits at once; nullptr: run.
  const int* gate = nullptr;
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_cp_async(uint64_t* b) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* b, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity) {
  while (!mbar_try_wait(b, parity)) __nanosleep(32);
}
// The producer runs ahead and mostly waits for the slowest consumer warp:
// back off instead of spinning, a polling warp steals issue slots from the
// consumer warps on its SMSP.
#ifndef SCONV_PRODUCER_SLEEP_NS
#define SCONV_PRODUCER_SLEEP_NS 256
#endif
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* b, unsigned parity) {
  while (!mbar_try_wait(b, parity)) __nanosleep(SCONV_PRODUCER_SLEEP_NS);
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
// TMA: one CC x KK x KT box of the transposed filters wt[C][KK][Kp] into the
// stage's weight region; completion is counted on the stage's `full` barrier.
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}

template <int R>
__device__ __forceinline__ int ws_lane_chan(int lane, int r) {
  if constexpr (R >= 4) {
    return (r / 4) * 128 + lane * 4 + (r % 4);
  } else {
    return lane * R + r;
  }
}

template <int R>
__device__ __forceinline__ void ws_lds_w(float (&dst)[R], const float* row, int lane) {
  if constexpr (R >= 4) {
#pragma unroll
    for (int g = 0; g < R / 4; ++g) {
      const float4 a = *reinterpret_cast<const float4*>(row + g * 128 + lane * 4);
      dst[4 * g + 0] = a.x;
      dst[4 * g + 1] = a.y;
      dst[4 * g + 2] = a.z;
      dst[4 * g + 3] = a.w;
    }
  } else {
    const float2 a = *reinterpret_cast<const float2*>(row + lane * 2);
    dst[0] = a.x;
    dst[1] = a.y;
  }
}

// Keeps a zero-skip block behind its uniform branch (see SCONV_KEEP_BRANCH);
// __syncwarp emits no instruction in converged code but is not if-converted,
// and it lets ptxas batch the mask-bit predicates ahead of the branches.
#ifndef SCONV_WS_GUARD
#define SCONV_WS_GUARD 2
#endif

// Window-row prefetch (RP, ecr_channel) pays while most window rows hold a
// nonzero (-3..-5% at s = 0.5-0.8) and costs a wasted shared-memory read per
// empty row, which the LSU-bound high-sparsity case cannot afford (+5% at
// s = 0.9, +17% at 0.95).  Choosing it inside one kernel -- per channel, per
// chunk, or per launch with both consumer loops compiled into one function --
// cost 1-14% on every path (profiles/r02/ab_row_prefetch.txt), so the two
// loops are separate instantiations and the launch picks one on the device
// (WsArgs::gate) from the sampled input density.
template <class Cfg>
__global__ void ws_density_gate_kernel(const float* x, unsigned total, int* gate) {
  // 1024 threads, one sample each: one per stratum of the input, at a hashed
  // offset; gate = 1 iff at least SCONV_WS_RP_DENSITY_PCT percent are nonzero
  const unsigned i = threadIdx.x, n = blockDim.x, stratum = total / n;
  const unsigned q = stratum ? i * stratum + (i * 0x9E3779B1u) % stratum : i;
  const int nz = __syncthreads_count(q < total && x[q] != 0.0f);
  if (i == 0) *gate = 100 * nz >= SCONV_WS_RP_DENSITY_PCT * int(stratum ? n : total);
}

template <class Cfg, bool FAST, bool RP = false>
__global__ void __launch_bounds__(Cfg::NT, Cfg::MINB)
    ecr_ws_kernel(const WsArgs a, const __grid_constant__ CUtensorMap wmap) {
  static_assert(!RP || Cfg::RPOK, "row prefetch is instantiated for the 3x3 one-body configs");
  if (a.gate && (*a.gate != 0) != RP) return;  // the other instantiation runs this launch
  constexpr int KH = Cfg::KH, KW = Cfg::KW, S = Cfg::S, TH = Cfg::TH, TW = Cfg::TW, R = Cfg::R;
  constexpr int KK = Cfg::KK, KT = Cfg::KT, CC = Cfg::CC, NS = Cfg::NS, P = Cfg::P;
  constexpr int WPC = Cfg::WPC, WPH = Cfg::WPH, WPW = Cfg::WPW, PITCH = Cfg::PITCH;
  constexpr int PATCH = Cfg::PATCH, NP = Cfg::NP;

  extern __shared__ float4 smem_raw[];
  float* smem = reinterpret_cast<float*>(smem_raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::RING);
  uint64_t* empty = full + NS;

  const int tid = threadIdx.x;
  // The shuffle makes the warp index provably warp-uniform to ptxas: with a
  // plain tid >> 5 the role split below is a "divergent" branch, the ballot
  // masks land in vector registers and every zero-skip branch pays a vector
  // bit test right before it (plus BRA.DIV checks for the guard).
  const int warp = __shfl_sync(kFull, tid >> 5, 0), lane = tid & 31;
  // K-blocks vary fastest over the linear grid, so the CTAs that read the same
  // input patches run together and the patch is fetched from HBM once.
  // Work items (tile group x K-block), K-blocks fastest; a CTA takes items
  // blockIdx.x, + gridDim.x, ... (one each unless the host launched a
  // persistent grid: then the ring runs on across items -- the producer
  // stages the next item's first chunks while the consumers store the last
  // one's outputs -- and a CTA's fill and drain are paid once).
  const int kblocks = (a.K + KT - 1) / KT;
  const int items = (a.total_tiles + WPC - 1) / WPC * kblocks;
  const int C = a.C, H = a.H, W = a.W, K = a.K;
  const int nchunks = (C + CC - 1) / CC;

  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 32 * NP + 1);  // cp.async lane arrivals + the TMA expect_tx arrival
      mbar_init(&empty[s], SCONV_EMPTY_ALL_LANES ? WPC * 32 : WPC);
    }
  }
  __syncthreads();

  if (warp >= WPC) {
    // ------------------------------ producer ------------------------------
    // producer warp pw copies cells (pairs) pw*32 + lane + 32*NP*e; pw 0 also
    // issues the weight TMA
    const int pl = NP == 1 ? lane : (warp - WPC) * 32 + lane;  // lane among the producer warps
    const size_t plane = static_cast<size_t>(H) * W;
    if constexpr (Cfg::PAIR) {
      // warp-uniform: 8-byte aligned cell pairs (every window row starts on
      // an even column; general-pool tiles may step by an odd stride)
      if ((W & 1) == 0 && ((a.tsx * S) & 1) == 0) {
        if (lane == 0)
          asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&wmap)) : "memory");
        for (int item = blockIdx.x, it = 0; item < items; item += gridDim.x, ++it) {
        const int cta = item / kblocks, k0 = (item - cta * kblocks) * KT, kbase = it * nchunks;
        // per pair: source pointer at channel 0 (the map base for pairs outside
        // the map: zero-filled, and base + c0 * plane stays inside the map),
        // valid bytes, and shared-memory byte offset within a stage
        const float* src0[Cfg::PAIRS_PER_LANE];
        int bytes[Cfg::PAIRS_PER_LANE];
        unsigned dst_b[Cfg::PAIRS_PER_LANE];
#pragma unroll
        for (int e = 0; e < Cfg::PAIRS_PER_LANE; ++e) {
          const int q = pl + 32 * NP * e;
          const int wi = q / (Cfg::NPOS / 2), pp = q - wi * (Cfg::NPOS / 2);
          const int Y = pp / (WPW / 2), X = 2 * (pp - Y * (WPW / 2));
          const int t = cta * WPC + wi;
          const int n = t / a.tiles_per_img, tt = t - n * a.tiles_per_img;
          const int ty = tt / a.tiles_x, tx = tt - ty * a.tiles_x;
          const int iy = ty * a.tsy * S + Y, ix = tx * a.tsx * S + X;
          const bool ok = q < Cfg::PAIRS && t < a.total_tiles && iy < H && ix < W;
          bytes[e] = ok ? (ix + 1 < W ? 8 : 4) : 0;
          src0[e] = ok ? a.x + (static_cast<size_t>(n) * C * H + iy) * W + ix : a.x;
          dst_b[e] = 4u * ((wi * CC) * PATCH + Y * PITCH + X);
        }
        for (int k = 0; k < nchunks; ++k) {
          const int kk = kbase + k, s = kk % NS;
          if (kk >= NS) mbar_wait_sleep(&empty[s], ((kk / NS) + 1) & 1);
          float* in_s = smem + s * Cfg::STAGE;
          float* w_s = in_s + Cfg::IN_STAGE;
          const unsigned in_b = smem_u32(in_s);
          const int c0 = k * CC;
          const size_t coff = static_cast<size_t>(c0) * plane;
          const bool whole = c0 + CC <= C;  // uniform: no channel tail in this chunk
#pragma unroll
          for (int e = 0; e < Cfg::PAIRS_PER_LANE; ++e) {
            if (pl + 32 * NP * e < Cfg::PAIRS) {
              const float* src = src0[e] + coff;
              const unsigned dst = in_b + dst_b[e];
#pragma unroll
              for (int ch = 0; ch < CC; ++ch, src += plane)
                cp_async8_s(dst + 4u * ch * PATCH, src, whole || c0 + ch < C ? bytes[e] : 0);
            }
          }
          if (pl == 0) {
            mbar_arrive_expect_tx(&full[s], Cfg::W_BYTES);
            tma_load_3d(w_s, &wmap, k0, 0, c0, &full[s]);
          }
          mbar_arrive_cp_async(&full[s]);
        }
        }  // items
        cp_async_wait<0>();
        return;
      }
    }
    if (lane == 0)
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&wmap)) : "memory");
    for (int item = blockIdx.x, it = 0; item < items; item += gridDim.x, ++it) {
    const int cta = item / kblocks, k0 = (item - cta * kblocks) * KT, kbase = it * nchunks;
    const float* src0[Cfg::CELLS_PER_LANE];
    bool ok[Cfg::CELLS_PER_LANE];
    unsigned dst_b[Cfg::CELLS_PER_LANE];
#pragma unroll
    for (int e = 0; e < Cfg::CELLS_PER_LANE; ++e) {
      const int q = pl + 32 * NP * e;
      const int wi = q / Cfg::NPOS, pos = q - (q / Cfg::NPOS) * Cfg::NPOS;
      const int Y = pos / WPW, X = pos - (pos / WPW) * WPW;
      const int t = cta * WPC + wi;
      const int n = t / a.tiles_per_img, tt = t - n * a.tiles_per_img;
      const int ty = tt / a.tiles_x, tx = tt - ty * a.tiles_x;
      const int iy = ty * a.tsy * S + Y, ix = tx * a.tsx * S + X;
      ok[e] = q < Cfg::CELLS && t < a.total_tiles && iy < H && ix < W;
      src0[e] = ok[e] ? a.x + (static_cast<size_t>(n) * C * H + iy) * W + ix : a.x;
      dst_b[e] = 4u * ((wi * CC) * PATCH + Y * PITCH + X);
    }
    for (int k = 0; k < nchunks; ++k) {
      const int kk = kbase + k, s = kk % NS;
      if (kk >= NS) mbar_wait_sleep(&empty[s], ((kk / NS) + 1) & 1);
      float* in_s = smem + s * Cfg::STAGE;
      float* w_s = in_s + Cfg::IN_STAGE;
      const unsigned in_b = smem_u32(in_s);
      const int c0 = k * CC;
      const size_t coff = static_cast<size_t>(c0) * plane;
      const bool whole = c0 + CC <= C;
#pragma unroll
      for (int e = 0; e < Cfg::CELLS_PER_LANE; ++e) {
        if (pl + 32 * NP * e < Cfg::CELLS) {
          const float* src = src0[e] + coff;
          const unsigned dst = in_b + dst_b[e];
#pragma unroll
          for (int ch = 0; ch < CC; ++ch, src += plane)
            cp_async4_s(dst + 4u * ch * PATCH, src, ok[e] && (whole || c0 + ch < C));
        }
      }
      if (pl == 0) {  // weights: one TMA box, zero-filled past C and Kp
        mbar_arrive_expect_tx(&full[s], Cfg::W_BYTES);
        tma_load_3d(w_s, &wmap, k0, 0, c0, &full[s]);
      }
      mbar_arrive_cp_async(&full[s]);
    }
    }  // items
    cp_async_wait<0>();
    return;
  }

  // ------------------------------- consumers -------------------------------
  // Lane l tests sub-patch cells l and l+32 (bit = Y*PITCH + X).
  const bool t0 = (lane % PITCH) < WPW && (lane / PITCH) < WPH;
  const bool t1 = ((lane + 32) % PITCH) < WPW && ((lane + 32) / PITCH) < WPH;
  constexpr bool TWO = WPH * PITCH > 32;
#if SCONV_WS_OPAQUE_LANE
  // The lane index as a shuffle result: ptxas cannot rematerialise it, so the
  // per-channel weight loads keep it in a register instead of re-reading
  // SR_TID.X (an S2R, ~8% of the stall samples at s = 0.95) every channel.
  // (R >= 4 only: the R = 2 configs measured +0.3..1.4% with it.)
  const int wlane = R >= 4 ? __shfl_sync(kFull, lane, lane) : lane;
#else
  const int wlane = lane;
#endif
  for (int item = blockIdx.x, it = 0; item < items; item += gridDim.x, ++it) {
  const int cta = item / kblocks, k0 = (item - cta * kblocks) * KT, kbase = it * nchunks;
  const int t = cta * WPC + warp;
  const bool active = t < a.total_tiles;
  const int n = active ? t / a.tiles_per_img : 0;
  const int tt = t - n * a.tiles_per_img;
  const int ty = tt / a.tiles_x, tx = tt - (tt / a.tiles_x) * a.tiles_x;

  float acc[TH][TW][R];
#pragma unroll
  for (int i = 0; i < TH; ++i)
#pragma unroll
    for (int j = 0; j < TW; ++j)
#pragma unroll
      for (int r = 0; r < R; ++r) acc[i][j][r] = 0.0f;

  for (int k = 0; k < nchunks; ++k) {
    const int kk = kbase + k, s = kk % NS;
    mbar_wait(&full[s], (kk / NS) & 1);
    if (active) {
      const float* ic = smem + s * Cfg::STAGE + warp * CC * PATCH;
      const float* wsrc = smem + s * Cfg::STAGE + Cfg::IN_STAGE;
      const int cn = min(CC, C - k * CC);
#pragma unroll Cfg::CU
      for (int c = 0; c < cn; ++c, ic += PATCH, wsrc += KK * KT) {
        const unsigned m0 = __ballot_sync(kFull, t0 && ic[lane] != 0.0f);
        const unsigned m1 = TWO ? __ballot_sync(kFull, t1 && ic[lane + 32] != 0.0f) : 0u;

        float wr[KK][R];
#pragma unroll
        for (int ij = 0; ij < KK; ++ij) ws_lds_w<R>(wr[ij], wsrc + ij * KT, wlane);

        // SPARSE_PCT 100: one body for every channel, no density test; 0: the
        // predicated body, empty windows skipped
        if constexpr (Cfg::SPARSE_PCT >= 100)
          ecr_channel<KH, KW, S, TH, TW, R, WPH, WPW, PITCH, PITCH, FAST, true, false, RP>(acc, wr, ic,
                                                                                       m0, m1);
        else if constexpr (Cfg::SPARSE_PCT <= 0) {
          if (m0 | m1)
            ecr_channel<KH, KW, S, TH, TW, R, WPH, WPW, PITCH, PITCH, FAST, false>(acc, wr, ic, m0, m1);
        } else if ((__popc(m0) + __popc(m1)) * 100 <= Cfg::NPOS * Cfg::SPARSE_PCT)
          ecr_channel<KH, KW, S, TH, TW, R, WPH, WPW, PITCH, PITCH, FAST, true>(acc, wr, ic, m0, m1);
        else
          ecr_channel<KH, KW, S, TH, TW, R, WPH, WPW, PITCH, PITCH, FAST, false>(acc, wr, ic, m0,
                                                                                m1);
      }
    }
#if SCONV_EMPTY_ALL_LANES
    mbar_arrive(&empty[s]);  // every lane releases its own reads (count WPC * 32)
#else
    // lane 0 releases the stage for the warp: __syncwarp orders the other
    // lanes' shared-memory reads before its mbarrier.arrive (release), and
    // the producer's try_wait (acquire) orders them before its next copies.
    // (compute-sanitizer racecheck does not follow this chain and reports the
    // copies as WAR hazards; built with SCONV_EMPTY_ALL_LANES=1 every lane
    // arrives and racecheck is clean: profiles/r02/sanitizer.md.)
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
#endif
  }
  if constexpr (P < 0) {
    // every consumer (active or not) has released its last stage: the ring
    // is free once the producer's copies have all landed, which the last
    // `full` wait of each consumer already observed
    asm volatile("bar.sync 1, %0;" ::"r"(WPC * 32) : "memory");
  }
  if (!active) continue;

  // ---- epilogue ------------------------------------------------------------
  const int oy0 = ty * a.tsy, ox0 = tx * a.tsx;
  if constexpr (P < 0) {
    // Any pool (pecr_conv_pool, src/pecr.cpp:147-167): the warp's conv tile
    // goes to its slice of the (now idle) ring, then each lane folds the
    // pool windows of its own channels in window raster order -- max from
    // +0 (ReLU folded), or the mean of max(v, 0) -- with no pre-pool value
    // leaving the SM.
    float* eb = smem + warp * (TH * TW * KT);
#pragma unroll
    for (int u = 0; u < TH; ++u)
#pragma unroll
      for (int v = 0; v < TW; ++v)
#pragma unroll
        for (int r = 0; r < R; ++r) eb[(u * TW + v) * KT + ws_lane_chan<R>(lane, r)] = acc[u][v][r];
    __syncwarp();
    const int pm = a.mode;
    const int PTH = (TH - a.ph) / a.ps + 1, PTW = (TW - a.pw) / a.ps + 1;
    const int py0 = ty * PTH, px0 = tx * PTW;
    for (int r = 0; r < R; ++r) {
      const int ch = ws_lane_chan<R>(lane, r), kk = k0 + ch;
      if (kk >= K) continue;
      float* dst = a.y + (static_cast<size_t>(n) * K + kk) * a.PHo * a.PWo;
      for (int py = 0; py < PTH && py0 + py < a.PHo; ++py)
        for (int px = 0; px < PTW && px0 + px < a.PWo; ++px) {
          PoolFold f;
          const float* wb = eb + (py * a.ps * TW + px * a.ps) * KT + ch;
          for (int du = 0; du < a.ph; ++du)
            for (int dv = 0; dv < a.pw; ++dv) f.add(wb[(du * TW + dv) * KT], pm);
          dst[(py0 + py) * a.PWo + px0 + px] = f.result(pm, a.ph * a.pw);
        }
    }
  } else if constexpr (P == 0) {
    if (a.mode) relu_tile(acc);  // fused Activation::kRelu (forward)
    const bool vec = (TW % 4 == 0) && (a.OW % 4 == 0);
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int kk = k0 + ws_lane_chan<R>(lane, r);
      if (kk >= K) continue;
      float* dst = a.y + ((static_cast<size_t>(n) * K + kk) * a.OH + oy0) * a.OW + ox0;
#pragma unroll
      for (int oy = 0; oy < TH; ++oy) {
        if (oy0 + oy >= a.OH) continue;
        if (vec) {
#pragma unroll
          for (int q = 0; q < TW / 4; ++q)
            if (ox0 + 4 * q < a.OW)
              *reinterpret_cast<float4*>(dst + oy * a.OW + 4 * q) =
                  make_float4(acc[oy][4 * q][r], acc[oy][4 * q + 1][r], acc[oy][4 * q + 2][r],
                              acc[oy][4 * q + 3][r]);
        } else {
#pragma unroll
          for (int ox = 0; ox < TW; ++ox)
            if (ox0 + ox < a.OW) dst[oy * a.OW + ox] = acc[oy][ox][r];
        }
      }
    }
  } else {
    const int PHo = a.OH / P, PWo = a.OW / P;
    const int py0 = oy0 / P, px0 = ox0 / P;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int kk = k0 + ws_lane_chan<R>(lane, r);
      if (kk >= K) continue;
      float* dst = a.y + ((static_cast<size_t>(n) * K + kk) * PHo + py0) * PWo + px0;
#pragma unroll
      for (int py = 0; py < TH / P; ++py) {
        if (py0 + py >= PHo) continue;
#pragma unroll
        for (int px = 0; px < TW / P; ++px) {
          if (px0 + px >= PWo) continue;
          PoolFold f;
#pragma unroll
          for (int u = 0; u < P; ++u)
#pragma unroll
            for (int v = 0; v < P; ++v) f.add(acc[py * P + u][px * P + v][r], a.mode);
          dst[py * PWo + px] = f.result(a.mode, P * P);
        }
      }
    }
  }
  }  // items
}

}  // namespace sconv_cu
