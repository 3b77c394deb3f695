// sconv_cuda.cu -- C ABI of libsconv_cuda.so (declared in include/sconv_cuda.h).
//
// Host launch / partition layer: argument validation with the reference's
// error taxonomy, per-context stream + workspace, host<->device staging for
// host-pointer calls, kernel selection, and the multi-GPU shard driver.  It
// replaces plan()/dispatch() (src/exec.cpp:8-36, include/sconv/exec.hpp:57-120)
// for the ECR / PECR entry points.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "host/internal.h"
#include "kernels/format.cuh"
#include "kernels/generic.cuh"
#include "kernels/ingest.cuh"
#include "kernels/smallc.cuh"
#include "kernels/smallc2.cuh"
#include "kernels/pointwise.cuh"
#include "kernels/scan.cuh"
#include "host/tma.h"

using namespace sconv_cu;
using namespace sconv_cu::host;

namespace sconv_cu {
namespace host {

thread_local std::string g_noctx_err;

int fail(sconv_cu_ctx* ctx, int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  (ctx ? ctx->err : g_noctx_err) = buf;
  return code;
}

unsigned grid_for(size_t work, int threads, int num_sms) {
  const size_t blocks = (work + threads - 1) / threads;
  return static_cast<unsigned>(std::min<size_t>(std::max<size_t>(blocks, 1), size_t(num_sms) * 64));
}

int finish_launch(sconv_cu_ctx* ctx, const char* what) {
  ctx->launches++;
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(ctx, SCONV_ERR_CUDA, "launch %s: %s", what, cudaGetErrorString(e));
  return SCONV_OK;
}

}  // namespace host
}  // namespace sconv_cu


namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// Bump allocator over the context workspace (grown on demand; growth drains
// the stream first because queued work may still read the old buffer).
struct Arena {
  sconv_cu_ctx* ctx;
  std::vector<size_t> sizes;
  int host = -1;  // >= 0: one of the async host-call workspaces (ctx->hws[host])
  bool grew = false;  // a host workspace was (re)allocated on ctx->stream
  size_t add(size_t bytes) {
    sizes.push_back((bytes + 255) & ~size_t{255});
    return sizes.size() - 1;
  }
  int commit(std::vector<char*>& out) {
    size_t total = 0;
    for (size_t s : sizes) total += s;
    char*& base = host >= 0 ? ctx->hws[host] : ctx->ws;
    size_t& cap_ = host >= 0 ? ctx->hws_cap[host] : ctx->ws_cap;
    if (total > cap_) {
      size_t cap = std::max(total, cap_ + cap_ / 2);
      if (host >= 0) cap = ctx->hws_max = std::max(ctx->hws_max, cap);
      ctx->mem_gen++;  // a captured forward graph must not replay old addresses
      // queued work may still read the old buffer (a host workspace is idle:
      // its previous call was waited for before this one took it)
      if (host < 0) {
        CK(cudaStreamSynchronize(ctx->stream));
        if (base) CK(cudaFree(base));
        base = nullptr;
        cap_ = 0;
        CK(cudaMalloc(&base, cap));
      } else {
        // stream-ordered, from the context's own pool: no device-wide
        // synchronisation (cudaFree would stall every call in flight)
        if (base) CK(cudaFreeAsync(base, ctx->stream));
        base = nullptr;
        cap_ = 0;
        CK(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&base), cap, ctx->pool, ctx->stream));
        grew = true;
      }
      cap_ = cap;
    }
    out.clear();
    size_t off = 0;
    for (size_t s : sizes) {
      out.push_back(base + off);
      off += s;
    }
    return SCONV_OK;
  }
};

int conv_dims(sconv_cu_ctx* ctx, int w, int h, int kw, int kh, int stride, int* ow, int* oh) {
  // conv_output_dims, src/tensor.cpp:44-55
  if (w < 1 || h < 1 || kw < 1 || kh < 1) return fail(ctx, SCONV_ERR_SHAPE, "dims must be positive");
  if (stride < 1) return fail(ctx, SCONV_ERR_CONFIG, "stride must be >= 1");
  if (kw > w || kh > h)
    return fail(ctx, SCONV_ERR_SHAPE, "kernel %dx%d larger than map %dx%d", kw, kh, w, h);
  *ow = (w - kw) / stride + 1;
  *oh = (h - kh) / stride + 1;
  return SCONV_OK;
}

int pack_count(sconv_cu_ctx* ctx, int in, int k, int cs, int p, int ps, int* out) {
  // Eq. 3, src/pecr.cpp:62-81
  if (in < 1 || k < 1 || cs < 1 || p < 1 || ps < 1)
    return fail(ctx, SCONV_ERR_CONFIG, "pack count arguments must be positive");
  const int num = in - k + cs - cs * p + ps * cs;
  const int den = ps * cs;
  if (num <= 0 || num % den != 0)
    return fail(ctx, SCONV_ERR_CONFIG,
                "pool tiling does not divide extent %d: (%d - %d + %d - %d + %d) / %d is not a "
                "positive integer",
                in, in, k, cs, cs * p, den, den);
  *out = num / den;
  return SCONV_OK;
}

// The kernel family of one fused ECR / PECR call.  One function decides it,
// for the launch (fused_conv) and the launch-plan query (sconv_cu_plan).
struct KernelChoice {
  bool smallc = false;      // ecr_smallc_kernel (C <= 4)
  bool sc2 = false;         // ... as the persistent ecr_smallc2_kernel (ECR, OW % 4 == 0)
  int ws = 0;               // v3 warp-specialised config id (reg_v3.inc)
  int which = 0;            // v2 tiled config id (reg_v2.cu)
  bool pool_after = false;  // PECR pool no epilogue fuses: conv, then pecr_pool_fold_kernel
  int P = 0;                // epilogue: 2 = fused 2x2/2 pool, -1 = fused general pool, 0 = none
  int pw = 0;               // 1x1 ECR as the dense ordered GEMM (pointwise.cuh): pw_tile id
  bool tiled() const { return smallc || ws || which || pw; }
};

// Tile of the pointwise GEMM for N*P columns and K filters (0: not used).
// Its CTAs walk the C channels in order, 8 per stage, one barrier each, so a
// CTA's time is set by C; it pays only with >= 2 CTAs per SM of 8x8-output
// threads (>= 1 for 64 x 128).  Measured on the config-2 1x1 layers (tools/gpu_runs/gpu_r2_pw.sh):
// inception 4a 1x1 (294 CTAs of 64x128) 94 -> 68 us; on 5a 1x1 (100 CTAs)
// and 4a.7 (25) the v3 1x1 configs stay as fast or faster, and smaller
// thread tiles (more warps, less work per barrier) were slower still.
struct PwTile {
  int bm, bn, tm, tn;
};
constexpr PwTile kPwTiles[] = {{128, 128, 8, 8}, {64, 128, 8, 8}};
int pw_tile(long long cols, int k, bool forced) {
  auto ctas = [&](int bm, int bn) { return ((cols + bn - 1) / bn) * ((k + bm - 1) / bm); };
  if (k % 128 == 0 && ctas(128, 128) >= 2 * 148) return 1;
  if (forced || ctas(64, 128) >= 148) return 2;
  return 0;
}
void pw_dims(int id, int* bm, int* bn) {
  *bm = kPwTiles[id - 1].bm;
  *bn = kPwTiles[id - 1].bn;
}

int choose_kernel(sconv_cu_ctx* ctx, int n, int c, int k, int kh, int kw, int stride, int OH,
                  int OW, bool pecr, int pw, int ph, int ps, unsigned flags, KernelChoice* out) {
  KernelChoice ch;
  const int P = (pecr && pw == ph && pw == ps) ? pw : 0;
  const int Pk = pecr ? (P ? P : -1) : 0;  // -1: a pool the epilogue cannot fold
  const int forced = (flags >> 8) & 0xff;
  const bool generic = flags & SCONV_F_GENERIC;
  const long tiles4 = long(n) * ((OH + 3) / 4) * ((OW + 3) / 4) * ((k + 127) / 128);
  const long tiles2 = long(n) * ((OH + 1) / 2) * ((OW + 1) / 2);
  const bool tileable = kh == 3 && kw == 3 && stride == 1 && (Pk == 0 || Pk == 2) && k >= 32;
  if (forced == 'M' && !tileable)
    return fail(ctx, SCONV_ERR_ARG, "forced kernel M does not apply to this shape");
  if (!generic) {
    // few input channels (VGG conv1_1): the per-warp small-C kernel (smallc.cuh)
    ch.smallc = tileable && (forced == 'M' || (!forced && c <= 4));
    ch.ws = ch.smallc ? 0 : pick_ws(k, c, OW, kh, kw, stride, Pk, tiles4, tiles2);
    ch.which = ch.ws || ch.smallc ? 0 : pick_tiled(k, kh, kw, stride, Pk);
    // PECR with a pool other than 2x2/2: the kernels whose tiles hold whole
    // pool windows fold it in the epilogue (P = -1); a geometry none of them
    // fits (pool larger than the conv tile, strided conv) falls back to a
    // tiled conv into a workspace + pecr_pool_fold_kernel (the pre-pool map
    // then does reach HBM).
    if (pecr && Pk != 2 && !ch.tiled() && !forced) {
      if (kh == 3 && kw == 3 && stride == 1 && k >= 32 && c <= 4 && pw <= 4 && ph <= 4) {
        ch.smallc = true;
        ch.P = -1;
      } else if ((ch.ws = pick_ws_pool(k, kh, kw, stride, pw, ph)) != 0) {
        ch.P = -1;
      } else {
        ch.smallc = kh == 3 && kw == 3 && stride == 1 && k >= 32 && c <= 4;
        ch.ws = ch.smallc ? 0 : pick_ws(k, c, OW, kh, kw, stride, 0, tiles4, tiles2);
        ch.which = ch.smallc || ch.ws ? 0 : pick_tiled(k, kh, kw, stride, 0);
        ch.pool_after = ch.tiled();
      }
    }
    // 1x1 stride-1 ECR: the dense ordered GEMM (pointwise.cuh) -- a window
    // is one cell per channel, so the zero-skipping kernels' per-channel
    // ballot / test / branch chain costs more than the multiplies it skips
    // (forced 'Y'; SCONV_NO_PW=1 keeps the v3 1x1 configs)
    static const bool pw_off = std::getenv("SCONV_NO_PW") != nullptr;  // dev A/B
    const int pwt = kh == 1 && kw == 1 && stride == 1 && Pk == 0
                        ? pw_tile(static_cast<long long>(n) * OH * OW, k, forced == 'Y') : 0;
    if (pwt && ((!forced && !pw_off) || forced == 'Y')) {
      ch.pw = pwt;
      ch.ws = ch.which = 0;
      ch.smallc = false;
    } else if (forced == 'Y') {
      return fail(ctx, SCONV_ERR_ARG, "forced kernel Y does not apply to this shape");
    }
    if (forced && forced != 'M' && forced != 'Y') {
      if (forced >= 1 && forced <= kNumCfgs) {
        if (tileable) {
          ch.which = forced;
          ch.ws = 0;
        }
      } else if (forced >= 'A' && forced <= 'W') {
        const int id = forced - 'A' + 1;
        const bool general = id >= 18 && id <= 20;
        if (general ? !(pecr && Pk != 2 && pick_ws_pool(k, kh, kw, stride, pw, ph) == id)
                    : !ws_applies(id, k, kh, kw, stride, Pk))
          return fail(ctx, SCONV_ERR_ARG, "forced kernel %c does not apply to this shape", forced);
        ch.ws = id;
        ch.which = 0;
        ch.smallc = false;
        ch.P = general ? -1 : 0;
      } else {
        return fail(ctx, SCONV_ERR_ARG, "unknown forced kernel id %d", forced);
      }
    }
  }
  if (ch.P != -1) ch.P = ch.tiled() && !ch.pool_after && Pk == 2 ? 2 : 0;
  // plain ECR on a few channels: the persistent small-C kernel (smallc2.cuh)
  // when its strips tile the map with whole float4 rows and the filters fit
  // its shared-memory budget; forced 'M' keeps the per-tile kernel
  static const bool sc2_off = std::getenv("SCONV_NO_SC2") != nullptr;  // dev A/B
  ch.sc2 = ch.smallc && ch.P == 0 && !ch.pool_after && forced != 'M' && !sc2_off;
  *out = ch;
  return SCONV_OK;
}

// Warp tiles of the small-C kernel per image: 4x4 conv outputs, or (P = -1)
// the tiles of whole pool windows.
long smallc_tiles(const KernelChoice& ch, int OH, int OW, int pw, int ph, int ps) {
  if (ch.P < 0) {
    const int pth = (4 - ph) / ps + 1, ptw = (4 - pw) / ps + 1;
    const int PHo = (OH - ph) / ps + 1, PWo = (OW - pw) / ps + 1;
    return long((PHo + pth - 1) / pth) * ((PWo + ptw - 1) / ptw);
  }
  return long((OH + 3) / 4) * ((OW + 3) / 4);
}

// CTAs one launch of `nb` images takes (chunk sizing below).
long ctas_for(const KernelChoice& ch, int nb, int k, int OH, int OW, size_t y_img, int pw, int ph,
              int ps) {
  sconv_launch_plan pl{};
  if (ch.smallc) return (nb * smallc_tiles(ch, OH, OW, pw, ph, ps) + 7) / 8 * ((k + 63) / 64);
  if (ch.pw) {
    int bm, bn;
    pw_dims(ch.pw, &bm, &bn);
    return (long(nb) * OH * OW + bn - 1) / bn * ((k + bm - 1) / bm);
  }
  if (ch.ws) {
    plan_ws(&pl, ch.ws, nb, k, OH, OW, pw, ph, ps);
    return long(pl.grid_x) * pl.grid_y * pl.grid_z;
  }
  if (ch.which) {
    plan_for(&pl, ch.which, nb, k, OH, OW);
    return long(pl.grid_x) * pl.grid_y * pl.grid_z;
  }
  return long((size_t(nb) * y_img + 255) / 256);
}

// Image chunks (first image, images) of one call.  Host pointers: the batch
// flows through a three-stage ring (H2D of chunk i+1, compute of chunk i, D2H
// of chunk i-1 on three streams), so both PCIe directions stay busy.  Device
// pointers: one chunk, unless a launch limit cuts it.
std::vector<std::pair<int, int>> plan_chunks(const sconv_cu_ctx* ctx, const KernelChoice& ch, int n,
                                             int k, int OH, int OW, size_t x_elems, size_t y_elems,
                                             bool dev, bool async, int pw, int ph, int ps) {
  static const int chunk_env = [] {  // dev override (tools/e2e_probe.py)
    const char* e = std::getenv("SCONV_CHUNKS");
    return e ? std::atoi(e) : 0;
  }();
  const size_t y_img = y_elems / size_t(n);
  int nchunk = 1;
  if (!dev && n > 1) {
    if (chunk_env > 0) {
      nchunk = std::min(n, chunk_env);
    } else if (async) {
      // asynchronous calls overlap each other's transfers, so two halves
      // (the minimum that puts H2D and D2H on their own streams) beat a finer
      // intra-call pipeline (tools/async_probe.py: 62 ms per VGG-19 step vs
      // 75 with the synchronous chunking, 100 with 16 chunks)
      nchunk = 2;
    } else {
      // whole waves: a chunk holds the images whose CTAs fill (just under) one
      // wave of 2 CTAs per SM, or a multiple of that when there would
      // otherwise be more than 16 chunks (e.g. conv4_2: 28 CTAs per image ->
      // 10-image chunks = 0.95 wave; 11 would spill 12 CTAs into a 2nd wave;
      // tools/e2e_probe.py: conv4_2 loses 20% at 4-image chunks)
      const double per_img = std::max(1.0, double(ctas_for(ch, n, k, OH, OW, y_img, pw, ph, ps)) / n);
      const int wave = std::max(1, static_cast<int>(2.0 * ctx->num_sms / per_img));
      const int chunk = wave * std::max(1, (n + 16 * wave - 1) / (16 * wave));
      nchunk = std::max(1, (n + chunk - 1) / chunk);
    }
  }
  // Launch limits: the kernels index a launch's input and output with 32-bit
  // offsets (the producer warps keep per-lane int offsets), so a launch
  // covers at most 2^30 elements of either; the v2 tiled kernels put the
  // images in grid.z (at most 65535).
  const size_t lim = size_t(1) << 30;
  const size_t big = std::max(x_elems, y_elems);
  nchunk = std::max(nchunk, static_cast<int>(std::min<size_t>(size_t(n), (big + lim - 1) / lim)));
  if (ch.which) nchunk = std::max(nchunk, (n + 65534) / 65535);
  const int per = (n + nchunk - 1) / nchunk;
  // With 4+ chunks the first and last are a quarter size, which shortens the
  // pipeline fill (first H2D before any compute) and drain (last compute +
  // D2H after the final H2D) of every synchronous call.
  std::vector<std::pair<int, int>> chunks;
  const int edge = nchunk >= 4 ? std::max(1, per / 4) : per;
  int n0 = 0;
  if (nchunk >= 4) {
    chunks.push_back({0, edge});
    n0 = edge;
  }
  const int tail = nchunk >= 4 ? std::min(edge, n - n0) : 0;
  while (n0 < n - tail) {
    const int nb = std::min(per, n - tail - n0);
    chunks.push_back({n0, nb});
    n0 += nb;
  }
  if (tail > 0) chunks.push_back({n0, tail});
  return chunks;
}

// SCONV_F_CACHE_FILTERS: the cached slab for (pointer, shape), or nullptr.
sconv_filter_entry* find_filters(sconv_cu_ctx* ctx, const float* src, bool host, int k, int c, int kk,
                                 int kp) {
  for (sconv_filter_entry& e : ctx->fcache)
    if (e.src == src && e.host == host && e.k == k && e.c == c && e.kk == kk && e.kp == kp) return &e;
  return nullptr;
}

void free_filter_entry(sconv_filter_entry& e) {
  if (e.dev) cudaFree(e.dev);
  if (e.wt) cudaFree(e.wt);
  e.dev = e.wt = nullptr;
}

// The lanes-over-pixels small-C kernel reads its filters from the constant
// bank (c_sc2_w).  A launch takes one of kSc2Slots slots per device, copies its
// [C][9][64] K-block there on its stream (D2D), and records an event the next
// user of the slot waits on, so launches on any streams / contexts never see
// each other's filters.  A stream that is capturing a graph uses the
// per-tile kernel instead (the slot's event would cross the capture).
struct Sc2SlotTable {
  std::mutex mu;
  int next = 0;
  cudaEvent_t ev[kSc2Slots] = {};
  float* base = nullptr;  // device address of c_sc2_w (floats)
};
Sc2SlotTable& sc2_slots(int device) {
  static std::mutex mu;
  static std::map<int, std::unique_ptr<Sc2SlotTable>> tables;  // one per device
  std::lock_guard<std::mutex> lock(mu);
  std::unique_ptr<Sc2SlotTable>& t = tables[device];
  if (!t) t.reset(new Sc2SlotTable);
  return *t;
}

template <int C, bool FAST, bool RELU, bool TMA>
int launch_smallc2_c(sconv_cu_ctx* ctx, cudaStream_t cs, SmallC2Args a, const float* wt,
                     const CUtensorMap& ymap) {
  auto kern = ecr_smallc2_kernel<C, FAST, RELU, TMA>;
  const int smem = sc2_smem_bytes(C, 64);
  static std::once_flag attr_once[64];
  cudaError_t attr_err = cudaSuccess;
  std::call_once(attr_once[ctx->device & 63], [&] {
    attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  });
  CK(attr_err);
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem));
  const long grid = std::min<long>((a.total_items + kSc2Warps - 1) / kSc2Warps,
                                   long(std::max(1, per_sm)) * ctx->num_sms);
  Sc2SlotTable& t = sc2_slots(ctx->device);
  std::lock_guard<std::mutex> lock(t.mu);
  if (!t.base) CK(cudaGetSymbolAddress(reinterpret_cast<void**>(&t.base), c_sc2_w));
  for (int kb = 0; kb < a.Kp / 64; ++kb) {
    const int slot = t.next;
    t.next = (t.next + 1) % kSc2Slots;
    if (t.ev[slot]) CK(cudaStreamWaitEvent(cs, t.ev[slot], 0));
    else CK(cudaEventCreateWithFlags(&t.ev[slot], cudaEventDisableTiming));
    CK(cudaMemcpy2DAsync(t.base + size_t(slot) * kSc2SlotFloats, 64 * sizeof(float), wt + kb * 64,
                         size_t(a.Kp) * sizeof(float), 64 * sizeof(float), size_t(C) * 9,
                         cudaMemcpyDeviceToDevice, cs));
    a.slot = slot;
    a.k0 = kb * 64;
    kern<<<static_cast<unsigned>(grid), 256, smem, cs>>>(a, ymap);
    TRY(finish_launch(ctx, "ecr_smallc2_kernel"));
    CK(cudaEventRecord(t.ev[slot], cs));
  }
  return SCONV_OK;
}

template <int C, bool FAST>
int launch_smallc2_t(sconv_cu_ctx* ctx, cudaStream_t cs, const SmallC2Args& a, const float* wt) {
  // outputs by TMA store when the row pitch allows a tensor map (OW % 4 == 0)
  CUtensorMap ymap;
  std::memset(&ymap, 0, sizeof(ymap));
  bool tma = a.OW % 4 == 0 && !std::getenv("SCONV_SC2_STG");
  if (tma) {
    const CUresult r = encode_output_map(a.y, a.N, a.K, a.OH, a.OW, 32, kSc2Rows, kSc2BoxK, &ymap);
    tma = r == CUDA_SUCCESS;
  }
  if (tma) return a.relu ? launch_smallc2_c<C, FAST, true, true>(ctx, cs, a, wt, ymap)
                         : launch_smallc2_c<C, FAST, false, true>(ctx, cs, a, wt, ymap);
  return a.relu ? launch_smallc2_c<C, FAST, true, false>(ctx, cs, a, wt, ymap)
                : launch_smallc2_c<C, FAST, false, false>(ctx, cs, a, wt, ymap);
}

int launch_smallc2(sconv_cu_ctx* ctx, cudaStream_t cs, const float* dx, const float* wt, float* dy,
                   int nb, int c, int h, int w, int k, int Kp, int OH, int OW, int relu, bool fast) {
  const int bands = (OH + kSc2Rows - 1) / kSc2Rows, strips = (OW + 31) / 32;
  if (nb == 0 || bands == 0 || strips == 0) return SCONV_OK;
  // the kernel splits (item, filter group) units with 32-bit arithmetic
  const int per = std::max(1, static_cast<int>(std::min<long>(nb, (1L << 26) / (long(bands) * strips))));
  for (int n0 = 0; n0 < nb; n0 += per) {
    const int m = std::min(per, nb - n0);
    SmallC2Args a{dx + size_t(n0) * c * h * w, wt, dy + size_t(n0) * k * OH * OW, m, c, h, w, k, Kp,
                  OH, OW, bands, strips, m * bands * strips, relu, 0, 0};
    int rc = SCONV_OK;
    switch (c * 2 + (fast ? 1 : 0)) {
      case 2: rc = launch_smallc2_t<1, false>(ctx, cs, a, wt); break;
      case 3: rc = launch_smallc2_t<1, true>(ctx, cs, a, wt); break;
      case 4: rc = launch_smallc2_t<2, false>(ctx, cs, a, wt); break;
      case 5: rc = launch_smallc2_t<2, true>(ctx, cs, a, wt); break;
      case 6: rc = launch_smallc2_t<3, false>(ctx, cs, a, wt); break;
      case 7: rc = launch_smallc2_t<3, true>(ctx, cs, a, wt); break;
      case 8: rc = launch_smallc2_t<4, false>(ctx, cs, a, wt); break;
      case 9: rc = launch_smallc2_t<4, true>(ctx, cs, a, wt); break;
      default: return fail(ctx, SCONV_ERR_ARG, "small-C kernel: C = %d", c);
    }
    TRY(rc);
  }
  return SCONV_OK;
}

// One kernel launch over images [0, nb) of a chunk (device buffers).
int launch_chunk(sconv_cu_ctx* ctx, const KernelChoice& ch, cudaStream_t cs, const float* dx,
                 const float* dw, const float* wt, float* dconv, float* dy, int nb, int c, int h,
                 int w, int k, int Kp, int kh, int kw, int stride, int OH, int OW, int pw, int ph,
                 int ps, int mode, int PHo, int PWo, bool pecr, bool fast) {
  const int model = ch.pool_after ? 0 : mode;
  cudaStreamCaptureStatus capturing = cudaStreamCaptureStatusNone;
  if (ch.sc2) CK(cudaStreamIsCapturing(cs, &capturing));
  if (ch.sc2 && capturing == cudaStreamCaptureStatusNone) {
    TRY(launch_smallc2(ctx, cs, dx, wt, dconv, nb, c, h, w, k, Kp, OH, OW, model, fast));
  } else if (ch.smallc) {
    SmallCArgs a{dx, wt, dconv, nb, c, h, w, k, Kp, OH, OW, 0, 0, 0, model};
    if (ch.P < 0) {  // tiles of whole pool windows
      const int pth = (4 - ph) / ps + 1, ptw = (4 - pw) / ps + 1;
      a.pw = pw, a.ph = ph, a.ps = ps, a.PHo = PHo, a.PWo = PWo;
      a.tsy = pth * ps, a.tsx = ptw * ps;
      a.tiles_x = (PWo + ptw - 1) / ptw;
      a.tiles_per_img = a.tiles_x * ((PHo + pth - 1) / pth);
    } else {
      a.tiles_x = (OW + 3) / 4;
      a.tiles_per_img = a.tiles_x * ((OH + 3) / 4);
    }
    a.total_tiles = a.tiles_per_img * nb;
    const dim3 grid((a.total_tiles + 7) / 8, (k + 63) / 64);
    if (ch.P < 0)
      fast ? ecr_smallc_kernel<-1, true><<<grid, 256, 0, cs>>>(a)
           : ecr_smallc_kernel<-1, false><<<grid, 256, 0, cs>>>(a);
    else if (ch.P == 2)
      fast ? ecr_smallc_kernel<2, true><<<grid, 256, 0, cs>>>(a)
           : ecr_smallc_kernel<2, false><<<grid, 256, 0, cs>>>(a);
    else
      fast ? ecr_smallc_kernel<0, true><<<grid, 256, 0, cs>>>(a)
           : ecr_smallc_kernel<0, false><<<grid, 256, 0, cs>>>(a);
    TRY(finish_launch(ctx, "ecr_smallc_kernel"));
  } else if (ch.pw) {
    const long long cols = static_cast<long long>(nb) * OH * OW;
    PwArgs a{dx, wt, dconv, nb, c, OH * OW, k, Kp, cols, model};
    int bm, bn;
    pw_dims(ch.pw, &bm, &bn);
    const dim3 grid(static_cast<unsigned>((cols + bn - 1) / bn), static_cast<unsigned>((k + bm - 1) / bm));
#define SCONV_PW_LAUNCH(BM, BN, TM, TN)                                                          \
  (fast ? pw_gemm_kernel<BM, BN, TM, TN, true><<<grid, PwCfg<BM, BN, TM, TN>::NT, 0, cs>>>(a)   \
        : pw_gemm_kernel<BM, BN, TM, TN, false><<<grid, PwCfg<BM, BN, TM, TN>::NT, 0, cs>>>(a))
    if (ch.pw == 1)
      SCONV_PW_LAUNCH(128, 128, 8, 8);
    else
      SCONV_PW_LAUNCH(64, 128, 8, 8);
#undef SCONV_PW_LAUNCH
    TRY(finish_launch(ctx, "pw_gemm_kernel"));
  } else if (ch.ws) {
    WsArgs a{dx, wt, dconv, nb, c, h, w, k, Kp, OH, OW, 0, 0, 0, model};
    if (ch.P < 0) a.pw = pw, a.ph = ph, a.ps = ps, a.PHo = PHo, a.PWo = PWo;
    TRY(fast ? launch_ws_fast(ctx, ch.ws, ch.P, a) : launch_ws_exact(ctx, ch.ws, ch.P, a));
  } else if (ch.which) {
    TiledArgs a{dx, wt, dconv, c, h, w, k, OH, OW, 0, model};
    TRY(launch_tiled(ctx, fast, ch.which, ch.P, a, nb));
  } else {
    GenericArgs a{dx, dw, dy, nb, c, h, w, k, kh, kw, stride, OH, OW, pw, ph, ps, mode, PHo, PWo};
    const size_t y_img = pecr ? size_t(k) * PHo * PWo : size_t(k) * OH * OW;
    const unsigned g = grid_for(size_t(nb) * y_img, 256, ctx->num_sms);
    if (pecr) {
      fast ? pecr_generic_kernel<true><<<g, 256, 0, cs>>>(a) : pecr_generic_kernel<false><<<g, 256, 0, cs>>>(a);
      TRY(finish_launch(ctx, "pecr_generic_kernel"));
    } else {
      fast ? ecr_generic_kernel<true><<<g, 256, 0, cs>>>(a) : ecr_generic_kernel<false><<<g, 256, 0, cs>>>(a);
      TRY(finish_launch(ctx, "ecr_generic_kernel"));
    }
  }
  if (ch.pool_after) {
    const size_t planes = size_t(nb) * k;
    pecr_pool_fold_kernel<<<grid_for(planes * PHo * PWo, 256, ctx->num_sms), 256, 0, cs>>>(
        dconv, dy, planes, OH, OW, pw, ph, ps, mode, PHo, PWo);
    TRY(finish_launch(ctx, "pecr_pool_fold_kernel"));
  }
  return SCONV_OK;
}

// A batch in the compressed-ingest layout (include/sconv_cuda.h).
struct PackedIn {
  const uint32_t* bits;
  const int64_t* base;
  const float* values;
};

// Expands images [n0, n0 + nb) of a packed batch into dense x (device).
// bits / base point at image n0's; values[0] is the absolute offset value0.
int expand_chunk(sconv_cu_ctx* ctx, cudaStream_t cs, const uint32_t* bits, const int64_t* base,
                 const float* values, int64_t value0, int nb, int64_t elems, float* x) {
  int64_t words = (elems + 31) / 32, blocks = (words + 31) / 32;
  ExpandArgs ea{bits, base, values, value0, nb, elems, words, blocks, x};
  const size_t warps = size_t(nb) * blocks;
  expand_packed_kernel<<<grid_for(warps * 32, 256, ctx->num_sms * 8), 256, 0, cs>>>(ea);
  return finish_launch(ctx, "expand_packed_kernel");
}

// Shared body of the fused ECR / PECR entries.  `pk`: the input comes in the
// compressed-ingest layout instead of dense x (x unused).
int fused_conv(sconv_cu_ctx* ctx, const float* x, int n, int c, int h, int w, const float* filt,
               int k, int kh, int kw, int stride, int pw, int ph, int ps, int mode, float* y,
               uint64_t* muls, uint64_t* adds, unsigned flags, const PackedIn* pk = nullptr) {
  if (!ctx) return fail(nullptr, SCONV_ERR_ARG, "null context");
  const bool pecr = pw > 0;
  if (n < 0 || k < 0) return fail(ctx, SCONV_ERR_SHAPE, "negative batch or filter count");
  if (c < 1) return fail(ctx, SCONV_ERR_SHAPE, "channels must be positive");
  int OW, OH;
  TRY(conv_dims(ctx, w, h, kw, kh, stride, &OW, &OH));
  int PWo = 0, PHo = 0;
  if (pecr) {
    if (mode != SCONV_POOL_MAX && mode != SCONV_POOL_MEAN)
      return fail(ctx, SCONV_ERR_CONFIG, "unknown pool mode %d", mode);
    TRY(pack_count(ctx, w, kw, stride, pw, ps, &PWo));
    TRY(pack_count(ctx, h, kh, stride, ph, ps, &PHo));
  }
  const bool dev = flags & SCONV_F_DEVICE, async = flags & SCONV_F_ASYNC, fast = flags & SCONV_F_FAST;
  if (async && (muls || adds)) return fail(ctx, SCONV_ERR_ARG, "counters need a synchronous call");
  // async host pointers: the call returns after enqueueing; x must stay
  // unchanged and y unread until sconv_cu_synchronize (pinned memory for
  // the copies to overlap).
  const bool host_async = async && !dev;
  if (n == 0 || k == 0) return SCONV_OK;
  const bool packed = pk != nullptr;
  if (packed) x = nullptr;
  if ((!packed && !x) || (packed && (!pk->bits || !pk->base)) || !filt || !y)
    return fail(ctx, SCONV_ERR_ARG, "null tensor pointer");
  if (dev && ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15))
    return fail(ctx, SCONV_ERR_ARG, "device x and y must be 16-byte aligned");
  KernelChoice ch;
  TRY(choose_kernel(ctx, n, c, k, kh, kw, stride, OH, OW, pecr, pw, ph, ps, flags, &ch));

  const size_t x_elems = size_t(n) * c * h * w, w_elems = size_t(k) * c * kh * kw;
  const size_t y_elems = pecr ? size_t(n) * k * PHo * PWo : size_t(n) * k * OH * OW;
  const int Kp = ch.smallc ? (k + 63) / 64 * 64 : ch.which ? k : (k + 3) / 4 * 4;
  const bool counters = muls || adds;
  const bool need_wt = ch.tiled();
  const bool cache = flags & SCONV_F_CACHE_FILTERS;

  DeviceGuard guard(ctx->device);
  const std::vector<std::pair<int, int>> chunks =
      plan_chunks(ctx, ch, n, k, OH, OW, x_elems, y_elems, dev, async, pw, ph, ps);
  const int nchunk = static_cast<int>(chunks.size());
  int per = 0;
  for (const auto& cp : chunks) per = std::max(per, cp.second);
  const size_t x_img = size_t(c) * h * w, y_img = y_elems / size_t(n);
  const int nbuf = dev ? 0 : std::min(nchunk, 3);
  const bool piped = !dev && nchunk > 1;
  // compressed ingest: per-image bitmap words / block offsets, and (host
  // pointers) the value count of every chunk, read off the host offsets
  const int64_t pk_words = (int64_t(x_img) + 31) / 32, pk_blocks = (pk_words + 31) / 32;
  std::vector<int64_t> chunk_v0(nchunk, 0), chunk_nv(nchunk, 0);
  int64_t pk_vmax = 0;
  if (packed && !dev) {
    for (int ci = 0; ci < nchunk; ++ci) {
      const int n0 = chunks[ci].first, nb = chunks[ci].second;
      chunk_v0[ci] = pk->base[int64_t(n0) * (pk_blocks + 1)];
      chunk_nv[ci] = pk->base[int64_t(n0 + nb - 1) * (pk_blocks + 1) + pk_blocks] - chunk_v0[ci];
      if (chunk_nv[ci] < 0) return fail(ctx, SCONV_ERR_FORMAT, "packed offsets decrease");
      if (chunk_nv[ci] > 0 && !pk->values) return fail(ctx, SCONV_ERR_ARG, "null packed values");
      pk_vmax = std::max(pk_vmax, chunk_nv[ci]);
    }
  }

  // Filters for SCONV_F_CACHE_FILTERS: the context's copy, made on first use.
  sconv_filter_entry* fe = cache ? find_filters(ctx, filt, !dev, k, c, kh * kw, need_wt ? Kp : 0) : nullptr;
  const bool fresh = cache && !fe;
  if (fresh) {
    if (ctx->fcache.size() >= 64) {  // bounded: drop the oldest entry
      CK(cudaDeviceSynchronize());
      free_filter_entry(ctx->fcache.front());
      ctx->fcache.erase(ctx->fcache.begin());
    }
    sconv_filter_entry e{filt, !dev, k, c, kh * kw, need_wt ? Kp : 0, nullptr, nullptr};
    if (!dev) CK(cudaMalloc(&e.dev, w_elems * 4));
    if (need_wt) CK(cudaMalloc(&e.wt, size_t(Kp) * c * kh * kw * 4));
    ctx->fcache.push_back(e);
    fe = &ctx->fcache.back();
  }

  Arena ar{ctx, {}};
  if (host_async) {  // take the next host workspace once its previous call is done
    ar.host = ctx->hws_next;
    ctx->hws_next = (ctx->hws_next + 1) % ctx->hws_n;
    if (!ctx->ev_hws[ar.host]) CK(cudaEventCreateWithFlags(&ctx->ev_hws[ar.host], cudaEventDisableTiming));
    else CK(cudaEventSynchronize(ctx->ev_hws[ar.host]));
  }
  size_t i_x[3] = {0, 0, 0}, i_y[3] = {0, 0, 0}, i_pix[3] = {0, 0, 0};
  size_t i_pb[3] = {0, 0, 0}, i_pbase[3] = {0, 0, 0}, i_pv[3] = {0, 0, 0};
  for (int b = 0; b < nbuf; ++b) {
    i_x[b] = ar.add(size_t(per) * x_img * 4);
    i_y[b] = ar.add(size_t(per) * y_img * 4);
    if (packed) {  // the chunk as it crosses PCIe
      i_pb[b] = ar.add(size_t(per) * pk_words * 4);
      i_pbase[b] = ar.add(size_t(per) * (pk_blocks + 1) * 8);
      i_pv[b] = ar.add(size_t(std::max<int64_t>(pk_vmax, 1)) * 4);
    }
  }
  if (dev && packed) i_x[0] = ar.add(size_t(per) * x_img * 4);  // expansion target
  const size_t i_w = dev || fe ? 0 : ar.add(w_elems * 4);
  const size_t i_wt = need_wt && !fe ? ar.add(size_t(Kp) * c * kh * kw * 4) : 0;
  for (int b = 0; b < (counters ? std::max(nbuf, 1) : 0); ++b) i_pix[b] = ar.add(size_t(per) * h * w * 4);
  const size_t i_conv = ch.pool_after ? ar.add(size_t(per) * k * OH * OW * 4) : 0;
  const size_t i_ops = ar.add(64);
  std::vector<char*> p;
  TRY(ar.commit(p));
  const float* dw = dev ? filt : fe ? fe->dev : reinterpret_cast<float*>(p[i_w]);
  auto* dops = reinterpret_cast<unsigned long long*>(p[i_ops]);
  const float* wt = !need_wt ? nullptr : fe ? fe->wt : reinterpret_cast<float*>(p[i_wt]);
  cudaStream_t st = ctx->stream;
  if (piped && !ctx->h2d) {
    CK(cudaStreamCreateWithFlags(&ctx->h2d, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&ctx->d2h, cudaStreamNonBlocking));
    for (int b = 0; b < 3; ++b) {
      CK(cudaEventCreateWithFlags(&ctx->ev_in[b], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ctx->ev_comp[b], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ctx->ev_out[b], cudaEventDisableTiming));
    }
    CK(cudaEventCreateWithFlags(&ctx->ev_done, cudaEventDisableTiming));
  }

  if (piped && host_async && ar.grew) {  // the new workspace exists in ctx->stream order
    CK(cudaEventRecord(ctx->ev_done, st));
    CK(cudaStreamWaitEvent(ctx->h2d, ctx->ev_done, 0));
    CK(cudaStreamWaitEvent(ctx->d2h, ctx->ev_done, 0));
  }
  // Filters: copy (host path) and re-layout for the tiled kernels, once per
  // call -- or once per cached slab.  Async host calls send them on the H2D
  // stream, ahead of this call's input chunks: issued on the context stream
  // they would queue behind every input copy already submitted to the H2D
  // engine (the previous calls' inputs).
  if (!dev && (!fe || fresh)) {
    if (host_async && piped) {
      CK(cudaMemcpyAsync(const_cast<float*>(dw), filt, w_elems * 4, cudaMemcpyHostToDevice, ctx->h2d));
      CK(cudaEventRecord(ctx->ev_done, ctx->h2d));
      CK(cudaStreamWaitEvent(st, ctx->ev_done, 0));
    } else {
      CK(cudaMemcpyAsync(const_cast<float*>(dw), filt, w_elems * 4, cudaMemcpyHostToDevice, st));
    }
  }
  if (need_wt && (!fe || fresh)) {
    const dim3 tgrid((Kp + 31) / 32, static_cast<unsigned>((size_t(c) * kh * kw + 31) / 32));
    transpose_filters_kernel<<<tgrid, dim3(32, 8), 0, st>>>(dw, const_cast<float*>(wt), k, Kp, c, kh * kw);
    TRY(finish_launch(ctx, "transpose_filters_kernel"));
  }
  if (counters) CK(cudaMemsetAsync(dops, 0, 16, st));
  if (piped && !host_async) {  // the copy streams start after everything queued so far
    CK(cudaEventRecord(ctx->ev_done, st));
    CK(cudaStreamWaitEvent(ctx->h2d, ctx->ev_done, 0));
    CK(cudaStreamWaitEvent(ctx->d2h, ctx->ev_done, 0));
  }
  // (async host calls own fresh ring slots: their first H2D copies need not
  // wait for the previous call's compute or D2H)

  for (int ci = 0; ci < nchunk; ++ci) {
    const int n0 = chunks[ci].first, nb = chunks[ci].second;
    if (nb <= 0) break;
    const int b = dev ? 0 : ci % nbuf;
    cudaStream_t cs = st;
    float* xslot = (!dev || packed) ? reinterpret_cast<float*>(p[i_x[b]]) : nullptr;
    const float* dx = (dev && !packed) ? x + size_t(n0) * x_img : xslot;
    float* dy = dev ? y + size_t(n0) * y_img : reinterpret_cast<float*>(p[i_y[b]]);
    float* dconv = ch.pool_after ? reinterpret_cast<float*>(p[i_conv]) : dy;  // conv kernels write here
    if (!dev) {
      cudaStream_t hs = piped ? ctx->h2d : st;
      if (piped && ci >= nbuf) CK(cudaStreamWaitEvent(hs, ctx->ev_comp[b], 0));  // x slot free
      if (packed) {  // bitmap, block offsets and nonzeros of the chunk's images
        CK(cudaMemcpyAsync(p[i_pb[b]], pk->bits + int64_t(n0) * pk_words,
                           size_t(nb) * pk_words * 4, cudaMemcpyHostToDevice, hs));
        CK(cudaMemcpyAsync(p[i_pbase[b]], pk->base + int64_t(n0) * (pk_blocks + 1),
                           size_t(nb) * (pk_blocks + 1) * 8, cudaMemcpyHostToDevice, hs));
        if (chunk_nv[ci] > 0)
          CK(cudaMemcpyAsync(p[i_pv[b]], pk->values + chunk_v0[ci], size_t(chunk_nv[ci]) * 4,
                             cudaMemcpyHostToDevice, hs));
      } else {
        CK(cudaMemcpyAsync(const_cast<float*>(dx), x + size_t(n0) * x_img, size_t(nb) * x_img * 4,
                           cudaMemcpyHostToDevice, hs));
      }
      if (piped) {
        CK(cudaEventRecord(ctx->ev_in[b], hs));
        CK(cudaStreamWaitEvent(cs, ctx->ev_in[b], 0));
        if (ci >= nbuf) CK(cudaStreamWaitEvent(cs, ctx->ev_out[b], 0));  // y slot drained
      }
    }
    if (packed) {  // compressed ingest: dense chunk rebuilt in HBM, then the conv
      if (dev)
        TRY(expand_chunk(ctx, cs, pk->bits + int64_t(n0) * pk_words,
                         pk->base + int64_t(n0) * (pk_blocks + 1), pk->values, 0, nb, x_img, xslot));
      else
        TRY(expand_chunk(ctx, cs, reinterpret_cast<uint32_t*>(p[i_pb[b]]),
                         reinterpret_cast<int64_t*>(p[i_pbase[b]]), reinterpret_cast<float*>(p[i_pv[b]]),
                         chunk_v0[ci], nb, x_img, xslot));
    }
    TRY(launch_chunk(ctx, ch, cs, dx, dw, wt, dconv, dy, nb, c, h, w, k, Kp, kh, kw, stride, OH, OW,
                     pw, ph, ps, mode, PHo, PWo, pecr, fast));
    if (counters) {  // integer atomics: order-free across chunks
      int32_t* pix = reinterpret_cast<int32_t*>(p[i_pix[b]]);
      pixel_nnz_kernel<<<grid_for(size_t(nb) * h * w, 256, ctx->num_sms), 256, 0, cs>>>(dx, nb, c, h,
                                                                                       w, pix);
      TRY(finish_launch(ctx, "pixel_nnz_kernel"));
      OpsArgs oa{pix, nb, h, w, kh, kw, stride, OH, OW, PHo, PWo, pecr ? pw : 0, ph, ps, dops};
      const size_t items = pecr ? size_t(nb) * PHo * PWo : size_t(nb) * OH * OW;
      ops_kernel<<<grid_for(items, 256, ctx->num_sms), 256, 0, cs>>>(oa);
      TRY(finish_launch(ctx, "ops_kernel"));
    }
    if (!dev) {
      cudaStream_t ds = piped ? ctx->d2h : st;
      if (piped) {
        CK(cudaEventRecord(ctx->ev_comp[b], cs));
        CK(cudaStreamWaitEvent(ds, ctx->ev_comp[b], 0));
      }
      CK(cudaMemcpyAsync(y + size_t(n0) * y_img, dy, size_t(nb) * y_img * 4, cudaMemcpyDeviceToHost,
                         ds));
      if (piped) CK(cudaEventRecord(ctx->ev_out[b], ds));
    }
  }
  if (host_async) {
    // the workspace is free once the last D2H (which follows the last kernel)
    // and the whole of the context stream's work for this call are done
    cudaStream_t ds = piped ? ctx->d2h : st;
    if (piped) {
      CK(cudaEventRecord(ctx->ev_done, st));
      CK(cudaStreamWaitEvent(ds, ctx->ev_done, 0));
    }
    CK(cudaEventRecord(ctx->ev_hws[ar.host], ds));
  } else if (piped) {  // join the copy streams back into the context stream
    CK(cudaEventRecord(ctx->ev_done, ctx->d2h));
    CK(cudaStreamWaitEvent(st, ctx->ev_done, 0));
    CK(cudaEventRecord(ctx->ev_done, ctx->h2d));
    CK(cudaStreamWaitEvent(st, ctx->ev_done, 0));
  }
  if (counters) {
    unsigned long long hops[2];
    CK(cudaMemcpyAsync(hops, dops, 16, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    // nnz is filter independent: every filter sees the same windows
    if (muls) *muls += hops[0] * static_cast<uint64_t>(k);
    if (adds) *adds += hops[1] * static_cast<uint64_t>(k);
  }
  if (!async) CK(cudaStreamSynchronize(st));
  return SCONV_OK;
}

template <typename F>
int run_multi(sconv_cu_ctx** ctxs, int nctx, int n, int k, size_t in_per_img, size_t w_per_filt,
              size_t out_per_map, const float* x, const float* filters, float* y, uint64_t* muls,
              uint64_t* adds, F&& call) {
  if (!ctxs || nctx < 1) return fail(nullptr, SCONV_ERR_ARG, "no contexts");
  std::vector<int> rc(nctx, SCONV_OK);
  std::vector<uint64_t> m(nctx, 0), a(nctx, 0);
  std::vector<std::vector<float>> tmp(nctx);
  std::vector<std::thread> pool;
  for (int r = 0; r < nctx; ++r) {
    pool.emplace_back([&, r] {
      int n0, n1, k0, k1;
      sconv_shard(n, k, nctx, r, &n0, &n1, &k0, &k1);
      if (n1 <= n0 || k1 <= k0) return;
      const bool ksplit = (k1 - k0) != k;
      float* out = y + size_t(n0) * k * out_per_map;
      if (ksplit) {
        tmp[r].resize(size_t(n1 - n0) * (k1 - k0) * out_per_map);
        out = tmp[r].data();
      }
      rc[r] = call(ctxs[r], x + size_t(n0) * in_per_img, n1 - n0, filters + size_t(k0) * w_per_filt,
                   k1 - k0, out, (muls ? &m[r] : nullptr), (adds ? &a[r] : nullptr));
      if (rc[r] == SCONV_OK && ksplit) {
        for (int i = 0; i < n1 - n0; ++i)
          std::memcpy(y + (size_t(n0 + i) * k + k0) * out_per_map,
                      tmp[r].data() + size_t(i) * (k1 - k0) * out_per_map,
                      size_t(k1 - k0) * out_per_map * 4);
      }
    });
  }
  for (auto& t : pool) t.join();
  for (int r = 0; r < nctx; ++r)
    if (rc[r] != SCONV_OK) {
      g_noctx_err = ctxs[r]->err;
      return rc[r];
    }
  for (int r = 0; r < nctx; ++r) {
    if (muls) *muls += m[r];
    if (adds) *adds += a[r];
  }
  return SCONV_OK;
}

}  // namespace

extern "C" {

const char* sconv_cu_version(void) { return "sconv_cuda 1 (sm_100a)"; }

int sconv_cu_device_count(int* count) {
  if (!count) return SCONV_ERR_ARG;
  const cudaError_t e = cudaGetDeviceCount(count);
  if (e != cudaSuccess) {
    *count = 0;
    return fail(nullptr, SCONV_ERR_CUDA, "cudaGetDeviceCount: %s", cudaGetErrorString(e));
  }
  return SCONV_OK;
}

int sconv_cu_ctx_create(int device, sconv_cu_ctx** out) {
  if (!out) return SCONV_ERR_ARG;
  *out = nullptr;
  sconv_cu_ctx* ctx = nullptr;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || device < 0 || device >= ndev)
    return fail(nullptr, SCONV_ERR_CUDA, "no CUDA device %d (%s)", device,
                e != cudaSuccess ? cudaGetErrorString(e) : "out of range");
  cudaDeviceProp prop;
  e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) return fail(nullptr, SCONV_ERR_CUDA, "%s", cudaGetErrorString(e));
  if (prop.major != 10)
    return fail(nullptr, SCONV_ERR_CUDA, "device %d is sm_%d%d; this library is built for sm_100a",
                device, prop.major, prop.minor);
  ctx = new sconv_cu_ctx();
  ctx->device = device;
  ctx->num_sms = prop.multiProcessorCount;
  {  // async host-call workspaces come from the context's own memory pool,
     // which keeps freed blocks mapped instead of trimming them at every sync
     // point (the device's default pool, which the application may use, is
     // left alone)
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    e = cudaMemPoolCreate(&ctx->pool, &props);
    if (e != cudaSuccess) {
      delete ctx;
      return fail(nullptr, SCONV_ERR_CUDA, "cudaMemPoolCreate: %s", cudaGetErrorString(e));
    }
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(ctx->pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  ctx->smem_optin = static_cast<int>(prop.sharedMemPerBlockOptin);
  DeviceGuard guard(device);
  e = cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete ctx;
    return fail(nullptr, SCONV_ERR_CUDA, "%s", cudaGetErrorString(e));
  }
  ctx->stream = ctx->own;
  e = cudaMalloc(&ctx->gate, sconv_cu_ctx::kGates * sizeof(int));
  if (e != cudaSuccess) {
    cudaStreamDestroy(ctx->own);
    cudaMemPoolDestroy(ctx->pool);
    delete ctx;
    return fail(nullptr, SCONV_ERR_CUDA, "%s", cudaGetErrorString(e));
  }
  if (const char* e = std::getenv("SCONV_HOST_ARENAS"))  // dev knob (tools/async_probe.py)
    ctx->hws_n = std::max(1, std::min(sconv_cu_ctx::kHostArenas, std::atoi(e)));
  *out = ctx;
  return SCONV_OK;
}

int sconv_cu_ctx_destroy(sconv_cu_ctx* ctx) {
  if (!ctx) return SCONV_ERR_ARG;
  {
    DeviceGuard guard(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->h2d) cudaStreamSynchronize(ctx->h2d);
    if (ctx->d2h) cudaStreamSynchronize(ctx->d2h);
    if (ctx->ws) cudaFree(ctx->ws);
    for (int a = 0; a < sconv_cu_ctx::kHostArenas; ++a) {
      if (ctx->ev_hws[a]) cudaEventSynchronize(ctx->ev_hws[a]);
      if (ctx->hws[a]) cudaFreeAsync(ctx->hws[a], ctx->stream);
      if (ctx->ev_hws[a]) cudaEventDestroy(ctx->ev_hws[a]);
    }
    cudaStreamSynchronize(ctx->stream);
    for (sconv_filter_entry& fe : ctx->fcache) free_filter_entry(fe);
    ctx->fcache.clear();
    if (ctx->pool) cudaMemPoolDestroy(ctx->pool);
    if (ctx->fwd) cudaFree(ctx->fwd);
    if (ctx->gate) cudaFree(ctx->gate);
    if (ctx->fwd_graph) cudaGraphExecDestroy(ctx->fwd_graph);
    if (ctx->ev_graph) cudaEventDestroy(ctx->ev_graph);
    if (ctx->own) cudaStreamDestroy(ctx->own);
    if (ctx->h2d) cudaStreamDestroy(ctx->h2d);
    if (ctx->d2h) cudaStreamDestroy(ctx->d2h);
    for (int b = 0; b < 3; ++b) {
      if (ctx->ev_in[b]) cudaEventDestroy(ctx->ev_in[b]);
      if (ctx->ev_comp[b]) cudaEventDestroy(ctx->ev_comp[b]);
      if (ctx->ev_out[b]) cudaEventDestroy(ctx->ev_out[b]);
    }
    if (ctx->ev_done) cudaEventDestroy(ctx->ev_done);
  }
  delete ctx;
  return SCONV_OK;
}

int sconv_cu_ctx_set_stream(sconv_cu_ctx* ctx, void* stream) {
  if (!ctx) return SCONV_ERR_ARG;
  DeviceGuard guard(ctx->device);
  CK(cudaStreamSynchronize(ctx->stream));  // workspace is stream-ordered
  ctx->stream = static_cast<cudaStream_t>(stream);
  return SCONV_OK;
}

int sconv_cu_ctx_use_own_stream(sconv_cu_ctx* ctx) {
  if (!ctx) return SCONV_ERR_ARG;
  DeviceGuard guard(ctx->device);
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->stream = ctx->own;
  return SCONV_OK;
}

void* sconv_cu_ctx_stream(sconv_cu_ctx* ctx) { return ctx ? ctx->stream : nullptr; }
int sconv_cu_ctx_device(sconv_cu_ctx* ctx) { return ctx ? ctx->device : -1; }

int sconv_cu_synchronize(sconv_cu_ctx* ctx) {
  if (!ctx) return SCONV_ERR_ARG;
  DeviceGuard guard(ctx->device);
  CK(cudaStreamSynchronize(ctx->stream));
  if (ctx->h2d) CK(cudaStreamSynchronize(ctx->h2d));  // async host-pointer calls
  if (ctx->d2h) CK(cudaStreamSynchronize(ctx->d2h));
  return SCONV_OK;
}

const char* sconv_cu_last_error(const sconv_cu_ctx* ctx) {
  return ctx ? ctx->err.c_str() : g_noctx_err.c_str();
}

uint64_t sconv_cu_launch_count(const sconv_cu_ctx* ctx) { return ctx ? ctx->launches : 0; }

int sconv_cu_release_filters(sconv_cu_ctx* ctx) {
  if (!ctx) return SCONV_ERR_ARG;
  DeviceGuard guard(ctx->device);
  CK(cudaDeviceSynchronize());  // cached slabs may be read by work in flight
  for (sconv_filter_entry& fe : ctx->fcache) free_filter_entry(fe);
  ctx->fcache.clear();
  ctx->tmaps.clear();
  return SCONV_OK;
}

int sconv_conv_output_dims(int in_w, int in_h, int k_w, int k_h, int stride, int* out_w,
                           int* out_h) {
  if (!out_w || !out_h) return SCONV_ERR_ARG;
  return conv_dims(nullptr, in_w, in_h, k_w, k_h, stride, out_w, out_h);
}

int sconv_pecr_pack_count(int in_extent, int k_extent, int conv_stride, int pool_extent,
                          int pool_stride, int* packs) {
  if (!packs) return SCONV_ERR_ARG;
  return pack_count(nullptr, in_extent, k_extent, conv_stride, pool_extent, pool_stride, packs);
}

int sconv_cu_plan(int n, int c, int h, int w, int k, int kh, int kw, int stride, int pool_w,
                  int pool_h, int pool_stride, unsigned flags, sconv_launch_plan* out) {
  if (!out) return SCONV_ERR_ARG;
  std::memset(out, 0, sizeof(*out));
  if (c < 1) return fail(nullptr, SCONV_ERR_SHAPE, "channels must be positive");
  int OW, OH;
  TRY(conv_dims(nullptr, w, h, kw, kh, stride, &OW, &OH));
  int PWo = OW, PHo = OH;
  if (pool_w > 0) {
    TRY(pack_count(nullptr, w, kw, stride, pool_w, pool_stride, &PWo));
    TRY(pack_count(nullptr, h, kh, stride, pool_h, pool_stride, &PHo));
  }
  KernelChoice ch;
  TRY(choose_kernel(nullptr, n, c, k, kh, kw, stride, OH, OW, pool_w > 0, pool_w, pool_h,
                    pool_stride, flags, &ch));
  const bool smallc = ch.smallc;
  const int ws = ch.ws, which = ch.which;
  if (ch.sc2) {  // persistent: grid = resident CTAs (at most one warp per item)
    const long items = long(n) * ((OH + kSc2Rows - 1) / kSc2Rows) * ((OW + 31) / 32);
    out->kernel = 301;
    out->grid_x = static_cast<int>(std::min<long>((items + kSc2Warps - 1) / kSc2Warps, 2L * 148));
    out->grid_y = out->grid_z = 1;
    out->block_threads = 256;
    out->smem_bytes = sc2_smem_bytes(c, (k + 63) / 64 * 64);
    out->tile_h = kSc2Rows;
    out->tile_w = 32;
    out->tile_k = 64;
  } else if (smallc) {
    const long tiles = long(n) * smallc_tiles(ch, OH, OW, pool_w, pool_h, pool_stride);
    out->kernel = 300;
    out->grid_x = static_cast<int>((tiles + 7) / 8);
    out->grid_y = (k + 63) / 64;
    out->grid_z = 1;
    out->block_threads = 256;
    out->smem_bytes = 8 * 48 * 4;
    out->tile_h = out->tile_w = 4;
    out->tile_k = 64;
  } else if (ch.pw) {
    int bm, bn;
    pw_dims(ch.pw, &bm, &bn);
    out->kernel = 400 + ch.pw;
    out->grid_x = static_cast<int>((long(n) * OH * OW + bn - 1) / bn);
    out->grid_y = (k + bm - 1) / bm;
    out->grid_z = 1;
    out->block_threads = bm / kPwTiles[ch.pw - 1].tm * (bn / kPwTiles[ch.pw - 1].tn);
    out->smem_bytes = 4 * 8 * (bm + bn) * 4;
    out->tile_h = 1;
    out->tile_w = bn;
    out->tile_k = bm;
  } else if (ws) {
    plan_ws(out, ws, n, k, OH, OW, ch.P < 0 ? pool_w : 0, pool_h, pool_stride);
  } else if (which) {
    plan_for(out, which, n, k, OH, OW);
  } else {
    const size_t work = size_t(n) * k * PHo * PWo;
    out->kernel = 0;
    out->grid_x = static_cast<int>(grid_for(work, 256, 148));
    out->grid_y = out->grid_z = 1;
    out->block_threads = 256;
    out->tile_h = out->tile_w = out->tile_k = 1;
  }
  return SCONV_OK;
}

// ---------------------------------------------------------------------------
// On-device multi-layer forward (forward(), src/pipeline.cpp:212-301)
// ---------------------------------------------------------------------------
namespace {

struct FwdLayerDims {
  int c, h, w;     // input
  int oh, ow;      // conv output
  int ph, pw;      // after pool (== oh, ow without pool)
};

// NetworkSpec::validate (src/pipeline.cpp:154-189) with the reference's error
// types, plus every layer's dims.
int forward_plan(sconv_cu_ctx* ctx, const sconv_layer* layers, int nl, int c, int h, int w,
                 std::vector<FwdLayerDims>* dims) {
  if (c < 1 || h < 1 || w < 1) return fail(ctx, SCONV_ERR_CONFIG, "network input dims must be positive");
  if (nl < 1 || !layers) return fail(ctx, SCONV_ERR_CONFIG, "network has no layers");
  dims->clear();
  for (int l = 0; l < nl; ++l) {
    const sconv_layer& L = layers[l];
    if (L.k < 1) return fail(ctx, SCONV_ERR_CONFIG, "layer %d: no filters", l);
    if (L.stride < 1) return fail(ctx, SCONV_ERR_CONFIG, "layer %d: conv stride must be >= 1", l);
    FwdLayerDims d{c, h, w, 0, 0, 0, 0};
    TRY(conv_dims(ctx, w, h, L.kw, L.kh, L.stride, &d.ow, &d.oh));
    d.pw = d.ow;
    d.ph = d.oh;
    if (L.pool_w != 0 || L.pool_h != 0) {
      if (L.pool_w < 1 || L.pool_h < 1) return fail(ctx, SCONV_ERR_SHAPE, "pool window must be positive");
      if (L.pool_stride < 1) return fail(ctx, SCONV_ERR_CONFIG, "pool stride must be >= 1");
      if (L.pool_mode != SCONV_POOL_MAX && L.pool_mode != SCONV_POOL_MEAN)
        return fail(ctx, SCONV_ERR_CONFIG, "layer %d: unknown pool mode %d", l, L.pool_mode);
      TRY(conv_dims(ctx, d.ow, d.oh, L.pool_w, L.pool_h, L.pool_stride, &d.pw, &d.ph));
    }
    dims->push_back(d);
    c = L.k;
    h = d.ph;
    w = d.pw;
  }
  return SCONV_OK;
}

}  // namespace

int sconv_cu_forward_dims(const sconv_layer* layers, int nlayers, int c, int h, int w, int* out_c,
                          int* out_h, int* out_w) {
  std::vector<FwdLayerDims> dims;
  TRY(forward_plan(nullptr, layers, nlayers, c, h, w, &dims));
  if (out_c) *out_c = layers[nlayers - 1].k;
  if (out_h) *out_h = dims.back().ph;
  if (out_w) *out_w = dims.back().pw;
  return SCONV_OK;
}

int sconv_cu_forward(sconv_cu_ctx* ctx, const float* x, int n, int c, int h, int w,
                     const sconv_layer* layers, int nlayers, int method, float* y,
                     float* const* layer_outputs, float* const* conv_outputs, uint64_t* muls,
                     uint64_t* adds, int32_t* pecr_fallback, unsigned flags) {
  if (!ctx) return fail(nullptr, SCONV_ERR_ARG, "null context");
  if (method != SCONV_METHOD_ECR && method != SCONV_METHOD_PECR)
    return fail(ctx, SCONV_ERR_CONFIG,
                "forward on the GPU runs the compressed methods (ECR, PECR); the dense method is "
                "the CPU reference's");
  if (n < 0) return fail(ctx, SCONV_ERR_SHAPE, "negative batch");
  if (flags & SCONV_F_ASYNC) return fail(ctx, SCONV_ERR_ARG, "forward is synchronous");
  std::vector<FwdLayerDims> dims;
  TRY(forward_plan(ctx, layers, nlayers, c, h, w, &dims));
  if (n == 0) return SCONV_OK;
  if (!x || !y) return fail(ctx, SCONV_ERR_ARG, "null tensor pointer");
  for (int l = 0; l < nlayers; ++l)
    if (!layers[l].filters) return fail(ctx, SCONV_ERR_ARG, "layer %d: null filters", l);
  const bool dev = flags & SCONV_F_DEVICE;
  const bool counters = muls || adds;
  if ((flags & SCONV_F_GRAPH) && (!dev || counters))
    return fail(ctx, SCONV_ERR_ARG, "SCONV_F_GRAPH needs device pointers and no counters");
  if (dev && ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y)) & 15))
    return fail(ctx, SCONV_ERR_ARG, "device x and y must be 16-byte aligned");

  // device residency: input, every layer's filters (host pointers only),
  // two activation buffers and one pre-pool conv buffer
  size_t act = size_t(c) * h * w, conv = 0, wtot = 0;
  for (int l = 0; l < nlayers; ++l) {
    const FwdLayerDims& d = dims[l];
    act = std::max(act, size_t(layers[l].k) * d.ph * d.pw);
    conv = std::max(conv, size_t(layers[l].k) * d.oh * d.ow);
    wtot += size_t(layers[l].k) * d.c * layers[l].kh * layers[l].kw;
  }
  auto up = [](size_t b) { return (b + 255) & ~size_t{255}; };
  const size_t b_act = up(size_t(n) * act * 4), b_conv = up(size_t(n) * conv * 4);
  const size_t b_w = dev ? 0 : up(wtot * 4);
  const size_t need = 2 * b_act + b_conv + b_w;
  DeviceGuard guard(ctx->device);
  cudaStream_t st = ctx->stream;
  if (need > ctx->fwd_cap) {
    CK(cudaStreamSynchronize(st));
    if (ctx->fwd) CK(cudaFree(ctx->fwd));
    ctx->fwd = nullptr;
    ctx->fwd_cap = 0;
    ctx->mem_gen++;
    CK(cudaMalloc(&ctx->fwd, need));
    ctx->fwd_cap = need;
  }
  float* buf[2] = {reinterpret_cast<float*>(ctx->fwd), reinterpret_cast<float*>(ctx->fwd + b_act)};
  float* cbuf = reinterpret_cast<float*>(ctx->fwd + 2 * b_act);
  float* wdev = reinterpret_cast<float*>(ctx->fwd + 2 * b_act + b_conv);
  std::vector<const float*> filt(nlayers);
  {  // one-time ingest (forward's h2d accounting, pipeline.cpp:222-227)
    size_t off = 0;
    for (int l = 0; l < nlayers; ++l) {
      const size_t cnt = size_t(layers[l].k) * dims[l].c * layers[l].kh * layers[l].kw;
      if (dev) {
        filt[l] = layers[l].filters;
      } else {
        CK(cudaMemcpyAsync(wdev + off, layers[l].filters, cnt * 4, cudaMemcpyHostToDevice, st));
        filt[l] = wdev + off;
      }
      off += cnt;
    }
  }
  const float* cur0 = x;
  if (!dev) {
    CK(cudaMemcpyAsync(buf[0], x, size_t(n) * c * h * w * 4, cudaMemcpyHostToDevice, st));
    cur0 = buf[0];
  }
  const unsigned kflags = (flags & (SCONV_F_FAST | SCONV_F_GENERIC | (0xffu << 8))) | SCONV_F_DEVICE |
                          (counters ? 0u : SCONV_F_ASYNC);
  const cudaMemcpyKind out_kind = dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
  uint64_t m_acc = 0, a_acc = 0;
  // Enqueue every layer on ctx->stream (no host synchronisation unless the
  // counters are requested), so the whole forward can be captured in a graph.
  auto enqueue = [&]() -> int {
  const float* cur = cur0;
  cudaStream_t st = ctx->stream;
  for (int l = 0; l < nlayers; ++l) {
    const sconv_layer& L = layers[l];
    const FwdLayerDims& d = dims[l];
    const bool pooled = L.pool_w != 0;
    const bool fuse = method == SCONV_METHOD_PECR && pooled && L.relu;
    if (pecr_fallback) pecr_fallback[l] = method == SCONV_METHOD_PECR && !fuse;
    float* next = buf[(cur == buf[0]) ? 1 : 0];
    uint64_t* pm = counters ? &m_acc : nullptr;
    uint64_t* pa = counters ? &a_acc : nullptr;
    int rc;
    const size_t conv_elems = size_t(n) * L.k * d.oh * d.ow;
    if (fuse) {
      rc = fused_conv(ctx, cur, n, d.c, d.h, d.w, filt[l], L.k, L.kh, L.kw, L.stride, L.pool_w,
                      L.pool_h, L.pool_stride, L.pool_mode, next, pm, pa, kflags);
    } else {
      const bool want_conv = conv_outputs && conv_outputs[l];
      // ReLU fused into the conv epilogue unless the pre-activation output is wanted
      const int relu_in_epi = L.relu && !want_conv;
      float* dst = pooled ? cbuf : next;
      rc = fused_conv(ctx, cur, n, d.c, d.h, d.w, filt[l], L.k, L.kh, L.kw, L.stride, 0, 0, 1,
                      relu_in_epi, dst, pm, pa, kflags);
      if (rc == SCONV_OK && want_conv)
        CK(cudaMemcpyAsync(conv_outputs[l], dst, conv_elems * 4, out_kind, st));
      if (rc == SCONV_OK && L.relu && !relu_in_epi) {
        relu_kernel<<<grid_for(conv_elems, 256, ctx->num_sms), 256, 0, st>>>(dst, conv_elems);
        TRY(finish_launch(ctx, "relu_kernel"));
      }
      if (rc == SCONV_OK && pooled) {
        const size_t planes = size_t(n) * L.k;
        pool_kernel<<<grid_for(planes * d.ph * d.pw, 256, ctx->num_sms), 256, 0, st>>>(
            cbuf, next, planes, d.oh, d.ow, L.pool_w, L.pool_h, L.pool_stride, L.pool_mode, d.ph,
            d.pw);
        TRY(finish_launch(ctx, "pool_kernel"));
      }
    }
    if (rc != SCONV_OK) {
      if (rc == SCONV_ERR_CUDA || rc == SCONV_ERR_ARG || rc == SCONV_ERR_DISPATCH) return rc;
      // per-layer failures surface as ConfigError (pipeline.cpp:293-297)
      const std::string why = ctx->err;
      return fail(ctx, SCONV_ERR_CONFIG, "layer %d failed: %s", l, why.c_str());
    }
    const size_t out_elems = size_t(n) * L.k * d.ph * d.pw;
    if (layer_outputs && layer_outputs[l])
      CK(cudaMemcpyAsync(layer_outputs[l], next, out_elems * 4, out_kind, st));
    if (l == nlayers - 1) CK(cudaMemcpyAsync(y, next, out_elems * 4, out_kind, st));
    cur = next;
  }
  return SCONV_OK;
  };

  if (!(flags & SCONV_F_GRAPH)) {
    TRY(enqueue());
  } else {
    // CUDA graph mode: the first call runs eagerly (sizing every workspace),
    // then captures the same launch sequence on the context's own stream;
    // later calls with identical arguments replay the graph (one launch for
    // the whole network).  The replay is ordered after prior work on the
    // caller's stream and before anything queued on it afterwards.
    std::string key(reinterpret_cast<const char*>(&n), sizeof n);
    auto add = [&](const void* p, size_t b) { key.append(reinterpret_cast<const char*>(p), b); };
    const void* ptrs[3] = {x, y, reinterpret_cast<const void*>(uintptr_t(method))};
    add(ptrs, sizeof ptrs);
    const int dims3[4] = {c, h, w, nlayers};
    add(dims3, sizeof dims3);
    add(layers, sizeof(sconv_layer) * nlayers);
    for (int l = 0; l < nlayers; ++l) {
      const void* o[2] = {layer_outputs ? layer_outputs[l] : nullptr,
                          conv_outputs ? conv_outputs[l] : nullptr};
      add(o, sizeof o);
    }
    add(&flags, sizeof flags);
    // a graph captured before any workspace it points into was reallocated
    // (a larger call on this context since) is stale: re-capture
    if (ctx->fwd_graph && ctx->fwd_key == key && ctx->fwd_gen == ctx->mem_gen) {
      CK(cudaEventRecord(ctx->ev_graph, st));
      CK(cudaStreamWaitEvent(ctx->own, ctx->ev_graph, 0));
      CK(cudaGraphLaunch(ctx->fwd_graph, ctx->own));
      CK(cudaEventRecord(ctx->ev_graph, ctx->own));
      CK(cudaStreamWaitEvent(st, ctx->ev_graph, 0));
      ctx->launches++;
    } else {
      TRY(enqueue());  // eager run: produces the result, sizes the workspaces
      CK(cudaStreamSynchronize(st));
      if (!ctx->ev_graph) CK(cudaEventCreateWithFlags(&ctx->ev_graph, cudaEventDisableTiming));
      if (ctx->fwd_graph) {
        cudaGraphExecDestroy(ctx->fwd_graph);
        ctx->fwd_graph = nullptr;
        ctx->fwd_key.clear();
      }
      struct StreamSwap {
        sconv_cu_ctx* c;
        cudaStream_t saved;
        ~StreamSwap() { c->stream = saved; }
      } swap{ctx, ctx->stream};
      ctx->stream = ctx->own;
      const uint64_t launches0 = ctx->launches;
      CK(cudaStreamBeginCapture(ctx->own, cudaStreamCaptureModeThreadLocal));
      const int rc = enqueue();
      cudaGraph_t graph = nullptr;
      const cudaError_t ec = cudaStreamEndCapture(ctx->own, &graph);
      ctx->launches = launches0;  // captured, not launched
      if (rc != SCONV_OK) {
        if (graph) cudaGraphDestroy(graph);
        return rc;
      }
      if (ec != cudaSuccess) return fail(ctx, SCONV_ERR_CUDA, "graph capture: %s", cudaGetErrorString(ec));
      cudaGraphExec_t exec = nullptr;
      const cudaError_t ei = cudaGraphInstantiate(&exec, graph, 0);
      cudaGraphDestroy(graph);
      if (ei != cudaSuccess) return fail(ctx, SCONV_ERR_CUDA, "graph instantiate: %s", cudaGetErrorString(ei));
      ctx->fwd_graph = exec;
      ctx->fwd_key = key;
      ctx->fwd_gen = ctx->mem_gen;
    }
  }
  CK(cudaStreamSynchronize(st));
  if (muls) *muls += m_acc;
  if (adds) *adds += a_acc;
  return SCONV_OK;
}

// ---------------------------------------------------------------------------
// Sparsity profiling (window_nnz_counts / sparsity_profile, src/dataset.cpp:249-286)
// ---------------------------------------------------------------------------
int sconv_cu_window_nnz(sconv_cu_ctx* ctx, const float* x, int n, int c, int h, int w, int kh,
                        int kw, int stride, int32_t* counts, double* raw, double* extended,
                        unsigned flags) {
  if (!ctx) return fail(nullptr, SCONV_ERR_ARG, "null context");
  if (n < 0) return fail(ctx, SCONV_ERR_SHAPE, "negative batch");
  if (c < 1) return fail(ctx, SCONV_ERR_SHAPE, "channels must be positive");
  int OW, OH;
  TRY(conv_dims(ctx, w, h, kw, kh, stride, &OW, &OH));
  if (n == 0) return SCONV_OK;
  if (!x) return fail(ctx, SCONV_ERR_ARG, "null tensor pointer");
  const bool dev = flags & SCONV_F_DEVICE;
  DeviceGuard guard(ctx->device);
  cudaStream_t st = ctx->stream;
  const size_t x_elems = size_t(n) * c * h * w, plane = size_t(h) * w;
  const size_t cnt_elems = size_t(n) * OH * OW;
  Arena ar{ctx, {}};
  const size_t i_x = dev ? 0 : ar.add(x_elems * 4);
  const size_t i_pix = ar.add(size_t(n) * plane * 4);
  const size_t i_cnt = (counts && !dev) ? ar.add(cnt_elems * 4) : 0;
  const size_t i_sum = ar.add(size_t(n) * 16);
  std::vector<char*> p;
  TRY(ar.commit(p));
  const float* dx = dev ? x : reinterpret_cast<float*>(p[i_x]);
  if (!dev) CK(cudaMemcpyAsync(const_cast<float*>(dx), x, x_elems * 4, cudaMemcpyHostToDevice, st));
  int32_t* pix = reinterpret_cast<int32_t*>(p[i_pix]);
  int32_t* dcnt = counts ? (dev ? counts : reinterpret_cast<int32_t*>(p[i_cnt])) : nullptr;
  auto* sums = reinterpret_cast<unsigned long long*>(p[i_sum]);  // [n] window, [n] raw
  CK(cudaMemsetAsync(sums, 0, size_t(n) * 16, st));
  pixel_nnz_kernel<<<grid_for(size_t(n) * plane, 256, ctx->num_sms), 256, 0, st>>>(dx, n, c, h, w, pix);
  TRY(finish_launch(ctx, "pixel_nnz_kernel"));
  OpsArgs oa{pix, n, h, w, kh, kw, stride, OH, OW, 0, 0, 0, 0, 0, nullptr};
  window_nnz_kernel<<<grid_for(cnt_elems, 256, ctx->num_sms), 256, 0, st>>>(oa, dcnt, sums);
  TRY(finish_launch(ctx, "window_nnz_kernel"));
  pixel_sum_kernel<<<grid_for(size_t(n) * plane, 256, ctx->num_sms), 256, 0, st>>>(pix, n, plane,
                                                                                 sums + n);
  TRY(finish_launch(ctx, "pixel_sum_kernel"));
  if (counts && !dev)
    CK(cudaMemcpyAsync(counts, dcnt, cnt_elems * 4, cudaMemcpyDeviceToHost, st));
  std::vector<unsigned long long> h_sums(size_t(n) * 2);
  CK(cudaMemcpyAsync(h_sums.data(), sums, size_t(n) * 16, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  // sparsity(): zero fraction of the map; extended: zero fraction of im2col
  const double map_sz = double(c) * h * w, col_sz = double(OH) * OW * c * kh * kw;
  for (int i = 0; i < n; ++i) {
    if (raw) raw[i] = double(uint64_t(map_sz) - h_sums[n + i]) / map_sz;
    if (extended) extended[i] = double(uint64_t(col_sz) - h_sums[i]) / col_sz;
  }
  return SCONV_OK;
}

int sconv_cu_ecr_conv(sconv_cu_ctx* ctx, const float* x, int n, int c, int h, int w,
                      const float* filters, int k, int kh, int kw, int stride, float* y,
                      uint64_t* muls, uint64_t* adds, unsigned flags) {
  return fused_conv(ctx, x, n, c, h, w, filters, k, kh, kw, stride, 0, 0, 1, 0, y, muls, adds,
                    flags);
}

int sconv_cu_pecr_conv_pool(sconv_cu_ctx* ctx, const float* x, int n, int c, int h, int w,
                            const float* filters, int k, int kh, int kw, int stride, int pool_w,
                            int pool_h, int pool_stride, int mode, float* y, uint64_t* muls,
                            uint64_t* adds, unsigned flags) {
  if (pool_w < 1 || pool_h < 1)
    return fail(ctx, SCONV_ERR_CONFIG, "pack count arguments must be positive");
  return fused_conv(ctx, x, n, c, h, w, filters, k, kh, kw, stride, pool_w, pool_h, pool_stride,
                    mode, y, muls, adds, flags);
}

int sconv_cu_ecr_conv_packed(sconv_cu_ctx* ctx, const uint32_t* bits, const int64_t* base,
                             const float* values, int n, int c, int h, int w, const float* filters,
                             int k, int kh, int kw, int stride, float* y, uint64_t* muls,
                             uint64_t* adds, unsigned flags) {
  const PackedIn pk{bits, base, values};
  return fused_conv(ctx, nullptr, n, c, h, w, filters, k, kh, kw, stride, 0, 0, 1, 0, y, muls, adds,
                    flags, &pk);
}

int sconv_cu_pecr_conv_pool_packed(sconv_cu_ctx* ctx, const uint32_t* bits, const int64_t* base,
                                   const float* values, int n, int c, int h, int w,
                                   const float* filters, int k, int kh, int kw, int stride,
                                   int pool_w, int pool_h, int pool_stride, int mode, float* y,
                                   uint64_t* muls, uint64_t* adds, unsigned flags) {
  if (pool_w < 1 || pool_h < 1)
    return fail(ctx, SCONV_ERR_CONFIG, "pack count arguments must be positive");
  const PackedIn pk{bits, base, values};
  return fused_conv(ctx, nullptr, n, c, h, w, filters, k, kh, kw, stride, pool_w, pool_h,
                    pool_stride, mode, y, muls, adds, flags, &pk);
}

int sconv_cu_unpack_maps(sconv_cu_ctx* ctx, const uint32_t* bits, const int64_t* base,
                         const float* values, int n, int c, int h, int w, float* x,
                         unsigned flags) {
  if (!ctx) return fail(nullptr, SCONV_ERR_ARG, "null context");
  if (n < 0 || c < 1 || h < 1 || w < 1) return fail(ctx, SCONV_ERR_SHAPE, "bad map dims");
  if (n == 0) return SCONV_OK;
  if (!(flags & SCONV_F_DEVICE)) return fail(ctx, SCONV_ERR_ARG, "sconv_cu_unpack_maps takes device pointers");
  if (!bits || !base || !x) return fail(ctx, SCONV_ERR_ARG, "null pointer");
  DeviceGuard guard(ctx->device);
  TRY(expand_chunk(ctx, ctx->stream, bits, base, values, 0, n, int64_t(c) * h * w, x));
  if (!(flags & SCONV_F_ASYNC)) CK(cudaStreamSynchronize(ctx->stream));
  return SCONV_OK;
}

int sconv_cu_ecr_convert(sconv_cu_ctx* ctx, const float* x, int c, int h, int w,
                         const float* filter, int kh, int kw, int stride, int32_t* ptr,
                         int32_t* offsets, float* f_data, float* k_data, unsigned flags) {
  if (!ctx) return fail(nullptr, SCONV_ERR_ARG, "null context");
  if (c < 1) return fail(ctx, SCONV_ERR_SHAPE, "channels must be positive");
  int OW, OH;
  TRY(conv_dims(ctx, w, h, kw, kh, stride, &OW, &OH));
  if (!x || !filter || !ptr || !offsets || !f_data || !k_data)
    return fail(ctx, SCONV_ERR_ARG, "null pointer");
  const bool dev = flags & SCONV_F_DEVICE;
  const size_t nwin = size_t(OH) * OW, slot = size_t(c) * kh * kw;
  DeviceGuard guard(ctx->device);
  Arena ar{ctx, {}};
  const size_t ix = dev ? 0 : ar.add(size_t(c) * h * w * 4), iw = dev ? 0 : ar.add(slot * 4);
  const size_t ip = dev ? 0 : ar.add(nwin * 4), io = dev ? 0 : ar.add(nwin * slot * 4);
  const size_t iff = dev ? 0 : ar.add(nwin * slot * 4), ik = dev ? 0 : ar.add(nwin * slot * 4);
  std::vector<char*> p;
  TRY(ar.commit(p));
  cudaStream_t st = ctx->stream;
  EcrExportArgs a{x, filter, c, h, w, kh, kw, stride, OH, OW, ptr, offsets, f_data, k_data};
  if (!dev) {
    a.x = reinterpret_cast<float*>(p[ix]);
    a.filter = reinterpret_cast<float*>(p[iw]);
    a.ptr = reinterpret_cast<int32_t*>(p[ip]);
    a.offsets = reinterpret_cast<int32_t*>(p[io]);
    a.f_data = reinterpret_cast<float*>(p[iff]);
    a.k_data = reinterpret_cast<float*>(p[ik]);
    CK(cudaMemcpyAsync(const_cast<float*>(a.x), x, size_t(c) * h * w * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(const_cast<float*>(a.filter), filter, slot * 4, cudaMemcpyHostToDevice, st));
  }
  ecr_export_kernel<<<grid_for(nwin * 32, 256, 1 << 20), 256, 0, st>>>(a);
  TRY(finish_launch(ctx, "ecr_export_kernel"));
  if (!dev) {
    CK(cudaMemcpyAsync(ptr, a.ptr, nwin * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(offsets, a.offsets, nwin * slot * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(f_data, a.f_data, nwin * slot * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(k_data, a.k_data, nwin * slot * 4, cudaMemcpyDeviceToHost, st));
  }
  if (!(flags & SCONV_F_ASYNC)) CK(cudaStreamSynchronize(st));
  return SCONV_OK;
}

int sconv_cu_ecr_spmv(sconv_cu_ctx* ctx, const int32_t* ptr, const float* f_data,
                      const float* k_data, int oh, int ow, int slot, float* y, uint64_t* muls,
                      uint64_t* adds, unsigned flags) {
  if (!ctx) return fail(nullptr, SCONV_ERR_ARG, "null context");
  if (oh < 1 || ow < 1 || slot < 1) return fail(ctx, SCONV_ERR_FORMAT, "empty ECR geometry");
  if (!ptr || !f_data || !k_data || !y) return fail(ctx, SCONV_ERR_ARG, "null pointer");
  const bool dev = flags & SCONV_F_DEVICE, fast = flags & SCONV_F_FAST;
  const size_t nwin = size_t(oh) * ow;
  if (!dev) {  // check_ecr ptr range on the host copy (src/ecr.cpp:32-38)
    for (size_t i = 0; i < nwin; ++i)
      if (ptr[i] < -1 || ptr[i] > slot)
        return fail(ctx, SCONV_ERR_FORMAT, "corrupted ptr value %d outside [-1, %d]", ptr[i], slot);
  }
  DeviceGuard guard(ctx->device);
  Arena ar{ctx, {}};
  const size_t ip = dev ? 0 : ar.add(nwin * 4), iff = dev ? 0 : ar.add(nwin * slot * 4);
  const size_t ik = dev ? 0 : ar.add(nwin * slot * 4), iy = dev ? 0 : ar.add(nwin * 4);
  const size_t iops = ar.add(64);
  std::vector<char*> p;
  TRY(ar.commit(p));
  cudaStream_t st = ctx->stream;
  auto* ops = reinterpret_cast<unsigned long long*>(p[iops]);
  EcrSpmvArgs a{ptr, f_data, k_data, static_cast<int>(nwin), slot, y, ops,
                reinterpret_cast<int*>(ops + 2)};
  if (!dev) {
    a.ptr = reinterpret_cast<int32_t*>(p[ip]);
    a.f_data = reinterpret_cast<float*>(p[iff]);
    a.k_data = reinterpret_cast<float*>(p[ik]);
    a.y = reinterpret_cast<float*>(p[iy]);
    CK(cudaMemcpyAsync(const_cast<int32_t*>(a.ptr), ptr, nwin * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(const_cast<float*>(a.f_data), f_data, nwin * slot * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(const_cast<float*>(a.k_data), k_data, nwin * slot * 4, cudaMemcpyHostToDevice, st));
  }
  CK(cudaMemsetAsync(ops, 0, 24, st));
  if (fast) {
    ecr_spmv_fast_kernel<<<grid_for(nwin * 32, 256, 1 << 20), 256, 0, st>>>(a);
  } else {
    ecr_spmv_exact_kernel<<<grid_for(nwin, 256, 1 << 20), 256, 0, st>>>(a);
  }
  TRY(finish_launch(ctx, "ecr_spmv_kernel"));
  unsigned long long h[3];
  CK(cudaMemcpyAsync(h, ops, 24, cudaMemcpyDeviceToHost, st));
  if (!dev) CK(cudaMemcpyAsync(y, a.y, nwin * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (static_cast<int>(h[2])) return fail(ctx, SCONV_ERR_FORMAT, "corrupted ptr value outside [-1, %d]", slot);
  if (muls) *muls += h[0];
  if (adds) *adds += h[1];
  return SCONV_OK;
}

int sconv_cu_pecr_count(sconv_cu_ctx* ctx, const float* x, int c, int h, int w, int kh, int kw,
                        int stride, int pool_w, int pool_h, int pool_stride, int32_t* count,
                        int64_t* pack_start, int64_t* total, unsigned flags) {
  if (!ctx) return fail(nullptr, SCONV_ERR_ARG, "null context");
  if (c < 1) return fail(ctx, SCONV_ERR_SHAPE, "channels must be positive");
  int OW, OH, PWo, PHo;
  TRY(conv_dims(ctx, w, h, kw, kh, stride, &OW, &OH));
  TRY(pack_count(ctx, w, kw, stride, pool_w, pool_stride, &PWo));
  TRY(pack_count(ctx, h, kh, stride, pool_h, pool_stride, &PHo));
  if (!x || !count || !pack_start || !total) return fail(ctx, SCONV_ERR_ARG, "null pointer");
  const bool dev = flags & SCONV_F_DEVICE;
  const int wpp = pool_w * pool_h, npacks = PHo * PWo;
  DeviceGuard guard(ctx->device);
  const int64_t nparts = (int64_t(npacks) + kScanChunk - 1) / kScanChunk;
  Arena ar{ctx, {}};
  const size_t ix = dev ? 0 : ar.add(size_t(c) * h * w * 4);
  const size_t ic = dev ? 0 : ar.add(size_t(npacks) * wpp * 4);
  const size_t is = dev ? 0 : ar.add(size_t(npacks + 1) * 8);
  const size_t ipart = ar.add(size_t(std::max<int64_t>(nparts, 1)) * 8);
  std::vector<char*> p;
  TRY(ar.commit(p));
  cudaStream_t st = ctx->stream;
  PecrFmtArgs a{x, c, h, w, kh, kw, stride, pool_w, pool_h, pool_stride, PHo, PWo, count,
                nullptr, nullptr, nullptr};
  int64_t* dstart = pack_start;
  if (!dev) {
    a.x = reinterpret_cast<float*>(p[ix]);
    a.count = reinterpret_cast<int32_t*>(p[ic]);
    dstart = reinterpret_cast<int64_t*>(p[is]);
    CK(cudaMemcpyAsync(const_cast<float*>(a.x), x, size_t(c) * h * w * 4, cudaMemcpyHostToDevice, st));
  }
  pecr_export_kernel<0><<<grid_for(size_t(npacks) * wpp * 32, 256, 1 << 20), 256, 0, st>>>(a);
  TRY(finish_launch(ctx, "pecr_export_kernel<count>"));
  // pack_start = exclusive prefix of the pack totals (kernels/scan.cuh)
  int64_t* part = reinterpret_cast<int64_t*>(p[ipart]);
  if (npacks == 0) {
    CK(cudaMemsetAsync(dstart, 0, 8, st));
  } else {
    pack_scan_partial<<<static_cast<unsigned>(nparts), kScanThreads, 0, st>>>(a.count, wpp, npacks, part);
    TRY(finish_launch(ctx, "pack_scan_partial"));
    pack_scan_partials<<<1, 1024, 0, st>>>(part, nparts);
    TRY(finish_launch(ctx, "pack_scan_partials"));
    pack_scan_final<<<static_cast<unsigned>(nparts), kScanThreads, 0, st>>>(a.count, wpp, npacks, part, dstart);
    TRY(finish_launch(ctx, "pack_scan_final"));
  }
  int64_t htotal = 0;
  CK(cudaMemcpyAsync(&htotal, dstart + npacks, 8, cudaMemcpyDeviceToHost, st));
  if (!dev) {
    CK(cudaMemcpyAsync(count, a.count, size_t(npacks) * wpp * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(pack_start, dstart, size_t(npacks + 1) * 8, cudaMemcpyDeviceToHost, st));
  }
  CK(cudaStreamSynchronize(st));
  *total = htotal;
  return SCONV_OK;
}

int sconv_cu_pecr_fill(sconv_cu_ctx* ctx, const float* x, int c, int h, int w, int kh, int kw,
                       int stride, int pool_w, int pool_h, int pool_stride,
                       const int64_t* pack_start, int64_t total, float* data, int32_t* index,
                       unsigned flags) {
  if (!ctx) return fail(nullptr, SCONV_ERR_ARG, "null context");
  if (c < 1) return fail(ctx, SCONV_ERR_SHAPE, "channels must be positive");
  int OW, OH, PWo, PHo;
  TRY(conv_dims(ctx, w, h, kw, kh, stride, &OW, &OH));
  TRY(pack_count(ctx, w, kw, stride, pool_w, pool_stride, &PWo));
  TRY(pack_count(ctx, h, kh, stride, pool_h, pool_stride, &PHo));
  if (!x || !pack_start || (total > 0 && (!data || !index)))
    return fail(ctx, SCONV_ERR_ARG, "null pointer");
  const bool dev = flags & SCONV_F_DEVICE;
  const int wpp = pool_w * pool_h, npacks = PHo * PWo;
  DeviceGuard guard(ctx->device);
  // counts are recomputed on device (cheap) so the fill needs no host state
  // beyond pack_start.
  Arena ar{ctx, {}};
  const size_t ix = dev ? 0 : ar.add(size_t(c) * h * w * 4);
  const size_t is = dev ? 0 : ar.add(size_t(npacks + 1) * 8);
  const size_t id = dev ? 0 : ar.add(size_t(std::max<int64_t>(total, 1)) * 4);
  const size_t ii = dev ? 0 : ar.add(size_t(std::max<int64_t>(total, 1)) * 4);
  const size_t ic = ar.add(size_t(npacks) * wpp * 4);
  std::vector<char*> p;
  TRY(ar.commit(p));
  cudaStream_t st = ctx->stream;
  PecrFmtArgs a{x, c, h, w, kh, kw, stride, pool_w, pool_h, pool_stride, PHo, PWo,
                reinterpret_cast<int32_t*>(p[ic]), pack_start, data, index};
  if (!dev) {
    a.x = reinterpret_cast<float*>(p[ix]);
    a.pack_start = reinterpret_cast<int64_t*>(p[is]);
    a.data = reinterpret_cast<float*>(p[id]);
    a.index = reinterpret_cast<int32_t*>(p[ii]);
    CK(cudaMemcpyAsync(const_cast<float*>(a.x), x, size_t(c) * h * w * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(const_cast<int64_t*>(a.pack_start), pack_start, size_t(npacks + 1) * 8,
                       cudaMemcpyHostToDevice, st));
  }
  const unsigned g = grid_for(size_t(npacks) * wpp * 32, 256, 1 << 20);
  pecr_export_kernel<0><<<g, 256, 0, st>>>(a);
  TRY(finish_launch(ctx, "pecr_export_kernel<count>"));
  pecr_export_kernel<1><<<g, 256, 0, st>>>(a);
  TRY(finish_launch(ctx, "pecr_export_kernel<fill>"));
  if (!dev && total > 0) {
    CK(cudaMemcpyAsync(data, a.data, size_t(total) * 4, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(index, a.index, size_t(total) * 4, cudaMemcpyDeviceToHost, st));
  }
  if (!(flags & SCONV_F_ASYNC)) CK(cudaStreamSynchronize(st));
  return SCONV_OK;
}

int sconv_cu_pecr_pool(sconv_cu_ctx* ctx, const int32_t* count, const int64_t* pack_start,
                       const float* data, const int32_t* index, int64_t total,
                       const float* kernel, int c, int kh, int kw, int packs_h, int packs_w,
                       int pool_w, int pool_h, int mode, float* y, uint64_t* muls, uint64_t* adds,
                       unsigned flags) {
  if (!ctx) return fail(nullptr, SCONV_ERR_ARG, "null context");
  if (c < 1 || kh < 1 || kw < 1 || packs_h < 1 || packs_w < 1 || pool_w < 1 || pool_h < 1)
    return fail(ctx, SCONV_ERR_FORMAT, "bad PECR geometry");
  if (mode != SCONV_POOL_MAX && mode != SCONV_POOL_MEAN)
    return fail(ctx, SCONV_ERR_CONFIG, "unknown pool mode %d", mode);
  if (!count || !pack_start || !kernel || !y || (total > 0 && (!data || !index)))
    return fail(ctx, SCONV_ERR_ARG, "null pointer");
  const bool dev = flags & SCONV_F_DEVICE, fast = flags & SCONV_F_FAST;
  const int wpp = pool_w * pool_h, npacks = packs_h * packs_w, cap = c * kh * kw;
  if (!dev) {  // check_pecr (src/pecr.cpp:40-55) on the host copy
    for (int pk = 0; pk < npacks; ++pk) {
      int64_t s = 0;
      for (int q = 0; q < wpp; ++q) {
        const int cn = count[size_t(pk) * wpp + q];
        if (cn < 0 || cn > cap)
          return fail(ctx, SCONV_ERR_FORMAT, "count entry %d outside [0, %d]", cn, cap);
        s += cn;
      }
      if (pack_start[pk] < 0 || pack_start[pk + 1] - pack_start[pk] != s || pack_start[pk + 1] > total)
        return fail(ctx, SCONV_ERR_FORMAT, "data/index length inconsistent with counts");
    }
    if (pack_start[npacks] != total)
      return fail(ctx, SCONV_ERR_FORMAT, "data/index length inconsistent with counts");
    for (int64_t q = 0; q < total; ++q)
      if (index[q] < 0 || index[q] >= cap)
        return fail(ctx, SCONV_ERR_FORMAT, "index entry %d out of range", index[q]);
  }
  DeviceGuard guard(ctx->device);
  Arena ar{ctx, {}};
  const size_t tb = size_t(std::max<int64_t>(total, 1)) * 4;
  const size_t ic = dev ? 0 : ar.add(size_t(npacks) * wpp * 4), is = dev ? 0 : ar.add(size_t(npacks + 1) * 8);
  const size_t id = dev ? 0 : ar.add(tb), ii = dev ? 0 : ar.add(tb);
  const size_t ik = dev ? 0 : ar.add(size_t(cap) * 4), iy = dev ? 0 : ar.add(size_t(npacks) * 4);
  const size_t iops = ar.add(64);
  std::vector<char*> p;
  TRY(ar.commit(p));
  cudaStream_t st = ctx->stream;
  auto* ops = reinterpret_cast<unsigned long long*>(p[iops]);
  PecrPoolArgs a{count, pack_start, data, index, kernel, npacks, wpp, cap, mode, y, ops,
                 reinterpret_cast<int*>(ops + 2)};
  if (!dev) {
    a.count = reinterpret_cast<int32_t*>(p[ic]);
    a.pack_start = reinterpret_cast<int64_t*>(p[is]);
    a.data = reinterpret_cast<float*>(p[id]);
    a.index = reinterpret_cast<int32_t*>(p[ii]);
    a.kernel = reinterpret_cast<float*>(p[ik]);
    a.y = reinterpret_cast<float*>(p[iy]);
    CK(cudaMemcpyAsync(const_cast<int32_t*>(a.count), count, size_t(npacks) * wpp * 4, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(const_cast<int64_t*>(a.pack_start), pack_start, size_t(npacks + 1) * 8, cudaMemcpyHostToDevice, st));
    if (total > 0) {
      CK(cudaMemcpyAsync(const_cast<float*>(a.data), data, size_t(total) * 4, cudaMemcpyHostToDevice, st));
      CK(cudaMemcpyAsync(const_cast<int32_t*>(a.index), index, size_t(total) * 4, cudaMemcpyHostToDevice, st));
    }
    CK(cudaMemcpyAsync(const_cast<float*>(a.kernel), kernel, size_t(cap) * 4, cudaMemcpyHostToDevice, st));
  }
  CK(cudaMemsetAsync(ops, 0, 24, st));
  if (dev) {
    pecr_check_kernel<<<(npacks + 255) / 256, 256, 0, st>>>(a, total);
    TRY(finish_launch(ctx, "pecr_check_kernel"));
  }
  if (fast) {
    pecr_pool_fast_kernel<<<grid_for(size_t(npacks) * 32, 256, 1 << 20), 256, 0, st>>>(a);
  } else {
    pecr_pool_exact_kernel<<<grid_for(npacks, 256, 1 << 20), 256, 0, st>>>(a);
  }
  TRY(finish_launch(ctx, "pecr_pool_kernel"));
  unsigned long long hh[3];
  CK(cudaMemcpyAsync(hh, ops, 24, cudaMemcpyDeviceToHost, st));
  if (!dev) CK(cudaMemcpyAsync(y, a.y, size_t(npacks) * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (static_cast<int>(hh[2])) return fail(ctx, SCONV_ERR_FORMAT, "corrupted PECR format");
  if (muls) *muls += hh[0];
  if (adds) *adds += hh[1];
  return SCONV_OK;
}

int sconv_cu_ecr_conv_multi(sconv_cu_ctx** ctxs, int nctx, const float* x, int n, int c, int h,
                            int w, const float* filters, int k, int kh, int kw, int stride,
                            float* y, uint64_t* muls, uint64_t* adds, unsigned flags) {
  if (flags & (SCONV_F_DEVICE | SCONV_F_ASYNC))
    return fail(nullptr, SCONV_ERR_ARG, "multi-device entry takes host pointers");
  int OW, OH;
  TRY(conv_dims(nullptr, w, h, kw, kh, stride, &OW, &OH));
  return run_multi(ctxs, nctx, n, k, size_t(c) * h * w, size_t(c) * kh * kw, size_t(OH) * OW, x,
                   filters, y, muls, adds,
                   [&](sconv_cu_ctx* cx, const float* xs, int ns, const float* ws, int ks,
                       float* ys, uint64_t* m, uint64_t* a) {
                     return sconv_cu_ecr_conv(cx, xs, ns, c, h, w, ws, ks, kh, kw, stride, ys, m,
                                              a, flags);
                   });
}

int sconv_cu_pecr_conv_pool_multi(sconv_cu_ctx** ctxs, int nctx, const float* x, int n, int c,
                                  int h, int w, const float* filters, int k, int kh, int kw,
                                  int stride, int pool_w, int pool_h, int pool_stride, int mode,
                                  float* y, uint64_t* muls, uint64_t* adds, unsigned flags) {
  if (flags & (SCONV_F_DEVICE | SCONV_F_ASYNC))
    return fail(nullptr, SCONV_ERR_ARG, "multi-device entry takes host pointers");
  int PWo, PHo;
  TRY(pack_count(nullptr, w, kw, stride, pool_w, pool_stride, &PWo));
  TRY(pack_count(nullptr, h, kh, stride, pool_h, pool_stride, &PHo));
  return run_multi(ctxs, nctx, n, k, size_t(c) * h * w, size_t(c) * kh * kw, size_t(PHo) * PWo,
                   x, filters, y, muls, adds,
                   [&](sconv_cu_ctx* cx, const float* xs, int ns, const float* ws, int ks,
                       float* ys, uint64_t* m, uint64_t* a) {
                     return sconv_cu_pecr_conv_pool(cx, xs, ns, c, h, w, ws, ks, kh, kw, stride,
                                                    pool_w, pool_h, pool_stride, mode, ys, m, a,
                                                    flags);
                   });
}

}  // extern "C"
