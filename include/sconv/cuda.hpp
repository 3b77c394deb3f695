// sconv/cuda.hpp -- batched C++ entry points over the C ABI (sconv_cuda.h)
// for reference callers: header-only, on top of the reference's UNCHANGED
// types (proj/include/sconv/{tensor,pipeline,metrics,errors,exec}.hpp).
//
// The drop-in (csrc/dropin/sconv_dropin.cpp) keeps the reference's per-filter
// two-phase API (ecr_convert -> ecr_spmv_conv, pecr_convert -> pecr_conv_pool),
// so after the CMake swap a reference caller of multichannel_conv or forward
// still moves an im2col-sized format across PCIe per (image, filter).  These
// entries are the batched alternative a C++ host calls directly:
//
//   sconv::cuda::multichannel_conv   all K filters of a layer in one fused
//                                    launch (src/pipeline.cpp:191-210), one
//                                    image or a batch
//   sconv::cuda::conv_pool           forward's fused conv + ReLU + pool branch
//                                    for a whole layer (pipeline.cpp:249-264)
//   sconv::cuda::forward             forward(net, input, method)
//                                    (pipeline.cpp:212-301) with the
//                                    activations resident in HBM
//
// Results are the reference's: EXACT (default) is bit-identical, FAST
// (Options::fast or $SCONV_CUDA_MODE=fast) within 1e-5 + 1e-5|ref|.  Status
// codes become the reference's exceptions.  Each host thread gets its own
// context (device Options::device, else $SCONV_CUDA_DEVICE, else 0), so the
// reference's "safe to call concurrently" contract holds.  Link
// libsconv_cuda.so; tests/dropin/cuda_hpp_test.cpp exercises every entry.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "sconv/errors.hpp"
#include "sconv/exec.hpp"
#include "sconv/metrics.hpp"
#include "sconv/pipeline.hpp"
#include "sconv/tensor.hpp"
#include "sconv_cuda.h"

namespace sconv::cuda {

struct Options {
  int device = -1;     // -1: $SCONV_CUDA_DEVICE, else 0
  int fast = -1;       // -1: $SCONV_CUDA_MODE == "fast"; 0 EXACT; 1 FAST
  bool keep_intermediates = true;  // forward: fill conv_outputs / layer_outputs like the reference
};

namespace detail {

[[noreturn]] inline void raise_status(int rc, const sconv_cu_ctx* c) {
  const std::string msg = sconv_cu_last_error(c);
  switch (rc) {
    case SCONV_ERR_SHAPE: throw ShapeError(msg);
    case SCONV_ERR_CONFIG: throw ConfigError(msg);
    case SCONV_ERR_FORMAT: throw FormatError(msg);
    case SCONV_ERR_IO: throw IoError(msg);
    case SCONV_ERR_DISPATCH: throw DispatchError(-1, -1, msg);
    case SCONV_ERR_ARG: throw std::invalid_argument(msg);
    default: throw std::runtime_error("sconv_cuda: " + msg);
  }
}

inline void check(int rc, const sconv_cu_ctx* c = nullptr) {
  if (rc != SCONV_OK) raise_status(rc, c);
}

inline int device_of(const Options& o) {
  if (o.device >= 0) return o.device;
  const char* e = std::getenv("SCONV_CUDA_DEVICE");
  return e ? std::atoi(e) : 0;
}

inline unsigned flags_of(const Options& o) {
  bool fast = o.fast == 1;
  if (o.fast < 0) {
    const char* e = std::getenv("SCONV_CUDA_MODE");
    fast = e && std::strcmp(e, "fast") == 0;
  }
  return fast ? SCONV_F_FAST : SCONV_F_EXACT;
}

// One context per (host thread, device), destroyed with the thread.
inline sconv_cu_ctx* context(int device) {
  struct Deleter {
    void operator()(sconv_cu_ctx* c) const { sconv_cu_ctx_destroy(c); }
  };
  thread_local std::map<int, std::unique_ptr<sconv_cu_ctx, Deleter>> ctxs;
  auto& slot = ctxs[device];
  if (!slot) {
    sconv_cu_ctx* c = nullptr;
    check(sconv_cu_ctx_create(device, &c));
    slot.reset(c);
  }
  return slot.get();
}

// Filters [K][C][kh][kw] from the reference's per-output-channel Filters.
inline std::vector<float> stack_filters(const std::vector<Filter>& filters, int channels) {
  if (filters.empty()) throw ConfigError("multichannel_conv requires filters");
  std::vector<float> w;
  w.reserve(filters.size() * filters[0].size());
  for (const Filter& f : filters) {
    if (f.channels != channels)  // ecr.cpp:53-56
      throw ShapeError("filter channels " + std::to_string(f.channels) + " != map channels " +
                       std::to_string(channels));
    if (f.height != filters[0].height || f.width != filters[0].width)
      throw ShapeError("filters must share dims");
    w.insert(w.end(), f.weights.begin(), f.weights.end());
  }
  return w;
}

// The images of a batch, one contiguous [N][C][H][W] buffer.
inline std::vector<float> stack_maps(const std::vector<FeatureMap>& maps) {
  if (maps.empty()) return {};
  const FeatureMap& m0 = maps[0];
  std::vector<float> x;
  x.reserve(maps.size() * m0.size());
  for (const FeatureMap& m : maps) {
    if (m.channels != m0.channels || m.height != m0.height || m.width != m0.width)
      throw ShapeError("batched maps must share dims");
    x.insert(x.end(), m.values.begin(), m.values.end());
  }
  return x;
}

inline std::vector<FeatureMap> split(std::vector<float>& y, int n, int k, int h, int w) {
  std::vector<FeatureMap> out;
  out.reserve(n);
  const size_t per = size_t(k) * h * w;
  for (int i = 0; i < n; ++i)
    out.emplace_back(k, h, w, std::vector<float>(y.begin() + i * per, y.begin() + (i + 1) * per));
  return out;
}

inline std::uint64_t map_bytes(int c, int h, int w) { return std::uint64_t(c) * h * w * 4; }

}  // namespace detail

/// multichannel_conv (src/pipeline.cpp:191-210) for a batch of maps: every
/// filter of every image in one fused ECR launch.  Method::kEcr only (the
/// dense method is the CPU reference's own).
inline std::vector<FeatureMap> multichannel_conv(const std::vector<FeatureMap>& maps,
                                                 const std::vector<Filter>& filters,
                                                 const ConvConfig& cfg, Method method = Method::kEcr,
                                                 const ExecConfig& exec = {},
                                                 OpCount* counters = nullptr, Options opt = {}) {
  if (method != Method::kEcr) throw ConfigError("sconv::cuda::multichannel_conv runs the ECR method");
  if (exec.workers < 1) throw ConfigError("workers must be >= 1");  // exec.hpp:62
  if (maps.empty()) return {};
  const FeatureMap& m0 = maps[0];
  std::vector<float> w = detail::stack_filters(filters, m0.channels);
  std::vector<float> x = detail::stack_maps(maps);
  int ow = 0, oh = 0;
  detail::check(sconv_conv_output_dims(m0.width, m0.height, filters[0].width, filters[0].height,
                                       cfg.stride, &ow, &oh));
  const int n = int(maps.size()), k = int(filters.size());
  std::vector<float> y(size_t(n) * k * oh * ow);
  sconv_cu_ctx* c = detail::context(detail::device_of(opt));
  std::uint64_t muls = 0, adds = 0;
  detail::check(sconv_cu_ecr_conv(c, x.data(), n, m0.channels, m0.height, m0.width, w.data(), k,
                                  filters[0].height, filters[0].width, cfg.stride, y.data(),
                                  counters ? &muls : nullptr, counters ? &adds : nullptr,
                                  detail::flags_of(opt)),
                c);
  if (counters) counters->merge(OpCount{muls, adds});
  return detail::split(y, n, k, oh, ow);
}

/// multichannel_conv for one map: the reference's signature plus Options.
inline FeatureMap multichannel_conv(const FeatureMap& map, const std::vector<Filter>& filters,
                                    const ConvConfig& cfg, Method method = Method::kEcr,
                                    const ExecConfig& exec = {}, OpCount* counters = nullptr,
                                    Options opt = {}) {
  return multichannel_conv(std::vector<FeatureMap>{map}, filters, cfg, method, exec, counters,
                           opt)[0];
}

/// forward's fused branch for a whole layer (src/pipeline.cpp:249-264):
/// conv + ReLU + pool of every filter -> K x packs_h x packs_w, per image.
inline std::vector<FeatureMap> conv_pool(const std::vector<FeatureMap>& maps,
                                         const std::vector<Filter>& filters, const ConvConfig& cfg,
                                         const PoolConfig& pool, OpCount* counters = nullptr,
                                         Options opt = {}) {
  if (maps.empty()) return {};
  const FeatureMap& m0 = maps[0];
  std::vector<float> w = detail::stack_filters(filters, m0.channels);
  std::vector<float> x = detail::stack_maps(maps);
  int pw = 0, ph = 0;
  detail::check(sconv_pecr_pack_count(m0.width, filters[0].width, cfg.stride, pool.width,
                                      pool.stride, &pw));
  detail::check(sconv_pecr_pack_count(m0.height, filters[0].height, cfg.stride, pool.height,
                                      pool.stride, &ph));
  const int n = int(maps.size()), k = int(filters.size());
  std::vector<float> y(size_t(n) * k * ph * pw);
  sconv_cu_ctx* c = detail::context(detail::device_of(opt));
  std::uint64_t muls = 0, adds = 0;
  detail::check(sconv_cu_pecr_conv_pool(
                    c, x.data(), n, m0.channels, m0.height, m0.width, w.data(), k,
                    filters[0].height, filters[0].width, cfg.stride, pool.width, pool.height,
                    pool.stride, pool.mode == PoolMode::kMean ? SCONV_POOL_MEAN : SCONV_POOL_MAX,
                    y.data(), counters ? &muls : nullptr, counters ? &adds : nullptr,
                    detail::flags_of(opt)),
                c);
  if (counters) counters->merge(OpCount{muls, adds});
  return detail::split(y, n, k, ph, pw);
}

inline FeatureMap conv_pool(const FeatureMap& map, const std::vector<Filter>& filters,
                            const ConvConfig& cfg, const PoolConfig& pool,
                            OpCount* counters = nullptr, Options opt = {}) {
  return conv_pool(std::vector<FeatureMap>{map}, filters, cfg, pool, counters, opt)[0];
}

/// forward(net, input, method) (src/pipeline.cpp:212-301) on the GPU: one
/// ingest of the input and every layer's filters, activations resident in
/// HBM, the fused PECR kernel on conv+pool layers with ReLU, ECR + epilogue
/// ReLU + pool otherwise (reported in pecr_fallback_layers).  `traffic` is the
/// reference's modeled report for the same network; conv_outputs holds the
/// reference's 1x1x1 placeholder on fused layers.
inline ForwardResult forward(const NetworkSpec& net, const FeatureMap& input, Method method,
                             const ExecConfig& exec = {}, Options opt = {}) {
  net.validate();
  if (input.channels != net.in_channels || input.height != net.in_height ||
      input.width != net.in_width)
    throw ShapeError("input dims do not match network spec");
  if (exec.workers < 1) throw ConfigError("workers must be >= 1");
  const int m = method == Method::kEcr ? SCONV_METHOD_ECR
                                       : method == Method::kPecr ? SCONV_METHOD_PECR : -1;
  if (m < 0) throw ConfigError("sconv::cuda::forward runs the compressed methods (ECR, PECR)");
  const int nl = int(net.layers.size());
  std::vector<std::vector<float>> w(nl);
  std::vector<sconv_layer> L(nl);
  for (int l = 0; l < nl; ++l) {
    const LayerSpec& s = net.layers[l];
    const int cin = l == 0 ? input.channels : net.layers[l - 1].filters.size();
    w[l] = detail::stack_filters(s.filters, cin);
    L[l] = {w[l].data(), int(s.filters.size()), s.filters[0].height, s.filters[0].width,
            s.conv.stride, s.activation == Activation::kRelu ? 1 : 0, s.pool ? s.pool->width : 0,
            s.pool ? s.pool->height : 0, s.pool ? s.pool->stride : 1,
            s.pool && s.pool->mode == PoolMode::kMean ? SCONV_POOL_MEAN : SCONV_POOL_MAX};
  }
  // per-layer dims: conv output and layer output
  std::vector<int> cc(nl), ch(nl), cw(nl), lh(nl), lw(nl);
  {
    int c = input.channels, h = input.height, wd = input.width;
    for (int l = 0; l < nl; ++l) {
      int oc = 0, oh = 0, ow = 0;
      detail::check(sconv_cu_forward_dims(&L[l], 1, c, h, wd, &oc, &oh, &ow));
      detail::check(sconv_conv_output_dims(wd, h, L[l].kw, L[l].kh, L[l].stride, &cw[l], &ch[l]));
      cc[l] = oc;
      lh[l] = oh;
      lw[l] = ow;
      c = oc, h = oh, wd = ow;
    }
  }
  ForwardResult r;
  std::vector<std::vector<float>> lo(nl), co(nl);
  std::vector<float*> lop(nl, nullptr), cop(nl, nullptr);
  std::vector<int32_t> fb(nl, 0);
  const bool fused_any = m == SCONV_METHOD_PECR;
  for (int l = 0; l < nl && opt.keep_intermediates; ++l) {
    lo[l].resize(size_t(cc[l]) * lh[l] * lw[l]);
    lop[l] = lo[l].data();
    const bool fuse = fused_any && net.layers[l].pool && L[l].relu;
    if (!fuse) {
      co[l].resize(size_t(cc[l]) * ch[l] * cw[l]);
      cop[l] = co[l].data();
    }
  }
  std::vector<float> y(static_cast<size_t>(cc[nl - 1]) * lh[nl - 1] * lw[nl - 1]);
  sconv_cu_ctx* c = detail::context(detail::device_of(opt));
  std::uint64_t muls = 0, adds = 0;
  detail::check(sconv_cu_forward(c, input.values.data(), 1, input.channels, input.height,
                                 input.width, L.data(), nl, m, y.data(),
                                 opt.keep_intermediates ? lop.data() : nullptr,
                                 opt.keep_intermediates ? cop.data() : nullptr, &muls, &adds,
                                 fb.data(), detail::flags_of(opt)),
                c);
  r.ops = OpCount{muls, adds};
  // the reference's traffic model (pipeline.cpp:222-300)
  r.traffic.host_to_device_bytes = detail::map_bytes(input.channels, input.height, input.width);
  int pc = input.channels, phh = input.height, pww = input.width;
  for (int l = 0; l < nl; ++l) {
    const std::uint64_t fbytes = std::uint64_t(w[l].size()) * 4;
    r.traffic.host_to_device_bytes += fbytes;
    r.traffic.global_loads_bytes += detail::map_bytes(pc, phh, pww) + fbytes;
    if (fb[l] || m == SCONV_METHOD_ECR || !net.layers[l].pool) {
      if (m == SCONV_METHOD_PECR) r.pecr_fallback_layers.push_back(l);
      r.traffic.global_stores_bytes += detail::map_bytes(cc[l], ch[l], cw[l]);
      if (net.layers[l].pool) {
        r.traffic.global_loads_bytes += detail::map_bytes(cc[l], ch[l], cw[l]);
        r.traffic.global_stores_bytes += detail::map_bytes(cc[l], lh[l], lw[l]);
      }
    } else {
      r.traffic.global_stores_bytes += detail::map_bytes(cc[l], lh[l], lw[l]);
    }
    if (opt.keep_intermediates) {
      r.conv_outputs.push_back(cop[l] ? FeatureMap(cc[l], ch[l], cw[l], std::move(co[l]))
                                      : FeatureMap(1, 1, 1));
      r.layer_outputs.emplace_back(cc[l], lh[l], lw[l], std::move(lo[l]));
    }
    pc = cc[l], phh = lh[l], pww = lw[l];
  }
  r.traffic.device_to_host_bytes = detail::map_bytes(pc, phh, pww);
  r.output = FeatureMap(pc, phh, pww, std::move(y));
  return r;
}

}  // namespace sconv::cuda
