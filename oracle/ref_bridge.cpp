// ref_bridge.cpp -- flat C entry points over the UNMODIFIED reference library.
//
// TEST INFRASTRUCTURE ONLY.  Built by oracle/Makefile together with the
// reference's own src/*.cpp (compiled in place from /root/reference, never
// copied) into oracle/_ref/libsconv_ref.so.  The whole reference namespace is
// renamed with -Dsconv=sconv_ref so it can share a process with the product's
// drop-in sconv:: symbols.  Used by tests/ to pin the C oracle and by
// bench.py's reference arm / cpu_baseline leg to time the reference itself.
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "sconv/dataset.hpp"
#include "sconv/ecr.hpp"
#include "sconv/errors.hpp"
#include "sconv/exec.hpp"
#include "sconv/pecr.hpp"
#include "sconv/pipeline.hpp"
#include "sconv/report.hpp"
#include "sconv/tensor.hpp"

using namespace sconv;  // == sconv_ref under -Dsconv=sconv_ref

namespace {

thread_local std::string g_err;

// 0 ok, 1 shape, 2 config, 3 format, 4 io, 5 dispatch, 9 other.
template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ShapeError& e) {
    g_err = e.what();
    return 1;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const FormatError& e) {
    g_err = e.what();
    return 3;
  } catch (const IoError& e) {
    g_err = e.what();
    return 4;
  } catch (const DispatchError& e) {
    g_err = e.what();
    return 5;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 9;
  }
}

FeatureMap as_map(const float* x, int C, int H, int W) {
  return FeatureMap(C, H, W, std::vector<float>(x, x + static_cast<std::size_t>(C) * H * W));
}

Filter as_filter(const float* w, int C, int kh, int kw) {
  return Filter(C, kh, kw, std::vector<float>(w, w + static_cast<std::size_t>(C) * kh * kw));
}

void add_ops(const OpCount& ops, uint64_t* muls, uint64_t* adds) {
  if (muls) *muls += ops.multiplications;
  if (adds) *adds += ops.additions;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_rng(uint64_t seed, int n, uint64_t* out) {
  Rng r(seed);
  for (int i = 0; i < n; ++i) out[i] = r.next();
}

int ref_generate(int h, int w, int c, double s, uint64_t seed, float* out) {
  return guarded([&] {
    const FeatureMap m = generate(h, w, c, s, seed);
    std::memcpy(out, m.values.data(), m.values.size() * sizeof(float));
  });
}

void ref_fixture_f5(float* out) {
  const FeatureMap m = fixture_f5();
  std::memcpy(out, m.values.data(), m.values.size() * sizeof(float));
}

void ref_fixture_k3(float* out) {
  const Filter f = fixture_k3();
  std::memcpy(out, f.weights.data(), f.weights.size() * sizeof(float));
}

int ref_conv_output_dims(int in_w, int in_h, int k_w, int k_h, int stride, int* ow, int* oh) {
  return guarded([&] {
    const OutputDims d = conv_output_dims(in_w, in_h, k_w, k_h, stride);
    *ow = d.width;
    *oh = d.height;
  });
}

int ref_dense_conv(const float* x, int C, int H, int W, const float* w, int kh, int kw,
                   int stride, float* y, uint64_t* muls, uint64_t* adds) {
  return guarded([&] {
    OpCount ops;
    const FeatureMap out = dense_conv(as_map(x, C, H, W), as_filter(w, C, kh, kw), {stride}, &ops);
    std::memcpy(y, out.values.data(), out.values.size() * sizeof(float));
    add_ops(ops, muls, adds);
  });
}

int ref_relu_pool(const float* x, int C, int H, int W, int relu_first, int pw, int ph, int ps,
                  int mode, float* y) {
  return guarded([&] {
    FeatureMap m = as_map(x, C, H, W);
    if (relu_first) m = relu(m);
    const FeatureMap out = pool(m, {pw, ph, ps, mode == 0 ? PoolMode::kMax : PoolMode::kMean});
    std::memcpy(y, out.values.data(), out.values.size() * sizeof(float));
  });
}

// ecr_convert -> flat arrays (ecr.cpp:51-97).
int ref_ecr_convert(const float* x, int C, int H, int W, const float* w, int kh, int kw,
                    int stride, int workers, int32_t* ptr, int32_t* offsets, float* f_data,
                    float* k_data) {
  return guarded([&] {
    ExecConfig ex;
    ex.workers = workers;
    const EcrMap e = ecr_convert(as_map(x, C, H, W), as_filter(w, C, kh, kw), {stride}, ex);
    const int ow = e.dims.out_w(), slot = e.dims.slot();
    for (std::size_t b = 0; b < e.block_rows.size(); ++b) {
      const EcrBlockRow& r = e.block_rows[b];
      const std::size_t base = b * ow * static_cast<std::size_t>(slot);
      std::memcpy(ptr + b * ow, r.ptr.data(), ow * sizeof(int32_t));
      std::memcpy(offsets + base, r.offsets.data(), r.offsets.size() * sizeof(int32_t));
      std::memcpy(f_data + base, r.f_data.data(), r.f_data.size() * sizeof(float));
      std::memcpy(k_data + base, r.k_data.data(), r.k_data.size() * sizeof(float));
    }
  });
}

// ecr_convert + ecr_spmv_conv for every (image, filter) pair, exactly the
// per-filter loop of multichannel_conv (pipeline.cpp:201-208).
int ref_ecr_conv(const float* x, int N, int C, int H, int W, const float* w, int K, int kh,
                 int kw, int stride, int workers, float* y, uint64_t* muls, uint64_t* adds) {
  return guarded([&] {
    ExecConfig ex;
    ex.workers = workers;
    const std::size_t in_sz = static_cast<std::size_t>(C) * H * W;
    const std::size_t f_sz = static_cast<std::size_t>(C) * kh * kw;
    std::size_t pos = 0;
    for (int n = 0; n < N; ++n) {
      const FeatureMap map = as_map(x + n * in_sz, C, H, W);
      for (int k = 0; k < K; ++k) {
        OpCount ops;
        const EcrMap e = ecr_convert(map, as_filter(w + k * f_sz, C, kh, kw), {stride}, ex);
        const FeatureMap out = ecr_spmv_conv(e, &ops, ex);
        std::memcpy(y + pos, out.values.data(), out.values.size() * sizeof(float));
        pos += out.values.size();
        add_ops(ops, muls, adds);
      }
    }
  });
}

int ref_pecr_pack_count(int in, int k, int cs, int p, int ps, int* out) {
  return guarded([&] { *out = pecr_pack_count(in, k, cs, p, ps); });
}

// pecr_convert -> flat arrays (pecr.cpp:83-131).  With data == nullptr only
// the total entry count is returned through *total.
int ref_pecr_convert(const float* x, int C, int H, int W, const float* w, int kh, int kw,
                     int stride, int pw, int ph, int ps, int workers, int32_t* count,
                     int64_t* pack_start, float* data, int32_t* index, int64_t* total) {
  return guarded([&] {
    ExecConfig ex;
    ex.workers = workers;
    const PecrMap p = pecr_convert(as_map(x, C, H, W), as_filter(w, C, kh, kw), {stride},
                                   {pw, ph, ps, PoolMode::kMax}, ex);
    int64_t pos = 0;
    std::size_t pk = 0;
    const int wpp = p.dims.windows_per_pack();
    for (const auto& row : p.pool_rows) {
      for (const PecrPoolPack& pack : row) {
        if (data) {
          pack_start[pk] = pos;
          std::memcpy(count + pk * wpp, pack.count.data(), wpp * sizeof(int32_t));
          std::memcpy(data + pos, pack.data.data(), pack.data.size() * sizeof(float));
          std::memcpy(index + pos, pack.index.data(), pack.index.size() * sizeof(int32_t));
        }
        pos += static_cast<int64_t>(pack.data.size());
        ++pk;
      }
    }
    if (data) pack_start[pk] = pos;
    *total = pos;
  });
}

// pecr_convert + pecr_conv_pool for every (image, filter) pair, exactly the
// fused branch of forward (pipeline.cpp:252-256).
int ref_pecr_conv(const float* x, int N, int C, int H, int W, const float* w, int K, int kh,
                  int kw, int stride, int pw, int ph, int ps, int mode, int workers, float* y,
                  uint64_t* muls, uint64_t* adds) {
  return guarded([&] {
    ExecConfig ex;
    ex.workers = workers;
    const PoolConfig pool{pw, ph, ps, mode == 0 ? PoolMode::kMax : PoolMode::kMean};
    const std::size_t in_sz = static_cast<std::size_t>(C) * H * W;
    const std::size_t f_sz = static_cast<std::size_t>(C) * kh * kw;
    std::size_t pos = 0;
    for (int n = 0; n < N; ++n) {
      const FeatureMap map = as_map(x + n * in_sz, C, H, W);
      for (int k = 0; k < K; ++k) {
        OpCount ops;
        const PecrMap p = pecr_convert(map, as_filter(w + k * f_sz, C, kh, kw), {stride}, pool, ex);
        const FeatureMap out = pecr_conv_pool(p, &ops, ex);
        std::memcpy(y + pos, out.values.data(), out.values.size() * sizeof(float));
        pos += out.values.size();
        add_ops(ops, muls, adds);
      }
    }
  });
}

int ref_window_nnz(const float* x, int C, int H, int W, int kh, int kw, int stride,
                   int32_t* counts) {
  return guarded([&] {
    const std::vector<int> c = window_nnz_counts(as_map(x, C, H, W), kw, kh, stride);
    std::memcpy(counts, c.data(), c.size() * sizeof(int32_t));
  });
}

int ref_checksum(const float* v, int64_t n, char* out17) {
  return guarded([&] {
    const std::string s = checksum_hex(std::vector<float>(v, v + n));
    std::memcpy(out17, s.c_str(), 17);
  });
}

// plan() (exec.cpp:8-36): fmt 0 = ECR, 1 = PECR.
int ref_plan(int in_w, int in_h, int k_w, int k_h, int stride, int channels, int fmt, int pw,
             int ph, int ps, int* blocks, int* threads, uint64_t* smem) {
  return guarded([&] {
    LayerDims d;
    d.in_w = in_w;
    d.in_h = in_h;
    d.k_w = k_w;
    d.k_h = k_h;
    d.stride = stride;
    d.channels = channels;
    if (fmt == 1) d.pool = PoolDims{pw, ph, ps};
    const Grid g = plan(d, fmt == 0 ? Format::kEcr : Format::kPecr);
    *blocks = g.blocks;
    *threads = g.threads_per_block;
    *smem = g.shared_bytes_per_block;
  });
}

// forward (pipeline.cpp:212-301) over a network given as flat arrays; writes
// every layer output (concatenated) and every conv output (concatenated, each
// at its conv-output size; fused layers' 1x1x1 placeholders leave theirs 0).
int ref_forward(const float* x, int C, int H, int W, int nl, const int* k, const int* kh,
                const int* kw, const int* stride, const int* relu, const int* pw, const int* ph,
                const int* ps, const int* pmode, const float* const* filters, int method,
                int workers, float* layer_out, float* conv_out, uint64_t* muls, uint64_t* adds,
                int* fallback) {
  return guarded([&] {
    NetworkSpec net;
    net.in_channels = C;
    net.in_height = H;
    net.in_width = W;
    int c = C;
    for (int l = 0; l < nl; ++l) {
      LayerSpec L;
      for (int f = 0; f < k[l]; ++f)
        L.filters.push_back(as_filter(filters[l] + static_cast<std::size_t>(f) * c * kh[l] * kw[l],
                                      c, kh[l], kw[l]));
      L.conv.stride = stride[l];
      L.activation = relu[l] ? Activation::kRelu : Activation::kNone;
      if (pw[l] > 0) {
        L.kind = LayerKind::kConvPool;
        L.pool = PoolConfig{pw[l], ph[l], ps[l], pmode[l] == 0 ? PoolMode::kMax : PoolMode::kMean};
      }
      net.layers.push_back(std::move(L));
      c = k[l];
    }
    ExecConfig ex;
    ex.workers = workers;
    const Method m = method == 0 ? Method::kDense : method == 1 ? Method::kEcr : Method::kPecr;
    const ForwardResult r = forward(net, as_map(x, C, H, W), m, ex);
    std::size_t p = 0, q = 0;
    int ih = H, iw = W;
    for (int l = 0; l < nl; ++l) {
      const auto& v = r.layer_outputs[l].values;
      std::memcpy(layer_out + p, v.data(), v.size() * sizeof(float));
      p += v.size();
      const bool fused = m == Method::kPecr && pw[l] > 0 && relu[l];
      const auto& cv = r.conv_outputs[l].values;
      if (!fused) std::memcpy(conv_out + q, cv.data(), cv.size() * sizeof(float));
      q += static_cast<std::size_t>(k[l]) * ((ih - kh[l]) / stride[l] + 1) *
           ((iw - kw[l]) / stride[l] + 1);
      ih = r.layer_outputs[l].height;
      iw = r.layer_outputs[l].width;
      fallback[l] = 0;
    }
    for (int l : r.pecr_fallback_layers) fallback[l] = 1;
    add_ops(r.ops, muls, adds);
  });
}

// sparsity_profile (dataset.cpp:270-286) of one map.
int ref_sparsity_profile(const float* x, int C, int H, int W, int kw, int kh, int stride,
                         double* raw, double* ext) {
  return guarded([&] {
    const auto p = sparsity_profile({as_map(x, C, H, W)}, kw, kh, stride);
    *raw = p[0].raw;
    *ext = p[0].extended;
  });
}

// save / load (dataset.cpp:232-243) of the reference, FMAP or CSV by extension.
int ref_save_map(const char* path, const float* x, int C, int H, int W) {
  return guarded([&] { save(as_map(x, C, H, W), path); });
}

int ref_load_map(const char* path, float* out, int64_t cap, int* C, int* H, int* W) {
  return guarded([&] {
    const FeatureMap m = load(path);
    *C = m.channels, *H = m.height, *W = m.width;
    if (static_cast<int64_t>(m.values.size()) > cap) throw std::runtime_error("capacity");
    std::memcpy(out, m.values.data(), m.values.size() * sizeof(float));
  });
}

int ref_hardware_concurrency() { return static_cast<int>(std::thread::hardware_concurrency()); }

}  // extern "C"
