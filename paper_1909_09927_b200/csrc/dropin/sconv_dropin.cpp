// sconv_dropin.cpp -- GPU drop-in for the reference's ECR / PECR translation
// units (proj/src/ecr.cpp, proj/src/pecr.cpp).
//
// Compiled against the reference's UNCHANGED public headers
// (proj/include/sconv/{ecr,pecr,tensor,exec,metrics,errors}.hpp): every
// signature below is the reference's, byte for byte.  A maintainer swaps
// src/ecr.cpp + src/pecr.cpp for this file in src/CMakeLists.txt and links
// libsconv_cuda.so; the rest of libsconv (tensor, exec,
// metrics, dataset, pipeline, report) is untouched, so multichannel_conv and
// forward() run on the GPU through these entry points.
//
// Each call runs on a per-thread CUDA context (device $SCONV_CUDA_DEVICE,
// default 0), so the reference's "safe to call concurrently" contract holds.
// Arithmetic is EXACT (bit-identical to the reference) unless
// $SCONV_CUDA_MODE=fast.  C ABI statuses map onto the reference exceptions.
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "sconv/ecr.hpp"
#include "sconv/errors.hpp"
#include "sconv/exec.hpp"
#include "sconv/pecr.hpp"
#include "sconv/tensor.hpp"
#include "sconv_cuda.h"

namespace sconv {

namespace {

struct ThreadCtx {
  sconv_cu_ctx* h = nullptr;
  ~ThreadCtx() {
    if (h) sconv_cu_ctx_destroy(h);
  }
};

[[noreturn]] void raise_status(int rc, const sconv_cu_ctx* c) {
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

void check(int rc, const sconv_cu_ctx* c = nullptr) {
  if (rc != SCONV_OK) raise_status(rc, c);
}

sconv_cu_ctx* ctx() {
  thread_local ThreadCtx t;
  if (!t.h) {
    const char* e = std::getenv("SCONV_CUDA_DEVICE");
    check(sconv_cu_ctx_create(e ? std::atoi(e) : 0, &t.h));
  }
  return t.h;
}

unsigned flags() {
  const char* e = std::getenv("SCONV_CUDA_MODE");
  return (e && std::strcmp(e, "fast") == 0) ? SCONV_F_FAST : SCONV_F_EXACT;
}

// dispatch() rejects workers < 1 (include/sconv/exec.hpp:62); keep that.
void check_exec(const ExecConfig& exec) {
  if (exec.workers < 1) throw ConfigError("workers must be >= 1");
}

void check_channels(const FeatureMap& map, const Filter& filter) {
  if (filter.channels != map.channels) {  // ecr.cpp:53-56, pecr.cpp:87-90
    throw ShapeError("filter channels " + std::to_string(filter.channels) +
                     " != map channels " + std::to_string(map.channels));
  }
}

OutputDims out_dims(int in_w, int in_h, int k_w, int k_h, int stride) {
  int ow = 0, oh = 0;
  check(sconv_conv_output_dims(in_w, in_h, k_w, k_h, stride, &ow, &oh));
  return {ow, oh};
}

}  // namespace

EcrGridShape ecr_grid_shape(int in_w, int in_h, int k_w, int k_h, int stride) {
  const OutputDims o = out_dims(in_w, in_h, k_w, k_h, stride);
  return {o.height, o.width};
}

EcrMap ecr_convert(const FeatureMap& map, const Filter& filter, const ConvConfig& cfg,
                   const ExecConfig& exec) {
  check_channels(map, filter);
  const OutputDims o = out_dims(map.width, map.height, filter.width, filter.height, cfg.stride);
  check_exec(exec);
  EcrMap ecr;
  ecr.dims = {map.width, map.height, filter.width, filter.height, cfg.stride, map.channels};
  const std::size_t slot = static_cast<std::size_t>(ecr.dims.slot());
  const std::size_t nwin = static_cast<std::size_t>(o.width) * o.height;
  std::vector<int32_t> ptr(nwin), offsets(nwin * slot);
  std::vector<float> f_data(nwin * slot), k_data(nwin * slot);
  sconv_cu_ctx* c = ctx();
  check(sconv_cu_ecr_convert(c, map.values.data(), map.channels, map.height, map.width,
                             filter.weights.data(), filter.height, filter.width, cfg.stride,
                             ptr.data(), offsets.data(), f_data.data(), k_data.data(), flags()),
        c);
  ecr.block_rows.resize(o.height);
  const std::size_t row = static_cast<std::size_t>(o.width) * slot;
  for (int b = 0; b < o.height; ++b) {
    EcrBlockRow& r = ecr.block_rows[b];
    r.f_data.assign(f_data.begin() + b * row, f_data.begin() + (b + 1) * row);
    r.k_data.assign(k_data.begin() + b * row, k_data.begin() + (b + 1) * row);
    r.offsets.assign(offsets.begin() + b * row, offsets.begin() + (b + 1) * row);
    r.ptr.assign(ptr.begin() + static_cast<std::size_t>(b) * o.width,
                 ptr.begin() + static_cast<std::size_t>(b + 1) * o.width);
  }
  return ecr;
}

FeatureMap ecr_spmv_conv(const EcrMap& ecr, OpCount* counters, const ExecConfig& exec) {
  // structural half of check_ecr (ecr.cpp:22-42); ptr ranges are checked by
  // the library and come back as FormatError too.
  const EcrDims& d = ecr.dims;
  const int threads = d.out_w(), slot = d.slot();
  if (static_cast<int>(ecr.block_rows.size()) != d.out_h())
    throw FormatError("block row count does not match output height");
  const std::size_t want = static_cast<std::size_t>(threads) * slot;
  for (const EcrBlockRow& r : ecr.block_rows) {
    if (r.f_data.size() != want || r.k_data.size() != want || r.offsets.size() != want ||
        static_cast<int>(r.ptr.size()) != threads)
      throw FormatError("block row arrays do not match thread count");
  }
  check_exec(exec);
  const std::size_t nwin = static_cast<std::size_t>(threads) * d.out_h();
  std::vector<int32_t> ptr;
  std::vector<float> f, k;
  ptr.reserve(nwin);
  f.reserve(nwin * slot);
  k.reserve(nwin * slot);
  for (const EcrBlockRow& r : ecr.block_rows) {
    ptr.insert(ptr.end(), r.ptr.begin(), r.ptr.end());
    f.insert(f.end(), r.f_data.begin(), r.f_data.end());
    k.insert(k.end(), r.k_data.begin(), r.k_data.end());
  }
  FeatureMap out(1, d.out_h(), d.out_w());
  uint64_t muls = 0, adds = 0;
  sconv_cu_ctx* c = ctx();
  check(sconv_cu_ecr_spmv(c, ptr.data(), f.data(), k.data(), d.out_h(), d.out_w(), slot,
                          out.values.data(), &muls, &adds, flags()),
        c);
  if (counters) counters->merge(OpCount{muls, adds});
  return out;
}

std::vector<float> ecr_window(const EcrMap& ecr, int block, int thread) {
  const EcrDims& d = ecr.dims;
  if (block < 0 || block >= d.out_h() || thread < 0 || thread >= d.out_w())
    throw ShapeError("window index out of range");
  const EcrBlockRow& row = ecr.block_rows[block];
  const std::size_t base = static_cast<std::size_t>(thread) * d.slot();
  std::vector<float> window(d.slot(), 0.0f);
  const int nnz = row.ptr[thread] < 0 ? 0 : row.ptr[thread];
  for (int p = 0; p < nnz; ++p) window[row.offsets[base + p]] = row.f_data[base + p];
  return window;
}

int pecr_pack_count(int in_extent, int k_extent, int conv_stride, int pool_extent,
                    int pool_stride) {
  int packs = 0;
  check(sconv_pecr_pack_count(in_extent, k_extent, conv_stride, pool_extent, pool_stride,
                              &packs));
  return packs;
}

PecrMap pecr_convert(const FeatureMap& map, const Filter& filter, const ConvConfig& conv,
                     const PoolConfig& pool, const ExecConfig& exec) {
  check_channels(map, filter);
  out_dims(map.width, map.height, filter.width, filter.height, conv.stride);
  const int packs_w = pecr_pack_count(map.width, filter.width, conv.stride, pool.width,
                                      pool.stride);
  const int packs_h = pecr_pack_count(map.height, filter.height, conv.stride, pool.height,
                                      pool.stride);
  check_exec(exec);
  PecrMap pecr;
  pecr.dims = {map.width, map.height, filter.width, filter.height, conv.stride, map.channels,
               pool};
  pecr.kernel = filter.weights;
  const int wpp = pecr.dims.windows_per_pack();
  const std::size_t npacks = static_cast<std::size_t>(packs_h) * packs_w;
  std::vector<int32_t> count(npacks * wpp);
  std::vector<int64_t> start(npacks + 1);
  int64_t total = 0;
  sconv_cu_ctx* c = ctx();
  check(sconv_cu_pecr_count(c, map.values.data(), map.channels, map.height, map.width,
                            filter.height, filter.width, conv.stride, pool.width, pool.height,
                            pool.stride, count.data(), start.data(), &total, flags()),
        c);
  std::vector<float> data(static_cast<std::size_t>(total));
  std::vector<int32_t> index(static_cast<std::size_t>(total));
  check(sconv_cu_pecr_fill(c, map.values.data(), map.channels, map.height, map.width,
                           filter.height, filter.width, conv.stride, pool.width, pool.height,
                           pool.stride, start.data(), total, data.data(), index.data(), flags()),
        c);
  pecr.pool_rows.assign(packs_h, std::vector<PecrPoolPack>(packs_w));
  for (int b = 0; b < packs_h; ++b) {
    for (int t = 0; t < packs_w; ++t) {
      const std::size_t pk = static_cast<std::size_t>(b) * packs_w + t;
      PecrPoolPack& pack = pecr.pool_rows[b][t];
      pack.count.assign(count.begin() + pk * wpp, count.begin() + (pk + 1) * wpp);
      pack.data.assign(data.begin() + start[pk], data.begin() + start[pk + 1]);
      pack.index.assign(index.begin() + start[pk], index.begin() + start[pk + 1]);
    }
  }
  return pecr;
}

FeatureMap pecr_conv_pool(const PecrMap& pecr, OpCount* counters, const ExecConfig& exec) {
  // structural half of check_pecr (pecr.cpp:24-58); count / index ranges
  // and data lengths are checked by the library (FormatError).
  const PecrDims& d = pecr.dims;
  const int packs_w = pecr_pack_count(d.in_w, d.k_w, d.conv_stride, d.pool.width, d.pool.stride);
  const int packs_h = pecr_pack_count(d.in_h, d.k_h, d.conv_stride, d.pool.height, d.pool.stride);
  if (pecr.packs_h() != packs_h) throw FormatError("pack row count mismatch");
  const std::size_t cap = static_cast<std::size_t>(d.channels) * d.k_h * d.k_w;
  if (pecr.kernel.size() != cap) throw FormatError("kernel length does not match dims");
  const int wpp = d.windows_per_pack();
  std::vector<int32_t> count;
  std::vector<int64_t> start{0};
  std::vector<float> data;
  std::vector<int32_t> index;
  for (const auto& row : pecr.pool_rows) {
    if (static_cast<int>(row.size()) != packs_w) throw FormatError("pack count mismatch");
    for (const PecrPoolPack& pack : row) {
      if (static_cast<int>(pack.count.size()) != wpp)
        throw FormatError("count length does not match windows per pack");
      if (pack.data.size() != pack.index.size())
        throw FormatError("data/index length inconsistent with counts");
      count.insert(count.end(), pack.count.begin(), pack.count.end());
      data.insert(data.end(), pack.data.begin(), pack.data.end());
      index.insert(index.end(), pack.index.begin(), pack.index.end());
      start.push_back(start.back() + static_cast<int64_t>(pack.data.size()));
    }
  }
  check_exec(exec);
  FeatureMap out(1, packs_h, packs_w);
  uint64_t muls = 0, adds = 0;
  sconv_cu_ctx* c = ctx();
  check(sconv_cu_pecr_pool(c, count.data(), start.data(), data.data(), index.data(), start.back(),
                           pecr.kernel.data(), d.channels, d.k_h, d.k_w, packs_h, packs_w,
                           d.pool.width, d.pool.height,
                           d.pool.mode == PoolMode::kMax ? SCONV_POOL_MAX : SCONV_POOL_MEAN,
                           out.values.data(), &muls, &adds, flags()),
        c);
  if (counters) counters->merge(OpCount{muls, adds});
  return out;
}

std::vector<float> pecr_window(const PecrMap& pecr, int pack_row, int pack_col, int n) {
  const PecrDims& d = pecr.dims;
  if (pack_row < 0 || pack_row >= pecr.packs_h() || pack_col < 0 ||
      pack_col >= pecr.packs_w() || n < 0 || n >= d.windows_per_pack())
    throw ShapeError("pack window index out of range");
  const PecrPoolPack& pack = pecr.pool_rows[pack_row][pack_col];
  std::size_t pos = 0;
  for (int m = 0; m < n; ++m) pos += static_cast<std::size_t>(pack.count[m]);
  std::vector<float> window(static_cast<std::size_t>(d.channels) * d.k_h * d.k_w, 0.0f);
  for (std::size_t p = pos; p < pos + static_cast<std::size_t>(pack.count[n]); ++p)
    window[pack.index[p]] = pack.data[p];
  return window;
}

}  // namespace sconv
