// cuda_hpp_test.cpp -- TEST INFRASTRUCTURE: include/sconv/cuda.hpp (the
// batched C++ entry points) against the unmodified reference, both in one
// binary: the reference's own src/*.cpp (CPU, namespace sconv) and
// sconv::cuda::* (GPU, through libsconv_cuda.so).
//
//   cuda_hpp_test          parity: bit-identical outputs, equal OpCounts,
//                          equal ForwardResult (ops, traffic model, fallback
//                          layers, per-layer outputs), the reference errors
//   cuda_hpp_test --time   one VGG-19 layer through the reference
//                          multichannel_conv / forward's fused branch on all
//                          host cores vs the batched GPU entries (JSON line)
#include <chrono>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "sconv/cuda.hpp"
#include "sconv/dataset.hpp"
#include "sconv/ecr.hpp"
#include "sconv/pecr.hpp"
#include "sconv/pipeline.hpp"

using namespace sconv;

static int failures = 0;
#define EXPECT(cond)                                                   \
  do {                                                                 \
    if (!(cond)) {                                                     \
      std::fprintf(stderr, "FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++failures;                                                      \
    }                                                                  \
  } while (0)

static bool same_bits(const FeatureMap& a, const FeatureMap& b) {
  return a.channels == b.channels && a.height == b.height && a.width == b.width &&
         std::memcmp(a.values.data(), b.values.data(), a.values.size() * 4) == 0;
}

static std::vector<Filter> filters(int k, int c, int kh, std::uint64_t seed) {
  std::vector<Filter> f;
  for (int j = 0; j < k; ++j) {
    FeatureMap g = generate(kh, kh, c, 0.0, seed + j);
    for (float& v : g.values) v -= 0.5f;
    f.emplace_back(c, kh, kh, g.values);
  }
  return f;
}

// forward's fused branch on the CPU reference: per filter pecr_convert +
// pecr_conv_pool, stacked (src/pipeline.cpp:249-264)
static FeatureMap ref_conv_pool(const FeatureMap& m, const std::vector<Filter>& fs, const ConvConfig& cfg,
                                const PoolConfig& pool, OpCount* ops, const ExecConfig& exec) {
  std::vector<float> vals;
  int h = 0, w = 0;
  for (const Filter& f : fs) {
    const FeatureMap o = pecr_conv_pool(pecr_convert(m, f, cfg, pool, exec), ops, exec);
    h = o.height, w = o.width;
    vals.insert(vals.end(), o.values.begin(), o.values.end());
  }
  return FeatureMap(int(fs.size()), h, w, vals);
}

static void parity() {
  const ExecConfig exec{4};
  // multichannel_conv: one map and a batch
  std::vector<FeatureMap> maps;
  for (int i = 0; i < 3; ++i) maps.push_back(generate(20, 22, 16, 0.7, 40 + i));
  const auto fs = filters(64, 16, 3, 900);
  for (const FeatureMap& m : maps) {
    OpCount a, b;
    const FeatureMap ref = multichannel_conv(m, fs, ConvConfig{1}, Method::kEcr, exec, &a);
    const FeatureMap got = cuda::multichannel_conv(m, fs, ConvConfig{1}, Method::kEcr, exec, &b);
    EXPECT(same_bits(ref, got));
    EXPECT(a == b);
  }
  {
    OpCount a, b;
    const auto got = cuda::multichannel_conv(maps, fs, ConvConfig{1}, Method::kEcr, exec, &b);
    for (size_t i = 0; i < maps.size(); ++i)
      EXPECT(same_bits(multichannel_conv(maps[i], fs, ConvConfig{1}, Method::kEcr, exec, &a), got[i]));
    EXPECT(a == b);
  }
  // conv + ReLU + pool (2x2/2 and an overlapping 3x3/2)
  for (const PoolConfig pool : {PoolConfig{2, 2, 2, PoolMode::kMax}, PoolConfig{3, 3, 2, PoolMode::kMean}}) {
    // Eq. 3 needs an even extent for 2x2/2 (20 -> 18 -> 9) and an odd one for 3x3/2 (19 -> 17 -> 8)
    const int ext = pool.width == 2 ? 20 : 19;
    const FeatureMap m = generate(ext, ext, 16, 0.6, 77);
    OpCount a, b;
    const FeatureMap ref = ref_conv_pool(m, fs, ConvConfig{1}, pool, &a, exec);
    const FeatureMap got = cuda::conv_pool(m, fs, ConvConfig{1}, pool, &b);
    EXPECT(same_bits(ref, got));
    EXPECT(a == b);
  }
  // forward: conv+ReLU, conv+ReLU+pool (fused), conv without ReLU + pool (fallback)
  NetworkSpec net;
  net.in_channels = 8, net.in_height = 30, net.in_width = 30;
  LayerSpec l0;
  l0.filters = filters(32, 8, 3, 100);
  LayerSpec l1;
  l1.kind = LayerKind::kConvPool;
  l1.filters = filters(32, 32, 3, 200);
  l1.pool = PoolConfig{2, 2, 2, PoolMode::kMax};
  LayerSpec l2;
  l2.kind = LayerKind::kConvPool;
  l2.filters = filters(48, 32, 3, 300);
  l2.pool = PoolConfig{3, 3, 1, PoolMode::kMean};
  l2.activation = Activation::kNone;
  net.layers = {l0, l1, l2};
  const FeatureMap in = generate(30, 30, 8, 0.7, 5);
  for (Method method : {Method::kEcr, Method::kPecr}) {
    const ForwardResult ref = forward(net, in, method, exec);
    const ForwardResult got = cuda::forward(net, in, method, exec);
    EXPECT(same_bits(ref.output, got.output));
    EXPECT(ref.ops == got.ops);
    EXPECT(ref.traffic == got.traffic);
    EXPECT(ref.pecr_fallback_layers == got.pecr_fallback_layers);
    EXPECT(ref.layer_outputs.size() == got.layer_outputs.size());
    for (size_t l = 0; l < ref.layer_outputs.size(); ++l) {
      EXPECT(same_bits(ref.layer_outputs[l], got.layer_outputs[l]));
      EXPECT(same_bits(ref.conv_outputs[l], got.conv_outputs[l]));
    }
  }
  // the reference's exception types
  bool threw = false;
  try {
    cuda::multichannel_conv(in, filters(4, 3, 3, 1), ConvConfig{1});
  } catch (const ShapeError&) {
    threw = true;
  }
  EXPECT(threw);
  threw = false;
  try {
    cuda::conv_pool(in, filters(4, 8, 3, 1), ConvConfig{1}, PoolConfig{3, 3, 3, PoolMode::kMax});
  } catch (const ConfigError&) {
    threw = true;
  }
  EXPECT(threw);
  threw = false;
  try {
    cuda::forward(net, in, Method::kDense);
  } catch (const ConfigError&) {
    threw = true;
  }
  EXPECT(threw);
}

template <class F>
static double seconds(F&& f, int reps) {
  f();  // warm (contexts, workspaces)
  const auto t0 = std::chrono::steady_clock::now();
  for (int r = 0; r < reps; ++r) f();
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / reps;
}

// VGG-19 conv3_2 (256 -> 256 @ 56, valid 3x3 on a 58x58 map) and
// conv3_4's fused conv+ReLU+pool, sparsity 0.7: reference on every host core
// vs the batched GPU entries (host buffers in, host buffers out).
static void timing() {
  const int workers = int(std::thread::hardware_concurrency());
  const ExecConfig exec{workers};
  const auto fs = filters(256, 256, 3, 3'500'000);
  std::vector<FeatureMap> maps;
  for (int i = 0; i < 16; ++i) maps.push_back(generate(58, 58, 256, 0.7, 3'000'000 + i));
  const int cpu_k = 16;  // reference sample: 16 filters, extrapolated x 256
  const std::vector<Filter> fs16(fs.begin(), fs.begin() + cpu_k);
  const double ref_ecr = seconds([&] { multichannel_conv(maps[0], fs16, ConvConfig{1}, Method::kEcr, exec); }, 1) *
                         (256.0 / cpu_k);
  const PoolConfig pool{2, 2, 2, PoolMode::kMax};
  const double ref_pecr =
      seconds([&] { ref_conv_pool(maps[0], fs16, ConvConfig{1}, pool, nullptr, exec); }, 1) * (256.0 / cpu_k);
  const double gpu1 = seconds([&] { cuda::multichannel_conv(maps[0], fs, ConvConfig{1}); }, 10);
  const double gpu16 = seconds([&] { cuda::multichannel_conv(maps, fs, ConvConfig{1}); }, 5);
  const double gpup1 = seconds([&] { cuda::conv_pool(maps[0], fs, ConvConfig{1}, pool); }, 10);
  const double gpup16 = seconds([&] { cuda::conv_pool(maps, fs, ConvConfig{1}, pool); }, 5);
  std::printf(
      "{\"layer\": \"VGG-19 conv3_2 (ECR) / conv3_4 (PECR 2x2/2), 256->256 @56, s=0.7\", "
      "\"host_threads\": %d, \"ref_ecr_ms_per_image\": %.3f, \"ref_pecr_ms_per_image\": %.3f, "
      "\"ref_sample\": \"%d of 256 filters, extrapolated\", "
      "\"cuda_ecr_ms_batch1\": %.3f, \"cuda_ecr_ms_per_image_batch16\": %.3f, "
      "\"cuda_pecr_ms_batch1\": %.3f, \"cuda_pecr_ms_per_image_batch16\": %.3f, "
      "\"what\": \"sconv::cuda::multichannel_conv / conv_pool (include/sconv/cuda.hpp) with host "
      "FeatureMaps in and out (H2D + kernel + D2H) vs the reference's multichannel_conv / fused "
      "branch on all host cores\"}\n",
      workers, ref_ecr * 1e3, ref_pecr * 1e3, cpu_k, gpu1 * 1e3, gpu16 * 1e3 / 16, gpup1 * 1e3,
      gpup16 * 1e3 / 16);
}

int main(int argc, char** argv) {
  if (argc > 1 && std::strcmp(argv[1], "--time") == 0) {
    timing();
    return 0;
  }
  parity();
  if (failures) {
    std::printf("cuda_hpp_test: %d failure(s)\n", failures);
    return 1;
  }
  std::printf("cuda_hpp_test: ok\n");
  return 0;
}
