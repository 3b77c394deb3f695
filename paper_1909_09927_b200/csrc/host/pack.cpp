// pack.cpp -- host side of the compressed ingest: a batch of dense maps
// [n][C][H][W] -> nonzero bitmap + block offsets + packed nonzero values
// (layout in include/sconv_cuda.h, "compressed ingest").  The GPU expands it
// back (kernels/ingest.cuh) right before the convolution, so only the
// nonzeros and one bit per element cross PCIe -- the transfer saving the
// paper attributes to its compressed formats.  Zero test as
// ecr_convert's (src/ecr.cpp:84): v != 0.0f, so -0 is a zero.
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "sconv_cuda.h"

namespace {

constexpr int64_t kBlockElems = 1024;  // one device warp expands 32 words = 1024 elements

int64_t count_nonzeros(const float* x, int64_t e) {
  int64_t nz = 0;
  for (int64_t i = 0; i < e; ++i) nz += x[i] != 0.0f;
  return nz;
}

// Packs one image: bits[words], base[blocks + 1] (absolute, from `first`),
// values from `first`.
void pack_one(const float* x, int64_t e, uint32_t* bits, int64_t* base, float* values, int64_t first) {
  const int64_t words = (e + 31) / 32, blocks = (words + 31) / 32;
  int64_t pos = first;
  for (int64_t b = 0; b < blocks; ++b) {
    base[b] = pos;
    const int64_t w1 = std::min(words, (b + 1) * 32);
    for (int64_t wi = b * 32; wi < w1; ++wi) {
      const int64_t e0 = wi * 32, e1 = std::min(e, e0 + 32);
      uint32_t m = 0;
      for (int64_t i = e0; i < e1; ++i) {
        const float v = x[i];
        if (v != 0.0f) {
          m |= 1u << (i - e0);
          values[pos++] = v;
        }
      }
      bits[wi] = m;
    }
  }
  base[blocks] = pos;
}

template <typename F>
void parallel_images(int n, int threads, F&& f) {
  int nt = threads > 0 ? threads : static_cast<int>(std::thread::hardware_concurrency());
  nt = std::max(1, std::min(nt, n));
  std::atomic<int> next{0};
  auto worker = [&] {
    for (int i; (i = next.fetch_add(1)) < n;) f(i);
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) pool.emplace_back(worker);
  worker();
  for (auto& t : pool) t.join();
}

}  // namespace

extern "C" {

int sconv_packed_dims(int c, int h, int w, int64_t* words, int64_t* blocks) {
  if (c < 1 || h < 1 || w < 1) return SCONV_ERR_SHAPE;
  const int64_t e = int64_t(c) * h * w;
  const int64_t wd = (e + 31) / 32;
  if (words) *words = wd;
  if (blocks) *blocks = (wd + 31) / 32;
  return SCONV_OK;
}

int sconv_pack_maps(const float* x, int n, int c, int h, int w, uint32_t* bits, int64_t* base,
                    float* values, int64_t capacity, int64_t* nnz, int threads) {
  if (n < 0 || !nnz || (n > 0 && !x)) return SCONV_ERR_ARG;
  if (c < 1 || h < 1 || w < 1) return SCONV_ERR_SHAPE;
  const int64_t e = int64_t(c) * h * w, words = (e + 31) / 32, blocks = (words + 31) / 32;
  std::vector<int64_t> counts(size_t(n) + 1, 0);
  parallel_images(n, threads, [&](int i) { counts[i + 1] = count_nonzeros(x + i * e, e); });
  for (int i = 0; i < n; ++i) counts[i + 1] += counts[i];
  *nnz = counts[n];
  if (!bits && !base && !values) return SCONV_OK;  // size query
  if (!bits || !base || (counts[n] > 0 && !values)) return SCONV_ERR_ARG;
  if (counts[n] > capacity) return SCONV_ERR_ARG;
  parallel_images(n, threads, [&](int i) {
    pack_one(x + i * e, e, bits + i * words, base + i * (blocks + 1), values, counts[i]);
  });
  return SCONV_OK;
}

}  // extern "C"
