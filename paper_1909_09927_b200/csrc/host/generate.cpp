// generate.cpp -- host side of the C ABI that needs no device: synthetic
// inputs bit-identical to sconv::generate, the FNV-1a checksum, and the
// multi-GPU shard rule.
//
// sconv::generate (src/dataset.cpp:77-100) is a sequential Fisher-Yates
// shuffle driven by xoshiro256**; it cannot be split inside one map without
// changing its bits, so the batch form runs one map per host thread.  The
// permutation uses 32-bit indices when the map has < 2^32 elements (same
// swaps, half the memory traffic of the reference's size_t array).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "sconv_cuda.h"

namespace {

struct Xoshiro256ss {  // Rng, src/dataset.cpp:55-75
  uint64_t s[4];
  explicit Xoshiro256ss(uint64_t seed) {
    for (auto& v : s) {  // SplitMix64 seeding
      seed += 0x9E3779B97F4A7C15ull;
      uint64_t z = seed;
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      v = z ^ (z >> 31);
    }
  }
  static uint64_t rotl(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }
  uint64_t next() {
    const uint64_t out = rotl(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return out;
  }
  double unit() { return static_cast<double>((next() >> 11) + 1) * 0x1.0p-53; }
};

template <typename Idx>
void generate_into(size_t total, double sparsity, uint64_t seed, float* out) {
  const size_t zeros = static_cast<size_t>(std::floor(sparsity * static_cast<double>(total)));
  Xoshiro256ss rng(seed);
  std::vector<Idx> perm(total);
  for (size_t i = 0; i < total; ++i) perm[i] = static_cast<Idx>(i);
  for (size_t i = total - 1; i > 0; --i) {
    const size_t j = static_cast<size_t>(rng.next() % static_cast<uint64_t>(i + 1));
    std::swap(perm[i], perm[j]);
  }
  // Mark zeros in the output itself (NaN-free sentinel: bit pattern 1).
  std::memset(out, 0, total * sizeof(float));
  uint32_t one = 1;
  float mark;
  std::memcpy(&mark, &one, 4);
  for (size_t i = 0; i < zeros; ++i) out[perm[i]] = mark;
  for (size_t p = 0; p < total; ++p) {
    uint32_t bits;
    std::memcpy(&bits, &out[p], 4);
    out[p] = bits == 1u ? 0.0f : static_cast<float>(rng.unit());
  }
}

int generate_one(int h, int w, int c, double s, uint64_t seed, float* out) {
  if (!(s >= 0.0 && s <= 1.0)) return SCONV_ERR_CONFIG;
  if (h < 1 || w < 1 || c < 1) return SCONV_ERR_SHAPE;
  if (!out) return SCONV_ERR_ARG;
  const size_t total = static_cast<size_t>(c) * h * w;
  if (total < (size_t{1} << 32))
    generate_into<uint32_t>(total, s, seed, out);
  else
    generate_into<uint64_t>(total, s, seed, out);
  return SCONV_OK;
}

}  // namespace

extern "C" {

int sconv_generate(int height, int width, int channels, double sparsity, uint64_t seed,
                   float* out) {
  return generate_one(height, width, channels, sparsity, seed, out);
}

int sconv_generate_batch(int count, int height, int width, int channels, double sparsity,
                         const uint64_t* seeds, float* out, int threads) {
  if (count < 0 || (count > 0 && (!seeds || !out))) return SCONV_ERR_ARG;
  if (!(sparsity >= 0.0 && sparsity <= 1.0)) return SCONV_ERR_CONFIG;
  if (height < 1 || width < 1 || channels < 1) return SCONV_ERR_SHAPE;
  const size_t per = static_cast<size_t>(channels) * height * width;
  int nt = threads > 0 ? threads : static_cast<int>(std::thread::hardware_concurrency());
  nt = std::max(1, std::min(nt, count));
  std::atomic<int> next{0};
  std::atomic<int> rc{SCONV_OK};
  auto worker = [&] {
    for (int i; (i = next.fetch_add(1)) < count;) {
      const int r = generate_one(height, width, channels, sparsity, seeds[i], out + i * per);
      if (r != SCONV_OK) rc.store(r);
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < nt; ++t) pool.emplace_back(worker);
  worker();
  for (auto& t : pool) t.join();
  return rc.load();
}

uint64_t sconv_checksum(const float* values, int64_t n) {  // src/report.cpp:14-30
  uint64_t h = 0xcbf29ce484222325ull;
  for (int64_t i = 0; i < n; ++i) {
    uint32_t bits;
    std::memcpy(&bits, values + i, 4);
    for (int sh = 0; sh < 32; sh += 8) {
      h ^= (bits >> sh) & 0xffu;
      h *= 0x100000001b3ull;
    }
  }
  return h;
}

// Contiguous partition like dispatch's block-row split (exec.hpp:91-93):
// part p of `parts` covers [total*p/parts, total*(p+1)/parts).
int sconv_shard(int n, int k, int world, int rank, int* n_begin, int* n_end, int* k_begin,
                int* k_end) {
  if (!n_begin || !n_end || !k_begin || !k_end) return SCONV_ERR_ARG;
  if (world < 1 || rank < 0 || rank >= world) return SCONV_ERR_CONFIG;
  if (n < 0 || k < 0) return SCONV_ERR_SHAPE;
  auto cut = [](int total, int parts, int p) {
    return static_cast<int>(static_cast<int64_t>(total) * p / parts);
  };
  if (n >= world || k < world) {
    *n_begin = cut(n, world, rank);
    *n_end = cut(n, world, rank + 1);
    *k_begin = 0;
    *k_end = k;
  } else {
    *n_begin = 0;
    *n_end = n;
    *k_begin = cut(k, world, rank);
    *k_end = cut(k, world, rank + 1);
  }
  return SCONV_OK;
}

}  // extern "C"
