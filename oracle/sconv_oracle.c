/*
 * sconv_oracle.c -- plain-C restatement of the reference ECR/PECR path.
 * TEST INFRASTRUCTURE ONLY (see sconv_oracle.h for the rules and pinning).
 *
 * Build: oracle/Makefile, -O2 -ffp-contract=off.  The reference is compiled
 * for x86-64 without FMA, so every `acc += a*b` below is a rounded multiply
 * followed by a rounded add; the contraction ban keeps it that way.
 */
#include "sconv_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- Rng: dataset.cpp:23-75 ------------------------------------------- */

static uint64_t sm64(uint64_t* x) { /* SplitMix64, dataset.cpp:23-29 */
  uint64_t z = (*x += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static uint64_t rol64(uint64_t v, int k) { return (v << k) | (v >> (64 - k)); }

void orc_rng_seed(orc_rng* r, uint64_t seed) { /* Rng::Rng, :55-57 */
  for (int i = 0; i < 4; ++i) r->s[i] = sm64(&seed);
}

uint64_t orc_rng_next(orc_rng* r) { /* xoshiro256**, Rng::next :59-69 */
  uint64_t* s = r->s;
  const uint64_t out = rol64(s[1] * 5, 7) * 9;
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = rol64(s[3], 45);
  return out;
}

double orc_rng_next_unit(orc_rng* r) { /* (0,1], :71-73 */
  return (double)((orc_rng_next(r) >> 11) + 1) * 0x1.0p-53;
}

/* generate: dataset.cpp:77-100.  Exactly floor(s*N) zeros placed at the
 * first positions of a Fisher-Yates permutation (next()%(i+1) swaps from the
 * top), then one next_unit() per nonzero in storage order. */
int orc_generate(int height, int width, int channels, double sparsity,
                 uint64_t seed, float* out) {
  if (!(sparsity >= 0.0 && sparsity <= 1.0)) return ORC_CONFIG;
  if (channels < 1 || height < 1 || width < 1) return ORC_SHAPE;
  const size_t total = (size_t)channels * height * width;
  const size_t zeros = (size_t)floor(sparsity * (double)total);
  size_t* perm = (size_t*)malloc(total * sizeof(size_t));
  unsigned char* zero = (unsigned char*)calloc(total, 1);
  orc_rng rng;
  orc_rng_seed(&rng, seed);
  for (size_t i = 0; i < total; ++i) perm[i] = i;
  for (size_t i = total - 1; i > 0; --i) {
    const size_t j = (size_t)(orc_rng_next(&rng) % (uint64_t)(i + 1));
    const size_t t = perm[i];
    perm[i] = perm[j];
    perm[j] = t;
  }
  for (size_t i = 0; i < zeros; ++i) zero[perm[i]] = 1;
  for (size_t p = 0; p < total; ++p)
    out[p] = zero[p] ? 0.0f : (float)orc_rng_next_unit(&rng);
  free(perm);
  free(zero);
  return ORC_OK;
}

/* ---- tensor.cpp -------------------------------------------------------- */

int orc_conv_output_dims(int in_w, int in_h, int k_w, int k_h, int stride,
                         int* out_w, int* out_h) { /* tensor.cpp:44-55 */
  if (in_w < 1 || in_h < 1 || k_w < 1 || k_h < 1) return ORC_SHAPE;
  if (stride < 1) return ORC_CONFIG;
  if (k_w > in_w || k_h > in_h) return ORC_SHAPE;
  *out_w = (in_w - k_w) / stride + 1;
  *out_h = (in_h - k_h) / stride + 1;
  return ORC_OK;
}

#define AT(m, H, W, c, y, x) ((m)[((size_t)(c) * (H) + (y)) * (W) + (x)])

int orc_dense_conv(const float* map, int C, int H, int W, const float* filt,
                   int kh, int kw, int stride, float* out, uint64_t* muls,
                   uint64_t* adds) { /* tensor.cpp:57-87 */
  int ow, oh;
  int rc = orc_conv_output_dims(W, H, kw, kh, stride, &ow, &oh);
  if (rc) return rc;
  for (int y = 0; y < oh; ++y)
    for (int x = 0; x < ow; ++x) {
      float acc = 0.0f;
      for (int c = 0; c < C; ++c)
        for (int i = 0; i < kh; ++i)
          for (int j = 0; j < kw; ++j) {
            const float prod =
                AT(map, H, W, c, y * stride + i, x * stride + j) *
                AT(filt, kh, kw, c, i, j);
            acc = acc + prod;
          }
      out[(size_t)y * ow + x] = acc;
    }
  if (muls) *muls += (uint64_t)oh * ow * C * kh * kw;
  /* per-channel convention: first term of each channel is not an add */
  if (adds) *adds += (uint64_t)oh * ow * C * (kh * kw - 1);
  return ORC_OK;
}

void orc_relu(const float* in, int64_t n, float* out) { /* tensor.cpp:89-95 */
  for (int64_t i = 0; i < n; ++i) out[i] = in[i] > 0.0f ? in[i] : 0.0f;
}

int orc_pool(const float* in, int C, int H, int W, int pw, int ph, int ps,
             int mode, float* out) { /* tensor.cpp:97-129 */
  if (pw < 1 || ph < 1) return ORC_SHAPE;
  if (ps < 1) return ORC_CONFIG;
  int ow, oh;
  int rc = orc_conv_output_dims(W, H, pw, ph, ps, &ow, &oh);
  if (rc) return rc;
  const float cnt = (float)(pw * ph);
  for (int c = 0; c < C; ++c)
    for (int y = 0; y < oh; ++y)
      for (int x = 0; x < ow; ++x) {
        float r;
        if (mode == 0) {
          r = AT(in, H, W, c, y * ps, x * ps);
          for (int i = 0; i < ph; ++i)
            for (int j = 0; j < pw; ++j) {
              const float v = AT(in, H, W, c, y * ps + i, x * ps + j);
              if (v > r) r = v;
            }
        } else {
          float s = 0.0f;
          for (int i = 0; i < ph; ++i)
            for (int j = 0; j < pw; ++j) s = s + AT(in, H, W, c, y * ps + i, x * ps + j);
          r = s / cnt;
        }
        AT(out, oh, ow, c, y, x) = r;
      }
  return ORC_OK;
}

/* ---- ECR: ecr.cpp ------------------------------------------------------ */

int orc_ecr_convert(const float* map, int C, int H, int W, const float* filt,
                    int kh, int kw, int stride, int32_t* ptr, int32_t* offsets,
                    float* f_data, float* k_data) { /* ecr.cpp:51-97 */
  int ow, oh;
  int rc = orc_conv_output_dims(W, H, kw, kh, stride, &ow, &oh);
  if (rc) return rc;
  const int slot = C * kh * kw;
  for (int b = 0; b < oh; ++b)
    for (int t = 0; t < ow; ++t) {
      const size_t base = ((size_t)b * ow + t) * slot;
      int n = 0;
      for (int c = 0; c < C; ++c)
        for (int i = 0; i < kh; ++i)
          for (int j = 0; j < kw; ++j) {
            const float v = AT(map, H, W, c, b * stride + i, t * stride + j);
            if (v != 0.0f) { /* -0.0 is zero, ecr.cpp:84 */
              f_data[base + n] = v;
              k_data[base + n] = AT(filt, kh, kw, c, i, j);
              offsets[base + n] = (c * kh + i) * kw + j;
              ++n;
            }
          }
      for (int p = n; p < slot; ++p) { /* filler, ecr.cpp:64-70 */
        f_data[base + p] = 0.0f;
        k_data[base + p] = 0.0f;
        offsets[base + p] = -1;
      }
      ptr[(size_t)b * ow + t] = n ? n : -1; /* sentinel, ecr.cpp:93 */
    }
  return ORC_OK;
}

int orc_ecr_spmv_conv(const int32_t* ptr, const float* f_data,
                      const float* k_data, int o_h, int o_w, int slot,
                      float* out, uint64_t* muls, uint64_t* adds) {
  /* check_ecr ptr range, ecr.cpp:32-38 */
  for (size_t w = 0; w < (size_t)o_h * o_w; ++w)
    if (ptr[w] < -1 || ptr[w] > slot) return ORC_FORMAT;
  uint64_t m = 0, a = 0;
  for (size_t w = 0; w < (size_t)o_h * o_w; ++w) { /* ecr.cpp:109-124 */
    const int nnz = ptr[w];
    if (nnz == -1) {
      out[w] = 0.0f;
      continue;
    }
    const size_t base = w * slot;
    float acc = 0.0f;
    for (int p = 0; p < nnz; ++p) {
      const float prod = f_data[base + p] * k_data[base + p];
      acc = acc + prod;
    }
    out[w] = acc;
    m += (uint64_t)nnz;
    a += nnz > 0 ? (uint64_t)(nnz - 1) : 0;
  }
  if (muls) *muls += m;
  if (adds) *adds += a;
  return ORC_OK;
}

int orc_ecr_conv_batched(const float* x, int N, int C, int H, int W,
                         const float* w, int K, int kh, int kw, int stride,
                         float* y, uint64_t* muls, uint64_t* adds) {
  /* multichannel_conv's per-filter loop (pipeline.cpp:191-210), with the
   * convert+SpMV pair fused per window: same terms, same order, same ops. */
  int ow, oh;
  int rc = orc_conv_output_dims(W, H, kw, kh, stride, &ow, &oh);
  if (rc) return rc;
  const size_t in_sz = (size_t)C * H * W, f_sz = (size_t)C * kh * kw;
  uint64_t m = 0, a = 0;
  for (int n = 0; n < N; ++n) {
    const float* map = x + n * in_sz;
    for (int k = 0; k < K; ++k) {
      const float* filt = w + k * f_sz;
      float* out = y + ((size_t)n * K + k) * oh * ow;
      for (int b = 0; b < oh; ++b)
        for (int t = 0; t < ow; ++t) {
          float acc = 0.0f;
          int nnz = 0;
          for (int c = 0; c < C; ++c)
            for (int i = 0; i < kh; ++i)
              for (int j = 0; j < kw; ++j) {
                const float v = AT(map, H, W, c, b * stride + i, t * stride + j);
                if (v != 0.0f) {
                  const float prod = v * AT(filt, kh, kw, c, i, j);
                  acc = acc + prod;
                  ++nnz;
                }
              }
          out[(size_t)b * ow + t] = nnz ? acc : 0.0f;
          m += (uint64_t)nnz;
          a += nnz > 0 ? (uint64_t)(nnz - 1) : 0;
        }
    }
  }
  if (muls) *muls += m;
  if (adds) *adds += a;
  return ORC_OK;
}

/* ---- PECR: pecr.cpp ---------------------------------------------------- */

int orc_pecr_pack_count(int in_extent, int k_extent, int conv_stride,
                        int pool_extent, int pool_stride, int* packs) {
  /* Eq. 3, pecr.cpp:62-81 */
  if (in_extent < 1 || k_extent < 1 || conv_stride < 1 || pool_extent < 1 ||
      pool_stride < 1)
    return ORC_CONFIG;
  const int num = in_extent - k_extent + conv_stride -
                  conv_stride * pool_extent + pool_stride * conv_stride;
  const int den = pool_stride * conv_stride;
  if (num <= 0 || num % den != 0) return ORC_CONFIG;
  *packs = num / den;
  return ORC_OK;
}

static int pecr_geom(int C, int H, int W, int kh, int kw, int stride, int pw,
                     int ph, int ps, int* packs_w, int* packs_h) {
  int ow, oh;
  (void)C;
  int rc = orc_conv_output_dims(W, H, kw, kh, stride, &ow, &oh); /* :90 */
  if (rc) return rc;
  rc = orc_pecr_pack_count(W, kw, stride, pw, ps, packs_w);
  if (rc) return rc;
  return orc_pecr_pack_count(H, kh, stride, ph, ps, packs_h);
}

/* Window n of pack (b,t) starts at (b*cs*ps + (n/pw)*cs, t*cs*ps + (n%pw)*cs)
 * -- pecr.cpp:106-112. */
int64_t orc_pecr_total(const float* map, int C, int H, int W, int kh, int kw,
                       int stride, int pw, int ph, int ps) {
  int pW, pH;
  int rc = pecr_geom(C, H, W, kh, kw, stride, pw, ph, ps, &pW, &pH);
  if (rc) return -(int64_t)rc;
  int64_t total = 0;
  for (int b = 0; b < pH; ++b)
    for (int t = 0; t < pW; ++t)
      for (int n = 0; n < pw * ph; ++n) {
        const int wy = b * stride * ps + (n / pw) * stride;
        const int wx = t * stride * ps + (n % pw) * stride;
        for (int c = 0; c < C; ++c)
          for (int i = 0; i < kh; ++i)
            for (int j = 0; j < kw; ++j)
              total += AT(map, H, W, c, wy + i, wx + j) != 0.0f;
      }
  return total;
}

int orc_pecr_convert(const float* map, int C, int H, int W, int kh, int kw,
                     int stride, int pw, int ph, int ps, int32_t* count,
                     int64_t* pack_start, float* data, int32_t* index) {
  /* pecr.cpp:83-131 */
  int pW, pH;
  int rc = pecr_geom(C, H, W, kh, kw, stride, pw, ph, ps, &pW, &pH);
  if (rc) return rc;
  int64_t pos = 0;
  for (int b = 0; b < pH; ++b)
    for (int t = 0; t < pW; ++t) {
      const size_t pk = (size_t)b * pW + t;
      pack_start[pk] = pos;
      for (int n = 0; n < pw * ph; ++n) {
        const int wy = b * stride * ps + (n / pw) * stride;
        const int wx = t * stride * ps + (n % pw) * stride;
        int num = 0;
        for (int c = 0; c < C; ++c)
          for (int i = 0; i < kh; ++i)
            for (int j = 0; j < kw; ++j) {
              const float v = AT(map, H, W, c, wy + i, wx + j);
              if (v != 0.0f) {
                data[pos] = v;
                index[pos] = (c * kh + i) * kw + j;
                ++pos;
                ++num;
              }
            }
        count[pk * (pw * ph) + n] = num; /* 0 allowed, no sentinel */
      }
    }
  pack_start[(size_t)pH * pW] = pos;
  return ORC_OK;
}

int orc_pecr_conv_pool(const int32_t* count, const int64_t* pack_start,
                       const float* data, const int32_t* index,
                       const float* kernel, int C, int kh, int kw,
                       int packs_h, int packs_w, int pw, int ph, int mode,
                       float* out, uint64_t* muls, uint64_t* adds) {
  /* pecr.cpp:133-172; format checks as check_pecr :40-55 */
  const int cap = C * kh * kw, wpp = pw * ph;
  for (size_t pk = 0; pk < (size_t)packs_h * packs_w; ++pk) {
    int64_t tot = 0;
    for (int n = 0; n < wpp; ++n) {
      const int cn = count[pk * wpp + n];
      if (cn < 0 || cn > cap) return ORC_FORMAT;
      tot += cn;
    }
    if (pack_start[pk + 1] - pack_start[pk] != tot) return ORC_FORMAT;
    for (int64_t p = pack_start[pk]; p < pack_start[pk + 1]; ++p)
      if (index[p] < 0 || index[p] >= cap) return ORC_FORMAT;
  }
  uint64_t m = 0, a = 0;
  for (size_t pk = 0; pk < (size_t)packs_h * packs_w; ++pk) {
    int64_t p = pack_start[pk];
    float best = 0.0f; /* ReLU folded into the max, :149 */
    float sum = 0.0f;
    for (int n = 0; n < wpp; ++n) {
      const int cn = count[pk * wpp + n];
      float acc = 0.0f;
      for (int q = 0; q < cn; ++q, ++p) {
        const float prod = data[p] * kernel[index[p]];
        acc = acc + prod;
      }
      if (mode == 0) {
        if (acc > best) best = acc;
      } else {
        sum = sum + (acc > 0.0f ? acc : 0.0f);
      }
      m += (uint64_t)cn;
      a += cn > 0 ? (uint64_t)(cn - 1) : 0;
    }
    out[pk] = mode == 0 ? best : sum / (float)wpp;
  }
  if (muls) *muls += m;
  if (adds) *adds += a;
  return ORC_OK;
}

int orc_pecr_conv_pool_batched(const float* x, int N, int C, int H, int W,
                               const float* w, int K, int kh, int kw,
                               int stride, int pw, int ph, int ps, int mode,
                               float* y, uint64_t* muls, uint64_t* adds) {
  /* forward()'s fused branch (pipeline.cpp:249-264): per filter, per pack,
   * p_w*p_h sequential window dots then the pooling fold of :157-167. */
  int pW, pH;
  int rc = pecr_geom(C, H, W, kh, kw, stride, pw, ph, ps, &pW, &pH);
  if (rc) return rc;
  const size_t in_sz = (size_t)C * H * W, f_sz = (size_t)C * kh * kw;
  const int wpp = pw * ph;
  uint64_t m = 0, a = 0;
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < K; ++k) {
      const float* map = x + n * in_sz;
      const float* filt = w + k * f_sz;
      float* out = y + ((size_t)n * K + k) * pH * pW;
      for (int b = 0; b < pH; ++b)
        for (int t = 0; t < pW; ++t) {
          float best = 0.0f, sum = 0.0f;
          for (int q = 0; q < wpp; ++q) {
            const int wy = b * stride * ps + (q / pw) * stride;
            const int wx = t * stride * ps + (q % pw) * stride;
            float acc = 0.0f;
            int cn = 0;
            for (int c = 0; c < C; ++c)
              for (int i = 0; i < kh; ++i)
                for (int j = 0; j < kw; ++j) {
                  const float v = AT(map, H, W, c, wy + i, wx + j);
                  if (v != 0.0f) {
                    const float prod = v * AT(filt, kh, kw, c, i, j);
                    acc = acc + prod;
                    ++cn;
                  }
                }
            if (mode == 0) {
              if (acc > best) best = acc;
            } else {
              sum = sum + (acc > 0.0f ? acc : 0.0f);
            }
            m += (uint64_t)cn;
            a += cn > 0 ? (uint64_t)(cn - 1) : 0;
          }
          out[(size_t)b * pW + t] = mode == 0 ? best : sum / (float)wpp;
        }
    }
  if (muls) *muls += m;
  if (adds) *adds += a;
  return ORC_OK;
}

/* ---- dataset.cpp:249-268, report.cpp:14-30 ------------------------------ */

int orc_window_nnz(const float* map, int C, int H, int W, int kh, int kw,
                   int stride, int32_t* counts) {
  int ow, oh;
  int rc = orc_conv_output_dims(W, H, kw, kh, stride, &ow, &oh);
  if (rc) return rc;
  for (int y = 0; y < oh; ++y)
    for (int x = 0; x < ow; ++x) {
      int nnz = 0;
      for (int c = 0; c < C; ++c)
        for (int i = 0; i < kh; ++i)
          for (int j = 0; j < kw; ++j)
            nnz += AT(map, H, W, c, y * stride + i, x * stride + j) != 0.0f;
      counts[(size_t)y * ow + x] = nnz;
    }
  return ORC_OK;
}

uint64_t orc_checksum(const float* v, int64_t n) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (int64_t i = 0; i < n; ++i) {
    uint32_t bits;
    memcpy(&bits, &v[i], 4);
    for (int s = 0; s < 32; s += 8) {
      h ^= (bits >> s) & 0xffu;
      h *= 0x100000001b3ull;
    }
  }
  return h;
}
