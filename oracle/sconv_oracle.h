/*
 * sconv_oracle.h -- CPU restatement of the reference ECR/PECR hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_1909_09927_b200/)
 * may include, link or call this; only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs use it, and only as the
 * checker.  The product fails loudly when its CUDA library is missing.
 *
 * Parity pinning: every function here is checked (tests/test_oracle.py)
 * against the tests/golden fixtures, which tests/golden/make_golden.py produced by
 * running the UNMODIFIED reference library (oracle/_ref/libsconv_ref.so,
 * built by oracle/Makefile from /root/reference/proj/src), and, when
 * oracle/_ref is present, directly against the reference on seeded inputs.
 *
 * Layouts are flat, channel-major row-major, exactly as FeatureMap/Filter
 * (reference include/sconv/tensor.hpp:12-49):
 *   map     [C][H][W]             filter [C][kh][kw]
 *   ECR     ptr[o_h*o_w]; offsets/f_data/k_data[o_h*o_w*slot]   (ecr.hpp:26-45)
 *   PECR    count[packs_h*packs_w*wpp]; pack_start[packs+1];
 *           data/index[total] concatenated pack-major             (pecr.hpp:35-52)
 *
 * Return codes mirror the reference exception types (errors.hpp:9-26).
 */
#ifndef SCONV_ORACLE_H
#define SCONV_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  ORC_OK = 0,
  ORC_SHAPE = 1,  /* ShapeError  */
  ORC_CONFIG = 2, /* ConfigError */
  ORC_FORMAT = 3  /* FormatError */
};

/* Rng: xoshiro256** seeded via SplitMix64 (dataset.cpp:55-75). */
typedef struct { uint64_t s[4]; } orc_rng;
void orc_rng_seed(orc_rng* r, uint64_t seed);
uint64_t orc_rng_next(orc_rng* r);
double orc_rng_next_unit(orc_rng* r);

/* generate(height, width, channels, sparsity, seed) (dataset.cpp:77-100). */
int orc_generate(int height, int width, int channels, double sparsity,
                 uint64_t seed, float* out);

int orc_conv_output_dims(int in_w, int in_h, int k_w, int k_h, int stride,
                         int* out_w, int* out_h);

int orc_dense_conv(const float* map, int C, int H, int W, const float* filt,
                   int kh, int kw, int stride, float* out, uint64_t* muls,
                   uint64_t* adds);

void orc_relu(const float* in, int64_t n, float* out);
int orc_pool(const float* in, int C, int H, int W, int pw, int ph, int ps,
             int mode, float* out);

/* ECR (ecr.cpp:51-128). */
int orc_ecr_convert(const float* map, int C, int H, int W, const float* filt,
                    int kh, int kw, int stride, int32_t* ptr, int32_t* offsets,
                    float* f_data, float* k_data);
int orc_ecr_spmv_conv(const int32_t* ptr, const float* f_data,
                      const float* k_data, int o_h, int o_w, int slot,
                      float* out, uint64_t* muls, uint64_t* adds);
/* Composition ecr_convert -> ecr_spmv_conv over N images x K filters,
 * output [N][K][o_h][o_w]; arithmetic identical to the two-phase path. */
int orc_ecr_conv_batched(const float* x, int N, int C, int H, int W,
                         const float* w, int K, int kh, int kw, int stride,
                         float* y, uint64_t* muls, uint64_t* adds);

/* PECR (pecr.cpp:62-172). */
int orc_pecr_pack_count(int in_extent, int k_extent, int conv_stride,
                        int pool_extent, int pool_stride, int* packs);
int64_t orc_pecr_total(const float* map, int C, int H, int W, int kh, int kw,
                       int stride, int pw, int ph, int ps);
int orc_pecr_convert(const float* map, int C, int H, int W, int kh, int kw,
                     int stride, int pw, int ph, int ps, int32_t* count,
                     int64_t* pack_start, float* data, int32_t* index);
int orc_pecr_conv_pool(const int32_t* count, const int64_t* pack_start,
                       const float* data, const int32_t* index,
                       const float* kernel, int C, int kh, int kw,
                       int packs_h, int packs_w, int pw, int ph, int mode,
                       float* out, uint64_t* muls, uint64_t* adds);
int orc_pecr_conv_pool_batched(const float* x, int N, int C, int H, int W,
                               const float* w, int K, int kh, int kw,
                               int stride, int pw, int ph, int ps, int mode,
                               float* y, uint64_t* muls, uint64_t* adds);

/* window_nnz_counts (dataset.cpp:249-268). */
int orc_window_nnz(const float* map, int C, int H, int W, int kh, int kw,
                   int stride, int32_t* counts);

/* checksum_hex (report.cpp:14-30): FNV-1a 64 over LE float bytes. */
uint64_t orc_checksum(const float* v, int64_t n);

#ifdef __cplusplus
}
#endif

#endif
