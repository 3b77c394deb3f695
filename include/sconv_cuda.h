/*
 * sconv_cuda.h -- C ABI of the B200 (sm_100a) ECR / PECR sparse-convolution
 * library (libsconv_cuda.so).
 *
 * This is the thin layer the reference's C++ host API calls into.  Plain
 * pointers and sizes only; no C++ or torch types cross it.  Each entry point
 * names the reference interface it replaces (paths relative to
 * /root/reference/proj).  Layouts follow FeatureMap/Filter
 * (include/sconv/tensor.hpp:12-49): channel-major then row-major fp32.
 *
 *   x  [N][C][H][W]   input maps (valid convolution, no padding)
 *   w  [K][C][kh][kw] filters (one Filter per output channel, as in
 *                     LayerSpec::filters, include/sconv/pipeline.hpp:17-23)
 *   y  [N][K][oh][ow] ECR output, or [N][K][packs_h][packs_w] PECR output
 *
 * Error model: every function returns an sconv_status.  The C++ drop-in
 * (paper_1909_09927_b200/csrc/dropin/) maps them onto the reference
 * exception types of include/sconv/errors.hpp:9-26 and exec.hpp:43-51.
 * sconv_cu_last_error() holds the message of the last failure on a context.
 *
 * Threading: a context owns one CUDA stream on one device and is not safe to
 * share between host threads without external synchronisation; any number of
 * contexts may run concurrently (the reference's "pure and reentrant"
 * contract).
 */
#ifndef SCONV_CUDA_H
#define SCONV_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SCONV_CUDA_ABI_VERSION 1

typedef enum {
  SCONV_OK = 0,
  SCONV_ERR_SHAPE = 1,    /* sconv::ShapeError   (errors.hpp:9-12)  */
  SCONV_ERR_CONFIG = 2,   /* sconv::ConfigError  (errors.hpp:14-17) */
  SCONV_ERR_FORMAT = 3,   /* sconv::FormatError  (errors.hpp:19-22) */
  SCONV_ERR_IO = 4,       /* sconv::IoError      (errors.hpp:24-26) */
  SCONV_ERR_DISPATCH = 5, /* sconv::DispatchError (exec.hpp:43-51)  */
  SCONV_ERR_CUDA = 6,     /* device / runtime failure -> std::runtime_error */
  SCONV_ERR_ARG = 7       /* null pointer or bad handle -> std::invalid_argument */
} sconv_status;

/* ---- flags ------------------------------------------------------------ */
/* Arithmetic.  EXACT (default) accumulates every output in the reference's
 * c -> i -> j order with separately rounded multiply and add: bit-identical
 * to ecr_spmv_conv / pecr_conv_pool.  FAST contracts each term into one FFMA
 * (same order); results stay within |a-b| <= 1e-5 + 1e-5*|b| of the
 * reference. */
#define SCONV_F_EXACT 0u
#define SCONV_F_FAST (1u << 0)
/* Every tensor pointer is a device pointer on the context's device (no
 * host<->device copies).  Without it all pointers are host pointers.  Device
 * maps x and outputs y must be 16-byte aligned (SCONV_ERR_ARG otherwise: the
 * kernels move 8- and 16-byte vectors). */
#define SCONV_F_DEVICE (1u << 1)
/* Return right after enqueueing (no synchronisation); counters must be NULL.
 * With SCONV_F_DEVICE the work is ordered on the context stream.  With host
 * pointers the call owns one of 6 rotating workspaces and its own
 * H2D / compute / D2H ring, so consecutive calls overlap their transfers;
 * the inputs must stay unchanged and the outputs unread until
 * sconv_cu_synchronize(ctx) (use pinned memory for the copies to overlap). */
#define SCONV_F_ASYNC (1u << 2)
/* Force the generic (one thread per output) kernels; testing only. */
#define SCONV_F_GENERIC (1u << 3)
/* sconv_cu_forward only, with SCONV_F_DEVICE and no counters: capture the
 * network's launches in a CUDA graph on the first call and replay it while
 * the arguments (pointers, shapes, layers, flags) stay the same. */
#define SCONV_F_GRAPH (1u << 4)
/* The caller promises that the filter values at this filters pointer (same
 * pointer, same K x C x kh x kw) do not change between calls, as for the
 * layer weights of an inference network: the context keeps the kernels'
 * re-laid-out copy ([C][kh*kw][Kp], plus the filters' device copy for host
 * pointers) and reuses it instead of copying / transposing every call.
 * sconv_cu_release_filters drops the cached copies. */
#define SCONV_F_CACHE_FILTERS (1u << 5)
/* Force one tiled kernel configuration (testing / tuning only): 1..6 = v2
 * TiledCfg1..6 (ignored when the shape is not a 3x3 stride-1 tile);
 * 'A'..'L', 'N'..'Q' = v3 WsA..WsQ, 'R'..'T' = the general-pool WsR..WsT
 * (PECR with a pool other than 2x2/2), 'U' / 'V' = the ECR-only 2x7 / 7x2
 * tiles, 'W' = 6x6 tiles in one 15-consumer CTA per SM, 'Y' = the 1x1
 * dense ordered GEMM (kernels/pointwise.cuh) (csrc/reg_v3.inc;
 * SCONV_ERR_ARG when the config does not fit the
 * window / stride / pool); 'M' = the small-C kernel.
 * 0 (default) lets the launch layer pick. */
#define SCONV_F_KERNEL(id) (((unsigned)(id) & 0xffu) << 8)

typedef enum { SCONV_POOL_MAX = 0, SCONV_POOL_MEAN = 1 } sconv_pool_mode;

typedef struct sconv_cu_ctx sconv_cu_ctx;

/* ---- context ------------------------------------------------------------ */
const char* sconv_cu_version(void);
int sconv_cu_device_count(int* count);
int sconv_cu_ctx_create(int device, sconv_cu_ctx** out);
int sconv_cu_ctx_destroy(sconv_cu_ctx* ctx);
/* Run on an external cudaStream_t (e.g. torch's current stream).  The value
 * is used as is: NULL is the legacy default stream.  Both calls drain the
 * previous stream first (the context workspace is stream-ordered). */
int sconv_cu_ctx_set_stream(sconv_cu_ctx* ctx, void* stream);
/* Go back to the context's own non-blocking stream. */
int sconv_cu_ctx_use_own_stream(sconv_cu_ctx* ctx);
void* sconv_cu_ctx_stream(sconv_cu_ctx* ctx);
int sconv_cu_ctx_device(sconv_cu_ctx* ctx);
int sconv_cu_synchronize(sconv_cu_ctx* ctx);
const char* sconv_cu_last_error(const sconv_cu_ctx* ctx);
/* Number of kernels this context has launched (evidence counter). */
uint64_t sconv_cu_launch_count(const sconv_cu_ctx* ctx);
/* Drop every filter copy kept for SCONV_F_CACHE_FILTERS calls (waits for the
 * context's work first). */
int sconv_cu_release_filters(sconv_cu_ctx* ctx);

/* ---- geometry (host only) ---------------------------------------------- */
/* conv_output_dims, src/tensor.cpp:44-55. */
int sconv_conv_output_dims(int in_w, int in_h, int k_w, int k_h, int stride,
                           int* out_w, int* out_h);
/* pecr_pack_count (Eq. 3), src/pecr.cpp:62-81. */
int sconv_pecr_pack_count(int in_extent, int k_extent, int conv_stride,
                          int pool_extent, int pool_stride, int* packs);

/* The CUDA launch chosen for a layer (replaces the simulated grid of
 * plan(), src/exec.cpp:8-36, for reporting).  pool_w == 0 -> ECR. */
typedef struct {
  int kernel;          /* 0 generic, 1 tiled 3x3, ... */
  int grid_x, grid_y, grid_z;
  int block_threads;
  int smem_bytes;
  int tile_h, tile_w, tile_k; /* outputs per CTA */
} sconv_launch_plan;
int sconv_cu_plan(int n, int c, int h, int w, int k, int kh, int kw, int stride,
                  int pool_w, int pool_h, int pool_stride, unsigned flags,
                  sconv_launch_plan* out);

/* ---- hot path: fused, batched ------------------------------------------ */
/* ECR convolution of N maps by K filters.  Replaces the per-filter
 * ecr_convert -> ecr_spmv_conv pair (src/ecr.cpp:51-128) as driven by
 * multichannel_conv (src/pipeline.cpp:191-210): the window compaction is done
 * on chip and never written to HBM.  Windows with no nonzero produce +0.0
 * (ptr == -1 law, ecr.cpp:112-115).  muls/adds (optional, accumulated with
 * +=) equal the sum over all (image, filter) calls of OpCount from
 * ecr_spmv_conv: per window nnz and max(nnz-1, 0). */
int sconv_cu_ecr_conv(sconv_cu_ctx* ctx, const float* x, int n, int c, int h,
                      int w, const float* filters, int k, int kh, int kw,
                      int stride, float* y, uint64_t* muls, uint64_t* adds,
                      unsigned flags);

/* PECR fused convolution + ReLU + pooling.  Replaces pecr_convert ->
 * pecr_conv_pool (src/pecr.cpp:83-172) as driven by forward's fused branch
 * (src/pipeline.cpp:249-264).  Max mode starts the running max at +0.0
 * (ReLU folded, pecr.cpp:149,157-158); mean mode sums max(acc, 0) over the
 * p_w*p_h windows in raster order then divides (pecr.cpp:159-167).  The
 * pre-pool convolution output never reaches HBM.  ConfigError unless Eq. 3
 * tiles both axes exactly. */
int sconv_cu_pecr_conv_pool(sconv_cu_ctx* ctx, const float* x, int n, int c,
                            int h, int w, const float* filters, int k, int kh,
                            int kw, int stride, int pool_w, int pool_h,
                            int pool_stride, int mode, float* y,
                            uint64_t* muls, uint64_t* adds, unsigned flags);

/* ---- on-device multi-layer forward ------------------- */
/* forward(net, input, method) of src/pipeline.cpp:212-301 for N images, with
 * every activation resident in HBM: one ingest of the input and all filters,
 * one egress of the output (plus any per-layer outputs requested).  Layer l:
 *   PECR method, pooled layer with ReLU -> fused conv+ReLU+pool
 *     (sconv_cu_pecr_conv_pool; the pre-pool output never reaches HBM);
 *   otherwise -> ECR conv, ReLU (fused into the conv epilogue unless
 *     conv_outputs[l] asks for the pre-activation map), then pool() if the
 *     layer pools; pecr_fallback[l] = 1 for these layers under PECR
 *     (ForwardResult::pecr_fallback_layers).
 * Validation follows NetworkSpec::validate (pipeline.cpp:154-189); a layer
 * that then fails (e.g. Eq. 3 not integral under PECR) is a ConfigError
 * "layer l failed: ..." (pipeline.cpp:293-297).  The dense method is the CPU
 * reference's and is refused (ConfigError).  With SCONV_F_DEVICE every
 * pointer (x, filters, y, layer/conv outputs) is a device pointer.
 * layer_outputs / conv_outputs: NULL or nlayers pointers, each NULL or a
 * buffer for [N][k][..] of that layer (conv_outputs of fused layers are not
 * written: the reference stores a 1x1x1 placeholder there). */
#define SCONV_METHOD_ECR 1
#define SCONV_METHOD_PECR 2
typedef struct {
  const float* filters; /* [k][c][kh][kw], c = the previous layer's k */
  int k, kh, kw, stride;
  int relu;             /* Activation::kRelu */
  int pool_w, pool_h, pool_stride, pool_mode; /* pool_w == 0: LayerKind::kConv */
} sconv_layer;
int sconv_cu_forward_dims(const sconv_layer* layers, int nlayers, int c, int h,
                          int w, int* out_c, int* out_h, int* out_w);
int sconv_cu_forward(sconv_cu_ctx* ctx, const float* x, int n, int c, int h,
                     int w, const sconv_layer* layers, int nlayers, int method,
                     float* y, float* const* layer_outputs,
                     float* const* conv_outputs, uint64_t* muls,
                     uint64_t* adds, int32_t* pecr_fallback, unsigned flags);

/* ---- sparsity profiling (src/dataset.cpp:249-286) ----------------------
 * window_nnz_counts for N maps: counts[N][oh][ow] (NULL: not written) = the
 * nonzeros of every conv window over all channels; raw[N] / extended[N]
 * (NULL: not written) = sparsity_profile's zero fraction of the map and of
 * its im2col extension.  Integer counts, exact ratios. */
int sconv_cu_window_nnz(sconv_cu_ctx* ctx, const float* x, int n, int c, int h,
                        int w, int kh, int kw, int stride, int32_t* counts,
                        double* raw, double* extended, unsigned flags);

/* ---- feature-map files (src/dataset.cpp:115-247) ------------------------
 * FMAP ("FMAP", u32le version 1, C, H, W, then LE fp32 values) or CSV by the
 * path's extension, with the reference's validation: IoError when the file
 * cannot be opened, FormatError on a bad magic / version / header / dims /
 * truncated payload / unparsable value.  Host only (no CUDA). */
const char* sconv_io_last_error(void);
int sconv_map_file_dims(const char* path, int* c, int* h, int* w);
/* capacity: floats available at out (ArgError when the map is larger). */
int sconv_load_map(const char* path, float* out, int64_t capacity, int* c,
                   int* h, int* w);
int sconv_save_map(const char* path, const float* values, int c, int h, int w);
/* N files of identical dims into out[N][C][H][W] (e.g. a pinned buffer for
 * the batched entries), on `threads` host threads (<= 0: all cores); the
 * lowest failing file's error is reported, ShapeError when dims differ. */
int sconv_load_maps(const char* const* paths, int n, float* out, int c, int h,
                    int w, int threads);

/* ---- formats: the reference's two-phase API (one map, one filter) ------- */
/* ecr_convert (src/ecr.cpp:51-97) by warp-ballot compaction.  Writes the
 * fixed-slot EcrMap arrays of include/sconv/ecr.hpp:35-45, flattened
 * [oh][ow][slot] (slot = c*kh*kw): nonzeros in c->i->j order, their paired
 * weights and offsets, filler 0.0 / 0.0 / -1, and ptr[oh][ow] = nnz or -1. */
int sconv_cu_ecr_convert(sconv_cu_ctx* ctx, const float* x, int c, int h,
                         int w, const float* filter, int kh, int kw, int stride,
                         int32_t* ptr, int32_t* offsets, float* f_data,
                         float* k_data, unsigned flags);

/* ecr_spmv_conv (src/ecr.cpp:99-128) over an EcrMap: FormatError when a ptr
 * lies outside [-1, slot] (check_ecr, ecr.cpp:22-42). */
int sconv_cu_ecr_spmv(sconv_cu_ctx* ctx, const int32_t* ptr,
                      const float* f_data, const float* k_data, int oh, int ow,
                      int slot, float* y, uint64_t* muls, uint64_t* adds,
                      unsigned flags);

/* pecr_convert (src/pecr.cpp:83-131), phase 1: per pack and window nonzero
 * counts count[packs_h][packs_w][pool_w*pool_h] and the exclusive prefix
 * pack_start[packs_h*packs_w + 1]; *total = entries of the whole map. */
int sconv_cu_pecr_count(sconv_cu_ctx* ctx, const float* x, int c, int h, int w,
                        int kh, int kw, int stride, int pool_w, int pool_h,
                        int pool_stride, int32_t* count, int64_t* pack_start,
                        int64_t* total, unsigned flags);
/* phase 2: data/index of every pack, concatenated pack-major
 * (PecrPoolPack::data / index, include/sconv/pecr.hpp:39-43). */
int sconv_cu_pecr_fill(sconv_cu_ctx* ctx, const float* x, int c, int h, int w,
                       int kh, int kw, int stride, int pool_w, int pool_h,
                       int pool_stride, const int64_t* pack_start, int64_t total,
                       float* data, int32_t* index, unsigned flags);

/* pecr_conv_pool (src/pecr.cpp:133-172) over a PecrMap; FormatError on the
 * check_pecr violations of pecr.cpp:24-58 (count range, data/index length,
 * index range). */
int sconv_cu_pecr_pool(sconv_cu_ctx* ctx, const int32_t* count,
                       const int64_t* pack_start, const float* data,
                       const int32_t* index, int64_t total,
                       const float* kernel, int c, int kh, int kw, int packs_h,
                       int packs_w, int pool_w, int pool_h, int mode, float* y,
                       uint64_t* muls, uint64_t* adds, unsigned flags);

/* ---- multi-GPU partition (replaces dispatch's worker partition,
 *      include/sconv/exec.hpp:89-107) --------------------------------------
 * Contiguous shard of the (image, filter) grid owned by `rank` of `world`:
 * images are split when n >= world, otherwise output channels.  Every output
 * is produced by exactly one rank with the same per-output order, so results
 * are bit-identical for any world size. */
int sconv_shard(int n, int k, int world, int rank, int* n_begin, int* n_end,
                int* k_begin, int* k_end);

/* One host thread driving several devices (dispatch's fork/join over GPUs):
 * shards by sconv_shard, runs every context's stream concurrently, joins.
 * Host pointers only. */
int sconv_cu_ecr_conv_multi(sconv_cu_ctx** ctxs, int nctx, const float* x,
                            int n, int c, int h, int w, const float* filters,
                            int k, int kh, int kw, int stride, float* y,
                            uint64_t* muls, uint64_t* adds, unsigned flags);
int sconv_cu_pecr_conv_pool_multi(sconv_cu_ctx** ctxs, int nctx,
                                  const float* x, int n, int c, int h, int w,
                                  const float* filters, int k, int kh, int kw,
                                  int stride, int pool_w, int pool_h,
                                  int pool_stride, int mode, float* y,
                                  uint64_t* muls, uint64_t* adds,
                                  unsigned flags);

/* ---- compressed ingest ---------------------------------------------------
 * A batch of n maps [C][H][W] can cross PCIe as its nonzero bitmap plus the
 * packed nonzeros instead of dense fp32 (the transfer saving the paper
 * credits its compressed formats with); the GPU expands it in
 * HBM right before the convolution.  Per image, E = C*H*W elements:
 *   bits   [n][words]       words = ceil(E / 32); bit e % 32 of word e / 32
 *                           set iff element e is nonzero (v != 0.0f: -0 is a
 *                           zero, as in ecr_convert, src/ecr.cpp:84)
 *   base   [n][blocks + 1]  blocks = ceil(words / 32) (1024 elements each):
 *                           offset in `values` of the block's first nonzero;
 *                           base[i][blocks] = one past image i's last one
 *   values [nnz]            every image's nonzeros in element order
 * Offsets are absolute, so image i's nonzeros start at base[i][0].  With host
 * pointers the calls copy exactly these bytes; with SCONV_F_DEVICE they read
 * them from device memory. */
int sconv_packed_dims(int c, int h, int w, int64_t* words, int64_t* blocks);
/* Pack dense maps (host, `threads` threads, 0 = all cores).  With bits,
 * base and values all NULL only *nnz is computed (size query); otherwise
 * values must hold `capacity` >= nnz floats. */
int sconv_pack_maps(const float* x, int n, int c, int h, int w, uint32_t* bits,
                    int64_t* base, float* values, int64_t capacity,
                    int64_t* nnz, int threads);
/* sconv_cu_ecr_conv / sconv_cu_pecr_conv_pool on a packed batch; outputs,
 * flags and results are those of the dense entries (bit-identical). */
int sconv_cu_ecr_conv_packed(sconv_cu_ctx* ctx, const uint32_t* bits,
                             const int64_t* base, const float* values, int n,
                             int c, int h, int w, const float* filters, int k,
                             int kh, int kw, int stride, float* y,
                             uint64_t* muls, uint64_t* adds, unsigned flags);
int sconv_cu_pecr_conv_pool_packed(sconv_cu_ctx* ctx, const uint32_t* bits,
                                   const int64_t* base, const float* values,
                                   int n, int c, int h, int w,
                                   const float* filters, int k, int kh, int kw,
                                   int stride, int pool_w, int pool_h,
                                   int pool_stride, int mode, float* y,
                                   uint64_t* muls, uint64_t* adds,
                                   unsigned flags);
/* Expand a packed batch into dense x [n][C][H][W] (device pointers only). */
int sconv_cu_unpack_maps(sconv_cu_ctx* ctx, const uint32_t* bits,
                         const int64_t* base, const float* values, int n, int c,
                         int h, int w, float* x, unsigned flags);

/* ---- synthetic inputs (host) ------------------------------------------- */
/* Bit-identical to sconv::generate (src/dataset.cpp:77-100): xoshiro256**
 * seeded by SplitMix64, floor(s*N) zeros at Fisher-Yates positions, nonzeros
 * in (0,1].  The batch form fills maps[i] = generate(h, w, c, s, seeds[i])
 * with up to `threads` host threads (0 = all cores). */
int sconv_generate(int height, int width, int channels, double sparsity,
                   uint64_t seed, float* out);
int sconv_generate_batch(int count, int height, int width, int channels,
                         double sparsity, const uint64_t* seeds, float* out,
                         int threads);
/* checksum_hex (src/report.cpp:14-30) as an integer: FNV-1a 64. */
uint64_t sconv_checksum(const float* values, int64_t n);

#ifdef __cplusplus
}
#endif

#endif /* SCONV_CUDA_H */
