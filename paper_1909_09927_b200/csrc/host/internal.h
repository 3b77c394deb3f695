// internal.h -- declarations shared by the translation units of
// libsconv_cuda.so (not part of the C ABI): the context object, the error
// helpers, and the v2 / v3 kernel registries (reg_v2.cu, reg_v3_*.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "kernels/ecr_tiled.cuh"
#include "kernels/ecr_ws.cuh"
#include "sconv_cuda.h"

// A filter slab kept for SCONV_F_CACHE_FILTERS calls: keyed by the caller's
// pointer and shape; `dev` is the device copy (host-pointer calls) and `wt`
// the kernels' [C][kh*kw][Kp] re-layout.
struct sconv_filter_entry {
  const float* src;
  bool host;
  int k, c, kk, kp;
  float* dev;
  float* wt;
};
// Encoded TMA descriptors of the weight slabs (reg_v3.inc), keyed by address
// and box: encoding is pure host work, repeated otherwise on every launch.
struct sconv_tmap_entry {
  const float* wt;
  int c, kk, kp, kt, cc;
  CUtensorMap map;
};

struct sconv_cu_ctx {
  int device = 0;
  // Stream-ordered allocations of this context (async host workspaces) come
  // from its own pool, so raising the pool's release threshold does not
  // change the device's default pool for the host application.
  cudaMemPool_t pool = nullptr;
  // Bumped whenever a workspace the captured forward graph may point into
  // (ws, hws, fwd) is reallocated: the graph is re-captured instead of
  // replaying stale addresses.
  uint64_t mem_gen = 0;
  uint64_t fwd_gen = 0;
  std::vector<sconv_filter_entry> fcache;
  std::vector<sconv_tmap_entry> tmaps;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  std::string err;
  uint64_t launches = 0;
  char* ws = nullptr;
  size_t ws_cap = 0;
  int num_sms = 148;
  int smem_optin = 0;
  // Workspaces of asynchronous host-pointer calls (SCONV_F_ASYNC without
  // SCONV_F_DEVICE): a call in flight owns one of these until its last D2H
  // (ev_hws) -- the rotation lets the H2D of the next call overlap the
  // compute / D2H of the previous ones.
  static constexpr int kHostArenas = 16;  // capacity; hws_n are used
  int hws_n = 6;
  size_t hws_max = 0;  // largest host workspace so far: a growing one jumps to it
  char* hws[kHostArenas] = {};
  size_t hws_cap[kHostArenas] = {};
  cudaEvent_t ev_hws[kHostArenas] = {};
  int hws_next = 0;
  // host-pointer pipeline: copy streams and per-buffer events (fused_conv)
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t ev_in[3] = {}, ev_comp[3] = {}, ev_out[3] = {};
  cudaEvent_t ev_done = nullptr;
  char* fwd = nullptr;              // sconv_cu_forward: resident activations + filters
  size_t fwd_cap = 0;
  cudaGraphExec_t fwd_graph = nullptr;  // SCONV_F_GRAPH: the captured forward
  std::string fwd_key;                  // ... and the arguments it was captured for
  cudaEvent_t ev_graph = nullptr;
  // Row-prefetch gates of ecr_ws_kernel launches (ws_density_gate_kernel
  // writes one, the two variants read it), taken round robin: a slot is
  // reused only kGates launches later on the context's stream.
  static constexpr int kGates = 64;
  int* gate = nullptr;
  unsigned gate_next = 0;
};

namespace sconv_cu {
namespace host {

int fail(sconv_cu_ctx* ctx, int code, const char* fmt, ...);
int finish_launch(sconv_cu_ctx* ctx, const char* what);
unsigned grid_for(size_t work, int threads, int num_sms);

#define CK(expr)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(ctx, SCONV_ERR_CUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                  __FILE__, __LINE__);                                                    \
  } while (0)

#define TRY(expr)                 \
  do {                            \
    const int rc_ = (expr);       \
    if (rc_ != SCONV_OK) return rc_; \
  } while (0)

// v2 tiled registry (reg_v2.cu): config id for a shape (0 = generic), launch, plan.
constexpr int kNumCfgs = 7;
int pick_tiled(int K, int kh, int kw, int S, int P);
int launch_tiled(sconv_cu_ctx* ctx, bool fast, int which, int P, const TiledArgs& a, int N);
void plan_for(sconv_launch_plan* p, int which, int N, int K, int OH, int OW);

// v3 warp-specialised registry (reg_v3.cu / reg_v3_exact.cu / reg_v3_fast.cu).
int pick_ws(int K, int C, int OW, int kh, int kw, int S, int P, long tiles4 = 1L << 40,
            long tiles2 = 1L << 40);
bool ws_applies(int id, int K, int kh, int kw, int S, int P);  // forced-config shape check
int launch_ws_fast(sconv_cu_ctx* ctx, int which, int P, const WsArgs& a);
int launch_ws_exact(sconv_cu_ctx* ctx, int which, int P, const WsArgs& a);
void plan_ws(sconv_launch_plan* p, int which, int N, int K, int OH, int OW, int pw = 0, int ph = 0,
             int ps = 1);
int pick_ws_pool(int K, int kh, int kw, int S, int pw, int ph);  // general-pool config, 0 = none

}  // namespace host
}  // namespace sconv_cu
