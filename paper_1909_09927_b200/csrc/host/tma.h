// tma.h -- tensor-map encoding for the filter staging of the v3/v4 kernels
// (host side; used by the v3 registry, reg_v3.inc).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

namespace sconv_cu {

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
inline EncodeTiledFn encode_tiled() {
  static EncodeTiledFn fn = [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return static_cast<EncodeTiledFn>(nullptr);
    return reinterpret_cast<EncodeTiledFn>(p);
  }();
  return fn;
}

// Tensor map over the transposed filters wt[C][KK][Kp] (fp32), box KT x KK x CC.
// Returns CUDA_SUCCESS, or CUDA_ERROR_NOT_SUPPORTED when the driver entry
// point is missing.
inline CUresult encode_weight_map(const float* wt, int C, int KK, int Kp, int KT, int CC,
                                  CUtensorMap* map) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return CUDA_ERROR_NOT_SUPPORTED;
  const cuuint64_t dims[3] = {cuuint64_t(Kp), cuuint64_t(KK), cuuint64_t(C)};
  const cuuint64_t strides[2] = {cuuint64_t(Kp) * 4, cuuint64_t(KK) * Kp * 4};
  const cuuint32_t box[3] = {cuuint32_t(KT), cuuint32_t(KK), cuuint32_t(CC)};
  const cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(wt), dims, strides, box,
             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

// Tensor map over a conv output y[N][K][OH][OW] (fp32) for TMA stores of
// box_w x box_h x box_k tiles of one image; out-of-range parts of a box are
// clipped by the hardware.  Needs OW % 4 == 0 (16-byte row pitch).
inline CUresult encode_output_map(float* y, int N, int K, int OH, int OW, int box_w, int box_h,
                                  int box_k, CUtensorMap* map) {
  EncodeTiledFn enc = encode_tiled();
  if (!enc) return CUDA_ERROR_NOT_SUPPORTED;
  const cuuint64_t dims[4] = {cuuint64_t(OW), cuuint64_t(OH), cuuint64_t(K), cuuint64_t(N)};
  const cuuint64_t strides[3] = {cuuint64_t(OW) * 4, cuuint64_t(OH) * OW * 4,
                                 cuuint64_t(K) * OH * OW * 4};
  const cuuint32_t box[4] = {cuuint32_t(box_w), cuuint32_t(box_h), cuuint32_t(box_k), 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, y, dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

}  // namespace sconv_cu
