// common.cuh -- small device helpers shared by the sconv sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace sconv_cu {

constexpr unsigned kFull = 0xffffffffu;

// One multiply-accumulate term.  EXACT mode reproduces the reference's x86-64
// arithmetic (`acc += a*b` compiled without FMA: rounded product, rounded
// sum -- src/ecr.cpp:117-120, src/pecr.cpp:152-155).  FAST mode contracts the
// term into a single FFMA.
template <bool FAST>
__device__ __forceinline__ float mac(float acc, float a, float b) {
  if constexpr (FAST) {
    return __fmaf_rn(a, b, acc);
  } else {
    return __fadd_rn(acc, __fmul_rn(a, b));
  }
}

// Two FAST terms in one packed FFMA2 (sm_100a `fma.rn.f32x2`, the scalar
// operand broadcast to both halves): {a0,a1} += {w0,w1} * v.  Same rounding
// as two FFMAs; one issue slot instead of two, which leaves room for the
// zero-skip branches of the ECR main loop.
__device__ __forceinline__ void ffma2(float& a0, float& a1, float w0, float w1, float v) {
  asm("{\n\t.reg .b64 a, w, v;\n\t"
      "mov.b64 a, {%0, %1};\n\t"
      "mov.b64 w, {%2, %3};\n\t"
      "mov.b64 v, {%4, %4};\n\t"
      "fma.rn.f32x2 a, w, v, a;\n\t"
      "mov.b64 {%0, %1}, a;\n\t}"
      : "+f"(a0), "+f"(a1)
      : "f"(w0), "f"(w1), "f"(v));
}

// Two EXACT terms, {a0,a1} += {w0,w1}*v as a rounded product then a rounded
// sum per half -- the reference's `acc += a*b` without contraction
// (src/ecr.cpp:117-120) -- in three issue slots instead of four: one packed
// FMUL2 and two scalar FADDs.  (A packed mul.rn.f32x2 followed by a packed
// add.rn.f32x2 is NOT used: ptxas 12.9 fuses that pair into an FFMA2 even
// with -fmad=false, which would round once instead of twice.)
//
// exact2_mul: that FMUL2 + two FADDs.  exact2: two issue slots -- the products
// by a packed FFMA with a -0 addend (w*v + -0 rounds exactly like w*v, +0
// products included), then one packed FADD; the -0 is read from constant
// memory, whose contents ptxas cannot assume, so it cannot turn the FFMA2 into
// an FMUL2 and fuse it with the add.  The branchy ECR bodies are issue-bound
// and take exact2 (EXACT conv1_2 -12%, conv4_2 -7%); the dense small-C kernel
// is FMA-pipe-bound, where FFMA2 + FADD2 cost more pipe cycles than FMUL2 +
// two FADDs (conv1_1 +24%), and keeps exact2_mul.
__device__ __forceinline__ void exact2_mul(float& a0, float& a1, float w0, float w1, float v) {
  asm("{\n\t.reg .b64 w, v, t;\n\t.reg .f32 t0, t1;\n\t"
      "mov.b64 w, {%2, %3};\n\t"
      "mov.b64 v, {%4, %4};\n\t"
      "mul.rn.f32x2 t, w, v;\n\t"
      "mov.b64 {t0, t1}, t;\n\t"
      "add.rn.f32 %0, %0, t0;\n\t"
      "add.rn.f32 %1, %1, t1;\n\t}"
      : "+f"(a0), "+f"(a1)
      : "f"(w0), "f"(w1), "f"(v));
}
#ifndef SCONV_EXACT_FMA
#define SCONV_EXACT_FMA 1
#endif
__constant__ float c_sconv_negzero = -0.0f;
__device__ __forceinline__ void exact2(float& a0, float& a1, float w0, float w1, float v) {
#if SCONV_EXACT_FMA
  asm("{\n\t.reg .b64 w, v, z, t, a;\n\t"
      "mov.b64 w, {%2, %3};\n\t"
      "mov.b64 v, {%4, %4};\n\t"
      "mov.b64 z, {%5, %5};\n\t"
      "fma.rn.f32x2 t, w, v, z;\n\t"
      "mov.b64 a, {%0, %1};\n\t"
      "add.rn.f32x2 a, a, t;\n\t"
      "mov.b64 {%0, %1}, a;\n\t}"
      : "+f"(a0), "+f"(a1)
      : "f"(w0), "f"(w1), "f"(v), "f"(c_sconv_negzero));
#else
  exact2_mul(a0, a1, w0, w1, v);
#endif
}

// Keeps ptxas from if-converting a zero-skip block into predicated FMAs
// (which would issue -- and occupy the FMA pipe -- for every zero too).  It
// emits one PMTRIG, which touches no registers; ptxas will not predicate a
// block that holds it, so the block stays behind a uniform BRA.U.
#define SCONV_KEEP_BRANCH() asm volatile("pmevent 0;")

// Pooling fold of pecr_conv_pool (src/pecr.cpp:147-167).
struct PoolFold {
  float best = 0.0f;  // max mode: running max starts at +0.0 -> ReLU folded
  float sum = 0.0f;   // mean mode: sum of max(acc, 0) in window raster order
  __device__ __forceinline__ void add(float acc, int mode) {
    if (mode == 0) {
      if (acc > best) best = acc;
    } else {
      sum = __fadd_rn(sum, acc > 0.0f ? acc : 0.0f);
    }
  }
  __device__ __forceinline__ float result(int mode, int windows) const {
    return mode == 0 ? best : __fdiv_rn(sum, static_cast<float>(windows));
  }
};

// Activation::kRelu applied in an ECR epilogue (relu(), src/tensor.cpp:89-95:
// v > 0 ? v : +0, so -0 and NaN become +0).  For P == 0 launches the `mode`
// argument (the pool mode of PECR launches) carries this flag.
__device__ __forceinline__ float relu_f(float v) { return v > 0.0f ? v : 0.0f; }

template <int A, int B, int R>
__device__ __forceinline__ void relu_tile(float (&acc)[A][B][R]) {
#pragma unroll
  for (int i = 0; i < A; ++i)
#pragma unroll
    for (int j = 0; j < B; ++j)
#pragma unroll
      for (int r = 0; r < R; ++r) acc[i][j][r] = relu_f(acc[i][j][r]);
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ void cp_async4(float* smem, const float* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int bytes = valid ? 4 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes)
               : "memory");
}

// 8-byte copy, src_bytes in {0, 4, 8}: the rest of the 8 bytes is zero-filled.
__device__ __forceinline__ void cp_async8(float* smem, const float* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes)
               : "memory");
}

// The same with the shared-memory destination as a byte address (the
// producers keep stage-relative offsets and add immediates).
__device__ __forceinline__ void cp_async4_s(unsigned smem, const float* gmem, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(smem), "l"(gmem), "r"(valid ? 4 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async8_s(unsigned smem, const float* gmem, int src_bytes) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem), "l"(gmem), "r"(src_bytes)
               : "memory");
}

__device__ __forceinline__ void cp_async16(float* smem, const float* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int bytes = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }

template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Deterministic integer reduction of a per-thread value into *dst
// (block reduce, one 64-bit atomic per block; integer sums are order-free).
__device__ __forceinline__ void block_add_u64(unsigned long long v, unsigned long long* dst) {
  __shared__ unsigned long long part[32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(kFull, v, o);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) part[w] = v;
  __syncthreads();
  if (w == 0) {
    const int nw = (blockDim.x + 31) >> 5;
    v = (threadIdx.x < static_cast<unsigned>(nw)) ? part[threadIdx.x] : 0ull;
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(kFull, v, o);
    if (threadIdx.x == 0 && v) atomicAdd(dst, v);
  }
  __syncthreads();
}

}  // namespace sconv_cu
