// Does a predicated-off FFMA2 cost FMA-pipe cycles?  (dev micro-benchmark)
// Each warp runs ITER x 16 FFMA2 on independent accumulators, guarded by a
// warp-uniform predicate taken from a kernel argument; time p = 1 vs p = 0.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void ffma2(float& a0, float& a1, float w0, float w1, float v) {
  asm("{\n\t.reg .b64 a, w, v;\n\tmov.b64 a, {%0, %1};\n\tmov.b64 w, {%2, %3};\n\tmov.b64 v, {%4, %4};\n\t"
      "fma.rn.f32x2 a, w, v, a;\n\tmov.b64 {%0, %1}, a;\n\t}"
      : "+f"(a0), "+f"(a1) : "f"(w0), "f"(w1), "f"(v));
}
__global__ void k(float* out, int iters, unsigned p, float v) {
  float a[32];
  for (int i = 0; i < 32; ++i) a[i] = threadIdx.x * 0.001f + i;
  const float w0 = 1.0001f, w1 = 0.9999f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      const unsigned bit = (p >> (i / 2)) & 1u;  // per-block predicate, as the ECR cell test
      if (bit) ffma2(a[i], a[i + 1], w0, w1, v);
    }
  }
  float s = 0;
  for (int i = 0; i < 32; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* out;
  cudaMalloc(&out, 148 * 8 * 1024 * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 20000;
  for (int warps = 8; warps <= 32; warps *= 2) {
    for (unsigned p : {0u, 0xffffu}) {
      k<<<148, warps * 32>>>(out, 100, p, 0.5f);
      cudaEventRecord(a);
      k<<<148, warps * 32>>>(out, iters, p, 0.5f);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double ffma2 = 148.0 * warps * iters * 16;
      int clk;
      cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
      const double cycles = ms * 1e-3 * clk * 1e3;
      printf("warps/SM %2d mask=%#06x: %.3f ms, %.2f SMSP-cycles per FFMA2 per warp-slot (2.0 = pipe-bound)\n",
             warps, p, ms, cycles / (ffma2 / 148 / 4));
    }
  }
  return 0;
}
