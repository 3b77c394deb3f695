// FFMA issue-rate microbenchmark (dev tool): per-SM FFMA/clk for
// (a) acc = v*w + acc with v shared (reuse), w and acc distinct registers,
// (b) the same with immediate-free 3 distinct registers per FFMA.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, int iters, float seed) {
  float acc[32], w[16];
  for (int i = 0; i < 32; ++i) acc[i] = seed * i;
  for (int i = 0; i < 16; ++i) w[i] = seed + i * 0.5f + threadIdx.x;
  float v = seed * threadIdx.x;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      if (MODE == 0) acc[i] = fmaf(v, w[i & 15], acc[i]);
      else acc[i] = fmaf(w[(i + 3) & 15], w[i & 15], acc[i]);
    }
    v = v * 1.0000001f;
  }
  float s = 0;
  for (int i = 0; i < 32; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* d; cudaMalloc(&d, 148 * 8 * 1024 * 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (int mode = 0; mode < 2; ++mode)
    for (int warps : {4, 8, 16, 32}) {
      const int iters = 20000;
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      auto run = [&] { if (mode == 0) k<0><<<sms * 2, warps * 16>>>(d, iters, 1.0f); else k<1><<<sms * 2, warps * 16>>>(d, iters, 1.0f); };
      run(); cudaDeviceSynchronize();
      cudaEventRecord(a); run(); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double fmas = double(sms) * 2 * warps * 16 * iters * 32.0;
      printf("mode %d warps/SM %2d: %.1f TFLOP/s (%.1f%% of 148*128*2*%.0fMHz)\n", mode, warps,
             2 * fmas / ms / 1e9, 100 * fmas / ms / 1e-3 / (sms * 128.0 * clk * 1e3), clk / 1e3);
    }
}
