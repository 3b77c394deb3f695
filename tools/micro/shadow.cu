// Dev microbenchmark: which instructions hide in the second cycle of an
// FFMA2?  Each step = 4 FFMA2 + X, X in {nothing, 1 uniform op, 2 uniform
// ops, 1 not-taken uniform branch, 1 LDS (uniform address)}.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void fma2(float& a0, float& a1, float w0, float w1, float v) {
  asm volatile("{\n\t.reg .b64 a, w, v;\n\tmov.b64 a, {%0, %1};\n\tmov.b64 w, {%2, %3};\n\t"
      "mov.b64 v, {%4, %4};\n\tfma.rn.f32x2 a, w, v, a;\n\tmov.b64 {%0, %1}, a;\n\t}"
      : "+f"(a0), "+f"(a1) : "f"(w0), "f"(w1), "f"(v));
}

template <int MODE>
__global__ void __launch_bounds__(128) k(float* out, const unsigned* pats, int iters, float seed) {
  __shared__ float sv[64];
  if (threadIdx.x < 64) sv[threadIdx.x] = seed * (threadIdx.x + 1);
  __syncthreads();
  float acc[32], w[16];
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = seed * i;
#pragma unroll
  for (int i = 0; i < 16; ++i) w[i] = seed + i * 0.5f + threadIdx.x;
  const int lane = threadIdx.x & 31;
  float v = seed * lane;
  unsigned u = __ballot_sync(0xffffffffu, (pats[0] >> lane) & 1u);
  unsigned u2 = u * 3u;
  float sink = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int s = 0; s < 16; ++s) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int a = (8 * s + 2 * q) & 31;
        fma2(acc[a], acc[a + 1], w[(2 * q + s) & 15], w[(2 * q + 1 + s) & 15], v);
      }
      if (MODE == 1 || MODE == 2) u = (u >> 1) ^ (u2 + s);   // uniform ALU
      if (MODE == 2) u2 = (u2 << 3) + u;
      if (MODE == 3) { if (u == 0xdeadbeefu + s) asm volatile("pmevent 1;"); }
      if (MODE == 4) sink += sv[(u + s) & 63];
    }
    v = v * 1.0000001f;
  }
  float r = sink;
#pragma unroll
  for (int i = 0; i < 32; ++i) r += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r + (u ^ u2) * 1e-30f;
}

template <int MODE>
void run(float* d, unsigned* pats, int sms, int clk) {
  const int iters = 20000;
  for (int bps : {4, 8}) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k<MODE><<<sms * bps, 128>>>(d, pats, iters, 1.0f);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    k<MODE><<<sms * bps, 128>>>(d, pats, iters, 1.0f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double cyc = ms * 1e-3 * clk * 1e3;
    const double steps = 16.0 * iters * bps;
    printf("shadow mode %d warps/SMSP %d: %.2f cyc per step (4 FFMA2 = 8.0 ideal), FMA %.1f%%\n", MODE, bps,
           cyc / steps, 100 * 8.0 / (cyc / steps));
  }
}

int main() {
  float* d;
  cudaMalloc(&d, 148 * 8 * 128 * 4);
  unsigned* pats;
  cudaMalloc(&pats, 16 * 4);
  cudaMemset(pats, 0x5a, 64);
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  run<0>(d, pats, sms, clk);
  run<1>(d, pats, sms, clk);
  run<2>(d, pats, sms, clk);
  run<3>(d, pats, sms, clk);
  run<4>(d, pats, sms, clk);
}
