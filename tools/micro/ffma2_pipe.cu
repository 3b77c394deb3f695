// Dev microbenchmark: FFMA vs FFMA2 throughput, alone and with one
// interleaved ALU op (does FFMA2 leave issue slots for other work?).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void fma2(float& a0, float& a1, float w0, float w1, float v) {
  asm volatile("{\n\t.reg .b64 a, w, v;\n\tmov.b64 a, {%0, %1};\n\tmov.b64 w, {%2, %3};\n\t"
      "mov.b64 v, {%4, %4};\n\tfma.rn.f32x2 a, w, v, a;\n\tmov.b64 {%0, %1}, a;\n\t}"
      : "+f"(a0), "+f"(a1) : "f"(w0), "f"(w1), "f"(v));
}

template <int MODE>  // 0 FFMA, 1 FFMA2, 2 FFMA + ALU, 3 FFMA2 + ALU, 4 FFMA2 + 2 ALU
__global__ void __launch_bounds__(128) k(float* out, int iters, float seed) {
  float acc[32], w[8];
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = seed * i;
#pragma unroll
  for (int i = 0; i < 8; ++i) w[i] = seed + i * 0.5f + threadIdx.x;
  float v = seed * threadIdx.x;
  unsigned x0 = threadIdx.x, x1 = threadIdx.x * 3, x2 = threadIdx.x * 7, x3 = threadIdx.x * 11;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 32; i += 2) {
      if (MODE == 0 || MODE == 2) {
        acc[i] = fmaf(w[i & 7], v, acc[i]);
        acc[i + 1] = fmaf(w[(i + 1) & 7], v, acc[i + 1]);
      } else {
        fma2(acc[i], acc[i + 1], w[i & 7], w[(i + 1) & 7], v);
      }
      if (MODE == 2) {
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x0) : "r"(x1), "r"(x2));
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x1) : "r"(x2), "r"(x3));
      }
      if (MODE == 3 || MODE == 4) {
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x0) : "r"(x1), "r"(x2));
      }
      if (MODE == 4) {
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x1) : "r"(x2), "r"(x3));
      }
    }
    v = v * 1.0000001f;
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + (x0 ^ x1) * 1e-30f;
}

template <int MODE>
void run(float* d, int sms, int clk) {
  const int iters = 20000;
  for (int bps : {2, 4, 8}) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k<MODE><<<sms * bps, 128>>>(d, iters, 1.0f);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    k<MODE><<<sms * bps, 128>>>(d, iters, 1.0f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double fmas = double(sms) * bps * 128 * iters * 32.0;
    const double per = fmas / (ms * 1e-3) / (sms * clk * 1e3);
    printf("mode %d warps/SM %2d: %.1f FMA/clk/SM (%.1f%% of 128)\n", MODE, bps * 4, per, per / 1.28);
  }
}

int main() {
  float* d;
  cudaMalloc(&d, 148 * 8 * 128 * 4);
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  run<0>(d, sms, clk);
  run<1>(d, sms, clk);
  run<2>(d, sms, clk);
  run<3>(d, sms, clk);
  run<4>(d, sms, clk);
}
