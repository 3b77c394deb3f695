// Dev microbenchmark: per-nonzero jump-table dispatch (switch over the set
// bits of a warp-uniform mask) instead of one branch per position.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void fma2(float& a0, float& a1, float w0, float w1, float v) {
  asm("{\n\t.reg .b64 a, w, v;\n\tmov.b64 a, {%0, %1};\n\tmov.b64 w, {%2, %3};\n\t"
      "mov.b64 v, {%4, %4};\n\tfma.rn.f32x2 a, w, v, a;\n\tmov.b64 {%0, %1}, a;\n\t}"
      : "+f"(a0), "+f"(a1) : "f"(w0), "f"(w1), "f"(v));
}

#define CASE(P)                                                        \
  case P:                                                              \
    _Pragma("unroll") for (int q = 0; q < NB; ++q) {                   \
      const int a = (2 * (P * NB + q)) & 31;                           \
      fma2(acc[a], acc[a + 1], w[(2 * q + P) & 15], w[(2 * q + 1 + P) & 15], v); \
    }                                                                  \
    break;

template <int NB, int MODE>  // MODE 0: LDS v per nonzero; MODE 1: v from registers via shfl-free select
__global__ void __launch_bounds__(128) k(float* out, const unsigned* pats, int iters, float seed) {
  __shared__ float sv[32];
  if (threadIdx.x < 32) sv[threadIdx.x] = seed * (threadIdx.x + 1);
  __syncthreads();
  float acc[32], w[16];
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = seed * i;
#pragma unroll
  for (int i = 0; i < 16; ++i) w[i] = seed + i * 0.5f + threadIdx.x;
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
    unsigned m = __ballot_sync(0xffffffffu, (pats[it & 15] >> lane) & 1u);
    while (m) {
      const int p = __ffs(m) - 1;
      m &= m - 1;
      const float v = sv[p];
      switch (p) {
        CASE(0) CASE(1) CASE(2) CASE(3) CASE(4) CASE(5) CASE(6) CASE(7)
        CASE(8) CASE(9) CASE(10) CASE(11) CASE(12) CASE(13) CASE(14) CASE(15)
        CASE(16) CASE(17) CASE(18) CASE(19) CASE(20) CASE(21) CASE(22) CASE(23)
        CASE(24) CASE(25) CASE(26) CASE(27) CASE(28) CASE(29) CASE(30) CASE(31)
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NB>
void run(float* d, unsigned* pats, int sms, int clk, int taken16, const char* what) {
  const int iters = 4000;
  for (int bps : {4, 8}) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k<NB, 0><<<sms * bps, 128>>>(d, pats, iters, 1.0f);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    k<NB, 0><<<sms * bps, 128>>>(d, pats, iters, 1.0f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double blocks = taken16 / 16.0 * iters;
    const double cyc = ms * 1e-3 * clk * 1e3;
    const double fma = blocks * NB * 2 * 32 * bps;
    printf("%-10s switch NB %d warps/SMSP %d: %.1f%% of FMA peak, %.1f cyc per nonzero, %.2f cyc per position\n",
           what, NB, bps, 100 * fma / cyc / 32, cyc / (blocks * bps), cyc / (32.0 * iters * bps));
  }
}

int main() {
  float* d;
  cudaMalloc(&d, 148 * 8 * 128 * 4);
  unsigned* pats;
  cudaMalloc(&pats, 16 * 4);
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  unsigned h[16];
  for (double dens : {1.0, 0.5, 0.3}) {
    unsigned long long s = 12345;
    int taken = 0;
    for (int i = 0; i < 16; ++i) {
      h[i] = 0;
      for (int b = 0; b < 32; ++b) {
        s = s * 6364136223846793005ull + 1442695040888963407ull;
        if ((s >> 40) % 1000 < dens * 1000) { h[i] |= 1u << b; ++taken; }
      }
    }
    cudaMemcpy(pats, h, sizeof(h), cudaMemcpyHostToDevice);
    char what[32];
    snprintf(what, 32, "dens %.1f", dens);
    run<2>(d, pats, sms, clk, taken, what);
    run<4>(d, pats, sms, clk, taken, what);
    run<8>(d, pats, sms, clk, taken, what);
  }
}
