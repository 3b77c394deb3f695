// Dev microbenchmark: cost of the ECR zero-skip branch on sm_100a.
// 32 positions per iteration; position p runs NB FFMA2 iff bit p of a
// warp-uniform mask (a ballot) is set.  v lives in registers (no LDS).
// MODE 0: no branch (all blocks run)  MODE 1: if(bit) { pmevent; block }
// MODE 2: if(bit) { block } (ptxas may predicate)
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void fma2(float& a0, float& a1, float w0, float w1, float v) {
  asm("{\n\t.reg .b64 a, w, v;\n\tmov.b64 a, {%0, %1};\n\tmov.b64 w, {%2, %3};\n\t"
      "mov.b64 v, {%4, %4};\n\tfma.rn.f32x2 a, w, v, a;\n\tmov.b64 {%0, %1}, a;\n\t}"
      : "+f"(a0), "+f"(a1) : "f"(w0), "f"(w1), "f"(v));
}

template <int MODE, int NB>
__global__ void __launch_bounds__(128) k(float* out, const unsigned* pats, int iters, float seed) {
  float acc[32], w[16], vv[8];
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = seed * i;
#pragma unroll
  for (int i = 0; i < 16; ++i) w[i] = seed + i * 0.5f + threadIdx.x;
#pragma unroll
  for (int i = 0; i < 8; ++i) vv[i] = seed * (threadIdx.x + i);
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
    const unsigned m = __ballot_sync(0xffffffffu, (pats[it & 15] >> lane) & 1u);
#pragma unroll
    for (int p = 0; p < 32; ++p) {
      const bool run = MODE == 0 || ((m >> p) & 1u);
      if (run) {
        if (MODE == 1) asm volatile("pmevent 0;");
        const float v = vv[p & 7];
#pragma unroll
        for (int q = 0; q < NB; ++q) {
          const int a = (2 * (p * NB + q)) & 31;
          fma2(acc[a], acc[a + 1], w[(2 * q) & 15], w[(2 * q + 1) & 15], v);
        }
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 32; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE, int NB>
void run(float* d, unsigned* pats, int sms, int clk, int taken16, const char* what) {
  const int iters = 4000;
  for (int bps : {4, 8}) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k<MODE, NB><<<sms * bps, 128>>>(d, pats, iters, 1.0f);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    k<MODE, NB><<<sms * bps, 128>>>(d, pats, iters, 1.0f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double blocks = MODE == 0 ? 32.0 * iters : taken16 / 16.0 * iters;  // per thread
    const double cyc = ms * 1e-3 * clk * 1e3;                                   // per SMSP
    const double warps_per_smsp = bps;                                          // 4 warps/CTA
    const double fma = blocks * NB * 2 * 32 * warps_per_smsp;                    // per SMSP
    printf("%-10s mode %d NB %d warps/SMSP %d: %.1f%% of FMA peak, %.1f cyc per executed block per warp-slot, %.2f cyc per position\n",
           what, MODE, NB, bps, 100 * fma / cyc / 32, cyc / (blocks * warps_per_smsp),
           cyc / (32.0 * iters * warps_per_smsp));
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
    if (dens == 1.0) { run<0, 2>(d, pats, sms, clk, taken, "nobranch"); run<0, 8>(d, pats, sms, clk, taken, "nobranch"); }
    run<1, 2>(d, pats, sms, clk, taken, what);
    run<1, 4>(d, pats, sms, clk, taken, what);
    run<1, 8>(d, pats, sms, clk, taken, what);
    run<2, 2>(d, pats, sms, clk, taken, what);
    run<2, 8>(d, pats, sms, clk, taken, what);
  }
}
