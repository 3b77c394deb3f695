// Dev microbenchmark: vector-predicate BRA vs uniform-predicate BRA.U for the
// ECR zero-skip branch (32 positions, NB FFMA2 per taken position).
// MODE 0: no branch; MODE 1: mask from a ballot (vector), MODE 2: mask from a
// uniform load (UR), MODE 3: MODE 2 with the block entered by an inverted
// test (zero cell = taken jump over).
#include <cstdio>
#include <cuda_runtime.h>
__constant__ unsigned cpats[16];

__device__ __forceinline__ void fma2(float& a0, float& a1, float w0, float w1, float v) {
  asm("{\n\t.reg .b64 a, w, v;\n\tmov.b64 a, {%0, %1};\n\tmov.b64 w, {%2, %3};\n\t"
      "mov.b64 v, {%4, %4};\n\tfma.rn.f32x2 a, w, v, a;\n\tmov.b64 {%0, %1}, a;\n\t}"
      : "+f"(a0), "+f"(a1) : "f"(w0), "f"(w1), "f"(v));
}

template <int MODE, int NB>
__global__ void __launch_bounds__(128) k(float* out, const unsigned* __restrict__ pats, int iters, float seed) {
  float acc[32], w[16], vv[8];
#pragma unroll
  for (int i = 0; i < 32; ++i) acc[i] = seed * i;
#pragma unroll
  for (int i = 0; i < 16; ++i) w[i] = seed + i * 0.5f + threadIdx.x;
#pragma unroll
  for (int i = 0; i < 8; ++i) vv[i] = seed * (threadIdx.x + i);
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
    unsigned m;
    if (MODE == 1) m = __ballot_sync(0xffffffffu, (pats[it & 15] >> lane) & 1u);
    else m = cpats[it & 15];  // constant bank, uniform index -> UR
#pragma unroll
    for (int p = 0; p < 32; ++p) {
      const bool run = MODE == 0 || ((m >> p) & 1u);
      if (run) {
        if (MODE != 0) asm volatile("pmevent 0;");
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
    const double blocks = MODE == 0 ? 32.0 * iters : taken16 / 16.0 * iters;
    const double cyc = ms * 1e-3 * clk * 1e3;
    const double fma = blocks * NB * 2 * 32 * bps;
    printf("%-8s mode %d NB %2d warps/SMSP %d: %.1f%% of FMA peak, %.2f cyc per position\n", what, MODE, NB,
           bps, 100 * fma / cyc / 32, cyc / (32.0 * iters * bps));
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
  for (double dens : {1.0, 0.3}) {
    unsigned h[16];
    unsigned long long st = 12345;
    int taken = 0;
    for (int i = 0; i < 16; ++i) {
      h[i] = 0;
      for (int b = 0; b < 32; ++b) {
        st = st * 6364136223846793005ull + 1442695040888963407ull;
        if ((st >> 33) % 1000 < dens * 1000) { h[i] |= 1u << b; ++taken; }
      }
    }
    cudaMemcpy(pats, h, sizeof h, cudaMemcpyHostToDevice);
    cudaMemcpyToSymbol(cpats, h, sizeof h);
    char what[16];
    snprintf(what, sizeof what, "dens %.1f", dens);
    run<0, 4>(d, pats, sms, clk, taken, what);
    run<1, 4>(d, pats, sms, clk, taken, what);
    run<2, 4>(d, pats, sms, clk, taken, what);
    run<1, 8>(d, pats, sms, clk, taken, what);
    run<2, 8>(d, pats, sms, clk, taken, what);
    run<1, 16>(d, pats, sms, clk, taken, what);
    run<2, 16>(d, pats, sms, clk, taken, what);
  }
  return 0;
}
