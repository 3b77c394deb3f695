// Dev microbenchmark: does packed FFMA2 (fma.rn.f32x2, sm_100a) free issue
// slots for the zero-skip overhead of the ECR main loop?
//   mode 0: scalar FFMA, 2*NB per taken branch
//   mode 1: FFMA2 with a broadcast scalar operand, NB per taken branch
// Each iteration ballots a 32-bit nonzero mask (like the kernel) and walks
// its 32 bits with uniform branches.  Reports useful FMA/clk/SM.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ void fma2(float2& acc, float2 w, float v) {
  unsigned long long a = *reinterpret_cast<unsigned long long*>(&acc);
  const unsigned long long b = *reinterpret_cast<const unsigned long long*>(&w);
  unsigned long long vv;
  asm("mov.b64 %0, {%1, %1};" : "=l"(vv) : "f"(v));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a) : "l"(b), "l"(vv));
  acc = *reinterpret_cast<float2*>(&a);
}

template <int MODE, int NB>
__global__ void __launch_bounds__(256) kb(float* out, const float* vals, int iters, float seed) {
  __shared__ float sv[64 * 32];
  for (int i = threadIdx.x; i < 64 * 32; i += blockDim.x) sv[i] = vals[i];
  __syncthreads();
  float2 acc[16], w[8];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = make_float2(seed * i, seed);
#pragma unroll
  for (int i = 0; i < 8; ++i) w[i] = make_float2(seed + i * 0.5f + threadIdx.x, seed - i);
  const int lane = threadIdx.x & 31;
  for (int it = 0; it < iters; ++it) {
    const float* row = sv + (it & 63) * 32;
    const unsigned m = __ballot_sync(0xffffffffu, row[lane] != 0.0f);
#pragma unroll
    for (int p = 0; p < 32; ++p) {
      if ((m >> p) & 1u) {
        const float v = row[p];
#pragma unroll
        for (int q = 0; q < NB; ++q) {
          float2& a = acc[(p * NB + q) & 15];
          const float2 ww = w[(p + q) & 7];
          if (MODE == 0) {
            a.x = fmaf(ww.x, v, a.x);
            a.y = fmaf(ww.y, v, a.y);
          } else {
            fma2(a, ww, v);
          }
        }
      }
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i].x + acc[i].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE, int NB>
void run(float* d, const float* vals, int sms, int clk, double dens, long long taken_per_64) {
  const int iters = 20000;
  for (int blocks_per_sm : {1, 2, 4}) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    kb<MODE, NB><<<sms * blocks_per_sm, 256>>>(d, vals, iters, 1.0f);
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    kb<MODE, NB><<<sms * blocks_per_sm, 256>>>(d, vals, iters, 1.0f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double taken = double(taken_per_64) * (iters / 64.0);
    const double fmas = double(sms) * blocks_per_sm * 256 * taken * NB * 2;
    const double per_clk_sm = fmas / (ms * 1e-3) / (sms * clk * 1e3);
    printf("mode %d NB %d dens %.2f warps/SM %2d: %.1f FMA/clk/SM (%.1f%% of 128), %.1f TFLOP/s\n",
           MODE, NB, dens, blocks_per_sm * 8, per_clk_sm, per_clk_sm / 1.28, 2 * fmas / ms / 1e9);
  }
}

int main() {
  float* d;
  cudaMalloc(&d, 148 * 4 * 256 * 4);
  float* vals;
  cudaMalloc(&vals, 64 * 32 * 4);
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  for (double dens : {1.0, 0.3}) {
    float h[64 * 32];
    long long taken = 0;
    srand(1);
    for (int i = 0; i < 64 * 32; ++i) {
      const bool nz = (rand() / (double)RAND_MAX) < dens;
      h[i] = nz ? 0.5f + (i % 7) * 0.01f : 0.0f;
      taken += nz;
    }
    cudaMemcpy(vals, h, sizeof(h), cudaMemcpyHostToDevice);
    run<0, 4>(d, vals, sms, clk, dens, taken);
    run<1, 4>(d, vals, sms, clk, dens, taken);
    run<0, 8>(d, vals, sms, clk, dens, taken);
    run<1, 8>(d, vals, sms, clk, dens, taken);
  }
  printf("clk %d MHz, %d SMs\n", clk / 1000, sms);
}
