// Do legacy HMMA (mma.sync tf32) and MUFU (ex2/rcp) overlap on sm_100a?  Per-warp
// instruction streams: HMMA only, MUFU only, and both interleaved 1:1 / 45:36.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 1024
__device__ __forceinline__ void mma(float (&c)[4], unsigned a0, unsigned a1, unsigned a2, unsigned a3, unsigned b0, unsigned b1) {
  asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
template <int NH, int NM>
__global__ void kern(float* out, float seed) {
  float acc[8][4];
  float m[8];
  unsigned a = __float_as_uint(seed + threadIdx.x * 1e-3f), b = __float_as_uint(seed * 0.5f);
  for (int c = 0; c < 8; ++c) { m[c] = seed * c * 1e-3f; for (int j = 0; j < 4; ++j) acc[c][j] = 0.f; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (c < NH) mma(acc[c], a, a ^ c, a, a, b, b ^ c);
      if (c < NM) m[c] = ex2(m[c]) * -0.5f;
    }
  }
  float s = 0;
  for (int c = 0; c < 8; ++c) { s += m[c]; for (int j = 0; j < 4; ++j) s += acc[c][j]; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int NH, int NM>
void run(const char* name, int sms, int warps_per_sm) {
  const int threads = 128, blocks = sms * warps_per_sm / 4;
  float* o; cudaMalloc(&o, sizeof(float) * threads * blocks);
  kern<NH, NM><<<blocks, threads>>>(o, 1.0f);
  cudaEvent_t x, y; cudaEventCreate(&x); cudaEventCreate(&y);
  cudaEventRecord(x);
  kern<NH, NM><<<blocks, threads>>>(o, 1.0f);
  cudaEventRecord(y); cudaEventSynchronize(y);
  float ms; cudaEventElapsedTime(&ms, x, y);
  double warps = (double)blocks * threads / 32;
  double clk = 1.965e9 * ms / 1e3;
  printf("%-28s warps/SM %2d  %7.3f ms  per-SMSP clk per warp-iter %.1f\n", name, warps_per_sm, ms,
         clk / (warps / sms / 4) / ITERS);
  cudaFree(o);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {8, 16}) {
    run<8, 0>("8 HMMA", sms, w);
    run<0, 8>("8 MUFU.EX2", sms, w);
    run<8, 8>("8 HMMA + 8 MUFU interleaved", sms, w);
    run<8, 6>("8 HMMA + 6 MUFU interleaved", sms, w);
  }
  return 0;
}
