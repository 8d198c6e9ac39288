// Which pipe runs F2FP (cvt.rn.f16x2.f32) on sm_100a?  Throughput alone and mixed with
// MUFU.EX2; per-warp independent chains.
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#define ITERS 1024
template <int NF, int NM>
__global__ void kern(float* out, float seed) {
  float m[8];
  float f[8];
  for (int c = 0; c < 8; ++c) { m[c] = seed * c * 1e-3f; f[c] = seed + c + threadIdx.x * 1e-3f; }
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (c < NF) {
        __half2 h = __floats2half2_rn(f[c], f[(c + 1) & 7]);
        f[c] = __int_as_float(*reinterpret_cast<int*>(&h)) * 1.0001f + 1e-3f;
      }
      if (c < NM) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(m[c])); m[c] = y * -0.5f; }
    }
  }
  float s = 0;
  for (int c = 0; c < 8; ++c) s += m[c] + f[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int NF, int NM>
void run(const char* name, int sms) {
  const int threads = 256, blocks = sms * 4;
  float* o; cudaMalloc(&o, sizeof(float) * threads * blocks);
  kern<NF, NM><<<blocks, threads>>>(o, 1.0f);
  cudaEvent_t x, y; cudaEventCreate(&x); cudaEventCreate(&y);
  cudaEventRecord(x);
  kern<NF, NM><<<blocks, threads>>>(o, 1.0f);
  cudaEventRecord(y); cudaEventSynchronize(y);
  float ms; cudaEventElapsedTime(&ms, x, y);
  double warp_iters = (double)blocks * threads / 32 * ITERS;
  printf("%-24s %7.3f ms  per-SM clk per warp-iteration %.2f\n", name, ms, 1.965e9 * ms / 1e3 / (warp_iters / sms));
  cudaFree(o);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<8, 0>("8 F2FP", sms);
  run<0, 8>("8 MUFU.EX2", sms);
  run<8, 8>("8 F2FP + 8 EX2", sms);
  return 0;
}
