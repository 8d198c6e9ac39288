// FP64 throughput on sm_100a: mma.sync m8n8k4 f64 (DMMA) vs DFMA, operands in
// registers, independent accumulator chains.  Design input for the query omega prep.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 2048
__global__ void k_dmma(double* out, double seed) {
  double acc[8][2];
  double a = seed + threadIdx.x * 1e-3, b = seed * 0.5;
  for (int c = 0; c < 8; ++c) acc[c][0] = acc[c][1] = 0.0;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int c = 0; c < 8; ++c) s += acc[c][0] + acc[c][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dfma(double* out, double seed) {
  double acc[8];
  double a = seed + threadIdx.x * 1e-3, b = seed * 0.5;
  for (int c = 0; c < 8; ++c) acc[c] = 0.0;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) acc[c] = fma(a, b, acc[c]);
  }
  double s = 0;
  for (int c = 0; c < 8; ++c) s += acc[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <typename K>
void run(const char* name, K kern, int sms, double flops_per_op_per_warp) {
  const int threads = 256, blocks = sms * 4;
  double* o; cudaMalloc(&o, sizeof(double) * threads * blocks);
  kern<<<blocks, threads>>>(o, 1.0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<<<blocks, threads>>>(o, 1.0);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ops = (double)blocks * threads / 32 * ITERS * 8;
  printf("%-32s %8.3f ms  %8.2f TFLOP/s\n", name, ms, ops * flops_per_op_per_warp / ms / 1e9);
  cudaFree(o);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run("mma.sync m8n8k4 f64 (DMMA)", k_dmma, sms, 2.0 * 8 * 8 * 4);
  run("DFMA", k_dfma, sms, 2.0 * 32);
  return 0;
}
