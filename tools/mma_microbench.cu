// Throughput of legacy warp-level mma.sync on sm_100a (TF32 m16n8k8, BF16 m16n8k16),
// operands in registers, independent accumulator chains.  Design input for the GP build.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 2048
template <int OP>
__global__ void kern(float* out, float seed) {
  float acc[8][4];
  unsigned a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(seed + threadIdx.x * 1e-3f + i);
  for (int i = 0; i < 2; ++i) b[i] = __float_as_uint(seed * 0.5f + i);
  for (int c = 0; c < 8; ++c) for (int j = 0; j < 4; ++j) acc[c][j] = 0.f;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (OP == 0)
        asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(acc[c][0]), "+f"(acc[c][1]), "+f"(acc[c][2]), "+f"(acc[c][3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      else
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(acc[c][0]), "+f"(acc[c][1]), "+f"(acc[c][2]), "+f"(acc[c][3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
    }
  }
  float s = 0;
  for (int c = 0; c < 8; ++c) for (int j = 0; j < 4; ++j) s += acc[c][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int OP>
void run(const char* name, int sms, double flops_per_mma) {
  const int threads = 256, blocks = sms * 4;
  float* o; cudaMalloc(&o, sizeof(float) * threads * blocks);
  kern<OP><<<blocks, threads>>>(o, 1.0f);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<OP><<<blocks, threads>>>(o, 1.0f);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double mmas = (double)blocks * threads / 32 * ITERS * 8;
  printf("%-32s %8.3f ms  %8.1f TFLOP/s\n", name, ms, mmas * flops_per_mma / ms / 1e9);
  cudaFree(o);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0>("mma.sync m16n8k8 tf32", sms, 2.0 * 16 * 8 * 8);
  run<1>("mma.sync m16n8k16 bf16", sms, 2.0 * 16 * 8 * 16);
  return 0;
}
