// TMEM load shape check: tcgen05.ld.16x32bx2 (lanes 0-15 of a warp's sub-partition, the
// second half-warp reading columns + imm offset) — the GP-info epilogue's access pattern.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc05_ld_test tools/tc05_ld_test.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k(uint32_t* out) {
  __shared__ uint32_t tb_s;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tb_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = tb_s;
  // cell (lane L, column c) = L * 1000 + c
  for (int c0 = 0; c0 < 128; c0 += 4) {
    const uint32_t L = warp * 32 + lane;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(tb + c0 + ((uint32_t)(warp * 32) << 16)),
                 "r"(L * 1000 + c0), "r"(L * 1000 + c0 + 1), "r"(L * 1000 + c0 + 2), "r"(L * 1000 + c0 + 3));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t r[4];
  asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x4.b32 {%0, %1, %2, %3}, [%4], 36;"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(tb + 8 + ((uint32_t)(warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int i = 0; i < 4; ++i) out[t * 4 + i] = r[i];
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tb));
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, 128 * 4 * 4);
  k<<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  uint32_t h[512];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%s\n", cudaGetErrorString(e));
  for (int t = 0; t < 128; t += (t % 32 == 15 ? 1 : (t % 32 == 16 ? 15 : 1))) {
    if (t % 32 > 1 && t % 32 < 15) continue;
    if (t % 32 > 17 && t % 32 < 31) continue;
    printf("thread %3d:", t);
    for (int i = 0; i < 4; ++i) printf(" (lane %u col %u)", h[t * 4 + i] / 1000, h[t * 4 + i] % 1000);
    printf("\n");
  }
  return 0;
}
