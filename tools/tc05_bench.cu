// tcgen05.mma issue throughput, kind::tf32, M=128, N in {24,32,64}, SS vs TS, one CTA per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(const void* base, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(base) >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
template <int MODE, int N, int NACC>
__global__ void k(long long* cyc, int iters) {
  __shared__ __align__(128) float sa[128 * 32];
  __shared__ __align__(128) float sb[64 * 32];
  __shared__ uint32_t tb_s;
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 128 * 32; i += blockDim.x) sa[i] = 0.001f * (i % 7);
  for (int i = t; i < 64 * 32; i += blockDim.x) sb[i] = 0.002f * (i % 5);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tb_s)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = tb_s;
  long long t0 = clock64();
  if (t == 0) {
    const uint32_t idesc = make_idesc(128, N);
    uint64_t da[4], db[4];
    for (int ks = 0; ks < 4; ++ks) { da[ks] = make_desc(sa + ks * 64, 128, 1024); db[ks] = make_desc(sb + ks * 64, 128, 1024); }
    for (int it = 0; it < iters; it += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t d = tb + (u % NACC) * N;
        if (MODE == 0)
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                       "l"(da[u & 3]), "l"(db[u & 3]), "r"(idesc), "r"(1));
        else
          asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                       "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
                       "r"(tb + 224 + (u & 3) * 8), "l"(db[u & 3]), "r"(idesc), "r"(1));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
  }
  asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
  long long t1 = clock64();
  if (t == 0 && blockIdx.x == 0) *cyc = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(256));
}
template <int MODE, int N, int NACC>
void run(const char* name) {
  long long* d; cudaMalloc(&d, 8);
  const int iters = 8192;
  k<MODE, N, NACC><<<148, 128>>>(d, iters);
  cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<MODE, N, NACC><<<148, 128>>>(d, iters);
  cudaEventRecord(b); cudaError_t e = cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  double flops = 2.0 * 128 * N * 8 * iters * 148;
  printf("%-24s %s  %.1f cycles/MMA  %.1f TFLOP/s\n", name, cudaGetErrorString(e), (double)c / iters, flops / ms / 1e9);
}
int main() {
  run<0, 24, 1>("SS N24 acc1");
  run<0, 24, 2>("SS N24 acc2");
  run<0, 24, 4>("SS N24 acc4");
  run<0, 24, 8>("SS N24 acc8");
  run<1, 24, 8>("TS N24 acc8");
  run<0, 32, 6>("SS N32 acc6");
  run<1, 32, 6>("TS N32 acc6");
  return 0;
}
