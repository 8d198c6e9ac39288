// tcgen05.mma kind::f16 (FP16 in, FP32 accumulate) for the GP-info contraction shapes:
//  1. correctness + TMEM placement of D for M=64 and M=128 (K-major, no swizzle, SS);
//  2. issue throughput per shape, one CTA per SM, NACC independent accumulators.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc05_f16_bench tools/tc05_f16_bench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
// kind::f16: D f32 (bit 4), A f16 (0), B f16 (0), both K-major
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// element (r, k) of an R x 16 tile, K-major no swizzle: 8-row groups of 2 core matrices (8 x 8 halves)
__host__ __device__ inline int koff(int r, int k) { return (r >> 3) * 128 + (k >> 3) * 64 + (r & 7) * 8 + (k & 7); }

template <int M, int N, int DLANE = 0>
__global__ void k_layout(const __half* A, const __half* B, float* D /*[128][N]*/) {
  __shared__ __align__(128) __half sa[128 * 16];
  __shared__ __align__(128) __half sb[256 * 16];
  __shared__ uint32_t tb_s;
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x, warp = t >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tb_s)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = t; i < M * 16; i += blockDim.x) sa[koff(i / 16, i % 16)] = A[i];
  for (int i = t; i < N * 16; i += blockDim.x) sb[koff(i / 16, i % 16)] = B[i];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = tb_s;
  // clear D region: every warp writes zeros to its lanes, columns [0, 256)
  {
    uint32_t z[32];
    for (int i = 0; i < 32; ++i) z[i] = 0x7fc00000u;  // NaN marker: untouched cells stay NaN
    for (int c0 = 0; c0 < 256; c0 += 32) {
      const uint32_t addr = tb + c0 + ((uint32_t)(warp * 32) << 16);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                   "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(addr),
                   "r"(z[0]), "r"(z[1]), "r"(z[2]), "r"(z[3]), "r"(z[4]), "r"(z[5]), "r"(z[6]), "r"(z[7]), "r"(z[8]),
                   "r"(z[9]), "r"(z[10]), "r"(z[11]), "r"(z[12]), "r"(z[13]), "r"(z[14]), "r"(z[15]), "r"(z[16]),
                   "r"(z[17]), "r"(z[18]), "r"(z[19]), "r"(z[20]), "r"(z[21]), "r"(z[22]), "r"(z[23]), "r"(z[24]),
                   "r"(z[25]), "r"(z[26]), "r"(z[27]), "r"(z[28]), "r"(z[29]), "r"(z[30]), "r"(z[31]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (t == 0) {
    const uint64_t da = make_desc(smem_u32(sa), 128, 256), db = make_desc(smem_u32(sb), 128, 256);
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tb + ((uint32_t)DLANE << 16)), "l"(da), "l"(db),
                 "r"(idesc_f16(M, N)), "r"(0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
  }
  asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t r[8];
    const uint32_t addr = tb + c0 + ((uint32_t)(warp * 32) << 16);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) D[t * N + c0 + j] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(256));
}

template <int M, int N, int DLANE = 0>
int layout_test() {
  __half *hA = (__half*)malloc(2 * M * 16), *hB = (__half*)malloc(2 * N * 16);
  float* hD = (float*)malloc(4 * 128 * N);
  srand(M * 7 + N);
  for (int i = 0; i < M * 16; ++i) hA[i] = __float2half((float)(rand() % 64 - 32) / 16.f);
  for (int i = 0; i < N * 16; ++i) hB[i] = __float2half((float)(rand() % 64 - 32) / 32.f);
  __half *dA, *dB; float* dD;
  cudaMalloc(&dA, 2 * M * 16); cudaMalloc(&dB, 2 * N * 16); cudaMalloc(&dD, 4 * 128 * N);
  cudaMemcpy(dA, hA, 2 * M * 16, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, 2 * N * 16, cudaMemcpyHostToDevice);
  k_layout<M, N, DLANE><<<1, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(hD, dD, 4 * 128 * N, cudaMemcpyDeviceToHost);
  // for every row r of the product find the TMEM lane holding it
  int bad = 0;
  printf("M=%d N=%d dlane=%d: %s; row -> lane:", M, N, DLANE, cudaGetErrorString(e));
  for (int r = 0; r < M; ++r) {
    int found = -1;
    for (int lane = 0; lane < 128 && found < 0; ++lane) {
      bool ok = true;
      for (int c = 0; c < N && ok; ++c) {
        double s = 0;
        for (int k = 0; k < 16; ++k) s += (double)__half2float(hA[r * 16 + k]) * __half2float(hB[c * 16 + k]);
        ok = fabs(s - hD[lane * N + c]) < 1e-4;
      }
      if (ok) found = lane;
    }
    if (found < 0) ++bad;
    if (r % 8 == 0 || found != r) printf(" %d:%d", r, found);
  }
  int nan_lanes = 0;
  for (int lane = 0; lane < 128; ++lane) nan_lanes += std::isnan(hD[lane * N]);
  printf("\n  rows without a lane: %d; lanes still NaN: %d\n", bad, nan_lanes);
  cudaFree(dA); cudaFree(dB); cudaFree(dD);
  return bad;
}

template <int M, int N, int NACC>
__global__ void k_rate(long long* cyc, int iters) {
  __shared__ __align__(128) __half sa[2][128 * 16];
  __shared__ __align__(128) __half sb[2][256 * 16];
  __shared__ uint32_t tb_s;
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 2 * 128 * 16; i += blockDim.x) (&sa[0][0])[i] = __float2half(0.001f * (i % 7));
  for (int i = t; i < 2 * 256 * 16; i += blockDim.x) (&sb[0][0])[i] = __float2half(0.002f * (i % 5));
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tb_s)), "r"(512));
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
    const uint32_t idesc = idesc_f16(M, N);
    uint64_t da[2], db[2];
    for (int ks = 0; ks < 2; ++ks) {
      da[ks] = make_desc(smem_u32(sa[ks]), 128, 256);
      db[ks] = make_desc(smem_u32(sb[ks]), 128, 256);
    }
    for (int it = 0; it < iters; it += 8) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const uint32_t d = tb + (u % NACC) * ((N + 15) & ~15);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                     "l"(da[u & 1]), "l"(db[u & 1]), "r"(idesc), "r"(1));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
  }
  asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
  long long t1 = clock64();
  if (t == 0 && blockIdx.x == 0) *cyc = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512));
}
template <int M, int N, int NACC>
void rate(const char* name) {
  long long* d; cudaMalloc(&d, 8);
  const int iters = 8192;
  k_rate<M, N, NACC><<<148, 128>>>(d, iters);
  cudaDeviceSynchronize();
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k_rate<M, N, NACC><<<148, 128>>>(d, iters);
  cudaEventRecord(b); cudaError_t e = cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  long long c; cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  double flops = 2.0 * M * N * 16 * (double)iters * 148;
  printf("%-28s %s  %6.1f cycles/MMA  %7.1f TFLOP/s\n", name, cudaGetErrorString(e), (double)c / iters, flops / ms / 1e9);
}
int main(int argc, char** argv) {
  if (argc > 1) { layout_test<64, 144, 16>(); return 0; }
  int bad = layout_test<64, 144>() + layout_test<128, 144>() + layout_test<64, 48>();
  rate<64, 144, 3>("f16 SS M64 N144 acc3");
  rate<64, 144, 1>("f16 SS M64 N144 acc1");
  rate<128, 144, 3>("f16 SS M128 N144 acc3");
  rate<64, 80, 4>("f16 SS M64 N80 acc4");
  rate<128, 48, 4>("f16 SS M128 N48 acc4");
  rate<128, 32, 4>("f16 SS M128 N32 acc4");
  rate<64, 256, 2>("f16 SS M64 N256 acc2");
  rate<128, 256, 2>("f16 SS M128 N256 acc2");
  rate<64, 72, 4>("f16 SS M64 N72 acc4");
  printf("%s\n", bad ? "LAYOUT FAILURES" : "layouts ok");
  return 0;
}
