// tcgen05.mma kind::f16 with BOTH operands MN-major (no swizzle), the layout the GP-info
// build's producers write (a thread = one landmark = one K index stores 8 consecutive
// M/N elements as one 16-byte vector).  Checks which of LBO / SBO is the MN-group stride,
// over 4 accumulated K=16 steps, M=64, N=144.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tc05_mn_test tools/tc05_mn_test.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
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
// kind::f16, D f32, A/B f16, A and B MN-major (bits 15, 16)
__host__ __device__ constexpr uint32_t idesc_mn(int M, int N) {
  return (1u << 4) | (1u << 15) | (1u << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
constexpr int M = 64, N = 144, KS = 4, K = 16 * KS;
// MN-major: 16-byte vectors of 8 MN-consecutive elements; vector (g = mn/8, k):
//   byte offset = kstep*BLK + g*GS + (k%16/8)*KG + (k%8)*16
// with GS = MN-group stride, KG = K-group (8 rows) stride
template <int MODE>
__global__ void k_mn(const __half* A /*[M][K]*/, const __half* B /*[N][K]*/, float* D /*[M][N]*/) {
  __shared__ __align__(1024) __half sa[KS * M * 16];
  __shared__ __align__(1024) __half sb[KS * N * 16];
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
  // layout: MN groups contiguous (GS = 128 B), K groups at KG = (MN/8)*128
  const int GA = 128, KGA = (M / 8) * 128, BLKA = M * 16 * 2;
  const int GB = 128, KGB = (N / 8) * 128, BLKB = N * 16 * 2;
  for (int i = t; i < M * K; i += blockDim.x) {
    const int m = i / K, k = i % K;
    const int off = (k / 16) * BLKA + (m / 8) * GA + ((k % 16) / 8) * KGA + (k % 8) * 16 + (m % 8) * 2;
    sa[off / 2] = A[i];
  }
  for (int i = t; i < N * K; i += blockDim.x) {
    const int n = i / K, k = i % K;
    const int off = (k / 16) * BLKB + (n / 8) * GB + ((k % 16) / 8) * KGB + (k % 8) * 16 + (n % 8) * 2;
    sb[off / 2] = B[i];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = tb_s;
  if (t == 0) {
    for (int ks = 0; ks < KS; ++ks) {
      uint64_t da, db;
      if (MODE == 0) {  // LBO = MN-group stride, SBO = K-group stride
        da = make_desc(smem_u32(sa) + ks * BLKA, GA, KGA);
        db = make_desc(smem_u32(sb) + ks * BLKB, GB, KGB);
      } else {          // swapped
        da = make_desc(smem_u32(sa) + ks * BLKA, KGA, GA);
        db = make_desc(smem_u32(sb) + ks * BLKB, KGB, GB);
      }
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tb), "l"(da), "l"(db),
                   "r"(idesc_mn(M, N)), "r"(ks > 0 ? 1u : 0u));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
  }
  asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // M=64: row r lives in lane (r/16)*32 + r%16
  const int lane = t & 31;
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t r[8];
    const uint32_t addr = tb + c0 + ((uint32_t)(warp * 32) << 16);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (lane < 16)
      for (int j = 0; j < 8; ++j) D[(warp * 16 + lane) * N + c0 + j] = __uint_as_float(r[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(256));
}

int main(int argc, char** argv) {
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  __half *hA = (__half*)malloc(2 * M * K), *hB = (__half*)malloc(2 * N * K);
  float* hD = (float*)malloc(4 * M * N);
  srand(3);
  for (int i = 0; i < M * K; ++i) hA[i] = __float2half((float)(rand() % 64 - 32) / 16.f);
  for (int i = 0; i < N * K; ++i) hB[i] = __float2half((float)(rand() % 64 - 32) / 32.f);
  __half *dA, *dB; float* dD;
  cudaMalloc(&dA, 2 * M * K); cudaMalloc(&dB, 2 * N * K); cudaMalloc(&dD, 4 * M * N);
  cudaMemcpy(dA, hA, 2 * M * K, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, 2 * N * K, cudaMemcpyHostToDevice);
  int ok_modes = 0;
  for (int mode = 0; mode < 2; ++mode) {
    if (only >= 0 && mode != only) continue;
    cudaMemset(dD, 0, 4 * M * N);
    if (mode == 0) k_mn<0><<<1, 128>>>(dA, dB, dD); else k_mn<1><<<1, 128>>>(dA, dB, dD);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hD, dD, 4 * M * N, cudaMemcpyDeviceToHost);
    double err = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double s = 0;
        for (int k = 0; k < K; ++k) s += (double)__half2float(hA[m * K + k]) * __half2float(hB[n * K + k]);
        err = fmax(err, fabs(s - hD[m * N + n]));
      }
    printf("MN-major mode %d (%s): %s maxerr %.3e\n", mode, mode ? "LBO=K-group, SBO=MN-group" : "LBO=MN-group, SBO=K-group",
           cudaGetErrorString(e), err);
    if (e == cudaSuccess && err < 1e-3) ok_modes |= 1 << mode;
  }
  printf("ok modes mask %d\n", ok_modes);
  return ok_modes ? 0 : 1;
}
