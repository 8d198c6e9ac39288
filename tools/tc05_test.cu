// Standalone validation of the tcgen05 building blocks used by the GP-info build:
// TMEM alloc, smem matrix descriptors (K-major, no swizzle), instruction descriptor
// for kind::tf32, tcgen05.mma SS and TS (A from TMEM), commit->mbarrier, tcgen05.ld.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major, SWIZZLE_NONE: core matrix = 8 rows x 16 B; LBO = K-direction core stride,
// SBO = M/N-direction 8-row-group stride (both bytes, encoded >> 4); version 1 (sm100).
__device__ __forceinline__ uint64_t make_desc(const void* base, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(base) >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version
  return d;                // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
}
// kind::tf32 instruction descriptor: D f32, A/B tf32, K-major both, N>>3, M>>4
__host__ __device__ constexpr uint32_t make_idesc(int M, int N) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// element (r, k) of an R x K tile in the K-major no-swizzle layout with LBO=128, SBO=256*(K/8)
__device__ __forceinline__ int kmaj_off(int r, int k, int K) {
  // per 8-row group: (K/4) core matrices of 128 B each, consecutive along K
  return (r / 8) * (K / 4) * 32 + (k / 4) * 32 + (r % 8) * 4 + (k % 4);  // in floats
}

template <int MODE>  // 0: SS, 1: TS (A from TMEM)
__global__ void k_test(const float* A, const float* B, float* D, int M, int N, int K) {
  __shared__ __align__(128) float sa[128 * 32];
  __shared__ __align__(128) float sb[32 * 32];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)), "r"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = t; i < M * K; i += blockDim.x) { int r = i / K, k = i % K; sa[kmaj_off(r, k, K)] = A[i]; }
  for (int i = t; i < N * K; i += blockDim.x) { int r = i / K, k = i % K; sb[kmaj_off(r, k, K)] = B[i]; }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tb = tmem_base;
  const uint32_t dcol = tb;         // D at columns [0, 32)
  const uint32_t acol = tb + 64;    // A (TS mode) at columns [64, 64+K)
  if (MODE == 1) {
    // each thread writes its A row (lane = row) into TMEM: K columns
    uint32_t v[32];
    for (int k = 0; k < 32; ++k) v[k] = (t < M && k < K) ? __float_as_uint(A[t * K + k]) : 0u;
    const uint32_t addr = acol + ((uint32_t)(warp * 32) << 16);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                 "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(addr),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]),
                 "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]),
                 "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]),
                 "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31]));
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (t == 0) {
    const uint32_t idesc = make_idesc(M, N);
    for (int ks = 0; ks < K / 8; ++ks) {
      // K-step ks covers k in [8ks, 8ks+8): 2 core matrices along K starting at (ks*2)*32 floats
      const uint64_t db = make_desc(sb + ks * 2 * 32, 128, (K / 4) * 128);
      const uint32_t acc = ks > 0 ? 1u : 0u;
      if (MODE == 0) {
        const uint64_t da = make_desc(sa + ks * 2 * 32, 128, (K / 4) * 128);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(dcol),
                     "l"(da), "l"(db), "r"(idesc), "r"(acc));
      } else {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(dcol),
                     "r"(acol + ks * 8), "l"(db), "r"(idesc), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
  }
  // wait for the MMA
  asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t r[32];
  const uint32_t addr = dcol + ((uint32_t)(warp * 32) << 16);
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                 "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                 "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
               : "r"(addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  if (t < M)
    for (int j = 0; j < N; ++j) D[t * N + j] = __uint_as_float(r[j]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(128));
}

static float tf32r(float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xffffe000u; float y; memcpy(&y, &u, 4); return y; }

int main() {
  const int M = 128, N = 24;
  int fails = 0;
  for (int mode = 0; mode < 2; ++mode)
    for (int K : {8, 32}) {
      float *hA = (float*)malloc(4 * M * K), *hB = (float*)malloc(4 * N * K), *hD = (float*)malloc(4 * M * N);
      srand(1 + K + mode);
      for (int i = 0; i < M * K; ++i) hA[i] = tf32r((float)(rand() % 1000) / 250.f - 2.f);
      for (int i = 0; i < N * K; ++i) hB[i] = tf32r((float)(rand() % 1000) / 300.f - 1.5f);
      float *dA, *dB, *dD;
      cudaMalloc(&dA, 4 * M * K); cudaMalloc(&dB, 4 * N * K); cudaMalloc(&dD, 4 * M * N);
      cudaMemcpy(dA, hA, 4 * M * K, cudaMemcpyHostToDevice);
      cudaMemcpy(dB, hB, 4 * N * K, cudaMemcpyHostToDevice);
      cudaMemset(dD, 0, 4 * M * N);
      if (mode == 0) k_test<0><<<1, 128>>>(dA, dB, dD, M, N, K); else k_test<1><<<1, 128>>>(dA, dB, dD, M, N, K);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(hD, dD, 4 * M * N, cudaMemcpyDeviceToHost);
      double maxerr = 0;
      for (int i = 0; i < M; ++i)
        for (int j = 0; j < N; ++j) {
          double s = 0;
          for (int k = 0; k < K; ++k) s += (double)hA[i * K + k] * hB[j * K + k];
          maxerr = fmax(maxerr, fabs(s - hD[i * N + j]));
        }
      printf("mode %s K=%d: %s maxerr %.3e  D[0][0]=%g D[77][5]=%g\n", mode ? "TS" : "SS", K, cudaGetErrorString(e), maxerr,
             hD[0], hD[77 * N + 5]);
      if (e != cudaSuccess || maxerr > 1e-3) ++fails;
      cudaFree(dA); cudaFree(dB); cudaFree(dD);
    }
  printf("%s\n", fails ? "FAILED" : "ALL OK");
  return fails;
}
