// Throughput microbenchmark for the pipes the FIF build/query/PC kernels use
// (FP32 FMA, FP64 FMA, MUFU ex2/rcp/rsq, FP64<->FP32 conversions, and mixes).
// Reports thread-ops per clock per SM. Not part of the product; design input.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 4096
#define CHAINS 8
template <int OP>
__global__ void kern(float* outf, double* outd, float seed, long long* clk) {
  float f[CHAINS]; double d[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) { f[c] = seed + threadIdx.x * 1e-3f + c; d[c] = f[c]; }
  long long t0 = clock64();
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      if (OP == 0) f[c] = fmaf(f[c], 0.999f, 0.001f);
      if (OP == 1) d[c] = fma(d[c], 0.999, 0.001);
      if (OP == 2) { float r; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(f[c])); f[c] = r; }
      if (OP == 3) { float r; asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(f[c])); f[c] = r; }
      if (OP == 4) { float r; asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(r) : "d"(d[c])); d[c] = (double)0 + __int_as_float(__float_as_int(r) ^ 1) ; }
      if (OP == 5) { double r; asm volatile("cvt.f64.f32 %0, %1;" : "=d"(r) : "f"(f[c])); f[c] = __int_as_float(__double2hiint(r) ^ 3); }
      if (OP == 6) { float r, s; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(f[c]));
                     asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(s) : "d"(d[c])); f[c] = r; d[c] = (double)0 + __int_as_float(__float_as_int(s) ^ 1); }
      if (OP == 7) { float r, s; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(f[c]));
                     asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(s) : "f"(r)); f[c] = s; }
      if (OP == 8) { float r; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(f[c])); f[c] = r;
                     d[c] = fma(d[c], 0.999, 0.001); }
      if (OP == 9) { float r; asm volatile("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(f[c])); f[c] = r; }
      if (OP == 10) { d[c] = __ddiv_rn(1.0, d[c]); }
      if (OP == 11) { float r; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(f[c]));
                      f[c] = fmaf(r, 0.999f, 0.001f); f[c] = fmaf(f[c], 0.999f, 0.001f); f[c] = fmaf(f[c], 0.999f, 0.001f); f[c] = fmaf(f[c], 0.999f, 0.001f);}
      if (OP == 12) { int x = __float_as_int(f[c]); x = __funnelshift_l(x, x ^ 7, 3) + 0x40000000; f[c] = __int_as_float(x); }
      if (OP == 14) { unsigned long long a, d; asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(f[c]), "f"(f[c] + 1.f));
                      asm volatile("fma.rn.f32x2 %0, %1, %1, %1;" : "=l"(d) : "l"(a));
                      float x, y; asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(d)); f[c] = x - y; }
      if (OP == 15) { unsigned long long a, b, d; asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(f[c]), "f"(f[c]));
                      b = a;
#pragma unroll
                      for (int r = 0; r < 4; ++r) { asm volatile("fma.rn.f32x2 %0, %1, %2, %1;" : "=l"(d) : "l"(a), "l"(b)); a = d; }
                      float x, y; asm("mov.b64 {%0, %1}, %2;" : "=f"(x), "=f"(y) : "l"(a)); f[c] = x + y; }
      if (OP == 13) { double r; asm volatile("cvt.f64.f32 %0, %1;" : "=d"(r) : "f"(f[c]));
                      float e; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(f[c])); f[c] = __int_as_float(__double2hiint(r) ^ 3) + e; }
    }
  }
  long long t1 = clock64();
  float sf = 0; double sd = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) { sf += f[c]; sd += d[c]; }
  outf[blockIdx.x * blockDim.x + threadIdx.x] = sf;
  outd[blockIdx.x * blockDim.x + threadIdx.x] = sd;
  if (threadIdx.x == 0 && blockIdx.x == 0) *clk = t1 - t0;
}
template <int OP>
void run(const char* name, int sms) {
  const int threads = 512, blocks = sms * 4;
  float* of; double* od; long long* clk;
  cudaMalloc(&of, sizeof(float) * threads * blocks);
  cudaMalloc(&od, sizeof(double) * threads * blocks);
  cudaMalloc(&clk, 8);
  kern<OP><<<blocks, threads>>>(of, od, 1.0f, clk);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<OP><<<blocks, threads>>>(of, od, 1.0f, clk);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  long long c; cudaMemcpy(&c, clk, 8, cudaMemcpyDeviceToHost);
  double ops = (double)threads * blocks * ITERS * CHAINS;
  int clkkhz; cudaDeviceGetAttribute(&clkkhz, cudaDevAttrClockRate, 0);
  // per-SM per-clock from wall time at the measured clock (approx via clock64 of block 0)
  double per_sm_per_clk_block0 = (double)threads * 4 * ITERS * CHAINS / c;  // 4 blocks/SM resident
  printf("%-28s  %8.3f ms  %10.3f Gop/s  ~%6.1f ops/clk/SM (clock64 basis)\n", name, ms, ops / ms / 1e6,
         per_sm_per_clk_block0);
  cudaFree(of); cudaFree(od); cudaFree(clk);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("SMs %d\n", sms);
  run<0>("FFMA", sms);
  run<1>("DFMA", sms);
  run<2>("MUFU.EX2", sms);
  run<3>("MUFU.RCP", sms);
  run<9>("MUFU.RSQ", sms);
  run<4>("F2F.F32.F64 (+LOP)", sms);
  run<5>("F2F.F64.F32 (+LOP)", sms);
  run<6>("EX2 + F2F.F32.F64", sms);
  run<13>("EX2 + F2F.F64.F32", sms);
  run<7>("EX2 + RCP", sms);
  run<8>("EX2 + DFMA", sms);
  run<11>("EX2 + 4 FFMA", sms);
  run<12>("SHF+IADD (ALU)", sms);
  run<10>("DDIV (__ddiv_rn)", sms);
  run<15>("4x FFMA2 (=8 FMA)", sms);
  return 0;
}
