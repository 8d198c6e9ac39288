// fif_gp_t5.cuh — GP info build on the 5th-generation tensor cores (tcgen05 + TMEM).
// Included by fif_build.cu (uses its pair_prologue / entries21 / voxel_split / h16_split2).
//
// Replaces _nb_build_gp's info branch (kernels.py:471-524): per voxel,
//   S[s][e] = sum_l vs(s, l) E(l, e)      (samples x landmarks) x (landmarks x 21 entries)
// with vs the GP sigmoids and E the packed 6x6 pair information (kernels.py:363-424);
// the reference's kinv @ S is applied at export / query time (field.py, fif_query.cu).
//
// One CTA (1 per SM) owns 3 voxels and streams 64-landmark tiles:
//  * 12 producer warps, thread = (voxel, landmark, sample half).  Each computes the pair's
//    bearing and weight once, then (half 0) the 21 entries and (both halves) its share of
//    the N_s sigmoids, splits every value into FP16 hi + lo, and stores 8 consecutive
//    entries / samples as one 16-byte vector into the MN-major UMMA operand tiles:
//      A (M = 64 rows): row 16 gi + 8 part + e % 8 holds part (hi/lo) of entry e = 8 gi + e % 8
//      B (N = 16 NG):   column s holds the hi sigmoid of sample s, column 8 NG + s the lo one
//    The sample directions (ax * zs, 3 x N_s floats) are kernel parameters, so the exponent
//    argument's FMAs take them straight from the constant bank.
//  * 1 MMA thread (warp 15) issues, per voxel and 16-landmark k-step, ONE
//    tcgen05.mma.kind::f16 M=64 N=16NG K=16 (FP32 accumulate in TMEM): the single product
//    [E_hi; E_lo] x [vs_hi, vs_lo]^T carries hi*hi, hi*lo, lo*hi (and lo*lo) in separate
//    accumulators, i.e. the 3-pass FP16 split of the mma.sync kernel in one instruction
//    (measured: M64 N144 K16 = 72 cycles; 4.5 cycles per pair vs the 8.75-cycle MUFU
//    floor of the sigmoids).  tcgen05.commit frees the stage's smem for the producers.
//  * 3 epilogue warps (TMEM sub-partitions 0-2 hold the 48 used D rows) drain a voxel's
//    accumulator every 512 landmarks (tcgen05.ld), add the four partial products in FP32
//    (hi/lo rows meet through one shuffle) and accumulate into FP64 sums in shared memory;
//    the voxels' flushes are staggered so the tensor pipe never waits on all three.
// FP16 range: entries are scaled by one exact power of two per voxel (a pre-pass bounds
// max |E| <= 2 w (1 + |p|^2) over the voxel's landmarks, so max|A'| < 2^14) and sigmoids
// by 2^12 (folded into the reciprocal's argument); values under FP16's normal range keep
// an absolute error <= 2^-37 max|E| per product, as in k_gp_info_h16.
#pragma once
// (included inside namespace fif)

#ifndef T5_VOX_N
#define T5_VOX_N 3                  // voxels per CTA (TMEM: 3 x 16 NG <= 480 of 512 columns)
#endif
#ifndef T5_STAGES_N
#define T5_STAGES_N 2
#endif
constexpr int T5_VOX = T5_VOX_N;
constexpr int T5_TILE = 64;         // landmarks per pipeline stage
constexpr int T5_KS = T5_TILE / 16; // MMAs per voxel per stage
constexpr int T5_STAGES = T5_STAGES_N;
constexpr int T5_FLUSH = 8;         // FP32 accumulation span: 8 tiles = 512 landmarks
#ifndef T5_PARTS
#define T5_PARTS 2                  // sample parts per (voxel, landmark) pair: one thread each
#endif
constexpr int T5_PWARPS = T5_VOX * T5_PARTS * 2;  // producer warps: voxels x parts x 2 landmark halves
// T5_DECOUPLE: the producer work is split by pipe.  The T5_PWARPS "sigmoid" warps compute
// only the (MUFU-heavy) sigmoids; T5_EWARPS "entry" warps, thread = (voxel, landmark), run
// one tile ahead: landmark load, the pair's bearing (handed to the sigmoid warps through a
// 2-slot shared-memory ring), the 21 entries and their A-tile stores (no MUFU).  Sharing an
// SM sub-partition, the two kinds overlap instead of meeting the XU pipe in lock step.
#ifndef T5_DECOUPLE
#define T5_DECOUPLE 0  // measured slower (139.3 vs 120.6 ms): DESIGN 8b
#endif
constexpr int T5_EWARPS = T5_DECOUPLE ? T5_VOX * 2 : 0;
// warp roles after the producers: 3 epilogue warps whose warp % 4 = 0, 1, 2 (the TMEM
// sub-partitions holding D rows 0-47) and one MMA warp, then the entry warps
constexpr int T5_EPI0 = (T5_PWARPS % 4 == 0) ? T5_PWARPS : ((T5_PWARPS + 1 + 3) / 4) * 4;
constexpr int T5_MMAW = (T5_PWARPS % 4 == 0) ? T5_PWARPS + 3 : T5_PWARPS;
constexpr int T5_E0 = T5_EPI0 + 3 + (T5_MMAW > T5_EPI0 ? 1 : 0);  // first entry warp
constexpr int T5_THREADS = (T5_E0 + T5_EWARPS) * 32;
static_assert(T5_MMAW < T5_EPI0 || T5_MMAW == T5_EPI0 + 3, "warp roles");
static_assert(!T5_DECOUPLE || T5_PARTS == 2, "decoupled producers: 2 sample parts");
constexpr int T5_NFULL = (T5_PWARPS + T5_EWARPS + 1) * 32;  // stage-full named barrier: writers + MMA warp
constexpr int T5_NU = (T5_PWARPS + T5_EWARPS) * 32;         // bearing-ring named barriers
constexpr int T5_MAX_NG = 10;       // N_s <= 80
constexpr int T5_BLK_A = 64 * 16 * 2;  // bytes per k-step of A (M = 64)

constexpr int T5_BAR_BYTES = 384;  // mbarriers (8 shared + 24 per-voxel), TMEM slot, scale bits (rounded up)
// PARTS = 4: part 0 shares each pair's bearing with parts 1-3 through shared memory
// ([stage][voxel][landmark] float4, after the barriers) and a named barrier per
// (voxel, landmark half, stage): ids 1 + T5_STAGES ...
#ifndef T5_SHARE_U
#define T5_SHARE_U (T5_PARTS >= 4 && !T5_DECOUPLE)  // part 0 computes each pair's bearing once for all parts
#endif
static_assert(!(T5_SHARE_U && T5_DECOUPLE), "T5_SHARE_U and T5_DECOUPLE are exclusive");
// bearing ring: [stage][voxel][landmark] float4 (SHARE_U: per pipeline stage; DECOUPLE: 2 slots)
constexpr int T5_USH_BYTES = T5_SHARE_U ? T5_STAGES * T5_VOX * T5_TILE * 16 : T5_DECOUPLE ? 2 * T5_VOX * T5_TILE * 16 : 0;
static_assert(1 + T5_STAGES + (T5_SHARE_U ? 2 * T5_VOX * T5_STAGES : 0) <= 16, "named barrier ids");
constexpr int T5_SMEM_MAX = 227 * 1024;  // opt-in shared memory per CTA on sm_100
struct __align__(16) T5Z {
  float z[3][8 * T5_MAX_NG];  // ax * zs[s][c] (T5_QUAD; else zs[s ^ 1][c], pairs swapped), FP32, 0 past N_s
};

__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  // no-swizzle canonical layout, sm100 descriptor version 1; MN-major operands:
  // LBO = stride between 8-deep K groups, SBO = stride between 8-wide M/N groups
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
// kind::f16 instruction descriptor: D FP32, A/B FP16, both MN-major, M = 64, N = 16 NG
template <int NG>
__host__ __device__ constexpr uint32_t t5_idesc() {
  return (1u << 4) | (1u << 15) | (1u << 16) | ((uint32_t)((16 * NG) >> 3) << 17) | ((uint32_t)(64 >> 4) << 24);
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t addr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(addr));
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// 16x32bx2 load of H consecutive columns per half-warp (second half at +H), H split into
// power-of-two chunks (x32 / x16 / x8 / x4 / x2 / x1)
template <int H, int C0 = 0>
__device__ __forceinline__ void tmem_ld_half(uint32_t addr, float* v) {
  if constexpr (C0 < H) {
    constexpr int REM = H - C0;
    constexpr int N = REM >= 32 ? 32 : REM >= 16 ? 16 : REM >= 8 ? 8 : REM >= 4 ? 4 : REM >= 2 ? 2 : 1;
    uint32_t* r = reinterpret_cast<uint32_t*>(v + C0);
    if constexpr (N == 32)
      asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                   "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32], %33;"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                     "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                     "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
                     "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
                     "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
                   : "r"(addr + C0), "n"(H));
    else if constexpr (N == 16)
      asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, "
                   "[%16], %17;"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                     "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
                     "=r"(r[15])
                   : "r"(addr + C0), "n"(H));
    else if constexpr (N == 8)
      asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                   : "r"(addr + C0), "n"(H));
    else if constexpr (N == 4)
      asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x4.b32 {%0,%1,%2,%3}, [%4], %5;"
                   : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                   : "r"(addr + C0), "n"(H));
    else if constexpr (N == 2)
      asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x2.b32 {%0,%1}, [%2], %3;"
                   : "=r"(r[0]), "=r"(r[1])
                   : "r"(addr + C0), "n"(H));
    else
      asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x1.b32 {%0}, [%1], %2;" : "=r"(r[0]) : "r"(addr + C0), "n"(H));
    tmem_ld_half<H, C0 + N>(addr, v);
  }
}

// hi/lo FP16 sigmoids 2^12 / (1 + 2^x), x = (ax z_s) . u + bx, for sample groups [G0, G1),
// stored as 16-byte vectors (8 samples) at column groups g (hi) and NG + g (lo)
#ifndef T5_ROTATE_ROLES
#define T5_ROTATE_ROLES 1
#endif
#ifndef T5_EPI_CHUNK
#define T5_EPI_CHUNK 1
#endif
#ifndef T5_NAMED
#define T5_NAMED 1
#endif
#ifndef T5_EPI_SLEEP
#define T5_EPI_SLEEP 2000
#endif
#ifndef T5_PROD_SLEEP
#define T5_PROD_SLEEP 64
#endif
#ifndef T5_MMA_SLEEP
#define T5_MMA_SLEEP 20
#endif
#ifndef T5_SLEEPWAIT
#define T5_SLEEPWAIT 1
#endif
// T5_PERVOX: every voxel of the CTA is its own pipeline: its 4 producer warps, stages and
// accumulator buffers have their own mbarriers ([voxel][stage / buffer]); the MMA thread
// polls them and issues a voxel's MMAs as soon as ITS stage is written, and the voxels'
// producers start T5_STAGGER_NS apart (the idea: one voxel's landmark load / prologue /
// stage wait overlaps the others' XU-bound sigmoid phase instead of all 12 warps meeting
// there).  Measured slower: 120.4 ms (stagger 300 or 600 ns), 121.1 ms (no stagger) vs
// 118.5 ms with the shared named barriers, rows bit-identical.
#ifndef T5_PERVOX
#define T5_PERVOX 0
#endif
#ifndef T5_STAGGER_NS
#define T5_STAGGER_NS 300
#endif
#ifndef T5_EARLY_PROBE
#define T5_EARLY_PROBE 0  // measured slower (121.3 vs 118.5 ms): DESIGN 8b
#endif
#ifndef T5_PIPE_PROLOGUE
#define T5_PIPE_PROLOGUE 0  // measured slower (121.0 vs 118.5 ms, 120 registers): DESIGN 8b
#endif
#ifndef T5_FAST_ISSUE
#define T5_FAST_ISSUE 1
#endif
#ifndef T5_XPAIR
#define T5_XPAIR 1
#endif
#ifndef T5_SPLIT_TRUNC
#define T5_SPLIT_TRUNC 1
#endif
#ifndef T5_SPLIT2
#define T5_SPLIT2 1
#endif
// FP16 hi + lo of two FP32 values.  T5_SPLIT_TRUNC: hi = x with its 13 low mantissa bits
// cleared (exactly representable in FP16 wherever FP16 is normal), lo = x - hi exact in
// FP32, both converted once -- the converted halves feed only the 16-byte operand stores,
// so they are allocated straight into the store's register quad (the round-to-nearest
// variant converts hi back to FP32 for the residual and needs register moves to build the
// quad).  |x - hi - lo16| <= 2^-21 |x| (2^-22 with round-to-nearest hi); below FP16's
// normal range both keep the absolute error <= 2^-25 (in scaled units).
// T5_SPLIT2: residuals as one packed FP32x2 subtraction.
__device__ __forceinline__ void t5_split2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
#if T5_SPLIT_TRUNC
  const float h0 = __uint_as_float(__float_as_uint(x0) & 0xFFFFE000u);
  const float h1 = __uint_as_float(__float_as_uint(x1) & 0xFFFFE000u);
  float d0, d1;
  unpack2(fsub2(pack2(x0, x1), pack2(h0, h1)), d0, d1);
  const __half2 h = __floats2half2_rn(h0, h1), l = __floats2half2_rn(d0, d1);
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
#else
  const __half2 h = __floats2half2_rn(x0, x1);
  const float2 b = __half22float2(h);
#if T5_SPLIT2
  float d0, d1;
  unpack2(fsub2(pack2(x0, x1), pack2(b.x, b.y)), d0, d1);
  const __half2 l = __floats2half2_rn(d0, d1);
#else
  const __half2 l = __floats2half2_rn(x0 - b.x, x1 - b.y);
#endif
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
#endif
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// polling with a sleep between probes (the epilogue waits ~7 000 cycles between flushes)
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity, unsigned ns) {
#if T5_SLEEPWAIT
  (void)ns;
  mbar_wait_sleep(bar, parity);
#else
  while (!mbar_try(bar, parity)) __nanosleep(ns);
#endif
}
// plain polling with a fixed sleep between probes (the suspending try_wait re-probes every
// few dozen cycles, which at 3 waiting warps cost ~4 % of the kernel's issue slots)
__device__ __forceinline__ void mbar_wait_poll(uint64_t* bar, uint32_t parity, unsigned ns) {
  while (!mbar_try(bar, parity)) __nanosleep(ns);
}
#ifndef T5_PROD_WAIT
#define T5_PROD_WAIT 0  // producers' stage-empty wait: 0 = poll + T5_PROD_SLEEP ns, 1 = suspending try_wait, 2 = spin
#endif
__device__ __forceinline__ void t5_prod_wait(uint64_t* bar, uint32_t parity) {
#if T5_PROD_WAIT == 1
  mbar_wait_sleep(bar, parity);
#elif T5_PROD_WAIT == 2
  while (!mbar_try(bar, parity)) {
  }
#else
  mbar_wait_poll(bar, parity, T5_PROD_SLEEP);
#endif
}
// named barriers: the producers arrive (no wait) and the MMA warp blocks in hardware
__device__ __forceinline__ void named_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
// T5_QUAD: one MUFU reciprocal per FOUR sigmoids.  With y_i = 2^-12 (1 + 2^x_i) (pairs
// (y0, y2) and (y1, y3) from two FFMA2), (y01, y23) = (y0 y1, y2 y3) is one FMUL2, r =
// 1 / (y01 y23), (a, b) = (y23 r, y01 r) one FMUL2, and the sigmoids 1 / y_i are
// (y1 a, y3 b) = (s0, s2) and (y0 a, y2 b) = (s1, s3), two FMUL2: 5 issue slots and one
// reciprocal per 4 samples instead of 4 and two (1.25 instead of 1.5 XU ops per sample).
// The product of four y stays finite for x <= 42 (y <= 2^31); the host selects this
// kernel only then.  Z holds the sample directions in order (no pair swap).
#ifndef T5_QUAD
#define T5_QUAD 0  // measured slower (123.0 vs 120.7 ms: the XU pipe is not what binds): DESIGN 8b
#endif
constexpr double T5_XMAX = T5_QUAD ? 42.0 : 60.0;  // host bound on bx + |ax|
// FP16 hi + lo of four sigmoids held as the pairs (s0, s2) and (s1, s3): hi = truncated
// (exact in FP16), lo = x - hi exact, residuals as two FADD2 on the pairs as they are
__device__ __forceinline__ void t5_split4(f32x2 s02, f32x2 s13, uint32_t& h01, uint32_t& h23, uint32_t& l01,
                                          uint32_t& l23) {
  float s0, s1, s2, s3;
  unpack2(s02, s0, s2);
  unpack2(s13, s1, s3);
  const float h0 = __uint_as_float(__float_as_uint(s0) & 0xFFFFE000u);
  const float h1 = __uint_as_float(__float_as_uint(s1) & 0xFFFFE000u);
  const float h2 = __uint_as_float(__float_as_uint(s2) & 0xFFFFE000u);
  const float h3 = __uint_as_float(__float_as_uint(s3) & 0xFFFFE000u);
  float d0, d1, d2, d3;
  unpack2(fsub2(s02, pack2(h0, h2)), d0, d2);
  unpack2(fsub2(s13, pack2(h1, h3)), d1, d3);
  const __half2 a = __floats2half2_rn(h0, h1), b = __floats2half2_rn(h2, h3);
  const __half2 c = __floats2half2_rn(d0, d1), d = __floats2half2_rn(d2, d3);
  h01 = *reinterpret_cast<const uint32_t*>(&a);
  h23 = *reinterpret_cast<const uint32_t*>(&b);
  l01 = *reinterpret_cast<const uint32_t*>(&c);
  l23 = *reinterpret_cast<const uint32_t*>(&d);
}
template <int NG, int G0, int G1>
__device__ __forceinline__ void t5_sigmoids(const T5Z& Z, float ux, float uy, float uz, float bx, uint32_t bdst) {
#if T5_QUAD
#pragma unroll
  for (int g = G0; g < G1; ++g) {
    uint32_t hv[4], lv[4];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int s0 = 8 * g + 4 * q;
      const f32x2 x01 = ffma2(splat2(ux), pack2(Z.z[0][s0], Z.z[0][s0 + 1]),
                              ffma2(splat2(uy), pack2(Z.z[1][s0], Z.z[1][s0 + 1]),
                                    ffma2(splat2(uz), pack2(Z.z[2][s0], Z.z[2][s0 + 1]), splat2(bx))));
      const f32x2 x23 = ffma2(splat2(ux), pack2(Z.z[0][s0 + 2], Z.z[0][s0 + 3]),
                              ffma2(splat2(uy), pack2(Z.z[1][s0 + 2], Z.z[1][s0 + 3]),
                                    ffma2(splat2(uz), pack2(Z.z[2][s0 + 2], Z.z[2][s0 + 3]), splat2(bx))));
      float x0, x1, x2, x3;
      unpack2(x01, x0, x1);
      unpack2(x23, x2, x3);
      const f32x2 y02 = ffma2(pack2(ex2_approx(x0), ex2_approx(x2)), splat2(0x1p-12f), splat2(0x1p-12f));
      const f32x2 y13 = ffma2(pack2(ex2_approx(x1), ex2_approx(x3)), splat2(0x1p-12f), splat2(0x1p-12f));
      float p01, p23;
      unpack2(fmul2(y02, y13), p01, p23);
      const float r = rcp_approx(p01 * p23);
      const f32x2 ab = fmul2(pack2(p23, p01), splat2(r));
      t5_split4(fmul2(y13, ab), fmul2(y02, ab), hv[2 * q], hv[2 * q + 1], lv[2 * q], lv[2 * q + 1]);
    }
    sts128(bdst + g * 128, hv[0], hv[1], hv[2], hv[3]);
    sts128(bdst + (NG + g) * 128, lv[0], lv[1], lv[2], lv[3]);
  }
#else
#pragma unroll
  for (int g = G0; g < G1; ++g) {
    uint32_t hv[4], lv[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int s0 = 8 * g + 2 * p;
#if T5_XPAIR
      const f32x2 x2 = ffma2(splat2(ux), pack2(Z.z[0][s0], Z.z[0][s0 + 1]),
                             ffma2(splat2(uy), pack2(Z.z[1][s0], Z.z[1][s0 + 1]),
                                   ffma2(splat2(uz), pack2(Z.z[2][s0], Z.z[2][s0 + 1]), splat2(bx))));
      float x0, x1;
      unpack2(x2, x0, x1);
#else
      const float x0 = fmaf(ux, Z.z[0][s0], fmaf(uy, Z.z[1][s0], fmaf(uz, Z.z[2][s0], bx)));
      const float x1 = fmaf(ux, Z.z[0][s0 + 1], fmaf(uy, Z.z[1][s0 + 1], fmaf(uz, Z.z[2][s0 + 1], bx)));
#endif
      float y0, y1;  // 2^-12 (1 + 2^x) for both, one FFMA2
      unpack2(ffma2(pack2(ex2_approx(x0), ex2_approx(x1)), splat2(0x1p-12f), splat2(0x1p-12f)), y0, y1);
      // one reciprocal for both sigmoids: r = 1 / (y0 y1), 1 / y1 = y0 r, 1 / y0 = y1 r (the
      // host launches this kernel only when x <= 60, so y0 y1 <= 2^98 stays finite; y >= 2^-12).
      // The host stores each sample pair's directions swapped in Z (x0 belongs to sample
      // s0 + 1), so (y0 r, y1 r) is (sigma(s0), sigma(s0 + 1)) in place: no register swap.
      const float r = rcp_approx(y0 * y1);
      float sg0, sg1;
      unpack2(fmul2(pack2(y0, y1), splat2(r)), sg0, sg1);
      t5_split2(sg0, sg1, hv[p], lv[p]);
    }
    sts128(bdst + g * 128, hv[0], hv[1], hv[2], hv[3]);
    sts128(bdst + (NG + g) * 128, lv[0], lv[1], lv[2], lv[3]);
  }
#endif
}

template <int NG, bool HAS_MASK>
__global__ void __launch_bounds__(T5_THREADS, 1)
k_gp_info_t5(const float4* __restrict__ lm, int64_t n_pad, VoxSrc src, int64_t v0, int64_t v1, int ns,
             const PairGate gate, int use_gbits, float inv_s2, float bx, const __grid_constant__ T5Z Z,
             double* __restrict__ out64, float* __restrict__ out32) {
  constexpr int NCOL = 16 * NG;                 // TMEM columns (and B rows) per voxel
  constexpr int BLK_B = NCOL * 16 * 2;          // bytes per k-step of B
  constexpr int STAGE_A = T5_KS * T5_BLK_A;     // bytes of one voxel's A tile
  constexpr int STAGE_B = T5_KS * BLK_B;
  constexpr int OFF_B = T5_STAGES * T5_VOX * STAGE_A;
  constexpr int OFF_ACC = OFF_B + T5_STAGES * T5_VOX * STAGE_B;
  constexpr int ACC_V = 8 * NG * 21;            // doubles per voxel
  constexpr int OFF_BAR = OFF_ACC + T5_VOX * ACC_V * 8;
  // sample-group boundaries of the parts; part 0 also computes the 21 entries (~ 13 samples of work)
  // (PARTS = 4: part 0's entries cost ~1.75 sample groups; the rest split over parts 1-3)
  constexpr int G1 = T5_PARTS == 1 ? NG : T5_PARTS == 2 ? NG / 2 : T5_PARTS == 3 ? (2 * NG + 4) / 9
                                                                   : (NG >= 6 ? (NG - 5 + 2) / 4 : 0);
  constexpr int G2 = T5_PARTS == 2 ? NG : T5_PARTS == 3 ? G1 + (NG - G1) * 3 / 7 : G1 + (NG - G1 + 2) / 3;
  constexpr int G3 = T5_PARTS == 4 ? G2 + (NG - G2 + 1) / 2 : NG;
  extern __shared__ __align__(1024) unsigned char smem[];
  double* acc = reinterpret_cast<double*>(smem + OFF_ACC);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* empty = full + T5_STAGES;
  uint64_t* ffull = empty + T5_STAGES;  // [2] accumulator buffer b holds a finished span
  uint64_t* fempty = ffull + 2;         // [2] the epilogue has drained buffer b
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(fempty + 2);
  int* sbits = reinterpret_cast<int*>(tmem_slot + 1);
  uint64_t* vfull = reinterpret_cast<uint64_t*>(smem + OFF_BAR + 128);  // T5_PERVOX: [voxel][stage]
  uint64_t* vempty = vfull + T5_VOX * T5_STAGES;
  uint64_t* vffull = vempty + T5_VOX * T5_STAGES;                        // [voxel][buffer]
  uint64_t* vfempty = vffull + T5_VOX * 2;
  static_assert(128 + 8 * (2 * T5_VOX * T5_STAGES + 4 * T5_VOX) <= T5_BAR_BYTES, "barrier bytes");
  constexpr bool PERVOX = T5_PERVOX && T5_FAST_ISSUE && !T5_PIPE_PROLOGUE && !T5_DECOUPLE && !T5_SHARE_U;
  // masked builds: the pre-pass evaluates each pair's matchability gate once and keeps the
  // answers as bits ([voxel][n_pad / 32] words) for the main loop (when they fit)
  float4* ush = reinterpret_cast<float4*>(smem + OFF_BAR + T5_BAR_BYTES);  // PARTS = 4 bearing share
  uint32_t* gbits = reinterpret_cast<uint32_t*>(smem + OFF_BAR + T5_BAR_BYTES + T5_USH_BYTES);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int64_t vbase = v0 + (int64_t)blockIdx.x * T5_VOX;
  const int ntiles = (int)(n_pad / T5_TILE);

  for (int i = t; i < T5_VOX * ACC_V; i += T5_THREADS) acc[i] = 0.0;
  if (t < T5_VOX) sbits[t] = 0;
  if (t == 0) {
    for (int s = 0; s < T5_STAGES; ++s) {
      mbar_init(&full[s], T5_PWARPS);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&ffull[b], 1);
      mbar_init(&fempty[b], 3);
    }
    for (int i = 0; i < T5_VOX * T5_STAGES; ++i) {
      mbar_init(&vfull[i], 2 * T5_PARTS);  // the voxel's producer warps
      mbar_init(&vempty[i], 1);
    }
    for (int i = 0; i < T5_VOX * 2; ++i) {
      mbar_init(&vffull[i], 1);
      mbar_init(&vfempty[i], 3);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();  // sbits zeroed before the pre-pass's atomicMax
  if (warp == T5_MMAW) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // producers: voxel centre, then the pre-pass bound on max |E| of their voxel
  // producer warp w: voxel pj = w / (2 PARTS); its role r (sample part, landmark half) is
  // rotated by the voxel so each SM sub-partition (w % 4) mixes heavy part-0 warps (entries +
  // their samples) with light ones instead of holding the same role for all three voxels
#if T5_ROTATE_ROLES
  const int prole = ((warp % (2 * T5_PARTS)) + warp / (2 * T5_PARTS)) % (2 * T5_PARTS);
#else
  const int prole = warp % (2 * T5_PARTS);
#endif
  const int pj = warp / (2 * T5_PARTS), ph = prole >> 1, pk = ((prole & 1) << 5) | lane;
  const int64_t pv = vbase + pj;
  const bool pvok = warp < T5_PWARPS && pv < v1;
  float ch[3] = {0.f, 0.f, 0.f}, cl[3] = {0.f, 0.f, 0.f};
  if (warp < T5_PWARPS) {
    voxel_split(src, pvok ? pv : v0, ch, cl);
    // Pre-pass: the voxel's bound 2 w (1 + |p|^2) >= 2 max|E| (|c2| <= |p|; the factor 2 also
    // covers the rounding of w = inv_s2 rsqrt(n^2)^2 in the build), w = inv_s2 / n^2, as
    // the fraction bn / bd = max (1 + |p|^2) / n^2 (no division per landmark); n^2 from the
    // same hi/lo difference as pair_prologue, the same skip rule.
    auto frac_update = [&](float4 a, float4 b, const float* c_h, const float* c_l, float& bn, float& bd) {
      const float dx = __fadd_rn(__fsub_rn(a.x, c_h[0]), __fsub_rn(b.x, c_l[0]));
      const float dy = __fadd_rn(__fsub_rn(a.y, c_h[1]), __fsub_rn(b.y, c_l[1]));
      const float dz = __fadd_rn(__fsub_rn(a.z, c_h[2]), __fsub_rn(b.z, c_l[2]));
      const float n2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
      const float num = 1.0f + a.w;
      if (n2 > 1e-30f && b.w != 0.f && num * bd > bn * n2) {
        bn = num;
        bd = n2;
      }
    };
    if (!HAS_MASK) {
      // unmasked: each producer thread loads a landmark once for all three voxels (a third
      // of the L2 traffic of per-voxel scans; the pre-pass is L2-bandwidth-bound)
      float vh[T5_VOX][3], vl[T5_VOX][3], bn[T5_VOX], bd[T5_VOX];
#pragma unroll
      for (int j = 0; j < T5_VOX; ++j) {
        voxel_split(src, vbase + j < v1 ? vbase + j : v0, vh[j], vl[j]);
        bn[j] = 0.f;
        bd[j] = 1.f;
      }
      constexpr int PT = T5_PWARPS * 32;
      for (int64_t i0 = warp * 32 + lane; i0 < n_pad; i0 += 2 * PT) {
        float4 a[2], b[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int64_t i = i0 + PT * u;
          a[u] = i < n_pad ? lm[2 * i] : make_float4(0.f, 0.f, 0.f, 0.f);
          b[u] = i < n_pad ? lm[2 * i + 1] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int j = 0; j < T5_VOX; ++j) frac_update(a[u], b[u], vh[j], vl[j], bn[j], bd[j]);
      }
#pragma unroll
      for (int j = 0; j < T5_VOX; ++j) {
        float mx = (vbase + j < v1 && bn[j] > 0.f) ? 2.0f * inv_s2 * __fdiv_rn(bn[j], bd[j]) : 0.f;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane == 0) atomicMax(&sbits[j], __float_as_int(mx));
      }
    } else {
      // masked: the voxel's own threads evaluate each pair's gate once (kept as bits)
      float mx = 0.f;
      if (pvok) {
        float bn = 0.f, bd = 1.f;
        constexpr int PT = 64 * T5_PARTS;  // pre-pass threads per voxel
        for (int64_t i0 = ph * 64 + pk; i0 < n_pad; i0 += 4 * PT) {
          float4 a[4], b[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int64_t i = i0 + PT * u;
            a[u] = i < n_pad ? lm[2 * i] : make_float4(0.f, 0.f, 0.f, 0.f);
            b[u] = i < n_pad ? lm[2 * i + 1] : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (b[u].w != 0.f && !gate_keep(gate, pv, i0 + PT * u)) b[u].w = 0.f;
            if (use_gbits) {  // warp = 32 consecutive landmarks: one word (none past n_pad: the
                              // next voxel's words follow)
              const unsigned wbits = __ballot_sync(0xffffffffu, b[u].w != 0.f);
              if (lane == 0 && i0 + PT * u < n_pad) gbits[pj * (n_pad >> 5) + ((i0 + PT * u) >> 5)] = wbits;
            }
            frac_update(a[u], b[u], ch, cl, bn, bd);
          }
        }
        mx = bn > 0.f ? 2.0f * inv_s2 * __fdiv_rn(bn, bd) : 0.f;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (lane == 0) atomicMax(&sbits[pj], __float_as_int(mx));
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  auto voxel_scale = [&](int j) {  // exact power of two with max|s E| < 2^14
    const int bits = sbits[j];
    if (bits <= 0) return 1.0f;
    const int ex = ((bits >> 23) & 0xff) - 127;
    return __int_as_float(min(254, max(1, 127 + 13 - ex)) << 23);
  };
  // FP32 accumulation spans: tiles [8k, 8k + 8) for every voxel (so a voxel's rounding does
  // not depend on which CTA, slab or centre list it lands in).  Span k accumulates in TMEM
  // buffer k & 1: an M = 64 MMA writes D rows to lanes 0-15 of each sub-partition, or to
  // lanes 16-31 with lane offset 16 in the D address (measured), so both buffers share the
  // voxel's 16 NG columns and the epilogue drains one while the tensor pipe fills the other.
  auto span_end = [&](int tt) { return (tt % T5_FLUSH) == T5_FLUSH - 1 || tt == ntiles - 1; };
  const uint32_t sbase = smem_u32(smem);

  if (T5_DECOUPLE && warp < T5_PWARPS) {
    // ───────────── sigmoid warps (decoupled producers) ─────────────
    const uint32_t kofs_b = (pk >> 4) * BLK_B + ((pk >> 3) & 1) * (256 * NG) + (pk & 7) * 16;
    for (int tt = 0; tt < ntiles; ++tt) {
      const int s = tt % T5_STAGES, u = tt & 1;
      named_sync(1 + T5_STAGES + u, T5_NU);  // the entry warps have written tile tt's bearings
      const float4 u4 = ush[(u * T5_VOX + pj) * T5_TILE + pk];
      named_arrive(3 + T5_STAGES + u, T5_NU);  // slot u may be refilled (tile tt + 2)
      if (tt >= T5_STAGES) t5_prod_wait(&empty[s], ((tt / T5_STAGES) - 1) & 1);
      const uint32_t bdst = sbase + OFF_B + (s * T5_VOX + pj) * STAGE_B + kofs_b;
      if (ph == 0)
        t5_sigmoids<NG, 0, G1>(Z, u4.x, u4.y, u4.z, bx, bdst);
      else
        t5_sigmoids<NG, G1, NG>(Z, u4.x, u4.y, u4.z, bx, bdst);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      named_arrive(1 + s, T5_NFULL);  // stage s: this warp's B columns written
    }
  } else if (T5_DECOUPLE && warp >= T5_E0) {
    // ───────────── entry warps: bearing, 21 entries, A tile (one tile ahead) ─────────────
    const int ew = warp - T5_E0, ej = ew >> 1, ek = ((ew & 1) << 5) | lane;
    const int64_t ev = vbase + ej;
    const bool evok = ev < v1;
    float ech[3], ecl[3];
    voxel_split(src, evok ? ev : v0, ech, ecl);
    const float inv_s2_s = inv_s2 * voxel_scale(ej);  // exact: a power of two
    const uint32_t kofs_a = (ek >> 4) * T5_BLK_A + ((ek >> 3) & 1) * 1024 + (ek & 7) * 16;
    float4 na = lm[2 * ek], nb = lm[2 * ek + 1];
    for (int tt = 0; tt < ntiles; ++tt) {
      const int s = tt % T5_STAGES, u = tt & 1;
      const float4 a = na;
      float4 b = nb;
      if (tt + 1 < ntiles) {
        const int64_t ni = (int64_t)(tt + 1) * T5_TILE + ek;
        na = lm[2 * ni];
        nb = lm[2 * ni + 1];
      }
      if (!evok) b.w = 0.f;
      if (HAS_MASK && b.w != 0.f) {
        const int64_t i = (int64_t)tt * T5_TILE + ek;
        const bool keep = use_gbits ? ((gbits[ej * (n_pad >> 5) + (i >> 5)] >> (i & 31)) & 1u) != 0
                                    : gate_keep(gate, ev, i);
        if (!keep) b.w = 0.f;
      }
      const PairF q = pair_prologue(a, b, ech, ecl, inv_s2_s);  // w (and every entry) carries the voxel scale
      if (tt >= 2) named_sync(3 + T5_STAGES + u, T5_NU);  // the sigmoid warps have read tile tt - 2
      ush[(u * T5_VOX + ej) * T5_TILE + ek] = make_float4(q.ux, q.uy, q.uz, 0.f);
      named_arrive(1 + T5_STAGES + u, T5_NU);
      float e[24];
      entries21(q, a, e);
      e[21] = e[22] = e[23] = 0.f;
      uint32_t hv[3][4], lv[3][4];
#pragma unroll
      for (int gi = 0; gi < 3; ++gi)
#pragma unroll
        for (int p = 0; p < 4; ++p) t5_split2(e[8 * gi + 2 * p], e[8 * gi + 2 * p + 1], hv[gi][p], lv[gi][p]);
      if (tt >= T5_STAGES) t5_prod_wait(&empty[s], ((tt / T5_STAGES) - 1) & 1);
      const uint32_t adst = sbase + (s * T5_VOX + ej) * STAGE_A + kofs_a;
#pragma unroll
      for (int gi = 0; gi < 3; ++gi) {
        sts128(adst + (2 * gi) * 128, hv[gi][0], hv[gi][1], hv[gi][2], hv[gi][3]);
        sts128(adst + (2 * gi + 1) * 128, lv[gi][0], lv[gi][1], lv[gi][2], lv[gi][3]);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      named_arrive(1 + s, T5_NFULL);  // stage s: this warp's A rows written
    }
    // consume the sigmoid warps' releases of the last two tiles (no barrier left half-arrived)
    for (int tt = ntiles > 2 ? ntiles : 2; tt < ntiles + 2; ++tt) named_sync(3 + T5_STAGES + (tt & 1), T5_NU);
  } else if (warp < T5_PWARPS) {
    // ───────────── producers ─────────────
    const float inv_s2_s = inv_s2 * voxel_scale(pj);  // exact: a power of two
    const uint32_t kofs_a = (pk >> 4) * T5_BLK_A + ((pk >> 3) & 1) * 1024 + (pk & 7) * 16;
    const uint32_t kofs_b = (pk >> 4) * BLK_B + ((pk >> 3) & 1) * (256 * NG) + (pk & 7) * 16;
#if T5_PIPE_PROLOGUE && T5_PARTS == 2 && !T5_SHARE_U
    // The pair prologue (landmark, gate, bearing: a dependent chain through rsqrt and its Newton
    // step) of tile tt + 1 sits in the middle of tile tt's sigmoid stream, where ptxas
    // interleaves it with independent work, instead of at the loop top where every warp of
    // the scheduler waits on it at the same time.
    auto prep = [&](int tile, float4 a, float4 b) {
      if (!pvok) b.w = 0.f;
      if (HAS_MASK && b.w != 0.f) {
        const int64_t i = (int64_t)tile * T5_TILE + pk;
        const bool keep = use_gbits ? ((gbits[pj * (n_pad >> 5) + (i >> 5)] >> (i & 31)) & 1u) != 0
                                    : gate_keep(gate, pv, i);
        if (!keep) b.w = 0.f;
      }
      return pair_prologue(a, b, ch, cl, inv_s2_s);  // w (and every entry) carries the voxel scale
    };
    float4 a_cur = lm[2 * pk];
    PairF q_cur = prep(0, a_cur, lm[2 * pk + 1]);
    float4 na = a_cur, nb = make_float4(0.f, 0.f, 0.f, 0.f);
    if (ntiles > 1) {
      na = lm[2 * (T5_TILE + pk)];
      nb = lm[2 * (T5_TILE + pk) + 1];
    }
    for (int tt = 0; tt < ntiles; ++tt) {
      const int s = tt % T5_STAGES;
      if (tt >= T5_STAGES) t5_prod_wait(&empty[s], ((tt / T5_STAGES) - 1) & 1);
      const float4 a_nxt = na, b_nxt = nb;  // tile tt + 1's landmark (loaded during tile tt - 1)
      if (tt + 2 < ntiles) {
        const int64_t ni = (int64_t)(tt + 2) * T5_TILE + pk;
        na = lm[2 * ni];
        nb = lm[2 * ni + 1];
      }
      const uint32_t adst = sbase + (s * T5_VOX + pj) * STAGE_A + kofs_a;
      const uint32_t bdst = sbase + OFF_B + (s * T5_VOX + pj) * STAGE_B + kofs_b;
      PairF q_nxt = q_cur;
      // (T5_PIPE_PROLOGUE == 2: after the tile's last store instead, where the sigmoid
      // temporaries are dead and the stores' completion, which the proxy fence waits for,
      // overlaps the prologue)
      if (ph == 0) {
        constexpr int GA = T5_PIPE_PROLOGUE == 2 ? 0 : G1 / 2;
        t5_sigmoids<NG, 0, GA>(Z, q_cur.ux, q_cur.uy, q_cur.uz, bx, bdst);
        if (T5_PIPE_PROLOGUE != 2 && tt + 1 < ntiles) q_nxt = prep(tt + 1, a_nxt, b_nxt);
        float e[24];
        entries21(q_cur, a_cur, e);
        e[21] = e[22] = e[23] = 0.f;
#pragma unroll
        for (int gi = 0; gi < 3; ++gi) {
          uint32_t hv[4], lv[4];
#pragma unroll
          for (int p = 0; p < 4; ++p) t5_split2(e[8 * gi + 2 * p], e[8 * gi + 2 * p + 1], hv[p], lv[p]);
          sts128(adst + (2 * gi) * 128, hv[0], hv[1], hv[2], hv[3]);
          sts128(adst + (2 * gi + 1) * 128, lv[0], lv[1], lv[2], lv[3]);
        }
        t5_sigmoids<NG, GA, G1>(Z, q_cur.ux, q_cur.uy, q_cur.uz, bx, bdst);
      } else {
        constexpr int GB = T5_PIPE_PROLOGUE == 2 ? G1 : G1 + (G2 - G1) / 2;
        t5_sigmoids<NG, G1, GB>(Z, q_cur.ux, q_cur.uy, q_cur.uz, bx, bdst);
        if (T5_PIPE_PROLOGUE != 2 && tt + 1 < ntiles) q_nxt = prep(tt + 1, a_nxt, b_nxt);
        t5_sigmoids<NG, GB, G2>(Z, q_cur.ux, q_cur.uy, q_cur.uz, bx, bdst);
      }
      if (T5_PIPE_PROLOGUE == 2 && tt + 1 < ntiles) q_nxt = prep(tt + 1, a_nxt, b_nxt);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
#if T5_NAMED
      named_arrive(1 + s, T5_NFULL);  // stage s written (the MMA warp syncs on it)
#else
      if (lane == 0) mbar_arrive(&full[s]);
#endif
      a_cur = a_nxt;
      q_cur = q_nxt;
    }
#else
    float4 na = lm[2 * pk], nb = lm[2 * pk + 1];
    if (PERVOX && T5_STAGGER_NS > 0 && pj > 0) __nanosleep(pj * T5_STAGGER_NS);
    for (int tt = 0; tt < ntiles; ++tt) {
      const int s = tt % T5_STAGES;
      // T5_EARLY_PROBE: the stage-empty barrier is probed before the pair prologue, so the
      // probe's own latency (a try_wait takes ~100 cycles to answer even when the phase is
      // complete) overlaps the prologue instead of following it
      uint64_t* ebar = PERVOX ? &vempty[pj * T5_STAGES + s] : &empty[s];
      bool stage_free = tt < T5_STAGES;
      if (T5_EARLY_PROBE && tt >= T5_STAGES) stage_free = mbar_try(ebar, ((tt / T5_STAGES) - 1) & 1);
      const float4 a = na;
      float4 b = nb;
      if (tt + 1 < ntiles) {
        const int64_t ni = (int64_t)(tt + 1) * T5_TILE + pk;
        na = lm[2 * ni];
        nb = lm[2 * ni + 1];
      }
      if (!pvok) b.w = 0.f;
      if (HAS_MASK && b.w != 0.f) {
        const int64_t i = (int64_t)tt * T5_TILE + pk;
        const bool keep = use_gbits ? ((gbits[pj * (n_pad >> 5) + (i >> 5)] >> (i & 31)) & 1u) != 0
                                    : gate_keep(gate, pv, i);
        if (!keep) b.w = 0.f;
      }
      PairF q;
      if (!T5_SHARE_U || ph == 0) q = pair_prologue(a, b, ch, cl, inv_s2_s);  // w (and every entry) carries the voxel scale
      if (!stage_free) t5_prod_wait(ebar, ((tt / T5_STAGES) - 1) & 1);
      if (T5_SHARE_U) {  // part 0 hands its bearing to the other parts (the slot is free: its last
                            // readers finished the tile whose MMA freed this stage)
        const int bid = 1 + T5_STAGES + ((pj * 2 + (pk >> 5)) * T5_STAGES + s);
        float4* slot = ush + (s * T5_VOX + pj) * T5_TILE + pk;
        if (ph == 0) {
          *slot = make_float4(q.ux, q.uy, q.uz, 0.f);
          __syncwarp();
          named_arrive(bid, 32 * T5_PARTS);
        } else {
          named_sync(bid, 32 * T5_PARTS);
          const float4 u4 = *slot;
          q.ux = u4.x, q.uy = u4.y, q.uz = u4.z, q.w = 0.f;
        }
      }
      const uint32_t adst = sbase + (s * T5_VOX + pj) * STAGE_A + kofs_a;
      const uint32_t bdst = sbase + OFF_B + (s * T5_VOX + pj) * STAGE_B + kofs_b;
      if (ph == 0) {
        float e[24];
        entries21(q, a, e);
        e[21] = e[22] = e[23] = 0.f;
#pragma unroll
        for (int gi = 0; gi < 3; ++gi) {
          uint32_t hv[4], lv[4];
#pragma unroll
          for (int p = 0; p < 4; ++p) t5_split2(e[8 * gi + 2 * p], e[8 * gi + 2 * p + 1], hv[p], lv[p]);
          sts128(adst + (2 * gi) * 128, hv[0], hv[1], hv[2], hv[3]);
          sts128(adst + (2 * gi + 1) * 128, lv[0], lv[1], lv[2], lv[3]);
        }
        t5_sigmoids<NG, 0, G1>(Z, q.ux, q.uy, q.uz, bx, bdst);
      } else if (T5_PARTS == 2 || ph == 1) {
        t5_sigmoids<NG, G1, G2>(Z, q.ux, q.uy, q.uz, bx, bdst);
      } else if (T5_PARTS == 3 || ph == 2) {
        t5_sigmoids<NG, G2, G3>(Z, q.ux, q.uy, q.uz, bx, bdst);
      } else {
        t5_sigmoids<NG, G3, NG>(Z, q.ux, q.uy, q.uz, bx, bdst);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (PERVOX) {
        if (lane == 0) mbar_arrive(&vfull[pj * T5_STAGES + s]);  // this warp's share of the voxel's stage
      } else {
#if T5_NAMED
        named_arrive(1 + s, T5_NFULL);  // stage s written (the MMA warp syncs on it)
#else
        if (lane == 0) mbar_arrive(&full[s]);
#endif
      }
    }
#endif  // T5_PIPE_PROLOGUE
  } else if (warp == T5_MMAW) {
    // ───────────── MMA issue (one thread) ─────────────
    // T5_FAST_ISSUE: the issuing thread is chosen by elect.sync (ptxas then keeps the operands
    // in uniform registers instead of a per-instruction R2UR waterfall) and the shared memory
    // descriptors are {loop-invariant low word + constant, constant high word} with the stage
    // unrolled: ~3 instead of ~21 instructions per MMA (the stage's release, tcgen05.commit
    // after the last MMA, is that much earlier).
    {
      constexpr uint32_t idesc = t5_idesc<NG>();
#if T5_FAST_ISSUE
      constexpr uint32_t HI = (128u >> 4) | (1u << 14);  // SBO = 128, descriptor version 1 (bit 46)
      const uint32_t sb4 = sbase >> 4;                   // (< 2^14: shared memory is < 256 KB)
      const uint32_t alo = sb4 | ((uint32_t)(1024 >> 4) << 16);
      const uint32_t blo = (sb4 + (OFF_B >> 4)) | ((uint32_t)((256 * NG) >> 4) << 16);
      auto issue = [&](auto stage, bool first, uint32_t dbase) {
        constexpr int S = decltype(stage)::value;
#pragma unroll
        for (int j = 0; j < T5_VOX; ++j)
#pragma unroll
          for (int ks = 0; ks < T5_KS; ++ks) {
            const uint32_t a = alo + (uint32_t)(((S * T5_VOX + j) * STAGE_A + ks * T5_BLK_A) >> 4);
            const uint32_t b = blo + (uint32_t)(((S * T5_VOX + j) * STAGE_B + ks * BLK_B) >> 4);
            const uint32_t accf = (!first || ks > 0) ? 1u : 0u;
            asm volatile("{\n\t.reg .pred p;\n\t.reg .b64 da, db;\n\tsetp.ne.b32 p, %5, 0;\n\t"
                         "mov.b64 da, {%1, %3};\n\tmov.b64 db, {%2, %3};\n\t"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %4, p;\n\t}" ::"r"(dbase + j * NCOL),
                         "r"(a), "r"(b), "r"(HI), "r"(idesc), "r"(accf));
          }
      };
#endif
#if T5_FAST_ISSUE
      if (PERVOX) {
        // one elected thread serves the three voxel pipelines round robin: the MMAs of a
        // voxel's tile as soon as its stage is written (and, for a span's first tile, its
        // accumulator buffer drained: never blocking on that, the other voxels need service)
        auto issue1 = [&](auto voxel, auto stage, bool first, uint32_t d) {
          constexpr int J = decltype(voxel)::value, S = decltype(stage)::value;
#pragma unroll
          for (int ks = 0; ks < T5_KS; ++ks) {
            const uint32_t a = alo + (uint32_t)(((S * T5_VOX + J) * STAGE_A + ks * T5_BLK_A) >> 4);
            const uint32_t b = blo + (uint32_t)(((S * T5_VOX + J) * STAGE_B + ks * BLK_B) >> 4);
            const uint32_t accf = (!first || ks > 0) ? 1u : 0u;
            asm volatile("{\n\t.reg .pred p;\n\t.reg .b64 da, db;\n\tsetp.ne.b32 p, %5, 0;\n\t"
                         "mov.b64 da, {%1, %3};\n\tmov.b64 db, {%2, %3};\n\t"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %4, p;\n\t}" ::"r"(d),
                         "r"(a), "r"(b), "r"(HI), "r"(idesc), "r"(accf));
          }
        };
        static_assert(!(T5_PERVOX && T5_FAST_ISSUE) || T5_STAGES == 2, "per-voxel pipelines: 2 stages");
        uint32_t elected;
        asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(elected));
        if (elected) {
          int st[T5_VOX];
#pragma unroll
          for (int j = 0; j < T5_VOX; ++j) st[j] = 0;
          int left = T5_VOX * ntiles;
          auto serve = [&](auto voxel) {
            constexpr int J = decltype(voxel)::value;
            const int tt = st[J], s = tt & 1;
            const int k = tt / T5_FLUSH, b = k & 1;
            const bool first = tt % T5_FLUSH == 0;
            if (!(tt < ntiles && mbar_try(&vfull[J * T5_STAGES + s], (tt >> 1) & 1) &&
                  (!first || k < 2 || mbar_try(&vfempty[J * 2 + b], ((k >> 1) - 1) & 1))))
              return false;
            tc_fence_after();
            const uint32_t d = tmem + ((uint32_t)(16 * b) << 16) + J * NCOL;
            if (s == 0)
              issue1(voxel, std::integral_constant<int, 0>{}, first, d);
            else
              issue1(voxel, std::integral_constant<int, 1>{}, first, d);
            if (span_end(tt))
              asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                               smem_u32(&vffull[J * 2 + b]))
                           : "memory");
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             smem_u32(&vempty[J * T5_STAGES + s]))
                         : "memory");
            ++st[J];
            --left;
            return true;
          };
          while (left > 0) {
            bool any = serve(std::integral_constant<int, 0>{});
            if constexpr (T5_VOX > 1) any |= serve(std::integral_constant<int, 1>{});
            if constexpr (T5_VOX > 2) any |= serve(std::integral_constant<int, 2>{});
            if (!any) __nanosleep(T5_MMA_SLEEP);
          }
        }
      } else
#endif
      for (int tt = 0; tt < ntiles; ++tt) {
        const int s = tt % T5_STAGES;
        const int k = tt / T5_FLUSH, b = k & 1;
        __syncwarp();
#if T5_NAMED
        named_sync(1 + s, T5_NFULL);  // all 32 lanes (bar.sync is warp-aligned)
#else
        mbar_wait_backoff(&full[s], (tt / T5_STAGES) & 1, T5_MMA_SLEEP);
#endif
        tc_fence_after();
#if T5_FAST_ISSUE
        uint32_t elected;
        asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(elected));
        if (elected) {
#else
        if (lane == 0) {  // one thread issues
#endif
          const bool first = tt % T5_FLUSH == 0;
          if (first && k >= 2) {  // buffer b last held span k - 2: drained long ago, normally
            mbar_wait_backoff(&fempty[b], ((k >> 1) - 1) & 1, T5_MMA_SLEEP);
            tc_fence_after();
          }
#if T5_FAST_ISSUE
          static_assert(T5_STAGES <= 3, "stage unrolling");
          const uint32_t dbase = tmem + ((uint32_t)(16 * b) << 16);
          if (s == 0)
            issue(std::integral_constant<int, 0>{}, first, dbase);
          else if (s == 1)
            issue(std::integral_constant<int, 1>{}, first, dbase);
          else
            issue(std::integral_constant<int, T5_STAGES - 1>{}, first, dbase);
#else
#pragma unroll
          for (int j = 0; j < T5_VOX; ++j) {
            const uint32_t a0 = sbase + (s * T5_VOX + j) * STAGE_A;
            const uint32_t b0 = sbase + OFF_B + (s * T5_VOX + j) * STAGE_B;
            const uint32_t d = tmem + ((uint32_t)(16 * b) << 16) + j * NCOL;
#pragma unroll
            for (int ks = 0; ks < T5_KS; ++ks) {
              const uint64_t da = umma_desc(a0 + ks * T5_BLK_A, 1024, 128);
              const uint64_t db = umma_desc(b0 + ks * BLK_B, 256 * NG, 128);
              const uint32_t accf = (!first || ks > 0) ? 1u : 0u;
              asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                           "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                           "l"(da), "l"(db), "r"(idesc), "r"(accf));
            }
          }
#endif
          if (span_end(tt))
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             smem_u32(&ffull[b]))
                         : "memory");
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                           smem_u32(&empty[s]))
                       : "memory");
        }
      }
    }
    __syncwarp();
  } else if (warp >= T5_EPI0 && warp < T5_EPI0 + 3) {
    // ───────────── epilogue: TMEM -> FP64 sums (warps 12-14 = sub-partitions 0-2) ─────────────
    // 16x32bx2 loads: lane L < 16 reads D row 16 sp + L, columns [0, H) of a sample block,
    // lane 16 + L the same row's columns [H, 2H) (H = 4 NG): the whole snapshot (hi and lo
    // sample columns) lands in registers with one wait, the accumulator is released, and
    // the FP64 accumulation runs while the tensor pipe refills it.
    constexpr int H = 4 * NG;
    const int sp = warp & 3;
    const int L = lane & 15, part = L >> 3, e = 8 * sp + (L & 7), q = lane >> 4;
    const bool row_ok = e < 21;
    const int nspans = (ntiles + T5_FLUSH - 1) / T5_FLUSH;
    for (int k = 0; k < nspans; ++k) {
      const int b = k & 1;
      if (!PERVOX) {
        mbar_wait_poll(&ffull[b], (k >> 1) & 1, T5_EPI_SLEEP);
        tc_fence_after();
      }
#pragma unroll 1
      for (int j = 0; j < T5_VOX; ++j) {
        if (PERVOX) {
          mbar_wait_poll(&vffull[j * 2 + b], (k >> 1) & 1, T5_EPI_SLEEP);
          tc_fence_after();
        }
        const uint32_t row = tmem + ((uint32_t)(32 * sp + 16 * b) << 16) + j * NCOL;
        double* aj = acc + j * ACC_V;
#if T5_EPI_CHUNK
        // 4 columns per load pair: few registers (the buffer is not needed again for 8 tiles)
#pragma unroll 1
        for (int c0 = 0; c0 < H; c0 += 4) {
          uint32_t hr[4], lr[4];
          asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x4.b32 {%0,%1,%2,%3}, [%4], %5;"
                       : "=r"(hr[0]), "=r"(hr[1]), "=r"(hr[2]), "=r"(hr[3]) : "r"(row + c0), "n"(H));
          asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x4.b32 {%0,%1,%2,%3}, [%4], %5;"
                       : "=r"(lr[0]), "=r"(lr[1]), "=r"(lr[2]), "=r"(lr[3]) : "r"(row + 8 * NG + c0), "n"(H));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            float v = __uint_as_float(hr[i]) + __uint_as_float(lr[i]);
            v += __shfl_xor_sync(0xffffffffu, v, 8);
            const int sm = q * H + c0 + i;
            if ((i & 1) == part && row_ok && sm < ns) aj[sm * 21 + e] += (double)v;
          }
        }
#else
        float hi[H], lo[H];
        tmem_ld_half<H>(row, hi);
        tmem_ld_half<H>(row + 8 * NG, lo);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int i = 0; i < H; ++i) {
          float v = hi[i] + lo[i];
          v += __shfl_xor_sync(0xffffffffu, v, 8);  // + the other part's row (entry hi / lo)
          const int sm = q * H + i;
          if ((i & 1) == part && row_ok && sm < ns) aj[sm * 21 + e] += (double)v;  // unscaled (exact 2^k at the end)
        }
#endif
        if (PERVOX) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&vfempty[j * 2 + b]);
        }
      }
      if (!PERVOX) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&fempty[b]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // write the voxels' FP64 sums (and the FP32 query copy)
  const int per = ns * 21;
  for (int i = t; i < T5_VOX * per; i += T5_THREADS) {
    const int j = i / per, r = i - j * per;
    const int64_t v = vbase + j;
    if (v >= v1) continue;
    const double x = acc[j * ACC_V + r] * (0x1p-12 / (double)voxel_scale(j));  // exact power of two
    out64[(v - v0) * per + r] = x;
    if (out32) out32[(v - v0) * per + r] = (float)x;
  }
  if (warp == T5_MMAW) {
    __syncwarp();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int NG>
constexpr size_t t5_smem_bytes() {  // without the gate bits (T5_VOX * n_pad / 8 bytes more when used)
  return (size_t)T5_STAGES * T5_VOX * T5_KS * (T5_BLK_A + 16 * NG * 16 * 2) + (size_t)T5_VOX * 8 * NG * 21 * 8 +
         T5_BAR_BYTES + T5_USH_BYTES;
}

