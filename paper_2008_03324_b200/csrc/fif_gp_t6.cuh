// fif_gp_t6.cuh — GP info build on tcgen05 with the sigmoid exponent arguments ALSO on the
// tensor cores (FIF_BUILD_T6; a measured alternative to the default k_gp_info_t5, see the
// result at the end).  Included by fif_build.cu after fif_gp_t5.cuh (shares its helpers).
//
// k_gp_info_t5 spends, per (pair, sample), 1.5 FFMA2 + a constant-bank load on the exponent
// argument x = (ax z_s) . u + bx and computes every pair's bearing twice (once per sample
// part): ~20 % of its issue slots.  Here
//   X[l][s] = sum_c u_c(l) (ax z_s)_c                    (landmarks x 3) x (3 x samples)
// is one more tcgen05.mma per (voxel, 64-landmark tile): kind::f16, M = 128, N = 16-aligned
// 8 NG, K = 16, FP32 accumulate.  The K = 16 slots carry the FP16 splits u = uh + ul (22
// bits) and ax z = zh + zm + zl (33 bits, host-made): uh zh, uh zm, uh zl, ul zh, ul zm (15
// products; everything dropped is < 2^-30 |x|).  The bias moves into the sigmoid's FFMA2:
//   2^-12 (1 + 2^(x' + bx)) = fma(2^x', 2^(bx - 12), 2^-12).
// Rows: A_x row 32 sp + lane belongs to the producer thread of TMEM sub-partition sp, so the
// 64 landmarks of a tile appear twice (once per sample part) and each thread reads ITS x
// values with one 32x32b tcgen05.ld of its own lane (32-40 columns) — no FFMA2, no constant
// loads.  The pair's bearing for tile t + 1 is computed during tile t (while the X loads of
// tile t are in flight), written K-major into the voxel's single A_x slot, and the MMA thread
// issues X(t + 1) once the voxel's four warps have X(t) in registers.
//
// TMEM (512 columns): S accumulators 3 x XN, X 3 x XN (XN = 80 at N_s = 70): X cannot be
// double-buffered.  To fit even that, the S product drops the separate hi/lo sample columns of
// k_gp_info_t5: per k-step TWO N = 8 NG MMAs accumulate into the same 48 D rows,
//   [E_lo; E_hi; 0] x vs_hi  and  [E_hi; 0; ...] x vs_lo
// (A tile K-group = [lo0 lo1 lo2 hi0 hi1 hi2 Z Z Z] x 128 B; the second MMA's descriptor
// starts at hi0, so its rows 24-47 read the zero groups and rows 48-63, never read back,
// run into the next K-group), i.e. rows 0-23 = E_lo vs_hi + E_hi vs_lo, rows 24-47 = E_hi
// vs_hi (lo x lo, <= 2^-22 relative, is dropped as in k_gp_info_h16).  The two rows of an
// entry sit in different epilogue warps; the warps walk the voxels in rotated order so that
// no FP64 cell has two writers at a time.
// Every voxel is its own pipeline (own stages, mbarriers, X and S columns); one elected
// thread polls the barriers and issues all MMAs (descriptors = loop-invariant low word +
// constant, ~3 instructions per MMA).  3 voxels per CTA, 64-landmark stages, 12 producer
// warps, lane-offset TMEM double buffering of the S spans, FP16 hi + lo by truncation, one
// reciprocal per pair of sigmoids and aligned 512-landmark FP32 spans are k_gp_info_t5's.
//
// Result (config 2, GP-70, B200): same precision as t5 (max-entry / voxel-Frobenius 1.15e-6
// vs 1.08e-6), 17 % fewer warp instructions, the sigmoid phase XU-saturated (1 220 cycles
// per tile vs ~2 200), but 135.4 ms vs 120.6 ms: with one X buffer the chain "X(t) read ->
// A_x(t + 1) -> barrier -> MMA thread -> in-order tensor queue -> X(t + 1) landed" (plus its
// extra proxy fences) is exposed once per tile, and the producers wait ~20 % of their time
// for X (profiles/r02_t6_*.txt, DESIGN 8b).
#pragma once
// (included inside namespace fif)

#ifndef T6_DEBUG
#define T6_DEBUG 0  // waits report their state and trap when nothing happens for a long time
#endif

#ifndef T6_G1_N
#define T6_G1_N 1
#define T6_G1_D 2
#endif
#define T6_G1(NG) ((NG) * T6_G1_N / T6_G1_D)  // sample groups of part 0 (which also computes the 21 entries)
#ifndef T6_X_FIRST
#define T6_X_FIRST 1
#endif
#ifndef T6_PROBE
#define T6_PROBE 0  // timing probes (wrong results): 1 = no second S MMA, 2 = no FP64 adds in the epilogue,
                    // 3 = producers do not wait for X, 4 = empty epilogue, 5 = no S MMAs
#endif
constexpr int T6_KG_A = 9 * 128;        // bytes per K-group of A: [lo0 lo1 lo2 hi0 hi1 hi2 Z Z Z]
constexpr int T6_BLK_A = 2 * T6_KG_A;   // bytes per k-step of A
constexpr int T6_AX_BYTES = 128 * 32;   // A_x per voxel: 128 rows x K = 16 halves, K-major
constexpr int T6_MAX_NG = 9;            // shared memory: N_s <= 72
constexpr int T6_XN_MAX = 80;
constexpr int T6_EPIBAR = 1;            // named barrier of the three epilogue warps
constexpr int T6_BAR_BYTES = 384;       // 30 mbarriers, TMEM slot, scale bits
#ifndef T6_STAGGER_NS
#define T6_STAGGER_NS 300  // start delay of voxel j's producers: j x this (de-phases the voxels' pipelines)
#endif
static_assert(T5_VOX == 3 && T5_PARTS == 2 && T5_STAGES == 2 && !T5_DECOUPLE && T5_PWARPS == 12,
              "k_gp_info_t6 is written for 3 voxels x 2 sample parts x 2 stages");

// B_x: the sample directions ax z_s as FP16 zh + zm + zl in the K-major UMMA layout
// (element (n, k) at (n / 8) 256 + (k / 8) 128 + (n % 8) 16 + (k % 8) 2 bytes), K slots
//   [zh.x zh.y | zh.z zh.z | zm.x zm.y | zm.z zm.z || zl.x zl.y | zl.z 0 | zh.x zh.y | zm.x zm.y]
// against the A_x row [A B A B | A B C C], A = (uh.x, uh.y), B = (uh.z, ul.z), C = (ul.x, ul.y).
struct __align__(16) T6Z {
  uint4 v[2 * T6_XN_MAX];
};

__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// 32x32b load of N consecutive columns of this thread's TMEM lane, split into x32 / x16 / x8 chunks
template <int N, int C0 = 0>
__device__ __forceinline__ void tmem_ld_row(uint32_t addr, uint32_t* r) {
  if constexpr (C0 < N) {
    constexpr int REM = N - C0;
    constexpr int W = REM >= 32 ? 32 : REM >= 16 ? 16 : 8;
    static_assert(REM % 8 == 0, "whole sample groups");
    uint32_t* p = r + C0;
    if constexpr (W == 32)
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
                   "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
                   : "=r"(p[0]), "=r"(p[1]), "=r"(p[2]), "=r"(p[3]), "=r"(p[4]), "=r"(p[5]), "=r"(p[6]), "=r"(p[7]),
                     "=r"(p[8]), "=r"(p[9]), "=r"(p[10]), "=r"(p[11]), "=r"(p[12]), "=r"(p[13]), "=r"(p[14]),
                     "=r"(p[15]), "=r"(p[16]), "=r"(p[17]), "=r"(p[18]), "=r"(p[19]), "=r"(p[20]), "=r"(p[21]),
                     "=r"(p[22]), "=r"(p[23]), "=r"(p[24]), "=r"(p[25]), "=r"(p[26]), "=r"(p[27]), "=r"(p[28]),
                     "=r"(p[29]), "=r"(p[30]), "=r"(p[31])
                   : "r"(addr + C0));
    else if constexpr (W == 16)
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : "=r"(p[0]), "=r"(p[1]), "=r"(p[2]), "=r"(p[3]), "=r"(p[4]), "=r"(p[5]), "=r"(p[6]), "=r"(p[7]),
                     "=r"(p[8]), "=r"(p[9]), "=r"(p[10]), "=r"(p[11]), "=r"(p[12]), "=r"(p[13]), "=r"(p[14]),
                     "=r"(p[15])
                   : "r"(addr + C0));
    else
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                   : "=r"(p[0]), "=r"(p[1]), "=r"(p[2]), "=r"(p[3]), "=r"(p[4]), "=r"(p[5]), "=r"(p[6]), "=r"(p[7])
                   : "r"(addr + C0));
    tmem_ld_row<N, C0 + W>(addr, r);
  }
}

// kind::f16 instruction descriptors: D FP32, A/B FP16
template <int NG>
__host__ __device__ constexpr uint32_t t6_idesc_s() {  // S: both MN-major, M = 64, N = 8 NG
  return (1u << 4) | (1u << 15) | (1u << 16) | ((uint32_t)((8 * NG) >> 3) << 17) | ((uint32_t)(64 >> 4) << 24);
}
template <int XN>
__host__ __device__ constexpr uint32_t t6_idesc_x() {  // X: both K-major, M = 128, N = XN
  return (1u << 4) | ((uint32_t)(XN >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void t6_mma(uint32_t d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t accf) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
               "l"(da), "l"(db), "r"(idesc), "r"(accf));
}
// the same with the descriptors as {low word, high word}: the high word is a constant
__device__ __forceinline__ void t6_mma_lo(uint32_t d, uint32_t a_lo, uint32_t b_lo, uint32_t hi, uint32_t idesc,
                                          uint32_t accf) {
  asm volatile("{\n\t.reg .pred p;\n\t.reg .b64 da, db;\n\tsetp.ne.b32 p, %5, 0;\n\t"
               "mov.b64 da, {%1, %3};\n\tmov.b64 db, {%2, %3};\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], da, db, %4, p;\n\t}" ::"r"(d),
               "r"(a_lo), "r"(b_lo), "r"(hi), "r"(idesc), "r"(accf));
}
// one elected thread of a converged warp (elect.sync: ptxas keeps the guarded region's
// operands in uniform registers instead of a per-instruction R2UR waterfall loop)
#ifndef T6_ELECT
#define T6_ELECT 1
#endif
__device__ __forceinline__ bool t6_elect(int lane) {
#if T6_ELECT
  uint32_t pred;
  asm volatile("{\n\t.reg .pred p;\n\telect.sync _|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(pred));
  return pred != 0;
#else
  return lane == 0;
#endif
}
__device__ __forceinline__ void t6_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// hi/lo FP16 sigmoids 2^12 / (1 + 2^(x' + bx)) of sample groups [G0, G1) from the X values in
// registers (column c of X holds sample c ^ 1, so the paired reciprocal's products come out
// in sample order, as in t5_sigmoids); cexp = 2^(bx - 12).  SKIP trailing sample pairs of the
// last group are padding (columns >= N_s, never read back) and are not computed.
// With every x already in registers nothing orders the transcendentals, and the compiler
// hoists all the ex2 of a tile into one burst that floods the XU queue while the FMA pipe
// idles.  The pairs are therefore software-pipelined by hand in three stages (ex2 of pair
// i + 2, reciprocal of pair i + 1, split + store of pair i) with the MUFU instructions as
// volatile asm, which keeps their program order: ex2 ex2 rcp ex2 ex2 rcp ...
__device__ __forceinline__ float ex2_approx_v(float x) {
  float r;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rcp_approx_v(float x) {
  float r;
  asm volatile("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// spin on an mbarrier phase; T6_DEBUG: report and trap instead of hanging
__device__ __forceinline__ void t6_spin(uint64_t* bar, uint32_t parity, int tag, int a, int b) {
#if T6_DEBUG
  long long n = 0;
  while (!mbar_try(bar, parity)) {
    if (++n > 20000000) {
      if ((threadIdx.x & 31) == 0) printf("t6 stuck tag %d block %d warp %d: %d %d\n", tag, blockIdx.x, threadIdx.x >> 5, a, b);
      __trap();
    }
  }
#else
  (void)tag, (void)a, (void)b;
  while (!mbar_try(bar, parity)) {
  }
#endif
}
#ifndef T6_PIPE
#define T6_PIPE 1
#endif
template <int NG, int G0, int G1, int SKIP>
__device__ __forceinline__ void t6_sigmoids(const uint32_t* xr, float cexp, uint32_t bdst) {
  constexpr int NP = 4 * (G1 - G0) - (G1 == NG ? SKIP : 0);  // sample pairs to compute
  static_assert(SKIP >= 0 && SKIP < 4, "padding pairs of the last group");
#if T6_PIPE
  float ea[3], eb[3], r[2];
  f32x2 y[2];
  uint32_t hv[4], lv[4];
#pragma unroll
  for (int st = 0; st < NP + 2; ++st) {
    if (st < NP) {  // stage A: both ex2 of pair st
      ea[st % 3] = ex2_approx_v(__uint_as_float(xr[2 * st]));
      eb[st % 3] = ex2_approx_v(__uint_as_float(xr[2 * st + 1]));
    }
    if (st >= 1 && st - 1 < NP) {  // stage B: y = 2^-12 (1 + 2^x), one reciprocal for the pair
      const int p = st - 1;
      y[p % 2] = ffma2(pack2(ea[p % 3], eb[p % 3]), splat2(cexp), splat2(0x1p-12f));
      float y0, y1;
      unpack2(y[p % 2], y0, y1);
      r[p % 2] = rcp_approx_v(y0 * y1);
    }
    if (st >= 2) {  // stage C: sigmoids, FP16 hi + lo, store per group of 8 samples
      const int p = st - 2;
      float sg0, sg1;
      unpack2(fmul2(y[p % 2], splat2(r[p % 2])), sg0, sg1);
      t5_split2(sg0, sg1, hv[p % 4], lv[p % 4]);
      if (p % 4 == 3 || p == NP - 1) {
#pragma unroll
        for (int i = p % 4 + 1; i < 4; ++i) hv[i] = lv[i] = 0u;
        const int g = G0 + p / 4;
        sts128(bdst + g * 128, hv[0], hv[1], hv[2], hv[3]);
        sts128(bdst + (NG + g) * 128, lv[0], lv[1], lv[2], lv[3]);
      }
    }
  }
#else
#pragma unroll
  for (int g = G0; g < G1; ++g) {
    uint32_t hv[4], lv[4];
#pragma unroll
    for (int p = 0; p < 4; ++p) {
      const int c = 8 * (g - G0) + 2 * p;
      if (4 * (g - G0) + p >= NP) {  // padded pair: never read back
        hv[p] = 0u;
        lv[p] = 0u;
        continue;
      }
      float y0, y1;
      unpack2(ffma2(pack2(ex2_approx(__uint_as_float(xr[c])), ex2_approx(__uint_as_float(xr[c + 1]))), splat2(cexp),
                    splat2(0x1p-12f)),
              y0, y1);
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

template <int NG>
struct T6Layout {
  static constexpr int NCOL = 8 * NG;                    // S columns per voxel (N of the S MMAs)
  static constexpr int XN = (NCOL + 15) / 16 * 16;       // X columns per voxel; TMEM column stride of S and X
  static constexpr int BLK_B = 2 * NCOL * 16 * 2;        // bytes per k-step of B ([vs_hi | vs_lo] column groups)
  static constexpr int STAGE_A = T5_KS * T6_BLK_A;
  static constexpr int STAGE_B = T5_KS * BLK_B;
  static constexpr int OFF_B = T5_STAGES * T5_VOX * STAGE_A;
  static constexpr int OFF_ACC = OFF_B + T5_STAGES * T5_VOX * STAGE_B;
  static constexpr int ACC_V = NCOL * 21;                // doubles per voxel
  static constexpr int OFF_BAR = OFF_ACC + T5_VOX * ACC_V * 8;
  static constexpr int OFF_AX = OFF_BAR + T6_BAR_BYTES;
  static constexpr int OFF_BX = OFF_AX + T5_VOX * T6_AX_BYTES;
  static constexpr int BYTES = OFF_BX + XN * 32;
  static constexpr int XBASE = T5_VOX * XN;              // first X column
  static_assert(2 * T5_VOX * XN <= 512, "TMEM columns");
  static_assert(OFF_B % 16 == 0 && OFF_AX % 16 == 0 && OFF_BX % 16 == 0 && OFF_ACC % 8 == 0, "alignment");
};

template <int NG, int SKIP>
__global__ void __launch_bounds__(T5_THREADS, 1)
k_gp_info_t6(const float4* __restrict__ lm, int64_t n_pad, VoxSrc src, int64_t v0, int64_t v1, int ns, float inv_s2,
             float cexp, const __grid_constant__ T6Z Z, double* __restrict__ out64, float* __restrict__ out32) {
  using LY = T6Layout<NG>;
  constexpr int XN = LY::XN, BLK_B = LY::BLK_B, STAGE_A = LY::STAGE_A, STAGE_B = LY::STAGE_B;
  constexpr int OFF_B = LY::OFF_B, OFF_ACC = LY::OFF_ACC, ACC_V = LY::ACC_V, OFF_BAR = LY::OFF_BAR;
  constexpr int OFF_AX = LY::OFF_AX, OFF_BX = LY::OFF_BX, XBASE = LY::XBASE;
  constexpr int G1 = T6_G1(NG);
  static_assert(G1 >= 1 && G1 < NG, "both sample parts need at least one group");
  extern __shared__ __align__(1024) unsigned char smem[];
  double* acc = reinterpret_cast<double*>(smem + OFF_ACC);
  // Every voxel of the CTA is its own pipeline (4 producer warps, its stages, its X and S
  // columns) with its own mbarriers, [voxel][stage / buffer]; the MMA thread polls them:
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + OFF_BAR);  // [3][2] stage written by the voxel's 4 warps
  uint64_t* empty = full + T5_VOX * 2;                           // [3][2] stage consumed by the S MMAs
  uint64_t* ffull = empty + T5_VOX * 2;                          // [3][2] accumulator buffer b holds a finished span
  uint64_t* fempty = ffull + T5_VOX * 2;                         // [3][2] the epilogue has drained buffer b
  uint64_t* axr = fempty + T5_VOX * 2;                           // [3] X(t - 1) read and A_x(t) written by the 4 warps
  uint64_t* xfull = axr + T5_VOX;                                // [3] X(t) has landed in TMEM
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xfull + T5_VOX);
  int* sbits = reinterpret_cast<int*>(tmem_slot + 1);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int64_t vbase = v0 + (int64_t)blockIdx.x * T5_VOX;
  const int ntiles = (int)(n_pad / T5_TILE);

  for (int i = t; i < T5_VOX * ACC_V; i += T5_THREADS) acc[i] = 0.0;
  {  // A tiles: the zero groups stay zero for the whole kernel
    uint4* a4 = reinterpret_cast<uint4*>(smem);
    for (int i = t; i < OFF_B / 16; i += T5_THREADS) a4[i] = make_uint4(0u, 0u, 0u, 0u);
    uint4* bx4 = reinterpret_cast<uint4*>(smem + OFF_BX);
    for (int i = t; i < 2 * XN; i += T5_THREADS) bx4[i] = Z.v[i];
  }
  if (t < T5_VOX) sbits[t] = 0;
  if (t == 0) {
    for (int i = 0; i < T5_VOX * 2; ++i) {
      mbar_init(&full[i], 4);
      mbar_init(&empty[i], 1);
      mbar_init(&ffull[i], 1);
      mbar_init(&fempty[i], 3);
    }
    for (int j = 0; j < T5_VOX; ++j) {
      mbar_init(&axr[j], 4);
      mbar_init(&xfull[j], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // zeros and B_x visible to the tensor core
  __syncthreads();  // sbits zeroed before the pre-pass's atomicMax
  if (warp == T5_MMAW) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // producer warp w: TMEM sub-partition sp = w % 4, voxel pj = w / 4; its role (sample part ph,
  // landmark half) is rotated by the voxel so every sub-partition mixes part-0 warps (entries +
  // G1 sample groups) with part-1 warps
  const int sp = warp & 3, pj = warp >> 2;
#if T5_ROTATE_ROLES
  const int prole = (sp + pj) & 3;
#else
  const int prole = sp;
#endif
  const int ph = prole >> 1, pk = ((prole & 1) << 5) | lane;
  const int64_t pv = vbase + pj;
  const bool pvok = warp < T5_PWARPS && pv < v1;
  float ch[3] = {0.f, 0.f, 0.f}, cl[3] = {0.f, 0.f, 0.f};
  if (warp < T5_PWARPS) {
    voxel_split(src, pvok ? pv : v0, ch, cl);
    // Pre-pass (as k_gp_info_t5, unmasked): the voxel's bound 2 w (1 + |p|^2) >= 2 max|E| as
    // the fraction max (1 + |p|^2) / n^2; each thread loads a landmark once for all three voxels
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
        for (int j = 0; j < T5_VOX; ++j) {
          const float dx = __fadd_rn(__fsub_rn(a[u].x, vh[j][0]), __fsub_rn(b[u].x, vl[j][0]));
          const float dy = __fadd_rn(__fsub_rn(a[u].y, vh[j][1]), __fsub_rn(b[u].y, vl[j][1]));
          const float dz = __fadd_rn(__fsub_rn(a[u].z, vh[j][2]), __fsub_rn(b[u].z, vl[j][2]));
          const float n2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
          const float num = 1.0f + a[u].w;
          if (n2 > 1e-30f && b[u].w != 0.f && num * bd[j] > bn[j] * n2) {
            bn[j] = num;
            bd[j] = n2;
          }
        }
    }
#pragma unroll
    for (int j = 0; j < T5_VOX; ++j) {
      float mx = (vbase + j < v1 && bn[j] > 0.f) ? 2.0f * inv_s2 * __fdiv_rn(bn[j], bd[j]) : 0.f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (lane == 0) atomicMax(&sbits[j], __float_as_int(mx));
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
  auto span_end = [&](int tt) { return (tt % T5_FLUSH) == T5_FLUSH - 1 || tt == ntiles - 1; };
  const uint32_t sbase = smem_u32(smem);

  if (warp < T5_PWARPS && ntiles > 0) {
    // ───────────── producers ─────────────
    const float inv_s2_s = inv_s2 * voxel_scale(pj);  // exact: a power of two
    const uint32_t kofs_a = (pk >> 4) * T6_BLK_A + ((pk >> 3) & 1) * T6_KG_A + (pk & 7) * 16;
    const uint32_t kofs_b = (pk >> 4) * BLK_B + ((pk >> 3) & 1) * (256 * NG) + (pk & 7) * 16;
    const int xrow = sp * 32 + lane;  // A_x row = D row = this thread's TMEM lane
    const uint32_t axdst = sbase + OFF_AX + pj * T6_AX_BYTES + (xrow >> 3) * 256 + (xrow & 7) * 16;
    const uint32_t xaddr = tmem + ((uint32_t)(32 * sp) << 16) + XBASE + pj * XN + (ph == 0 ? 0 : 8 * G1);
    auto store_ax = [&](const PairF& q) {  // u = uh + ul in FP16 (uh: 10 mantissa bits, exact)
      const float hx = __uint_as_float(__float_as_uint(q.ux) & 0xFFFFE000u);
      const float hy = __uint_as_float(__float_as_uint(q.uy) & 0xFFFFE000u);
      const float hz = __uint_as_float(__float_as_uint(q.uz) & 0xFFFFE000u);
      const __half2 A = __floats2half2_rn(hx, hy), B = __floats2half2_rn(hz, q.uz - hz),
                    C = __floats2half2_rn(q.ux - hx, q.uy - hy);
      const uint32_t wa = *reinterpret_cast<const uint32_t*>(&A), wb = *reinterpret_cast<const uint32_t*>(&B),
                     wc = *reinterpret_cast<const uint32_t*>(&C);
      sts128(axdst, wa, wb, wa, wb);
      sts128(axdst + 128, wa, wb, wc, wc);
    };
    float4 a_cur = lm[2 * pk];
    PairF q_cur;
    {
      float4 b = lm[2 * pk + 1];
      if (!pvok) b.w = 0.f;
      q_cur = pair_prologue(a_cur, b, ch, cl, inv_s2_s);  // w (and every entry) carries the voxel scale
      store_ax(q_cur);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&axr[pj]);
    }
    if (T6_STAGGER_NS > 0 && pj > 0) __nanosleep(pj * T6_STAGGER_NS);
    float4 na = a_cur, nb = make_float4(0.f, 0.f, 0.f, 0.f);
    if (ntiles > 1) {
      na = lm[2 * (T5_TILE + pk)];
      nb = lm[2 * (T5_TILE + pk) + 1];
    }
    for (int tt = 0; tt < ntiles; ++tt) {
      const int s = tt % T5_STAGES;
      // this thread's exponent arguments of tile tt: one row of X(tt) (landed during tile tt - 1)
      constexpr int XR = 8 * (G1 > NG - G1 ? G1 : NG - G1);
      uint32_t xr[XR];
      if (T6_PROBE != 3) t6_spin(&xfull[pj], tt & 1, 1, pj, tt);
      tc_fence_after();
      if (ph == 0)
        tmem_ld_row<8 * G1>(xaddr, xr);
      else
        tmem_ld_row<8 * (NG - G1)>(xaddr, xr);
      // bearing of tile tt + 1 (its landmark was loaded a tile ago) while the X loads are in flight
      const float4 a_nxt = na;
      float4 b_nxt = nb;
      if (!pvok || tt + 1 >= ntiles) b_nxt.w = 0.f;
      const PairF q_nxt = pair_prologue(a_nxt, b_nxt, ch, cl, inv_s2_s);
      tc_wait_ld();  // X(tt) is in registers: its columns may be overwritten ...
      tc_fence_before();
      if (tt + 1 < ntiles) {  // ... and X(tt) landed also means the X MMA has read A_x(tt)
        store_ax(q_nxt);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&axr[pj]);
      if (tt + 2 < ntiles) {  // landmark of tile tt + 2: consumed after this tile's sigmoids
        const int64_t ni = (int64_t)(tt + 2) * T5_TILE + pk;
        na = lm[2 * ni];
        nb = lm[2 * ni + 1];
      }
#if T6_DEBUG
      if (tt >= T5_STAGES) t6_spin(&empty[pj * 2 + s], ((tt / T5_STAGES) - 1) & 1, 2, pj, tt);
#else
      if (tt >= T5_STAGES) t5_prod_wait(&empty[pj * 2 + s], ((tt / T5_STAGES) - 1) & 1);
#endif
      const uint32_t adst = sbase + (s * T5_VOX + pj) * STAGE_A + kofs_a;
      const uint32_t bdst = sbase + OFF_B + (s * T5_VOX + pj) * STAGE_B + kofs_b;
      if (ph == 0) {
        t6_sigmoids<NG, 0, G1, SKIP>(xr, cexp, bdst);  // (first: the X registers die before the entries)
        float e[24];
        entries21(q_cur, a_cur, e);
        e[21] = e[22] = e[23] = 0.f;
#pragma unroll
        for (int gi = 0; gi < 3; ++gi) {
          uint32_t hv[4], lv[4];
#pragma unroll
          for (int p = 0; p < 4; ++p) t5_split2(e[8 * gi + 2 * p], e[8 * gi + 2 * p + 1], hv[p], lv[p]);
          sts128(adst + gi * 128, lv[0], lv[1], lv[2], lv[3]);
          sts128(adst + (3 + gi) * 128, hv[0], hv[1], hv[2], hv[3]);
        }
      } else {
        t6_sigmoids<NG, G1, NG, SKIP>(xr, cexp, bdst);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[pj * 2 + s]);  // this warp's share of the voxel's stage s is written
      a_cur = a_nxt;
      q_cur = q_nxt;
    }
  } else if (warp == T5_MMAW && ntiles > 0) {
    // ───────────── MMA issue (one thread) ─────────────
    // 27 MMAs per tile: the issuing thread must not spend ~20 instructions on each (at that
    // cost the single MMA warp, not the producers, bounds the kernel: measured).  The shared
    // memory descriptors are {low word, constant high word}; the low word (address >> 4 and
    // the K-group stride) of every (stage, voxel, k-step) operand is a loop-invariant base
    // plus a compile-time constant, with the stage unrolled.
    constexpr uint32_t idesc_s = t6_idesc_s<NG>();
    constexpr uint32_t idesc_x = t6_idesc_x<XN>();
    constexpr uint32_t HI_S = (128u >> 4) | (1u << 14);  // SBO = 128, descriptor version 1 (bit 46)
    constexpr uint32_t HI_X = (256u >> 4) | (1u << 14);  // SBO = 256
    const uint32_t sb4 = sbase >> 4;                     // (< 2^14: shared memory is < 256 KB)
    const uint32_t alo = sb4 | ((uint32_t)(T6_KG_A >> 4) << 16);
    const uint32_t blo = (sb4 + (OFF_B >> 4)) | ((uint32_t)((256 * NG) >> 4) << 16);
    const uint32_t axlo = (sb4 + (OFF_AX >> 4)) | ((128u >> 4) << 16);
    const uint32_t bxlo = (sb4 + (OFF_BX >> 4)) | ((128u >> 4) << 16);
    auto issue_x = [&](auto voxel) {  // X(t) = A_x(t) (128 x 16) B_x^T (16 x XN) of one voxel
      constexpr int J = decltype(voxel)::value;
      t6_mma_lo(tmem + XBASE + J * XN, axlo + J * (T6_AX_BYTES >> 4), bxlo, HI_X, idesc_x, 0u);
      t6_commit(&xfull[J]);
    };
    auto issue_s = [&](auto voxel, auto stage, bool first, uint32_t d) {
      constexpr int J = decltype(voxel)::value, S = decltype(stage)::value;
#pragma unroll
      for (int ks = 0; ks < T5_KS; ++ks) {
        if (T6_PROBE == 5) continue;
        const uint32_t a = alo + (uint32_t)(((S * T5_VOX + J) * STAGE_A + ks * T6_BLK_A) >> 4);
        const uint32_t bb = blo + (uint32_t)(((S * T5_VOX + J) * STAGE_B + ks * BLK_B) >> 4);
        // rows [E_lo; E_hi; 0] x vs_hi, then rows [E_hi; 0; ..] x vs_lo into the same D rows
        t6_mma_lo(d, a, bb, HI_S, idesc_s, (ks > 0 || !first) ? 1u : 0u);
#if T6_PROBE != 1  // (timing probe 1: without the second S MMA; wrong results)
        t6_mma_lo(d, a + ((3 * 128) >> 4), bb + ((NG * 128) >> 4), HI_S, idesc_s, 1u);
#endif
      }
    };
    // One elected thread serves the three voxel pipelines round robin: X(t) of a voxel as soon
    // as its producers have read X(t - 1) and written A_x(t), the S MMAs of a tile as soon as
    // its stage is written.  xt / st: next tile whose X / S MMAs are to be issued.
    if (t6_elect(lane)) {
      int xt[T5_VOX], st[T5_VOX];
#pragma unroll
      for (int j = 0; j < T5_VOX; ++j) xt[j] = st[j] = 0;
      int left = 2 * T5_VOX * ntiles;
      auto serve = [&](auto voxel) {
        constexpr int J = decltype(voxel)::value;
        bool any = false;
        if (xt[J] < ntiles && mbar_try(&axr[J], xt[J] & 1)) {
          tc_fence_after();
          issue_x(voxel);
          ++xt[J];
          --left;
          any = true;
        }
        const int tt = st[J], s = tt & 1;
        const int k = tt / T5_FLUSH, b = k & 1;
        const bool first = tt % T5_FLUSH == 0;
        // a span's first tile also needs its accumulator buffer drained (it last held span k - 2).
        // Never block on that: the epilogue walks the voxels together, so a voxel that runs
        // ahead must let this thread serve the others, or they would wait for each other.
        // T6_X_FIRST: the S MMAs of tile tt are held back until X(tt + 2) is issued (its A_x is
        // written ~P1 after tile tt's stage): otherwise every X queues behind a tile's worth of
        // S MMAs in the in-order tensor pipe and the producers wait even longer for it
        // (139.4 vs 135.5 ms).  Probing all barriers first and issuing every ready X before any
        // S was slower (142.7 ms).
        if (tt < ntiles && (!T6_X_FIRST || xt[J] >= tt + 3 || xt[J] >= ntiles) &&
            mbar_try(&full[J * 2 + s], (tt >> 1) & 1) &&
            (!first || k < 2 || mbar_try(&fempty[J * 2 + b], ((k >> 1) - 1) & 1))) {
          tc_fence_after();
          const uint32_t d = tmem + ((uint32_t)(16 * b) << 16) + J * XN;
          if (s == 0)
            issue_s(voxel, std::integral_constant<int, 0>{}, first, d);
          else
            issue_s(voxel, std::integral_constant<int, 1>{}, first, d);
          if (span_end(tt)) t6_commit(&ffull[J * 2 + b]);
          t6_commit(&empty[J * 2 + s]);
          ++st[J];
          --left;
          any = true;
        }
        return any;
      };
#if T6_DEBUG
      long long idle = 0;
#endif
      while (left > 0) {
        const bool a0 = serve(std::integral_constant<int, 0>{});
        const bool a1 = serve(std::integral_constant<int, 1>{});
        const bool a2 = serve(std::integral_constant<int, 2>{});
        if (!(a0 | a1 | a2)) __nanosleep(T5_MMA_SLEEP);
#if T6_DEBUG
        idle = (a0 | a1 | a2) ? 0 : idle + 1;
        if (idle > 2000000) {
          if (blockIdx.x == 0)
            printf("t6 stuck: left %d ntiles %d xt %d %d %d st %d %d %d\n", left, ntiles, xt[0], xt[1], xt[2], st[0],
                   st[1], st[2]);
          __trap();
        }
#endif
      }
    }
    __syncwarp();
  } else if (warp >= T5_EPI0 && warp < T5_EPI0 + 3 && ntiles > 0) {
    // ───────────── epilogue: TMEM -> FP64 sums (warps 12-14 = sub-partitions 0-2) ─────────────
    // D rows 0-23: E_lo vs_hi + E_hi vs_lo of entries 0-23, rows 24-47: E_hi vs_hi.  Lane L < 16
    // of warp sp holds row 16 sp + L, columns [0, H); lane 16 + L the same row's columns [H, 2H).
    // Both row sets add into the same FP64 cells, and the two rows of an entry sit in different
    // warps.  No cell gets two writers at a time because the warps walk the voxels in rotated
    // order (warp sp: voxels sp, sp + 1, sp + 2 mod 3) with a named barrier after each step:
    // one pass per warp and span (the first version ran two phases over all voxels; its
    // critical warp was 94 % busy and the MMA thread waited for drained buffers: measured).
    constexpr int H = 4 * NG;
    constexpr int CH = (H % 12 == 0) ? 12 : (H % 8 == 0) ? 8 : 4;  // columns per wait
    const int L = lane & 15, q = lane >> 4;
    const int row = 16 * sp + L;
    const int e = row >= 24 ? row - 24 : row;
    const bool row_ok = e < 21;
    const int nspans = (ntiles + T5_FLUSH - 1) / T5_FLUSH;
    for (int k = 0; k < nspans; ++k) {
      const int b = k & 1;
#pragma unroll 1
      for (int step = 0; step < T5_VOX; ++step) {
        const int j = (sp + step) % T5_VOX;
#if T6_DEBUG
        t6_spin(&ffull[j * 2 + b], (k >> 1) & 1, 4, j, k);
#else
        mbar_wait_poll(&ffull[j * 2 + b], (k >> 1) & 1, T5_EPI_SLEEP);
#endif
        tc_fence_after();
        const uint32_t radr = tmem + ((uint32_t)(32 * sp + 16 * b) << 16) + j * XN;
        double* aj = acc + j * ACC_V + e;
        if (T6_PROBE != 4) {
#pragma unroll 1
          for (int c0 = 0; c0 < H; c0 += CH) {
            uint32_t r[CH];
#pragma unroll
            for (int u = 0; u < CH; u += 4)
              asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x4.b32 {%0,%1,%2,%3}, [%4], %5;"
                           : "=r"(r[u]), "=r"(r[u + 1]), "=r"(r[u + 2]), "=r"(r[u + 3])
                           : "r"(radr + c0 + u), "n"(H));
            tc_wait_ld();
#pragma unroll
            for (int i = 0; i < CH; ++i) {
              const int sm = q * H + c0 + i;
              if (T6_PROBE != 2 && row_ok && sm < ns) aj[sm * 21] += (double)__uint_as_float(r[i]);
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&fempty[j * 2 + b]);
        named_sync(T6_EPIBAR, 96);
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

// Host: the B_x image of the sample directions (column n holds sample n ^ 1)
inline uint16_t t6_half_bits(double x) {
  const __half h = __double2half(x);
  return static_cast<__half_raw>(h).x;
}
inline void t6_fill_z(T6Z& z, const double* zs_host, int ns, double ax, int xn) {
  uint16_t img[2 * T6_XN_MAX * 8];
  for (auto& w : img) w = 0;
  for (int n = 0; n < xn; ++n) {
    const int s = n ^ 1;
    if (s >= ns) continue;
    uint16_t zh[3], zm[3], zl[3];
    for (int c = 0; c < 3; ++c) {
      const double v = ax * zs_host[3 * s + c];
      zh[c] = t6_half_bits(v);
      const double r1 = v - (double)__half2float(__half(__half_raw{zh[c]}));
      zm[c] = t6_half_bits(r1);
      const double r2 = r1 - (double)__half2float(__half(__half_raw{zm[c]}));
      zl[c] = t6_half_bits(r2);
    }
    uint16_t* k0 = img + ((n / 8) * 256 + (n % 8) * 16) / 2;  // K slots 0-7
    uint16_t* k1 = k0 + 64;                                    // K slots 8-15
    k0[0] = zh[0], k0[1] = zh[1], k0[2] = zh[2], k0[3] = zh[2];
    k0[4] = zm[0], k0[5] = zm[1], k0[6] = zm[2], k0[7] = zm[2];
    k1[0] = zl[0], k1[1] = zl[1], k1[2] = zl[2], k1[3] = 0;
    k1[4] = zh[0], k1[5] = zh[1], k1[6] = zm[0], k1[7] = zm[1];
  }
  memcpy(z.v, img, sizeof(img));
}
