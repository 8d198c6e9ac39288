// fif_build.cu — field build (positional information factors), sm_100a.
//
// Replaces the voxel x landmark loops of the reference:
//   _nb_build_quad / _nb_build_quad_par  kernels.py:427-468, 527-568
//   _nb_build_gp                         kernels.py:471-524
//   per-pair 6x6 information             _nb_fim_flat_into kernels.py:363-424
//
// N-body structure: a CTA owns a tile of voxels; landmark tiles stream through
// shared memory and are broadcast to every thread.  Per-pair arithmetic is FP32
// on a difference d = p - c that is exact to ~1 ulp (landmarks and centres are
// pre-split into float hi/lo pairs), partial sums over short landmark runs are
// FP32 and are flushed into FP64 / double-float accumulators so the final
// factors carry ~1e-9 relative error (the query-parity budget).
// GP trace evaluates the sigmoid's cosine in FP64 (FP64 pipe is otherwise idle)
// because the kinv epilogue amplifies S errors ~200x.
#include <cstdarg>
#include <cstring>
#include <mutex>
#include <type_traits>

#include <cuda_fp16.h>

#include "fif_common.cuh"
#include "fif_gate.cuh"

namespace fif {

// ─────────────────────────── landmark table ────────────────────────────
// Per landmark 2 x float4: {ph.x, ph.y, ph.z, |p|^2}, {pl.x, pl.y, pl.z, valid}
// with p = ph + pl.  Rows past n are zero with valid = 0 (zero contribution).
constexpr int kLmPad = 256;

__global__ void k_prep_landmarks(const double* __restrict__ pts, int64_t n, int64_t n_pad, float4* __restrict__ tab) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_pad) return;
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f), b = make_float4(0.f, 0.f, 0.f, 0.f);
  if (i < n) {
    double px = pts[3 * i], py = pts[3 * i + 1], pz = pts[3 * i + 2];
    split_f32(px, a.x, b.x);
    split_f32(py, a.y, b.y);
    split_f32(pz, a.z, b.z);
    a.w = __double2float_rn(px * px + py * py + pz * pz);
    b.w = 1.0f;
  }
  tab[2 * i] = a;
  tab[2 * i + 1] = b;
}

// Per-pair prologue shared by the quad kernels and GP-info phase A.
struct PairF {
  float ux, uy, uz, w;  // unit bearing c->p and w = 1/(sigma^2 n^2) (0 if skipped)
};

__device__ __forceinline__ PairF pair_prologue(float4 a, float4 b, const float ch[3], const float cl[3], float inv_s2) {
  float dx = __fadd_rn(__fsub_rn(a.x, ch[0]), __fsub_rn(b.x, cl[0]));
  float dy = __fadd_rn(__fsub_rn(a.y, ch[1]), __fsub_rn(b.y, cl[1]));
  float dz = __fadd_rn(__fsub_rn(a.z, ch[2]), __fsub_rn(b.z, cl[2]));
  float n2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
  // the reference skips n2 < 1e-300 (kernels.py:444); in FP32 a coincident
  // landmark gives n2 == 0 and is skipped through rn = 0
  bool ok = n2 > 1e-30f && b.w != 0.f;
  float rn = ok ? rsqrtf(n2) : 0.f;
  // one Newton step: rsqrt to ~1 ulp
  rn = fmaf(0.5f * rn, fmaf(-n2 * rn, rn, 1.0f), rn);
  PairF q;
  q.ux = dx * rn;
  q.uy = dy * rn;
  q.uz = dz * rn;
  q.w = inv_s2 * rn * rn;
  return q;
}

__device__ __forceinline__ void voxel_split(const VoxSrc& src, int64_t v, float ch[3], float cl[3]) {
  double cx, cy, cz;
  voxel_center(src, v, cx, cy, cz);
  split_f32(cx, ch[0], cl[0]);
  split_f32(cy, ch[1], cl[1]);
  split_f32(cz, ch[2], cl[2]);
}

// ─────────────────────────── quad (FP64) ───────────────────────────────
// Quad factors feed queries whose value can cancel to ~1e-3 of the factor
// magnitude (nearest-landmark terms dominate sums weighted by 1/n^2), so the
// per-pair arithmetic is FP64 (B200 FP64 = 1/2 FP32 rate, separate pipe).
// EXACT=true reproduces _nb_build_quad's operation order bit for bit (IEEE sqrt
// and division, no FMA, landmark-sequential sums); EXACT=false uses FMA and an
// rsqrt+Newton reciprocal (~1e-16 relative, ~2x faster).
// Landmark tile: double4 {px, py, pz, |p|^2}.
constexpr int QD_THREADS = 128;
constexpr int QD_TILE = 128;

__global__ void k_prep_landmarks64(const double* __restrict__ pts, int64_t n, int64_t n_pad, double4* __restrict__ tab) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_pad) return;
  double4 a = make_double4(0.0, 0.0, 0.0, -1.0);  // pp < 0 marks padding
  if (i < n) {
    double px = pts[3 * i], py = pts[3 * i + 1], pz = pts[3 * i + 2];
    a = make_double4(px, py, pz, __dadd_rn(__dadd_rn(__dmul_rn(px, px), __dmul_rn(py, py)), __dmul_rn(pz, pz)));
  }
  tab[i] = a;
}

__device__ __forceinline__ double rsqrt_nr(double n2) {
  double r;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(n2));
  double h = n2 * r;
  r = fma(0.5 * r, fma(-h, r, 1.0), r);
  h = n2 * r;
  r = fma(0.5 * r, fma(-h, r, 1.0), r);
  return r;
}

struct PairD {
  double ux, uy, uz, w;  // w = 0 when the pair is skipped
};

template <bool EXACT>
__device__ __forceinline__ PairD pair64(double4 p, double cx, double cy, double cz, double inv_s2, bool keep) {
  PairD q;
  double dx = __dsub_rn(p.x, cx), dy = __dsub_rn(p.y, cy), dz = __dsub_rn(p.z, cz);
  double n2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  keep = keep && p.w >= 0.0 && n2 >= 1e-300;  // kernels.py:444
  if (!keep) {
    q.ux = q.uy = q.uz = q.w = 0.0;
    return q;
  }
  if (EXACT) {
    double n = __dsqrt_rn(n2);
    q.ux = __ddiv_rn(dx, n);
    q.uy = __ddiv_rn(dy, n);
    q.uz = __ddiv_rn(dz, n);
    q.w = __ddiv_rn(inv_s2, n2);
  } else {
    double r = rsqrt_nr(n2);
    q.ux = dx * r;
    q.uy = dy * r;
    q.uz = dz * r;
    q.w = inv_s2 * r * r;
  }
  return q;
}

// Entries of the 6x6 block (kernels.py:385-423) in packed order, FP64.
// EXACT: the reference's expressions with IEEE rounding of every operation.
#define MUL(a, b) (EXACT ? __dmul_rn((a), (b)) : ((a) * (b)))
#define ADD(a, b) (EXACT ? __dadd_rn((a), (b)) : ((a) + (b)))
#define SUB(a, b) (EXACT ? __dsub_rn((a), (b)) : ((a) - (b)))
template <bool EXACT>
__device__ __forceinline__ void c2_of(const PairD& q, double4 p, double& c2x, double& c2y, double& c2z) {
  c2x = SUB(MUL(p.y, q.uz), MUL(p.z, q.uy));
  c2y = SUB(MUL(p.z, q.ux), MUL(p.x, q.uz));
  c2z = SUB(MUL(p.x, q.uy), MUL(p.y, q.ux));
}
template <bool EXACT>
__device__ __forceinline__ double entry64(int e, const PairD& q, double4 p, double c2x, double c2y, double c2z) {
  const double w = q.w, nw = -q.w, ux = q.ux, uy = q.uy, uz = q.uz, px = p.x, py = p.y, pz = p.z, pp = p.w;
  switch (e) {
    case 0: return MUL(w, SUB(1.0, MUL(ux, ux)));
    case 1: return MUL(w, MUL(-ux, uy));
    case 2: return MUL(w, MUL(-ux, uz));
    case 3: return MUL(nw, MUL(ux, c2x));
    case 4: return MUL(nw, ADD(-pz, MUL(ux, c2y)));
    case 5: return MUL(nw, ADD(py, MUL(ux, c2z)));
    case 6: return MUL(w, SUB(1.0, MUL(uy, uy)));
    case 7: return MUL(w, MUL(-uy, uz));
    case 8: return MUL(nw, ADD(pz, MUL(uy, c2x)));
    case 9: return MUL(nw, MUL(uy, c2y));
    case 10: return MUL(nw, ADD(-px, MUL(uy, c2z)));
    case 11: return MUL(w, SUB(1.0, MUL(uz, uz)));
    case 12: return MUL(nw, ADD(-py, MUL(uz, c2x)));
    case 13: return MUL(nw, ADD(px, MUL(uz, c2y)));
    case 14: return MUL(nw, MUL(uz, c2z));
    case 15: return MUL(w, SUB(SUB(pp, MUL(px, px)), MUL(c2x, c2x)));
    case 16: return MUL(w, SUB(MUL(-px, py), MUL(c2x, c2y)));
    case 17: return MUL(w, SUB(MUL(-px, pz), MUL(c2x, c2z)));
    case 18: return MUL(w, SUB(SUB(pp, MUL(py, py)), MUL(c2y, c2y)));
    case 19: return MUL(w, SUB(MUL(-py, pz), MUL(c2y, c2z)));
    default: return MUL(w, SUB(ADD(MUL(-pz, pz), pp), MUL(c2z, c2z)));
  }
}

// One thread per voxel; out (rows,10) f64 = sum_i vp_i[k] tr_i (kernels.py:459-461).
template <bool EXACT, bool HAS_MASK>
__global__ void __launch_bounds__(QD_THREADS) k_quad_trace(const double4* __restrict__ lm, int64_t n_pad, int64_t n_real,
                                                           VoxSrc src, int64_t v0, int64_t v1,
                                                           const PairGate gate, double inv_s2,
                                                           double* __restrict__ out) {
  __shared__ double4 tile[QD_TILE];
  const int64_t v = v0 + blockIdx.x * (int64_t)QD_THREADS + threadIdx.x;
  const bool active = v < v1;
  double cx, cy, cz;
  voxel_center(src, active ? v : v0, cx, cy, cz);
  double acc[10];
#pragma unroll
  for (int k = 0; k < 10; ++k) acc[k] = 0.0;
  for (int64_t base = 0; base < n_pad; base += QD_TILE) {
    __syncthreads();
    for (int j = threadIdx.x; j < QD_TILE; j += QD_THREADS) tile[j] = lm[base + j];
    __syncthreads();
#pragma unroll 2
    for (int j = 0; j < QD_TILE; ++j) {
      const double4 p = tile[j];
      bool keep = active;
      if (HAS_MASK) {
        int64_t i = base + j;
        keep = keep && i < n_real && gate_keep(gate, v, i);
      }
      const PairD q = pair64<EXACT>(p, cx, cy, cz, inv_s2, keep);
      double tr;
      if (EXACT) {
        double c2x, c2y, c2z;
        c2_of<true>(q, p, c2x, c2y, c2z);
        // out[0] + out[7] + out[14] + out[21] + out[28] + out[35]  (kernels.py:424)
        tr = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(entry64<true>(0, q, p, c2x, c2y, c2z),
                                                                entry64<true>(6, q, p, c2x, c2y, c2z)),
                                                      entry64<true>(11, q, p, c2x, c2y, c2z)),
                                            entry64<true>(15, q, p, c2x, c2y, c2z)),
                                  entry64<true>(18, q, p, c2x, c2y, c2z)),
                        entry64<true>(20, q, p, c2x, c2y, c2z));
        const double vp[10] = {__dmul_rn(q.ux, q.ux), __dmul_rn(q.uy, q.uy), __dmul_rn(q.uz, q.uz),
                               __dmul_rn(q.ux, q.uy), __dmul_rn(q.ux, q.uz), __dmul_rn(q.uy, q.uz),
                               q.ux, q.uy, q.uz, 1.0};
        if (q.w != 0.0) {
#pragma unroll
          for (int k = 0; k < 10; ++k) acc[k] = __dadd_rn(acc[k], __dmul_rn(vp[k], tr));
        }
      } else {
        // trace = w (2 + |p|^2 + (p.u)^2) in closed form
        const double pu = fma(p.x, q.ux, fma(p.y, q.uy, p.z * q.uz));
        tr = q.w * fma(pu, pu, 2.0 + p.w);
        const double tx = tr * q.ux, ty = tr * q.uy, tz = tr * q.uz;
        acc[0] = fma(tx, q.ux, acc[0]);
        acc[1] = fma(ty, q.uy, acc[1]);
        acc[2] = fma(tz, q.uz, acc[2]);
        acc[3] = fma(tx, q.uy, acc[3]);
        acc[4] = fma(tx, q.uz, acc[4]);
        acc[5] = fma(ty, q.uz, acc[5]);
        acc[6] += tx;
        acc[7] += ty;
        acc[8] += tz;
        acc[9] += tr;
      }
    }
  }
  if (active) {
#pragma unroll
    for (int k = 0; k < 10; ++k) out[(v - v0) * 10 + k] = acc[k];
  }
}

// Info: warp-uniform entry groups; warp (w % 4) owns a subset of the 21 unique
// entries for the CTA's 32 voxels (one per lane), FP64 accumulators in registers.
// G0: TL {0,1,2,6,7,11}  G1: TR {3,4,5,8,9}  G2: {10,12,13,14,15}  G3: BR {16..20}
constexpr int QI_THREADS = 128;
constexpr int QI_TILE = 32;  // landmarks per phase-A/B tile of k_quad_info
template <int G> struct QGroup { static constexpr int NE = G == 0 ? 6 : 5; };
__host__ __device__ constexpr int qidx(int G, int t) {
  return G == 0 ? (t < 3 ? t : (t < 5 ? t + 3 : 11))
       : G == 1 ? (t < 3 ? 3 + t : 5 + t)
       : G == 2 ? (t == 0 ? 10 : 11 + t)
       : 16 + t;
}

template <int G, bool EXACT, bool HAS_MASK>
__device__ __forceinline__ void quad_info_tiles(const double4* __restrict__ lm, double4* tile, double* rec,
                                                int64_t n_pad, int64_t n_real, int64_t v, int64_t v0, bool active,
                                                double cx, double cy, double cz, const PairGate gate,
                                                double inv_s2, double* __restrict__ out) {
  constexpr int NE = QGroup<G>::NE;
  constexpr int RS = QI_TILE * 32;  // stride between record components
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc[10 * NE];
#pragma unroll
  for (int t = 0; t < 10 * NE; ++t) acc[t] = 0.0;
  for (int64_t base = 0; base < n_pad; base += QI_TILE) {
    __syncthreads();
    for (int j = threadIdx.x; j < QI_TILE; j += QI_THREADS) tile[j] = lm[base + j];
    __syncthreads();
    // phase A: pair (voxel = lane, landmark j), j = warp, warp + 4, ...
#pragma unroll 1
    for (int j = warp; j < QI_TILE; j += QI_THREADS / 32) {
      const double4 p = tile[j];
      bool keep = active;
      if (HAS_MASK) {
        const int64_t i = base + j;
        keep = keep && i < n_real && gate_keep(gate, v, i);
      }
      const PairD q = pair64<EXACT>(p, cx, cy, cz, inv_s2, keep);
      double c2x, c2y, c2z;
      c2_of<EXACT>(q, p, c2x, c2y, c2z);
      double* r = rec + j * 32 + lane;
      r[0] = q.ux;
      r[RS] = q.uy;
      r[2 * RS] = q.uz;
      r[3 * RS] = q.w;
      r[4 * RS] = c2x;
      r[5 * RS] = c2y;
      r[6 * RS] = c2z;
    }
    __syncthreads();
    // phase B: this warp's entry group
#pragma unroll 2
    for (int j = 0; j < QI_TILE; ++j) {
      const double4 p = tile[j];
      const double* r = rec + j * 32 + lane;
      const PairD q{r[0], r[RS], r[2 * RS], r[3 * RS]};
      const double c2x = r[4 * RS], c2y = r[5 * RS], c2z = r[6 * RS];
      double e[NE];
#pragma unroll
      for (int t = 0; t < NE; ++t) e[t] = entry64<EXACT>(qidx(G, t), q, p, c2x, c2y, c2z);
      const double vp[10] = {MUL(q.ux, q.ux), MUL(q.uy, q.uy), MUL(q.uz, q.uz), MUL(q.ux, q.uy),
                             MUL(q.ux, q.uz), MUL(q.uy, q.uz), q.ux, q.uy, q.uz, 1.0};
#pragma unroll
      for (int k = 0; k < 10; ++k)
#pragma unroll
        for (int t = 0; t < NE; ++t)
          acc[k * NE + t] = EXACT ? __dadd_rn(acc[k * NE + t], __dmul_rn(vp[k], e[t])) : fma(vp[k], e[t], acc[k * NE + t]);
    }
  }
  if (active) {
    double* o = out + (v - v0) * 210;
#pragma unroll
    for (int k = 0; k < 10; ++k)
#pragma unroll
      for (int t = 0; t < NE; ++t) o[k * 21 + qidx(G, t)] = acc[k * NE + t];
  }
}
#undef MUL
#undef ADD
#undef SUB

// Phase A computes each (voxel, landmark) pair's bearing, weight and c2 = p x u once, into
// shared memory (component-major [7][QI_TILE][32], so both the stores and each entry
// group's reads are conflict-free); phase B: warp G accumulates its entry group for the
// same 32 voxels (lane = voxel).  Skipped pairs are stored as zeros, so their products
// add +-0 -- bit-identical to skipping them, as the accumulators are never -0.
#ifndef QI_MINB
#define QI_MINB 3  // 12 warps per SM (<= 168 registers): 67.6 -> 65.5 ms on config 2
#endif
template <bool EXACT, bool HAS_MASK>
__global__ void __launch_bounds__(QI_THREADS, QI_MINB) k_quad_info(const double4* __restrict__ lm, int64_t n_pad, int64_t n_real,
                                                          VoxSrc src, int64_t v0, int64_t v1,
                                                          const PairGate gate, double inv_s2,
                                                          double* __restrict__ out) {
  extern __shared__ __align__(16) unsigned char qi_raw[];
  double4* tile = reinterpret_cast<double4*>(qi_raw);                        // [QI_TILE]
  double* rec = reinterpret_cast<double*>(tile + QI_TILE);                   // [7][QI_TILE][32]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t v = v0 + blockIdx.x * (int64_t)32 + lane;
  const bool active = v < v1;
  double cx, cy, cz;
  voxel_center(src, active ? v : v0, cx, cy, cz);
  switch (warp) {
    case 0: quad_info_tiles<0, EXACT, HAS_MASK>(lm, tile, rec, n_pad, n_real, v, v0, active, cx, cy, cz, gate, inv_s2, out); break;
    case 1: quad_info_tiles<1, EXACT, HAS_MASK>(lm, tile, rec, n_pad, n_real, v, v0, active, cx, cy, cz, gate, inv_s2, out); break;
    case 2: quad_info_tiles<2, EXACT, HAS_MASK>(lm, tile, rec, n_pad, n_real, v, v0, active, cx, cy, cz, gate, inv_s2, out); break;
    default: quad_info_tiles<3, EXACT, HAS_MASK>(lm, tile, rec, n_pad, n_real, v, v0, active, cx, cy, cz, gate, inv_s2, out); break;
  }
}

// ─────────────────────────── GP, trace ─────────────────────────────────
// CTA = VB voxels x ceil(N_s/GT_G) threads; thread (v, gi) owns samples gi + s*tpv.
// Phase A: per (voxel, landmark) pair, FP64 bearing u and FP32 trace tr into smem
// (the reference's exact d, n2 and skip rule).  Phase B: for each landmark a
// thread loads the 32-byte pair record once and evaluates GT_G sigmoids with the
// cosine in FP64 (the kinv epilogue amplifies S errors ~200x),
// converts the exponent argument to FP32 on the integer ALU, and accumulates
// tr * vs into FP32 partials flushed into double-float accumulators.
constexpr int GT_TILE = 64;
constexpr int GT_FLUSH = 8;
#ifndef GT_G_N
#define GT_G_N 4
#endif
constexpr int GT_G = GT_G_N;
constexpr int GT_THREADS = 256;
#ifndef GT_MINB
#define GT_MINB 3
#endif
// Sigmoid reciprocals.  GT_PAIR (default): one MUFU rcp per pair of sigmoids,
// r = 1 / ((1 + 2^x0)(1 + 2^x1)) with x clamped to 63 -- a quarter less MUFU/MIO traffic
// for 2 FMULs and 2 clamps: config 2 113.7 -> 110.1 ms (106.1 unclamped, which is only safe
// for |x| <= 63; a per-CTA proof plus a fallback path measured 111.8, a per-landmark
// branch 115.0).  Otherwise GT_RCP: 0 one MUFU rcp per sigmoid, 1 scalar FMA-pipe Newton,
// 2 packed (FFMA2) Newton -- measured 113.7 / 133.5 / 140.3 ms: moving the reciprocal to
// the FMA pipe costs more issue slots and latency than the MUFU time it frees.
#ifndef GT_PAIR
#define GT_PAIR 1
#endif
#ifndef GT_RCP
#define GT_RCP 0
#endif
static_assert(GT_G % 2 == 0, "paired sigmoids need an even GT_G");
struct __align__(16) PairT {
  double ux, uy, uz;
  float tr, pad;
};

template <bool HAS_MASK>
__global__ void __launch_bounds__(GT_THREADS, GT_MINB) k_gp_trace(const double* __restrict__ pts, int64_t n_real, VoxSrc src,
                                                         int64_t v0, int64_t v1, int vb, int ns,
                                                         const double* __restrict__ zs, const PairGate gate,
                                                         double inv_s2, double ax, double bx,
                                                         double* __restrict__ out64, float* __restrict__ out32) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int pstride = GT_TILE + 1;                                // records per voxel (+1: bank spread)
  PairT* pairs = reinterpret_cast<PairT*>(smem_raw);              // [vb][pstride]
  double* cen = reinterpret_cast<double*>(pairs + vb * pstride);  // [vb][3]
  double* lp = cen + 3 * vb;                                      // [GT_TILE][3] landmark tile
  const int t = threadIdx.x, nt = blockDim.x;
  const int tpv = (ns + GT_G - 1) / GT_G;
  const int64_t vbase = v0 + blockIdx.x * (int64_t)vb;
  if (t < vb) {
    int64_t v = vbase + t;
    double cx = 0, cy = 0, cz = 0;
    if (v < v1) voxel_center(src, v, cx, cy, cz);
    cen[3 * t] = cx;
    cen[3 * t + 1] = cy;
    cen[3 * t + 2] = cz;
  }
  const int vl = t / tpv, gi = t - vl * tpv;
  const bool worker = vl < vb;
  const bool active = worker && (vbase + vl) < v1;
  // x = ax (u . z) + bx = (ax zx) ux + (ax zy) uy + (ax zz) uz + bx
  double zx[GT_G], zy[GT_G], zz[GT_G];
#pragma unroll
  for (int s = 0; s < GT_G; ++s) {
    const int g = gi + s * tpv;
    const bool ok = worker && g < ns;
    // exact power-of-two pre-scale for the two-op FP64 -> FP32 conversion below
    zx[s] = ok ? ax * zs[3 * g] * kF32Bias : 0.0;
    zy[s] = ok ? ax * zs[3 * g + 1] * kF32Bias : 0.0;
    zz[s] = ok ? ax * zs[3 * g + 2] * kF32Bias : 0.0;
  }
  const double bxs = bx * kF32Bias;
  DF acc[GT_G];
#pragma unroll
  for (int s = 0; s < GT_G; ++s) acc[s].init();
  const int npairs = vb * GT_TILE;
  for (int64_t base = 0; base < n_real; base += GT_TILE) {
    __syncthreads();
    for (int j = t; j < GT_TILE * 3; j += nt) {
      int64_t i = base + j / 3;
      lp[j] = i < n_real ? pts[3 * base + j] : 0.0;
    }
    __syncthreads();
    // phase A: FP64 per-pair quantities
    for (int pidx = t; pidx < npairs; pidx += nt) {
      const int pv = pidx / GT_TILE, pj = pidx - pv * GT_TILE;
      const int64_t i = base + pj;
      const double px = lp[3 * pj], py = lp[3 * pj + 1], pz = lp[3 * pj + 2];
      const double dx = px - cen[3 * pv], dy = py - cen[3 * pv + 1], dz = pz - cen[3 * pv + 2];
      const double n2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
      bool ok = i < n_real && n2 >= 1e-300 && (vbase + pv) < v1;  // kernels.py:494
      if (HAS_MASK && ok) ok = gate_keep(gate, vbase + pv, i);
      PairT pr;
      if (ok) {
        const double rn = rsqrt_nr(n2);
        const double ux = dx * rn, uy = dy * rn, uz = dz * rn;
        const double w = inv_s2 * rn * rn;
        const double pu = px * ux + py * uy + pz * uz;
        const double pp = px * px + py * py + pz * pz;
        pr.ux = ux;
        pr.uy = uy;
        pr.uz = uz;
        pr.tr = (float)(w * (2.0 + pp + pu * pu));
      } else {
        pr.ux = pr.uy = pr.uz = 0.0;
        pr.tr = 0.f;
      }
      pr.pad = 0.f;
      pairs[pv * pstride + pj] = pr;
    }
    __syncthreads();
    if (worker) {
      const PairT* pv = pairs + vl * pstride;
#pragma unroll 1
      for (int j0 = 0; j0 < GT_TILE; j0 += GT_FLUSH) {
        float part[GT_G];
#pragma unroll
        for (int s = 0; s < GT_G; ++s) part[s] = 0.f;
#pragma unroll 2
        for (int j = j0; j < j0 + GT_FLUSH; ++j) {
          const PairT pr = pv[j];
          if constexpr (GT_PAIR) {
#pragma unroll
            for (int s = 0; s < GT_G; s += 2) {
              // two sigmoids, one reciprocal: r = 1 / ((1 + 2^x0)(1 + 2^x1)),
              // vs0 = (1 + 2^x1) r, vs1 = (1 + 2^x0) r; x <= 63 keeps the product finite
              // (a sigmoid below 2^-63 is then off by < 2^-63 absolute)
              const float x0 =
                  fminf(f64s_to_f32_alu(fma(pr.ux, zx[s], fma(pr.uy, zy[s], fma(pr.uz, zz[s], bxs)))), 63.f);
              const float x1 =
                  fminf(f64s_to_f32_alu(fma(pr.ux, zx[s + 1], fma(pr.uy, zy[s + 1], fma(pr.uz, zz[s + 1], bxs)))), 63.f);
              const float a0 = 1.0f + ex2_approx(x0), a1 = 1.0f + ex2_approx(x1);
              const float tr_r = pr.tr * rcp_approx(a0 * a1);
              part[s] = fmaf(tr_r, a1, part[s]);
              part[s + 1] = fmaf(tr_r, a0, part[s + 1]);
            }
          } else {
#if GT_RCP == 2
            const f32x2 tr2 = splat2(pr.tr);
#pragma unroll
            for (int s = 0; s < GT_G; s += 2) {
              // -k_s (u.z - cos a) log2(e) in FP64 (zx..bxs carry the exact 2^-896
              // pre-scale of f64s_to_f32_alu), converted to FP32 with two ALU ops;
              // clamped so 1 + 2^x stays finite for the FMA-pipe reciprocal
              const float x0 = fminf(f64s_to_f32_alu(fma(pr.ux, zx[s], fma(pr.uy, zy[s], fma(pr.uz, zz[s], bxs)))), 126.f);
              const float x1 =
                  fminf(f64s_to_f32_alu(fma(pr.ux, zx[s + 1], fma(pr.uy, zy[s + 1], fma(pr.uz, zz[s + 1], bxs)))), 126.f);
              const f32x2 ny = ffma2(pack2(ex2_approx(x0), ex2_approx(x1)), splat2(-1.0f), splat2(-1.0f));
              const f32x2 vs = rcp_nr2_neg(ny);
              float p0, p1;
              unpack2(ffma2(tr2, vs, pack2(part[s], part[s + 1])), p0, p1);
              part[s] = p0;
              part[s + 1] = p1;
            }
#else
#pragma unroll
            for (int s = 0; s < GT_G; ++s) {
              // -k_s (u.z - cos a) log2(e) in FP64 (zx..bxs carry the exact 2^-896
              // pre-scale of f64s_to_f32_alu), converted to FP32 with two ALU ops
              const float x = f64s_to_f32_alu(fma(pr.ux, zx[s], fma(pr.uy, zy[s], fma(pr.uz, zz[s], bxs))));
#if GT_RCP == 1
              const float vs = rcp_nr_neg(-1.0f - ex2_approx(fminf(x, 126.f)));
#else
              const float vs = rcp_approx(1.0f + ex2_approx(x));
#endif
              part[s] = fmaf(pr.tr, vs, part[s]);
            }
#endif
          }
        }
#pragma unroll
        for (int s = 0; s < GT_G; ++s) acc[s].add(part[s]);
      }
    }
  }
  if (active) {
    const int64_t r = vbase + vl - v0;
#pragma unroll
    for (int s = 0; s < GT_G; ++s) {
      const int g = gi + s * tpv;
      if (g >= ns) continue;
      const double v = acc[s].value();
      out64[r * ns + g] = v;
      if (out32) out32[r * ns + g] = (float)v;
    }
  }
}

// ─────────────────────────── GP, info ──────────────────────────────────
// Phase A: per pair, u and the 21 unique entries of w*block in FP32, laid out
// for packed FP32x2 math: float4 {ux, uy, uz, e20}, then e0..e19 as 5 float4.
// Phase B: thread (v, g) evaluates vs_g once per landmark and accumulates
// vs_g * entries with FFMA2 (sm_100 packed FP32) into FP32 partials, flushed
// every GI_FLUSH_TILES tiles into FP64 accumulators (F2F on the MUFU pipe + DADD
// on the otherwise idle FP64 pipe).
constexpr int GI_TILE = 32;
constexpr int GI_THREADS_MAX = 320;

// All 21 packed entries (FP32) for one pair.
__device__ __forceinline__ void entries21(const PairF& q, float4 a, float* e) {
  const float w = q.w, ux = q.ux, uy = q.uy, uz = q.uz;
  const float px = a.x, py = a.y, pz = a.z, pp = a.w;
  const float wx = w * ux, wy = w * uy, wz = w * uz;
  const float c2x = fmaf(py, uz, -pz * uy), c2y = fmaf(pz, ux, -px * uz), c2z = fmaf(px, uy, -py * ux);
  e[0] = fmaf(-wx, ux, w);
  e[1] = -wx * uy;
  e[2] = -wx * uz;
  e[3] = -w * (ux * c2x);
  e[4] = -w * fmaf(ux, c2y, -pz);
  e[5] = -w * fmaf(ux, c2z, py);
  e[6] = fmaf(-wy, uy, w);
  e[7] = -wy * uz;
  e[8] = -w * fmaf(uy, c2x, pz);
  e[9] = -w * (uy * c2y);
  e[10] = -w * fmaf(uy, c2z, -px);
  e[11] = fmaf(-wz, uz, w);
  e[12] = -w * fmaf(uz, c2x, -py);
  e[13] = -w * fmaf(uz, c2y, px);
  e[14] = -w * (uz * c2z);
  e[15] = w * fmaf(-c2x, c2x, fmaf(-px, px, pp));
  e[16] = w * fmaf(-c2x, c2y, -px * py);
  e[17] = w * fmaf(-c2x, c2z, -px * pz);
  e[18] = w * fmaf(-c2y, c2y, fmaf(-py, py, pp));
  e[19] = w * fmaf(-c2y, c2z, -py * pz);
  e[20] = w * fmaf(-c2z, c2z, fmaf(-pz, pz, pp));
}


// ── phase A of the GP info kernels on FP32x2 pairs: the same landmark against two voxels
// (lo half: voxel A, hi half: voxel B), every operation of pair_prologue / entries21
// issued once as FFMA2 / FMUL2 / FADD2 (rsqrt stays per lane on MUFU).
struct PairF2 {
  f32x2 ux, uy, uz, w;
};
// ch2/cl2: centre hi/lo of both voxels; okA/okB: the pair is kept (landmark valid, voxel in range, mask)
__device__ __forceinline__ PairF2 pair_prologue2(float4 a, float4 b, const f32x2 ch2[3], const f32x2 cl2[3],
                                                 float inv_s2, bool okA, bool okB) {
  const f32x2 dx = fadd2(fsub2(splat2(a.x), ch2[0]), fsub2(splat2(b.x), cl2[0]));
  const f32x2 dy = fadd2(fsub2(splat2(a.y), ch2[1]), fsub2(splat2(b.y), cl2[1]));
  const f32x2 dz = fadd2(fsub2(splat2(a.z), ch2[2]), fsub2(splat2(b.z), cl2[2]));
  const f32x2 n2 = ffma2(dx, dx, ffma2(dy, dy, fmul2(dz, dz)));
  float nA, nB;
  unpack2(n2, nA, nB);
  const f32x2 rn0 = pack2(okA && nA > 1e-30f ? rsqrtf(nA) : 0.f, okB && nB > 1e-30f ? rsqrtf(nB) : 0.f);
  // one Newton step: rsqrt to ~1 ulp
  const f32x2 rn = ffma2(fmul2(splat2(0.5f), rn0), ffma2(fmul2(fneg2(n2), rn0), rn0, splat2(1.0f)), rn0);
  PairF2 q;
  q.ux = fmul2(dx, rn);
  q.uy = fmul2(dy, rn);
  q.uz = fmul2(dz, rn);
  q.w = fmul2(fmul2(splat2(inv_s2), rn), rn);
  return q;
}
// entries21 for both voxels of a PairF2 (same landmark a)
__device__ __forceinline__ void entries21x2(const PairF2& q, float4 a, f32x2* e) {
  const f32x2 w = q.w, ux = q.ux, uy = q.uy, uz = q.uz;
  const f32x2 px = splat2(a.x), py = splat2(a.y), pz = splat2(a.z), pp = splat2(a.w);
  const f32x2 nw = fneg2(w);
  const f32x2 wx = fmul2(w, ux), wy = fmul2(w, uy), wz = fmul2(w, uz);
  const f32x2 c2x = ffma2(py, uz, fneg2(fmul2(pz, uy))), c2y = ffma2(pz, ux, fneg2(fmul2(px, uz))),
              c2z = ffma2(px, uy, fneg2(fmul2(py, ux)));
  e[0] = ffma2(fneg2(wx), ux, w);
  e[1] = fmul2(fneg2(wx), uy);
  e[2] = fmul2(fneg2(wx), uz);
  e[3] = fmul2(nw, fmul2(ux, c2x));
  e[4] = fmul2(nw, ffma2(ux, c2y, fneg2(pz)));
  e[5] = fmul2(nw, ffma2(ux, c2z, py));
  e[6] = ffma2(fneg2(wy), uy, w);
  e[7] = fmul2(fneg2(wy), uz);
  e[8] = fmul2(nw, ffma2(uy, c2x, pz));
  e[9] = fmul2(nw, fmul2(uy, c2y));
  e[10] = fmul2(nw, ffma2(uy, c2z, fneg2(px)));
  e[11] = ffma2(fneg2(wz), uz, w);
  e[12] = fmul2(nw, ffma2(uz, c2x, fneg2(py)));
  e[13] = fmul2(nw, ffma2(uz, c2y, px));
  e[14] = fmul2(nw, fmul2(uz, c2z));
  e[15] = fmul2(w, ffma2(fneg2(c2x), c2x, ffma2(fneg2(px), px, pp)));
  e[16] = fmul2(w, ffma2(fneg2(c2x), c2y, fneg2(fmul2(px, py))));
  e[17] = fmul2(w, ffma2(fneg2(c2x), c2z, fneg2(fmul2(px, pz))));
  e[18] = fmul2(w, ffma2(fneg2(c2y), c2y, ffma2(fneg2(py), py, pp)));
  e[19] = fmul2(w, ffma2(fneg2(c2y), c2z, fneg2(fmul2(py, pz))));
  e[20] = fmul2(w, ffma2(fneg2(c2z), c2z, ffma2(fneg2(pz), pz, pp)));
}

// Shared-memory reads cost one wavefront per 128 lane-bytes even when every lane
// reads the same address (measured: LDS.128 broadcast ~ 4 wavefronts), so each
// thread handles GI_G samples (g, g+tpv, g+2tpv, ...) of one voxel and reuses
// every 96-byte pair record GI_G times; FP64 accumulators live in shared memory
// ([21*GI_G][blockDim] doubles) and are refreshed every GI_FLUSH_TILES tiles.
constexpr int GI_G = 4;
constexpr int GI_FLUSH_TILES = 4;  // FP32 partials span 128 landmarks
constexpr int GI_VB_THREADS = 128;

template <bool HAS_MASK>
__global__ void __launch_bounds__(GI_VB_THREADS, 2)
k_gp_info(const float4* __restrict__ lm, int64_t n_pad, int64_t n_real, VoxSrc src, int64_t v0, int64_t v1, int vb,
          int ns, const double* __restrict__ zs, const PairGate gate, float inv_s2, float ax, float bx,
          double* __restrict__ out64, float* __restrict__ out32) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tpv = (ns + GI_G - 1) / GI_G;                        // threads per voxel
  const int pstride = GI_TILE * 6 + 1;                           // float4 per voxel (+1: bank spread)
  const int nt = blockDim.x;
  double* accs = reinterpret_cast<double*>(smem_raw);            // [21*GI_G][nt]
  float4* pairs = reinterpret_cast<float4*>(accs + 21 * GI_G * nt);  // [vb][pstride]
  float4* tile = pairs + vb * pstride;                           // [GI_TILE][2]
  float* cs = reinterpret_cast<float*>(tile + GI_TILE * 2);      // [vb][6]
  const int t = threadIdx.x;
  const int64_t vbase = v0 + blockIdx.x * (int64_t)vb;
  if (t < vb) {
    int64_t v = vbase + t;
    float ch[3], cl[3];
    voxel_split(src, v < v1 ? v : v0, ch, cl);
    for (int k = 0; k < 3; ++k) {
      cs[6 * t + k] = ch[k];
      cs[6 * t + 3 + k] = cl[k];
    }
  }
  for (int k = 0; k < 21 * GI_G; ++k) accs[k * nt + t] = 0.0;
  const int vl = t / tpv, gi = t - vl * tpv;
  const bool worker = vl < vb;
  const bool active = worker && (vbase + vl) < v1;
  float zx[GI_G], zy[GI_G], zz[GI_G];
#pragma unroll
  for (int s = 0; s < GI_G; ++s) {
    const int g = gi + s * tpv;
    const bool ok = worker && g < ns;
    zx[s] = ok ? (float)zs[3 * g] : 0.f;
    zy[s] = ok ? (float)zs[3 * g + 1] : 0.f;
    zz[s] = ok ? (float)zs[3 * g + 2] : 0.f;
  }
  float2 part[GI_G][10];
  float part20[GI_G];
#pragma unroll
  for (int s = 0; s < GI_G; ++s) {
    part20[s] = 0.f;
#pragma unroll
    for (int k = 0; k < 10; ++k) part[s][k] = make_float2(0.f, 0.f);
  }
  const int npairs = vb * GI_TILE;
  int tiles = 0;
  for (int64_t base = 0; base < n_pad; base += GI_TILE) {
    __syncthreads();
    for (int j = t; j < GI_TILE * 2; j += nt) tile[j] = lm[2 * base + j];
    __syncthreads();
    for (int pidx = t; pidx < npairs; pidx += nt) {
      const int pv = pidx / GI_TILE, pj = pidx - pv * GI_TILE;
      float4 a = tile[2 * pj], b = tile[2 * pj + 1];
      if ((vbase + pv) >= v1) b.w = 0.f;
      if (HAS_MASK) {
        int64_t i = base + pj;
        if (b.w != 0.f && !gate_keep(gate, vbase + pv, i)) b.w = 0.f;
      }
      const float* c = cs + 6 * pv;
      const float ch[3] = {c[0], c[1], c[2]}, cl[3] = {c[3], c[4], c[5]};
      const PairF q = pair_prologue(a, b, ch, cl, inv_s2);
      float e[21];
      entries21(q, a, e);
      float4* dst = pairs + pv * pstride + pj * 6;
      dst[0] = make_float4(q.ux, q.uy, q.uz, e[20]);
#pragma unroll
      for (int k = 0; k < 5; ++k) dst[1 + k] = make_float4(e[4 * k], e[4 * k + 1], e[4 * k + 2], e[4 * k + 3]);
    }
    __syncthreads();
    if (worker) {
      const float4* pv = pairs + vl * pstride;
      // software pipeline: the sigmoids of landmarks j+2, j+3 (2 x GI_G independent
      // MUFU chains) are issued before the FFMA2 block of landmarks j, j+1.
      float vs[2][GI_G], e20[2];
      auto sigmoids = [&](int j, float (&out)[2][GI_G], float (&oe)[2]) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const float4 r0 = pv[6 * (j + u)];
          oe[u] = r0.w;
#pragma unroll
          for (int s = 0; s < GI_G; ++s) {
            const float cg = fmaf(r0.x, zx[s], fmaf(r0.y, zy[s], r0.z * zz[s]));
            out[u][s] = rcp_approx(1.0f + ex2_approx(fmaf(cg, ax, bx)));
          }
        }
      };
      sigmoids(0, vs, e20);
#pragma unroll 1
      for (int j0 = 0; j0 < GI_TILE; j0 += 2) {
        float vn[2][GI_G], en[2];
        sigmoids((j0 + 2) & (GI_TILE - 1), vn, en);  // wraps harmlessly on the last step
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const float4* p = pv + 6 * (j0 + u);
#pragma unroll
          for (int k = 0; k < 5; ++k) {
            const float4 r = p[1 + k];
            const float2 lo = make_float2(r.x, r.y), hi = make_float2(r.z, r.w);
#pragma unroll
            for (int s = 0; s < GI_G; ++s) {
              const float2 v2 = make_float2(vs[u][s], vs[u][s]);
              part[s][2 * k] = __ffma2_rn(v2, lo, part[s][2 * k]);
              part[s][2 * k + 1] = __ffma2_rn(v2, hi, part[s][2 * k + 1]);
            }
          }
#pragma unroll
          for (int s = 0; s < GI_G; ++s) part20[s] = fmaf(vs[u][s], e20[u], part20[s]);
        }
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          e20[u] = en[u];
#pragma unroll
          for (int s = 0; s < GI_G; ++s) vs[u][s] = vn[u][s];
        }
      }
      if (++tiles == GI_FLUSH_TILES || base + GI_TILE >= n_pad) {
        tiles = 0;
#pragma unroll
        for (int s = 0; s < GI_G; ++s) {
#pragma unroll
          for (int k = 0; k < 10; ++k) {
            accs[(21 * s + 2 * k) * nt + t] += (double)part[s][k].x;
            accs[(21 * s + 2 * k + 1) * nt + t] += (double)part[s][k].y;
            part[s][k] = make_float2(0.f, 0.f);
          }
          accs[(21 * s + 20) * nt + t] += (double)part20[s];
          part20[s] = 0.f;
        }
      }
    }
  }
  if (active) {
    const int64_t r = vbase + vl - v0;
    for (int s = 0; s < GI_G; ++s) {
      const int g = gi + s * tpv;
      if (g >= ns) continue;
      double* o = out64 + (r * ns + g) * 21;
      float* o32 = out32 ? out32 + (r * ns + g) * 21 : nullptr;
#pragma unroll
      for (int e = 0; e < 21; ++e) {
        const double v = accs[(21 * s + e) * nt + t];
        o[e] = v;
        if (o32) o32[e] = (float)v;
      }
    }
  }
}

// ─────────────────────────── GP, info on the tensor pipe ────────────────
// S_v[g][e] = sum_j vs_v(j, g) E_v(j, e) is, per voxel, a (samples x landmarks) x
// (landmarks x entries) matrix product whose A operand (the sigmoids) is generated
// on the fly.  Each warp owns one voxel and up to 5 m16 sample tiles; per k-step of
// 8 landmarks a lane evaluates 4 sigmoids per m-tile (exactly the A-fragment entries
// it holds: no redundant MUFU work) and the warp issues mma.sync m16n8k8 TF32 with a
// 3-term split (hi*hi + hi*lo + lo*hi ~ FP32 products) into FP32 accumulators that are
// flushed to FP64 (shared memory) every GC_FLUSH landmarks.  B fragments (entries,
// pre-split into TF32 hi/lo by phase A) are read from a bank-conflict-free layout.
constexpr int GC_TILE = 64;       // landmarks per smem tile
#ifndef GC_FLUSH_TILES
#define GC_FLUSH_TILES 8          // FP32 accumulators span 512 landmarks, then FP64
#endif
constexpr int GC_MT = 5;          // m16 tiles per warp (80 samples)
constexpr int GC_WARPS = 4;
constexpr int GC_NT = 3;          // n8 tiles (24 >= 21 entries)

// TF32 split by truncation (1 LOP3; cvt.rna.tf32 costs ~5 instructions on sm_100):
// hi keeps 10 explicit mantissa bits, lo = x - hi is exact in FP32 and is truncated
// again, so hi + lo == x to 2^-22 relative.
__device__ __forceinline__ uint32_t tf32_hi(float x) { return __float_as_uint(x) & 0xffffe000u; }
__device__ __forceinline__ void tf32_split(float x, uint32_t& hi, uint32_t& lo) {
  hi = tf32_hi(x);
  lo = tf32_hi(x - __uint_as_float(hi));
}
__device__ __forceinline__ void mma_tf32(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// DEAD_TOP: the upper 8 rows of the warp's last m-tile are padding (e.g. N_s = 70 with
// 5 m-tiles): their sigmoids are skipped at compile time (A rows = 0, no MUFU work).
template <bool HAS_MASK, bool DEAD_TOP>
__global__ void __launch_bounds__(GC_WARPS * 32, 2)
k_gp_info_tc(const float4* __restrict__ lm, int64_t n_pad, int64_t n_real, VoxSrc src, int64_t v0, int64_t v1,
             int ns, int wpv, const double* __restrict__ zs, const PairGate gate, float inv_s2, float ax,
             float bx, double* __restrict__ out64, float* __restrict__ out32) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int vpc = GC_WARPS / wpv;                                   // voxels per CTA
  float* eh = reinterpret_cast<float*>(smem_raw);                   // [vpc][GC_TILE][24] entries (FP32)
  float4* uu = reinterpret_cast<float4*>(eh + vpc * GC_TILE * 24);  // [vpc][GC_TILE] bearings
  float4* tile = uu + vpc * GC_TILE;                                // [GC_TILE][2] landmarks
  float* cs = reinterpret_cast<float*>(tile + GC_TILE * 2);         // [vpc][6] centre hi/lo
  double* acc = reinterpret_cast<double*>(cs + ((6 * vpc + 1) & ~1));  // [GC_WARPS][GC_MT*GC_NT*4][32]
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int vl = warp / wpv, mg = warp - vl * wpv;
  const int64_t vbase = v0 + blockIdx.x * (int64_t)vpc;
  const int64_t myv = vbase + vl;
  if (t < vpc) {
    const int64_t v = vbase + t;
    float ch[3], cl[3];
    voxel_split(src, v < v1 ? v : v0, ch, cl);
    for (int k = 0; k < 3; ++k) {
      cs[6 * t + k] = ch[k];
      cs[6 * t + 3 + k] = cl[k];
    }
  }
  double* myacc = acc + (size_t)warp * GC_MT * GC_NT * 4 * 32;
  for (int i = 0; i < GC_MT * GC_NT * 4; ++i) myacc[i * 32 + lane] = 0.0;
  // sample directions of this lane's A rows: rows gid and gid+8 of each m-tile; folded
  // into the exponent argument x = (ax z) . u + bx
  float zr[GC_MT][2][3];
#pragma unroll
  for (int m = 0; m < GC_MT; ++m)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int g = (mg * GC_MT + m) * 16 + gid + 8 * h;
      const bool ok = g < ns;
      zr[m][h][0] = ok ? (float)(ax * zs[3 * g]) : 0.f;
      zr[m][h][1] = ok ? (float)(ax * zs[3 * g + 1]) : 0.f;
      zr[m][h][2] = ok ? (float)(ax * zs[3 * g + 2]) : 0.f;
    }
  float c[GC_MT][GC_NT][4];
#pragma unroll
  for (int m = 0; m < GC_MT; ++m)
#pragma unroll
    for (int n = 0; n < GC_NT; ++n)
#pragma unroll
      for (int i = 0; i < 4; ++i) c[m][n][i] = 0.f;
  const int npairs = vpc * GC_TILE;
  int tiles = 0;
  for (int64_t base = 0; base < n_pad; base += GC_TILE) {
    __syncthreads();
    for (int j = t; j < GC_TILE * 2; j += blockDim.x) tile[j] = lm[2 * base + j];
    __syncthreads();
    // phase A: per (voxel, landmark) bearing + 21 entries, entries split to TF32 hi/lo
    for (int pidx = t; pidx < npairs; pidx += blockDim.x) {
      const int pv = pidx / GC_TILE, pj = pidx - pv * GC_TILE;
      float4 a = tile[2 * pj], b = tile[2 * pj + 1];
      if ((vbase + pv) >= v1) b.w = 0.f;
      if (HAS_MASK) {
        const int64_t i = base + pj;
        if (b.w != 0.f && !gate_keep(gate, vbase + pv, i)) b.w = 0.f;
      }
      const float* cc = cs + 6 * pv;
      const float ch[3] = {cc[0], cc[1], cc[2]}, cl[3] = {cc[3], cc[4], cc[5]};
      const PairF q = pair_prologue(a, b, ch, cl, inv_s2);
      float e[21];
      entries21(q, a, e);
      float4* dh = reinterpret_cast<float4*>(eh + (pv * GC_TILE + pj) * 24);
#pragma unroll
      for (int k = 0; k < 5; ++k) dh[k] = make_float4(e[4 * k], e[4 * k + 1], e[4 * k + 2], e[4 * k + 3]);
      dh[5] = make_float4(e[20], 0.f, 0.f, 0.f);
      uu[pv * GC_TILE + pj] = make_float4(q.ux, q.uy, q.uz, 0.f);
    }
    __syncthreads();
    if (vl < vpc) {
      const float* ehv = eh + vl * GC_TILE * 24;
      const float4* uv = uu + vl * GC_TILE;
      // A fragments (TF32 hi/lo) for one k-step: all 20 sigmoid chains of the 5 m-tiles
      // are independent, so their MUFU latencies overlap; the next k-step's fragments are
      // computed while the tensor pipe works through this step's 45 MMAs.
      // a0 (row gid, col tig), a1 (row gid+8, col tig), a2 (row gid, col tig+4), a3 (row gid+8, col tig+4)
      // sigmoids of m-tile m for landmarks k0 + {tig, tig+4}, split to TF32 hi/lo
      auto afrag_m = [&](int k0, int m, uint32_t (&ah)[4], uint32_t (&al)[4]) {
        const float4 u0 = uv[k0 + tig], u1 = uv[k0 + tig + 4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int h = i & 1;
          if (DEAD_TOP && h == 1 && m == GC_MT - 1) {
            ah[i] = al[i] = 0u;
            continue;
          }
          const float4 u = (i < 2) ? u0 : u1;
          const float x = fmaf(u.x, zr[m][h][0], fmaf(u.y, zr[m][h][1], fmaf(u.z, zr[m][h][2], bx)));
          tf32_split(rcp_approx(1.0f + ex2_approx(x)), ah[i], al[i]);
        }
      };
      uint32_t ah[GC_MT][4], al[GC_MT][4];
#pragma unroll
      for (int m = 0; m < GC_MT; ++m) afrag_m(0, m, ah[m], al[m]);
#pragma unroll 1
      for (int k0 = 0; k0 < GC_TILE; k0 += 8) {
        // B fragments: rows (landmarks) k0+tig, k0+tig+4; column (entry) 8n + gid
        // (each (landmark, entry) element is held by exactly one lane: split here, once)
        uint32_t bh[GC_NT][2], bl[GC_NT][2];
#pragma unroll
        for (int n = 0; n < GC_NT; ++n) {
          tf32_split(ehv[(k0 + tig) * 24 + 8 * n + gid], bh[n][0], bl[n][0]);
          tf32_split(ehv[(k0 + tig + 4) * 24 + 8 * n + gid], bh[n][1], bl[n][1]);
        }
        const int kn = (k0 + 8) & (GC_TILE - 1);  // next step (wraps harmlessly on the last)
        uint32_t nh[GC_MT][4], nl[GC_MT][4];
        // The MMA passes (15 accumulators each, so dependent MMAs are 15 apart) are
        // interleaved with the next step's sigmoid chains so the MUFU pipe and the
        // tensor pipe work at the same time inside one warp.
#pragma unroll
        for (int m = 0; m < GC_MT; ++m)
#pragma unroll
          for (int n = 0; n < GC_NT; ++n) mma_tf32(c[m][n], ah[m], bh[n][0], bh[n][1]);
        afrag_m(kn, 0, nh[0], nl[0]);
        afrag_m(kn, 1, nh[1], nl[1]);
#pragma unroll
        for (int m = 0; m < GC_MT; ++m)
#pragma unroll
          for (int n = 0; n < GC_NT; ++n) mma_tf32(c[m][n], ah[m], bl[n][0], bl[n][1]);
        afrag_m(kn, 2, nh[2], nl[2]);
        afrag_m(kn, 3, nh[3], nl[3]);
#pragma unroll
        for (int m = 0; m < GC_MT; ++m)
#pragma unroll
          for (int n = 0; n < GC_NT; ++n) mma_tf32(c[m][n], al[m], bh[n][0], bh[n][1]);
        afrag_m(kn, 4, nh[4], nl[4]);
#pragma unroll
        for (int m = 0; m < GC_MT; ++m)
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            ah[m][i] = nh[m][i];
            al[m][i] = nl[m][i];
          }
      }
      if (++tiles == GC_FLUSH_TILES || base + GC_TILE >= n_pad) {
        tiles = 0;
#pragma unroll
        for (int m = 0; m < GC_MT; ++m)
#pragma unroll
          for (int n = 0; n < GC_NT; ++n)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              myacc[((m * GC_NT + n) * 4 + i) * 32 + lane] += (double)c[m][n][i];
              c[m][n][i] = 0.f;
            }
      }
    }
  }
  if (vl < vpc && myv < v1) {
    const int64_t r = myv - v0;
    // C fragment: c0 (row gid, col 2tig), c1 (row gid, col 2tig+1), c2 (row gid+8, 2tig), c3 (row gid+8, 2tig+1)
#pragma unroll
    for (int m = 0; m < GC_MT; ++m)
#pragma unroll
      for (int n = 0; n < GC_NT; ++n)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int g = (mg * GC_MT + m) * 16 + gid + ((i >> 1) << 3);
          const int en = 8 * n + 2 * tig + (i & 1);
          if (g >= ns || en >= 21) continue;
          const double v = myacc[((m * GC_NT + n) * 4 + i) * 32 + lane];
          out64[(r * ns + g) * 21 + en] = v;
          if (out32) out32[(r * ns + g) * 21 + en] = (float)v;
        }
  }
}

// ─────────────────── GP, info on the tensor pipe: FP16 split ─────────────
// Same contraction as k_gp_info_tc, as mma.sync m16n8k16 with FP16 operands: one MMA
// covers 16 landmarks (twice the TF32 k8 step at the same instruction cost), with the
// same 3-term split (hi*hi + hi*lo + lo*hi: ~22-bit products, FP32 accumulation).
// FP16's range is managed by exact power-of-two scales:
//   A' = 2^12 vs (sigmoid in (0, 1]; the scale folds into the reciprocal's argument),
//   B' = s E with s = 2^(13 - floor(log2 max|E|)) per voxel, lowered (and the FP32
//   accumulators rescaled by the same power of two) whenever a landmark tile holds a
//   larger entry, reset after every FP64 flush; the flush divides by 2^12 s exactly.
// Entries below max|E| 2^-17 keep an absolute error <= 2^-37 max|E| (FP16 subnormal
// spacing), far under the FP32 accumulation error of the voxel's sums.
// phase A (bearings, entries) for two voxels at once on FP32x2 pairs: 160.2 -> 156.4 ms
#ifndef GH_PACKED_A
#define GH_PACKED_A 1
#endif
// exponent arguments of rows gid / gid + 8 as FFMA2 pairs (u splats, zs pairs) and their
// 2^-12 (1 + 2^x) as one FFMA2: 165.0 -> 160.6 ms, bit-identical results
#ifndef GH_XPAIR
#define GH_XPAIR 1
#endif
// one reciprocal per pair of sigmoids (1 / (y0 y1)): 165.1 -> 164.0 ms, but it needs
// |x| <= 62 (a host-checked template variant would double the instantiations; the clamp
// that avoids it costs more than the gain: 166.5 ms) -- off
#ifndef GH_PAIR_RCP
#define GH_PAIR_RCP 0
#endif
// packed FP32x2 arithmetic where pairs of sigmoids or entries meet (bit mask):
// 1 split residuals (FADD2), 2 sigmoid denominators (FFMA2), 4 B-operand scaling (FMUL2).
// With the row-paired exponent arguments (GH_XPAIR) the residual pairs need register
// moves: 2 alone is best (155.4 ms vs 156.2 with 3 and 157.2 with 7)
#ifndef GH_PACKED
#define GH_PACKED 2
#endif
__device__ __forceinline__ void h16_split2(float x0, float x1, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(x0, x1);
  const float2 b = __half22float2(h);
#if GH_PACKED & 1
  f32x2 d;  // both residuals in one packed FP32x2 subtraction
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(pack2(x0, x1)), "l"(pack2(b.x, b.y)));
  float d0, d1;
  unpack2(d, d0, d1);
  const __half2 l = __floats2half2_rn(d0, d1);
#else
  const __half2 l = __floats2half2_rn(x0 - b.x, x1 - b.y);
#endif
  hi = *reinterpret_cast<const uint32_t*>(&h);
  lo = *reinterpret_cast<const uint32_t*>(&l);
}
__device__ __forceinline__ void mma_f16(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
#ifdef GH_NO_MMA  // timing probe only (wrong results): the kernel without its tensor-core work
  c[0] += __uint_as_float((a[0] ^ a[1] ^ a[2] ^ a[3] ^ b0 ^ b1) & 0x3f800000u);
  return;
#endif
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
constexpr int H16_BEXP = 13;  // |B'| < 2^14
#ifndef GH_WARPS
#define GH_WARPS 4  // warps (voxels) per CTA
#endif
#ifndef GH_MINB
#define GH_MINB 3  // 12 warps per SM when the shared memory allows it (N_s <= 70)
#endif
// sample m16 tiles whose sigmoid reciprocals run as packed FMA-pipe Newton (the rest on
// MUFU).  Measured on config 2: 0 tiles 166.1 ms, 2: 168.9, 3: 173.5, 5: 187.9 -- MUFU
// stays (the kernel is issue/latency-limited, not MUFU-throughput-limited).
#ifndef GH_NR_MT
#define GH_NR_MT 0
#endif

template <bool HAS_MASK, bool DEAD_TOP>
__global__ void __launch_bounds__(GH_WARPS * 32, GH_MINB)
k_gp_info_h16(const float4* __restrict__ lm, int64_t n_pad, int64_t n_real, VoxSrc src, int64_t v0, int64_t v1,
              int ns, int wpv, const double* __restrict__ zs, const PairGate gate, float inv_s2, float ax,
              float bx, double* __restrict__ out64, float* __restrict__ out32) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int vpc = GH_WARPS / wpv;                                   // voxels per CTA
  float* eh = reinterpret_cast<float*>(smem_raw);                   // [vpc][GC_TILE][21] entries (FP32)
  float4* uu = reinterpret_cast<float4*>(eh + ((vpc * GC_TILE * 21 + 3) & ~3));  // [vpc][GC_TILE] bearings
  float4* tile = uu + vpc * GC_TILE;                                // [GC_TILE][2] landmarks
  float* cs = reinterpret_cast<float*>(tile + GC_TILE * 2);         // [vpc][6] centre hi/lo
  int* tmax = reinterpret_cast<int*>(cs + 6 * GH_WARPS);            // [vpc] max |entry| of the tile (bits)
  double* acc = reinterpret_cast<double*>(tmax + 2 * GH_WARPS);     // [GH_WARPS][rw][21] FP64 sums (valid rows only)
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int gid = lane >> 2, tig = lane & 3;
  const int vl = warp / wpv, mg = warp - vl * wpv;
  const int64_t vbase = v0 + blockIdx.x * (int64_t)vpc;
  const int64_t myv = vbase + vl;
  if (t < vpc) {
    const int64_t v = vbase + t;
    float ch[3], cl[3];
    voxel_split(src, v < v1 ? v : v0, ch, cl);
    for (int k = 0; k < 3; ++k) {
      cs[6 * t + k] = ch[k];
      cs[6 * t + 3 + k] = cl[k];
    }
  }
  const int rw = min(GC_MT * 16, ns);                               // sample rows per warp slot
  const int g0 = mg * GC_MT * 16;                                   // first sample row of this warp
  double* myacc = acc + (size_t)warp * rw * 21;
  for (int i = lane; i < rw * 21; i += 32) myacc[i] = 0.0;
  float zr[GC_MT][2][3];
#pragma unroll
  for (int m = 0; m < GC_MT; ++m)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int g = (mg * GC_MT + m) * 16 + gid + 8 * h;
      const bool ok = g < ns;
      zr[m][h][0] = ok ? (float)(ax * zs[3 * g]) : 0.f;
      zr[m][h][1] = ok ? (float)(ax * zs[3 * g + 1]) : 0.f;
      zr[m][h][2] = ok ? (float)(ax * zs[3 * g + 2]) : 0.f;
    }
#if GH_XPAIR
  // rows gid and gid + 8 of each m-tile as FP32x2 pairs: the exponent arguments of both
  // rows come out of three FFMA2 per landmark
  f32x2 zr2[GC_MT][3];
#pragma unroll
  for (int m = 0; m < GC_MT; ++m)
#pragma unroll
    for (int c3 = 0; c3 < 3; ++c3) zr2[m][c3] = pack2(zr[m][0][c3], zr[m][1][c3]);
  const f32x2 bx2 = splat2(bx);
#endif
  float c[GC_MT][GC_NT][4];
#pragma unroll
  for (int m = 0; m < GC_MT; ++m)
#pragma unroll
    for (int n = 0; n < GC_NT; ++n)
#pragma unroll
      for (int i = 0; i < 4; ++i) c[m][n][i] = 0.f;
  float s_cur = 0x1p100f;  // B scale of the current FP32 accumulation span (power of two)
  const int npairs = vpc * GC_TILE;
  int tiles = 0;
  for (int64_t base = 0; base < n_pad; base += GC_TILE) {
    __syncthreads();
    for (int j = t; j < GC_TILE * 2; j += blockDim.x) tile[j] = lm[2 * base + j];
    if (t < vpc) tmax[t] = 0;
    __syncthreads();
    // phase A: per (voxel, landmark) bearing + 21 entries, and the voxel's max |entry|
#if GH_PACKED_A
    if (npairs == 2 * (int)blockDim.x) {  // two voxels per thread (pv, pv + blockDim / tile) against landmark pj, packed
      const int pv = t / GC_TILE, pj = t - pv * GC_TILE;  // warp-uniform pv (32 | GC_TILE)
      const float4 a = tile[2 * pj], b = tile[2 * pj + 1];
      const int pv2 = pv + (int)blockDim.x / GC_TILE;  // the thread's second voxel
      bool okA = b.w != 0.f && (vbase + pv) < v1, okB = b.w != 0.f && (vbase + pv2) < v1;
      if (HAS_MASK) {
        const int64_t i = base + pj;
        if (okA && !gate_keep(gate, vbase + pv, i)) okA = false;
        if (okB && !gate_keep(gate, vbase + pv2, i)) okB = false;
      }
      const float* cA = cs + 6 * pv;
      const float* cB = cs + 6 * pv2;
      const f32x2 ch2[3] = {pack2(cA[0], cB[0]), pack2(cA[1], cB[1]), pack2(cA[2], cB[2])};
      const f32x2 cl2[3] = {pack2(cA[3], cB[3]), pack2(cA[4], cB[4]), pack2(cA[5], cB[5])};
      const PairF2 q = pair_prologue2(a, b, ch2, cl2, inv_s2, okA, okB);
      f32x2 e[21];
      entries21x2(q, a, e);
      // |entry| <= w max(1, 2|p|, |p|^2) <= w (1 + |p|^2) (|c2| <= |p|); x2 covers FP32 rounding
      float mxA, mxB;
      unpack2(ffma2(splat2(a.w), fmul2(splat2(2.0f), q.w), fmul2(splat2(2.0f), q.w)), mxA, mxB);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        mxA = fmaxf(mxA, __shfl_xor_sync(0xffffffffu, mxA, o));
        mxB = fmaxf(mxB, __shfl_xor_sync(0xffffffffu, mxB, o));
      }
      if (lane == 0) {
        atomicMax(&tmax[pv], __float_as_int(mxA));
        atomicMax(&tmax[pv2], __float_as_int(mxB));
      }
      float* dA = eh + (pv * GC_TILE + pj) * 21;
      float* dB = eh + (pv2 * GC_TILE + pj) * 21;
#pragma unroll
      for (int k2 = 0; k2 < 21; ++k2) unpack2(e[k2], dA[k2], dB[k2]);
      float uxA, uxB, uyA, uyB, uzA, uzB;
      unpack2(q.ux, uxA, uxB);
      unpack2(q.uy, uyA, uyB);
      unpack2(q.uz, uzA, uzB);
      uu[pv * GC_TILE + pj] = make_float4(uxA, uyA, uzA, 0.f);
      uu[pv2 * GC_TILE + pj] = make_float4(uxB, uyB, uzB, 0.f);
    } else
#endif
    for (int pidx = t; pidx < npairs; pidx += blockDim.x) {
      const int pv = pidx / GC_TILE, pj = pidx - pv * GC_TILE;  // warp-uniform pv (32 | GC_TILE)
      float4 a = tile[2 * pj], b = tile[2 * pj + 1];
      if ((vbase + pv) >= v1) b.w = 0.f;
      if (HAS_MASK) {
        const int64_t i = base + pj;
        if (b.w != 0.f && !gate_keep(gate, vbase + pv, i)) b.w = 0.f;
      }
      const float* cc = cs + 6 * pv;
      const float ch[3] = {cc[0], cc[1], cc[2]}, cl[3] = {cc[3], cc[4], cc[5]};
      const PairF q = pair_prologue(a, b, ch, cl, inv_s2);
      float e[21];
      entries21(q, a, e);
      // |entry| <= w max(1, 2|p|, |p|^2) <= w (1 + |p|^2) (|c2| <= |p|); x2 covers FP32 rounding
      float mx = fmaf(a.w, 2.0f * q.w, 2.0f * q.w);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (lane == 0) atomicMax(&tmax[pv], __float_as_int(mx));
      float* dh = eh + (pv * GC_TILE + pj) * 21;
#pragma unroll
      for (int k = 0; k < 21; ++k) dh[k] = e[k];
      uu[pv * GC_TILE + pj] = make_float4(q.ux, q.uy, q.uz, 0.f);
    }
    __syncthreads();
    if (vl < vpc) {
      const float tm = __int_as_float(tmax[vl]);
      if (tm > 0.f) {  // lower the B scale if this tile holds a larger entry (exact rescale)
        const int ex = ((__float_as_int(tm) >> 23) & 0xff) - 127;
        const int be = min(254, max(1, 127 + H16_BEXP - ex));
        const float s_need = __int_as_float(be << 23);
        if (s_need < s_cur) {
          const float r = s_need / s_cur;
#pragma unroll
          for (int m = 0; m < GC_MT; ++m)
#pragma unroll
            for (int n = 0; n < GC_NT; ++n)
#pragma unroll
              for (int i = 0; i < 4; ++i) c[m][n][i] *= r;
          s_cur = s_need;
        }
      }
      // entries 21..23 of an n8 tile read the next pair's values: they only feed the
      // discarded accumulator columns 21..23 (each MMA output column is independent)
      const float* ehv = eh + vl * GC_TILE * 21;
      const float4* uv = uu + vl * GC_TILE;
      // A fragment (m16n8k16, f16): reg0 (row gid, k 2tig..+1), reg1 (row gid+8, k 2tig..+1),
      // reg2 (row gid, k 2tig+8..+9), reg3 (row gid+8, k 2tig+8..+9); low half = lower k
#if GH_XPAIR
      auto afrag_m = [&](int k0, int m, uint32_t (&ah)[4], uint32_t (&al)[4]) {
        const float4 u[4] = {uv[k0 + 2 * tig], uv[k0 + 2 * tig + 1], uv[k0 + 2 * tig + 8], uv[k0 + 2 * tig + 9]};
        if (DEAD_TOP && m == GC_MT - 1) {  // rows gid + 8 are padding: row gid alone
#pragma unroll
          for (int r = 0; r < 4; r += 2) {
            const int kb = r;
            float sg[2];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const float4 uj = u[kb + j];
              const float x = fmaf(uj.x, zr[m][0][0], fmaf(uj.y, zr[m][0][1], fmaf(uj.z, zr[m][0][2], bx)));
              sg[j] = rcp_approx(fmaf(ex2_approx(x), 0x1p-12f, 0x1p-12f));
            }
            h16_split2(sg[0], sg[1], ah[r], al[r]);
            ah[r + 1] = al[r + 1] = 0u;
          }
          return;
        }
#pragma unroll
        for (int kb = 0; kb < 4; kb += 2) {
          float sg[2][2];  // [row half h][landmark j]
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const float4 uj = u[kb + j];
            const f32x2 x2 = ffma2(splat2(uj.x), zr2[m][0], ffma2(splat2(uj.y), zr2[m][1], ffma2(splat2(uj.z), zr2[m][2], bx2)));
            float x0, x1;
            unpack2(x2, x0, x1);
            float y0, y1;  // 2^-12 (1 + 2^x) for both rows, one FFMA2
            unpack2(ffma2(pack2(ex2_approx(x0), ex2_approx(x1)), splat2(0x1p-12f), splat2(0x1p-12f)), y0, y1);
            sg[0][j] = rcp_approx(y0);
            sg[1][j] = rcp_approx(y1);
          }
          h16_split2(sg[0][0], sg[0][1], ah[kb], al[kb]);          // reg kb: row gid
          h16_split2(sg[1][0], sg[1][1], ah[kb + 1], al[kb + 1]);  // reg kb + 1: row gid + 8
        }
      };
#else
      auto afrag_m = [&](int k0, int m, uint32_t (&ah)[4], uint32_t (&al)[4]) {
        const float4 u[4] = {uv[k0 + 2 * tig], uv[k0 + 2 * tig + 1], uv[k0 + 2 * tig + 8], uv[k0 + 2 * tig + 9]};
#pragma unroll
        for (int r = 0; r < 4; ++r) {
          const int h = r & 1, kb = (r >> 1) * 2;
          if (DEAD_TOP && h == 1 && m == GC_MT - 1) {
            ah[r] = al[r] = 0u;
            continue;
          }
          float sg[2];
          if (m < GH_NR_MT) {  // reciprocal on the FMA pipe (packed Newton), x clamped so y stays finite
            float ex[2];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const float4 uj = u[kb + j];
              const float x = fmaf(uj.x, zr[m][h][0], fmaf(uj.y, zr[m][h][1], fmaf(uj.z, zr[m][h][2], bx)));
              ex[j] = ex2_approx(fminf(x, 126.f));
            }
            const f32x2 ny = ffma2(pack2(ex[0], ex[1]), splat2(-0x1p-12f), splat2(-0x1p-12f));
            unpack2(rcp_nr2_neg(ny), sg[0], sg[1]);  // 2^12 / (1 + 2^x)
          } else {
#if GH_PAIR_RCP
            // one reciprocal for both: r = 1 / (y0 y1), sg0 = y1 r, sg1 = y0 r; x <= 63 keeps
            // the product finite (a sigmoid below 2^-63 is then off by < 2^-63 absolute)
            float ex[2];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const float4 uj = u[kb + j];
              ex[j] = ex2_approx(fminf(fmaf(uj.x, zr[m][h][0], fmaf(uj.y, zr[m][h][1], fmaf(uj.z, zr[m][h][2], bx))), 63.f));
            }
            const float y0 = fmaf(ex[0], 0x1p-12f, 0x1p-12f), y1 = fmaf(ex[1], 0x1p-12f, 0x1p-12f);
            const float r = rcp_approx(y0 * y1);
            sg[0] = y1 * r;
            sg[1] = y0 * r;
#elif GH_PACKED & 2
            float ex[2];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const float4 uj = u[kb + j];
              ex[j] = ex2_approx(fmaf(uj.x, zr[m][h][0], fmaf(uj.y, zr[m][h][1], fmaf(uj.z, zr[m][h][2], bx))));
            }
            float y0, y1;  // 2^-12 (1 + 2^x) for both, one FFMA2
            unpack2(ffma2(pack2(ex[0], ex[1]), splat2(0x1p-12f), splat2(0x1p-12f)), y0, y1);
            sg[0] = rcp_approx(y0);  // 2^12 / (1 + 2^x)
            sg[1] = rcp_approx(y1);
#else
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const float4 uj = u[kb + j];
              const float x = fmaf(uj.x, zr[m][h][0], fmaf(uj.y, zr[m][h][1], fmaf(uj.z, zr[m][h][2], bx)));
              sg[j] = rcp_approx(fmaf(ex2_approx(x), 0x1p-12f, 0x1p-12f));  // 2^12 / (1 + 2^x)
            }
#endif
          }
          h16_split2(sg[0], sg[1], ah[r], al[r]);
        }
      };
#endif
      uint32_t ah[GC_MT][4], al[GC_MT][4];
#pragma unroll
      for (int m = 0; m < GC_MT; ++m) afrag_m(0, m, ah[m], al[m]);
      // one k16 step; NEXT: the following step's sigmoids are evaluated between the MMA
      // passes (the tile's last step has no successor: its passes run back to back, so
      // no sigmoid is computed twice)
      auto kstep = [&](int k0, auto next_tag) {
        constexpr bool NEXT = decltype(next_tag)::value;
        // B fragment (f16): reg0 (k 2tig..+1, col gid), reg1 (k 2tig+8..+9, col gid)
        uint32_t bh[GC_NT][2], bl[GC_NT][2];
#pragma unroll
        for (int n = 0; n < GC_NT; ++n) {
          const float* eb = ehv + 8 * n + gid;
#if GH_PACKED & 4
          float b0, b1, b2, b3;  // scaled by s_cur, two FMUL2
          unpack2(fmul2(pack2(eb[(k0 + 2 * tig) * 21], eb[(k0 + 2 * tig + 1) * 21]), splat2(s_cur)), b0, b1);
          unpack2(fmul2(pack2(eb[(k0 + 2 * tig + 8) * 21], eb[(k0 + 2 * tig + 9) * 21]), splat2(s_cur)), b2, b3);
          h16_split2(b0, b1, bh[n][0], bl[n][0]);
          h16_split2(b2, b3, bh[n][1], bl[n][1]);
#else
          h16_split2(eb[(k0 + 2 * tig) * 21] * s_cur, eb[(k0 + 2 * tig + 1) * 21] * s_cur, bh[n][0], bl[n][0]);
          h16_split2(eb[(k0 + 2 * tig + 8) * 21] * s_cur, eb[(k0 + 2 * tig + 9) * 21] * s_cur, bh[n][1], bl[n][1]);
#endif
        }
        const int kn = k0 + 16;
        uint32_t nh[GC_MT][4], nl[GC_MT][4];
#pragma unroll
        for (int m = 0; m < GC_MT; ++m)
#pragma unroll
          for (int n = 0; n < GC_NT; ++n) mma_f16(c[m][n], ah[m], bh[n][0], bh[n][1]);
        if (NEXT) {
          afrag_m(kn, 0, nh[0], nl[0]);
          afrag_m(kn, 1, nh[1], nl[1]);
        }
#pragma unroll
        for (int m = 0; m < GC_MT; ++m)
#pragma unroll
          for (int n = 0; n < GC_NT; ++n) mma_f16(c[m][n], ah[m], bl[n][0], bl[n][1]);
        if (NEXT) {
          afrag_m(kn, 2, nh[2], nl[2]);
          afrag_m(kn, 3, nh[3], nl[3]);
        }
#pragma unroll
        for (int m = 0; m < GC_MT; ++m)
#pragma unroll
          for (int n = 0; n < GC_NT; ++n) mma_f16(c[m][n], al[m], bh[n][0], bh[n][1]);
        if (NEXT) {
          afrag_m(kn, 4, nh[4], nl[4]);
#pragma unroll
          for (int m = 0; m < GC_MT; ++m)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              ah[m][i] = nh[m][i];
              al[m][i] = nl[m][i];
            }
        }
      };
#pragma unroll 1
      for (int k0 = 0; k0 < GC_TILE - 16; k0 += 16) kstep(k0, std::true_type{});
      kstep(GC_TILE - 16, std::false_type{});
      if (++tiles == GC_FLUSH_TILES || base + GC_TILE >= n_pad) {
        tiles = 0;
        const double unscale = 0x1p-12 / (double)s_cur;  // exact power of two
#pragma unroll
        for (int m = 0; m < GC_MT; ++m)
#pragma unroll
          for (int n = 0; n < GC_NT; ++n)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int gl = m * 16 + gid + ((i >> 1) << 3), en = 8 * n + 2 * tig + (i & 1);
              if (g0 + gl < ns && en < 21) myacc[gl * 21 + en] += (double)c[m][n][i] * unscale;
              c[m][n][i] = 0.f;
            }
        s_cur = 0x1p100f;
      }
    }
  }
  if (vl < vpc && myv < v1) {
    const int64_t ob = ((myv - v0) * ns + g0) * 21;
    const int tot = min(GC_MT * 16, ns - g0) * 21;
    for (int i = lane; i < tot; i += 32) {
      const double v = myacc[i];
      out64[ob + i] = v;
      if (out32) out32[ob + i] = (float)v;
    }
  }
}

#include "fif_gp_t5.cuh"
#include "fif_gp_t6.cuh"

// ─────────────────────────── exports ───────────────────────────────────
// Expand packed (rows, nv, 21) to the reference's (rows, nv*36).
__global__ void k_expand36(const double* __restrict__ in, int64_t blocks, double* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= blocks * 36) return;
  int64_t b = i / 36;
  int rc = (int)(i - b * 36), r = rc / 6, c = rc - r * 6;
  int lo = r < c ? r : c, hi = r < c ? c : r;
  out[i] = in[b * 21 + packed_index(lo, hi)];
}

// F = kinv @ S per voxel (kinv symmetric; reference factor of kernels.py:511-523).
// S (rows, ns, W), W = 1 (trace) or 21 (info); out (rows, ns, W) f64.
__global__ void k_gp_apply_kinv(const double* __restrict__ S, int64_t rows, int ns, int W,
                                const double* __restrict__ kinv, double* __restrict__ out) {
  extern __shared__ double sm[];  // S row [ns*W]
  const int64_t r = blockIdx.x;
  const int n = ns * W;
  for (int j = threadIdx.x; j < n; j += blockDim.x) sm[j] = S[r * n + j];
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    int k = j / W, e = j - k * W;
    double s = 0.0;
    for (int gidx = 0; gidx < ns; ++gidx) s = fma(kinv[(int64_t)k * ns + gidx], sm[gidx * W + e], s);
    out[r * n + j] = s;
  }
}

// Reference-layout export of GP rows (N_s <= 84): out = kinv @ S per voxel, expanded to the
// reference's 36 entries per block in the same kernel (info) -- the GEMM kinv (N_s x N_s) x
// [S_v0 | S_v1 | ...] over groups of voxels, FP64.  kinv is staged once per persistent CTA,
// transposed (kT[g][k] = kinv[k][g]) so a thread's 28 consecutive k for one g are 14
// broadcast LDS.128; thread = (column c = voxel-in-group x entry, k group of 28), 28 FP64
// register accumulators, the same fma(kinv[k][g], S[g][e], acc) chain in g order as
// k_gp_apply_kinv (bit-identical output).  Columns per CTA: 84 = 4 voxels x 21 (info) or
// 84 voxels x 1 (trace).
constexpr int GX_NC = 84, GX_KG = 28, GX_KS = 84;  // columns, k per thread group, kT row stride
template <int W>
__global__ void __launch_bounds__(256, 2) k_gp_export(const double* __restrict__ S, int64_t rows, int ns,
                                                      const double* __restrict__ kinv, double* __restrict__ out) {
  constexpr int VB = GX_NC / W;
  extern __shared__ __align__(16) double gx_sm[];
  double* kT = gx_sm;                   // [ns][GX_KS]
  double* st = gx_sm + ns * GX_KS;      // [ns][GX_NC]
  for (int i = threadIdx.x; i < ns * GX_KS; i += blockDim.x) {
    const int g = i / GX_KS, k = i - g * GX_KS;
    kT[i] = k < ns ? kinv[(int64_t)k * ns + g] : 0.0;
  }
  const int t = threadIdx.x, grp = t / GX_NC, c = t - grp * GX_NC, k0 = GX_KG * grp;
  const int vb = c / W, e = c - vb * W;
  int plo = 0, phi = 0;  // packed entry e -> (row, col) of the upper triangle
  if (W == 21) {
    int r = 0, rem = e;
    while (rem >= 6 - r) rem -= 6 - r, ++r;
    plo = r;
    phi = r + rem;
  }
  const int64_t groups = (rows + VB - 1) / VB;
  for (int64_t gi = blockIdx.x; gi < groups; gi += gridDim.x) {
    const int64_t v0 = gi * VB;
    const int nvb = (int)(rows - v0 < VB ? rows - v0 : VB);
    __syncthreads();  // previous group's tile consumed (and kT written, first time)
    for (int i = threadIdx.x; i < VB * ns * W; i += blockDim.x) {
      const int b = i / (ns * W), r = i - b * (ns * W), g = r / W, ee = r - g * W;
      st[g * GX_NC + b * W + ee] = b < nvb ? S[(v0 + b) * ns * W + r] : 0.0;
    }
    __syncthreads();
    if (grp < 3 && k0 < ns && vb < nvb) {
      double acc[GX_KG];
#pragma unroll
      for (int i = 0; i < GX_KG; ++i) acc[i] = 0.0;
      for (int g = 0; g < ns; ++g) {
        const double sv = st[g * GX_NC + c];
        const double2* kp = reinterpret_cast<const double2*>(kT + g * GX_KS + k0);
#pragma unroll
        for (int i = 0; i < GX_KG / 2; ++i) {
          const double2 kk = kp[i];
          acc[2 * i] = fma(kk.x, sv, acc[2 * i]);
          acc[2 * i + 1] = fma(kk.y, sv, acc[2 * i + 1]);
        }
      }
      const int64_t v = v0 + vb;
#pragma unroll
      for (int i = 0; i < GX_KG; ++i) {
        const int k = k0 + i;
        if (k < ns) {
          if (W == 21) {
            double* o = out + (v * ns + k) * 36;
            o[plo * 6 + phi] = acc[i];
            if (plo != phi) o[phi * 6 + plo] = acc[i];
          } else {
            out[v * ns + k] = acc[i];
          }
        }
      }
    }
  }
}

}  // namespace fif

using namespace fif;

extern "C" int64_t fif_build_scratch_bytes(int64_t n_points) {
  int64_t n_pad = ((n_points + kLmPad - 1) / kLmPad) * kLmPad;
  if (n_pad == 0) n_pad = kLmPad;
  return n_pad * 2 * (int64_t)sizeof(float4);
}

// The build proper; `gate` (when has_gate) is the per-pair matchability test: an explicit
// mask (fif_build) or the fused gate predicates (fif_build_matched).
static int build_impl(int factor_kind, const fif_model* model, const double* d_points, int64_t n_points,
                      const fif_grid* grid, const double* d_centers, int64_t v_begin, int64_t v_end, PairGate gate,
                      bool has_gate, double sigma, uint32_t build_flags, void* d_scratch, double* d_out64,
                      float* d_out32, void* stream) {
  FIF_CHECK_ARG(model != nullptr, "fif_build: model is NULL");
  FIF_CHECK_ARG(factor_kind == FIF_KIND_INFO || factor_kind == FIF_KIND_TRACE, "fif_build: bad factor_kind %d",
                factor_kind);
  FIF_CHECK_ARG(model->kind == FIF_MODEL_QUAD || model->kind == FIF_MODEL_GP, "fif_build: bad model kind %d",
                model->kind);
  FIF_CHECK_ARG(v_end >= v_begin && v_begin >= 0, "fif_build: bad voxel range [%lld,%lld)", (long long)v_begin,
                (long long)v_end);
  FIF_CHECK_ARG(d_out64 != nullptr, "fif_build: d_out64 is NULL");
  FIF_CHECK_ARG(sigma > 0, "fif_build: sigma must be positive");
  FIF_CHECK_ARG(n_points >= 0, "fif_build: n_points < 0");
  FIF_CHECK_ARG(n_points == 0 || d_points != nullptr, "fif_build: d_points is NULL");
  FIF_CHECK_ARG(d_centers != nullptr || grid != nullptr, "fif_build: need a grid or explicit centres");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t rows = v_end - v_begin;
  const bool trace = factor_kind == FIF_KIND_TRACE;
  const int nv = model->kind == FIF_MODEL_QUAD ? 10 : model->n_v;
  const int64_t width = trace ? nv : (int64_t)nv * 21;
  if (rows == 0) return FIF_OK;
  if (n_points == 0) {
    // no landmarks: every factor is exactly zero (field.py:248-252 builds an empty map)
    cudaMemsetAsync(d_out64, 0, sizeof(double) * rows * width, st);
    if (d_out32) cudaMemsetAsync(d_out32, 0, sizeof(float) * rows * width, st);
    FIF_CHECK_LAUNCH("fif_build(memset)");
    return FIF_OK;
  }
  VoxSrc src{};
  src.centers = d_centers;
  if (grid) {
    src.ox = grid->origin[0];
    src.oy = grid->origin[1];
    src.oz = grid->origin[2];
    src.vs = grid->voxel_size;
    src.nx = grid->dims[0];
    src.ny = grid->dims[1];
    src.nz = grid->dims[2];
    if (!d_centers) {
      FIF_CHECK_ARG(grid->voxel_size > 0 && grid->dims[0] > 0 && grid->dims[1] > 0 && grid->dims[2] > 0,
                    "fif_build: empty grid");
      FIF_CHECK_ARG(v_end <= grid->dims[0] * grid->dims[1] * grid->dims[2], "fif_build: v_end beyond grid");
    }
  }
  const double inv_s2 = 1.0 / (sigma * sigma);
  const bool has_mask = has_gate;
  gate.src = src;
  int64_t n_pad = ((n_points + kLmPad - 1) / kLmPad) * kLmPad;
  float4* lm = reinterpret_cast<float4*>(d_scratch);
  FIF_CHECK_ARG(d_scratch != nullptr || (model->kind == FIF_MODEL_GP && trace), "fif_build: d_scratch is NULL");
  const bool need_lm = model->kind == FIF_MODEL_GP && !trace;
  if (need_lm) {
    FIF_CHECK_ARG(d_scratch != nullptr, "fif_build: d_scratch is NULL");
    k_prep_landmarks<<<(unsigned)((n_pad + 255) / 256), 256, 0, st>>>(d_points, n_points, n_pad, lm);
    FIF_CHECK_LAUNCH("k_prep_landmarks");
  }
  if (model->kind == FIF_MODEL_QUAD) {
    const bool exact = (build_flags & FIF_BUILD_EXACT) != 0;
    double4* lm64 = reinterpret_cast<double4*>(d_scratch);
    k_prep_landmarks64<<<(unsigned)((n_pad + 255) / 256), 256, 0, st>>>(d_points, n_points, n_pad, lm64);
    FIF_CHECK_LAUNCH("k_prep_landmarks64");
    if (trace) {
      unsigned blocks = (unsigned)((rows + QD_THREADS - 1) / QD_THREADS);
#define QT_LAUNCH(E, M) k_quad_trace<E, M><<<blocks, QD_THREADS, 0, st>>>(lm64, n_pad, n_points, src, v_begin, v_end, gate, inv_s2, d_out64)
      if (exact) { if (has_mask) QT_LAUNCH(true, true); else QT_LAUNCH(true, false); }
      else { if (has_mask) QT_LAUNCH(false, true); else QT_LAUNCH(false, false); }
#undef QT_LAUNCH
      FIF_CHECK_LAUNCH("k_quad_trace");
    } else {
      unsigned blocks = (unsigned)((rows + 31) / 32);
      const size_t qi_smem = sizeof(double4) * QI_TILE + sizeof(double) * 7 * QI_TILE * 32;
      static std::atomic<uint64_t> qi_attr{0};
      if (needs_setup(qi_attr)) {
        for (auto f : {k_quad_info<true, true>, k_quad_info<true, false>, k_quad_info<false, true>, k_quad_info<false, false>})
          cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qi_smem);
        mark_setup(qi_attr);
      }
#define QI_LAUNCH(E, M) \
  k_quad_info<E, M><<<blocks, QI_THREADS, qi_smem, st>>>(lm64, n_pad, n_points, src, v_begin, v_end, gate, inv_s2, d_out64)
      if (exact) { if (has_mask) QI_LAUNCH(true, true); else QI_LAUNCH(true, false); }
      else { if (has_mask) QI_LAUNCH(false, true); else QI_LAUNCH(false, false); }
#undef QI_LAUNCH
      FIF_CHECK_LAUNCH("k_quad_info");
    }
    return FIF_OK;
  }
  // GP
  const int ns = model->n_v;
  FIF_CHECK_ARG(ns >= 1 && ns <= 1024, "fif_build: N_s=%d out of range", ns);
  FIF_CHECK_ARG(model->zs != nullptr, "fif_build: GP model without zs");
  // sigmoid 1/(1 + exp(-k_s (c - cos a))) = 1/(1 + 2^(c*ax + bx))
  const double LOG2E = 1.4426950408889634;
  const double ax = -model->k_s * LOG2E;
  const double bx = model->k_s * model->cos_alpha * LOG2E;
  FIF_CHECK_ARG(ns <= GI_THREADS_MAX, "fif_build: N_s=%d exceeds %d", ns, GI_THREADS_MAX);
  if (trace) {
    const int tpv = (ns + GT_G - 1) / GT_G;
    int vbt = GT_THREADS / tpv;
    if (vbt < 1) vbt = 1;
    if (vbt > 32) vbt = 32;  // N_s <= 28: the pair records of more voxels would not fit the 96 KB opt-in below
    const int threads_t = ((vbt * tpv + 31) / 32) * 32;
    FIF_CHECK_ARG(threads_t <= GT_THREADS, "fif_build: N_s=%d too large for k_gp_trace", ns);
    const unsigned blocks_t = (unsigned)((rows + vbt - 1) / vbt);
    size_t smem = sizeof(PairT) * vbt * (GT_TILE + 1) + sizeof(double) * 3 * vbt + sizeof(double) * 3 * GT_TILE;
    static std::atomic<uint64_t> carve{0};
    if (needs_setup(carve)) {
      for (auto f : {k_gp_trace<true>, k_gp_trace<false>}) {
        cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
      }
      mark_setup(carve);
    }
    if (has_mask)
      k_gp_trace<true><<<blocks_t, threads_t, smem, st>>>(d_points, n_points, src, v_begin, v_end, vbt, ns, model->zs,
                                                          gate, inv_s2, ax, bx, d_out64, d_out32);
    else
      k_gp_trace<false><<<blocks_t, threads_t, smem, st>>>(d_points, n_points, src, v_begin, v_end, vbt, ns,
                                                           model->zs, gate, inv_s2, ax, bx, d_out64, d_out32);
    FIF_CHECK_LAUNCH("k_gp_trace");
  } else if ((build_flags & FIF_BUILD_T6) && !(build_flags & (FIF_BUILD_SIMT | FIF_BUILD_TF32 | FIF_BUILD_H16)) &&
             model->zs_host != nullptr && !has_mask && ns > 8 && ns <= 8 * T6_MAX_NG && bx + fabs(ax) <= T5_XMAX &&
             fabs(ax) <= 100.0 && fabs(bx - 12.0) <= 100.0 && !T5_QUAD) {
    // tcgen05 path with the exponent arguments x' = (ax zs) . u on the tensor cores as well (one
    // M=128 K=16 MMA per voxel per 64 landmarks) and the bias folded into the sigmoid:
    // 2^-12 (1 + 2^(x' + bx)) = fma(2^x', 2^(bx - 12), 2^-12); |ax| <= 100 keeps 2^x' finite
    const int ng = (ns + 7) / 8;
    T6Z z;
    t6_fill_z(z, model->zs_host, ns, ax, (8 * ng + 15) / 16 * 16);
    const float cexp = (float)exp2(bx - 12.0);
    const unsigned blocks6 = (unsigned)((rows + T5_VOX - 1) / T5_VOX);
    int rc = FIF_OK;
#define T6_LAUNCH(NG, SKIP)                                                                                  \
  do {                                                                                                       \
    constexpr int sm = T6Layout<NG>::BYTES;                                                                  \
    static_assert(sm <= T5_SMEM_MAX, "k_gp_info_t6 shared memory");                                          \
    static std::atomic<uint64_t> attr{0};                                                                    \
    if (needs_setup(attr)) {                                                                                 \
      cudaFuncSetAttribute(k_gp_info_t6<NG, SKIP>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);         \
      mark_setup(attr);                                                                                      \
    }                                                                                                        \
    k_gp_info_t6<NG, SKIP><<<blocks6, T5_THREADS, sm, st>>>(lm, n_pad, src, v_begin, v_end, ns, (float)inv_s2, \
                                                            cexp, z, d_out64, d_out32);                      \
  } while (0)
  // (one trailing sample pair of padding, N_s <= 8 NG - 2, is skipped at compile time: N_s = 70)
#define T6_CASE(NG)                              \
  case NG:                                       \
    if (ns <= 8 * NG - 2) T6_LAUNCH(NG, 1);      \
    else T6_LAUNCH(NG, 0);                       \
    break;
    switch (ng) {
      T6_CASE(2) T6_CASE(3) T6_CASE(4) T6_CASE(5) T6_CASE(6) T6_CASE(7) T6_CASE(8) T6_CASE(9)
      default: rc = FIF_ERR_UNSUPPORTED;
    }
#undef T6_LAUNCH
#undef T6_CASE
    if (rc != FIF_OK) {
      set_error("fif_build: N_s=%d unsupported by k_gp_info_t6", ns);
      return rc;
    }
    FIF_CHECK_LAUNCH("k_gp_info_t6");
  } else if (!(build_flags & (FIF_BUILD_SIMT | FIF_BUILD_TF32 | FIF_BUILD_H16)) && model->zs_host != nullptr &&
             ns <= 8 * T5_MAX_NG && bx + fabs(ax) <= T5_XMAX) {
    // (x = (ax zs) . u + bx <= bx + |ax| <= T5_XMAX keeps the shared sigmoid reciprocal finite)
    // tcgen05 path: one tcgen05.mma (M=64, N=16 NG, K=16) per voxel per 16 landmarks, TMEM accumulators
    const int ng = (ns + 7) / 8;
    T5Z z{};
    for (int sidx = 0; sidx < ns; ++sidx)  // (pair sigmoids: sample s at slot s ^ 1, see t5_sigmoids)
      for (int c = 0; c < 3; ++c) z.z[c][T5_QUAD ? sidx : sidx ^ 1] = (float)(ax * model->zs_host[3 * sidx + c]);
    const unsigned blocks5 = (unsigned)((rows + T5_VOX - 1) / T5_VOX);
    int rc = FIF_OK;
#define T5_CASE(NG)                                                                                         \
  case NG: {                                                                                                \
    constexpr size_t sm = t5_smem_bytes<NG>();                                                              \
    const size_t gb = (size_t)T5_VOX * (n_pad / 8);                                                         \
    static const bool no_gb = getenv("FIF_T5_NO_GATE_BITS") != nullptr;                                     \
    const int use_gb = has_mask && !no_gb && sm + gb <= T5_SMEM_MAX;                                        \
    static std::atomic<uint64_t> attr{0};                                                                   \
    if (needs_setup(attr)) {                                                                                \
      cudaFuncSetAttribute(k_gp_info_t5<NG, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, T5_SMEM_MAX); \
      cudaFuncSetAttribute(k_gp_info_t5<NG, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);  \
      mark_setup(attr);                                                                                     \
    }                                                                                                       \
    if (has_mask)                                                                                           \
      k_gp_info_t5<NG, true><<<blocks5, T5_THREADS, sm + (use_gb ? gb : 0), st>>>(                            \
          lm, n_pad, src, v_begin, v_end, ns, gate, use_gb, (float)inv_s2, (float)bx, z, d_out64, d_out32);  \
    else                                                                                                    \
      k_gp_info_t5<NG, false><<<blocks5, T5_THREADS, sm, st>>>(lm, n_pad, src, v_begin, v_end, ns, gate, 0, \
                                                               (float)inv_s2, (float)bx, z, d_out64, d_out32); \
    break;                                                                                                  \
  }
    switch (ng) {
      T5_CASE(1) T5_CASE(2) T5_CASE(3) T5_CASE(4) T5_CASE(5) T5_CASE(6) T5_CASE(7) T5_CASE(8) T5_CASE(9) T5_CASE(10)
      default: rc = FIF_ERR_UNSUPPORTED;
    }
#undef T5_CASE
    if (rc != FIF_OK) {
      set_error("fif_build: N_s=%d unsupported by k_gp_info_t5", ns);
      return rc;
    }
    FIF_CHECK_LAUNCH("k_gp_info_t5");
  } else if (!(build_flags & (FIF_BUILD_SIMT | FIF_BUILD_TF32))) {
    // tensor-pipe path, FP16 split (mma.sync m16n8k16): a warp covers 80 samples of one voxel
    const int wpv = (ns + 16 * GC_MT - 1) / (16 * GC_MT);
    FIF_CHECK_ARG(wpv >= 1 && wpv <= GH_WARPS, "fif_build: N_s=%d too large for k_gp_info_h16", ns);
    const int vpc = GH_WARPS / wpv;
    const unsigned blocks_c = (unsigned)((rows + vpc - 1) / vpc);
    const int rw = ns < GC_MT * 16 ? ns : GC_MT * 16;
    size_t smem = sizeof(float) * ((vpc * GC_TILE * 21 + 3) & ~3) + sizeof(float4) * (vpc * GC_TILE + GC_TILE * 2) +
                  sizeof(float) * 6 * GH_WARPS + sizeof(int) * 2 * GH_WARPS + sizeof(double) * GH_WARPS * rw * 21;
    static std::atomic<uint64_t> carve_h{0};
    if (needs_setup(carve_h)) {
      for (auto f : {k_gp_info_h16<true, true>, k_gp_info_h16<false, true>, k_gp_info_h16<true, false>,
                     k_gp_info_h16<false, false>}) {
        cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      }
      mark_setup(carve_h);
    }
    const bool dead_top = wpv == 1 && (GC_MT - 1) * 16 + 8 >= ns;
#define GH_LAUNCH(M, D)                                                                                        \
  k_gp_info_h16<M, D><<<blocks_c, GH_WARPS * 32, smem, st>>>(lm, n_pad, n_points, src, v_begin, v_end, ns, wpv, \
                                                            model->zs, gate, (float)inv_s2, (float)ax, (float)bx, \
                                                            d_out64, d_out32)
    if (has_mask) { if (dead_top) GH_LAUNCH(true, true); else GH_LAUNCH(true, false); }
    else { if (dead_top) GH_LAUNCH(false, true); else GH_LAUNCH(false, false); }
#undef GH_LAUNCH
    FIF_CHECK_LAUNCH("k_gp_info_h16");
  } else if (!(build_flags & FIF_BUILD_SIMT)) {
    // tensor-pipe path (mma.sync TF32x3): a warp covers 80 samples of one voxel
    const int wpv = (ns + 16 * GC_MT - 1) / (16 * GC_MT);
    FIF_CHECK_ARG(wpv >= 1 && wpv <= GC_WARPS, "fif_build: N_s=%d too large for k_gp_info_tc", ns);
    const int vpc = GC_WARPS / wpv;
    const unsigned blocks_c = (unsigned)((rows + vpc - 1) / vpc);
    size_t smem = sizeof(float) * (vpc * GC_TILE * 24) + sizeof(float4) * (vpc * GC_TILE + GC_TILE * 2) +
                  sizeof(float) * ((6 * vpc + 1) & ~1) + sizeof(double) * GC_WARPS * GC_MT * GC_NT * 4 * 32;
    static std::atomic<uint64_t> carve_tc{0};
    if (needs_setup(carve_tc)) {
      for (auto f : {k_gp_info_tc<true, true>, k_gp_info_tc<false, true>, k_gp_info_tc<true, false>,
                     k_gp_info_tc<false, false>}) {
        cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      }
      mark_setup(carve_tc);
    }
    // the top 8 rows of the last warp's last m-tile are padding for every warp of the
    // voxel only when wpv == 1; with wpv > 1 earlier warps' tiles are real
    const bool dead_top = wpv == 1 && (GC_MT - 1) * 16 + 8 >= ns;
#define GC_LAUNCH(M, D)                                                                                       \
  k_gp_info_tc<M, D><<<blocks_c, GC_WARPS * 32, smem, st>>>(lm, n_pad, n_points, src, v_begin, v_end, ns, wpv, \
                                                           model->zs, gate, (float)inv_s2, (float)ax, (float)bx, \
                                                           d_out64, d_out32)
    if (has_mask) { if (dead_top) GC_LAUNCH(true, true); else GC_LAUNCH(true, false); }
    else { if (dead_top) GC_LAUNCH(false, true); else GC_LAUNCH(false, false); }
#undef GC_LAUNCH
    FIF_CHECK_LAUNCH("k_gp_info_tc");
  } else {
    const int tpv = (ns + GI_G - 1) / GI_G;
    int vbi = GI_VB_THREADS / tpv;
    if (vbi < 1) vbi = 1;
    const int threads_i = ((vbi * tpv + 31) / 32) * 32;
    FIF_CHECK_ARG(threads_i <= GI_VB_THREADS || vbi == 1, "fif_build: N_s=%d too large for k_gp_info", ns);
    const unsigned blocks_i = (unsigned)((rows + vbi - 1) / vbi);
    size_t smem = sizeof(double) * 21 * GI_G * threads_i + sizeof(float4) * (vbi * (GI_TILE * 6 + 1) + GI_TILE * 2) +
                  sizeof(float) * 6 * vbi;
    static std::atomic<uint64_t> carve{0};
    if (needs_setup(carve)) {  // prefer the max shared-memory carveout so several CTAs fit per SM
      for (auto f : {k_gp_info<true>, k_gp_info<false>}) {
        cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      }
      mark_setup(carve);
    }
    if (has_mask)
      k_gp_info<true><<<blocks_i, threads_i, smem, st>>>(lm, n_pad, n_points, src, v_begin, v_end, vbi, ns, model->zs,
                                                         gate, (float)inv_s2, (float)ax, (float)bx, d_out64, d_out32);
    else
      k_gp_info<false><<<blocks_i, threads_i, smem, st>>>(lm, n_pad, n_points, src, v_begin, v_end, vbi, ns,
                                                          model->zs, gate, (float)inv_s2, (float)ax, (float)bx,
                                                          d_out64, d_out32);
    FIF_CHECK_LAUNCH("k_gp_info");
  }
  return FIF_OK;
}

extern "C" int fif_build(int factor_kind, const fif_model* model, const double* d_points, int64_t n_points,
                         const fif_grid* grid, const double* d_centers, int64_t v_begin, int64_t v_end,
                         const uint8_t* d_mask, double sigma, uint32_t build_flags, void* d_scratch, double* d_out64,
                         float* d_out32, void* stream) {
  PairGate gate{};
  gate.mask = d_mask;
  gate.v0 = v_begin;
  gate.n = n_points;
  return build_impl(factor_kind, model, d_points, n_points, grid, d_centers, v_begin, v_end, gate, d_mask != nullptr,
                    sigma, build_flags, d_scratch, d_out64, d_out32, stream);
}

extern "C" int fif_build_matched(int factor_kind, const fif_model* model, const double* d_points, int64_t n_points,
                                 const double* d_centers, int64_t rows, const fif_match* match,
                                 const double* d_view_dirs, double sigma, uint32_t build_flags, void* d_scratch,
                                 double* d_out64, float* d_out32, void* stream) {
  FIF_CHECK_ARG(match != nullptr && d_centers != nullptr, "fif_build_matched: NULL match / centres");
  FIF_CHECK_ARG(!(match->flags & FIF_MATCH_CONE) || d_view_dirs,
                "fif_build_matched: view cone requires landmark view directions");
  FIF_CHECK_ARG(!(match->flags & FIF_MATCH_OCCLUDE) || ((match->n_spheres == 0 || match->spheres) &&
                                                        (match->n_boxes == 0 || match->boxes)),
                "fif_build_matched: occlusion needs the sphere / box arrays");
  PairGate gate{};
  gate.m = *match;
  gate.pts = d_points;
  gate.vdir = d_view_dirs;
  gate.v0 = 0;
  gate.n = n_points;
  return build_impl(factor_kind, model, d_points, n_points, nullptr, d_centers, 0, rows, gate, match->flags != 0,
                    sigma, build_flags, d_scratch, d_out64, d_out32, stream);
}

extern "C" int fif_export_reference(int factor_kind, const fif_model* model, const double* d_in64, int64_t rows,
                                    double* d_out, void* stream) {
  FIF_CHECK_ARG(model != nullptr, "fif_export_reference: NULL model");
  FIF_CHECK_ARG(rows >= 0, "fif_export_reference: rows < 0");
  if (rows == 0) return FIF_OK;  // an empty field (no occupied voxel) exports nothing
  FIF_CHECK_ARG(d_in64 != nullptr && d_out != nullptr, "fif_export_reference: NULL argument");
  cudaStream_t st = (cudaStream_t)stream;
  const bool trace = factor_kind == FIF_KIND_TRACE;
  const int nv = model->kind == FIF_MODEL_QUAD ? 10 : model->n_v;
  const double* src = d_in64;
  double* tmp = nullptr;
  if (model->kind == FIF_MODEL_GP) {
    FIF_CHECK_ARG(model->kinv != nullptr, "fif_export_reference: GP model without kinv");
    const int W = trace ? 1 : 21;
    if (nv <= GX_KS) {  // fused GEMM + expansion
      const size_t smem = sizeof(double) * (size_t)nv * (GX_KS + GX_NC);
      static std::atomic<uint64_t> gx_attr{0};
      if (needs_setup(gx_attr)) {
        cudaFuncSetAttribute(k_gp_export<21>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(sizeof(double) * GX_KS * (GX_KS + GX_NC)));
        cudaFuncSetAttribute(k_gp_export<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(sizeof(double) * GX_KS * (GX_KS + GX_NC)));
        mark_setup(gx_attr);
      }
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      const int64_t groups = (rows + GX_NC / W - 1) / (GX_NC / W);
      const unsigned grid = (unsigned)std::min<int64_t>(groups, (int64_t)sms * 2);
      if (trace)
        k_gp_export<1><<<grid, 256, smem, st>>>(d_in64, rows, nv, model->kinv, d_out);
      else
        k_gp_export<21><<<grid, 256, smem, st>>>(d_in64, rows, nv, model->kinv, d_out);
      FIF_CHECK_LAUNCH("k_gp_export");
      return FIF_OK;
    }
    double* dst = d_out;
    if (!trace) {
      if (cudaMallocAsync(&tmp, sizeof(double) * rows * nv * 21, st) != cudaSuccess) {
        set_error("fif_export_reference: cudaMallocAsync failed");
        return FIF_ERR_CUDA;
      }
      dst = tmp;
    }
    size_t smem = sizeof(double) * nv * W;
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_gp_apply_kinv, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_gp_apply_kinv<<<(unsigned)rows, 256, smem, st>>>(d_in64, rows, nv, W, model->kinv, dst);
    FIF_CHECK_LAUNCH("k_gp_apply_kinv");
    if (trace) return FIF_OK;
    src = tmp;
  } else if (trace) {
    cudaMemcpyAsync(d_out, d_in64, sizeof(double) * rows * 10, cudaMemcpyDeviceToDevice, st);
    FIF_CHECK_LAUNCH("fif_export_reference(copy)");
    return FIF_OK;
  }
  int64_t blocks36 = rows * nv;
  k_expand36<<<(unsigned)((blocks36 * 36 + 255) / 256), 256, 0, st>>>(src, blocks36, d_out);
  FIF_CHECK_LAUNCH("k_expand36");
  if (tmp) cudaFreeAsync(tmp, st);
  return FIF_OK;
}
