// fif_query.cu — batched pose queries with analytic pose gradients, sm_100a.
//
// Replaces the per-query loops of the reference:
//   _nb_query_fim_batch_quad/gp      kernels.py:752-777  (+ _nb_query_fim 674-726)
//   _nb_field_metric_batch_quad/gp   kernels.py:1493-1522 (+ _nb_query_metric 1429-1472,
//                                    _nb_metric_one 1405-1426, _nb_metric_of 602-608)
// and adds the analytic gradient w.r.t. a decoupled world-frame pose perturbation
// t' = t + dt, R' = exp(dtheta^) R, which the reference lacks.
//
// One warp per query.  Corner location and trilinear weights are FP64 with the
// reference's exact operation order (bit-exact indices / status).  Rotation
// weights: quad v^r(z) (kernels.py:638-649); GP omega = kinv v^r(z) in FP64 so
// the field can hold the pre-kinv sums S in FP32.  The field
// rows are streamed once per corner (HBM-bound) and blended in FP64.
#include "fif_common.cuh"
#include "fif_linalg.cuh"

#include <cstdlib>

#include <cub/cub.cuh>

namespace fif {


struct QueryGeom {
  double ox, oy, oz, vs;
  int64_t nx, ny, nz;
};

// Corner table for one query. Returns status; fills rows[8], w[8], dw[8][3].
// Nearest: one corner (n=1) with w=1, dw=0.
__device__ __forceinline__ int locate(const QueryGeom& gm, const int32_t* __restrict__ slots, double px, double py,
                                      double pz, bool trilinear, int& ncorner, int64_t rows[8], double w[8],
                                      double dw[8][3]) {
  if (!trilinear) {
    // kernels.py:628-635
    int64_t ix = (int64_t)floor(__ddiv_rn(__dsub_rn(px, gm.ox), gm.vs));
    int64_t iy = (int64_t)floor(__ddiv_rn(__dsub_rn(py, gm.oy), gm.vs));
    int64_t iz = (int64_t)floor(__ddiv_rn(__dsub_rn(pz, gm.oz), gm.vs));
    if (ix < 0 || iy < 0 || iz < 0 || ix >= gm.nx || iy >= gm.ny || iz >= gm.nz) return FIF_STATUS_OUT_OF_FIELD;
    ncorner = 1;
    rows[0] = slots ? (int64_t)slots[(ix * gm.ny + iy) * gm.nz + iz] : (iz * gm.ny + iy) * gm.nx + ix;
    w[0] = 1.0;
    dw[0][0] = dw[0][1] = dw[0][2] = 0.0;
    return FIF_STATUS_OK;
  }
  // kernels.py:679-702
  double gx = __dsub_rn(__ddiv_rn(__dsub_rn(px, gm.ox), gm.vs), 0.5);
  double gy = __dsub_rn(__ddiv_rn(__dsub_rn(py, gm.oy), gm.vs), 0.5);
  double gz = __dsub_rn(__ddiv_rn(__dsub_rn(pz, gm.oz), gm.vs), 0.5);
  int64_t bx = (int64_t)floor(gx), by = (int64_t)floor(gy), bz = (int64_t)floor(gz);
  double fx = __dsub_rn(gx, (double)bx), fy = __dsub_rn(gy, (double)by), fz = __dsub_rn(gz, (double)bz);
  if (bx + 1 == gm.nx && fx == 0.0) { bx -= 1; fx = 1.0; }
  if (by + 1 == gm.ny && fy == 0.0) { by -= 1; fy = 1.0; }
  if (bz + 1 == gm.nz && fz == 0.0) { bz -= 1; fz = 1.0; }
  if (bx < 0 || by < 0 || bz < 0 || bx + 1 >= gm.nx || by + 1 >= gm.ny || bz + 1 >= gm.nz)
    return FIF_STATUS_OUT_OF_FIELD;
  ncorner = 8;
  const double inv_vs = 1.0 / gm.vs;
  int k = 0;
  for (int dx = 0; dx < 2; ++dx) {
    double wx = dx ? fx : __dsub_rn(1.0, fx);
    for (int dy = 0; dy < 2; ++dy) {
      double wy = dy ? fy : __dsub_rn(1.0, fy);
      for (int dz = 0; dz < 2; ++dz, ++k) {
        double wz = dz ? fz : __dsub_rn(1.0, fz);
        w[k] = __dmul_rn(__dmul_rn(wx, wy), wz);
        dw[k][0] = (dx ? inv_vs : -inv_vs) * wy * wz;
        dw[k][1] = (dy ? inv_vs : -inv_vs) * wx * wz;
        dw[k][2] = (dz ? inv_vs : -inv_vs) * wx * wy;
        int64_t ix = bx + dx, iy = by + dy, iz = bz + dz;
        rows[k] = slots ? (int64_t)slots[(ix * gm.ny + iy) * gm.nz + iz] : (iz * gm.ny + iy) * gm.nx + ix;
      }
    }
  }
  return FIF_STATUS_OK;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__constant__ int kPackR[21] = {0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 1, 2, 2, 2, 2, 3, 3, 3, 4, 4, 5};
__constant__ int kPackC[21] = {0, 1, 2, 3, 4, 5, 1, 2, 3, 4, 5, 2, 3, 4, 5, 3, 4, 5, 4, 5, 5};
__constant__ int kIsDiag[21] = {1, 0, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 1, 0, 1};


struct QueryOut {
  double* trace;
  double* trace_grad;
  double* fim;
  double* fim_grad;
  double* det;
  double* det_grad;
  double* lmin;
  double* lmin_grad;
  uint8_t* status;
};

// ───────────────────────── prep: corners + rotation weights ─────────────
// Per query q: status, 8 corner rows (int32, -1 = empty/absent), corner weights
// cw[q][c] = {w, dw/dx, dw/dy, dw/dz}, and rotation weights wt[q][k] = {omega_k,
// d omega_k/dz_x, d omega_k/dz_y, d omega_k/dz_z} (one double4 per sample k, FP64),
// where omega = v^r (quad, kernels.py:638-649) or kinv v^r (GP, kernels.py:652-657;
// kinv symmetric so omega . S == v^r . (kinv S)).  A CTA handles QP_Q queries.
// GP: v^r into smem, then one thread per (k, group of QP_G queries) runs the FP64
// matrix-vector products with kinv read through L1 (coalesced over k) and v^r
// broadcast from smem; the three derivative rows reuse t = kinv_gk v^r_g:
// d omega_a = inv_l2 kinv (v^r . zs_a).
constexpr int QP_Q = 64;
constexpr int QP_G = 4;
constexpr int QP_THREADS = 256;

__global__ void __launch_bounds__(QP_THREADS) k_query_prep(fif_model m, QueryGeom gm, const int32_t* __restrict__ slots,
                                                          const double* __restrict__ pos, const double* __restrict__ axes,
                                                          int64_t nq, int trilinear, uint8_t* __restrict__ status,
                                                          int32_t* __restrict__ rows, double4* __restrict__ cw,
                                                          double4* __restrict__ wt, const int32_t* __restrict__ perm) {
  extern __shared__ double sv[];  // [QP_Q][nv] v^r, then zs [nv][3]
  const int nv = m.kind == FIF_MODEL_QUAD ? 10 : m.n_v;
  const int64_t q0 = blockIdx.x * (int64_t)QP_Q;
  const int t = threadIdx.x;
  // corners and trilinear weights: one thread per query (FP64, reference order)
  if (t < QP_Q && q0 + t < nq) {  // (QP_Q <= QP_THREADS)
    const int64_t q = q0 + t;
    int nc = 0;
    int64_t r[8];
    double w[8], dw[8][3];
    const int64_t qo = perm ? (int64_t)perm[q] : q;  // slot q holds query qo (locality order)
    const int st = locate(gm, slots, pos[3 * qo], pos[3 * qo + 1], pos[3 * qo + 2], trilinear != 0, nc, r, w, dw);
    status[q] = (uint8_t)st;
    for (int c = 0; c < 8; ++c) {
      const bool ok = st == FIF_STATUS_OK && c < nc;
      rows[q * 8 + c] = ok ? (int32_t)r[c] : -1;
      cw[q * 8 + c] = ok ? make_double4(w[c], dw[c][0], dw[c][1], dw[c][2]) : make_double4(0, 0, 0, 0);
    }
  }
  if (m.kind == FIF_MODEL_QUAD) {
    for (int idx = t; idx < QP_Q * 10; idx += blockDim.x) {
      const int qi = idx / 10, k = idx - qi * 10;
      const int64_t q = q0 + qi;
      if (q >= nq) continue;
      const int64_t qo = perm ? (int64_t)perm[q] : q;
      const double zx = axes[3 * qo], zy = axes[3 * qo + 1], zz = axes[3 * qo + 2];
      const double k2 = m.k2, k1 = m.k1, k0 = m.k0, t2 = 2.0 * k2;
      double v = 0, gx = 0, gy = 0, gz = 0;
      switch (k) {
        case 0: v = __dmul_rn(__dmul_rn(k2, zx), zx); gx = t2 * zx; break;
        case 1: v = __dmul_rn(__dmul_rn(k2, zy), zy); gy = t2 * zy; break;
        case 2: v = __dmul_rn(__dmul_rn(k2, zz), zz); gz = t2 * zz; break;
        case 3: v = __dmul_rn(__dmul_rn(t2, zx), zy); gx = t2 * zy; gy = t2 * zx; break;
        case 4: v = __dmul_rn(__dmul_rn(t2, zx), zz); gx = t2 * zz; gz = t2 * zx; break;
        case 5: v = __dmul_rn(__dmul_rn(t2, zy), zz); gy = t2 * zz; gz = t2 * zy; break;
        case 6: v = __dmul_rn(k1, zx); gx = k1; break;
        case 7: v = __dmul_rn(k1, zy); gy = k1; break;
        case 8: v = __dmul_rn(k1, zz); gz = k1; break;
        default: v = k0; break;
      }
      wt[q * 10 + k] = make_double4(v, gx, gy, gz);
    }
    return;
  }
  // GP: v^r into smem (kernels.py:652-657 sample kernel), zs / l^2 staged after it
  const double inv_l2 = 1.0 / (m.ell * m.ell);
  double* zs = sv + QP_Q * nv;
  for (int idx = t; idx < 3 * nv; idx += blockDim.x) zs[idx] = m.zs[idx] * inv_l2;
  for (int idx = t; idx < QP_Q * nv; idx += blockDim.x) {
    const int qi = idx / nv, g = idx - qi * nv;
    const int64_t q = q0 + qi;
    if (q >= nq) {
      sv[idx] = 0.0;
      continue;
    }
    const int64_t qo = perm ? (int64_t)perm[q] : q;
    const double c = __dadd_rn(__dadd_rn(__dmul_rn(axes[3 * qo], m.zs[3 * g]), __dmul_rn(axes[3 * qo + 1], m.zs[3 * g + 1])),
                               __dmul_rn(axes[3 * qo + 2], m.zs[3 * g + 2]));
    sv[idx] = m.sig2 * exp(__dmul_rn(__dsub_rn(c, 1.0), inv_l2));
  }
  __syncthreads();
  // one thread per (k, group of QP_G queries): each kinv element read once feeds
  // QP_G queries; zs is warp-uniform, v^r uniform within the query group.
  for (int idx = t; idx < (QP_Q / QP_G) * nv; idx += blockDim.x) {
    const int qg = idx / nv, k = idx - qg * nv;
    const double* v = sv + qg * QP_G * nv;
    const double* kc = m.kinv + k;
    double a[QP_G][4];
#pragma unroll
    for (int i = 0; i < QP_G; ++i) a[i][0] = a[i][1] = a[i][2] = a[i][3] = 0.0;
#pragma unroll 2
    for (int g = 0; g < nv; ++g) {
      const double kg = __ldg(kc + (int64_t)g * nv);
      const double z0 = zs[3 * g], z1 = zs[3 * g + 1], z2 = zs[3 * g + 2];
#pragma unroll
      for (int i = 0; i < QP_G; ++i) {
        const double tg = kg * v[i * nv + g];
        a[i][0] += tg;
        a[i][1] = fma(tg, z0, a[i][1]);
        a[i][2] = fma(tg, z1, a[i][2]);
        a[i][3] = fma(tg, z2, a[i][3]);
      }
    }
#pragma unroll
    for (int i = 0; i < QP_G; ++i) {
      const int64_t q = q0 + qg * QP_G + i;
      if (q < nq) wt[q * nv + k] = make_double4(a[i][0], a[i][1], a[i][2], a[i][3]);
    }
  }
}

// GP prep on the FP64 tensor core: Omega[(q, a)][k] = sum_g U[(q, a)][g] kinv[g][k],
// U[(q, 0)] = v^r(q), U[(q, a)] = v^r(q) . zs_a / l^2, as mma.sync m8n8k4 f64 (DMMA,
// IEEE FP64 products and sums): an m8 tile = 2 queries x 4 weight rows, kinv staged
// once per CTA in smem (zero padded to a multiple of 8), v^r per query in smem.
// Same outputs as k_query_prep; used when kinv fits in shared memory.
constexpr int QD_Q = 32;
constexpr int QD_THREADS = 256;

__device__ __forceinline__ void dmma_884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// QQ queries per CTA: 32 for streaming batches, 8 for small batches (more CTAs, so the
// latency-bound prep spreads over more SMs)
// RPQ weight rows per query in an m8 tile: 4 (omega and its 3 z-derivatives) when
// gradients are wanted, else 1 (8 queries per tile, a quarter of the DMMAs)
template <int QQ, int RPQ>
struct QDShape {
  static constexpr int MTILES = QQ * RPQ / 8;
  static constexpr int NWARPS = MTILES < 8 ? MTILES : 8;
  static constexpr int THREADS = 32 * NWARPS;
  static constexpr int MT_PER_WARP = MTILES / NWARPS;
};
template <int NT, int QQ, int RPQ>
__global__ void __launch_bounds__(QDShape<QQ, RPQ>::THREADS, 3) k_query_prep_gp(fif_model m, QueryGeom gm,
                                                              const int32_t* __restrict__ slots,
                                                              const double* __restrict__ pos,
                                                              const double* __restrict__ axes, int64_t nq,
                                                              int trilinear, uint8_t* __restrict__ status,
                                                              int32_t* __restrict__ rows, double4* __restrict__ cw,
                                                              double* __restrict__ wt,
                                                              const int32_t* __restrict__ perm) {
  extern __shared__ double smd[];
  constexpr int NP8 = 8 * NT, KS = NP8 / 4;
  constexpr int MT_PER_WARP = QDShape<QQ, RPQ>::MT_PER_WARP;
  constexpr int NWARPS = QDShape<QQ, RPQ>::NWARPS;
  constexpr int QPM = 8 / RPQ;  // queries per m8 tile
  const int nv = m.n_v;
  // kinv row-major (stride nv) landed by one TMA bulk copy; rows nv..NP8-1 read by the
  // padded k-steps are zeroed (their A entries are zero too, and 0 x NaN would not be)
  double* kf = smd;                                  // [NP8][nv] (+ tail)
  double* sv = kf + ((NP8 * nv + 8 + 15) & ~15);     // [QQ][NP8] v^r
  double* sa = sv + QQ * NP8;                        // [NP8][4] {1, zs/l^2}
  double* sz = sa + 4 * NP8;                         // [QQ][4] optical axes of the CTA's queries
  __shared__ __align__(8) uint64_t kbar;
  const int64_t q0 = blockIdx.x * (int64_t)QQ;
  const int t = threadIdx.x;
  const uint32_t kbytes = (uint32_t)(nv * nv * sizeof(double));
  const bool use_tma = (kbytes % 16u) == 0 && (reinterpret_cast<uintptr_t>(m.kinv) & 15) == 0;
  if (use_tma) {
    if (t == 0) {
      mbar_init(&kbar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      mbar_expect_tx(&kbar, kbytes);
      tma_bulk_g2s(kf, m.kinv, kbytes, &kbar);
    }
  } else {
    for (int idx = t; idx < nv * nv; idx += blockDim.x) kf[idx] = m.kinv[idx];
  }
  for (int idx = nv * nv + t; idx < NP8 * nv + 8; idx += blockDim.x) kf[idx] = 0.0;
  if (t < QQ && q0 + t < nq) {  // corners and trilinear weights (FP64, reference order)
    const int64_t q = q0 + t;
    int nc = 0;
    int64_t r[8];
    double w[8], dw[8][3];
    const int64_t qo = perm ? (int64_t)perm[q] : q;  // slot q holds query qo (locality order)
    sz[4 * t] = axes[3 * qo];
    sz[4 * t + 1] = axes[3 * qo + 1];
    sz[4 * t + 2] = axes[3 * qo + 2];
    const int st = locate(gm, slots, pos[3 * qo], pos[3 * qo + 1], pos[3 * qo + 2], trilinear != 0, nc, r, w, dw);
    status[q] = (uint8_t)st;
    for (int c = 0; c < 8; ++c) {
      const bool ok = st == FIF_STATUS_OK && c < nc;
      rows[q * 8 + c] = ok ? (int32_t)r[c] : -1;
      cw[q * 8 + c] = ok ? make_double4(w[c], dw[c][0], dw[c][1], dw[c][2]) : make_double4(0, 0, 0, 0);
    }
  }
  const double inv_l2 = 1.0 / (m.ell * m.ell);
  for (int g = t; g < NP8; g += blockDim.x) {
    const bool ok = g < nv;
    sa[4 * g] = ok ? 1.0 : 0.0;
    sa[4 * g + 1] = ok ? m.zs[3 * g] * inv_l2 : 0.0;
    sa[4 * g + 2] = ok ? m.zs[3 * g + 1] * inv_l2 : 0.0;
    sa[4 * g + 3] = ok ? m.zs[3 * g + 2] * inv_l2 : 0.0;
  }
  __syncthreads();  // sz (the queries' optical axes) staged by the locating threads
  auto vr_of = [&](int qi, double z0, double z1, double z2) {  // kernels.py:652-657
    const double c = __dadd_rn(__dadd_rn(__dmul_rn(sz[4 * qi], z0), __dmul_rn(sz[4 * qi + 1], z1)),
                               __dmul_rn(sz[4 * qi + 2], z2));
    return m.sig2 * exp(__dmul_rn(__dsub_rn(c, 1.0), inv_l2));
  };
  if ((int)blockDim.x >= NP8) {  // thread owns sample g (its zs in registers), strides over queries
    const int gq = blockDim.x / NP8, g = t % NP8, qs = t / NP8;
    if (qs < gq) {
      const bool gok = g < nv;
      const double z0 = gok ? m.zs[3 * g] : 0.0, z1 = gok ? m.zs[3 * g + 1] : 0.0, z2 = gok ? m.zs[3 * g + 2] : 0.0;
      for (int qi = qs; qi < QQ; qi += gq) sv[qi * NP8 + g] = (q0 + qi < nq && gok) ? vr_of(qi, z0, z1, z2) : 0.0;
    }
  } else {
    for (int idx = t; idx < QQ * NP8; idx += blockDim.x) {
      const int qi = idx / NP8, g = idx - qi * NP8;
      sv[idx] = (q0 + qi < nq && g < nv) ? vr_of(qi, m.zs[3 * g], m.zs[3 * g + 1], m.zs[3 * g + 2]) : 0.0;
    }
  }
  if (use_tma) mbar_wait(&kbar, 0);
  __syncthreads();
  const int warp = t >> 5, lane = t & 31;
  const int row = lane >> 2, tq = lane & 3;  // A/C row; A col = B row = tq
  const int qq = row / RPQ, a = row % RPQ;  // m8 row -> (query of the tile, weight row)
  // each warp owns MT_PER_WARP m-tiles (2 queries each) and all NT n-tiles: every B
  // fragment load feeds MT_PER_WARP DMMAs, every A fragment NT DMMAs
  double c[MT_PER_WARP][NT][2];
#pragma unroll
  for (int i = 0; i < MT_PER_WARP; ++i)
#pragma unroll
    for (int n = 0; n < NT; ++n) c[i][n][0] = c[i][n][1] = 0.0;
  // B[g][k] = kinv[g][k] with g = 4 ks + tq, k = 8 n + row; columns k >= nv read the
  // next row (finite) and only feed discarded outputs
  const double* kfl = kf + tq * nv + row;
#pragma unroll 1
  for (int ks = 0; ks < KS; ++ks) {
    const int g = 4 * ks + tq;
    const double sg = RPQ == 1 ? 1.0 : sa[4 * g + a];
    double av[MT_PER_WARP];
#pragma unroll
    for (int i = 0; i < MT_PER_WARP; ++i) {
      const int qi = (warp + i * NWARPS) * QPM + qq;
      av[i] = RPQ == 1 ? sv[qi * NP8 + g] : sv[qi * NP8 + g] * sg;
    }
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const double b = kfl[4 * ks * nv + 8 * n];
#pragma unroll
      for (int i = 0; i < MT_PER_WARP; ++i) dmma_884(c[i][n][0], c[i][n][1], av[i], b);
    }
  }
#pragma unroll
  for (int i = 0; i < MT_PER_WARP; ++i) {
    const int64_t q = q0 + (warp + i * NWARPS) * QPM + qq;
    if (q >= nq) continue;
#pragma unroll
    for (int n = 0; n < NT; ++n) {
      const int k = n * 8 + 2 * tq;
      if (k < nv) wt[(q * nv + k) * 4 + a] = c[i][n][0];
      if (k + 1 < nv) wt[(q * nv + k + 1) * 4 + a] = c[i][n][1];
    }
  }
}

template <int NT, int QQ, int RPQ>
static void launch_prep_gp(size_t smem, int64_t q, cudaStream_t st, const fif_model& m, const QueryGeom& gm,
                           const int32_t* slots, const double* pos, const double* axes, int trilinear,
                           uint8_t* status, int32_t* rows, double4* cw, double* wt, const int32_t* perm) {
  auto kern = k_query_prep_gp<NT, QQ, RPQ>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  kern<<<(unsigned)((q + QQ - 1) / QQ), QDShape<QQ, RPQ>::THREADS, smem, st>>>(m, gm, slots, pos, axes, q, trilinear, status,
                                                                     rows, cw, wt, perm);
}

// ───────────────────────── contraction: info fields ─────────────────────
// One warp per query, lane e < 21 owns packed entry e.  Each warp streams its
// queries through a private QW_STAGES-deep ring of k-chunks: one chunk = KC
// samples of all NC corner rows (KC*21 contiguous entries of each row, one TMA
// bulk copy per corner, 16-B aligned superset) plus the KC rotation weights, all
// completing on the stage's mbarrier.  Lane 0 refills a stage as soon as the warp
// has consumed it, so the next chunks (of this or the next query) are in flight
// while the warp computes
//     G_c += omega_k S_c,k          (every corner: the 6x6 blend and d/dt)
//     R_a += d omega_k/dz_a . (sum_c w_c S_c,k)   (rotation gradient, blend first)
// in FP64 from the smem copy.  No block-level synchronisation: warps are
// independent streams, the block only shares a zero row used for absent corners.
constexpr int QW_WARPS = 4;
// warps per CTA: the streaming variants (2-3 stages) run 4 independent query warps per
// CTA; the small-batch variant (QW_SMALL_STAGES: every k-chunk of a query in flight at
// once, latency- rather than bandwidth-bound) runs one warp per CTA
constexpr int QW_SMALL_STAGES = 8;
__host__ __device__ constexpr int qw_wpb(int stages) { return stages >= QW_SMALL_STAGES ? 1 : QW_WARPS; }

// k-chunk length: 840 bytes of each corner row per stage for FP32 and FP64 rows.
template <typename T>
struct QWShape {
  static constexpr int KC = sizeof(T) == 4 ? 10 : 5;
  static constexpr uint32_t CHUNK = KC * 21 * sizeof(T);
  static constexpr uint32_t CAP = (CHUNK + 32 + 15) & ~15u;  // + alignment slack both ends
};
// per-warp METRIC scratch: per corner G (21) and, with metric gradients, H_a (3 x 21)
template <bool METRIC, bool MGRAD>
__host__ __device__ constexpr uint32_t qw_cf() {
  return METRIC ? (MGRAD ? 84u : 21u) : 0u;
}
template <typename T, int NC, int STAGES, bool METRIC, bool MGRAD>
__host__ __device__ constexpr uint32_t qw_warp_bytes() {
  return 64 + STAGES * (NC * QWShape<T>::CAP + QWShape<T>::KC * 32) + 8 * 8 * qw_cf<METRIC, MGRAD>();
}

// Outputs of one query from its per-corner contractions G_c (lane = packed entry),
// the blended rotation derivatives R (or per-corner H for metric gradients), the
// corner weights (lane c holds corner c's {w, dw} in my_cw) and r_lane (row of corner
// `lane`, -1 = absent).  Shared by the streaming and the small-batch kernels.
template <int NC, bool GRAD, bool METRIC, bool MGRAD>
__device__ __forceinline__ void emit_outputs(const QueryOut& out, int64_t qo, int st, int lane, bool on,
                                             const double (&w)[NC], const double (&G)[NC], double R0, double R1,
                                             double R2, const double (&H)[MGRAD ? NC : 1][3], double4 my_cw,
                                             double* cfim, const double* __restrict__ axes, int32_t r_lane) {
  constexpr unsigned FULL = 0xffffffffu;
  constexpr uint32_t CF = qw_cf<METRIC, MGRAD>();
  if (MGRAD) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      R0 = fma(w[c], H[c][0], R0);
      R1 = fma(w[c], H[c][1], R1);
      R2 = fma(w[c], H[c][2], R2);
      if (on) {
        cfim[c * CF + 21 + lane] = H[c][0];
        cfim[c * CF + 42 + lane] = H[c][1];
        cfim[c * CF + 63 + lane] = H[c][2];
      }
    }
  }
  double val = 0, pgx = 0, pgy = 0, pgz = 0;
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    val = fma(w[c], G[c], val);
    if (GRAD) {
      pgx = fma(__shfl_sync(FULL, my_cw.y, c), G[c], pgx);
      pgy = fma(__shfl_sync(FULL, my_cw.z, c), G[c], pgy);
      pgz = fma(__shfl_sync(FULL, my_cw.w, c), G[c], pgz);
    }
    if (METRIC && on) cfim[c * CF + lane] = G[c];
  }
  const double zx = axes[3 * qo], zy = axes[3 * qo + 1], zz = axes[3 * qo + 2];
  const double tgx = zy * R2 - zz * R1, tgy = zz * R0 - zx * R2, tgz = zx * R1 - zy * R0;  // z x d/dz
  if (out.fim && on) {
    const int pr = kPackR[lane], pc = kPackC[lane];
    out.fim[qo * 36 + pr * 6 + pc] = val;
    out.fim[qo * 36 + pc * 6 + pr] = val;
  }
  if (GRAD && out.fim_grad && on) {
    const int pr = kPackR[lane], pc = kPackC[lane];
    const double g6[6] = {pgx, pgy, pgz, tgx, tgy, tgz};
#pragma unroll
    for (int d = 0; d < 6; ++d) {
      out.fim_grad[qo * 216 + d * 36 + pr * 6 + pc] = g6[d];
      out.fim_grad[qo * 216 + d * 36 + pc * 6 + pr] = g6[d];
    }
  }
  if (out.trace || (GRAD && out.trace_grad)) {
    const bool dg = on && kIsDiag[lane];
    const double tv = warp_sum(dg ? val : 0.0);
    if (out.trace && lane == 0) out.trace[qo] = tv;
    if (GRAD && out.trace_grad) {
      const double g6[6] = {pgx, pgy, pgz, tgx, tgy, tgz};
#pragma unroll
      for (int d = 0; d < 6; ++d) {
        const double sgl = warp_sum(dg ? g6[d] : 0.0);
        if (lane == d) out.trace_grad[qo * 6 + d] = sgl;
      }
    }
  }
  if (METRIC) {
    __syncwarp();
    double mv_det = 0, mv_lmin = 0, gd[3] = {0, 0, 0}, gl[3] = {0, 0, 0};
    if (lane < NC) {
      const double* cf = cfim + lane * CF;
      if (r_lane >= 0) {
        if (out.det) {
          double a[36], inv[36];
          unpack21(cf, a);
          bool ok;
          if (MGRAD && out.det_grad) {
            mv_det = det6_core<true>(a, inv, ok);
            if (ok)
#pragma unroll
              for (int ax = 0; ax < 3; ++ax) {  // d det = det tr(F^-1 dF), dF packed symmetric
                double t = 0.0;
#pragma unroll
                for (int x = 0; x < 21; ++x) {
                  const int r = pack_r(x), c = pack_c(x);
                  t = fma(r == c ? inv[7 * r] : inv[6 * r + c] + inv[6 * c + r], cf[21 * (1 + ax) + x], t);
                }
                gd[ax] = mv_det * t;
              }
          } else {
            mv_det = det6_core<false>(a, inv, ok);
          }
        }
        if (out.lmin) {
          double a[36], v6[6];
          unpack21(cf, a);
          if (MGRAD && out.lmin_grad) {
            mv_lmin = lmin6_core<true>(a, v6);
#pragma unroll
            for (int ax = 0; ax < 3; ++ax) {  // d lambda = v^T dF v
              double t = 0.0;
#pragma unroll
              for (int x = 0; x < 21; ++x) {
                const int r = pack_r(x), c = pack_c(x);
                t = fma(r == c ? v6[r] * v6[r] : 2.0 * v6[r] * v6[c], cf[21 * (1 + ax) + x], t);
              }
              gl[ax] = t;
            }
          } else {
            mv_lmin = lmin6_core<false>(a, v6);
          }
        }
      }
    }
    double mdet = 0, mlmin = 0;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const double dd = __shfl_sync(0xffffffffu, mv_det, c), ll = __shfl_sync(0xffffffffu, mv_lmin, c);
      if (w[c] != 0.0) {
        mdet = fma(w[c], dd, mdet);
        mlmin = fma(w[c], ll, mlmin);
      }
    }
    if (lane == 0) {
      if (out.det) out.det[qo] = mdet;
      if (out.lmin) out.lmin[qo] = mlmin;
    }
    if (MGRAD) {
      // lane c < NC holds its corner's (w, dw) in my_cw; other lanes hold zeros
      auto blend_grad = [&](double val_c, const double (&gz)[3], double* dst) {
        const double tx = warp_sum(my_cw.y * val_c), ty = warp_sum(my_cw.z * val_c), tz = warp_sum(my_cw.w * val_c);
        const double zxg = warp_sum(my_cw.x * gz[0]), zyg = warp_sum(my_cw.x * gz[1]), zzg = warp_sum(my_cw.x * gz[2]);
        const double g6[6] = {tx, ty, tz, zy * zzg - zz * zyg, zz * zxg - zx * zzg, zx * zyg - zy * zxg};
        if (lane < 6) dst[qo * 6 + lane] = g6[lane];
      };
      if (out.det_grad) blend_grad(mv_det, gd, out.det_grad);
      if (out.lmin_grad) blend_grad(mv_lmin, gl, out.lmin_grad);
    }
  }
  if (out.status && lane == 0) out.status[qo] = (uint8_t)st;
}

template <typename T, int NC, int STAGES, bool GRAD, bool METRIC, bool MGRAD>
__global__ void __launch_bounds__(qw_wpb(STAGES) * 32, STAGES == 2 ? 3 : (STAGES == 3 ? 2 : 3))
k_query_info(int nv, const T* __restrict__ field,
                                                             const double* __restrict__ axes, int64_t nq,
                                                             const uint8_t* __restrict__ status,
                                                             const int32_t* __restrict__ rows,
                                                             const double4* __restrict__ cw,
                                                             const double4* __restrict__ wt, QueryOut out,
                                                             const int32_t* __restrict__ perm) {
  using SH = QWShape<T>;
  constexpr int KC = SH::KC;
  constexpr uint32_t CAP = SH::CAP;
  constexpr uint32_t STAGE = NC * CAP + KC * 32;
  constexpr unsigned FULL = 0xffffffffu;
  constexpr uint32_t CF = qw_cf<METRIC, MGRAD>();
  static_assert(!MGRAD || (METRIC && GRAD), "metric gradients need METRIC and GRAD");
  extern __shared__ __align__(128) unsigned char qraw[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const T* zero_row = reinterpret_cast<const T*>(qraw);  // [CHUNK] zeros, shared
  unsigned char* wbase = qraw + ((SH::CHUNK + 127) & ~127u) + (size_t)warp * ((qw_warp_bytes<T, NC, STAGES, METRIC, MGRAD>() + 127) & ~127u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(wbase);
  unsigned char* stages = wbase + 64;
  double* cfim = reinterpret_cast<double*>(stages + STAGES * STAGE);  // METRIC: [8][CF]
  for (int i = threadIdx.x; i < (int)(SH::CHUNK / 4); i += blockDim.x) reinterpret_cast<float*>(qraw)[i] = 0.f;
  if (lane == 0) {
    for (int b = 0; b < STAGES; ++b) mbar_init(&bars[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t rw = (int64_t)nv * 21;
  const int nch = (nv + KC - 1) / KC;
  constexpr int WPB = qw_wpb(STAGES);
  const int64_t tw = (int64_t)gridDim.x * WPB;
  const int64_t qfirst = blockIdx.x * (int64_t)WPB + warp;
  const int64_t nmine = qfirst < nq ? (nq - qfirst + tw - 1) / tw : 0;
  auto qof = [&](int64_t i) { return qfirst + i * tw; };
  auto row_of = [&](int64_t i) -> int32_t {  // lane c < NC: corner c's row of my i-th query
    return (i < nmine && lane < NC) ? __ldg(rows + qof(i) * 8 + lane) : -1;
  };

  // ── producer (whole warp; lane c < NC copies corner c, lane NC the weights) ──
  int64_t pi = 0;
  int pj = 0, pb = 0;
  int32_t p_r = row_of(0), pn_r = row_of(1);
  auto produce = [&]() {
    if (pi >= nmine) return;
    const int64_t q = qof(pi);
    const int k0 = pj * KC, kn = min(KC, nv - k0);
    uintptr_t a0 = 0;
    uint32_t bytes = 0;
    if (lane < NC) {
      if (p_r >= 0) {
        const uintptr_t src = reinterpret_cast<uintptr_t>(field + (int64_t)p_r * rw + (int64_t)k0 * 21);
        a0 = src & ~(uintptr_t)15;
        bytes = (uint32_t)(((src + kn * 21 * sizeof(T) + 15) & ~(uintptr_t)15) - a0);
      }
    } else if (lane == NC) {
      a0 = reinterpret_cast<uintptr_t>(wt + q * nv + k0);
      bytes = (uint32_t)kn * 32u;
    }
    const uint32_t total = __reduce_add_sync(FULL, bytes);
    if (lane == 0) mbar_expect_tx(&bars[pb], total);
    __syncwarp();
    if (bytes) tma_bulk_g2s(stages + (size_t)pb * STAGE + (lane < NC ? lane : NC) * CAP,
                            reinterpret_cast<const void*>(a0), bytes, &bars[pb]);
    if (++pb == STAGES) pb = 0;
    if (++pj == nch) {
      pj = 0;
      ++pi;
      p_r = pn_r;
      pn_r = row_of(pi + 1);
    }
  };
  for (int s = 0; s < STAGES - 1; ++s) produce();

  // ── consumer ──
  const bool on = lane < 21;
  const int e = on ? lane : 0;
  int32_t c_r = row_of(0);
  double4 c_cw = lane < NC && nmine > 0 ? cw[qof(0) * 8 + lane] : make_double4(0, 0, 0, 0);
  int c_st = nmine > 0 ? status[qof(0)] : 0;
  int cb = 0;
  uint32_t cphase = 0;
  for (int64_t i = 0; i < nmine; ++i) {
    const int64_t q = qof(i);                                // slot (locality order)
    const int64_t qo = perm ? (int64_t)perm[q] : q;         // caller's query index
    const int st = c_st;
    int32_t r[NC];
    double w[NC], G[NC];
    uint32_t off[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      r[c] = __shfl_sync(FULL, c_r, c);
      w[c] = __shfl_sync(FULL, c_cw.x, c);
      off[c] = (uint32_t)(reinterpret_cast<uintptr_t>(field + (int64_t)(r[c] < 0 ? 0 : r[c]) * rw) & 15);
      G[c] = 0.0;
    }
    const double4 my_cw = c_cw;
    const int32_t my_r = c_r;  // row of corner `lane` (lanes < NC)
    // prefetch the next query's metadata
    c_r = row_of(i + 1);
    if (i + 1 < nmine) {
      c_cw = lane < NC ? cw[qof(i + 1) * 8 + lane] : make_double4(0, 0, 0, 0);
      c_st = status[qof(i + 1)];
    }
    double R0 = 0, R1 = 0, R2 = 0;
    double H[MGRAD ? NC : 1][3];
#pragma unroll
    for (int c = 0; c < (MGRAD ? NC : 1); ++c) H[c][0] = H[c][1] = H[c][2] = 0.0;
    for (int j = 0; j < nch; ++j) {
      __syncwarp();  // every lane is done with the stage produce() refills next
      if (lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      produce();
      mbar_wait(&bars[cb], cphase);
      if (st == FIF_STATUS_OK && on) {
        const int k0 = j * KC, kn = min(KC, nv - k0);
        const unsigned char* sb = stages + (size_t)cb * STAGE;
        const T* src[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c)
          src[c] = r[c] >= 0
                       ? reinterpret_cast<const T*>(sb + c * CAP + ((off[c] + (uint32_t)(k0 * 21 * sizeof(T))) & 15u)) + e
                       : zero_row + e;
        const double4* wk = reinterpret_cast<const double4*>(sb + NC * CAP);
        auto step = [&](int kk) {
          const double4 om = wk[kk];
          double sv[NC];
#pragma unroll
          for (int c = 0; c < NC; ++c) sv[c] = (double)src[c][kk * 21];
#pragma unroll
          for (int c = 0; c < NC; ++c) G[c] = fma(om.x, sv[c], G[c]);
          if (MGRAD) {
            // per-corner rotation derivatives (the metric gradients need each corner's dF)
#pragma unroll
            for (int c = 0; c < NC; ++c) {
              H[c][0] = fma(om.y, sv[c], H[c][0]);
              H[c][1] = fma(om.z, sv[c], H[c][1]);
              H[c][2] = fma(om.w, sv[c], H[c][2]);
            }
          } else if (GRAD) {
            // blend over corners as two independent chains (halves the DFMA dependency depth)
            double b0 = 0.0, b1 = 0.0;
#pragma unroll
            for (int c = 0; c < NC; c += 2) {
              b0 = fma(w[c], sv[c], b0);
              if (c + 1 < NC) b1 = fma(w[c + 1], sv[c + 1], b1);
            }
            const double bl = b0 + b1;
            R0 = fma(om.y, bl, R0);
            R1 = fma(om.z, bl, R1);
            R2 = fma(om.w, bl, R2);
          }
        };
        if (kn == KC) {
#pragma unroll
          for (int kk = 0; kk < KC; ++kk) step(kk);
        } else {
#pragma unroll 1
          for (int kk = 0; kk < kn; ++kk) step(kk);
        }
      }
      if (++cb == STAGES) {
        cb = 0;
        cphase ^= 1u;
      }
    }
    // ── query complete: outputs ──
    if (st != FIF_STATUS_OK) {
      if (out.fim) for (int i2 = lane; i2 < 36; i2 += 32) out.fim[qo * 36 + i2] = 0.0;
      if (out.fim_grad) for (int i2 = lane; i2 < 216; i2 += 32) out.fim_grad[qo * 216 + i2] = 0.0;
      if (lane == 0) {
        if (out.trace) out.trace[qo] = 0.0;
        if (out.det) out.det[qo] = 0.0;
        if (out.lmin) out.lmin[qo] = 0.0;
      }
      if (out.trace_grad && lane < 6) out.trace_grad[qo * 6 + lane] = 0.0;
      if (out.det_grad && lane < 6) out.det_grad[qo * 6 + lane] = 0.0;
      if (out.lmin_grad && lane < 6) out.lmin_grad[qo * 6 + lane] = 0.0;
      if (out.status && lane == 0) out.status[qo] = (uint8_t)st;
      continue;
    }
    emit_outputs<NC, GRAD, METRIC, MGRAD>(out, qo, st, lane, on, w, G, R0, R1, R2, H, my_cw, cfim, axes, my_r);
  }
}

// ───────────────────────── small batches: fused prep + k-split contraction ──
// Latency-bound regime (a few hundred queries or fewer, e.g. planner state checks):
// one CTA of QS_WARPS warps per query.  Thread 0 locates the corners and issues TMA
// bulk copies of the (whole) corner rows at once; while they land, the CTA evaluates
// v^r and omega = kinv v^r (+ derivatives) in FP64 into shared memory; then the warps
// split the sample range, lanes over packed entries, and warp 0 reduces the partials
// and emits the outputs (emit_outputs, as the streaming kernel).  GP fields, FP32 rows.
constexpr int QS_WARPS = 8;

template <int NC, bool GRAD, bool METRIC, bool MGRAD>
__host__ __device__ constexpr int qs_np() {
  return NC + (MGRAD ? 3 * NC : (GRAD ? 3 : 0));
}

template <int NC, bool GRAD, bool METRIC, bool MGRAD>
__global__ void __launch_bounds__(QS_WARPS * 32) k_query_small(fif_model m, QueryGeom gm,
                                                               const int32_t* __restrict__ slots,
                                                               const double* __restrict__ pos,
                                                               const double* __restrict__ axes, int64_t nq,
                                                               int trilinear, const float* __restrict__ field,
                                                               QueryOut out) {
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int NP = qs_np<NC, GRAD, METRIC, MGRAD>();
  constexpr uint32_t CF = qw_cf<METRIC, MGRAD>();
  const int nv = m.n_v;
  const int64_t rw = (int64_t)nv * 21;
  const uint32_t rowcap = (uint32_t)((rw * 4 + 16 + 15) & ~15ll);
  extern __shared__ __align__(128) unsigned char qsm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(qsm);
  int* meta_i = reinterpret_cast<int*>(qsm + 16);               // [0] status, [1..8] rows, [9..16] offsets
  double4* meta_cw = reinterpret_cast<double4*>(qsm + 128);      // [8]
  unsigned char* rowbuf = qsm + 128 + 8 * sizeof(double4);       // [NC][rowcap]
  double4* om = reinterpret_cast<double4*>(rowbuf + (size_t)NC * rowcap);  // [nv]
  double* vr = reinterpret_cast<double*>(om + nv);                // [nv]
  double* part = vr + ((nv + 1) & ~1);                            // [QS_WARPS][NP][32]
  double* cfim = part + QS_WARPS * NP * 32;                       // METRIC: [8][CF]
  double* kin = cfim + (METRIC ? 8 * CF : 0);                     // [nv][nv] kinv, landed once per CTA
  uint64_t* kbar = bar + 1;
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const uint32_t kbytes = (uint32_t)(nv * nv * sizeof(double));
  const bool k_tma = (kbytes % 16u) == 0 && (reinterpret_cast<uintptr_t>(m.kinv) & 15) == 0;
  if (t == 0) {
    mbar_init(bar, 1);
    mbar_init(kbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (k_tma) {
      mbar_expect_tx(kbar, kbytes);
      tma_bulk_g2s(kin, m.kinv, kbytes, kbar);
    }
  }
  if (!k_tma)
    for (int i = t; i < nv * nv; i += blockDim.x) kin[i] = m.kinv[i];
  __syncthreads();
  bool k_ready = !k_tma;
  const double inv_l2 = 1.0 / (m.ell * m.ell);
  uint32_t phase = 0;
  for (int64_t q = blockIdx.x; q < nq; q += gridDim.x) {
    if (t == 0) {  // corners, weights, status (FP64, reference order) and the row copies
      int nc = 0;
      int64_t r[8];
      double w[8], dw[8][3];
      const int st = locate(gm, slots, pos[3 * q], pos[3 * q + 1], pos[3 * q + 2], trilinear != 0, nc, r, w, dw);
      meta_i[0] = st;
      uint32_t total = 0;
      for (int c = 0; c < 8; ++c) {
        const bool ok = st == FIF_STATUS_OK && c < nc;
        const int32_t rr = ok ? (int32_t)r[c] : -1;
        meta_i[1 + c] = rr;
        meta_cw[c] = ok ? make_double4(w[c], dw[c][0], dw[c][1], dw[c][2]) : make_double4(0, 0, 0, 0);
        if (c < NC && rr >= 0) {
          const uintptr_t src = reinterpret_cast<uintptr_t>(field + (int64_t)rr * rw);
          meta_i[9 + c] = (int)(src & 15);
          total += (uint32_t)(((src + rw * 4 + 15) & ~(uintptr_t)15) - (src & ~(uintptr_t)15));
        }
      }
      if (st == FIF_STATUS_OK && total > 0) {
        mbar_expect_tx(bar, total);
        for (int c = 0; c < NC; ++c) {
          if (meta_i[1 + c] < 0) continue;
          const uintptr_t src = reinterpret_cast<uintptr_t>(field + (int64_t)meta_i[1 + c] * rw);
          const uintptr_t a0 = src & ~(uintptr_t)15;
          tma_bulk_g2s(rowbuf + (size_t)c * rowcap, reinterpret_cast<const void*>(a0),
                       (uint32_t)(((src + rw * 4 + 15) & ~(uintptr_t)15) - a0), bar);
        }
      }
    }
    __syncthreads();
    const int st = meta_i[0];
    if (st == FIF_STATUS_OK) {
      bool any_copy = false;
#pragma unroll
      for (int c = 0; c < NC; ++c) any_copy |= meta_i[1 + c] >= 0;
      // absent corners (sparse fields) read as zero rows
#pragma unroll
      for (int c = 0; c < NC; ++c)
        if (meta_i[1 + c] < 0)
          for (int i = t; i < (int)(rowcap / 4); i += blockDim.x) reinterpret_cast<float*>(rowbuf + (size_t)c * rowcap)[i] = 0.f;
      // v^r (kernels.py:652-657), then omega = kinv v^r and its z-derivatives (FP64)
      const double zx = axes[3 * q], zy = axes[3 * q + 1], zz = axes[3 * q + 2];
      for (int g = t; g < nv; g += blockDim.x) {
        const double c = __dadd_rn(__dadd_rn(__dmul_rn(zx, m.zs[3 * g]), __dmul_rn(zy, m.zs[3 * g + 1])),
                                   __dmul_rn(zz, m.zs[3 * g + 2]));
        vr[g] = m.sig2 * exp(__dmul_rn(__dsub_rn(c, 1.0), inv_l2));
      }
      if (!k_ready) {
        mbar_wait(kbar, 0);
        k_ready = true;
      }
      __syncthreads();
      for (int k = t; k < nv; k += blockDim.x) {
        double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll 4
        for (int g = 0; g < nv; ++g) {
          const double tg = kin[g * nv + k] * vr[g];
          a0 += tg;
          a1 = fma(tg, m.zs[3 * g], a1);
          a2 = fma(tg, m.zs[3 * g + 1], a2);
          a3 = fma(tg, m.zs[3 * g + 2], a3);
        }
        om[k] = make_double4(a0, a1 * inv_l2, a2 * inv_l2, a3 * inv_l2);
      }
      __syncthreads();
      if (any_copy) {
        mbar_wait(bar, phase);
        phase ^= 1u;
      }
      // k-split contraction: warp w covers samples [k0, k1), lane = packed entry
      const bool on = lane < 21;
      const int e = on ? lane : 0;
      const int kper = (nv + QS_WARPS - 1) / QS_WARPS;
      const int k0 = warp * kper, k1 = min(nv, k0 + kper);
      double w[NC], G[NC], H[MGRAD ? NC : 1][3];
      const float* src[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        w[c] = meta_cw[c].x;
        G[c] = 0.0;
        H[MGRAD ? c : 0][0] = H[MGRAD ? c : 0][1] = H[MGRAD ? c : 0][2] = 0.0;
        src[c] = reinterpret_cast<const float*>(rowbuf + (size_t)c * rowcap + (meta_i[1 + c] >= 0 ? meta_i[9 + c] : 0)) + e;
      }
      double R0 = 0, R1 = 0, R2 = 0;
      if (on) {
        for (int k = k0; k < k1; ++k) {
          const double4 o = om[k];
          double sv[NC];
#pragma unroll
          for (int c = 0; c < NC; ++c) sv[c] = (double)src[c][k * 21];
#pragma unroll
          for (int c = 0; c < NC; ++c) G[c] = fma(o.x, sv[c], G[c]);
          if (MGRAD) {
#pragma unroll
            for (int c = 0; c < NC; ++c) {
              H[MGRAD ? c : 0][0] = fma(o.y, sv[c], H[MGRAD ? c : 0][0]);
              H[MGRAD ? c : 0][1] = fma(o.z, sv[c], H[MGRAD ? c : 0][1]);
              H[MGRAD ? c : 0][2] = fma(o.w, sv[c], H[MGRAD ? c : 0][2]);
            }
          } else if (GRAD) {
            double bl = 0.0;
#pragma unroll
            for (int c = 0; c < NC; ++c) bl = fma(w[c], sv[c], bl);
            R0 = fma(o.y, bl, R0);
            R1 = fma(o.z, bl, R1);
            R2 = fma(o.w, bl, R2);
          }
        }
      }
      double* pw = part + (size_t)warp * NP * 32;
#pragma unroll
      for (int c = 0; c < NC; ++c) pw[c * 32 + lane] = G[c];
      if (MGRAD) {
#pragma unroll
        for (int c = 0; c < NC; ++c)
#pragma unroll
          for (int a = 0; a < 3; ++a) pw[(NC + 3 * c + a) * 32 + lane] = H[MGRAD ? c : 0][a];
      } else if (GRAD) {
        pw[NC * 32 + lane] = R0;
        pw[(NC + 1) * 32 + lane] = R1;
        pw[(NC + 2) * 32 + lane] = R2;
      }
      __syncthreads();
      if (warp == 0) {
        // reduce the warps' partials (fixed order), then the shared output emission
#pragma unroll
        for (int c = 0; c < NC; ++c) G[c] = 0.0;
        R0 = R1 = R2 = 0.0;
#pragma unroll
        for (int c = 0; c < (MGRAD ? NC : 1); ++c) H[c][0] = H[c][1] = H[c][2] = 0.0;
        for (int ww = 0; ww < QS_WARPS; ++ww) {
          const double* pp = part + (size_t)ww * NP * 32;
#pragma unroll
          for (int c = 0; c < NC; ++c) G[c] += pp[c * 32 + lane];
          if (MGRAD) {
#pragma unroll
            for (int c = 0; c < NC; ++c)
#pragma unroll
              for (int a = 0; a < 3; ++a) H[MGRAD ? c : 0][a] += pp[(NC + 3 * c + a) * 32 + lane];
          } else if (GRAD) {
            R0 += pp[NC * 32 + lane];
            R1 += pp[(NC + 1) * 32 + lane];
            R2 += pp[(NC + 2) * 32 + lane];
          }
        }
        const double4 my_cw = lane < NC ? meta_cw[lane] : make_double4(0, 0, 0, 0);
        const int32_t r_lane = lane < NC ? meta_i[1 + lane] : -1;
        emit_outputs<NC, GRAD, METRIC, MGRAD>(out, q, st, lane, on, w, G, R0, R1, R2, H, my_cw, cfim, axes,
                                              r_lane);
      }
    } else if (warp == 0) {
      if (out.fim) for (int i2 = lane; i2 < 36; i2 += 32) out.fim[q * 36 + i2] = 0.0;
      if (out.fim_grad) for (int i2 = lane; i2 < 216; i2 += 32) out.fim_grad[q * 216 + i2] = 0.0;
      if (lane == 0) {
        if (out.trace) out.trace[q] = 0.0;
        if (out.det) out.det[q] = 0.0;
        if (out.lmin) out.lmin[q] = 0.0;
      }
      if (out.trace_grad && lane < 6) out.trace_grad[q * 6 + lane] = 0.0;
      if (out.det_grad && lane < 6) out.det_grad[q * 6 + lane] = 0.0;
      if (out.lmin_grad && lane < 6) out.lmin_grad[q * 6 + lane] = 0.0;
      if (out.status && lane == 0) out.status[q] = (uint8_t)st;
    }
    __syncthreads();  // shared buffers are reused by the next query
  }
}

template <int NC, bool GRAD, bool METRIC, bool MGRAD>
static void launch_small(const fif_model& m, const QueryGeom& gm, const int32_t* slots, const double* pos,
                         const double* axes, int64_t q, int trilinear, const float* field, const QueryOut& out,
                         cudaStream_t st) {
  auto kern = k_query_small<NC, GRAD, METRIC, MGRAD>;
  const int nv = m.n_v;
  const size_t rowcap = ((size_t)nv * 21 * 4 + 16 + 15) & ~(size_t)15;
  const size_t smem = 128 + 8 * sizeof(double4) + NC * rowcap + sizeof(double4) * nv +
                      sizeof(double) * (((nv + 1) & ~1) + QS_WARPS * qs_np<NC, GRAD, METRIC, MGRAD>() * 32 +
                                        8 * qw_cf<METRIC, MGRAD>() + (size_t)nv * nv);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t cap = (int64_t)num_sms() * 4;
  kern<<<(unsigned)(q < cap ? q : cap), QS_WARPS * 32, smem, st>>>(m, gm, slots, pos, axes, q, trilinear, field, out);
}

// ───────────────────────── contraction: trace fields ────────────────────
constexpr int QC_WARPS = 8;
// Rows of n_v scalars: lanes stride over k, per-lane partial sums, warp reduction.
template <typename T, int NC, bool GRAD>
__global__ void __launch_bounds__(QC_WARPS * 32) k_query_trace(int nv, const T* __restrict__ field,
                                                              const double* __restrict__ axes, int64_t nq,
                                                              const uint8_t* __restrict__ status,
                                                              const int32_t* __restrict__ rows,
                                                              const double4* __restrict__ cw,
                                                              const double4* __restrict__ wt, QueryOut out,
                                                              const int32_t* __restrict__ perm) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t q = blockIdx.x * (int64_t)QC_WARPS + warp; q < nq; q += (int64_t)gridDim.x * QC_WARPS) {
    const int st = status[q];
    const int64_t qo = perm ? (int64_t)perm[q] : q;  // q: slot (locality order)
    if (st != FIF_STATUS_OK) {
      if (lane == 0 && out.trace) out.trace[qo] = 0.0;
      if (out.trace_grad && lane < 6) out.trace_grad[qo * 6 + lane] = 0.0;
      if (out.status && lane == 0) out.status[qo] = (uint8_t)st;
      continue;
    }
    const double4* wq = wt + q * nv;
    int32_t r[NC];
    double w[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      r[c] = rows[q * 8 + c];
      w[c] = cw[q * 8 + c].x;
    }
    double G[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) G[c] = 0.0;
    double R0 = 0, R1 = 0, R2 = 0;
    for (int k = lane; k < nv; k += 32) {
      double s[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) s[c] = r[c] >= 0 ? (double)__ldg(field + (int64_t)r[c] * nv + k) : 0.0;
      const double4 om = wq[k];
#pragma unroll
      for (int c = 0; c < NC; ++c) G[c] = fma(om.x, s[c], G[c]);
      if (GRAD) {
        double b = 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c) b = fma(w[c], s[c], b);
        R0 = fma(om.y, b, R0);
        R1 = fma(om.z, b, R1);
        R2 = fma(om.w, b, R2);
      }
    }
    double val = 0, pgx = 0, pgy = 0, pgz = 0;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const double g = warp_sum(G[c]);
      val = fma(w[c], g, val);
      if (GRAD) {
        const double4 d = cw[q * 8 + c];
        pgx = fma(d.y, g, pgx);
        pgy = fma(d.z, g, pgy);
        pgz = fma(d.w, g, pgz);
      }
    }
    if (lane == 0 && out.trace) out.trace[qo] = val;
    if (GRAD && out.trace_grad) {
      R0 = warp_sum(R0);
      R1 = warp_sum(R1);
      R2 = warp_sum(R2);
      const double zx = axes[3 * qo], zy = axes[3 * qo + 1], zz = axes[3 * qo + 2];
      const double g6[6] = {pgx, pgy, pgz, zy * R2 - zz * R1, zz * R0 - zx * R2, zx * R1 - zy * R0};
      if (lane < 6) out.trace_grad[qo * 6 + lane] = g6[lane];
    }
    if (out.status && lane == 0) out.status[qo] = (uint8_t)st;
  }
}

static unsigned query_blocks(int64_t q) {
  int64_t need = (q + QC_WARPS - 1) / QC_WARPS;
  int64_t cap = (int64_t)num_sms() * 32;
  return (unsigned)(need < cap ? (need > 0 ? need : 1) : cap);
}

// Locality order for large batches: queries are processed in Morton order of their
// base voxel (3 x 10 bits), so queries sharing corner rows run close in time and the
// rows are re-read from L2 rather than HBM; results go back to the caller's order.
__device__ __forceinline__ uint32_t spread10(uint32_t v) {
  v &= 1023u;
  v = (v | (v << 16)) & 0x030000FFu;
  v = (v | (v << 8)) & 0x0300F00Fu;
  v = (v | (v << 4)) & 0x030C30C3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}
__global__ void k_query_keys(QueryGeom gm, const double* __restrict__ pos, int64_t nq, uint32_t* __restrict__ keys,
                             int32_t* __restrict__ idx) {
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= nq) return;
  const double inv = 1.0 / gm.vs;
  auto cell = [&](double x, double o, int64_t n) -> uint32_t {
    double g = floor((x - o) * inv);
    g = fmin(fmax(g, 0.0), (double)(n - 1));
    return (uint32_t)((int64_t)g >> (n > 1024 ? 1 : 0));  // 10 bits per axis (coarsened for huge grids)
  };
  const uint32_t ix = cell(pos[3 * q], gm.ox, gm.nx), iy = cell(pos[3 * q + 1], gm.oy, gm.ny),
                 iz = cell(pos[3 * q + 2], gm.oz, gm.nz);
  keys[q] = (spread10(iz) << 2) | (spread10(iy) << 1) | spread10(ix);
  idx[q] = (int32_t)q;
}

template <typename T, int NC, int STAGES, bool GRAD, bool METRIC, bool MGRAD>
static void launch_info(int nv, const T* f, const double* axes, int64_t q, const uint8_t* status, const int32_t* rows,
                        const double4* cw, const double4* wt, const QueryOut& out, const int32_t* perm,
                        cudaStream_t st) {
  auto kern = k_query_info<T, NC, STAGES, GRAD, METRIC, MGRAD>;
  const size_t smem = ((QWShape<T>::CHUNK + 127) & ~127u) +
                      (size_t)qw_wpb(STAGES) * ((qw_warp_bytes<T, NC, STAGES, METRIC, MGRAD>() + 127) & ~127u);
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  constexpr int WPB = qw_wpb(STAGES);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, WPB * 32, smem);
  const int64_t need = (q + WPB - 1) / WPB;
  const int64_t cap = (int64_t)num_sms() * (per_sm > 0 ? per_sm : 1);
  kern<<<(unsigned)(need < cap ? need : cap), WPB * 32, smem, st>>>(nv, f, axes, q, status, rows, cw, wt, out, perm);
}

template <typename T, int NC>
static void launch_info_nc(bool grad, bool metric, bool mgrad, int nv, const T* f, const double* axes, int64_t q,
                           const uint8_t* status, const int32_t* rows, const double4* cw, const double4* wt,
                           const QueryOut& out, const int32_t* perm, cudaStream_t st) {
  // value/gradient streaming: 2 stages, 3 CTAs/SM; metric variants (det/lmin, LU and
  // Jacobi per corner, more registers): 3 stages, 2 CTAs/SM
  static const int stages_env = getenv("FIF_QW_STAGES") ? atoi(getenv("FIF_QW_STAGES")) : 2;
  if (q <= (int64_t)num_sms() * 3) {  // small batch: one query per CTA, all k-chunks in flight
    constexpr int S = QW_SMALL_STAGES;
    if (mgrad) launch_info<T, NC, S, true, true, true>(nv, f, axes, q, status, rows, cw, wt, out, perm, st);
    else if (metric && grad) launch_info<T, NC, S, true, true, false>(nv, f, axes, q, status, rows, cw, wt, out, perm, st);
    else if (metric) launch_info<T, NC, S, false, true, false>(nv, f, axes, q, status, rows, cw, wt, out, perm, st);
    else if (grad) launch_info<T, NC, S, true, false, false>(nv, f, axes, q, status, rows, cw, wt, out, perm, st);
    else launch_info<T, NC, S, false, false, false>(nv, f, axes, q, status, rows, cw, wt, out, perm, st);
    return;
  }
  if (metric) {
    if (mgrad) launch_info<T, NC, 3, true, true, true>(nv, f, axes, q, status, rows, cw, wt, out, perm, st);
    else if (grad) launch_info<T, NC, 3, true, true, false>(nv, f, axes, q, status, rows, cw, wt, out, perm, st);
    else launch_info<T, NC, 3, false, true, false>(nv, f, axes, q, status, rows, cw, wt, out, perm, st);
  } else if (stages_env == 3) {
    if (grad) launch_info<T, NC, 3, true, false, false>(nv, f, axes, q, status, rows, cw, wt, out, perm, st);
    else launch_info<T, NC, 3, false, false, false>(nv, f, axes, q, status, rows, cw, wt, out, perm, st);
  } else {
    if (grad) launch_info<T, NC, 2, true, false, false>(nv, f, axes, q, status, rows, cw, wt, out, perm, st);
    else launch_info<T, NC, 2, false, false, false>(nv, f, axes, q, status, rows, cw, wt, out, perm, st);
  }
}

template <typename T>
static int launch_contract(int kind, bool trilinear, bool grad, bool metric, bool mgrad, int nv, const void* field,
                           const double* axes, int64_t q, const uint8_t* status, const int32_t* rows,
                           const double4* cw, const double4* wt, const QueryOut& out, const int32_t* perm,
                           cudaStream_t st) {
  const T* f = reinterpret_cast<const T*>(field);
  if (kind == FIF_KIND_TRACE) {
    const unsigned blocks = query_blocks(q);
    const int threads = QC_WARPS * 32;
#define QT(NC, G) k_query_trace<T, NC, G><<<blocks, threads, 0, st>>>(nv, f, axes, q, status, rows, cw, wt, out, perm)
    if (trilinear) { if (grad) QT(8, true); else QT(8, false); }
    else { if (grad) QT(1, true); else QT(1, false); }
#undef QT
    FIF_CHECK_LAUNCH("k_query_trace");
    return FIF_OK;
  }
  if (trilinear) launch_info_nc<T, 8>(grad, metric, mgrad, nv, f, axes, q, status, rows, cw, wt, out, perm, st);
  else launch_info_nc<T, 1>(grad, metric, mgrad, nv, f, axes, q, status, rows, cw, wt, out, perm, st);
  FIF_CHECK_LAUNCH("k_query_info");
  return FIF_OK;
}

}  // namespace fif

using namespace fif;

extern "C" int fif_query(int factor_kind, const fif_model* model, const fif_grid* grid, const void* d_field,
                         const int32_t* d_slots, const double* d_positions, const double* d_axes, int64_t q, int mode,
                         uint32_t flags, double* d_trace, double* d_trace_grad, double* d_fim, double* d_fim_grad,
                         double* d_det, double* d_lmin, uint8_t* d_status, void* stream) {
  fif_query_out o{d_trace, d_trace_grad, d_fim, d_fim_grad, d_det, nullptr, d_lmin, nullptr, d_status};
  return fif_query_ex(factor_kind, model, grid, d_field, d_slots, d_positions, d_axes, q, mode, flags, &o, stream);
}

// Corner table of a batch of positions (debug / parity ABI fif_locate): exactly the
// locate() the query kernels run, with rows reported as the reference's x-major linear
// voxel index (field.py:81-83) so they compare with kernels._nb_locate_nearest /
// the trilinear corner block (kernels.py:628-635, 678-702) bit for bit.
__global__ void k_locate(QueryGeom gm, const double* __restrict__ pos, int64_t q, int trilinear,
                         int64_t* __restrict__ index, double* __restrict__ weight, uint8_t* __restrict__ status) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= q) return;
  int nc = 0;
  int64_t rows[8];
  double w[8], dw[8][3];
  const int s = locate(gm, nullptr, pos[3 * i], pos[3 * i + 1], pos[3 * i + 2], trilinear != 0, nc, rows, w, dw);
  status[i] = (uint8_t)s;
  for (int k = 0; k < 8; ++k) {
    int64_t lin = -1;
    double wk = 0.0;
    if (s == FIF_STATUS_OK && k < nc) {
      const int64_t j = rows[k];  // internal z-major row of the dense grid
      const int64_t ix = j % gm.nx, r = j / gm.nx, iy = r % gm.ny, iz = r / gm.ny;
      lin = (ix * gm.ny + iy) * gm.nz + iz;
      wk = w[k];
    }
    if (index) index[8 * i + k] = lin;
    if (weight) weight[8 * i + k] = wk;
  }
}

extern "C" int fif_locate(const fif_grid* grid, const double* d_positions, int64_t q, int mode, int64_t* d_index,
                          double* d_weight, uint8_t* d_status, void* stream) {
  FIF_CHECK_ARG(grid && d_status && (q == 0 || d_positions), "fif_locate: NULL argument");
  FIF_CHECK_ARG(q >= 0, "fif_locate: negative query count");
  FIF_CHECK_ARG(mode == FIF_MODE_NEAREST || mode == FIF_MODE_TRILINEAR, "fif_locate: unknown mode %d", mode);
  FIF_CHECK_ARG(grid->voxel_size > 0 && grid->dims[0] > 0 && grid->dims[1] > 0 && grid->dims[2] > 0,
                "fif_locate: empty grid");
  if (q == 0) return FIF_OK;
  QueryGeom gm{grid->origin[0], grid->origin[1], grid->origin[2], grid->voxel_size,
               grid->dims[0],   grid->dims[1],   grid->dims[2]};
  k_locate<<<(unsigned)((q + 255) / 256), 256, 0, (cudaStream_t)stream>>>(gm, d_positions, q,
                                                                         mode == FIF_MODE_TRILINEAR, d_index,
                                                                         d_weight, d_status);
  FIF_CHECK_LAUNCH("k_locate");
  return FIF_OK;
}

extern "C" int fif_query_ex(int factor_kind, const fif_model* model, const fif_grid* grid, const void* d_field,
                            const int32_t* d_slots, const double* d_positions, const double* d_axes, int64_t q,
                            int mode, uint32_t flags, const fif_query_out* o, void* stream) {
  return fif_query_ex2(factor_kind, model, grid, d_field, nullptr, d_slots, d_positions, d_axes, q, mode, flags, o,
                       stream);
}

extern "C" int fif_query_ex2(int factor_kind, const fif_model* model, const fif_grid* grid, const void* d_field,
                             const double* d_trace_rows, const int32_t* d_slots, const double* d_positions,
                             const double* d_axes, int64_t q, int mode, uint32_t flags, const fif_query_out* o,
                             void* stream) {
  FIF_CHECK_ARG(model && grid && o, "fif_query: NULL model/grid/outputs");
  FIF_CHECK_ARG(factor_kind == FIF_KIND_INFO || factor_kind == FIF_KIND_TRACE, "fif_query: bad factor_kind");
  FIF_CHECK_ARG(mode == FIF_MODE_NEAREST || mode == FIF_MODE_TRILINEAR, "fif_query: bad mode %d", mode);
  FIF_CHECK_ARG(q >= 0, "fif_query: q < 0");
  if (q == 0) return FIF_OK;
  FIF_CHECK_ARG(d_field && d_positions && d_axes, "fif_query: NULL field/positions/axes");
  FIF_CHECK_ARG(model->kind == FIF_MODEL_QUAD || (model->kind == FIF_MODEL_GP && model->zs && model->kinv),
                "fif_query: bad model");
  const bool info = factor_kind == FIF_KIND_INFO;
  const bool want_g = (flags & FIF_Q_GRAD) != 0;
  FIF_CHECK_ARG(info || !((o->fim && (flags & FIF_Q_FULL)) || (o->fim_grad && (flags & FIF_Q_FULL) && want_g) ||
                          (o->det && (flags & FIF_Q_DET)) || (o->lmin && (flags & FIF_Q_LMIN))),
                "fif_query: full FIM / det / lmin need an info field (WrongFactorKind)");
  FIF_CHECK_ARG(grid->voxel_size > 0, "fif_query: voxel_size <= 0");
  const int nv = model->kind == FIF_MODEL_QUAD ? 10 : model->n_v;
  FIF_CHECK_ARG(nv >= 1 && nv <= 1024, "fif_query: n_v out of range");
  // bound the per-call scratch (32 nv bytes of rotation weights per query): very large
  // batches run as consecutive slices of kQueryChunk queries on the same stream
  // (capped so the scratch of one slice stays near 1 GiB: 2^18..2^21 queries)
  int64_t kQueryChunk = ((int64_t)1 << 30) / ((int64_t)nv * 32 + 320);
  kQueryChunk = kQueryChunk < ((int64_t)1 << 18) ? ((int64_t)1 << 18) : (kQueryChunk > ((int64_t)1 << 21) ? ((int64_t)1 << 21) : kQueryChunk);
  if (q > kQueryChunk) {
    for (int64_t q0 = 0; q0 < q; q0 += kQueryChunk) {
      const int64_t n = q - q0 < kQueryChunk ? q - q0 : kQueryChunk;
      auto sl = [&](double* p, int64_t w) { return p ? p + q0 * w : nullptr; };
      fif_query_out os{sl(o->trace, 1),    sl(o->trace_grad, 6), sl(o->fim, 36),     sl(o->fim_grad, 216),
                       sl(o->det, 1),      sl(o->det_grad, 6),   sl(o->lmin, 1),     sl(o->lmin_grad, 6),
                       o->status ? o->status + q0 : nullptr};
      const int rc = fif_query_ex2(factor_kind, model, grid, d_field, d_trace_rows, d_slots, d_positions + 3 * q0,
                                   d_axes + 3 * q0, n, mode, flags, &os, stream);
      if (rc != FIF_OK) return rc;
    }
    return FIF_OK;
  }
  QueryGeom gm{grid->origin[0], grid->origin[1], grid->origin[2], grid->voxel_size,
               grid->dims[0],   grid->dims[1],   grid->dims[2]};
  QueryOut out{(flags & FIF_Q_TRACE) ? o->trace : nullptr,
               (flags & FIF_Q_TRACE) && want_g ? o->trace_grad : nullptr,
               (flags & FIF_Q_FULL) ? o->fim : nullptr,
               (flags & FIF_Q_FULL) && want_g ? o->fim_grad : nullptr,
               (flags & FIF_Q_DET) ? o->det : nullptr,
               (flags & FIF_Q_DET) && want_g ? o->det_grad : nullptr,
               (flags & FIF_Q_LMIN) ? o->lmin : nullptr,
               (flags & FIF_Q_LMIN) && want_g ? o->lmin_grad : nullptr,
               o->status};
  // trace outputs of an info field from its FP64 trace table (d_trace_rows): the trace
  // contraction runs as a trace-field contraction on those rows, the remaining outputs on
  // d_field, both from one prep (corners + rotation weights)
  const bool split_trace = info && d_trace_rows != nullptr && out.trace != nullptr;
  QueryOut out_tr{};
  if (split_trace) {
    out_tr.trace = out.trace;
    out_tr.trace_grad = out.trace_grad;
    out.trace = out.trace_grad = nullptr;
  }
  const bool main_work = out.trace || out.fim || out.det || out.lmin;
  if (split_trace && !main_work) {  // the trace contraction reports the status
    out_tr.status = out.status;
    out.status = nullptr;
  }
  const bool mgrad = info && (out.det_grad || out.lmin_grad);
  const bool grad = want_g && (out.trace_grad || out.fim_grad || mgrad);
  const bool grad_tr = want_g && out_tr.trace_grad;
  const bool metric = info && (out.det || out.lmin);
  const bool trilinear = mode == FIF_MODE_TRILINEAR;
  cudaStream_t st = (cudaStream_t)stream;
  // small GP info batches (latency-bound): one fused kernel, one CTA per query
  static const bool no_small = getenv("FIF_QUERY_NO_FUSED_SMALL") != nullptr;
  if (!split_trace && info && model->kind == FIF_MODEL_GP && !(flags & FIF_Q_FIELD_F64) &&
      q <= (int64_t)num_sms() * 3 && !no_small &&
      (size_t)nv * 21 * 4 * (trilinear ? 8 : 1) + (size_t)nv * nv * 8 <= 150 * 1024) {
    const float* ff = reinterpret_cast<const float*>(d_field);
    const int tri = trilinear ? 1 : 0;
#define QSM(NC)                                                                                              \
  do {                                                                                                       \
    if (mgrad) launch_small<NC, true, true, true>(*model, gm, d_slots, d_positions, d_axes, q, tri, ff, out, st); \
    else if (metric && grad) launch_small<NC, true, true, false>(*model, gm, d_slots, d_positions, d_axes, q, tri, ff, out, st); \
    else if (metric) launch_small<NC, false, true, false>(*model, gm, d_slots, d_positions, d_axes, q, tri, ff, out, st); \
    else if (grad) launch_small<NC, true, false, false>(*model, gm, d_slots, d_positions, d_axes, q, tri, ff, out, st); \
    else launch_small<NC, false, false, false>(*model, gm, d_slots, d_positions, d_axes, q, tri, ff, out, st); \
  } while (0)
    if (trilinear) QSM(8);
    else QSM(1);
#undef QSM
    FIF_CHECK_LAUNCH("k_query_small");
    return FIF_OK;
  }
  // stream-ordered scratch: status, rows, corner weights, rotation weights
  const size_t b_status = ((size_t)q + 255) & ~(size_t)255;
  const size_t b_rows = (size_t)q * 8 * sizeof(int32_t);
  const size_t b_cw = (size_t)q * 8 * sizeof(double4);
  const size_t b_wt = (size_t)q * nv * sizeof(double4);
  static std::atomic<uint64_t> pool_set{0};
  if (needs_setup(pool_set)) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      // keep up to 1 GiB of freed scratch reserved between calls (no re-allocation for
      // planner-sized batches); anything above is returned to the device at the next
      // synchronisation, so one huge batch does not pin memory torch may need later
      uint64_t thr = 1ull << 30;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    mark_setup(pool_set);
  }
  unsigned char* scratch = nullptr;
  if (cudaMallocAsync(&scratch, b_status + b_rows + b_cw + b_wt + 256, st) != cudaSuccess) {
    set_error("fif_query: cudaMallocAsync of %zu bytes failed", b_status + b_rows + b_cw + b_wt);
    return FIF_ERR_CUDA;
  }
  uint8_t* s_status = scratch;
  double4* s_cw = reinterpret_cast<double4*>(scratch + b_status);
  int32_t* s_rows = reinterpret_cast<int32_t*>(scratch + b_status + b_cw);
  double4* s_wt = reinterpret_cast<double4*>(scratch + b_status + b_cw + ((b_rows + 255) & ~(size_t)255));
  // locality order (Morton order of the base voxel) for batches large enough to pay for the sort
  int32_t* perm = nullptr;
  unsigned char* sort_buf = nullptr;
  static const int64_t sort_min = getenv("FIF_QUERY_SORT_MIN") ? atoll(getenv("FIF_QUERY_SORT_MIN")) : 262144;
  if (q >= sort_min && q < (int64_t)INT32_MAX && sort_min > 0) {
    size_t temp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, temp, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (const int32_t*)nullptr, (int32_t*)nullptr, (int)q, 0, 30, st);
    const size_t b4 = ((size_t)q * 4 + 255) & ~(size_t)255;
    if (cudaMallocAsync(&sort_buf, 4 * b4 + temp, st) != cudaSuccess) {
      set_error("fif_query: cudaMallocAsync for the locality sort failed");
      cudaFreeAsync(scratch, st);
      return FIF_ERR_CUDA;
    }
    uint32_t* keys = reinterpret_cast<uint32_t*>(sort_buf);
    uint32_t* keys2 = reinterpret_cast<uint32_t*>(sort_buf + b4);
    int32_t* idx = reinterpret_cast<int32_t*>(sort_buf + 2 * b4);
    perm = reinterpret_cast<int32_t*>(sort_buf + 3 * b4);
    k_query_keys<<<(unsigned)((q + 255) / 256), 256, 0, st>>>(gm, d_positions, q, keys, idx);
    FIF_CHECK_LAUNCH("k_query_keys");
    cub::DeviceRadixSort::SortPairs(sort_buf + 4 * b4, temp, keys, keys2, idx, perm, (int)q, 0, 30, st);
    FIF_CHECK_LAUNCH("fif_query(locality sort)");
  }
  const int np8 = (nv + 7) & ~7, ntiles = np8 / 8;
  const size_t dmma_smem =
      sizeof(double) * ((size_t)((np8 * nv + 8 + 15) & ~15) + (size_t)QD_Q * np8 + 4 * (size_t)np8 + 4 * (size_t)QD_Q);
  static const bool simt_prep = getenv("FIF_QUERY_PREP_SIMT") != nullptr;
  if (model->kind == FIF_MODEL_GP && ntiles <= 12 && !simt_prep) {
    double* wtd = reinterpret_cast<double*>(s_wt);
    const int tri = trilinear ? 1 : 0;
    const bool small = q <= 1024;
    const size_t sm = small ? dmma_smem - sizeof(double) * (size_t)(QD_Q - 8) * np8 : dmma_smem;
    const bool pgrad = grad || grad_tr;
    switch (ntiles) {
#define PG(NT)                                                                                                   \
  case NT:                                                                                                       \
    if (small && pgrad) launch_prep_gp<NT, 8, 4>(sm, q, st, *model, gm, d_slots, d_positions, d_axes, tri, s_status, \
                                                s_rows, s_cw, wtd, perm);                                        \
    else if (small) launch_prep_gp<NT, 8, 1>(sm, q, st, *model, gm, d_slots, d_positions, d_axes, tri, s_status,   \
                                             s_rows, s_cw, wtd, perm);                                           \
    else if (pgrad) launch_prep_gp<NT, 32, 4>(sm, q, st, *model, gm, d_slots, d_positions, d_axes, tri, s_status,   \
                                             s_rows, s_cw, wtd, perm);                                           \
    else launch_prep_gp<NT, 32, 1>(sm, q, st, *model, gm, d_slots, d_positions, d_axes, tri, s_status, s_rows,     \
                                   s_cw, wtd, perm);                                                             \
    break;
      PG(1) PG(2) PG(3) PG(4) PG(5) PG(6) PG(7) PG(8) PG(9) PG(10) PG(11) PG(12)
#undef PG
    }
    FIF_CHECK_LAUNCH("k_query_prep_gp");
  } else {
    const size_t prep_smem = sizeof(double) * (QP_Q + 3) * nv;
    if (prep_smem > 48 * 1024)
      cudaFuncSetAttribute(k_query_prep, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)prep_smem);
    k_query_prep<<<(unsigned)((q + QP_Q - 1) / QP_Q), QP_THREADS, prep_smem, st>>>(
        *model, gm, d_slots, d_positions, d_axes, q, trilinear ? 1 : 0, s_status, s_rows, s_cw, s_wt, perm);
    FIF_CHECK_LAUNCH("k_query_prep");
  }
  const bool f64 = model->kind == FIF_MODEL_QUAD || (flags & FIF_Q_FIELD_F64);
  int rc = FIF_OK;
  if (main_work || !split_trace)
    rc = f64 ? launch_contract<double>(factor_kind, trilinear, grad, metric, mgrad, nv, d_field, d_axes, q, s_status,
                                       s_rows, s_cw, s_wt, out, perm, st)
             : launch_contract<float>(factor_kind, trilinear, grad, metric, mgrad, nv, d_field, d_axes, q, s_status,
                                      s_rows, s_cw, s_wt, out, perm, st);
  if (rc == FIF_OK && split_trace)
    rc = launch_contract<double>(FIF_KIND_TRACE, trilinear, grad_tr, false, false, nv, d_trace_rows, d_axes, q,
                                 s_status, s_rows, s_cw, s_wt, out_tr, perm, st);
  if (sort_buf) cudaFreeAsync(sort_buf, st);
  cudaFreeAsync(scratch, st);
  return rc;
}
