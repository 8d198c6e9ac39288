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

namespace fif {

constexpr int Q_WARPS = 8;

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

// Rotation weights into smem: wt[0][k] = weight, wt[1+a][k] = d weight / d z_a.
// quad: v^r (kernels.py:638-649); GP: omega = kinv v^r with v^r_g = s2 exp((z.zs_g - 1)/l^2)
// (kernels.py:652-657) — kinv symmetric, so omega . S == v^r . (kinv S).
__device__ __forceinline__ void rotation_weights(const fif_model& m, int nv, double zx, double zy, double zz,
                                                 double* __restrict__ wt, double* __restrict__ tmp, int lane) {
  if (m.kind == FIF_MODEL_QUAD) {
    if (lane < 10) {
      const double k2 = m.k2, k1 = m.k1, k0 = m.k0, t2 = 2.0 * k2;
      double v = 0, gx = 0, gy = 0, gz = 0;
      switch (lane) {
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
      wt[lane] = v;
      wt[nv + lane] = gx;
      wt[2 * nv + lane] = gy;
      wt[3 * nv + lane] = gz;
    }
    __syncwarp();
    return;
  }
  const double inv_l2 = 1.0 / (m.ell * m.ell);
  for (int g = lane; g < nv; g += 32) {
    double zsx = m.zs[3 * g], zsy = m.zs[3 * g + 1], zsz = m.zs[3 * g + 2];
    double c = __dadd_rn(__dadd_rn(__dmul_rn(zx, zsx), __dmul_rn(zy, zsy)), __dmul_rn(zz, zsz));
    double vr = m.sig2 * exp(__dmul_rn(__dsub_rn(c, 1.0), inv_l2));
    tmp[g] = vr;
    double s = vr * inv_l2;
    tmp[nv + g] = s * zsx;
    tmp[2 * nv + g] = s * zsy;
    tmp[3 * nv + g] = s * zsz;
  }
  __syncwarp();
  for (int k = lane; k < nv; k += 32) {
    double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
    for (int g = 0; g < nv; ++g) {
      double kg = __ldg(m.kinv + (int64_t)g * nv + k);
      a0 = fma(kg, tmp[g], a0);
      a1 = fma(kg, tmp[nv + g], a1);
      a2 = fma(kg, tmp[2 * nv + g], a2);
      a3 = fma(kg, tmp[3 * nv + g], a3);
    }
    wt[k] = a0;
    wt[nv + k] = a1;
    wt[2 * nv + k] = a2;
    wt[3 * nv + k] = a3;
  }
  __syncwarp();
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// 6x6 determinant (partial-pivot LU) and smallest eigenvalue (cyclic Jacobi), FP64.
__device__ double det6(const double* a_in) {
  double a[36];
  for (int i = 0; i < 36; ++i) a[i] = a_in[i];
  double det = 1.0;
  for (int c = 0; c < 6; ++c) {
    int p = c;
    double best = fabs(a[6 * c + c]);
    for (int r = c + 1; r < 6; ++r)
      if (fabs(a[6 * r + c]) > best) { best = fabs(a[6 * r + c]); p = r; }
    if (best == 0.0) return 0.0;
    if (p != c) {
      for (int k = 0; k < 6; ++k) { double t = a[6 * c + k]; a[6 * c + k] = a[6 * p + k]; a[6 * p + k] = t; }
      det = -det;
    }
    double piv = a[6 * c + c];
    det *= piv;
    for (int r = c + 1; r < 6; ++r) {
      double f = a[6 * r + c] / piv;
      for (int k = c + 1; k < 6; ++k) a[6 * r + k] -= f * a[6 * c + k];
    }
  }
  return det;
}
__device__ double lmin6(const double* a_in) {
  double a[36];
  for (int i = 0; i < 36; ++i) a[i] = a_in[i];
  for (int sweep = 0; sweep < 64; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int r = 0; r < 6; ++r)
      for (int c = 0; c < 6; ++c) {
        double v = a[6 * r + c] * a[6 * r + c];
        tot += v;
        if (r != c) off += v;
      }
    if (off <= 1e-30 * tot || off == 0.0) break;
    for (int p = 0; p < 5; ++p)
      for (int q = p + 1; q < 6; ++q) {
        double apq = a[6 * p + q];
        if (apq == 0.0) continue;
        double theta = (a[6 * q + q] - a[6 * p + p]) / (2.0 * apq);
        double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        double cs = 1.0 / sqrt(t * t + 1.0), sn = t * cs;
        for (int k = 0; k < 6; ++k) {
          double akp = a[6 * k + p], akq = a[6 * k + q];
          a[6 * k + p] = cs * akp - sn * akq;
          a[6 * k + q] = sn * akp + cs * akq;
        }
        for (int k = 0; k < 6; ++k) {
          double apk = a[6 * p + k], aqk = a[6 * q + k];
          a[6 * p + k] = cs * apk - sn * aqk;
          a[6 * q + k] = sn * apk + cs * aqk;
        }
      }
  }
  double m = a[0];
  for (int k = 1; k < 6; ++k) m = fmin(m, a[7 * k]);
  return m;
}

__constant__ int kPackR[21] = {0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 1, 2, 2, 2, 2, 3, 3, 3, 4, 4, 5};
__constant__ int kPackC[21] = {0, 1, 2, 3, 4, 5, 1, 2, 3, 4, 5, 2, 3, 4, 5, 3, 4, 5, 4, 5, 5};
__constant__ int kIsDiag[21] = {1, 0, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 1, 0, 0, 1, 0, 1};

template <typename T>
__device__ __forceinline__ double ld_field(const T* __restrict__ p) {
  return (double)__ldg(p);
}

struct QueryOut {
  double* trace;
  double* trace_grad;
  double* fim;
  double* fim_grad;
  double* det;
  double* lmin;
  uint8_t* status;
};

// KIND: FIF_KIND_INFO rows (nv,21) | FIF_KIND_TRACE rows (nv)
template <typename T, int KIND, bool GRAD, bool METRIC>
__global__ void __launch_bounds__(Q_WARPS * 32) k_query(fif_model m, QueryGeom gm, const T* __restrict__ field,
                                                        const int32_t* __restrict__ slots,
                                                        const double* __restrict__ pos,
                                                        const double* __restrict__ axes, int64_t nq, int trilinear,
                                                        QueryOut out) {
  extern __shared__ double qsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nv = m.kind == FIF_MODEL_QUAD ? 10 : m.n_v;
  double* wt = qsm + warp * (8 * nv + 8 * 21);  // [4][nv] weights
  double* tmp = wt + 4 * nv;                     // [4][nv] GP scratch
  double* cornerfim = tmp + 4 * nv;              // [8][21] (METRIC)
  const int64_t rw = KIND == FIF_KIND_INFO ? (int64_t)nv * 21 : nv;
  for (int64_t q = blockIdx.x * (int64_t)Q_WARPS + warp; q < nq; q += (int64_t)gridDim.x * Q_WARPS) {
    const double px = pos[3 * q], py = pos[3 * q + 1], pz = pos[3 * q + 2];
    const double zx = axes[3 * q], zy = axes[3 * q + 1], zz = axes[3 * q + 2];
    int nc = 0;
    int64_t rows[8];
    double w[8], dw[8][3];
    const int st = locate(gm, slots, px, py, pz, trilinear != 0, nc, rows, w, dw);
    if (out.status && lane == 0) out.status[q] = (uint8_t)st;
    if (st != FIF_STATUS_OK) {
      if (KIND == FIF_KIND_INFO) {
        for (int j = lane; j < 36; j += 32) if (out.fim) out.fim[q * 36 + j] = 0.0;
        if (out.fim_grad) for (int j = lane; j < 216; j += 32) out.fim_grad[q * 216 + j] = 0.0;
      }
      if (lane == 0) {
        if (out.trace) out.trace[q] = 0.0;
        if (out.det) out.det[q] = 0.0;
        if (out.lmin) out.lmin[q] = 0.0;
      }
      if (out.trace_grad && lane < 6) out.trace_grad[q * 6 + lane] = 0.0;
      continue;
    }
    rotation_weights(m, nv, zx, zy, zz, wt, tmp, lane);
    // val, d/dt (3), d/dz (3)
    double val = 0, pgx = 0, pgy = 0, pgz = 0, rgx = 0, rgy = 0, rgz = 0;
    double mdet = 0, mlmin = 0;
    if (KIND == FIF_KIND_INFO) {
      const bool on = lane < 21;
      const int e = on ? lane : 0;
      for (int c = 0; c < nc; ++c) {
        if (rows[c] < 0) {
          if (METRIC && on) cornerfim[c * 21 + e] = 0.0;
          continue;  // empty voxel: exact zero factor (field.py:12)
        }
        const T* f = field + rows[c] * rw + e;
        double g0 = 0, g1 = 0, g2 = 0, g3 = 0;
        if (on) {
          int k = 0;
          for (; k + 4 <= nv; k += 4) {
            double f0 = ld_field(f + (k + 0) * 21), f1 = ld_field(f + (k + 1) * 21);
            double f2 = ld_field(f + (k + 2) * 21), f3 = ld_field(f + (k + 3) * 21);
            g0 = fma(wt[k], f0, g0); g0 = fma(wt[k + 1], f1, g0); g0 = fma(wt[k + 2], f2, g0); g0 = fma(wt[k + 3], f3, g0);
            if (GRAD) {
              g1 = fma(wt[nv + k], f0, g1); g1 = fma(wt[nv + k + 1], f1, g1);
              g1 = fma(wt[nv + k + 2], f2, g1); g1 = fma(wt[nv + k + 3], f3, g1);
              g2 = fma(wt[2 * nv + k], f0, g2); g2 = fma(wt[2 * nv + k + 1], f1, g2);
              g2 = fma(wt[2 * nv + k + 2], f2, g2); g2 = fma(wt[2 * nv + k + 3], f3, g2);
              g3 = fma(wt[3 * nv + k], f0, g3); g3 = fma(wt[3 * nv + k + 1], f1, g3);
              g3 = fma(wt[3 * nv + k + 2], f2, g3); g3 = fma(wt[3 * nv + k + 3], f3, g3);
            }
          }
          for (; k < nv; ++k) {
            double f0 = ld_field(f + k * 21);
            g0 = fma(wt[k], f0, g0);
            if (GRAD) {
              g1 = fma(wt[nv + k], f0, g1);
              g2 = fma(wt[2 * nv + k], f0, g2);
              g3 = fma(wt[3 * nv + k], f0, g3);
            }
          }
        }
        val = fma(w[c], g0, val);
        if (GRAD) {
          pgx = fma(dw[c][0], g0, pgx);
          pgy = fma(dw[c][1], g0, pgy);
          pgz = fma(dw[c][2], g0, pgz);
          rgx = fma(w[c], g1, rgx);
          rgy = fma(w[c], g2, rgy);
          rgz = fma(w[c], g3, rgz);
        }
        if (METRIC && on) cornerfim[c * 21 + e] = g0;
      }
      if (out.fim && lane < 21) {
        int r = kPackR[lane], cc = kPackC[lane];
        out.fim[q * 36 + r * 6 + cc] = val;
        out.fim[q * 36 + cc * 6 + r] = val;
      }
      // d/dtheta = z x d/dz
      const double tgx = zy * rgz - zz * rgy, tgy = zz * rgx - zx * rgz, tgz = zx * rgy - zy * rgx;
      if (GRAD && out.fim_grad && lane < 21) {
        int r = kPackR[lane], cc = kPackC[lane];
        double g[6] = {pgx, pgy, pgz, tgx, tgy, tgz};
        for (int j = 0; j < 6; ++j) {
          out.fim_grad[q * 216 + j * 36 + r * 6 + cc] = g[j];
          out.fim_grad[q * 216 + j * 36 + cc * 6 + r] = g[j];
        }
      }
      if (out.trace || (GRAD && out.trace_grad)) {
        const bool dg = lane < 21 && kIsDiag[lane];
        double tv = warp_sum(dg ? val : 0.0);
        if (out.trace && lane == 0) out.trace[q] = tv;
        if (GRAD && out.trace_grad) {
          double g[6] = {pgx, pgy, pgz, tgx, tgy, tgz};
          for (int j = 0; j < 6; ++j) {
            double s = warp_sum(dg ? g[j] : 0.0);
            if (lane == j) out.trace_grad[q * 6 + j] = s;
          }
        }
      }
      if (METRIC) {
        __syncwarp();
        // corner metric by lanes 0..nc-1, blended in the reference's corner order
        double mv_det = 0, mv_lmin = 0;
        if (lane < nc) {
          double a[36];
          for (int j = 0; j < 21; ++j) {
            double v = cornerfim[lane * 21 + j];
            a[kPackR[j] * 6 + kPackC[j]] = v;
            a[kPackC[j] * 6 + kPackR[j]] = v;
          }
          if (rows[lane] >= 0) {
            if (out.det) mv_det = det6(a);
            if (out.lmin) mv_lmin = lmin6(a);
          }
        }
        for (int c = 0; c < nc; ++c) {
          double dd = __shfl_sync(0xffffffffu, mv_det, c), ll = __shfl_sync(0xffffffffu, mv_lmin, c);
          if (w[c] != 0.0) {
            mdet = fma(w[c], dd, mdet);
            mlmin = fma(w[c], ll, mlmin);
          }
        }
        if (lane == 0) {
          if (out.det) out.det[q] = mdet;
          if (out.lmin) out.lmin[q] = mlmin;
        }
        __syncwarp();
      }
    } else {
      // trace field: lanes over k, 7 per-lane partial sums, warp reduction
      for (int c = 0; c < nc; ++c) {
        if (rows[c] < 0) continue;
        const T* f = field + rows[c] * rw;
        for (int k = lane; k < nv; k += 32) {
          double s = ld_field(f + k);
          double ws = wt[k] * s;
          val = fma(w[c], ws, val);
          if (GRAD) {
            pgx = fma(dw[c][0], ws, pgx);
            pgy = fma(dw[c][1], ws, pgy);
            pgz = fma(dw[c][2], ws, pgz);
            rgx = fma(w[c], wt[nv + k] * s, rgx);
            rgy = fma(w[c], wt[2 * nv + k] * s, rgy);
            rgz = fma(w[c], wt[3 * nv + k] * s, rgz);
          }
        }
      }
      val = warp_sum(val);
      if (out.trace && lane == 0) out.trace[q] = val;
      if (GRAD && out.trace_grad) {
        pgx = warp_sum(pgx); pgy = warp_sum(pgy); pgz = warp_sum(pgz);
        rgx = warp_sum(rgx); rgy = warp_sum(rgy); rgz = warp_sum(rgz);
        double g[6] = {pgx, pgy, pgz, zy * rgz - zz * rgy, zz * rgx - zx * rgz, zx * rgy - zy * rgx};
        if (lane < 6) out.trace_grad[q * 6 + lane] = g[lane];
      }
    }
    __syncwarp();
  }
}

template <typename T, int KIND, bool GRAD, bool METRIC>
static int launch_query(const fif_model& m, const QueryGeom& gm, const void* field, const int32_t* slots,
                        const double* pos, const double* axes, int64_t q, int mode, const QueryOut& out,
                        cudaStream_t st) {
  const int nv = m.kind == FIF_MODEL_QUAD ? 10 : m.n_v;
  size_t smem = sizeof(double) * Q_WARPS * (8 * nv + 8 * 21);
  auto kern = k_query<T, KIND, GRAD, METRIC>;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int64_t need = (q + Q_WARPS - 1) / Q_WARPS;
  int64_t cap = (int64_t)kSMs * 16;
  unsigned blocks = (unsigned)(need < cap ? need : cap);
  if (blocks == 0) blocks = 1;
  kern<<<blocks, Q_WARPS * 32, smem, st>>>(m, gm, reinterpret_cast<const T*>(field), slots, pos, axes, q,
                                           mode == FIF_MODE_TRILINEAR, out);
  FIF_CHECK_LAUNCH("k_query");
  return FIF_OK;
}

template <typename T, int KIND>
static int dispatch_query(bool grad, bool metric, const fif_model& m, const QueryGeom& gm, const void* field,
                          const int32_t* slots, const double* pos, const double* axes, int64_t q, int mode,
                          const QueryOut& out, cudaStream_t st) {
  if (KIND == FIF_KIND_TRACE) {
    return grad ? launch_query<T, KIND, true, false>(m, gm, field, slots, pos, axes, q, mode, out, st)
                : launch_query<T, KIND, false, false>(m, gm, field, slots, pos, axes, q, mode, out, st);
  }
  if (metric)
    return grad ? launch_query<T, KIND, true, true>(m, gm, field, slots, pos, axes, q, mode, out, st)
                : launch_query<T, KIND, false, true>(m, gm, field, slots, pos, axes, q, mode, out, st);
  return grad ? launch_query<T, KIND, true, false>(m, gm, field, slots, pos, axes, q, mode, out, st)
              : launch_query<T, KIND, false, false>(m, gm, field, slots, pos, axes, q, mode, out, st);
}

}  // namespace fif

using namespace fif;

extern "C" int fif_query(int factor_kind, const fif_model* model, const fif_grid* grid, const void* d_field,
                         const int32_t* d_slots, const double* d_positions, const double* d_axes, int64_t q, int mode,
                         uint32_t flags, double* d_trace, double* d_trace_grad, double* d_fim, double* d_fim_grad,
                         double* d_det, double* d_lmin, uint8_t* d_status, void* stream) {
  FIF_CHECK_ARG(model && grid, "fif_query: NULL model/grid");
  FIF_CHECK_ARG(factor_kind == FIF_KIND_INFO || factor_kind == FIF_KIND_TRACE, "fif_query: bad factor_kind");
  FIF_CHECK_ARG(mode == FIF_MODE_NEAREST || mode == FIF_MODE_TRILINEAR, "fif_query: bad mode %d", mode);
  FIF_CHECK_ARG(q >= 0, "fif_query: q < 0");
  if (q == 0) return FIF_OK;
  FIF_CHECK_ARG(d_field && d_positions && d_axes, "fif_query: NULL field/positions/axes");
  FIF_CHECK_ARG(model->kind == FIF_MODEL_QUAD || (model->kind == FIF_MODEL_GP && model->zs && model->kinv),
                "fif_query: bad model");
  const bool info = factor_kind == FIF_KIND_INFO;
  FIF_CHECK_ARG(info || !(d_fim || d_fim_grad || d_det || d_lmin),
                "fif_query: full FIM / det / lmin need an info field (WrongFactorKind)");
  FIF_CHECK_ARG(grid->voxel_size > 0, "fif_query: voxel_size <= 0");
  QueryGeom gm{grid->origin[0], grid->origin[1], grid->origin[2], grid->voxel_size,
               grid->dims[0],   grid->dims[1],   grid->dims[2]};
  QueryOut out{(flags & FIF_Q_TRACE) ? d_trace : nullptr,
               (flags & FIF_Q_TRACE) && (flags & FIF_Q_GRAD) ? d_trace_grad : nullptr,
               (flags & FIF_Q_FULL) ? d_fim : nullptr,
               (flags & FIF_Q_FULL) && (flags & FIF_Q_GRAD) ? d_fim_grad : nullptr,
               (flags & FIF_Q_DET) ? d_det : nullptr,
               (flags & FIF_Q_LMIN) ? d_lmin : nullptr,
               d_status};
  const bool grad = (flags & FIF_Q_GRAD) && (out.trace_grad || out.fim_grad);
  const bool metric = info && (out.det || out.lmin);
  cudaStream_t st = (cudaStream_t)stream;
  const bool f64 = model->kind == FIF_MODEL_QUAD || (flags & FIF_Q_FIELD_F64);
  if (f64) {
    return info ? dispatch_query<double, FIF_KIND_INFO>(grad, metric, *model, gm, d_field, d_slots, d_positions,
                                                        d_axes, q, mode, out, st)
                : dispatch_query<double, FIF_KIND_TRACE>(grad, metric, *model, gm, d_field, d_slots, d_positions,
                                                         d_axes, q, mode, out, st);
  }
  return info ? dispatch_query<float, FIF_KIND_INFO>(grad, metric, *model, gm, d_field, d_slots, d_positions, d_axes,
                                                     q, mode, out, st)
              : dispatch_query<float, FIF_KIND_TRACE>(grad, metric, *model, gm, d_field, d_slots, d_positions,
                                                      d_axes, q, mode, out, st);
}
