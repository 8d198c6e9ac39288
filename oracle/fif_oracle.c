/*
 * fif_oracle.c — CPU restatement of the reference FIF hot paths (TEST INFRASTRUCTURE).
 *
 * This file is the CHECKER for the CUDA product path, never the product: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load it.  It restates, in plain C with IEEE binary64 arithmetic and
 * no FMA contraction (compile with -ffp-contract=off), the numba kernels of the
 * reference package `fifield` 0.1.0 (/root/reference/pkg/src/fifield/kernels.py):
 *
 *   or_fim_flat        <- _nb_fim_flat_into        kernels.py:363-424
 *   or_build_quad      <- _nb_build_quad(_par)     kernels.py:427-468, 527-568
 *   or_build_gp        <- _nb_build_gp             kernels.py:471-524
 *   or_exact_fim       <- _nb_exact_fim            kernels.py:571-599
 *   or_pc_mask         <- visibility test inside _nb_exact_fim (kernels.py:580-595)
 *   or_locate_nearest  <- _nb_locate_nearest       kernels.py:628-635
 *   or_trilinear       <- corner logic in _nb_query_fim / _nb_query_metric
 *                         kernels.py:679-719, 1432-1468
 *   or_query_fim_batch <- _nb_query_fim_batch_*    kernels.py:752-777 (+ _nb_query_fim 674-726)
 *   or_metric_batch    <- _nb_field_metric_batch_* kernels.py:1493-1522 (+ _nb_query_metric
 *                         1429-1472, _nb_metric_one 1405-1426, _nb_metric_of 602-608)
 *   or_centers         <- GridConfig.centers       field.py:74-79
 *
 * Operation order follows the reference line by line (left-to-right sums,
 * mul-then-add, IEEE division), so the non-BLAS paths are bit-identical to the
 * numba reference; the GP build replaces the reference's BLAS np.dot calls
 * (kernels.py:505,511,519) by landmark-ordered loops, which changes only the
 * summation order (~1e-15 relative).  det / lmin use a partial-pivot LU and a
 * cyclic Jacobi eigen-solver in place of LAPACK (kernels.py:604-607).
 * Pinned against the tests/golden npz fixtures (generated from the reference itself).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define STATUS_OK 0
#define STATUS_OUT_OF_FIELD 1

static void set_threads(int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
}

int or_openmp_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* field.py:74-79 — origin + (idx + 0.5) * voxel_size, x-major / z-minor order. */
void or_centers(const double* origin, double vs, const int64_t* dims, double* out) {
  int64_t nx = dims[0], ny = dims[1], nz = dims[2], r = 0;
  for (int64_t ix = 0; ix < nx; ++ix)
    for (int64_t iy = 0; iy < ny; ++iy)
      for (int64_t iz = 0; iz < nz; ++iz, ++r) {
        out[3 * r + 0] = origin[0] + ((double)ix + 0.5) * vs;
        out[3 * r + 1] = origin[1] + ((double)iy + 0.5) * vs;
        out[3 * r + 2] = origin[2] + ((double)iz + 0.5) * vs;
      }
}

/* kernels.py:363-424.  Returns the block trace (sum of the six diagonal entries). */
double or_fim_flat(double px, double py, double pz, double tx, double ty, double tz, double inv_s2,
                   double* out) {
  double dx = px - tx, dy = py - ty, dz = pz - tz;
  double n2 = dx * dx + dy * dy + dz * dz;
  if (n2 < 1e-300) {
    for (int k = 0; k < 36; ++k) out[k] = 0.0;
    return 0.0;
  }
  double n = sqrt(n2);
  double ux = dx / n, uy = dy / n, uz = dz / n;
  double w = inv_s2 / n2;
  double c2x = py * uz - pz * uy;
  double c2y = pz * ux - px * uz;
  double c2z = px * uy - py * ux;
  double pp = px * px + py * py + pz * pz;
  out[0] = w * (1.0 - ux * ux);
  out[1] = w * (-ux * uy);
  out[2] = w * (-ux * uz);
  out[6] = out[1];
  out[7] = w * (1.0 - uy * uy);
  out[8] = w * (-uy * uz);
  out[12] = out[2];
  out[13] = out[8];
  out[14] = w * (1.0 - uz * uz);
  out[3] = -w * (ux * c2x);
  out[4] = -w * (-pz + ux * c2y);
  out[5] = -w * (py + ux * c2z);
  out[9] = -w * (pz + uy * c2x);
  out[10] = -w * (uy * c2y);
  out[11] = -w * (-px + uy * c2z);
  out[15] = -w * (-py + uz * c2x);
  out[16] = -w * (px + uz * c2y);
  out[17] = -w * (uz * c2z);
  out[18] = out[3];
  out[19] = out[9];
  out[20] = out[15];
  out[24] = out[4];
  out[25] = out[10];
  out[26] = out[16];
  out[30] = out[5];
  out[31] = out[11];
  out[32] = out[17];
  out[21] = w * (pp - px * px - c2x * c2x);
  out[22] = w * (-px * py - c2x * c2y);
  out[23] = w * (-px * pz - c2x * c2z);
  out[27] = out[22];
  out[28] = w * (pp - py * py - c2y * c2y);
  out[29] = w * (-py * pz - c2y * c2z);
  out[33] = out[23];
  out[34] = out[29];
  out[35] = w * (-pz * pz + pp - c2z * c2z);
  return out[0] + out[7] + out[14] + out[21] + out[28] + out[35];
}

/* kernels.py:427-468 (serial) / 527-568 (prange over voxels; identical arithmetic). */
void or_build_quad(const double* centers, int64_t nv, const double* points, int64_t npts, double sigma,
                   double k2, double k1, double k0, int want_trace, const uint8_t* mask, double* out,
                   int nthreads) {
  (void)k2; (void)k1; (void)k0;  /* the position vector does not depend on the coefficients */
  int64_t width = want_trace ? 10 : 360;
  double inv_s2 = 1.0 / (sigma * sigma);
  set_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t v = 0; v < nv; ++v) {
    double blk[36], vp[10];
    double* o = out + v * width;
    for (int64_t k = 0; k < width; ++k) o[k] = 0.0;
    double cx = centers[3 * v], cy = centers[3 * v + 1], cz = centers[3 * v + 2];
    for (int64_t i = 0; i < npts; ++i) {
      if (mask && mask[v * npts + i] == 0) continue;
      double px = points[3 * i], py = points[3 * i + 1], pz = points[3 * i + 2];
      double dx = px - cx, dy = py - cy, dz = pz - cz;
      double n2 = dx * dx + dy * dy + dz * dz;
      if (n2 < 1e-300) continue;
      double n = sqrt(n2);
      double ux = dx / n, uy = dy / n, uz = dz / n;
      vp[0] = ux * ux; vp[1] = uy * uy; vp[2] = uz * uz;
      vp[3] = ux * uy; vp[4] = ux * uz; vp[5] = uy * uz;
      vp[6] = ux; vp[7] = uy; vp[8] = uz; vp[9] = 1.0;
      double tr = or_fim_flat(px, py, pz, cx, cy, cz, inv_s2, blk);
      if (want_trace) {
        for (int k = 0; k < 10; ++k) o[k] += vp[k] * tr;
      } else {
        for (int k = 0; k < 10; ++k) {
          double vk = vp[k];
          double* ob = o + 36 * k;
          for (int e = 0; e < 36; ++e) ob[e] += vk * blk[e];
        }
      }
    }
  }
}

/* kernels.py:471-524.  Per voxel: u, keep, i6, tr for every landmark; cang = u zs^T;
 * vs = sigmoid(ks (cang - cos_alpha)) with skipped rows zeroed; vp = vs kinv;
 * trace: out[k] = sum_i vp[i,k] tr_i; info: out[k,e] = sum_i vp[i,k] i6[i,e].
 * The reference's BLAS products are evaluated here landmark by landmark.        */
void or_build_gp(const double* centers, int64_t nv, const double* points, int64_t npts, double sigma,
                 const double* zs, int ns, const double* kinv, double ks, double cos_alpha, int want_trace,
                 const uint8_t* mask, double* out, int nthreads) {
  int64_t width = want_trace ? ns : (int64_t)ns * 36;
  double inv_s2 = 1.0 / (sigma * sigma);
  set_threads(nthreads);
#pragma omp parallel
  {
    double* vs = (double*)malloc(sizeof(double) * ns);
    double* vp = (double*)malloc(sizeof(double) * ns);
#pragma omp for schedule(dynamic, 1)
    for (int64_t v = 0; v < nv; ++v) {
      double blk[36];
      double* o = out + v * width;
      for (int64_t k = 0; k < width; ++k) o[k] = 0.0;
      double cx = centers[3 * v], cy = centers[3 * v + 1], cz = centers[3 * v + 2];
      for (int64_t i = 0; i < npts; ++i) {
        if (mask && mask[v * npts + i] == 0) continue;  /* zero vs row: no contribution */
        double px = points[3 * i], py = points[3 * i + 1], pz = points[3 * i + 2];
        double dx = px - cx, dy = py - cy, dz = pz - cz;
        double n2 = dx * dx + dy * dy + dz * dz;
        if (n2 < 1e-300) continue;
        double n = sqrt(n2);
        double ux = dx / n, uy = dy / n, uz = dz / n;
        double tr = or_fim_flat(px, py, pz, cx, cy, cz, inv_s2, blk);
        for (int g = 0; g < ns; ++g) {
          double c = ux * zs[3 * g] + uy * zs[3 * g + 1] + uz * zs[3 * g + 2];
          vs[g] = 1.0 / (1.0 + exp(-ks * (c - cos_alpha)));
        }
        for (int k = 0; k < ns; ++k) vp[k] = 0.0;
        for (int g = 0; g < ns; ++g) {
          double s = vs[g];
          const double* kr = kinv + (int64_t)g * ns;
          for (int k = 0; k < ns; ++k) vp[k] += s * kr[k];
        }
        if (want_trace) {
          for (int k = 0; k < ns; ++k) o[k] += vp[k] * tr;
        } else {
          for (int k = 0; k < ns; ++k) {
            double vk = vp[k];
            double* ob = o + 36 * k;
            for (int e = 0; e < 36; ++e) ob[e] += vk * blk[e];
          }
        }
      }
    }
    free(vs);
    free(vp);
  }
}

/* The exact pinhole visibility test of kernels.py:580-595, same operation order. */
static inline int pc_visible(const double* rot, double tx, double ty, double tz, double px, double py,
                             double pz, double fx, double fy, double cx, double cy, double width,
                             double height) {
  double r00 = rot[0], r10 = rot[3], r20 = rot[6];
  double r01 = rot[1], r11 = rot[4], r21 = rot[7];
  double r02 = rot[2], r12 = rot[5], r22 = rot[8];
  double dx = px - tx, dy = py - ty, dz = pz - tz;
  double zc = r02 * dx + r12 * dy + r22 * dz;
  if (zc <= 0.0) return 0;
  double xc = r00 * dx + r10 * dy + r20 * dz;
  double yc = r01 * dx + r11 * dy + r21 * dz;
  double u_px = fx * xc / zc + cx;
  if (u_px < 0.0 || u_px >= width) return 0;
  double v_px = fy * yc / zc + cy;
  if (v_px < 0.0 || v_px >= height) return 0;
  return 1;
}

/* kernels.py:571-599 batched (743-749): out (Q,36). */
void or_exact_fim_batch(const double* rots, const double* ts, int64_t q, const double* points, int64_t npts,
                        double fx, double fy, double cx, double cy, double width, double height, double sigma,
                        double* out, int nthreads) {
  double inv_s2 = 1.0 / (sigma * sigma);
  set_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t j = 0; j < q; ++j) {
    double blk[36];
    double* fim = out + 36 * j;
    for (int e = 0; e < 36; ++e) fim[e] = 0.0;
    const double* rot = rots + 9 * j;
    double tx = ts[3 * j], ty = ts[3 * j + 1], tz = ts[3 * j + 2];
    for (int64_t i = 0; i < npts; ++i) {
      double px = points[3 * i], py = points[3 * i + 1], pz = points[3 * i + 2];
      if (!pc_visible(rot, tx, ty, tz, px, py, pz, fx, fy, cx, cy, width, height)) continue;
      or_fim_flat(px, py, pz, tx, ty, tz, inv_s2, blk);
      for (int e = 0; e < 36; ++e) fim[e] += blk[e];
    }
  }
}

/* Visibility mask (Q, N) u8 with the reference's exact test. */
void or_pc_mask(const double* rots, const double* ts, int64_t q, const double* points, int64_t npts, double fx,
                double fy, double cx, double cy, double width, double height, uint8_t* out, int nthreads) {
  set_threads(nthreads);
#pragma omp parallel for schedule(static)
  for (int64_t j = 0; j < q; ++j)
    for (int64_t i = 0; i < npts; ++i)
      out[j * npts + i] = (uint8_t)pc_visible(rots + 9 * j, ts[3 * j], ts[3 * j + 1], ts[3 * j + 2],
                                              points[3 * i], points[3 * i + 1], points[3 * i + 2], fx, fy, cx,
                                              cy, width, height);
}

/* kernels.py:628-635 */
int64_t or_locate_nearest(const double* origin, double vs, const int64_t* dims, const double* pos) {
  int64_t ix = (int64_t)floor((pos[0] - origin[0]) / vs);
  int64_t iy = (int64_t)floor((pos[1] - origin[1]) / vs);
  int64_t iz = (int64_t)floor((pos[2] - origin[2]) / vs);
  if (ix < 0 || iy < 0 || iz < 0 || ix >= dims[0] || iy >= dims[1] || iz >= dims[2]) return -1;
  return (ix * dims[1] + iy) * dims[2] + iz;
}

/* kernels.py:679-719: base corner, weights in (dx,dy,dz) order; returns status. */
int or_trilinear(const double* origin, double vs, const int64_t* dims, const double* pos, int64_t* idx,
                 double* wts) {
  double gx = (pos[0] - origin[0]) / vs - 0.5;
  double gy = (pos[1] - origin[1]) / vs - 0.5;
  double gz = (pos[2] - origin[2]) / vs - 0.5;
  int64_t bx = (int64_t)floor(gx), by = (int64_t)floor(gy), bz = (int64_t)floor(gz);
  double fxw = gx - (double)bx, fyw = gy - (double)by, fzw = gz - (double)bz;
  if (bx + 1 == dims[0] && fxw == 0.0) { bx -= 1; fxw = 1.0; }
  if (by + 1 == dims[1] && fyw == 0.0) { by -= 1; fyw = 1.0; }
  if (bz + 1 == dims[2] && fzw == 0.0) { bz -= 1; fzw = 1.0; }
  if (bx < 0 || by < 0 || bz < 0 || bx + 1 >= dims[0] || by + 1 >= dims[1] || bz + 1 >= dims[2])
    return STATUS_OUT_OF_FIELD;
  int k = 0;
  for (int dx = 0; dx < 2; ++dx) {
    double wx = dx == 1 ? fxw : 1.0 - fxw;
    for (int dy = 0; dy < 2; ++dy) {
      double wy = dy == 1 ? fyw : 1.0 - fyw;
      for (int dz = 0; dz < 2; ++dz, ++k) {
        double wz = dz == 1 ? fzw : 1.0 - fzw;
        wts[k] = wx * wy * wz;
        idx[k] = ((bx + dx) * dims[1] + (by + dy)) * dims[2] + (bz + dz);
      }
    }
  }
  return STATUS_OK;
}

/* kernels.py:638-657 */
static void quad_vr(double zx, double zy, double zz, double k2, double k1, double k0, double* vr) {
  vr[0] = k2 * zx * zx; vr[1] = k2 * zy * zy; vr[2] = k2 * zz * zz;
  vr[3] = 2.0 * k2 * zx * zy; vr[4] = 2.0 * k2 * zx * zz; vr[5] = 2.0 * k2 * zy * zz;
  vr[6] = k1 * zx; vr[7] = k1 * zy; vr[8] = k1 * zz; vr[9] = k0;
}
static void gp_vr(double zx, double zy, double zz, const double* zs, int ns, double sig2, double ell, double* vr) {
  double inv_l2 = 1.0 / (ell * ell);
  for (int g = 0; g < ns; ++g) {
    double c = zx * zs[3 * g] + zy * zs[3 * g + 1] + zz * zs[3 * g + 2];
    vr[g] = sig2 * exp((c - 1.0) * inv_l2);
  }
}

/* kernels.py:660-671 */
static void contract(const double* row, const double* vr, int nvr, double* fim) {
  for (int e = 0; e < 36; ++e) fim[e] = 0.0;
  for (int k = 0; k < nvr; ++k) {
    double vk = vr[k];
    if (vk == 0.0) continue;
    const double* b = row + 36 * k;
    for (int e = 0; e < 36; ++e) fim[e] += vk * b[e];
  }
}

/* kernels.py:674-726 */
static int query_fim_one(const int32_t* slots, const double* factors, int64_t width, const double* origin,
                         double vs, const int64_t* dims, const double* pos, const double* vr, int nvr,
                         int trilinear, double* fim) {
  double work[36];
  for (int e = 0; e < 36; ++e) fim[e] = 0.0;
  if (trilinear) {
    int64_t idx[8];
    double wts[8];
    if (or_trilinear(origin, vs, dims, pos, idx, wts) != STATUS_OK) return STATUS_OUT_OF_FIELD;
    for (int j = 0; j < 8; ++j) {
      double wgt = wts[j];
      if (wgt == 0.0) continue;
      int32_t row = slots[idx[j]];
      if (row < 0) continue;
      contract(factors + (int64_t)row * width, vr, nvr, work);
      for (int e = 0; e < 36; ++e) fim[e] += wgt * work[e];
    }
    return STATUS_OK;
  }
  int64_t lin = or_locate_nearest(origin, vs, dims, pos);
  if (lin < 0) return STATUS_OUT_OF_FIELD;
  int32_t row = slots[lin];
  if (row >= 0) contract(factors + (int64_t)row * width, vr, nvr, fim);
  return STATUS_OK;
}

/* model: 1 = quad (params k2,k1,k0), 2 = gp (zs, ns, sig2, ell).  kernels.py:752-777 */
void or_query_fim_batch(const int32_t* slots, const double* factors, int64_t width, const double* origin,
                        double vs, const int64_t* dims, const double* positions, const double* axes, int64_t q,
                        int model, double k2, double k1, double k0, const double* zs, int ns, double sig2,
                        double ell, int trilinear, double* out, int64_t* status, int nthreads) {
  set_threads(nthreads);
#pragma omp parallel
  {
    int nvr = model == 1 ? 10 : ns;
    double* vr = (double*)malloc(sizeof(double) * (size_t)nvr);
#pragma omp for schedule(static)
    for (int64_t i = 0; i < q; ++i) {
      const double* z = axes + 3 * i;
      if (model == 1) quad_vr(z[0], z[1], z[2], k2, k1, k0, vr);
      else gp_vr(z[0], z[1], z[2], zs, ns, sig2, ell, vr);
      status[i] = query_fim_one(slots, factors, width, origin, vs, dims, positions + 3 * i, vr, nvr, trilinear,
                                out + 36 * i);
    }
    free(vr);
  }
}

/* 6x6 determinant: LU with partial pivoting (the LAPACK getrf recipe). */
static double det6(const double* a_in) {
  double a[36];
  memcpy(a, a_in, sizeof(a));
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

/* Smallest eigenvalue of a symmetric 6x6: cyclic Jacobi sweeps. */
static double lmin6(const double* a_in) {
  double a[36];
  for (int r = 0; r < 6; ++r)
    for (int c = 0; c < 6; ++c) a[6 * r + c] = 0.5 * (a_in[6 * r + c] + a_in[6 * c + r]);
  for (int sweep = 0; sweep < 64; ++sweep) {
    double off = 0.0, tot = 0.0;
    for (int r = 0; r < 6; ++r)
      for (int c = 0; c < 6; ++c) {
        tot += a[6 * r + c] * a[6 * r + c];
        if (r != c) off += a[6 * r + c] * a[6 * r + c];
      }
    if (off <= 1e-30 * tot || off == 0.0) break;
    for (int p = 0; p < 5; ++p)
      for (int qq = p + 1; qq < 6; ++qq) {
        double apq = a[6 * p + qq];
        if (apq == 0.0) continue;
        double app = a[6 * p + p], aqq = a[6 * qq + qq];
        double theta = (aqq - app) / (2.0 * apq);
        double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
        double cs = 1.0 / sqrt(t * t + 1.0), sn = t * cs;
        for (int k = 0; k < 6; ++k) {
          double akp = a[6 * k + p], akq = a[6 * k + qq];
          a[6 * k + p] = cs * akp - sn * akq;
          a[6 * k + qq] = sn * akp + cs * akq;
        }
        for (int k = 0; k < 6; ++k) {
          double apk = a[6 * p + k], aqk = a[6 * qq + k];
          a[6 * p + k] = cs * apk - sn * aqk;
          a[6 * qq + k] = sn * apk + cs * aqk;
        }
      }
  }
  double m = a[0];
  for (int k = 1; k < 6; ++k) if (a[7 * k] < m) m = a[7 * k];
  return m;
}

/* kernels.py:602-608 */
double or_metric_of(const double* fim, int mid) {
  if (mid == 0) return det6(fim);
  if (mid == 1) return lmin6(fim);
  return fim[0] + fim[7] + fim[14] + fim[21] + fim[28] + fim[35];
}

/* kernels.py:1405-1426 */
static double metric_one(const double* factors, int64_t width, int32_t row, const double* vr, int nvr, int mid,
                         int is_trace) {
  if (row < 0) return 0.0;
  const double* f = factors + (int64_t)row * width;
  if (is_trace) {
    double val = 0.0;
    for (int k = 0; k < nvr; ++k) val += vr[k] * f[k];
    return val;
  }
  if (mid == 2) {
    double val = 0.0;
    for (int k = 0; k < nvr; ++k) {
      int b = 36 * k;
      val += vr[k] * (f[b] + f[b + 7] + f[b + 14] + f[b + 21] + f[b + 28] + f[b + 35]);
    }
    return val;
  }
  double work[36];
  contract(f, vr, nvr, work);
  return or_metric_of(work, mid);
}

/* kernels.py:1493-1522 with _nb_query_metric 1429-1472 */
void or_metric_batch(const int32_t* slots, const double* factors, int64_t width, const double* origin, double vs,
                     const int64_t* dims, const double* positions, const double* axes, int64_t q, int model,
                     double k2, double k1, double k0, const double* zs, int ns, double sig2, double ell, int mid,
                     int is_trace, int trilinear, double* vals, int64_t* status, int nthreads) {
  set_threads(nthreads);
#pragma omp parallel
  {
    int nvr = model == 1 ? 10 : ns;
    double* vr = (double*)malloc(sizeof(double) * (size_t)nvr);
#pragma omp for schedule(static)
    for (int64_t i = 0; i < q; ++i) {
      const double* z = axes + 3 * i;
      const double* pos = positions + 3 * i;
      if (model == 1) quad_vr(z[0], z[1], z[2], k2, k1, k0, vr);
      else gp_vr(z[0], z[1], z[2], zs, ns, sig2, ell, vr);
      if (trilinear) {
        int64_t idx[8];
        double wts[8];
        if (or_trilinear(origin, vs, dims, pos, idx, wts) != STATUS_OK) {
          vals[i] = 0.0;
          status[i] = STATUS_OUT_OF_FIELD;
          continue;
        }
        double val = 0.0;
        for (int j = 0; j < 8; ++j) {
          if (wts[j] == 0.0) continue;
          val += wts[j] * metric_one(factors, width, slots[idx[j]], vr, nvr, mid, is_trace);
        }
        vals[i] = val;
        status[i] = STATUS_OK;
      } else {
        int64_t lin = or_locate_nearest(origin, vs, dims, pos);
        if (lin < 0) {
          vals[i] = 0.0;
          status[i] = STATUS_OUT_OF_FIELD;
          continue;
        }
        vals[i] = metric_one(factors, width, slots[lin], vr, nvr, mid, is_trace);
        status[i] = STATUS_OK;
      }
    }
    free(vr);
  }
}
