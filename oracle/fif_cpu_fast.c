/* fif_cpu_fast.c — the reference's GP build algorithm as a reasonably fast CPU port,
 * used ONLY as bench.py's CPU baseline / reference arm (TEST INFRASTRUCTURE, like
 * fif_oracle.c; never part of the product path).
 *
 * Same algorithm as _nb_build_gp (kernels.py:471-524): per voxel and landmark the
 * sigmoid sample visibilities vs (kernels.py:506), vp = vs @ kinv (kernels.py:511)
 * and the per-landmark 6x6 FIM (kernels.py:363-424) accumulated as vp (x) I6
 * (kernels.py:519-523).  Where the reference hands the two products to BLAS over all
 * landmarks of a voxel, this port blocks the landmarks (FP_LB at a time) so both
 * products run as small cache-resident matrix products with vectorised (AVX2/FMA)
 * inner loops, and the sigmoid exponentials vectorised (glibc libmvec, hence
 * -ffast-math for this file only).  Results agree with fif_oracle.c's literal loops
 * to ~1e-13 (summation order, FMA contraction, vector exp); tests/test_host.py
 * checks that.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define FP_LB 64

/* kernels.py:363-424 — 36 entries row-major of the landmark's 6x6 block; returns the trace. */
static inline double fim_flat(double px, double py, double pz, double tx, double ty, double tz, double inv_s2,
                              double* out) {
  double dx = px - tx, dy = py - ty, dz = pz - tz;
  double n2 = dx * dx + dy * dy + dz * dz;
  double n = sqrt(n2);
  double ux = dx / n, uy = dy / n, uz = dz / n;
  double w = inv_s2 / n2;
  double c2x = py * uz - pz * uy, c2y = pz * ux - px * uz, c2z = px * uy - py * ux;
  double u[3] = {ux, uy, uz}, c2[3] = {c2x, c2y, c2z}, p[3] = {px, py, pz};
  double pp = px * px + py * py + pz * pz;
  /* S = skew(p) */
  double S[3][3] = {{0, -pz, py}, {pz, 0, -px}, {-py, px, 0}};
  double tr = 0.0;
  for (int r = 0; r < 3; ++r)
    for (int c = 0; c < 3; ++c) {
      double tl = w * ((r == c ? 1.0 : 0.0) - u[r] * u[c]);
      double trr = -w * (S[r][c] + u[r] * c2[c]);
      double br = w * ((r == c ? pp : 0.0) - p[r] * p[c] - c2[r] * c2[c]);
      out[r * 6 + c] = tl;
      out[r * 6 + 3 + c] = trr;
      out[(3 + c) * 6 + r] = trr;
      out[(3 + r) * 6 + 3 + c] = br;
      if (r == c) tr += tl + br;
    }
  return tr;
}

void fp_build_gp(const double* centers, int64_t nv, const double* points, int64_t npts, double sigma,
                 const double* zs, int ns, const double* kinv, double ks, double cos_alpha, int want_trace,
                 double* out, int nthreads) {
  const int64_t width = want_trace ? ns : (int64_t)ns * 36;
  const double inv_s2 = 1.0 / (sigma * sigma);
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif
#pragma omp parallel
  {
    double* vs = (double*)aligned_alloc(64, sizeof(double) * FP_LB * ns);
    double* vp = (double*)aligned_alloc(64, sizeof(double) * FP_LB * ns);
    double* blk = (double*)aligned_alloc(64, sizeof(double) * FP_LB * 36);
    double* trs = (double*)aligned_alloc(64, sizeof(double) * FP_LB);
#pragma omp for schedule(dynamic, 1)
    for (int64_t v = 0; v < nv; ++v) {
      double* o = out + v * width;
      memset(o, 0, sizeof(double) * width);
      const double cx = centers[3 * v], cy = centers[3 * v + 1], cz = centers[3 * v + 2];
      for (int64_t i0 = 0; i0 < npts; i0 += FP_LB) {
        int nb = 0;
        for (int64_t i = i0; i < npts && i < i0 + FP_LB; ++i) {
          const double px = points[3 * i], py = points[3 * i + 1], pz = points[3 * i + 2];
          const double dx = px - cx, dy = py - cy, dz = pz - cz;
          const double n2 = dx * dx + dy * dy + dz * dz;
          if (n2 < 1e-300) continue; /* kernels.py:494 */
          const double n = sqrt(n2);
          const double ux = dx / n, uy = dy / n, uz = dz / n;
          trs[nb] = fim_flat(px, py, pz, cx, cy, cz, inv_s2, blk + 36 * nb);
          double* s = vs + (int64_t)nb * ns;
#pragma omp simd
          for (int g = 0; g < ns; ++g) {
            const double c = ux * zs[3 * g] + uy * zs[3 * g + 1] + uz * zs[3 * g + 2];
            s[g] = 1.0 / (1.0 + exp(-ks * (c - cos_alpha)));
          }
          ++nb;
        }
        /* vp = vs @ kinv (nb x ns x ns) */
        for (int j = 0; j < nb; ++j) {
          double* pr = vp + (int64_t)j * ns;
          const double* sr = vs + (int64_t)j * ns;
          for (int k = 0; k < ns; ++k) pr[k] = 0.0;
          for (int g = 0; g < ns; ++g) {
            const double sg = sr[g];
            const double* kr = kinv + (int64_t)g * ns;
            for (int k = 0; k < ns; ++k) pr[k] += sg * kr[k];
          }
        }
        if (want_trace) {
          for (int j = 0; j < nb; ++j) {
            const double* pr = vp + (int64_t)j * ns;
            for (int k = 0; k < ns; ++k) o[k] += pr[k] * trs[j];
          }
        } else {
          /* o[k][e] += sum_j vp[j][k] blk[j][e] */
          for (int k = 0; k < ns; ++k) {
            double acc[36];
            for (int e = 0; e < 36; ++e) acc[e] = 0.0;
            for (int j = 0; j < nb; ++j) {
              const double vk = vp[(int64_t)j * ns + k];
              const double* b = blk + 36 * j;
              for (int e = 0; e < 36; ++e) acc[e] += vk * b[e];
            }
            double* ob = o + 36 * k;
            for (int e = 0; e < 36; ++e) ob[e] += acc[e];
          }
        }
      }
    }
    free(vs);
    free(vp);
    free(blk);
    free(trs);
  }
}
