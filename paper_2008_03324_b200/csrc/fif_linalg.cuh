// fif_linalg.cuh — 6x6 symmetric-matrix metrics in registers (det / lambda_min and
// their gradient helpers), shared by the field queries (fif_query.cu) and the
// point-cloud metric path (fif_pc.cu).  Replaces the LAPACK calls of
// _nb_metric_of (kernels.py:602-608): np.linalg.det (LU with partial pivoting) and
// np.linalg.eigvalsh(...)[0].
#pragma once
#include "fif_common.cuh"

namespace fif {

// 6x6 determinant (partial-pivot LU) and smallest eigenvalue (cyclic Jacobi), FP64.
// Every loop is fully unrolled with compile-time indices (row swaps and the pivot
// permutation as selects), so the matrices stay in registers instead of local memory.
// Arithmetic order is that of the straightforward loops (and of the oracle's).
__host__ __device__ constexpr int pack_r(int x) { return x < 6 ? 0 : x < 11 ? 1 : x < 15 ? 2 : x < 18 ? 3 : x < 20 ? 4 : 5; }
__host__ __device__ constexpr int pack_c(int x) { return pack_r(x) + x - (pack_r(x) * 6 - pack_r(x) * (pack_r(x) - 1) / 2); }

// LU with partial pivoting (rows swapped whole, multipliers kept below the diagonal so
// P A = L U); returns det, or 0 with ok = false for a singular matrix.  INV: F^-1.
template <bool INV>
__device__ __forceinline__ double det6_core(double (&a)[36], double (&inv)[36], bool& ok) {
  int perm[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) perm[i] = i;
  double det = 1.0;
  ok = false;
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    int p = c;
    double best = fabs(a[6 * c + c]);
#pragma unroll
    for (int r = c + 1; r < 6; ++r)
      if (fabs(a[6 * r + c]) > best) { best = fabs(a[6 * r + c]); p = r; }
    if (best == 0.0) return 0.0;
#pragma unroll
    for (int r = c + 1; r < 6; ++r) {
      const bool sw = p == r;
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        const double t = a[6 * c + k];
        a[6 * c + k] = sw ? a[6 * r + k] : t;
        a[6 * r + k] = sw ? t : a[6 * r + k];
      }
      if (INV) {
        const int tp = perm[c];
        perm[c] = sw ? perm[r] : tp;
        perm[r] = sw ? tp : perm[r];
      }
    }
    if (p != c) det = -det;
    const double piv = a[6 * c + c];
    det *= piv;
#pragma unroll
    for (int r = c + 1; r < 6; ++r) {
      const double f = a[6 * r + c] / piv;
#pragma unroll
      for (int k = c + 1; k < 6; ++k) a[6 * r + k] -= f * a[6 * c + k];
      if (INV) a[6 * r + c] = f;
    }
  }
  if (INV) {
    double rd[6];  // one division per pivot, then multiplies in the 6 back substitutions
#pragma unroll
    for (int i = 0; i < 6; ++i) rd[i] = 1.0 / a[6 * i + i];
#pragma unroll
    for (int j = 0; j < 6; ++j) {  // column j of A^-1: solve L U x = P e_j
      double x[6];
#pragma unroll
      for (int i = 0; i < 6; ++i) {
        double y = perm[i] == j ? 1.0 : 0.0;
#pragma unroll
        for (int k = 0; k < i; ++k) y -= a[6 * i + k] * x[k];
        x[i] = y;
      }
#pragma unroll
      for (int i = 5; i >= 0; --i) {
        double y = x[i];
#pragma unroll
        for (int k = i + 1; k < 6; ++k) y -= a[6 * i + k] * x[k];
        x[i] = y * rd[i];
      }
#pragma unroll
      for (int i = 0; i < 6; ++i) inv[6 * i + j] = x[i];
    }
  }
  ok = true;
  return det;
}

// cyclic Jacobi; VEC: accumulate the rotations and return the unit eigenvector of the
// smallest eigenvalue in vec
template <bool VEC>
__device__ __forceinline__ double lmin6_core(double (&a)[36], double (&vec)[6]) {
  double V[VEC ? 36 : 1];
  if (VEC) {
#pragma unroll
    for (int i = 0; i < (VEC ? 36 : 1); ++i) V[i] = (i % 7 == 0) ? 1.0 : 0.0;
  }
  for (int sweep = 0; sweep < 64; ++sweep) {
    double off = 0.0, tot = 0.0;
#pragma unroll
    for (int r = 0; r < 6; ++r)
#pragma unroll
      for (int c = 0; c < 6; ++c) {
        const double v = a[6 * r + c] * a[6 * r + c];
        tot += v;
        if (r != c) off += v;
      }
    if (off <= 1e-30 * tot || off == 0.0) break;
#pragma unroll
    for (int p = 0; p < 5; ++p)
#pragma unroll
      for (int q = p + 1; q < 6; ++q) {
        const double apq = a[6 * p + q];
        if (apq != 0.0) {
          const double theta = (a[6 * q + q] - a[6 * p + p]) / (2.0 * apq);
          const double t = (theta >= 0 ? 1.0 : -1.0) / (fabs(theta) + sqrt(theta * theta + 1.0));
          const double cs = rsqrt(fma(t, t, 1.0)), sn = t * cs;
#pragma unroll
          for (int k = 0; k < 6; ++k) {
            const double akp = a[6 * k + p], akq = a[6 * k + q];
            a[6 * k + p] = cs * akp - sn * akq;
            a[6 * k + q] = sn * akp + cs * akq;
            if (VEC) {
              const double vkp = V[6 * k + p], vkq = V[6 * k + q];
              V[6 * k + p] = cs * vkp - sn * vkq;
              V[6 * k + q] = sn * vkp + cs * vkq;
            }
          }
#pragma unroll
          for (int k = 0; k < 6; ++k) {
            const double apk = a[6 * p + k], aqk = a[6 * q + k];
            a[6 * p + k] = cs * apk - sn * aqk;
            a[6 * q + k] = sn * apk + cs * aqk;
          }
        }
      }
  }
  double m = a[0];
#pragma unroll
  for (int k = 1; k < 6; ++k) m = fmin(m, a[7 * k]);
  if (VEC) {
    double best = a[0];
    int im = 0;
#pragma unroll
    for (int k = 1; k < 6; ++k)
      if (a[7 * k] < best) { best = a[7 * k]; im = k; }
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      double v = V[6 * i];
#pragma unroll
      for (int k = 1; k < 6; ++k) v = im == k ? V[6 * i + k] : v;
      vec[i] = v;
    }
  }
  return m;
}

// unpack a corner's 21 packed entries into a symmetric 6x6 (registers)
__device__ __forceinline__ void unpack21(const double* cf, double (&a)[36]) {
#pragma unroll
  for (int x = 0; x < 21; ++x) {
    const double v = cf[x];
    a[pack_r(x) * 6 + pack_c(x)] = v;
    a[pack_c(x) * 6 + pack_r(x)] = v;
  }
}

}  // namespace fif
