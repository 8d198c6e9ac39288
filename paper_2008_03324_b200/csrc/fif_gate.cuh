// fif_gate.cuh — matchability gates (field.py:143-177, world.py:96-140) as a per-pair
// device predicate, shared by the mask kernel (fif_match.cu) and the build kernels
// (fif_build.cu), which evaluate it on the fly inside their pair loops so a masked build
// never materialises a (V, N) mask.
//
// Every operation is the reference's numpy FP64 arithmetic in numpy's own order (explicit
// round-to-nearest intrinsics, no FMA contraction unless numpy's BLAS fuses):
//   d = p - c;  dist = sqrt((dx*dx + dy*dy) + dz*dz)              np.linalg.norm(axis=2)
//   range: dist >= d_near, dist <= d_far                          field.py:153-158
//   cone:  u = d / max(dist, 1e-12); cos = (ux vx + uz vz) + uy vy field.py:159-165 (einsum)
//   occlusion (world.segment_blocked, start = c, end = p, seg = d, t_hi = 1 - 1e-6):
//     sphere: rel = c - s;  a = (sx sx + sz sz) + sy sy            einsum("ij,ij->i")
//             b = fma(2sz, rz, fma(2sx, rx, 2sy ry))               (2 seg) @ rel, OpenBLAS dgemv
//                 ((2sx rx + 2sy ry) + 2sz rz for a single landmark: numpy's own dot)
//             t = a > 0 ? clip(-b / (2 max(a, 1e-300)), 0, t_hi) : 0
//             blocked |= |c + t seg - s| < r - 1e-9
//     box:    lo + 1e-9, hi - 1e-9; slab test with inv = 1/seg (inf on flat axes, which use
//             the inside-the-slab rule), blocked |= enter < leave && leave > 0 && enter < t_hi
// The einsum / dgemv orders were measured against numpy 2.3 + its OpenBLAS in the
// authoring image (the GPU box runs the same image); tests/golden/match*.npz pin them.
#pragma once
#include "fif_common.cuh"

namespace fif {

struct PairGate {
  const uint8_t* mask;   // explicit (rows, n) mask, row = v - v0 (fif_build's d_mask), or NULL
  fif_match m;           // fused gates (flags FIF_MATCH_*) when mask == NULL
  const double* pts;     // (n,3) FP64 landmarks
  const double* vdir;    // (n,3) landmark view directions (cone)
  VoxSrc src;            // voxel centres (explicit array or grid), bit-exact FP64
  int64_t v0, n;
};

__device__ __forceinline__ double g_norm3(double x, double y, double z) {
  return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z)));
}

// np.minimum / np.maximum (NaN-propagating, unlike fmin / fmax)
__device__ __forceinline__ double np_min(double a, double b) { return (a != a || b != b) ? a + b : fmin(a, b); }
__device__ __forceinline__ double np_max(double a, double b) { return (a != a || b != b) ? a + b : fmax(a, b); }

// world.segment_blocked for one (start c, end p) pair
__device__ __forceinline__ bool g_blocked(const fif_match& m, double cx, double cy, double cz, double sx, double sy,
                                          double sz, bool single) {
  const double t_hi = 1.0 - 1e-6;
  for (int64_t k = 0; k < m.n_spheres; ++k) {
    const double* s = m.spheres + 4 * k;
    const double rx = __dsub_rn(cx, s[0]), ry = __dsub_rn(cy, s[1]), rz = __dsub_rn(cz, s[2]);
    const double a = __dadd_rn(__dadd_rn(__dmul_rn(sx, sx), __dmul_rn(sz, sz)), __dmul_rn(sy, sy));
    const double tx = 2.0 * sx, ty = 2.0 * sy, tz = 2.0 * sz;  // exact
    const double b = single ? __dadd_rn(__dadd_rn(__dmul_rn(tx, rx), __dmul_rn(ty, ry)), __dmul_rn(tz, rz))
                            : __fma_rn(tz, rz, __fma_rn(tx, rx, __dmul_rn(ty, ry)));
    double t = 0.0;
    if (a > 0) {
      t = __ddiv_rn(-b, 2.0 * fmax(a, 1e-300));
      t = fmin(fmax(t, 0.0), t_hi);
    }
    const double qx = __dsub_rn(__dadd_rn(cx, __dmul_rn(t, sx)), s[0]);
    const double qy = __dsub_rn(__dadd_rn(cy, __dmul_rn(t, sy)), s[1]);
    const double qz = __dsub_rn(__dadd_rn(cz, __dmul_rn(t, sz)), s[2]);
    if (g_norm3(qx, qy, qz) < __dsub_rn(s[3], 1e-9)) return true;
  }
  for (int64_t k = 0; k < m.n_boxes; ++k) {
    const double* bx = m.boxes + 6 * k;
    const double c3[3] = {cx, cy, cz}, s3[3] = {sx, sy, sz};
    double enter = -INFINITY, leave = INFINITY;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      const double lo = __dadd_rn(bx[ax], 1e-9), hi = __dsub_rn(bx[3 + ax], 1e-9);
      double tmin, tmax;
      if (s3[ax] != 0.0) {
        const double inv = __ddiv_rn(1.0, s3[ax]);
        const double t0 = __dmul_rn(__dsub_rn(lo, c3[ax]), inv), t1 = __dmul_rn(__dsub_rn(hi, c3[ax]), inv);
        tmin = np_min(t0, t1);
        tmax = np_max(t0, t1);
      } else {
        const bool inside = c3[ax] >= lo && c3[ax] <= hi;
        tmin = inside ? -INFINITY : INFINITY;
        tmax = inside ? INFINITY : -INFINITY;
      }
      enter = np_max(enter, tmin);
      leave = np_min(leave, tmax);
    }
    if (enter < leave && leave > 0.0 && enter < t_hi) return true;
  }
  return false;
}

// Matchability.mask for one (centre, landmark i) pair: true = the pair contributes.
__device__ __forceinline__ bool match_pair(const fif_match& m, double cx, double cy, double cz, const double* pts,
                                           const double* vdir, int64_t i, bool single) {
  const double dx = __dsub_rn(pts[3 * i], cx), dy = __dsub_rn(pts[3 * i + 1], cy), dz = __dsub_rn(pts[3 * i + 2], cz);
  if (m.flags & (FIF_MATCH_NEAR | FIF_MATCH_FAR | FIF_MATCH_CONE)) {
    const double dist = g_norm3(dx, dy, dz);
    if ((m.flags & FIF_MATCH_NEAR) && !(dist >= m.d_near)) return false;
    if ((m.flags & FIF_MATCH_FAR) && !(dist <= m.d_far)) return false;
    if (m.flags & FIF_MATCH_CONE) {
      const double safe = fmax(dist, 1e-12);
      const double ux = __ddiv_rn(dx, safe), uy = __ddiv_rn(dy, safe), uz = __ddiv_rn(dz, safe);
      const double c = __dadd_rn(__dadd_rn(__dmul_rn(ux, vdir[3 * i]), __dmul_rn(uz, vdir[3 * i + 2])),
                                 __dmul_rn(uy, vdir[3 * i + 1]));
      if (!(c >= m.cos_beta)) return false;
    }
  }
  if ((m.flags & FIF_MATCH_OCCLUDE) && g_blocked(m, cx, cy, cz, dx, dy, dz, single)) return false;
  return true;
}

// The build kernels' per-pair test: landmark i against voxel v (global index in [v0, v1)).
__device__ __forceinline__ bool gate_keep(const PairGate& g, int64_t v, int64_t i) {
  if (g.mask) return g.mask[(v - g.v0) * g.n + i] != 0;
  double cx, cy, cz;
  voxel_center(g.src, v, cx, cy, cz);
  return match_pair(g.m, cx, cy, cz, g.pts, g.vdir, i, g.n == 1);
}

}  // namespace fif
