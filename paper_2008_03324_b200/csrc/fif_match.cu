// fif_match.cu — matchability gates on the GPU, sm_100a.
//
// Replaces the range and view-cone parts of Matchability.mask (field.py:143-165),
// which the reference evaluates with (V, N, 3) float64 numpy temporaries.  Per
// (voxel centre c, landmark p), FP64 with the reference's numpy arithmetic:
//   d = p - c;  dist = sqrt((dx*dx + dy*dy) + dz*dz)        (np.linalg.norm, axis=2)
//   range:  dist >= d_near,  dist <= d_far                    (field.py:153-158)
//   cone:   u = d / max(dist, 1e-12);
//           cos = (ux*vx + uz*vz) + uy*vy >= cos_beta          (field.py:159-165; the
//           order numpy 2.3's einsum("vnk,nk->vn") uses, measured bit-exactly)
// No FMA contraction (explicit __d*_rn intrinsics), so the mask is bit-identical.
// Layout: one CTA row-strip per voxel, 4 landmarks per thread, uchar4 stores.
#include "fif_common.cuh"

namespace fif {

constexpr int MM_THREADS = 256;
constexpr int MM_PER_T = 4;

template <bool NEAR, bool FAR, bool CONE>
__global__ void __launch_bounds__(MM_THREADS) k_match_mask(fif_match m, const double* __restrict__ centers,
                                                           int64_t rows, const double* __restrict__ pts,
                                                           const double* __restrict__ vdir, int64_t n,
                                                           uint8_t* __restrict__ mask) {
  const int64_t i0 = (blockIdx.x * (int64_t)MM_THREADS + threadIdx.x) * MM_PER_T;
  if (i0 >= n) return;
  for (int64_t r = blockIdx.y; r < rows; r += gridDim.y) {
    const double cx = centers[3 * r], cy = centers[3 * r + 1], cz = centers[3 * r + 2];
    uint8_t ok[MM_PER_T];
#pragma unroll
    for (int j = 0; j < MM_PER_T; ++j) {
      const int64_t i = i0 + j;
      ok[j] = 0;
      if (i >= n) continue;
      const double dx = __dsub_rn(pts[3 * i], cx), dy = __dsub_rn(pts[3 * i + 1], cy),
                   dz = __dsub_rn(pts[3 * i + 2], cz);
      const double dist =
          __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz)));
      bool a = true;
      if (NEAR) a = a && dist >= m.d_near;
      if (FAR) a = a && dist <= m.d_far;
      if (CONE) {
        const double safe = fmax(dist, 1e-12);
        const double ux = __ddiv_rn(dx, safe), uy = __ddiv_rn(dy, safe), uz = __ddiv_rn(dz, safe);
        const double c = __dadd_rn(__dadd_rn(__dmul_rn(ux, vdir[3 * i]), __dmul_rn(uz, vdir[3 * i + 2])),
                                   __dmul_rn(uy, vdir[3 * i + 1]));
        a = a && c >= m.cos_beta;
      }
      ok[j] = a ? 1 : 0;
    }
    uint8_t* o = mask + r * n + i0;
    if (i0 + MM_PER_T <= n && ((reinterpret_cast<uintptr_t>(o) & 3) == 0)) {
      *reinterpret_cast<uchar4*>(o) = make_uchar4(ok[0], ok[1], ok[2], ok[3]);
    } else {
      for (int j = 0; j < MM_PER_T && i0 + j < n; ++j) o[j] = ok[j];
    }
  }
}

}  // namespace fif

using namespace fif;

extern "C" int fif_match_mask(const fif_match* m, const double* d_centers, int64_t rows, const double* d_points,
                              const double* d_view_dirs, int64_t n_points, uint8_t* d_mask, void* stream) {
  FIF_CHECK_ARG(m, "fif_match_mask: NULL match");
  FIF_CHECK_ARG(rows >= 0 && n_points >= 0, "fif_match_mask: negative size");
  if (rows == 0 || n_points == 0) return FIF_OK;
  FIF_CHECK_ARG(d_centers && d_points && d_mask, "fif_match_mask: NULL centers/points/mask");
  const bool cone = (m->flags & FIF_MATCH_CONE) != 0;
  FIF_CHECK_ARG(!cone || d_view_dirs, "fif_match_mask: view cone requires landmark view directions");
  const unsigned bx = (unsigned)((n_points + MM_THREADS * MM_PER_T - 1) / (MM_THREADS * MM_PER_T));
  const unsigned by = (unsigned)(rows < 65535 ? rows : 65535);
  const dim3 grid(bx, by);
  cudaStream_t st = (cudaStream_t)stream;
  const int sel = (m->flags & 7u);
#define MM(N, F, C) k_match_mask<N, F, C><<<grid, MM_THREADS, 0, st>>>(*m, d_centers, rows, d_points, d_view_dirs, n_points, d_mask)
  switch (sel) {
    case 0: MM(false, false, false); break;
    case 1: MM(true, false, false); break;
    case 2: MM(false, true, false); break;
    case 3: MM(true, true, false); break;
    case 4: MM(false, false, true); break;
    case 5: MM(true, false, true); break;
    case 6: MM(false, true, true); break;
    default: MM(true, true, true); break;
  }
#undef MM
  FIF_CHECK_LAUNCH("k_match_mask");
  return FIF_OK;
}
