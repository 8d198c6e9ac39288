// fif_match.cu — matchability gates on the GPU, sm_100a.
//
// Replaces Matchability.mask (field.py:143-177): range, view cone and ObstacleWorld
// occlusion (world.segment_blocked, world.py:96-140), which the reference evaluates with
// (V, N, 3) float64 numpy temporaries and a per-voxel Python loop.  The per-pair predicate
// (fif_gate.cuh match_pair) is the reference's numpy FP64 arithmetic in numpy's order, so
// the masks are bit-identical.  k_match_mask materialises a (rows, N) mask (parity aid and
// the Python-predicate path); builds evaluate the same predicate inside their pair loops
// (fif_build_matched) and only need the per-voxel occupancy of k_match_any.
#include "fif_gate.cuh"

namespace fif {

constexpr int MM_THREADS = 256;
constexpr int MM_PER_T = 4;

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
      ok[j] = (i < n && match_pair(m, cx, cy, cz, pts, vdir, i, n == 1)) ? 1 : 0;
    }
    uint8_t* o = mask + r * n + i0;
    if (i0 + MM_PER_T <= n && ((reinterpret_cast<uintptr_t>(o) & 3) == 0)) {
      *reinterpret_cast<uchar4*>(o) = make_uchar4(ok[0], ok[1], ok[2], ok[3]);
    } else {
      for (int j = 0; j < MM_PER_T && i0 + j < n; ++j) o[j] = ok[j];
    }
  }
}

// Occupancy of each centre under the gates (field.py:255-257: a voxel gets a row iff some
// landmark matches): one CTA per centre, early exit once any landmark passes.
__global__ void __launch_bounds__(MM_THREADS) k_match_any(fif_match m, const double* __restrict__ centers,
                                                          int64_t rows, const double* __restrict__ pts,
                                                          const double* __restrict__ vdir, int64_t n,
                                                          uint8_t* __restrict__ any) {
  __shared__ int found;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const double cx = centers[3 * r], cy = centers[3 * r + 1], cz = centers[3 * r + 2];
    if (threadIdx.x == 0) found = 0;
    __syncthreads();
    for (int64_t b = 0; b < n; b += MM_THREADS * 8) {
      bool hit = false;
      for (int64_t i = b + threadIdx.x; i < n && i < b + MM_THREADS * 8 && !hit; i += MM_THREADS)
        hit = match_pair(m, cx, cy, cz, pts, vdir, i, n == 1);
      if (hit) found = 1;
      __syncthreads();
      const int f = found;
      __syncthreads();
      if (f) break;
    }
    if (threadIdx.x == 0) any[r] = (uint8_t)found;
    __syncthreads();
  }
}

}  // namespace fif

using namespace fif;

static int check_match(const fif_match* m, const double* d_view_dirs) {
  FIF_CHECK_ARG(m, "fif_match: NULL match");
  FIF_CHECK_ARG(!(m->flags & FIF_MATCH_CONE) || d_view_dirs, "fif_match: view cone requires landmark view directions");
  FIF_CHECK_ARG(!(m->flags & FIF_MATCH_OCCLUDE) ||
                    ((m->n_spheres == 0 || m->spheres) && (m->n_boxes == 0 || m->boxes) && m->n_spheres >= 0 &&
                     m->n_boxes >= 0),
                "fif_match: occlusion needs the sphere / box arrays");
  return FIF_OK;
}

extern "C" int fif_match_mask(const fif_match* m, const double* d_centers, int64_t rows, const double* d_points,
                              const double* d_view_dirs, int64_t n_points, uint8_t* d_mask, void* stream) {
  if (int rc = check_match(m, d_view_dirs)) return rc;
  FIF_CHECK_ARG(rows >= 0 && n_points >= 0, "fif_match_mask: negative size");
  if (rows == 0 || n_points == 0) return FIF_OK;
  FIF_CHECK_ARG(d_centers && d_points && d_mask, "fif_match_mask: NULL centers/points/mask");
  const unsigned bx = (unsigned)((n_points + MM_THREADS * MM_PER_T - 1) / (MM_THREADS * MM_PER_T));
  const unsigned by = (unsigned)(rows < 65535 ? rows : 65535);
  k_match_mask<<<dim3(bx, by), MM_THREADS, 0, (cudaStream_t)stream>>>(*m, d_centers, rows, d_points, d_view_dirs,
                                                                      n_points, d_mask);
  FIF_CHECK_LAUNCH("k_match_mask");
  return FIF_OK;
}

extern "C" int fif_match_any(const fif_match* m, const double* d_centers, int64_t rows, const double* d_points,
                             const double* d_view_dirs, int64_t n_points, uint8_t* d_any, void* stream) {
  if (int rc = check_match(m, d_view_dirs)) return rc;
  FIF_CHECK_ARG(rows >= 0 && n_points >= 0, "fif_match_any: negative size");
  if (rows == 0) return FIF_OK;
  FIF_CHECK_ARG(d_centers && d_any && (n_points == 0 || d_points), "fif_match_any: NULL centers/points/out");
  cudaStream_t st = (cudaStream_t)stream;
  if (n_points == 0) {
    cudaMemsetAsync(d_any, 0, (size_t)rows, st);
    FIF_CHECK_LAUNCH("fif_match_any(memset)");
    return FIF_OK;
  }
  const int64_t cap = (int64_t)num_sms() * 8;
  k_match_any<<<(unsigned)(rows < cap ? rows : cap), MM_THREADS, 0, st>>>(*m, d_centers, rows, d_points, d_view_dirs,
                                                                         n_points, d_any);
  FIF_CHECK_LAUNCH("k_match_any");
  return FIF_OK;
}
