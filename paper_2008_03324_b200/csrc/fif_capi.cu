// fif_capi.cu — C-ABI plumbing: thread-local error string, launch counter,
// version, grid centres.
#include <cstdarg>
#include <cstdio>

#include "fif_common.cuh"

namespace fif {
static thread_local char g_err[512] = "";
static std::atomic<int64_t> g_launches{0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int num_sms() {
  static std::atomic<int> cache[64];
  int dev = 0;
  cudaGetDevice(&dev);
  int v = cache[dev & 63].load(std::memory_order_relaxed);
  if (v <= 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    cache[dev & 63].store(v, std::memory_order_relaxed);
  }
  return v;
}

__global__ void k_centers(VoxSrc s, int order, int64_t v0, int64_t v1, double* __restrict__ out) {
  int64_t v = v0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (v >= v1) return;
  double cx, cy, cz;
  if (order == 1) {
    voxel_center(s, v, cx, cy, cz);
  } else {
    int64_t iz = v % s.nz, r = v / s.nz, iy = r % s.ny, ix = r / s.ny;
    int64_t vz = (iz * s.ny + iy) * s.nx + ix;
    voxel_center(s, vz, cx, cy, cz);
  }
  out[3 * (v - v0)] = cx;
  out[3 * (v - v0) + 1] = cy;
  out[3 * (v - v0) + 2] = cz;
}
}  // namespace fif

using namespace fif;

extern "C" int fif_abi_version(void) { return FIF_ABI_VERSION; }
extern "C" const char* fif_last_error(void) { return g_err; }
extern "C" int64_t fif_launch_count(void) { return g_launches.load(); }

extern "C" int fif_grid_centers(const fif_grid* grid, int order, int64_t v_begin, int64_t v_end, double* d_out,
                                void* stream) {
  FIF_CHECK_ARG(grid && d_out, "fif_grid_centers: NULL argument");
  FIF_CHECK_ARG(order == 0 || order == 1, "fif_grid_centers: order must be 0 or 1");
  int64_t V = grid->dims[0] * grid->dims[1] * grid->dims[2];
  FIF_CHECK_ARG(0 <= v_begin && v_begin <= v_end && v_end <= V, "fif_grid_centers: bad range");
  if (v_end == v_begin) return FIF_OK;
  VoxSrc s{nullptr, grid->origin[0], grid->origin[1], grid->origin[2], grid->voxel_size,
           grid->dims[0], grid->dims[1], grid->dims[2]};
  int64_t n = v_end - v_begin;
  k_centers<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(s, order, v_begin, v_end, d_out);
  FIF_CHECK_LAUNCH("k_centers");
  return FIF_OK;
}
