// fif_pc.cu — point-cloud brute-force Fisher information (the paper's baseline), sm_100a.
//
// Replaces _nb_exact_fim / _nb_exact_fim_batch (kernels.py:571-599, 743-749).
// One warp per pose, lanes over landmarks; landmark tiles are staged once per
// CTA in shared memory and shared by its 16 poses.  The visibility test is the
// reference's FP64 arithmetic in its exact operation order (no FMA), with the
// two IEEE divisions replaced by sign tests on fma residuals wherever the
// residual is far from zero — the decision is then provably identical — and
// evaluated exactly otherwise.  Visible landmarks are compacted through a
// per-warp smem queue so the FP32 6x6 accumulation runs on full warps.
#include "fif_common.cuh"

namespace fif {

constexpr int PC_WARPS = 16;
constexpr int PC_TILE = 2048;
constexpr int PC_QCAP = 64;

struct PoseR {
  double r00, r01, r02, r10, r11, r12, r20, r21, r22, tx, ty, tz;
};

// Reference test (kernels.py:580-595): zc = r02 dx + r12 dy + r22 dz (left to right),
// u = fx xc / zc + cx rejected if < 0 or >= width, same for v.
__device__ __forceinline__ bool pc_visible(const PoseR& P, double px, double py, double pz, const fif_camera& cam,
                                           double cxw, double cyh) {
  const double dx = __dsub_rn(px, P.tx), dy = __dsub_rn(py, P.ty), dz = __dsub_rn(pz, P.tz);
  const double zc = __dadd_rn(__dadd_rn(__dmul_rn(P.r02, dx), __dmul_rn(P.r12, dy)), __dmul_rn(P.r22, dz));
  if (!(zc > 0.0)) return false;
  const double xc = __dadd_rn(__dadd_rn(__dmul_rn(P.r00, dx), __dmul_rn(P.r10, dy)), __dmul_rn(P.r20, dz));
  const double a = __dmul_rn(cam.fx, xc);
  // u_px = RN(RN(a / zc) + cx).  b0 = zc (a/zc + cx), b1 = zc (a/zc + cx - width), one rounding each.
  {
    const double b0 = fma(cam.cx, zc, a), b1 = fma(cxw, zc, a);
    const double m = 1e-12 * (fabs(a) + fabs(cam.cx) * zc + fabs(cam.width) * zc);
    if (b0 < -m || b1 > m) return false;
    if (!(b0 > m && b1 < -m)) {  // near an image border: evaluate exactly as the reference
      const double u = __dadd_rn(__ddiv_rn(a, zc), cam.cx);
      if (u < 0.0 || u >= cam.width) return false;
    }
  }
  const double yc = __dadd_rn(__dadd_rn(__dmul_rn(P.r01, dx), __dmul_rn(P.r11, dy)), __dmul_rn(P.r21, dz));
  const double b = __dmul_rn(cam.fy, yc);
  {
    const double b0 = fma(cam.cy, zc, b), b1 = fma(cyh, zc, b);
    const double m = 1e-12 * (fabs(b) + fabs(cam.cy) * zc + fabs(cam.height) * zc);
    if (b0 < -m || b1 > m) return false;
    if (!(b0 > m && b1 < -m)) {
      const double v = __dadd_rn(__ddiv_rn(b, zc), cam.cy);
      if (v < 0.0 || v >= cam.height) return false;
    }
  }
  return true;
}

// 21 unique entries of the per-landmark 6x6 (kernels.py:363-424) in packed order, FP32.
__device__ __forceinline__ void fim21(float dx, float dy, float dz, float px, float py, float pz, float inv_s2,
                                      float* e) {
  float n2 = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
  float rn = rsqrtf(n2);
  rn = fmaf(0.5f * rn, fmaf(-n2 * rn, rn, 1.0f), rn);
  float ux = dx * rn, uy = dy * rn, uz = dz * rn, w = inv_s2 * rn * rn;
  float pp = fmaf(px, px, fmaf(py, py, pz * pz));
  float wx = w * ux, wy = w * uy, wz = w * uz;
  float c2x = fmaf(py, uz, -pz * uy), c2y = fmaf(pz, ux, -px * uz), c2z = fmaf(px, uy, -py * ux);
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

__constant__ int kPR[21] = {0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 1, 2, 2, 2, 2, 3, 3, 3, 4, 4, 5};
__constant__ int kPC[21] = {0, 1, 2, 3, 4, 5, 1, 2, 3, 4, 5, 2, 3, 4, 5, 3, 4, 5, 4, 5, 5};

// Landmark table for the FP32 pre-test: p = hi + lo (float4 {hi.xyz, 0}, {lo.xyz, 0}).
__global__ void k_pc_prep(const double* __restrict__ pts, int64_t n, float4* __restrict__ tab) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  float hx, lx, hy, ly, hz, lz;
  split_f32(pts[3 * i], hx, lx);
  split_f32(pts[3 * i + 1], hy, ly);
  split_f32(pts[3 * i + 2], hz, lz);
  tab[2 * i] = make_float4(hx, hy, hz, 0.f);
  tab[2 * i + 1] = make_float4(lx, ly, lz, 0.f);
}

// FP32 pre-test with rigorous margins, branch-free: returns +1 (certainly visible
// under the reference's FP64 test), -1 (certainly invisible) or 0 (within the error
// band of z = 0 or of an image border: decide with the exact FP64 test).
// d = p - t is exact to ~1 ulp of |d| (hi/lo parts); every FP32 rounding below is
// bounded by a few ulp of |f| |d|_1, and the margins are 8-16 ulp of that.
struct PoseF {
  float r00, r01, r02, r10, r11, r12, r20, r21, r22, thx, thy, thz, tlx, tly, tlz;
};
struct CamF {
  float fx, fy, cx, cy, cxw, cyh, mz, mu, mv;
};
__device__ __forceinline__ int pc_pretest(const PoseF& P, float4 ph, float4 pl, const CamF& C, float& dx, float& dy,
                                          float& dz) {
  dx = (ph.x - P.thx) + (pl.x - P.tlx);
  dy = (ph.y - P.thy) + (pl.y - P.tly);
  dz = (ph.z - P.thz) + (pl.z - P.tlz);
  const float l1 = fabsf(dx) + fabsf(dy) + fabsf(dz);
  const float zc = fmaf(P.r02, dx, fmaf(P.r12, dy, P.r22 * dz));
  const float xc = fmaf(P.r00, dx, fmaf(P.r10, dy, P.r20 * dz));
  const float yc = fmaf(P.r01, dx, fmaf(P.r11, dy, P.r21 * dz));
  const float a = C.fx * xc, b = C.fy * yc;
  const float b0 = fmaf(C.cx, zc, a), b1 = fmaf(C.cxw, zc, a);
  const float c0 = fmaf(C.cy, zc, b), c1 = fmaf(C.cyh, zc, b);
  const float mz = C.mz * l1, m1 = C.mu * l1, m2 = C.mv * l1;
  const bool zpos = zc > mz, zneg = zc < -mz;
  const bool out = (b0 < -m1) | (b1 > m1) | (c0 < -m2) | (c1 > m2);
  const bool in = (b0 > m1) & (b1 < -m1) & (c0 > m2) & (c1 < -m2);
  return (zpos & in) ? 1 : ((zneg | (zpos & out)) ? -1 : 0);
}

template <bool MASK>
__global__ void __launch_bounds__(PC_WARPS * 32) k_pc_fim(const double* __restrict__ rot, const double* __restrict__ tr,
                                                          int64_t nq, const double* __restrict__ pts,
                                                          const float4* __restrict__ ptab, int64_t n, fif_camera cam,
                                                          float inv_s2, double* __restrict__ out,
                                                          uint8_t* __restrict__ mask) {
  extern __shared__ float4 pcsm[];
  float4 (*tile)[PC_TILE] = reinterpret_cast<float4 (*)[PC_TILE]>(pcsm);                     // [2][PC_TILE]
  float4 (*queue)[PC_QCAP][2] = reinterpret_cast<float4 (*)[PC_QCAP][2]>(pcsm + 2 * PC_TILE);  // [warps][cap][2]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double cxw = cam.cx - cam.width, cyh = cam.cy - cam.height;
  // margins: 16 ulp(fp32) x (|f| + |c| + |w|) per unit of |d|_1 (bounds every rounding
  // of the FP32 evaluation plus the FP64 reference's own roundings)
  CamF CF;
  CF.fx = (float)cam.fx; CF.fy = (float)cam.fy; CF.cx = (float)cam.cx; CF.cy = (float)cam.cy;
  CF.cxw = (float)cxw; CF.cyh = (float)cyh;
  CF.mz = 8.0f * 5.96e-8f;
  CF.mu = 16.0f * 5.96e-8f * (float)(fabs(cam.fx) + fabs(cam.cx) + fabs(cam.width));
  CF.mv = 16.0f * 5.96e-8f * (float)(fabs(cam.fy) + fabs(cam.cy) + fabs(cam.height));
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int64_t q0 = blockIdx.x * (int64_t)PC_WARPS; q0 < nq; q0 += (int64_t)gridDim.x * PC_WARPS) {
    const int64_t q = q0 + warp;
    const bool has_pose = q < nq;
    PoseR P;
    PoseF PF;
    {
      const int64_t qq = has_pose ? q : q0;
      const double* R = rot + 9 * qq;
      P.r00 = R[0]; P.r01 = R[1]; P.r02 = R[2];
      P.r10 = R[3]; P.r11 = R[4]; P.r12 = R[5];
      P.r20 = R[6]; P.r21 = R[7]; P.r22 = R[8];
      P.tx = tr[3 * qq]; P.ty = tr[3 * qq + 1]; P.tz = tr[3 * qq + 2];
      PF.r00 = (float)P.r00; PF.r01 = (float)P.r01; PF.r02 = (float)P.r02;
      PF.r10 = (float)P.r10; PF.r11 = (float)P.r11; PF.r12 = (float)P.r12;
      PF.r20 = (float)P.r20; PF.r21 = (float)P.r21; PF.r22 = (float)P.r22;
      split_f32(P.tx, PF.thx, PF.tlx);
      split_f32(P.ty, PF.thy, PF.tly);
      split_f32(P.tz, PF.thz, PF.tlz);
    }
    float acc[21];
#pragma unroll
    for (int e = 0; e < 21; ++e) acc[e] = 0.f;
    int qn = 0;  // queued entries (warp-uniform)
    for (int64_t base = 0; base < n; base += PC_TILE) {
      const int cnt = (int)min((int64_t)PC_TILE, n - base);
      __syncthreads();
      for (int j = threadIdx.x; j < cnt * 2; j += blockDim.x) tile[j & 1][j >> 1] = ptab[2 * base + j];
      __syncthreads();
      if (!has_pose) continue;
      for (int j0 = 0; j0 < cnt; j0 += 32) {
        const int j = j0 + lane;
        bool vis = false;
        float dx = 0.f, dy = 0.f, dz = 0.f;
        float4 ph = make_float4(0.f, 0.f, 0.f, 0.f);
        if (j < cnt) {
          ph = tile[0][j];
          const int pre = pc_pretest(PF, ph, tile[1][j], CF, dx, dy, dz);
          if (pre == 0) {
            const int64_t i = base + j;
            vis = pc_visible(P, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], cam, cxw, cyh);
          } else {
            vis = pre > 0;
          }
          if (MASK) mask[q * n + base + j] = (uint8_t)vis;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, vis);
        if (vis) {
          const int slot = qn + __popc(bal & lt_mask);
          queue[warp][slot][0] = make_float4(dx, dy, dz, 0.f);
          queue[warp][slot][1] = ph;
        }
        qn += __popc(bal);
        if (qn >= 32) {
          __syncwarp();
          const float4 d = queue[warp][lane][0], p = queue[warp][lane][1];
          float e[21];
          fim21(d.x, d.y, d.z, p.x, p.y, p.z, inv_s2, e);
#pragma unroll
          for (int k = 0; k < 21; ++k) acc[k] += e[k];
          __syncwarp();
          qn -= 32;
          if (lane < qn) {  // move the overflow to the front
            queue[warp][lane][0] = queue[warp][32 + lane][0];
            queue[warp][lane][1] = queue[warp][32 + lane][1];
          }
          __syncwarp();
        }
      }
    }
    if (has_pose) {
      __syncwarp();
      if (lane < qn) {
        const float4 d = queue[warp][lane][0], p = queue[warp][lane][1];
        float e[21];
        fim21(d.x, d.y, d.z, p.x, p.y, p.z, inv_s2, e);
#pragma unroll
        for (int k = 0; k < 21; ++k) acc[k] += e[k];
      }
#pragma unroll
      for (int k = 0; k < 21; ++k) {
        float v = acc[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        acc[k] = v;
      }
      double mine = 0.0;
#pragma unroll
      for (int k = 0; k < 21; ++k) if (lane == k) mine = (double)acc[k];
      if (lane < 21) {
        out[q * 36 + kPR[lane] * 6 + kPC[lane]] = mine;
        out[q * 36 + kPC[lane] * 6 + kPR[lane]] = mine;
      }
    }
  }
}

}  // namespace fif

using namespace fif;

extern "C" int fif_pc_fim(const double* d_rot, const double* d_t, int64_t q, const double* d_points, int64_t n_points,
                          const fif_camera* cam, double sigma, double* d_out, uint8_t* d_mask, void* stream) {
  FIF_CHECK_ARG(cam != nullptr, "fif_pc_fim: NULL camera");
  FIF_CHECK_ARG(sigma > 0, "fif_pc_fim: sigma must be positive");
  FIF_CHECK_ARG(q >= 0 && n_points >= 0, "fif_pc_fim: negative size");
  if (q == 0) return FIF_OK;
  FIF_CHECK_ARG(d_rot && d_t && d_out, "fif_pc_fim: NULL pointer");
  cudaStream_t st = (cudaStream_t)stream;
  if (n_points == 0) {  // fim.py:141-142: empty scene -> zeros
    cudaMemsetAsync(d_out, 0, sizeof(double) * 36 * q, st);
    FIF_CHECK_LAUNCH("fif_pc_fim(memset)");
    return FIF_OK;
  }
  FIF_CHECK_ARG(d_points != nullptr, "fif_pc_fim: NULL points");
  int64_t need = (q + PC_WARPS - 1) / PC_WARPS;
  int64_t cap = (int64_t)kSMs * 2;
  unsigned blocks = (unsigned)(need < cap ? need : cap);
  const float inv_s2 = (float)(1.0 / (sigma * sigma));
  float4* ptab = nullptr;
  if (cudaMallocAsync(&ptab, sizeof(float4) * 2 * n_points, st) != cudaSuccess) {
    set_error("fif_pc_fim: cudaMallocAsync failed");
    return FIF_ERR_CUDA;
  }
  k_pc_prep<<<(unsigned)((n_points + 255) / 256), 256, 0, st>>>(d_points, n_points, ptab);
  FIF_CHECK_LAUNCH("k_pc_prep");
  const size_t smem = sizeof(float4) * (2 * PC_TILE + PC_WARPS * PC_QCAP * 2);
  static bool attr = false;
  if (!attr) {
    for (auto f : {k_pc_fim<true>, k_pc_fim<false>}) {
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    }
    attr = true;
  }
  if (d_mask)
    k_pc_fim<true><<<blocks, PC_WARPS * 32, smem, st>>>(d_rot, d_t, q, d_points, ptab, n_points, *cam, inv_s2, d_out,
                                                        d_mask);
  else
    k_pc_fim<false><<<blocks, PC_WARPS * 32, smem, st>>>(d_rot, d_t, q, d_points, ptab, n_points, *cam, inv_s2,
                                                         d_out, d_mask);
  cudaFreeAsync(ptab, st);
  FIF_CHECK_LAUNCH("k_pc_fim");
  return FIF_OK;
}
