// fif_pc.cu — point-cloud brute-force Fisher information (the paper's baseline), sm_100a.
//
// Replaces _nb_exact_fim / _nb_exact_fim_batch (kernels.py:571-599, 743-749).
// One warp per pose, lanes over landmarks; landmark tiles are staged once per
// CTA in shared memory and shared by its 16 poses.  A producer warp streams the
// tiles with TMA bulk copies into a PC_NBUF-deep ring (mbarrier full/empty pairs),
// so pose warps never wait on each other: a warp with many visible landmarks may
// lag the others by up to PC_NBUF - 1 tiles.  The visibility test is the
// reference's FP64 arithmetic in its exact operation order (no FMA), with the
// two IEEE divisions replaced by sign tests on fma residuals wherever the
// residual is far from zero — the decision is then provably identical — and
// evaluated exactly otherwise.  Visible landmarks are compacted through a
// per-warp smem queue so the FP32 6x6 accumulation runs on full warps.
// Spatial culling: landmarks are sorted in Morton order and cut into groups of 32 with a
// bounding box each; a pose first evaluates its five affine visibility rows over each
// group's box (lane = group, 32 groups per tile), so groups that are certainly outside
// the view (most of them) are skipped and groups certainly inside go straight to the
// 6x6 accumulation; only groups the frustum boundary crosses run the per-landmark test.
#include "fif_common.cuh"
#include "fif_linalg.cuh"

#include <cub/cub.cuh>

namespace fif {

constexpr int PC_WARPS = 15;  // pose warps; + 1 producer warp = 4 warps per SM sub-partition
#ifndef PC_TILE_N
#define PC_TILE_N 1024
#endif
constexpr int PC_TILE = PC_TILE_N;
#ifndef PC_RING_LM
#define PC_RING_LM 4096
#endif
constexpr int PC_NBUF = PC_RING_LM / PC_TILE;  // 128 KB ring (hi + lo) at 4096 landmarks
constexpr int PC_QCAP = 64;
#ifndef PC_SLEEPWAIT
#define PC_SLEEPWAIT 1  // ring waits suspend in hardware instead of spinning
#endif
#if PC_SLEEPWAIT
#define PC_WAIT mbar_wait_sleep
#else
#define PC_WAIT mbar_wait
#endif
// pre-test image-border rows as FFMA2 pairs (landmark coordinates broadcast): config 3
// 73.6 -> 70.4 ms, bit-identical decisions (FFMA2 rounds each lane like FFMA)
#ifndef PC_PACKED
#define PC_PACKED 1
#endif

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

// Landmark tables in Morton order (slot k holds landmark i = order[k]): hi[k] = {p_hi.xyz,
// |p_hi|_1}, lo[k] = {p_lo.xyz, i as int bits}, p = p_hi + p_lo; *p1max = max |p_hi|_1
// (float bits, for the pre-test margins).
__global__ void k_pc_prep(const double* __restrict__ pts, int64_t n, const int32_t* __restrict__ order,
                          float4* __restrict__ tab, unsigned* __restrict__ p1max) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  float l1 = 0.f;
  if (k < n) {
    const int64_t i = order ? (int64_t)order[k] : k;
    float hx, lx, hy, ly, hz, lz;
    split_f32(pts[3 * i], hx, lx);
    split_f32(pts[3 * i + 1], hy, ly);
    split_f32(pts[3 * i + 2], hz, lz);
    l1 = fabsf(hx) + fabsf(hy) + fabsf(hz);
    tab[k] = make_float4(hx, hy, hz, l1);
    tab[n + k] = make_float4(lx, ly, lz, __int_as_float((int)i));
  }
  const unsigned m = __reduce_max_sync(0xffffffffu, __float_as_uint(l1));  // non-negative floats order as ints
  if ((threadIdx.x & 31) == 0) atomicMax(p1max, m);
}

// Box of each group of 32 consecutive table slots (over p_hi): centre c and a half
// extent e rounded up, so every p_hi of the group lies in [c - e, c + e].
__global__ void k_pc_groups(const float4* __restrict__ tab, int64_t n, float4* __restrict__ gbox) {
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g * 32 >= n) return;
  float mn[3] = {3.0e38f, 3.0e38f, 3.0e38f}, mx[3] = {-3.0e38f, -3.0e38f, -3.0e38f};
  const int64_t end = min(n, g * 32 + 32);
  for (int64_t k = g * 32; k < end; ++k) {
    const float4 p = tab[k];
    mn[0] = fminf(mn[0], p.x), mx[0] = fmaxf(mx[0], p.x);
    mn[1] = fminf(mn[1], p.y), mx[1] = fmaxf(mx[1], p.y);
    mn[2] = fminf(mn[2], p.z), mx[2] = fmaxf(mx[2], p.z);
  }
  float c[3], e[3];
  for (int a = 0; a < 3; ++a) {
    c[a] = 0.5f * (mn[a] + mx[a]);
    e[a] = fmaxf(__fsub_ru(mx[a], c[a]), __fsub_ru(c[a], mn[a]));
  }
  gbox[2 * g] = make_float4(c[0], c[1], c[2], 0.f);
  gbox[2 * g + 1] = make_float4(e[0], e[1], e[2], 0.f);
}

// 30-bit Morton key of each landmark over the landmarks' bounding box (part: k_pc_bbox)
__device__ __forceinline__ uint32_t spread10(uint32_t v) {
  v &= 0x3ffu;
  v = (v | (v << 16)) & 0x030000FFu;
  v = (v | (v << 8)) & 0x0300F00Fu;
  v = (v | (v << 4)) & 0x030C30C3u;
  v = (v | (v << 2)) & 0x09249249u;
  return v;
}
__global__ void k_pc_mkeys(const double* __restrict__ pts, int64_t n, const double* __restrict__ part, int nparts,
                           uint32_t* __restrict__ keys, int32_t* __restrict__ idx) {
  __shared__ double box[6];
  if (threadIdx.x < 6) {
    const bool is_lo = threadIdx.x < 3;
    double v = is_lo ? 1e300 : -1e300;
    for (int b = 0; b < nparts; ++b) v = is_lo ? fmin(v, part[b * 6 + threadIdx.x]) : fmax(v, part[b * 6 + threadIdx.x]);
    box[threadIdx.x] = v;
  }
  __syncthreads();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t c[3];
  for (int a = 0; a < 3; ++a) {
    const double ext = box[3 + a] - box[a];
    const double f = ext > 0 ? (pts[3 * i + a] - box[a]) / ext * 1024.0 : 0.0;
    c[a] = (uint32_t)fmin(fmax(f, 0.0), 1023.0);
  }
  keys[i] = spread10(c[0]) | (spread10(c[1]) << 1) | (spread10(c[2]) << 2);
  idx[i] = (int32_t)i;
}

// FP32 pre-test with rigorous margins, branch-free.  Every quantity the reference
// compares is an affine function of the landmark position p for a fixed pose:
//   zc = R2 . (p - t),  b0 = zc (u - 0) = (fx R0 + cx R2) . (p - t),  b1 = zc (u - W),
//   c0 = zc (v - 0),    c1 = zc (v - H)                 (u, v the pixel coordinates)
// and the reference sees the landmark iff zc > 0, b0 >= 0, b1 < 0, c0 >= 0, c1 < 0.
// The FP32 evaluation of w_k . p_hi + C_k (per-pose coefficients formed in FP64)
// differs from the exact value by at most ~6 u W_k (|p|_1 + |t|_1) (u = 2^-24, W_k =
// max |w_k|: coefficient and constant rounding, p_lo dropped, three FMA roundings), and
// the reference's FP64 decision by far less.  With the pose-uniform margin
// m_k = 16 u (W_k (max_i |p_i|_1 + |t|_1) + |C_k|), each row is stored normalised as
//   h_k = s_k (w_k . p + C_k) / m_k + 1      (s_k = +1, +1, -1, +1, -1: "inside" > 0)
// whose FP32 evaluation is within ~0.4 of its exact value (the normalisation's own
// roundings included), so h_k > 2 proves the row's condition and h_k < 0 refutes it.
// Returns +1 certainly visible, -1 certainly not, 0 otherwise: run the reference's
// exact FP64 test.
struct PoseAff {
  float w[5][3], c[5];
#if PC_PACKED
  f32x2 w12[3], w34[3], c12, c34;  // image-border rows (1, 2) and (3, 4) as FP32x2 pairs
#endif
};
// Group box test.  h_k over the box {c +- e}: h_k(c) +- sum_i |w_ki| e_i.  h_k(c) carries
// at most ~1.2 of FP32 error (|c|_1 <= 3 max_i |p_i|_1 against the margin's max |p|_1), the
// extent term 3 roundings (covered by the 1 + 2^-20 factor), so min_k > 3 proves every
// landmark's exact row value > 1 (all five conditions hold: certainly visible) and any
// row's max < -1 proves that row fails for every landmark (certainly invisible: for
// zc > 0 the failed image-border row rejects it, for zc <= 0 the first test does).
// Returns +1 / -1 / 0 (mixed).
__device__ __forceinline__ int pc_boxtest(const PoseAff& A, float4 c, float4 e) {
  float mn = 3.0e38f, mxmin = 3.0e38f;
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const float hc = fmaf(A.w[k][0], c.x, fmaf(A.w[k][1], c.y, fmaf(A.w[k][2], c.z, A.c[k])));
    const float ex = fmaf(fabsf(A.w[k][0]), e.x, fmaf(fabsf(A.w[k][1]), e.y, fabsf(A.w[k][2]) * e.z)) * 1.000001f;
    mn = fminf(mn, hc - ex);
    mxmin = fminf(mxmin, hc + ex);
  }
  return mn > 3.f ? 1 : (mxmin < -1.f ? -1 : 0);
}

__device__ __forceinline__ int pc_pretest(const PoseAff& A, float4 ph) {
  float h[5];
#if PC_PACKED
  h[0] = fmaf(A.w[0][0], ph.x, fmaf(A.w[0][1], ph.y, fmaf(A.w[0][2], ph.z, A.c[0])));
  const f32x2 X = splat2(ph.x), Y = splat2(ph.y), Z = splat2(ph.z);
  unpack2(ffma2(A.w12[0], X, ffma2(A.w12[1], Y, ffma2(A.w12[2], Z, A.c12))), h[1], h[2]);
  unpack2(ffma2(A.w34[0], X, ffma2(A.w34[1], Y, ffma2(A.w34[2], Z, A.c34))), h[3], h[4]);
#else
#pragma unroll
  for (int k = 0; k < 5; ++k) h[k] = fmaf(A.w[k][0], ph.x, fmaf(A.w[k][1], ph.y, fmaf(A.w[k][2], ph.z, A.c[k])));
#endif
  const float img = fminf(fminf(h[1], h[2]), fminf(h[3], h[4]));  // the four image-border rows
  const bool vis = fminf(h[0], img) > 2.f;
  const bool invis = (h[0] < 0.f) | ((h[0] > 2.f) & (img < 0.f));
  return vis ? 1 : (invis ? -1 : 0);
}

// 16-byte shared-memory load at a shared-window address (keeps the tile address
// arithmetic in 32-bit shared offsets)
__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}

constexpr int PC_GPT = PC_TILE / 32;  // landmark groups per tile (one per lane)
static_assert(PC_GPT <= 32 && PC_TILE % 32 == 0, "the box test maps one group to each lane");
template <bool MASK, bool CULL>
__global__ void __launch_bounds__((PC_WARPS + 1) * 32, 1) k_pc_fim(const double* __restrict__ rot, const double* __restrict__ tr,
                                                          int64_t nq, const double* __restrict__ pts,
                                                          const float4* __restrict__ ptab, const float4* __restrict__ gbox,
                                                          int64_t n, fif_camera cam,
                                                          const unsigned* __restrict__ p1max, float inv_s2, double* __restrict__ out,
                                                          uint8_t* __restrict__ mask, const int32_t* __restrict__ perm) {
  extern __shared__ float4 pcsm[];
  float4* ring_hi = pcsm;                                  // [PC_NBUF][PC_TILE]
  float4* ring_lo = pcsm + PC_NBUF * PC_TILE;              // [PC_NBUF][PC_TILE] (w = original index bits)
  float4* ring_box = pcsm + 2 * PC_NBUF * PC_TILE;         // [PC_NBUF][2 * PC_GPT] group centre / half extent
  float4* queues = ring_box + PC_NBUF * 2 * PC_GPT;        // [PC_WARPS][PC_QCAP][2]
  uint64_t* full = reinterpret_cast<uint64_t*>(queues + PC_WARPS * PC_QCAP * 2);  // [PC_NBUF]
  uint64_t* empty = full + PC_NBUF;                                                 // [PC_NBUF]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int b = 0; b < PC_NBUF; ++b) {
      mbar_init(&full[b], 1);
      mbar_init(&empty[b], PC_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t ntiles = (n + PC_TILE - 1) / PC_TILE;
  const int64_t qstride = (int64_t)gridDim.x * PC_WARPS;
  const int64_t npi = blockIdx.x * (int64_t)PC_WARPS < nq ? (nq - blockIdx.x * (int64_t)PC_WARPS + qstride - 1) / qstride : 0;
  if (warp == PC_WARPS) {  // producer: every tile of every pose group, in consumption order
    if (lane == 0) {
      int64_t seq = 0;
      for (int64_t it = 0; it < npi; ++it)
        for (int64_t t = 0; t < ntiles; ++t, ++seq) {
          const int b = (int)(seq % PC_NBUF);
          PC_WAIT(&empty[b], (uint32_t)(((seq / PC_NBUF) & 1) ^ 1));
          const int64_t base = t * PC_TILE;
          const int cnt = (int)min((int64_t)PC_TILE, n - base);
          const uint32_t bytes = (uint32_t)(cnt * sizeof(float4));
          const uint32_t bbytes = CULL ? (uint32_t)(((cnt + 31) / 32) * 2 * sizeof(float4)) : 0u;
          mbar_expect_tx(&full[b], 2 * bytes + bbytes);
          tma_bulk_g2s(ring_hi + b * PC_TILE, ptab + base, bytes, &full[b]);
          tma_bulk_g2s(ring_lo + b * PC_TILE, ptab + n + base, bytes, &full[b]);
          if (CULL) tma_bulk_g2s(ring_box + b * 2 * PC_GPT, gbox + 2 * (base / 32), bbytes, &full[b]);
        }
    }
    return;
  }
  float4* qd = queues + warp * PC_QCAP * 2;  // (d, p) of queued visible landmarks
  const double cxw = cam.cx - cam.width, cyh = cam.cy - cam.height;
  const unsigned lt_mask = (1u << lane) - 1u;
  int64_t seq = 0;
  for (int64_t it = 0; it < npi; ++it) {
    const int64_t q0 = blockIdx.x * (int64_t)PC_WARPS + it * qstride;
    const int64_t qs = q0 + warp;                                  // slot (similar poses adjacent)
    const int64_t q = qs < nq && perm ? (int64_t)perm[qs] : qs;  // caller's pose index
    const bool has_pose = qs < nq;
    PoseAff A;
    float thx, thy, thz, tlx, tly, tlz;
    {
      const int64_t qq = has_pose ? q : (perm ? (int64_t)perm[q0] : q0);
      const double* R = rot + 9 * qq;
      const double tx = tr[3 * qq], ty = tr[3 * qq + 1], tz = tr[3 * qq + 2];
      split_f32(tx, thx, tlx);
      split_f32(ty, thy, tly);
      split_f32(tz, thz, tlz);
      // affine rows in FP64: world-frame coefficients of zc, b0, b1, c0, c1
      const double R0[3] = {R[0], R[3], R[6]}, R1[3] = {R[1], R[4], R[7]}, R2[3] = {R[2], R[5], R[8]};
      const double lt = fabs(tx) + fabs(ty) + fabs(tz) + (double)__uint_as_float(*p1max);
#pragma unroll
      for (int k = 0; k < 5; ++k) {
        double w[3];
#pragma unroll
        for (int i = 0; i < 3; ++i)
          w[i] = k == 0 ? R2[i]
                        : k == 1 ? cam.fx * R0[i] + cam.cx * R2[i]
                                 : k == 2 ? cam.fx * R0[i] + cxw * R2[i]
                                          : k == 3 ? cam.fy * R1[i] + cam.cy * R2[i] : cam.fy * R1[i] + cyh * R2[i];
        const double c = -(w[0] * tx + w[1] * ty + w[2] * tz);
        const double wm = fmax(fabs(w[0]), fmax(fabs(w[1]), fabs(w[2])));
        const double mk = 16.0 * 0x1p-24 * (wm * lt + fabs(c)) * 1.000001;
        const double sc = (k == 2 || k == 4 ? -1.0 : 1.0) / mk;
#pragma unroll
        for (int i = 0; i < 3; ++i) A.w[k][i] = (float)(w[i] * sc);
        A.c[k] = (float)(c * sc + 1.0);
      }
#if PC_PACKED
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        A.w12[i] = pack2(A.w[1][i], A.w[2][i]);
        A.w34[i] = pack2(A.w[3][i], A.w[4][i]);
      }
      A.c12 = pack2(A.c[1], A.c[2]);
      A.c34 = pack2(A.c[3], A.c[4]);
#endif
    }
    float acc[21];
#pragma unroll
    for (int e = 0; e < 21; ++e) acc[e] = 0.f;
    int qn = 0;  // queued entries (warp-uniform)
    for (int64_t t = 0; t < ntiles; ++t, ++seq) {
      const int64_t base = t * PC_TILE;
      const int cnt = (int)min((int64_t)PC_TILE, n - base);
      const int bsel = (int)(seq % PC_NBUF);
      const uint32_t tile_hi = smem_u32(ring_hi + bsel * PC_TILE) + 16u * lane;  // this lane's first landmark
      const uint32_t tile_lo = smem_u32(ring_lo + bsel * PC_TILE) + 16u * lane;
      PC_WAIT(&full[bsel], (uint32_t)((seq / PC_NBUF) & 1));
      if (!has_pose) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[bsel]);
        continue;
      }
      // group decisions for this tile: lane g tests group g's box
      const int ngr = (cnt + 31) >> 5;
      unsigned todo = ngr >= 32 ? 0xffffffffu : (1u << ngr) - 1u;
      unsigned allvis = 0u;
      if (CULL) {
        int dec = -1;
        if (lane < ngr) {
          const uint32_t bx = smem_u32(ring_box + bsel * 2 * PC_GPT) + 32u * lane;
          dec = pc_boxtest(A, lds128(bx), lds128(bx + 16u));
        }
        allvis = __ballot_sync(0xffffffffu, dec > 0);
        todo &= ~__ballot_sync(0xffffffffu, dec < 0);
      }
      while (todo) {
        const int g = __ffs(todo) - 1;
        todo &= todo - 1;
        const int j0 = 32 * g, j = j0 + lane;
        if ((allvis >> g) & 1u) {  // every landmark of the group is visible: accumulate directly
          if (j < cnt) {
            const float4 ph = lds128(tile_hi + 16u * j0), pl = lds128(tile_lo + 16u * j0);
            const float dx = (ph.x - thx) + (pl.x - tlx), dy = (ph.y - thy) + (pl.y - tly),
                        dz = (ph.z - thz) + (pl.z - tlz);
            float e[21];
            fim21(dx, dy, dz, ph.x, ph.y, ph.z, inv_s2, e);
#pragma unroll
            for (int k = 0; k < 21; ++k) acc[k] += e[k];
            if (MASK) mask[q * n + __float_as_int(pl.w)] = 1;
          }
          continue;
        }
        bool vis = false;
        float4 ph = make_float4(0.f, 0.f, 0.f, 0.f), pl = ph;
        if (j < cnt) {
          ph = lds128(tile_hi + 16u * j0);
          const int pre = pc_pretest(A, ph);
          if (pre == 0) {  // within a margin: the reference's FP64 test (pose re-read: rare path)
            pl = lds128(tile_lo + 16u * j0);
            const int64_t i = __float_as_int(pl.w);  // original landmark index
            const double* R = rot + 9 * q;
            const PoseR P{R[0], R[1], R[2], R[3], R[4], R[5], R[6], R[7], R[8], tr[3 * q], tr[3 * q + 1], tr[3 * q + 2]};
            vis = pc_visible(P, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], cam, cxw, cyh);
          } else {
            vis = pre > 0;
          }
        }
        const unsigned bal = __ballot_sync(0xffffffffu, vis);
        if (vis) {
          // d = p - t, exact to ~1 ulp of |d| from the hi / lo parts
          pl = lds128(tile_lo + 16u * j0);
          if (MASK) mask[q * n + __float_as_int(pl.w)] = 1;
          const float dx = (ph.x - thx) + (pl.x - tlx), dy = (ph.y - thy) + (pl.y - tly),
                      dz = (ph.z - thz) + (pl.z - tlz);
          const int slot = qn + __popc(bal & lt_mask);
          qd[2 * slot] = make_float4(dx, dy, dz, 0.f);
          qd[2 * slot + 1] = ph;
        }
        qn += __popc(bal);
        if (qn >= 32) {
          __syncwarp();
          const float4 d = qd[2 * lane], p = qd[2 * lane + 1];
          float e[21];
          fim21(d.x, d.y, d.z, p.x, p.y, p.z, inv_s2, e);
#pragma unroll
          for (int k = 0; k < 21; ++k) acc[k] += e[k];
          __syncwarp();
          qn -= 32;
          if (lane < qn) {  // move the overflow to the front
            qd[2 * lane] = qd[2 * (32 + lane)];
            qd[2 * lane + 1] = qd[2 * (32 + lane) + 1];
          }
          __syncwarp();
        }
      }
      __syncwarp();  // every lane is done reading this tile
      if (lane == 0) mbar_arrive(&empty[bsel]);
    }
    if (has_pose) {
      __syncwarp();
      if (lane < qn) {
        const float4 d = qd[2 * lane], p = qd[2 * lane + 1];
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

// Pose order for load balance: the 15 pose warps of a CTA share landmark tiles, so the
// CTA runs at the pace of its slowest pose; grouping similar poses (coarse position cell
// and optical-axis direction) into the same CTA evens their visible-landmark counts.
// per-block min / max of the pose positions (pass 1), reduced by one block (pass 2)
constexpr int PK_BLOCKS = 512;
__global__ void k_pc_bbox(const double* __restrict__ tr, int64_t nq, double* __restrict__ part) {
  __shared__ double lo[3][256], hi[3][256];
  double l[3] = {1e300, 1e300, 1e300}, h[3] = {-1e300, -1e300, -1e300};
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nq; q += (int64_t)gridDim.x * blockDim.x)
    for (int a = 0; a < 3; ++a) {
      l[a] = fmin(l[a], tr[3 * q + a]);
      h[a] = fmax(h[a], tr[3 * q + a]);
    }
  for (int a = 0; a < 3; ++a) {
    lo[a][threadIdx.x] = l[a];
    hi[a][threadIdx.x] = h[a];
  }
  __syncthreads();
  for (int s2 = blockDim.x / 2; s2 > 0; s2 >>= 1) {
    if ((int)threadIdx.x < s2)
      for (int a = 0; a < 3; ++a) {
        lo[a][threadIdx.x] = fmin(lo[a][threadIdx.x], lo[a][threadIdx.x + s2]);
        hi[a][threadIdx.x] = fmax(hi[a][threadIdx.x], hi[a][threadIdx.x + s2]);
      }
    __syncthreads();
  }
  if (threadIdx.x < 3) {
    part[blockIdx.x * 6 + threadIdx.x] = lo[threadIdx.x][0];
    part[blockIdx.x * 6 + 3 + threadIdx.x] = hi[threadIdx.x][0];
  }
}
__global__ void k_pc_keys(const double* __restrict__ rot, const double* __restrict__ tr, int64_t nq,
                          const double* __restrict__ part, int nparts, uint32_t* __restrict__ keys,
                          int32_t* __restrict__ idx) {
  __shared__ double box[6];
  if (threadIdx.x < 6) {
    const bool is_lo = threadIdx.x < 3;
    double v = is_lo ? 1e300 : -1e300;
    for (int b = 0; b < nparts; ++b) v = is_lo ? fmin(v, part[b * 6 + threadIdx.x]) : fmax(v, part[b * 6 + threadIdx.x]);
    box[threadIdx.x] = v;
  }
  __syncthreads();
  const int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (q >= nq) return;
  auto cell = [&](int a) -> uint32_t {  // 16 cells per axis over the poses' bounding box
    const double ext = box[3 + a] - box[a];
    const double c = ext > 0 ? floor((tr[3 * q + a] - box[a]) / ext * 16.0) : 0.0;
    return (uint32_t)fmin(fmax(c, 0.0), 15.0);
  };
  const uint32_t pc = (cell(2) << 8) | (cell(1) << 4) | cell(0);
  // optical axis = R[:, 2]: dominant axis and sign (6 faces) x 4 x 4 face cells
  const double ax = rot[9 * q + 2], ay = rot[9 * q + 5], az = rot[9 * q + 8];
  const double fx = fabs(ax), fy = fabs(ay), fz = fabs(az);
  int face;
  double u, v;
  if (fx >= fy && fx >= fz) { face = ax > 0 ? 0 : 1; u = ay / fx; v = az / fx; }
  else if (fy >= fz) { face = ay > 0 ? 2 : 3; u = ax / fy; v = az / fy; }
  else { face = az > 0 ? 4 : 5; u = ax / fz; v = ay / fz; }
  const uint32_t ui = (uint32_t)fmin(3.0, (u + 1.0) * 2.0), vi = (uint32_t)fmin(3.0, (v + 1.0) * 2.0);
  keys[q] = (((uint32_t)face * 16u + ui * 4u + vi) << 12) | pc;
  idx[q] = (int32_t)q;
}

// World-from-camera rotation of a yaw-only pose, R = Rz(yaw) R_base, in the reference's
// operation order (kernels.py:615-621): row 0 = c b0 - s b1, row 1 = s b0 + c b1, row 2 = b2,
// every product and sum rounded separately (numba emits no FMA here).  cos / sin come from
// the host (libm), like the reference's np.cos / np.sin.
struct Mat3 {
  double m[9];
};
__global__ void k_yaw_rot(const double* __restrict__ cs, int64_t q, Mat3 b, double* __restrict__ rot) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= q) return;
  const double c = cs[2 * i], s = cs[2 * i + 1];
  double* r = rot + 9 * i;
#pragma unroll
  for (int col = 0; col < 3; ++col) {
    r[col] = __dsub_rn(__dmul_rn(c, b.m[col]), __dmul_rn(s, b.m[3 + col]));
    r[3 + col] = __dadd_rn(__dmul_rn(s, b.m[col]), __dmul_rn(c, b.m[3 + col]));
    r[6 + col] = b.m[6 + col];
  }
}

// Scalar metric of each 6x6 (kernels.py:602-608 _nb_metric_of): 0 det (partial-pivot LU),
// 1 smallest eigenvalue (cyclic Jacobi), 2 trace (diagonal summed left to right).
__global__ void k_metric6(const double* __restrict__ fim, int64_t q, int mid, double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= q) return;
  const double* f = fim + 36 * i;
  if (mid == FIF_METRIC_TRACE) {
    double t = f[0];
#pragma unroll
    for (int k = 1; k < 6; ++k) t = __dadd_rn(t, f[7 * k]);
    out[i] = t;
    return;
  }
  double a[36];
#pragma unroll
  for (int k = 0; k < 36; ++k) a[k] = f[k];
  if (mid == FIF_METRIC_DET) {
    bool ok;
    double inv[36];
    out[i] = det6_core<false>(a, inv, ok);
  } else {
    double v[6];
    out[i] = lmin6_core<false>(a, v);
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
  int64_t cap = (int64_t)num_sms();  // persistent: one CTA (16 warps, ~190 KB smem) per SM
  unsigned blocks = (unsigned)(need < cap ? need : cap);
  const float inv_s2 = (float)(1.0 / (sigma * sigma));
  // landmark tables in Morton order + group boxes: hi[n], lo[n], max |p|_1, boxes[2 ceil(n/32)]
  const int64_t ngroups = (n_points + 31) / 32;
  float4* ptab = nullptr;
  if (cudaMallocAsync(&ptab, sizeof(float4) * (2 * n_points + 1 + 2 * ngroups), st) != cudaSuccess) {
    set_error("fif_pc_fim: cudaMallocAsync failed");
    return FIF_ERR_CUDA;
  }
  unsigned* p1max = reinterpret_cast<unsigned*>(ptab + 2 * n_points);
  float4* gbox = ptab + 2 * n_points + 1;
  cudaMemsetAsync(p1max, 0, sizeof(unsigned), st);
  static const bool no_cull = getenv("FIF_PC_NOCULL") != nullptr;
  int32_t* order = nullptr;
  unsigned char* lbuf = nullptr;
  if (n_points >= 64 && n_points < (int64_t)INT32_MAX) {
    size_t temp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, temp, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (const int32_t*)nullptr, (int32_t*)nullptr, (int)n_points, 0, 30, st);
    const size_t b4 = ((size_t)n_points * 4 + 255) & ~(size_t)255, bp = sizeof(double) * 6 * PK_BLOCKS;
    if (cudaMallocAsync(&lbuf, 4 * b4 + bp + temp, st) != cudaSuccess) {
      cudaFreeAsync(ptab, st);
      set_error("fif_pc_fim: cudaMallocAsync (landmark order) failed");
      return FIF_ERR_CUDA;
    }
    uint32_t* keys = reinterpret_cast<uint32_t*>(lbuf);
    uint32_t* keys2 = reinterpret_cast<uint32_t*>(lbuf + b4);
    int32_t* idx = reinterpret_cast<int32_t*>(lbuf + 2 * b4);
    order = reinterpret_cast<int32_t*>(lbuf + 3 * b4);
    double* part = reinterpret_cast<double*>(lbuf + 4 * b4);
    k_pc_bbox<<<PK_BLOCKS, 256, 0, st>>>(d_points, n_points, part);
    k_pc_mkeys<<<(unsigned)((n_points + 255) / 256), 256, 0, st>>>(d_points, n_points, part, PK_BLOCKS, keys, idx);
    FIF_CHECK_LAUNCH("k_pc_mkeys");
    cub::DeviceRadixSort::SortPairs(lbuf + 4 * b4 + bp, temp, keys, keys2, idx, order, (int)n_points, 0, 30, st);
  }
  k_pc_prep<<<(unsigned)((n_points + 255) / 256), 256, 0, st>>>(d_points, n_points, order, ptab, p1max);
  FIF_CHECK_LAUNCH("k_pc_prep");
  k_pc_groups<<<(unsigned)((ngroups + 127) / 128), 128, 0, st>>>(ptab, n_points, gbox);
  FIF_CHECK_LAUNCH("k_pc_groups");
  if (lbuf) cudaFreeAsync(lbuf, st);
  if (d_mask) cudaMemsetAsync(d_mask, 0, (size_t)q * (size_t)n_points, st);  // the kernel writes the visible pairs
  const size_t smem = sizeof(float4) * (2 * PC_NBUF * PC_TILE + PC_NBUF * 2 * PC_GPT + PC_WARPS * PC_QCAP * 2) +
                      2 * PC_NBUF * sizeof(uint64_t);
  static std::atomic<uint64_t> attr{0};
  if (needs_setup(attr)) {
    for (auto f : {k_pc_fim<true, true>, k_pc_fim<false, true>, k_pc_fim<true, false>, k_pc_fim<false, false>}) {
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    }
    mark_setup(attr);
  }
  // similar poses share a CTA (load balance across its pose warps)
  int32_t* perm = nullptr;
  unsigned char* sbuf = nullptr;
  if (q >= (int64_t)PC_WARPS * num_sms() * 4 && q < (int64_t)INT32_MAX) {
    size_t temp = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, temp, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                    (const int32_t*)nullptr, (int32_t*)nullptr, (int)q, 0, 19, st);
    const size_t b4 = ((size_t)q * 4 + 255) & ~(size_t)255, bp = sizeof(double) * 6 * PK_BLOCKS;
    if (cudaMallocAsync(&sbuf, 4 * b4 + bp + temp, st) != cudaSuccess) {
      cudaFreeAsync(ptab, st);
      set_error("fif_pc_fim: cudaMallocAsync (pose order) failed");
      return FIF_ERR_CUDA;
    }
    uint32_t* keys = reinterpret_cast<uint32_t*>(sbuf);
    uint32_t* keys2 = reinterpret_cast<uint32_t*>(sbuf + b4);
    int32_t* idx = reinterpret_cast<int32_t*>(sbuf + 2 * b4);
    perm = reinterpret_cast<int32_t*>(sbuf + 3 * b4);
    double* part = reinterpret_cast<double*>(sbuf + 4 * b4);
    k_pc_bbox<<<PK_BLOCKS, 256, 0, st>>>(d_t, q, part);
    k_pc_keys<<<(unsigned)((q + 255) / 256), 256, 0, st>>>(d_rot, d_t, q, part, PK_BLOCKS, keys, idx);
    FIF_CHECK_LAUNCH("k_pc_keys");
    cub::DeviceRadixSort::SortPairs(sbuf + 4 * b4 + bp, temp, keys, keys2, idx, perm, (int)q, 0, 19, st);
  }
#define PC_LAUNCH(M, C)                                                                                       \
  k_pc_fim<M, C><<<blocks, (PC_WARPS + 1) * 32, smem, st>>>(d_rot, d_t, q, d_points, ptab, gbox, n_points, *cam, p1max, \
                                                            inv_s2, d_out, d_mask, perm)
  if (d_mask) { if (no_cull) PC_LAUNCH(true, false); else PC_LAUNCH(true, true); }
  else { if (no_cull) PC_LAUNCH(false, false); else PC_LAUNCH(false, true); }
#undef PC_LAUNCH
  if (sbuf) cudaFreeAsync(sbuf, st);
  cudaFreeAsync(ptab, st);
  FIF_CHECK_LAUNCH("k_pc_fim");
  return FIF_OK;
}

extern "C" int fif_pc_metric_yaw(const double* d_positions, const double* d_cos_sin, int64_t q, const double* d_points,
                                 int64_t n_points, const fif_camera* cam, double sigma, const double* r_base, int metric,
                                 double* d_values, double* d_fim, uint8_t* d_mask, void* stream) {
  FIF_CHECK_ARG(cam != nullptr && r_base != nullptr, "fif_pc_metric_yaw: NULL camera / r_base");
  FIF_CHECK_ARG(metric == FIF_METRIC_DET || metric == FIF_METRIC_LMIN || metric == FIF_METRIC_TRACE,
                "fif_pc_metric_yaw: unknown metric %d", metric);
  FIF_CHECK_ARG(q >= 0 && n_points >= 0, "fif_pc_metric_yaw: negative size");
  if (q == 0) return FIF_OK;
  FIF_CHECK_ARG(d_positions && d_cos_sin && d_values, "fif_pc_metric_yaw: NULL pointer");
  cudaStream_t st = (cudaStream_t)stream;
  Mat3 b;
  for (int k = 0; k < 9; ++k) b.m[k] = r_base[k];
  double* buf = nullptr;
  const size_t bytes = sizeof(double) * (size_t)q * (9 + (d_fim ? 0 : 36));
  if (cudaMallocAsync(&buf, bytes, st) != cudaSuccess) {
    set_error("fif_pc_metric_yaw: cudaMallocAsync of %zu bytes failed", bytes);
    return FIF_ERR_CUDA;
  }
  double* rot = buf;
  double* fim = d_fim ? d_fim : buf + 9 * q;
  k_yaw_rot<<<(unsigned)((q + 255) / 256), 256, 0, st>>>(d_cos_sin, q, b, rot);
  FIF_CHECK_LAUNCH("k_yaw_rot");
  int rc = fif_pc_fim(rot, d_positions, q, d_points, n_points, cam, sigma, fim, d_mask, stream);
  if (rc == FIF_OK) {
    k_metric6<<<(unsigned)((q + 127) / 128), 128, 0, st>>>(fim, q, metric, d_values);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      set_error("k_metric6: %s", cudaGetErrorString(e));
      rc = FIF_ERR_CUDA;
    } else {
      count_launch();
    }
  }
  cudaFreeAsync(buf, st);
  return rc;
}
