/*
 * fif_b200.h — C ABI of the B200-native Fisher Information Field hot paths.
 *
 * One shared library (paper_2008_03324_b200/libfif_b200.so), C linkage, no C++
 * exceptions across the boundary.  Every entry point takes caller-allocated
 * DEVICE pointers (e.g. torch tensors' data_ptr()), explicit sizes, a CUDA
 * stream (cudaStream_t passed as void*; NULL = legacy default stream) and
 * returns an int status: FIF_OK (0) or a negative error code, with the message
 * in fif_last_error() (thread-local).  Per-query out-of-field is an OUTPUT
 * (status array), never an error.  The library never frees caller memory.
 *
 * Each function names the reference (fifield 0.1.0, /root/reference/pkg/src/
 * fifield) interface it replaces; INTEGRATION.md shows the ctypes binding a
 * maintainer adds to fifield/kernels.py as a "cuda" backend.
 */
#ifndef FIF_B200_H
#define FIF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FIF_ABI_VERSION 2

/* return codes */
#define FIF_OK 0
#define FIF_ERR_ARG (-1)
#define FIF_ERR_CUDA (-2)
#define FIF_ERR_UNSUPPORTED (-3)

/* factor kinds (field.py:37 _FACTOR_CODES) */
#define FIF_KIND_INFO 0
#define FIF_KIND_TRACE 1
/* visibility models (field.py:39-40) */
#define FIF_MODEL_QUAD 1
#define FIF_MODEL_GP 2
/* query modes (field.py:42) */
#define FIF_MODE_NEAREST 0
#define FIF_MODE_TRILINEAR 1
/* per-query status (kernels.py:50-51) */
#define FIF_STATUS_OK 0
#define FIF_STATUS_OUT_OF_FIELD 1
/* fif_query output selection flags */
#define FIF_Q_TRACE 1u     /* tr(I) (trace field: vr . row; info field: trace of the contraction) */
#define FIF_Q_FULL 2u      /* full 6x6 information (info fields only)                            */
#define FIF_Q_GRAD 4u      /* analytic d/d[t; theta] of every requested output                   */
#define FIF_Q_DET 8u       /* det(I), blended per corner like kernels.py:1456-1468 (info only)   */
#define FIF_Q_LMIN 16u     /* smallest eigenvalue, blended per corner (info only)                */
#define FIF_Q_FIELD_F64 32u /* GP field operand is the FP64 S array instead of the FP32 copy     */
/* fif_build flags */
#define FIF_BUILD_EXACT 1u  /* quad: reproduce _nb_build_quad's FP64 operation order bit for bit     */
#define FIF_BUILD_SIMT 2u   /* GP info: FP32 SIMT (FFMA2) kernel instead of the tensor-pipe kernel   */
#define FIF_BUILD_TF32 4u   /* GP info: TF32x3 mma.sync kernel instead of the default tcgen05 one       */
#define FIF_BUILD_H16 8u    /* GP info: FP16-split mma.sync kernel instead of the default tcgen05 one  */
#define FIF_BUILD_T6 16u    /* GP info: k_gp_info_t6 (sigmoid exponent arguments on the tensor cores as well;
                               unmasked builds with 9 <= N_s <= 72, else the default kernel; measured slower
                               than the default k_gp_info_t5: DESIGN 8b) */

/* Axis-aligned voxel grid (field.py:45-98 GridConfig). */
typedef struct fif_grid {
  double origin[3];
  double voxel_size;
  int64_t dims[3];
} fif_grid;

/* Visibility model parameters (visibility.py QuadraticVisibility / GpVisibility).
 * zs / kinv are DEVICE pointers (N_s x 3 and N_s x N_s float64, row-major).      */
typedef struct fif_model {
  int32_t kind;      /* FIF_MODEL_QUAD or FIF_MODEL_GP                      */
  int32_t n_v;       /* 10 (quad) or N_s (GP)                               */
  double k2, k1, k0; /* quad coefficients (visibility.py:56-68)             */
  double k_s;        /* GP sigmoid sharpness (visibility.py:30)             */
  double cos_alpha;  /* cos(half FoV)                                       */
  double sig2, ell;  /* SE kernel sigma^2 and length scale (visibility.py:71-86) */
  const double* zs;  /* device (N_s,3) sample directions                    */
  const double* kinv;/* device (N_s,N_s) inverse Gram matrix                */
  const double* zs_host; /* optional host copy of zs: the sample directions become kernel
                            parameters of the tcgen05 GP-info build (NULL: mma.sync kernel) */
} fif_model;

/* Pinhole camera (fim.py:28-68), pixels. */
typedef struct fif_camera {
  double fx, fy, cx, cy, width, height;
} fif_camera;

int fif_abi_version(void);
const char* fif_last_error(void);

/* Voxel centres origin + (idx + 0.5) * voxel_size, bit-identical to
 * GridConfig.centers (field.py:74-79).  order 0: reference x-major / z-minor
 * linear index; order 1: internal z-major index.  Rows [v_begin, v_end).     */
int fif_grid_centers(const fif_grid* grid, int order, int64_t v_begin, int64_t v_end, double* d_out,
                     void* stream);

/* Bytes of device scratch fif_build needs for n_points landmarks. */
int64_t fif_build_scratch_bytes(int64_t n_points);

/* Field build — replaces kernels.build_quad_factors (kernels.py:1576-1582) and
 * kernels.build_gp_factors (kernels.py:1585-1590), i.e. the voxel x landmark
 * loops of _nb_build_quad (427-468) and _nb_build_gp (471-524).
 *
 * Voxels: if d_centers != NULL, rows [v_begin, v_end) of that (V,3) float64
 * array; else the grid's voxels with INTERNAL z-major indices [v_begin, v_end)
 * (a contiguous z-slab; the sharding unit).  Optional d_mask: (v_end-v_begin, N)
 * uint8 matchability mask (field.py:143-177), 0 = pair skipped.
 * Output d_out64 (rows = v_end - v_begin):
 *   quad trace (rows,10) f64 | quad info (rows,10,21) f64 packed upper-triangle,
 *   GP trace (rows,N_s) f64 S | GP info (rows,N_s,21) f64 S, where
 *   S = sum_i vs_i (x) I_i is the pre-kinv factor (reference factor = kinv @ S).
 * Optional d_out32: the same array in float32 (the query operand for GP).
 * d_scratch: fif_build_scratch_bytes(n_points) bytes.  build_flags:
 * FIF_BUILD_EXACT (quad only) selects the bit-exact reference arithmetic; the
 * FIF_BUILD_SIMT / TF32 / H16 / T6 flags select alternative GP info kernels (all
 * within the same tolerance; 0 = the fastest, k_gp_info_t5).                  */
int fif_build(int factor_kind, const fif_model* model, const double* d_points, int64_t n_points,
              const fif_grid* grid, const double* d_centers, int64_t v_begin, int64_t v_end,
              const uint8_t* d_mask, double sigma, uint32_t build_flags, void* d_scratch, double* d_out64,
              float* d_out32, void* stream);

/* Reference-layout rows (kernels.py:18-20): quad info expands the packed
 * upper triangle to 36 per block; GP rows become kinv @ S (FP64); trace rows
 * of quad are copied.  Row order is preserved.                                */
int fif_export_reference(int factor_kind, const fif_model* model, const double* d_in64, int64_t rows,
                         double* d_out, void* stream);

/* Batched pose query — replaces kernels.query_fim_batch_quad/gp
 * (kernels.py:1648-1677) and field_metric_yaw_batch_quad/gp (1707-1728),
 * plus the analytic pose gradient, which the reference lacks.
 * d_field: f64 rows (quad) or f32 S rows (GP; f64 with FIF_Q_FIELD_F64) laid
 * out as fif_build writes them.  d_slots: NULL for a dense internal z-major
 * field, else the (prod(dims),) int32 map from the reference linear index to
 * a row (-1 = empty voxel, reads as zero; field.py:264-266).
 * Inputs: positions (Q,3) f64, optical axes z = R[:,2] (Q,3) f64.
 * Outputs (each optional, NULL = not written):
 *   d_trace (Q) | d_trace_grad (Q,6) | d_fim (Q,36) | d_fim_grad (Q,6,36) |
 *   d_det (Q) | d_lmin (Q) | d_status (Q) uint8.
 * Gradient convention: d/d[t(3); theta(3)] with t' = t + dt, R' = exp(dtheta^) R.
 * lambda_min gradients (fif_query_ex) go through the eigenvector, whose sensitivity
 * to the FP32 copy grows like 1/gap: pass the f64 rows with FIF_Q_FIELD_F64 for
 * them (the Python Field does so automatically).                                */
int fif_query(int factor_kind, const fif_model* model, const fif_grid* grid, const void* d_field,
              const int32_t* d_slots, const double* d_positions, const double* d_axes, int64_t q, int mode,
              uint32_t flags, double* d_trace, double* d_trace_grad, double* d_fim, double* d_fim_grad,
              double* d_det, double* d_lmin, uint8_t* d_status, void* stream);

/* Output set of fif_query_ex; every pointer is optional (NULL = not written).
 * Shapes as in fif_query, plus d/d[t; theta] of the blended metrics:
 *   det_grad (Q,6), lmin_grad (Q,6)  (with FIF_Q_GRAD and FIF_Q_DET / FIF_Q_LMIN).
 * Per corner: d det F = det F tr(F^-1 dF) (0 for a singular corner),
 * d lambda_min = v^T dF v (v the unit eigenvector); blended like the values.  */
typedef struct fif_query_out {
  double* trace;
  double* trace_grad;
  double* fim;
  double* fim_grad;
  double* det;
  double* det_grad;
  double* lmin;
  double* lmin_grad;
  uint8_t* status;
} fif_query_out;

/* fif_query with the output set passed as a struct (adds the metric gradients). */
int fif_query_ex(int factor_kind, const fif_model* model, const fif_grid* grid, const void* d_field,
                 const int32_t* d_slots, const double* d_positions, const double* d_axes, int64_t q, int mode,
                 uint32_t flags, const fif_query_out* out, void* stream);

/* fif_query_ex with the trace outputs of an INFO field taken from d_trace_rows: its FP64
 * trace table (rows, n_v), T[r][k] = sum of the 6 diagonal entries of block k of the row
 * (the per-sample trace kernels.py:1414-1423 contracts).  With the FP32 GP query copy the
 * trace of the contraction cancels (omega = kinv v^r alternates in sign: measured 3.2e-4
 * relative on config-2 nearest queries, over the 1e-4 tolerance), so the trace is
 * contracted from FP64 rows (+8 n_v bytes per corner) while the 6x6, det and lambda_min
 * stream the FP32 rows; one prep serves both.  d_trace_rows NULL = fif_query_ex.      */
int fif_query_ex2(int factor_kind, const fif_model* model, const fif_grid* grid, const void* d_field,
                  const double* d_trace_rows, const int32_t* d_slots, const double* d_positions, const double* d_axes,
                  int64_t q, int mode, uint32_t flags, const fif_query_out* out, void* stream);

/* Point-cloud brute force — replaces kernels.exact_fim_batch
 * (kernels.py:1638-1645 -> _nb_exact_fim 571-599).  R (Q,9) row-major
 * world-from-camera rotations, t (Q,3), landmarks (N,3), all f64.
 * d_out (Q,36) f64.  Optional d_mask (Q,N) uint8: the exact-visibility mask
 * (bit-exact with the reference's FP64 test).                                 */
int fif_pc_fim(const double* d_rot, const double* d_t, int64_t q, const double* d_points, int64_t n_points,
               const fif_camera* cam, double sigma, double* d_out, uint8_t* d_mask, void* stream);

/* Scalar information metrics (kernels.py:602-608 _nb_metric_of / metric_id). */
#define FIF_METRIC_DET 0
#define FIF_METRIC_LMIN 1
#define FIF_METRIC_TRACE 2

/* Exact point-cloud metric at yaw-only poses — replaces kernels.pc_metric_yaw_batch
 * (kernels.py:1599-1606 -> _nb_pc_metric_yaw_batch 611-625), the exact comparator behind
 * rrt.ExactInfoRepr.metric_batch (rrt.py:54-71).  Per pose: R = Rz(yaw) r_base with the
 * reference's operation order, the point-cloud 6x6 of fif_pc_fim, then det / lambda_min /
 * trace.  d_positions (Q,3) f64; d_cos_sin (Q,2) f64 = cos, sin of each yaw, computed on
 * the HOST (libm, like np.cos / np.sin; the device's cos / sin would move mask bits);
 * r_base: HOST (3,3) row-major (rrt.R_CAM_MOUNT).  d_values (Q) f64.  Optional d_fim
 * (Q,36) and d_mask (Q,N) as in fif_pc_fim.                                            */
int fif_pc_metric_yaw(const double* d_positions, const double* d_cos_sin, int64_t q, const double* d_points,
                      int64_t n_points, const fif_camera* cam, double sigma, const double* r_base, int metric,
                      double* d_values, double* d_fim, uint8_t* d_mask, void* stream);

/* Corner table of a batch of positions — the bit-exact indexing rule of the queries as a
 * debug / parity entry point: kernels._nb_locate_nearest (kernels.py:628-635) and the
 * trilinear corner block of _nb_query_fim (678-702; twin _np_trilinear_corners 247-272).
 * d_index (Q,8) int64: the reference's x-major linear voxel indices (field.py:81-83);
 * d_weight (Q,8) f64; d_status (Q) uint8 (FIF_STATUS_*).  Nearest: corner 0 only
 * (weight 1), the other seven -1 / 0; out of field: all eight -1 / 0.  d_index and
 * d_weight are optional.                                                              */
int fif_locate(const fif_grid* grid, const double* d_positions, int64_t q, int mode, int64_t* d_index,
               double* d_weight, uint8_t* d_status, void* stream);

/* Matchability gates — replaces Matchability.mask (field.py:143-177) for range, view
 * cone and ObstacleWorld occlusion (world.segment_blocked, world.py:96-140).  d_mask (rows, n_points) uint8, row-major:
 * 1 = the (centre, landmark) pair contributes.  FP64, bit-identical with the
 * reference's numpy arithmetic (norm order (x^2 + y^2) + z^2; einsum order
 * (x + z) + y; occlusion as fif_gate.cuh documents).  Python predicates stay on
 * the host, as in the reference.                                               */
#define FIF_MATCH_NEAR 1u  /* dist >= d_near     */
#define FIF_MATCH_FAR 2u   /* dist <= d_far      */
#define FIF_MATCH_CONE 4u  /* cos(angle to view_dir) >= cos_beta (needs d_view_dirs (N,3)) */
#define FIF_MATCH_OCCLUDE 8u /* sight line centre -> landmark not blocked (world.segment_blocked) */
typedef struct fif_match {
  double d_near;
  double d_far;
  double cos_beta;
  uint32_t flags;
  /* occluders of an ObstacleWorld (world.py:18-56), DEVICE arrays:
   * spheres (n_spheres, 4) = centre xyz, radius; boxes (n_boxes, 6) = lo xyz, hi xyz */
  const double* spheres;
  int64_t n_spheres;
  const double* boxes;
  int64_t n_boxes;
} fif_match;
int fif_match_mask(const fif_match* match, const double* d_centers, int64_t rows, const double* d_points,
                   const double* d_view_dirs, int64_t n_points, uint8_t* d_mask, void* stream);

/* Per-centre occupancy under the gates: d_any (rows) uint8, 1 iff some landmark matches
 * (the reference gives a voxel a row iff its mask row has a 1, field.py:253-257).       */
int fif_match_any(const fif_match* match, const double* d_centers, int64_t rows, const double* d_points,
                  const double* d_view_dirs, int64_t n_points, uint8_t* d_any, void* stream);

/* Matchability-gated build with the gates FUSED into the build kernels' pair loops (no
 * (V, N) mask is materialised) — replaces the masked path of Field.build (field.py:229-268:
 * Matchability.mask, then build_*_factors(..., mask)).  Voxels: the (rows, 3) f64 centres
 * (normally the occupied voxels from fif_match_any, in the reference's row order).  Output
 * layout and d_scratch as fif_build.  match->flags == 0 builds unmasked.                  */
int fif_build_matched(int factor_kind, const fif_model* model, const double* d_points, int64_t n_points,
                      const double* d_centers, int64_t rows, const fif_match* match, const double* d_view_dirs,
                      double sigma, uint32_t build_flags, void* d_scratch, double* d_out64, float* d_out32,
                      void* stream);

/* Number of kernel launches issued by this library since load (for bench
 * accounting of gpu_launches). */
int64_t fif_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* FIF_B200_H */
