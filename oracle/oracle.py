"""ctypes front end of the C oracle (fif_oracle.c) — TEST INFRASTRUCTURE ONLY.

Mirrors the reference kernel boundary (`fifield.kernels`, kernels.py:1559-1732):
plain float64 arrays in, arrays out, integer status codes.  Only tests/,
__graft_entry__.smoke() and bench.py's CPU legs may import this module.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libfif_oracle.so")
_FAST_PATH = os.path.join(_HERE, "libfif_cpu_fast.so")
_lib = None
_fast = None

_d = ctypes.c_double
_i64 = ctypes.c_int64
_int = ctypes.c_int
_p = ctypes.c_void_p


def build() -> str:
    """Compile the oracle (make in oracle/). Idempotent."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.or_fim_flat.restype = _d
        L.or_fim_flat.argtypes = [_d] * 7 + [_p]
        L.or_build_quad.argtypes = [_p, _i64, _p, _i64, _d, _d, _d, _d, _int, _p, _p, _int]
        L.or_build_gp.argtypes = [_p, _i64, _p, _i64, _d, _p, _int, _p, _d, _d, _int, _p, _p, _int]
        L.or_exact_fim_batch.argtypes = [_p, _p, _i64, _p, _i64] + [_d] * 7 + [_p, _int]
        L.or_pc_mask.argtypes = [_p, _p, _i64, _p, _i64] + [_d] * 6 + [_p, _int]
        L.or_locate_nearest.restype = _i64
        L.or_locate_nearest.argtypes = [_p, _d, _p, _p]
        L.or_trilinear.restype = _int
        L.or_trilinear.argtypes = [_p, _d, _p, _p, _p, _p]
        L.or_centers.argtypes = [_p, _d, _p, _p]
        L.or_query_fim_batch.argtypes = [_p, _p, _i64, _p, _d, _p, _p, _p, _i64, _int, _d, _d, _d, _p, _int, _d,
                                         _d, _int, _p, _p, _int]
        L.or_metric_batch.argtypes = [_p, _p, _i64, _p, _d, _p, _p, _p, _i64, _int, _d, _d, _d, _p, _int, _d, _d,
                                      _int, _int, _int, _p, _p, _int]
        L.or_metric_of.restype = _d
        L.or_metric_of.argtypes = [_p, _int]
        L.or_openmp_max_threads.restype = _int
        _lib = L
    return _lib


def fast_lib():
    """The blocked / vectorised CPU port of the GP build (bench CPU legs only)."""
    global _fast
    if _fast is None:
        if not os.path.exists(_FAST_PATH):
            build()
        L = ctypes.CDLL(_FAST_PATH)
        L.fp_build_gp.argtypes = [_p, _i64, _p, _i64, _d, _p, _int, _p, _d, _d, _int, _p, _int]
        _fast = L
    return _fast


def build_gp_factors_fast(centers, points, sigma, zs, kinv, ks, cos_alpha, want_trace, nthreads=0):
    """The reference GP build (kernels.py:471-524) as a fast CPU port (no mask)."""
    c, p = _c(centers).reshape(-1, 3), _c(points).reshape(-1, 3)
    zs, kinv = _c(zs), _c(kinv)
    ns = zs.shape[0]
    out = np.empty((c.shape[0], ns if want_trace else 36 * ns))
    fast_lib().fp_build_gp(_ptr(c), c.shape[0], _ptr(p), p.shape[0], float(sigma), _ptr(zs), ns, _ptr(kinv),
                           float(ks), float(cos_alpha), int(bool(want_trace)), _ptr(out), int(nthreads))
    return out


def _c(a, dtype=np.float64):
    return np.ascontiguousarray(a, dtype=dtype)


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def max_threads() -> int:
    return int(lib().or_openmp_max_threads())


def centers(origin, voxel_size, dims):
    origin, dims = _c(origin), _c(dims, np.int64)
    out = np.empty((int(np.prod(dims)), 3))
    lib().or_centers(_ptr(origin), float(voxel_size), _ptr(dims), _ptr(out))
    return out


def fim_flat(p, t, inv_s2):
    out = np.empty(36)
    tr = lib().or_fim_flat(*map(float, p), *map(float, t), float(inv_s2), _ptr(out))
    return out.reshape(6, 6), tr


def build_quad_factors(centers, points, sigma, k2, k1, k0, want_trace, mask=None, nthreads=0):
    """kernels.build_quad_factors (kernels.py:1576) — (V,10) or (V,360) float64."""
    c, p = _c(centers).reshape(-1, 3), _c(points).reshape(-1, 3)
    m = _c(mask, np.uint8) if mask is not None else None
    out = np.empty((c.shape[0], 10 if want_trace else 360))
    lib().or_build_quad(_ptr(c), c.shape[0], _ptr(p), p.shape[0], float(sigma), float(k2), float(k1), float(k0),
                        int(bool(want_trace)), _ptr(m), _ptr(out), int(nthreads))
    return out


def build_gp_factors(centers, points, sigma, zs, kinv, ks, cos_alpha, want_trace, mask=None, nthreads=0):
    """kernels.build_gp_factors (kernels.py:1585) — (V,Ns) or (V,36 Ns) float64."""
    c, p = _c(centers).reshape(-1, 3), _c(points).reshape(-1, 3)
    zs, kinv = _c(zs), _c(kinv)
    ns = zs.shape[0]
    m = _c(mask, np.uint8) if mask is not None else None
    out = np.empty((c.shape[0], ns if want_trace else 36 * ns))
    lib().or_build_gp(_ptr(c), c.shape[0], _ptr(p), p.shape[0], float(sigma), _ptr(zs), ns, _ptr(kinv), float(ks),
                      float(cos_alpha), int(bool(want_trace)), _ptr(m), _ptr(out), int(nthreads))
    return out


def exact_fim_batch(rots, ts, points, camera, sigma=1.0, nthreads=0):
    """kernels.exact_fim_batch (kernels.py:1638) — (Q,6,6); camera = (fx,fy,cx,cy,w,h)."""
    r, t, p = _c(rots).reshape(-1, 9), _c(ts).reshape(-1, 3), _c(points).reshape(-1, 3)
    out = np.empty((t.shape[0], 36))
    fx, fy, cx, cy, w, h = map(float, camera)
    lib().or_exact_fim_batch(_ptr(r), _ptr(t), t.shape[0], _ptr(p), p.shape[0], fx, fy, cx, cy, w, h,
                             float(sigma), _ptr(out), int(nthreads))
    return out.reshape(-1, 6, 6)


def pc_mask(rots, ts, points, camera, nthreads=0):
    r, t, p = _c(rots).reshape(-1, 9), _c(ts).reshape(-1, 3), _c(points).reshape(-1, 3)
    out = np.empty((t.shape[0], p.shape[0]), dtype=np.uint8)
    fx, fy, cx, cy, w, h = map(float, camera)
    lib().or_pc_mask(_ptr(r), _ptr(t), t.shape[0], _ptr(p), p.shape[0], fx, fy, cx, cy, w, h, _ptr(out),
                     int(nthreads))
    return out.astype(bool)


def locate_nearest(origin, voxel_size, dims, pos):
    origin, dims, pos = _c(origin), _c(dims, np.int64), _c(pos)
    return int(lib().or_locate_nearest(_ptr(origin), float(voxel_size), _ptr(dims), _ptr(pos)))


def trilinear(origin, voxel_size, dims, pos):
    origin, dims, pos = _c(origin), _c(dims, np.int64), _c(pos)
    idx = np.empty(8, dtype=np.int64)
    w = np.empty(8)
    st = lib().or_trilinear(_ptr(origin), float(voxel_size), _ptr(dims), _ptr(pos), _ptr(idx), _ptr(w))
    return (idx, w) if st == 0 else None


def _model_args(model):
    """model: ('quad', k2, k1, k0) or ('gp', zs, sig2, ell)."""
    if model[0] == "quad":
        return 1, float(model[1]), float(model[2]), float(model[3]), None, 0, 0.0, 1.0
    zs = _c(model[1])
    return 2, 0.0, 0.0, 0.0, zs, zs.shape[0], float(model[2]), float(model[3])


def query_fim_batch(slots, factors, origin, voxel_size, dims, positions, axes, model, trilinear, nthreads=0):
    """kernels.query_fim_batch_quad/gp (kernels.py:1648-1677) -> (fims (Q,6,6), status (Q,))."""
    slots, factors = _c(slots, np.int32), _c(factors)
    origin, dims = _c(origin), _c(dims, np.int64)
    pos, ax = _c(positions).reshape(-1, 3), _c(axes).reshape(-1, 3)
    kind, k2, k1, k0, zs, ns, sig2, ell = _model_args(model)
    out = np.empty((pos.shape[0], 36))
    st = np.empty(pos.shape[0], dtype=np.int64)
    lib().or_query_fim_batch(_ptr(slots), _ptr(factors), factors.shape[1], _ptr(origin), float(voxel_size),
                             _ptr(dims), _ptr(pos), _ptr(ax), pos.shape[0], kind, k2, k1, k0, _ptr(zs), ns, sig2,
                             ell, int(bool(trilinear)), _ptr(out), _ptr(st), int(nthreads))
    return out.reshape(-1, 6, 6), st


def metric_batch(slots, factors, origin, voxel_size, dims, positions, axes, model, metric, is_trace, trilinear,
                 nthreads=0):
    """kernels.field_metric_yaw_batch_quad/gp (kernels.py:1707-1728) -> (values, status)."""
    mid = {"det": 0, "lmin": 1, "trace": 2}[metric]
    slots, factors = _c(slots, np.int32), _c(factors)
    origin, dims = _c(origin), _c(dims, np.int64)
    pos, ax = _c(positions).reshape(-1, 3), _c(axes).reshape(-1, 3)
    kind, k2, k1, k0, zs, ns, sig2, ell = _model_args(model)
    vals = np.empty(pos.shape[0])
    st = np.empty(pos.shape[0], dtype=np.int64)
    lib().or_metric_batch(_ptr(slots), _ptr(factors), factors.shape[1], _ptr(origin), float(voxel_size),
                          _ptr(dims), _ptr(pos), _ptr(ax), pos.shape[0], kind, k2, k1, k0, _ptr(zs), ns, sig2,
                          ell, mid, int(bool(is_trace)), int(bool(trilinear)), _ptr(vals), _ptr(st), int(nthreads))
    return vals, st


def metric_of(fim, metric):
    f = _c(fim).reshape(36)
    return float(lib().or_metric_of(_ptr(f), {"det": 0, "lmin": 1, "trace": 2}[metric]))
