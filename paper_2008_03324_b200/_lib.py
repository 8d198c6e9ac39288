"""ctypes binding of libfif_b200.so — the C ABI declared in include/fif_b200.h.

Fails loudly: there is no CPU fallback.  If the library is missing it is built
in-tree with nvcc (which only works where the CUDA toolkit is installed); if a
CUDA device is absent, every compute entry point raises.
"""
from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from ._build import LIB, build

FIF_OK = 0
KIND_INFO, KIND_TRACE = 0, 1
MODEL_QUAD, MODEL_GP = 1, 2
MODE_NEAREST, MODE_TRILINEAR = 0, 1
Q_TRACE, Q_FULL, Q_GRAD, Q_DET, Q_LMIN, Q_FIELD_F64 = 1, 2, 4, 8, 16, 32
BUILD_EXACT = 1
BUILD_SIMT = 2
BUILD_TF32 = 4
BUILD_H16 = 8
BUILD_T6 = 16
METRIC_IDS = {"det": 0, "lmin": 1, "trace": 2}  # kernels.metric_id (kernels.py:602-608)

EXPORTED = (
    "fif_abi_version", "fif_last_error", "fif_grid_centers", "fif_build_scratch_bytes", "fif_build",
    "fif_export_reference", "fif_query", "fif_query_ex", "fif_pc_fim", "fif_match_mask",
    "fif_launch_count", "fif_locate", "fif_pc_metric_yaw", "fif_match_any", "fif_build_matched",
    "fif_query_ex2",
)


class FifCudaError(RuntimeError):
    """A libfif_b200 entry point returned a non-zero status."""


class Grid(ctypes.Structure):
    _fields_ = [("origin", ctypes.c_double * 3), ("voxel_size", ctypes.c_double), ("dims", ctypes.c_int64 * 3)]


class Model(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32), ("n_v", ctypes.c_int32),
        ("k2", ctypes.c_double), ("k1", ctypes.c_double), ("k0", ctypes.c_double),
        ("k_s", ctypes.c_double), ("cos_alpha", ctypes.c_double),
        ("sig2", ctypes.c_double), ("ell", ctypes.c_double),
        ("zs", ctypes.c_void_p), ("kinv", ctypes.c_void_p), ("zs_host", ctypes.c_void_p),
    ]


class QueryOut(ctypes.Structure):
    """fif_query_out: device output pointers of fif_query_ex (NULL = not written)."""
    _fields_ = [(n, ctypes.c_void_p) for n in ("trace", "trace_grad", "fim", "fim_grad", "det", "det_grad",
                                                 "lmin", "lmin_grad", "status")]


class Match(ctypes.Structure):
    _fields_ = [("d_near", ctypes.c_double), ("d_far", ctypes.c_double), ("cos_beta", ctypes.c_double),
                ("flags", ctypes.c_uint32), ("spheres", ctypes.c_void_p), ("n_spheres", ctypes.c_int64),
                ("boxes", ctypes.c_void_p), ("n_boxes", ctypes.c_int64)]


MATCH_NEAR, MATCH_FAR, MATCH_CONE, MATCH_OCCLUDE = 1, 2, 4, 8


class Camera(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in ("fx", "fy", "cx", "cy", "width", "height")]


_lib = None
_lock = threading.Lock()
_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_int = ctypes.c_int
_d = ctypes.c_double


def load():
    """Load (building first if needed) and type the shared library."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB):
            build()
        L = ctypes.CDLL(LIB)
        L.fif_abi_version.restype = _int
        L.fif_last_error.restype = ctypes.c_char_p
        L.fif_launch_count.restype = _i64
        L.fif_build_scratch_bytes.restype = _i64
        L.fif_build_scratch_bytes.argtypes = [_i64]
        L.fif_grid_centers.restype = _int
        L.fif_grid_centers.argtypes = [ctypes.POINTER(Grid), _int, _i64, _i64, _p, _p]
        L.fif_build.restype = _int
        L.fif_build.argtypes = [_int, ctypes.POINTER(Model), _p, _i64, ctypes.POINTER(Grid), _p, _i64, _i64, _p, _d,
                                ctypes.c_uint32, _p, _p, _p, _p]
        L.fif_export_reference.restype = _int
        L.fif_export_reference.argtypes = [_int, ctypes.POINTER(Model), _p, _i64, _p, _p]
        L.fif_query.restype = _int
        L.fif_query.argtypes = [_int, ctypes.POINTER(Model), ctypes.POINTER(Grid), _p, _p, _p, _p, _i64, _int,
                                ctypes.c_uint32, _p, _p, _p, _p, _p, _p, _p, _p]
        L.fif_query_ex.restype = _int
        L.fif_query_ex.argtypes = [_int, ctypes.POINTER(Model), ctypes.POINTER(Grid), _p, _p, _p, _p, _i64, _int,
                                   ctypes.c_uint32, ctypes.POINTER(QueryOut), _p]
        L.fif_match_mask.restype = _int
        L.fif_match_mask.argtypes = [ctypes.POINTER(Match), _p, _i64, _p, _p, _i64, _p, _p]
        L.fif_pc_fim.restype = _int
        L.fif_pc_fim.argtypes = [_p, _p, _i64, _p, _i64, ctypes.POINTER(Camera), _d, _p, _p, _p]
        L.fif_locate.restype = _int
        L.fif_locate.argtypes = [ctypes.POINTER(Grid), _p, _i64, _int, _p, _p, _p, _p]
        L.fif_pc_metric_yaw.restype = _int
        L.fif_pc_metric_yaw.argtypes = [_p, _p, _i64, _p, _i64, ctypes.POINTER(Camera), _d,
                                        ctypes.POINTER(ctypes.c_double * 9), _int, _p, _p, _p, _p]
        L.fif_query_ex2.restype = _int
        L.fif_query_ex2.argtypes = [_int, ctypes.POINTER(Model), ctypes.POINTER(Grid), _p, _p, _p, _p, _p, _i64, _int,
                                    ctypes.c_uint32, ctypes.POINTER(QueryOut), _p]
        L.fif_match_any.restype = _int
        L.fif_match_any.argtypes = [ctypes.POINTER(Match), _p, _i64, _p, _p, _i64, _p, _p]
        L.fif_build_matched.restype = _int
        L.fif_build_matched.argtypes = [_int, ctypes.POINTER(Model), _p, _i64, _p, _i64, ctypes.POINTER(Match), _p, _d,
                                        ctypes.c_uint32, _p, _p, _p, _p]
        if L.fif_abi_version() != 2:
            raise FifCudaError(f"libfif_b200 ABI {L.fif_abi_version()} != 2")
        _lib = L
        return L


def check(status: int, what: str) -> None:
    if status != FIF_OK:
        msg = load().fif_last_error().decode(errors="replace")
        raise FifCudaError(f"{what} failed (status {status}): {msg}")


def launch_count() -> int:
    return int(load().fif_launch_count())


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None passes NULL)."""
    if t is None:
        return None
    return t.data_ptr()


def make_grid(origin, voxel_size, dims) -> Grid:
    g = Grid()
    o = np.asarray(origin, dtype=np.float64).reshape(3)
    d = np.asarray(dims, dtype=np.int64).reshape(3)
    for a in range(3):
        g.origin[a] = float(o[a])
        g.dims[a] = int(d[a])
    g.voxel_size = float(voxel_size)
    return g


def make_camera(cam_tuple) -> Camera:
    c = Camera()
    c.fx, c.fy, c.cx, c.cy, c.width, c.height = map(float, cam_tuple)
    return c
