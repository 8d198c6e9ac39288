"""GPU-resident Fisher Information Field — drop-in for fifield/field.py.

Build (field.py:229-268 -> kernels.build_*_factors) runs the sm_100a N-body
kernels of csrc/fif_build.cu; queries (field.py:313-457 -> kernels.query_* /
field_metric_*) run the warp-per-query kernel of csrc/fif_query.cu.  The public
surface — GridConfig, Matchability, Field.build / query_fim / query_fim_batch /
query_metric / metric_axis_batch / query_factor / add|remove|update_landmark /
memory_stats / serialize / deserialize and the slots / factors /
occupied_index3 attributes — matches the reference, so callers switch by import.

Device storage:
  * ALWAYS_MATCH fields are dense: one row per voxel in INTERNAL z-major order
    j = (iz*ny + iy)*nx + ix, so a z-slab is a contiguous row range (the
    multi-GPU shard unit).  `slots` maps the reference's x-major linear index to
    these rows, exactly like the reference's own slots array.
  * Matchability-masked fields keep the reference's occupied-row order and a
    device copy of `slots`.
  * quad: FP64 rows (n_v, 21 packed upper triangle) or (n_v,);
    GP: pre-kinv sums S = sum_i vs_i (x) I_i, FP64 master plus the FP32 copy the
    query kernel streams; queries form omega = kinv v^r in FP64.
  `factors` materialises the reference layout (kernels.py:18-20; GP: kinv @ S)
  on demand.
"""
from __future__ import annotations

import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import _device, _lib
from .errors import BadMagic, EmptyGrid, OutOfField, TruncatedFile, VersionMismatch, WrongFactorKind
from .fim import DEFAULT_SIGMA
from .geometry import Pose
from .visibility import GpVisibility, QuadraticVisibility, SeKernelParams, gp_build, model_from_reference

MAGIC = b"FIF1"
FORMAT_VERSION = 1
_FACTOR_CODES = {"info": 0, "trace": 1}
_FACTOR_NAMES = {v: k for k, v in _FACTOR_CODES.items()}
_MODEL_QUAD, _MODEL_GP = 1, 2
_MODES = ("nearest", "trilinear")
_PACK_R = np.array([0, 0, 0, 0, 0, 0, 1, 1, 1, 1, 1, 2, 2, 2, 2, 3, 3, 3, 4, 4, 5])
_PACK_C = np.array([0, 1, 2, 3, 4, 5, 1, 2, 3, 4, 5, 2, 3, 4, 5, 3, 4, 5, 4, 5, 5])
_PACK36 = _PACK_R * 6 + _PACK_C  # flat 6x6 position of each packed entry


@dataclass(frozen=True)
class GridConfig:
    """Axis-aligned voxel grid: min corner, voxel edge, voxel counts (field.py:45-98)."""

    origin: np.ndarray
    voxel_size: float
    dims: np.ndarray

    def __post_init__(self) -> None:
        origin = np.asarray(self.origin, dtype=np.float64).reshape(3).copy()
        dims = np.asarray(self.dims, dtype=np.int64).reshape(3).copy()
        if self.voxel_size <= 0:
            raise ValueError("voxel_size must be positive")
        if (dims < 1).any():
            raise EmptyGrid(f"dims {dims.tolist()} contain an empty axis")
        origin.flags.writeable = False
        dims.flags.writeable = False
        object.__setattr__(self, "origin", origin)
        object.__setattr__(self, "dims", dims)
        object.__setattr__(self, "voxel_size", float(self.voxel_size))

    @property
    def voxel_count(self) -> int:
        return int(np.prod(self.dims))

    @property
    def extent(self) -> np.ndarray:
        return self.dims * self.voxel_size

    def centers(self) -> np.ndarray:
        """(V,3) centres in the reference's x-major / z-minor order."""
        nx, ny, nz = (int(d) for d in self.dims)
        ix, iy, iz = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
        idx = np.stack([ix, iy, iz], axis=-1).reshape(-1, 3)
        return self.origin + (idx + 0.5) * self.voxel_size

    def linear_index(self, index3) -> np.ndarray:
        i = np.asarray(index3, dtype=np.int64)
        return (i[..., 0] * self.dims[1] + i[..., 1]) * self.dims[2] + i[..., 2]

    def index3_of(self, linear) -> np.ndarray:
        lin = np.asarray(linear, dtype=np.int64)
        iz = lin % self.dims[2]
        rest = lin // self.dims[2]
        return np.stack([rest // self.dims[1], rest % self.dims[1], iz], axis=-1)

    def internal_index(self, index3) -> np.ndarray:
        """Row of a voxel in the dense z-major device layout."""
        i = np.asarray(index3, dtype=np.int64)
        return (i[..., 2] * self.dims[1] + i[..., 1]) * self.dims[0] + i[..., 0]

    def index3_of_internal(self, j) -> np.ndarray:
        j = np.asarray(j, dtype=np.int64)
        ix = j % self.dims[0]
        rest = j // self.dims[0]
        return np.stack([ix, rest % self.dims[1], rest // self.dims[1]], axis=-1)

    def contains(self, position) -> bool:
        g = (np.asarray(position, dtype=np.float64) - self.origin) / self.voxel_size
        return bool((g >= 0).all() and (g < self.dims).all())

    def center_of(self, index3) -> np.ndarray:
        return self.origin + (np.asarray(index3, dtype=np.float64) + 0.5) * self.voxel_size


def _grid_of(cfg) -> GridConfig:
    if isinstance(cfg, GridConfig):
        return cfg
    return GridConfig(np.asarray(cfg.origin), float(cfg.voxel_size), np.asarray(cfg.dims))


def _world_arrays(occ):
    """(spheres (S,4), boxes (B,6)) float64 of an ObstacleWorld (world.py:44-56), duck-typed
    through its `spheres` (centre, radius) and `boxes` (lo, hi) lists; None if `occ` is not one."""
    spheres, boxes = getattr(occ, "spheres", None), getattr(occ, "boxes", None)
    if spheres is None and boxes is None:
        return None
    sph = np.array([[*np.asarray(s.center, dtype=np.float64).reshape(3), float(s.radius)] for s in (spheres or [])],
                   dtype=np.float64).reshape(-1, 4)
    box = np.array([[*np.asarray(b.lo, dtype=np.float64).reshape(3), *np.asarray(b.hi, dtype=np.float64).reshape(3)]
                    for b in (boxes or [])], dtype=np.float64).reshape(-1, 6)
    return sph, box


def _segment_blocked(occ, start, ends) -> np.ndarray:
    """world.segment_blocked (world.py:96-140) restated in numpy with the reference's
    expressions (host parity reference for the device gate)."""
    start = np.asarray(start, dtype=np.float64).reshape(3)
    ends = np.asarray(ends, dtype=np.float64).reshape(-1, 3)
    blocked = np.zeros(ends.shape[0], dtype=bool)
    sph, box = _world_arrays(occ)
    if sph.shape[0] == 0 and box.shape[0] == 0:
        return blocked
    seg = ends - start
    t_hi = 1.0 - 1e-6
    for cx, cy, cz, r in sph:
        c = np.array([cx, cy, cz])
        rel = start - c
        a = np.einsum("ij,ij->i", seg, seg)
        b = 2.0 * seg @ rel
        t = np.where(a > 0, np.clip(-b / (2 * np.maximum(a, 1e-300)), 0.0, t_hi), 0.0)
        dist = np.linalg.norm(start + t[:, None] * seg - c, axis=1)
        blocked |= dist < r - 1e-9
    for row in box:
        lo, hi = row[:3] + 1e-9, row[3:] - 1e-9
        with np.errstate(divide="ignore", invalid="ignore"):
            inv = np.where(seg != 0.0, 1.0 / seg, np.inf)
            t0, t1 = (lo - start) * inv, (hi - start) * inv
        tmin, tmax = np.minimum(t0, t1), np.maximum(t0, t1)
        flat = seg == 0.0
        inside = (start >= lo) & (start <= hi)
        tmin = np.where(flat, np.where(inside, -np.inf, np.inf), tmin)
        tmax = np.where(flat, np.where(inside, np.inf, -np.inf), tmax)
        enter, leave = tmin.max(axis=1), tmax.min(axis=1)
        blocked |= (enter < leave) & (leave > 0.0) & (enter < t_hi)
    return blocked


@dataclass(frozen=True)
class Matchability:
    """Which landmarks contribute to a voxel (field.py:101-180).  The default accepts every
    pair.  Range, view cone and ObstacleWorld occlusion are device predicates (fif_gate.cuh,
    the reference's FP64 arithmetic, bit-identical masks) that the build kernels evaluate
    inside their pair loops; a Python `predicate` is evaluated pairwise on the host, as in
    the reference, and applied as an explicit mask."""

    d_near: float | None = None
    d_far: float | None = None
    view_cone_beta: float | None = None
    occluders: object | None = None
    predicate: object | None = None

    @property
    def is_trivial(self) -> bool:
        return all(x is None for x in (self.d_near, self.d_far, self.view_cone_beta, self.occluders, self.predicate))

    def describe(self) -> str:
        if self.is_trivial:
            return "always"
        parts = []
        if self.d_near is not None or self.d_far is not None:
            parts.append(f"range[{self.d_near},{self.d_far}]")
        if self.view_cone_beta is not None:
            parts.append(f"viewcone[{self.view_cone_beta:.4f}]")
        if self.occluders is not None:
            parts.append("occlusion")
        if self.predicate is not None:
            parts.append("custom")
        return "+".join(parts)

    @property
    def gpu_gates(self) -> bool:
        """Gates evaluated on the GPU: range, view cone, ObstacleWorld occlusion."""
        return (self.d_near is not None or self.d_far is not None or self.view_cone_beta is not None
                or (self.occluders is not None and _world_arrays(self.occluders) is not None))

    @property
    def host_gates(self) -> bool:
        """Gates only the host can evaluate: a Python predicate, or an occluder object that is
        not an ObstacleWorld but provides segment_blocked(center, points)."""
        return self.predicate is not None or (self.occluders is not None and _world_arrays(self.occluders) is None)

    def device_match(self, device: torch.device, view_dirs=None):
        """(fif_match struct, device tensors it points to) for the GPU gates."""
        m = _lib.Match()
        m.flags = 0
        keep = []
        if self.d_near is not None:
            m.d_near, m.flags = float(self.d_near), m.flags | _lib.MATCH_NEAR
        if self.d_far is not None:
            m.d_far, m.flags = float(self.d_far), m.flags | _lib.MATCH_FAR
        vd = None
        if self.view_cone_beta is not None:
            if view_dirs is None:
                raise ValueError("view_cone_beta requires landmark view directions")
            m.cos_beta, m.flags = float(np.cos(self.view_cone_beta)), m.flags | _lib.MATCH_CONE
            vd = _device.to_device_f64(view_dirs, device, (3,))
            keep.append(vd)
        arrays = _world_arrays(self.occluders) if self.occluders is not None else None
        if arrays is not None:
            sph = torch.from_numpy(np.ascontiguousarray(arrays[0])).to(device)
            box = torch.from_numpy(np.ascontiguousarray(arrays[1])).to(device)
            keep += [sph, box]
            m.spheres, m.n_spheres = (sph.data_ptr() if sph.shape[0] else None), sph.shape[0]
            m.boxes, m.n_boxes = (box.data_ptr() if box.shape[0] else None), box.shape[0]
            m.flags |= _lib.MATCH_OCCLUDE
        return m, vd, keep

    def device_any(self, centers: torch.Tensor, points: torch.Tensor, view_dirs=None) -> torch.Tensor:
        """(V,) bool on the device: some landmark passes the GPU gates (fif_match_any)."""
        dev = points.device
        m, vd, _keep = self.device_match(dev, view_dirs)
        out = torch.empty(centers.shape[0], dtype=torch.uint8, device=dev)
        with torch.cuda.device(dev):
            _lib.check(_lib.load().fif_match_any(m, _lib.ptr(centers), centers.shape[0], _lib.ptr(points),
                                                 _lib.ptr(vd), points.shape[0], _lib.ptr(out),
                                                 _device.stream_handle(dev)), "fif_match_any")
        return out.bool()

    def device_mask(self, centers: torch.Tensor, points: torch.Tensor, view_dirs=None) -> torch.Tensor:
        """(V, N) uint8 mask on the device: the GPU gates (fif_match_mask, bit-identical with
        `mask`), AND the host-only gates."""
        dev = points.device
        V, N = centers.shape[0], points.shape[0]
        if self.gpu_gates:
            m, vd, _keep = self.device_match(dev, view_dirs)
            out = torch.empty((V, N), dtype=torch.uint8, device=dev)
            with torch.cuda.device(dev):
                _lib.check(_lib.load().fif_match_mask(m, _lib.ptr(centers), V, _lib.ptr(points), _lib.ptr(vd), N,
                                                      _lib.ptr(out), _device.stream_handle(dev)), "fif_match_mask")
        else:
            out = torch.ones((V, N), dtype=torch.uint8, device=dev)
        if self.host_gates:
            occ = None if (self.occluders is None or _world_arrays(self.occluders) is not None) else self.occluders
            host = Matchability(occluders=occ, predicate=self.predicate)
            hm = host.mask(_device.to_numpy(centers), _device.to_numpy(points), view_dirs)
            out &= torch.from_numpy(hm).to(dev)
        return out

    def mask(self, centers, points, view_dirs=None):
        """Host restatement of the reference's mask (field.py:143-177); the build evaluates the
        same gates on the device, this is the parity reference for them."""
        if self.is_trivial:
            return None
        d = points[None, :, :] - centers[:, None, :]
        dist = np.linalg.norm(d, axis=2)
        ok = np.ones(dist.shape, dtype=bool)
        if self.d_near is not None:
            ok &= dist >= self.d_near
        if self.d_far is not None:
            ok &= dist <= self.d_far
        if self.view_cone_beta is not None:
            if view_dirs is None:
                raise ValueError("view_cone_beta requires landmark view directions")
            cosang = np.einsum("vnk,nk->vn", d / np.maximum(dist, 1e-12)[..., None], view_dirs)
            ok &= cosang >= np.cos(self.view_cone_beta)
        if self.occluders is not None:
            if _world_arrays(self.occluders) is not None:
                blocked_fn = lambda c, p: _segment_blocked(self.occluders, c, p)  # noqa: E731
            else:
                blocked_fn = getattr(self.occluders, "segment_blocked", None)
                if blocked_fn is None:
                    raise TypeError("occluders must be an ObstacleWorld (spheres / boxes) or provide "
                                    "segment_blocked(center, points)")
            for v in range(centers.shape[0]):
                ok[v] &= ~np.asarray(blocked_fn(centers[v], points), dtype=bool)
        if self.predicate is not None:
            for v in range(centers.shape[0]):
                for n in range(points.shape[0]):
                    if ok[v, n] and not self.predicate(centers[v], points[n]):
                        ok[v, n] = False
        return ok.astype(np.uint8)


ALWAYS_MATCH = Matchability()


def _as_points(landmarks):
    """Scene, (N,3) array / tensor, or a single 3-vector -> (points, view_dirs)."""
    view_dirs = getattr(landmarks, "view_dirs", None)
    positions = getattr(landmarks, "positions", landmarks)
    if isinstance(positions, torch.Tensor):
        pts = positions.to(torch.float64).reshape(-1, 3).contiguous()
    else:
        pts = np.ascontiguousarray(np.asarray(positions, dtype=np.float64).reshape(-1, 3))
    if view_dirs is not None:
        view_dirs = np.ascontiguousarray(np.asarray(view_dirs, dtype=np.float64).reshape(-1, 3))
    return pts, view_dirs


class _DeviceModel:
    """ctypes fif_model with device copies of zs / kinv (kept alive here)."""

    def __init__(self, model, device: torch.device):
        self.model = model
        m = _lib.Model()
        self._keep = []
        if isinstance(model, QuadraticVisibility):
            m.kind, m.n_v = _lib.MODEL_QUAD, 10
            m.k2, m.k1, m.k0 = model.k2, model.k1, model.k0
        else:
            m.kind, m.n_v = _lib.MODEL_GP, model.n_v
            m.k_s, m.cos_alpha = model.k_s, float(np.cos(model.alpha))
            m.sig2, m.ell = model.params.sigma2, model.params.length_scale
            zs_h = np.ascontiguousarray(model.samples, dtype=np.float64)
            zs = torch.from_numpy(zs_h).to(device)
            kinv = torch.from_numpy(np.ascontiguousarray(model.kinv)).to(device)
            self._keep += [zs, kinv, zs_h]
            m.zs, m.kinv = zs.data_ptr(), kinv.data_ptr()
            m.zs_host = zs_h.ctypes.data  # sample directions as kernel parameters (tcgen05 build)
        self.c = m


# masked builds evaluate the matchability gates for at most this many (voxel, landmark)
# pairs at a time (one byte each), bounding device memory for large maps
_MASK_CHUNK_BYTES = 1 << 30

# GP info kernel: "t5" (default; tcgen05.mma FP16 split with TMEM accumulators, N_s <= 80,
# other N_s run "h16"), "t6" (t5 with the sigmoid exponent arguments on the tensor cores too;
# measured slower, kept as a cross-check), "h16" (mma.sync FP16 split, k16 per MMA), "tf32"
# (mma.sync TF32x3) or "simt" (FP32 FFMA2); the alternatives are kept as cross-checks.
GP_INFO_KERNEL = "t5"
_GP_INFO_FLAGS = {"t5": 0, "t6": _lib.BUILD_T6, "h16": _lib.BUILD_H16, "tf32": _lib.BUILD_TF32,
                  "simt": _lib.BUILD_SIMT}


def build_rows(points: torch.Tensor, model, want_trace: bool, sigma: float, device: torch.device, grid=None,
               centers: torch.Tensor | None = None, v_begin: int = 0, v_end: int | None = None,
               mask: torch.Tensor | None = None, dmodel: _DeviceModel | None = None, f32_copy: bool = True,
               exact: bool = False, out64: torch.Tensor | None = None, out32: torch.Tensor | None = None,
               scratch: torch.Tensor | None = None):
    """One fif_build launch: rows [v_begin, v_end) of the z-major grid (or of `centers`).
    Returns (f64 rows (R, width_packed), f32 copy or None); out64 / out32 (contiguous row
    ranges of a larger field) receive the rows when given."""
    # the C ABI reads plain double pointers: anything else would be reinterpreted silently
    if points.dtype != torch.float64 or points.dim() != 2 or points.shape[1] != 3 or not points.is_contiguous():
        raise TypeError(f"build_rows: points must be a contiguous (N, 3) float64 tensor, got {tuple(points.shape)} "
                        f"{points.dtype}")
    if centers is not None and (centers.dtype != torch.float64 or not centers.is_contiguous()):
        raise TypeError(f"build_rows: centers must be a contiguous float64 tensor, got {centers.dtype}")
    dm = dmodel or _DeviceModel(model, device)
    n_v = 10 if isinstance(model, QuadraticVisibility) else model.n_v
    width = n_v if want_trace else n_v * 21
    if v_end is None:
        v_end = centers.shape[0] if centers is not None else int(np.prod(grid.dims))
    rows = v_end - v_begin
    gp = isinstance(model, GpVisibility)
    if out64 is None:
        out64 = torch.empty((rows, width), dtype=torch.float64, device=device)
        out32 = torch.empty((rows, width), dtype=torch.float32, device=device) if (gp and f32_copy) else None
    assert out64.shape == (rows, width) and out64.is_contiguous()
    assert out32 is None or (out32.shape == (rows, width) and out32.is_contiguous())
    n = points.shape[0]
    if scratch is None:
        scratch = torch.empty(int(_lib.load().fif_build_scratch_bytes(n)), dtype=torch.uint8, device=device)
    g = _lib.make_grid(grid.origin, grid.voxel_size, grid.dims) if grid is not None else None
    kind = _lib.KIND_TRACE if want_trace else _lib.KIND_INFO
    with torch.cuda.device(device):  # the library launches on the current device
        st = _lib.load().fif_build(kind, dm.c, _lib.ptr(points), n, g, _lib.ptr(centers), v_begin, v_end,
                                   _lib.ptr(mask), float(sigma),
                                   (_lib.BUILD_EXACT if exact else 0) | _GP_INFO_FLAGS[GP_INFO_KERNEL],
                                   _lib.ptr(scratch), _lib.ptr(out64), _lib.ptr(out32), _device.stream_handle(device))
    _lib.check(st, "fif_build")
    return out64, out32


def build_matched_rows(points: torch.Tensor, model, want_trace: bool, sigma: float, device: torch.device,
                       centers: torch.Tensor, matchability: "Matchability", view_dirs=None,
                       dmodel: _DeviceModel | None = None, f32_copy: bool = True, exact: bool = False):
    """One fif_build_matched launch: rows for the given centres with the GPU gates of
    `matchability` evaluated inside the build kernels (no (V, N) mask)."""
    dm = dmodel or _DeviceModel(model, device)
    n_v = model.n_v
    width = n_v if want_trace else n_v * 21
    rows = centers.shape[0]
    out64 = torch.empty((rows, width), dtype=torch.float64, device=device)
    gp = isinstance(model, GpVisibility)
    out32 = torch.empty((rows, width), dtype=torch.float32, device=device) if (gp and f32_copy) else None
    if points.dtype != torch.float64 or not points.is_contiguous() or centers.dtype != torch.float64 or \
            not centers.is_contiguous():
        raise TypeError("build_matched_rows: points and centers must be contiguous float64 tensors")
    scratch = torch.empty(int(_lib.load().fif_build_scratch_bytes(points.shape[0])), dtype=torch.uint8, device=device)
    m, vd, _keep = matchability.device_match(device, view_dirs)
    kind = _lib.KIND_TRACE if want_trace else _lib.KIND_INFO
    with torch.cuda.device(device):
        _lib.check(_lib.load().fif_build_matched(kind, dm.c, _lib.ptr(points), points.shape[0], _lib.ptr(centers), rows,
                                                 m, _lib.ptr(vd), float(sigma),
                                                 (_lib.BUILD_EXACT if exact else 0) | _GP_INFO_FLAGS[GP_INFO_KERNEL],
                                                 _lib.ptr(scratch), _lib.ptr(out64), _lib.ptr(out32),
                                                 _device.stream_handle(device)), "fif_build_matched")
    return out64, out32


def _host_rows(host_out, rows: int, width: int) -> torch.Tensor:
    if host_out is None:
        return torch.empty((rows, width), dtype=torch.float64).pin_memory()
    if tuple(host_out.shape) != (rows, width) or host_out.dtype != torch.float64 or host_out.is_cuda:
        raise ValueError(f"host_out must be a host float64 tensor of shape ({rows}, {width})")
    return host_out


def _export_chunks(field: "Field", host_out: torch.Tensor, chunks, before_export=None) -> None:
    """Export each row range of `chunks` (device staging, two buffers) and copy it to
    host_out on a side stream; before_export(i) runs on the compute stream first (the
    pipelined build launches chunk i's rows there)."""
    dev = field.device
    if not chunks:
        if before_export is not None:
            before_export(-1)
        return
    comp = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(device=dev)
    cmax = max(b - a for a, b in chunks)
    stage = [torch.empty((cmax, field.row_width), dtype=torch.float64, device=dev) for _ in range(2)]
    freed = [None, None]
    with torch.cuda.device(dev):
        for i, (a, b) in enumerate(chunks):
            if before_export is not None:
                before_export(i)
            buf = stage[i & 1]
            if freed[i & 1] is not None:
                comp.wait_event(freed[i & 1])  # the D2H of chunk i - 2 has drained this buffer
            field._export_range(a, b, buf)
            ready = torch.cuda.Event()
            ready.record(comp)
            copy.wait_event(ready)
            with torch.cuda.stream(copy):
                host_out[a:b].copy_(buf[: b - a], non_blocking=True)
                done = torch.cuda.Event()
                done.record(copy)
            freed[i & 1] = done
        comp.wait_stream(copy)
        for t in stage:
            t.record_stream(copy)


# z-slab row chunks of a host_factors build (chunk i's export + D2H overlap chunk i + 1's build)
HOST_EXPORT_CHUNKS = 8


def _build_to_host(pts_dev, config, model, factor_kind, sigma, dev, exact, host_out) -> "Field":
    """Dense build in z-slab row chunks; chunk i's export + D2H overlap chunk i + 1's build
    (a voxel's rows do not depend on the chunking: fixed flush spans)."""
    want_trace = factor_kind == "trace"
    n_v = model.n_v
    width = n_v if want_trace else n_v * 21
    rows = config.voxel_count
    gp = isinstance(model, GpVisibility)
    s64 = torch.empty((rows, width), dtype=torch.float64, device=dev)
    s32 = torch.empty((rows, width), dtype=torch.float32, device=dev) if gp else None
    fld = Field(config, model, factor_kind, sigma, s64, s32, None, ALWAYS_MATCH, dense=True)
    host_out = _host_rows(host_out, rows, fld.row_width)
    per = -(-rows // max(1, HOST_EXPORT_CHUNKS))
    chunks = [(a, min(rows, a + per)) for a in range(0, rows, per)]
    scratch = torch.empty(int(_lib.load().fif_build_scratch_bytes(pts_dev.shape[0])), dtype=torch.uint8, device=dev)

    def build_chunk(i):
        if i < 0:
            return
        a, b = chunks[i]
        build_rows(pts_dev, model, want_trace, sigma, dev, grid=config, v_begin=a, v_end=b, dmodel=fld._dm,
                   exact=exact, out64=s64[a:b], out32=None if s32 is None else s32[a:b], scratch=scratch)

    _export_chunks(fld, host_out, chunks, build_chunk)
    torch.cuda.current_stream(dev).synchronize()  # the host factors are complete on return
    fld._ref_cache = host_out.numpy()
    return fld


def device_centers(config: GridConfig, device: torch.device, order: int = 0) -> torch.Tensor:
    """(V,3) voxel centres on the device (fif_grid_centers; order 0 = the reference's x-major
    linear order, 1 = internal z-major), bit-identical to GridConfig.centers."""
    V = config.voxel_count
    out = torch.empty((V, 3), dtype=torch.float64, device=device)
    g = _lib.make_grid(config.origin, config.voxel_size, config.dims)
    with torch.cuda.device(device):
        _lib.check(_lib.load().fif_grid_centers(g, order, 0, V, _lib.ptr(out), _device.stream_handle(device)),
                   "fif_grid_centers")
    return out


class Field:
    """Voxel map of positional factors for one visibility model (field.py:193-614)."""

    def __init__(self, config: GridConfig, model, factor_kind: str, sigma: float, store64: torch.Tensor,
                 store32: torch.Tensor | None = None, occupied_index3: np.ndarray | None = None,
                 matchability: Matchability = ALWAYS_MATCH, dense: bool = True):
        if factor_kind not in _FACTOR_CODES:
            raise ValueError(f"factor_kind must be one of {tuple(_FACTOR_CODES)}")
        self.config = _grid_of(config)
        self.model = model_from_reference(model)
        self.factor_kind = factor_kind
        self.sigma = float(sigma)
        self.matchability = matchability
        self.device = store64.device
        self._s64 = store64
        self._s32 = store32
        self._dense = dense
        self._is_info = factor_kind == "info"
        self._dm = _DeviceModel(self.model, self.device)
        self._grid_c = _lib.make_grid(self.config.origin, self.config.voxel_size, self.config.dims)
        self._ref_cache = None
        self._t64 = None
        if dense:
            self._occ3 = None
            self._slots_np = None
            self._slots_dev = None
        else:
            self._occ3 = np.ascontiguousarray(occupied_index3, dtype=np.int32).reshape(-1, 3)
            slots = np.full(self.config.voxel_count, -1, dtype=np.int32)
            if self._occ3.shape[0]:
                slots[self.config.linear_index(self._occ3)] = np.arange(self._occ3.shape[0], dtype=np.int32)
            self._slots_np = slots
            self._slots_dev = torch.from_numpy(slots).to(self.device)

    # ── attributes of the reference Field ───────────────────────────
    @property
    def row_width(self) -> int:
        return self.model.n_v * (36 if self._is_info else 1)

    @property
    def rows(self) -> int:
        return int(self._s64.shape[0])

    @property
    def slots(self) -> np.ndarray:
        if self._slots_np is None:
            cfg = self.config
            lin = np.arange(cfg.voxel_count, dtype=np.int64)
            self._slots_np = cfg.internal_index(cfg.index3_of(lin)).astype(np.int32)
        return self._slots_np

    @property
    def occupied_index3(self) -> np.ndarray:
        if self._occ3 is None:
            self._occ3 = self.config.index3_of_internal(np.arange(self.rows)).astype(np.int32)
        return self._occ3

    @property
    def factors(self) -> np.ndarray:
        """Reference-layout FP64 rows (rows ordered as `occupied_index3`)."""
        if self._ref_cache is None:
            self._ref_cache = _device.to_numpy(self.export_reference())
        return self._ref_cache

    def export_reference_to(self, host_out: torch.Tensor | None = None, chunk_rows: int = 1 << 14) -> np.ndarray:
        """All reference-layout rows into (pinned) host memory, chunk by chunk: the export
        kernel of chunk i + 1 overlaps the D2H copy of chunk i (a side copy stream, two
        device staging buffers).  Returns the host rows (also cached as `factors`)."""
        host_out = _host_rows(host_out, self.rows, self.row_width)
        _export_chunks(self, host_out, [(a, min(self.rows, a + chunk_rows)) for a in range(0, self.rows, chunk_rows)])
        torch.cuda.current_stream(self.device).synchronize()  # the host rows are complete on return
        self._ref_cache = host_out.numpy()
        return self._ref_cache

    def export_reference(self, rows: torch.Tensor | np.ndarray | None = None) -> torch.Tensor:
        """Device tensor of reference-layout rows (all, or the given row indices)."""
        src = self._s64 if rows is None else self._s64[torch.as_tensor(rows, device=self.device, dtype=torch.long)]
        src = src.contiguous()
        out = torch.empty((src.shape[0], self.row_width), dtype=torch.float64, device=self.device)
        kind = _lib.KIND_INFO if self._is_info else _lib.KIND_TRACE
        with torch.cuda.device(self.device):
            _lib.check(_lib.load().fif_export_reference(kind, self._dm.c, _lib.ptr(src), src.shape[0], _lib.ptr(out),
                                                        _device.stream_handle(self.device)), "fif_export_reference")
        return out

    def _export_range(self, a: int, b: int, out: torch.Tensor) -> None:
        kind = _lib.KIND_INFO if self._is_info else _lib.KIND_TRACE
        with torch.cuda.device(self.device):
            _lib.check(_lib.load().fif_export_reference(kind, self._dm.c, _lib.ptr(self._s64[a:b]), b - a,
                                                        _lib.ptr(out), _device.stream_handle(self.device)),
                       "fif_export_reference")

    @property
    def storage(self) -> dict:
        return {"f64": self._s64, "f32": self._s32}

    # ── construction ────────────────────────────────────────────────
    @staticmethod
    def build(landmarks, config, model, factor_kind: str = "info", matchability: Matchability = ALWAYS_MATCH,
              sigma: float = DEFAULT_SIGMA, parallel: bool = False, device=None, exact: bool = False,
              process_group=None, replicate: bool = True, host_factors: bool = False,
              host_out: torch.Tensor | None = None) -> "Field":
        """Build every voxel's factor on the GPU.  `parallel` is accepted for API
        compatibility (the GPU build is always parallel).  exact=True (quad model)
        reproduces the reference's FP64 operation order bit for bit.  With a torch.distributed
        `process_group` (one rank per GPU; the default group when it is the WORLD) the grid
        is built as z-slabs across the ranks (parallel.build_field): replicate=True returns the
        whole field on every rank, replicate=False this rank's slab.
        host_factors=True also hands back what the reference's build returns, the
        reference-layout FP64 `factors` in host memory: the grid is built in z-slab chunks
        and each chunk's export and D2H copy overlap the build of the next (`host_out`: an
        optional pinned (rows, row_width) float64 buffer to fill)."""
        if process_group is not None:
            import torch.distributed as dist

            if process_group is not dist.group.WORLD:
                raise NotImplementedError("sharded builds run on the default (WORLD) process group")
            if not matchability.is_trivial:
                raise NotImplementedError("sharded builds support ALWAYS_MATCH")
            from .parallel import build_field

            pts, _ = _as_points(landmarks)
            return build_field(pts, config, model, factor_kind, sigma, _device.require_cuda(device), replicate)
        config = _grid_of(config)
        if config.voxel_count == 0:
            raise EmptyGrid("grid has zero voxels")
        if factor_kind not in _FACTOR_CODES:
            raise ValueError(f"factor_kind must be one of {tuple(_FACTOR_CODES)}")
        model = model_from_reference(model)
        dev = _device.require_cuda(device)
        points, view_dirs = _as_points(landmarks)
        want_trace = factor_kind == "trace"
        n_v = model.n_v
        width = n_v if want_trace else n_v * 21
        gp = isinstance(model, GpVisibility)
        if points.shape[0] == 0:
            empty64 = torch.zeros((0, width), dtype=torch.float64, device=dev)
            return Field(config, model, factor_kind, sigma, empty64, empty64.float() if gp else None,
                         np.zeros((0, 3), np.int32), matchability, dense=False)
        pts_dev = _device.to_device_f64(points, dev, (3,))
        if matchability.is_trivial and host_factors:
            return _build_to_host(pts_dev, config, model, factor_kind, sigma, dev, exact, host_out)
        if matchability.is_trivial:
            s64, s32 = build_rows(pts_dev, model, want_trace, sigma, dev, grid=config, exact=exact)
            return Field(config, model, factor_kind, sigma, s64, s32, None, matchability, dense=True)
        if not matchability.host_gates:
            # gates fused into the build kernels: occupancy pass (fif_match_any), then the
            # occupied voxels' rows in the reference's linear order (field.py:253-265)
            cen = device_centers(config, dev)
            occ = torch.nonzero(matchability.device_any(cen, pts_dev, view_dirs)).flatten()
            if occ.numel() == 0:
                s64 = torch.zeros((0, width), dtype=torch.float64, device=dev)
                return Field(config, model, factor_kind, sigma, s64, s64.float() if gp else None,
                             np.zeros((0, 3), np.int32), matchability, dense=False)
            s64, s32 = build_matched_rows(pts_dev, model, want_trace, sigma, dev, cen[occ].contiguous(), matchability,
                                          view_dirs, exact=exact)
            lin = occ.cpu().numpy()
            return Field(config, model, factor_kind, sigma, s64, s32, config.index3_of(lin).astype(np.int32),
                         matchability, dense=False)
        # a Python predicate (host, as in the reference): explicit masks in voxel chunks bounded
        # to _MASK_CHUNK_BYTES, occupied rows kept in the reference's linear order
        centers = config.centers()
        n = points.shape[0]
        chunk = max(1, min(config.voxel_count, _MASK_CHUNK_BYTES // max(1, n)))
        parts64, parts32, lins = [], [], []
        for c0 in range(0, config.voxel_count, chunk):
            c1 = min(config.voxel_count, c0 + chunk)
            cen = torch.from_numpy(np.ascontiguousarray(centers[c0:c1])).to(dev)
            mask = matchability.device_mask(cen, pts_dev, view_dirs)
            occ = torch.nonzero(mask.any(dim=1)).flatten()
            if occ.numel() == 0:
                continue
            s64, s32 = build_rows(pts_dev, model, want_trace, sigma, dev, centers=cen[occ].contiguous(),
                                  mask=mask[occ].contiguous(), exact=exact)
            parts64.append(s64)
            if s32 is not None:
                parts32.append(s32)
            lins.append(occ.cpu().numpy() + c0)
        if parts64:
            s64 = torch.cat(parts64)
            s32 = torch.cat(parts32) if parts32 else None
            lin = np.concatenate(lins)
        else:
            s64 = torch.zeros((0, width), dtype=torch.float64, device=dev)
            s32 = s64.float() if gp else None
            lin = np.zeros(0, dtype=np.int64)
        return Field(config, model, factor_kind, sigma, s64, s32, config.index3_of(lin).astype(np.int32),
                     matchability, dense=False)

    # ── queries ─────────────────────────────────────────────────────
    def _check_mode(self, mode: str) -> bool:
        if mode not in _MODES:
            raise ValueError(f"mode must be one of {_MODES}")
        return mode == "trilinear"

    def _field_ptr(self, use_f64: bool):
        # trace-kind GP fields always contract the FP64 master: with the FP32 copy, the
        # trace omega . T cancels (omega = kinv v^r alternates in sign) to 3e-4 relative on
        # config-2 nearest queries, over the 1e-4 tolerance; FP64 rows are 8 N_s B per corner
        if (isinstance(self.model, QuadraticVisibility) or use_f64 or self._s32 is None
                or not self._is_info):
            return self._s64, True
        return self._s32, False

    def trace_table(self) -> torch.Tensor | None:
        """FP64 (rows, n_v) per-sample trace of a GP info field's pre-kinv rows (the
        diagonal kernels.py:1414-1423 sums, left to right); the trace outputs of info-field
        queries contract it instead of the FP32 copy (fif_query_ex2).  Built on first use."""
        if not (self._is_info and isinstance(self.model, GpVisibility)):
            return None
        if self._t64 is None or self._t64.shape[0] != self.rows:
            v = self._s64.view(self.rows, self.model.n_v, 21)
            t = v[:, :, 0].clone()
            for k in (6, 11, 15, 18, 20):  # packed diagonal entries (1,1) ... (5,5)
                t += v[:, :, k]
            self._t64 = t.contiguous()
        return self._t64

    def query_device(self, positions: torch.Tensor, axes: torch.Tensor, mode: str = "trilinear",
                     trace: bool = True, full: bool = False, grad: bool = False, det: bool = False,
                     lmin: bool = False, field_f64: bool = False, out: dict | None = None) -> dict:
        """Device-resident batched query: (Q,3) positions and optical axes, float64 CUDA
        tensors.  Returns a dict of device tensors (trace, trace_grad, fim (Q,36),
        fim_grad (Q,6,36), det, lmin, status)."""
        trilinear = self._check_mode(mode)
        if (full or det or lmin) and not self._is_info:
            raise WrongFactorKind("full FIM / det / lmin require an info-factor field")
        q = positions.shape[0]
        dev = self.device
        out = {} if out is None else out

        def buf(name, shape, dtype=torch.float64):
            t = out.get(name)
            if t is None or t.shape[0] != q:
                t = torch.empty((q, *shape), dtype=dtype, device=dev)
                out[name] = t
            return t

        flags = 0
        tr_t = trg_t = fim_t = fimg_t = det_t = lmin_t = detg_t = lming_t = None
        if trace:
            flags |= _lib.Q_TRACE
            tr_t = buf("trace", ())
            if grad:
                trg_t = buf("trace_grad", (6,))
        if full:
            flags |= _lib.Q_FULL
            fim_t = buf("fim", (36,))
            if grad:
                fimg_t = buf("fim_grad", (6, 36))
        if grad:
            flags |= _lib.Q_GRAD
        if det:
            flags |= _lib.Q_DET
            det_t = buf("det", ())
            if grad:
                detg_t = buf("det_grad", (6,))
        if lmin:
            flags |= _lib.Q_LMIN
            lmin_t = buf("lmin", ())
            if grad:
                lming_t = buf("lmin_grad", (6,))
        st_t = buf("status", (), torch.uint8)
        # lambda_min gradients read the FP64 master: d lambda = v^T dF v through the
        # eigenvector v, whose sensitivity to the FP32 copy's rounding grows like
        # 1 / (eigenvalue gap) (measured 6e-4 on near-degenerate golden voxels vs 9e-6)
        field_t, is64 = self._field_ptr(field_f64 or (lmin and grad))
        if is64 and isinstance(self.model, GpVisibility):
            flags |= _lib.Q_FIELD_F64
        kind = _lib.KIND_INFO if self._is_info else _lib.KIND_TRACE
        if self.rows == 0:
            for t in (tr_t, trg_t, fim_t, fimg_t, det_t, lmin_t, detg_t, lming_t):
                if t is not None:
                    t.zero_()
            # every voxel is empty: status still follows the grid geometry
            dummy = torch.zeros((1, field_t.shape[1] if field_t.dim() == 2 else 1), dtype=field_t.dtype, device=dev)
            field_t = dummy
        slots = None if self._dense else self._slots_dev
        if self.rows == 0:
            slots = torch.full((self.config.voxel_count,), -1, dtype=torch.int32, device=dev)
        o = _lib.QueryOut(*(_lib.ptr(t) for t in (tr_t, trg_t, fim_t, fimg_t, det_t, detg_t, lmin_t, lming_t, st_t)))
        # trace outputs of a GP info field come from the FP64 trace table (see trace_table)
        ttab = self.trace_table() if (trace and not is64 and self.rows > 0) else None
        with torch.cuda.device(dev):
            _lib.check(_lib.load().fif_query_ex2(kind, self._dm.c, self._grid_c, _lib.ptr(field_t), _lib.ptr(ttab),
                                                 _lib.ptr(slots), _lib.ptr(positions), _lib.ptr(axes), q,
                                                 _lib.MODE_TRILINEAR if trilinear else _lib.MODE_NEAREST, flags, o,
                                                 _device.stream_handle(dev)), "fif_query")
        return out

    def query_graph(self, batch: int, mode: str = "trilinear", outputs=("trace", "full"), grad: bool = False,
                    field_f64: bool = False) -> "QueryGraph":
        """A CUDA-graph-captured query of a fixed batch size (planner inner loops issue
        many small batches, where launch latency dominates): static device input/output
        buffers, one graph replay per call.  See QueryGraph.run."""
        return QueryGraph(self, batch, mode, outputs, grad, field_f64)

    def query_batch(self, positions, rotations=None, axes=None, outputs=("trace", "full"), grad: bool = False,
                    mode: str = "trilinear", to_numpy: bool = False) -> dict:
        """Batched query with optional analytic pose gradients (new in this build).

        outputs subset of {"trace", "full", "det", "lmin"}.  Gradients are d/d[t; theta]
        for t' = t + dt, R' = exp(dtheta^) R; shapes: trace_grad / det_grad / lmin_grad (Q,6),
        fim_grad (Q,6,6,6).  det/lmin gradients: per corner det F tr(F^-1 dF) and v^T dF v.
        """
        dev = self.device
        pos = _device.to_device_f64(positions, dev, (3,))
        if axes is None:
            if rotations is None:
                raise ValueError("pass rotations (Q,3,3) or axes (Q,3)")
            r = _device.to_device_f64(rotations, dev, (3, 3))
            ax = r[:, :, 2].contiguous()
        else:
            ax = _device.to_device_f64(axes, dev, (3,))
        outs = set(outputs)
        res = self.query_device(pos, ax, mode, trace="trace" in outs, full="full" in outs, grad=grad,
                                det="det" in outs, lmin="lmin" in outs)
        q = pos.shape[0]
        ret = {"in_field": res["status"] == 0}
        for k in ("trace", "trace_grad", "det", "det_grad", "lmin", "lmin_grad"):
            if k in res:
                ret[k] = res[k]
        if "fim" in res:
            ret["fim"] = res["fim"].view(q, 6, 6)
        if "fim_grad" in res:
            ret["fim_grad"] = res["fim_grad"].view(q, 6, 6, 6)
        if to_numpy:
            ret = {k: _device.to_numpy(v) for k, v in ret.items()}
        return ret

    def query_fim_batch(self, positions, rotations, mode: str = "nearest"):
        """(fims (Q,6,6), in_field (Q,)) — zeros outside coverage (field.py:345-379)."""
        if not self._is_info:
            raise WrongFactorKind("FIM query requires an info-factor field")
        self._check_mode(mode)
        r = self.query_batch(positions, rotations=rotations, outputs=("full",), mode=mode, to_numpy=True)
        return r["fim"], r["in_field"]

    def query_fim(self, pose: Pose, mode: str = "nearest") -> np.ndarray:
        if not self._is_info:
            raise WrongFactorKind("FIM query requires an info-factor field")
        self._check_mode(mode)
        fims, ok = self.query_fim_batch(pose.translation[None], pose.rotation[None], mode)
        if not ok[0]:
            raise OutOfField(f"position {pose.translation.tolist()} outside field coverage")
        return fims[0]

    def metric_axis_batch(self, positions, axes, metric: str = "det", mode: str = "nearest"):
        """(values, in_field) at (position, optical axis) pairs (field.py:418-457)."""
        if metric not in ("det", "lmin", "trace"):
            raise ValueError(f"unknown metric {metric!r}")
        if not self._is_info and metric != "trace":
            raise WrongFactorKind("det/lmin require an info-factor field")
        self._check_mode(mode)
        r = self.query_batch(positions, axes=axes, outputs=(metric,), mode=mode, to_numpy=True)
        return r[metric], r["in_field"]

    def query_metric(self, pose: Pose, metric: str = "det", mode: str = "nearest") -> float:
        if metric not in ("det", "lmin", "trace"):
            raise ValueError(f"unknown metric {metric!r}")
        if not self._is_info and metric != "trace":
            raise WrongFactorKind("det/lmin require an info-factor field")
        self._check_mode(mode)
        vals, ok = self.metric_axis_batch(pose.translation[None], pose.rotation[:, 2][None], metric, mode)
        if not ok[0]:
            raise OutOfField(f"position {pose.translation.tolist()} outside field coverage")
        return float(vals[0])

    def locate(self, positions, mode: str = "trilinear") -> dict:
        """Corner table of each position on the device (fif_locate): the bit-exact indexing
        rule the queries use (kernels.py:628-635 nearest, 678-702 trilinear).  Returns numpy
        arrays index (Q,8) int64 reference linear voxel indices (-1 = unused corner),
        weight (Q,8) and status (Q,) uint8 (0 ok, 1 out of field)."""
        trilinear = self._check_mode(mode)
        dev = self.device
        pos = _device.to_device_f64(positions, dev, (3,))
        q = pos.shape[0]
        idx = torch.empty((q, 8), dtype=torch.int64, device=dev)
        w = torch.empty((q, 8), dtype=torch.float64, device=dev)
        st = torch.empty(q, dtype=torch.uint8, device=dev)
        with torch.cuda.device(dev):
            _lib.check(_lib.load().fif_locate(self._grid_c, _lib.ptr(pos), q,
                                              _lib.MODE_TRILINEAR if trilinear else _lib.MODE_NEAREST, _lib.ptr(idx),
                                              _lib.ptr(w), _lib.ptr(st), _device.stream_handle(dev)), "fif_locate")
        return {"index": _device.to_numpy(idx), "weight": _device.to_numpy(w), "status": _device.to_numpy(st)}

    def query_factor(self, position, mode: str = "nearest") -> np.ndarray:
        """Raw (blended) reference-layout factor at a position (field.py:277-303): the
        corners come from the device locate (the queries' bit-exact rule), the rows from
        the reference-layout export, blended in FP64 in corner order like the reference."""
        trilinear = self._check_mode(mode)
        pos = np.asarray(position, dtype=np.float64).reshape(3)
        loc = self.locate(pos[None], mode)
        if loc["status"][0] != 0:
            if trilinear:
                raise OutOfField(f"position {pos.tolist()} lacks 8 interpolation neighbors")
            raise OutOfField(f"position {pos.tolist()} outside grid")
        ncorner = 8 if trilinear else 1
        idx, wts = loc["index"][0, :ncorner], loc["weight"][0, :ncorner]
        rows = self.slots[idx]
        out = np.zeros(self.row_width)
        valid = rows >= 0
        if valid.any():
            ref = _device.to_numpy(self.export_reference(rows[valid]))
            if not trilinear:
                out = ref[0].copy()
            else:
                for w, row in zip(wts[valid], ref):
                    if w != 0.0:
                        out += w * row
        return out.reshape(self.model.n_v, 6, 6) if self._is_info else out

    # ── incremental updates (field.py:461-505) ──────────────────────
    def _increment(self, points, view_dirs, sign: float) -> None:
        pts, vd = _as_points(points)
        if pts.shape[0] == 0:
            return
        dev = self.device
        pts_dev = _device.to_device_f64(pts, dev, (3,))
        want_trace = not self._is_info
        if self.matchability.is_trivial and self._dense:
            inc, _ = build_rows(pts_dev, self.model, want_trace, self.sigma, dev, grid=self.config,
                                dmodel=self._dm, f32_copy=False)
            self._s64.add_(inc, alpha=sign)
        else:
            cen = device_centers(self.config, dev)
            vdirs = vd if vd is not None else view_dirs
            mt = self.matchability
            if mt.is_trivial:
                mask = None
                touched = np.ones(self.config.voxel_count, bool)
            elif not mt.host_gates:  # fused gates: occupancy only
                mask = None
                touched = _device.to_numpy(mt.device_any(cen, pts_dev, vdirs))
            else:
                mask = mt.device_mask(cen, pts_dev, vdirs)
                touched = _device.to_numpy(mask.any(dim=1))
            if not touched.any():
                return
            lin = np.nonzero(touched)[0]
            sel = torch.from_numpy(lin).to(dev)
            sub_c = cen[sel].contiguous()
            if not mt.is_trivial and not mt.host_gates:
                inc, _ = build_matched_rows(pts_dev, self.model, want_trace, self.sigma, dev, sub_c, mt, vdirs,
                                            dmodel=self._dm, f32_copy=False)
            else:
                sub_m = None if mask is None else mask[sel].contiguous()
                inc, _ = build_rows(pts_dev, self.model, want_trace, self.sigma, dev, centers=sub_c, mask=sub_m,
                                    dmodel=self._dm, f32_copy=False)
            if self._dense:
                rows = self.slots[lin]
            else:
                rows = self._slots_np[lin]
                missing = rows < 0
                if missing.any():
                    start = self.rows
                    new_lin = lin[missing]
                    self._slots_np[new_lin] = np.arange(start, start + new_lin.size, dtype=np.int32)
                    self._slots_dev = torch.from_numpy(self._slots_np).to(dev)
                    self._s64 = torch.cat([self._s64, torch.zeros((new_lin.size, self._s64.shape[1]),
                                                                  dtype=torch.float64, device=dev)])
                    self._occ3 = np.vstack([self._occ3, self.config.index3_of(new_lin).astype(np.int32)])
                    rows = self._slots_np[lin]
            idx = torch.as_tensor(rows.astype(np.int64), device=dev)
            self._s64.index_add_(0, idx, inc, alpha=sign)
        if self._s32 is not None:
            self._s32 = self._s64.float()
        self._ref_cache = None
        self._t64 = None

    def add_landmarks(self, landmarks, view_dirs=None) -> None:
        self._increment(landmarks, view_dirs, +1.0)

    def remove_landmarks(self, landmarks, view_dirs=None) -> None:
        self._increment(landmarks, view_dirs, -1.0)

    add_landmark = add_landmarks
    remove_landmark = remove_landmarks

    def update_landmark(self, old, new) -> None:
        self.remove_landmarks(old)
        self.add_landmarks(new)

    # ── accounting and serialization (field.py:509-614) ─────────────
    def memory_stats(self) -> dict:
        scalars = self.row_width
        rows = self.rows
        bytes_factors = rows * scalars * 8
        bytes_index = self.config.voxel_count * 4 + rows * 12
        dev_bytes = self._s64.numel() * 8 + (self._s32.numel() * 4 if self._s32 is not None else 0)
        return {
            "voxel_count": rows, "grid_voxels": self.config.voxel_count, "n_v": self.model.n_v,
            "scalars_per_voxel": scalars, "bytes_factors": bytes_factors, "bytes_factors_float32": rows * scalars * 4,
            "bytes_index": bytes_index, "bytes_total": bytes_factors + bytes_index, "device_bytes": dev_bytes,
        }

    def serialize(self, path) -> None:
        """FIF1 file, readable by the reference's Field.deserialize."""
        m = self.model
        head = bytearray(MAGIC)
        head += struct.pack("<I", FORMAT_VERSION)
        head += struct.pack("<B", _FACTOR_CODES[self.factor_kind])
        if isinstance(m, QuadraticVisibility):
            head += struct.pack("<B", _MODEL_QUAD) + struct.pack("<d", m.alpha) + struct.pack("<3d", m.k2, m.k1, m.k0)
        else:
            head += struct.pack("<B", _MODEL_GP) + struct.pack("<d", m.alpha) + struct.pack("<I", m.n_v)
            head += np.ascontiguousarray(m.samples, dtype="<f8").tobytes()
            head += struct.pack("<4d", m.params.sigma2, m.params.length_scale, m.params.jitter, m.k_s)
        head += struct.pack("<d", self.sigma)
        head += np.ascontiguousarray(self.config.origin, dtype="<f8").tobytes()
        head += struct.pack("<d", self.config.voxel_size)
        head += struct.pack("<3I", *(int(d) for d in self.config.dims))
        head += struct.pack("<Q", self.rows)
        occ = self.occupied_index3
        order = np.argsort(self.config.linear_index(occ), kind="stable")
        fac = self.factors
        rec = np.empty(self.rows, dtype=np.dtype([("i", "<i4", (3,)), ("f", "<f8", (self.row_width,))]))
        rec["i"] = occ[order]
        rec["f"] = fac[order]
        with open(path, "wb") as f:
            f.write(bytes(head))
            f.write(rec.tobytes())

    @staticmethod
    def deserialize(path, expect_kind: str | None = None, device=None) -> "Field":
        with open(path, "rb") as f:
            data = f.read()
        off = 0

        def take(n: int) -> bytes:
            nonlocal off
            if off + n > len(data):
                raise TruncatedFile(f"needed {n} bytes at offset {off}, file has {len(data)}")
            chunk = data[off:off + n]
            off += n
            return chunk

        if take(4) != MAGIC:
            raise BadMagic("not a field file (bad magic)")
        (version,) = struct.unpack("<I", take(4))
        if version != FORMAT_VERSION:
            raise VersionMismatch(f"file version {version}, supported {FORMAT_VERSION}")
        (kind_code,) = struct.unpack("<B", take(1))
        if kind_code not in _FACTOR_NAMES:
            raise TruncatedFile(f"unknown factor kind code {kind_code}")
        factor_kind = _FACTOR_NAMES[kind_code]
        if expect_kind is not None and factor_kind != expect_kind:
            raise WrongFactorKind(f"file holds {factor_kind} factors, expected {expect_kind}")
        (model_code,) = struct.unpack("<B", take(1))
        if model_code == _MODEL_QUAD:
            (alpha,) = struct.unpack("<d", take(8))
            model = QuadraticVisibility(alpha, *struct.unpack("<3d", take(24)))
        elif model_code == _MODEL_GP:
            (alpha,) = struct.unpack("<d", take(8))
            (n_s,) = struct.unpack("<I", take(4))
            samples = np.frombuffer(take(24 * n_s), dtype="<f8").reshape(n_s, 3).copy()
            sigma2, ell, jitter, k_s = struct.unpack("<4d", take(32))
            model = gp_build(samples, SeKernelParams(sigma2, ell, jitter), alpha, k_s)  # kinv recomputed
        else:
            raise TruncatedFile(f"unknown model kind code {model_code}")
        (sigma,) = struct.unpack("<d", take(8))
        origin = np.frombuffer(take(24), dtype="<f8").copy()
        (voxel_size,) = struct.unpack("<d", take(8))
        dims = struct.unpack("<3I", take(12))
        (rows,) = struct.unpack("<Q", take(8))
        config = GridConfig(origin, voxel_size, np.asarray(dims, dtype=np.int64))
        width = model.n_v * (36 if factor_kind == "info" else 1)
        rec_t = np.dtype([("i", "<i4", (3,)), ("f", "<f8", (width,))])
        rec = np.frombuffer(take(rows * rec_t.itemsize), dtype=rec_t)
        occ3 = np.ascontiguousarray(rec["i"], dtype=np.int32)
        factors = np.ascontiguousarray(rec["f"], dtype=np.float64)
        if rows and ((occ3 < 0).any() or (occ3 >= np.asarray(dims)).any()):
            raise TruncatedFile("voxel index outside grid")
        dev = _device.require_cuda(device)
        s64 = _device.to_device_f64(_from_reference_rows(factors, model, factor_kind), dev)
        s64 = s64.reshape(rows, model.n_v * (21 if factor_kind == "info" else 1))  # explicit width: rows may be 0
        s32 = s64.float() if isinstance(model, GpVisibility) else None
        fld = Field(config, model, factor_kind, sigma, s64, s32, occ3, ALWAYS_MATCH, dense=False)
        fld._ref_cache = factors  # bitwise round trip of the stored reference rows
        return fld


def _from_reference_rows(factors: np.ndarray, model, factor_kind: str) -> np.ndarray:
    """Reference-layout rows -> device storage layout (packed; GP: S = K F)."""
    n_v = model.n_v
    factors = np.asarray(factors, dtype=np.float64).reshape(-1, n_v * (36 if factor_kind == "info" else 1))
    rows = factors.shape[0]
    if factor_kind == "info":
        packed = factors.reshape(rows, n_v, 36)[:, :, _PACK36]
    else:
        packed = factors.reshape(rows, n_v, 1)
    if isinstance(model, GpVisibility):
        from .visibility import _gram

        packed = np.einsum("gk,rkw->rgw", _gram(model.samples, model.params), packed)
    return np.ascontiguousarray(packed.reshape(rows, n_v * (21 if factor_kind == "info" else 1)))


def build(landmarks, config, model, factor_kind="info", matchability=ALWAYS_MATCH, sigma=DEFAULT_SIGMA,
          parallel=False, device=None, **kw) -> Field:
    """Module-level alias for Field.build (field.py:645-648)."""
    return Field.build(landmarks, config, model, factor_kind, matchability, sigma, parallel, device, **kw)


class QueryGraph:
    """Fixed-size batched query captured once into a CUDA graph (Field.query_graph).

    run(positions, axes) copies the inputs into the static device buffers (from host
    or device tensors; a short batch is padded by repeating its last pose), replays the
    graph and returns the static output tensors (valid until the next run); replay()
    skips the copies when the caller writes self.positions / self.axes directly.  The
    field must not change (add/remove landmarks) while the graph lives."""

    def __init__(self, field: Field, batch: int, mode: str, outputs, grad: bool, field_f64: bool):
        if batch <= 0:
            raise ValueError("batch must be positive")
        self.field, self.batch = field, int(batch)
        dev = field.device
        outs = set(outputs)
        self._kw = dict(trace="trace" in outs, full="full" in outs, det="det" in outs, lmin="lmin" in outs,
                        grad=grad, field_f64=field_f64)
        field._check_mode(mode)
        self._mode = mode
        self.positions = torch.zeros((self.batch, 3), dtype=torch.float64, device=dev)
        self.axes = torch.zeros((self.batch, 3), dtype=torch.float64, device=dev)
        self.axes[:, 2] = 1.0
        self.out: dict = {}
        s = torch.cuda.Stream(device=dev)
        s.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(s):  # warm-up outside capture: allocations, function attributes
            field.query_device(self.positions, self.axes, mode, out=self.out, **self._kw)
        torch.cuda.current_stream(dev).wait_stream(s)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=s):
            field.query_device(self.positions, self.axes, mode, out=self.out, **self._kw)

    def replay(self) -> dict:
        """Replay on the current contents of self.positions / self.axes (fill them in
        place, e.g. from a planner's own kernels, to skip the input copies)."""
        self.graph.replay()
        return self.out

    def run(self, positions, axes) -> dict:
        n = positions.shape[0]
        if n > self.batch or axes.shape[0] != n:
            raise ValueError(f"batch of {n} poses does not fit the captured size {self.batch}")
        p = positions if isinstance(positions, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(positions,
                                                                                                        np.float64))
        a = axes if isinstance(axes, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(axes, np.float64))
        self.positions[:n].copy_(p.reshape(-1, 3), non_blocking=True)
        self.axes[:n].copy_(a.reshape(-1, 3), non_blocking=True)
        if n < self.batch and n > 0:
            self.positions[n:].copy_(self.positions[n - 1:n].expand(self.batch - n, 3))
            self.axes[n:].copy_(self.axes[n - 1:n].expand(self.batch - n, 3))
        self.graph.replay()
        return self.out
