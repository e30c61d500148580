"""Signed-distance grids on the device and the query_sdf drop-in.

Mirrors the reference's ``gelsim.geometry.sdf`` surface that the hot path
needs: ``SdfGrid`` / ``SdfQuery`` (sdf.py:29-63), ``query_sdf``
(sdf.py:271-321) and the TSDF cache format (sdf.py:331-361).  Building an SDF
from a mesh (``build_sdf``, sdf.py:66-100) is offline asset preparation and
out of scope; ``analytic_grid`` samples closed-form shapes the same way
``build_sdf`` lays out its grid, for synthetic benchmarks and tests.
"""
from __future__ import annotations

import struct
import threading
import weakref
from dataclasses import dataclass

import numpy as np

from . import _device, _lib

SDF_MAGIC = b"TSDF"
SDF_VERSION = 1


@dataclass
class SdfGrid:
    """Discretised signed distance + unit gradient (sdf.py:29-54)."""

    origin: np.ndarray
    spacing: float
    dims: tuple
    values: np.ndarray      # (nx, ny, nz), negative inside
    gradients: np.ndarray   # (nx, ny, nz, 3)

    def __post_init__(self):
        self.origin = np.asarray(self.origin, dtype=np.float64)
        self.dims = tuple(int(d) for d in self.dims)
        if self.spacing <= 0:
            raise ValueError("spacing must be positive")

    @property
    def upper(self) -> np.ndarray:
        return self.origin + self.spacing * (np.array(self.dims) - 1)

    def save(self, path) -> None:
        write_sdf_cache(self, path)

    @classmethod
    def load(cls, path) -> "SdfGrid":
        return read_sdf_cache(path)


@dataclass
class SdfQuery:
    """Interpolated distance, unit normal and in-bounds flag (sdf.py:57-63)."""

    distance: object
    normal: object
    valid: object


class DeviceSdf:
    """An SDF grid uploaded once to one device as float64 {d, gx, gy, gz} cells."""

    def __init__(self, grid, device=None):
        dev = _device.resolve_device(device)
        lib = _lib.load()
        dims = np.asarray(tuple(int(d) for d in grid.dims), dtype=np.int32)
        values = np.ascontiguousarray(np.asarray(grid.values, dtype=np.float64))
        grads = np.ascontiguousarray(np.asarray(grid.gradients, dtype=np.float64))
        if values.shape != tuple(dims) or grads.shape != tuple(dims) + (3,):
            raise ValueError("SdfGrid values/gradients do not match dims")
        origin = np.ascontiguousarray(np.asarray(grid.origin, dtype=np.float64))
        handle = _lib.c_void_p()
        _lib.check(lib.tacsl_sdf_create(dev.index, values.ctypes.data, grads.ctypes.data, dims.ctypes.data,
                                        origin.ctypes.data, float(grid.spacing), _lib.ctypes.byref(handle)))
        self.handle = handle
        self.device = dev
        self.dims = tuple(int(d) for d in dims)
        self.origin = origin.copy()
        self.spacing = float(grid.spacing)
        self._finalizer = weakref.finalize(self, lib.tacsl_sdf_destroy, handle)

    def close(self) -> None:
        self._finalizer()


_cache_lock = threading.Lock()
_cache: dict = {}


def device_sdf(grid, device=None) -> DeviceSdf:
    """Upload `grid` once per (object, device); grids are immutable by contract
    (SPEC.md:81-82), so the handle is cached for the grid object's lifetime."""
    if isinstance(grid, DeviceSdf):
        return grid
    dev = _device.resolve_device(device)
    key = (id(grid), dev.index)
    with _cache_lock:
        hit = _cache.get(key)
        if hit is not None and hit[0]() is grid:
            return hit[1]
    dsdf = DeviceSdf(grid, dev)
    with _cache_lock:
        try:
            ref = weakref.ref(grid, lambda _r, k=key: _cache.pop(k, None))
        except TypeError:  # not weak-referenceable: cache by identity only while alive in caller
            ref = (lambda g=grid: g)
        _cache[key] = (ref, dsdf)
    return dsdf


def query_sdf(grid, points) -> SdfQuery:
    """Drop-in for gelsim.geometry.query_sdf (sdf.py:271-321), on the GPU.

    numpy points -> numpy SdfQuery (float64, bool); CUDA tensor points ->
    CUDA tensors.  Out-of-grid points: distance +inf, normal 0, valid False.
    """
    t = _device.torch()
    on_device = _device.is_cuda_tensor(points)
    dev = points.device if on_device else None
    dsdf = device_sdf(grid, dev)
    dev = dsdf.device
    pts = _device.to_device(points, t.float64, dev)
    single = pts.ndim == 1
    pts2 = pts.reshape(-1, 3)
    if pts2.shape[-1] != 3:
        raise ValueError("points must have a trailing dimension of 3")
    n = pts2.shape[0]
    dist = t.empty(n, dtype=t.float64, device=dev)
    normal = t.empty((n, 3), dtype=t.float64, device=dev)
    valid = t.empty(n, dtype=t.uint8, device=dev)
    lib = _lib.load()
    _lib.check(lib.tacsl_query_sdf(dsdf.handle, pts2.data_ptr(), n, dist.data_ptr(), normal.data_ptr(),
                                   valid.data_ptr(), _device.stream_handle(dev)))
    valid_b = valid.bool()
    if single:
        dist, normal, valid_b = dist[0], normal[0], valid_b[0]
    if on_device:
        return SdfQuery(distance=dist, normal=normal, valid=valid_b)
    if single:
        return SdfQuery(distance=np.float64(dist.item()), normal=normal.cpu().numpy(),
                        valid=np.bool_(valid_b.item()))
    return SdfQuery(distance=dist.cpu().numpy(), normal=normal.cpu().numpy(), valid=valid_b.cpu().numpy())


# ---------------------------------------------------------------------------
# TSDF cache (little-endian): magic, version, dims, origin f32, spacing f32,
# values f32, gradients f32 -- sdf.py:331-361
# ---------------------------------------------------------------------------


def relative_penetration_rate(q: SdfQuery, x_dot):
    """Drop-in for gelsim.geometry.relative_penetration_rate (sdf.py:324-328):
    d_dot = n . x_dot per query, on the GPU; raises InvalidQuery when any
    query was out of the grid.  numpy in -> numpy out, CUDA in -> CUDA out."""
    t = _device.torch()
    on_device = _device.is_cuda_tensor(q.normal)
    dev = _device.resolve_device(q.normal.device if on_device else None)
    normal = _device.to_device(q.normal, t.float64, dev)
    valid = _device.to_device(q.valid, t.uint8, dev) if not _device.is_cuda_tensor(q.valid) else \
        q.valid.to(t.uint8).contiguous()
    xd = _device.to_device(x_dot, t.float64, dev)
    shape = tuple(normal.shape[:-1])
    single_x = tuple(xd.shape) == (3,)
    if not single_x:
        xd = xd.expand(tuple(normal.shape)).contiguous()
    n = int(np.prod(shape, dtype=np.int64)) if shape else 1
    out = t.empty(shape, dtype=t.float64, device=dev)
    scratch = t.empty(1, dtype=t.int32, device=dev)
    _lib.check(_lib.load().tacsl_relative_penetration_rate(
        normal.data_ptr(), valid.data_ptr(), xd.data_ptr(), n, int(single_x), out.data_ptr(), scratch.data_ptr(),
        _device.stream_handle(dev)))
    if on_device:
        return out
    host = out.cpu().numpy()
    return host if shape else np.float64(host)


def write_sdf_cache(grid, path) -> None:
    with open(path, "wb") as fh:
        fh.write(SDF_MAGIC)
        fh.write(struct.pack("<I", SDF_VERSION))
        fh.write(struct.pack("<3I", *(int(d) for d in grid.dims)))
        fh.write(struct.pack("<3f", *np.asarray(grid.origin, dtype=np.float32)))
        fh.write(struct.pack("<f", np.float32(grid.spacing)))
        fh.write(np.asarray(grid.values).astype("<f4").tobytes(order="C"))
        fh.write(np.asarray(grid.gradients).astype("<f4").tobytes(order="C"))


def read_sdf_cache(path) -> SdfGrid:
    with open(path, "rb") as fh:
        if fh.read(4) != SDF_MAGIC:
            raise ValueError(f"{path}: not an SDF cache file")
        (version,) = struct.unpack("<I", fh.read(4))
        if version != SDF_VERSION:
            raise ValueError(f"{path}: unsupported version {version}")
        dims = struct.unpack("<3I", fh.read(12))
        origin = np.array(struct.unpack("<3f", fh.read(12)), dtype=np.float64)
        (spacing,) = struct.unpack("<f", fh.read(4))
        n = dims[0] * dims[1] * dims[2]
        values = np.frombuffer(fh.read(4 * n), dtype="<f4").reshape(dims).astype(np.float64)
        grads = np.frombuffer(fh.read(12 * n), dtype="<f4").reshape(dims + (3,)).astype(np.float64)
    return SdfGrid(origin=origin, spacing=float(spacing), dims=dims, values=values, gradients=grads)


# ---------------------------------------------------------------------------
# analytic grids (synthetic assets)
# ---------------------------------------------------------------------------


def _layout(lo, hi, dims, padding):
    """Grid placement of build_sdf (sdf.py:78-82): cubic cells sized by the
    tightest axis, centred on the padded bounds."""
    dims = np.array(dims)
    extent = (np.asarray(hi) - np.asarray(lo)) + 2.0 * padding
    spacing = float(np.max(extent / (dims - 1)))
    center = (np.asarray(lo) + np.asarray(hi)) / 2.0
    origin = center - spacing * (dims - 1) / 2.0
    return origin, spacing


def _sample(fn, origin, spacing, dims, fp32=True):
    xs = origin[0] + spacing * np.arange(dims[0])
    ys = origin[1] + spacing * np.arange(dims[1])
    zs = origin[2] + spacing * np.arange(dims[2])
    px, py, pz = np.meshgrid(xs, ys, zs, indexing="ij")
    values = fn(px, py, pz)
    grads = np.stack(np.gradient(values, spacing), axis=-1)
    grads = grads / np.maximum(np.linalg.norm(grads, axis=-1, keepdims=True), 1e-12)
    if fp32:  # TSDF-cache precision: the same float32-representable grid feeds every implementation
        values = values.astype(np.float32).astype(np.float64)
        grads = grads.astype(np.float32).astype(np.float64)
    return SdfGrid(origin=origin, spacing=spacing, dims=tuple(dims), values=values, gradients=grads)


def cylinder_grid(radius=0.008, height=0.05, dims=(32, 32, 64), padding=0.004, fp32=True) -> SdfGrid:
    """Capped cylinder along +z centred at the origin -- the peg of
    envs/peg_tasks.py:94-95 (make_cylinder(0.008, 0.05)) sampled exactly."""
    h = height / 2.0

    def fn(x, y, z):
        dr = np.hypot(x, y) - radius
        dz = np.abs(z) - h
        out = np.hypot(np.maximum(dr, 0.0), np.maximum(dz, 0.0))
        return out + np.minimum(np.maximum(dr, dz), 0.0)

    origin, spacing = _layout((-radius, -radius, -h), (radius, radius, h), dims, padding)
    return _sample(fn, origin, spacing, dims, fp32)


def box_grid(size=(0.1, 0.1, 0.02), dims=(48, 48, 24), padding=0.01, fp32=True) -> SdfGrid:
    """Axis-aligned box centred at the origin (make_box of the reference tests)."""
    half = np.asarray(size, dtype=np.float64) / 2.0

    def fn(x, y, z):
        qx, qy, qz = np.abs(x) - half[0], np.abs(y) - half[1], np.abs(z) - half[2]
        outside = np.sqrt(np.maximum(qx, 0) ** 2 + np.maximum(qy, 0) ** 2 + np.maximum(qz, 0) ** 2)
        return outside + np.minimum(np.maximum(qx, np.maximum(qy, qz)), 0.0)

    origin, spacing = _layout(-half, half, dims, padding)
    return _sample(fn, origin, spacing, dims, fp32)


def sphere_grid(radius=0.005, dims=(48, 48, 48), padding=0.002, fp32=True) -> SdfGrid:
    def fn(x, y, z):
        return np.sqrt(x * x + y * y + z * z) - radius

    origin, spacing = _layout((-radius,) * 3, (radius,) * 3, dims, padding)
    return _sample(fn, origin, spacing, dims, fp32)
