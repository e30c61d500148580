"""Penalty force field: drop-ins for ``gelsim.tactile`` hot-path functions.

* ``compute_force_field`` -- tactile/field.py:79-129 (K2 on the GPU)
* ``penalty_forces``      -- tactile/field.py:61-76
* ``net_wrench``          -- tactile/field.py:132-141
* ``PenaltyParams``, ``ForceField``, ``TactilePointGrid``,
  ``sample_tactile_points`` -- field.py:28-58, points.py:13-67 (set-up types;
  flat pads -- curved-gel projection is asset preparation, out of scope).
"""
from __future__ import annotations

import threading
import weakref
from dataclasses import dataclass

import numpy as np

from . import _device, _lib
from .errors import DimensionMismatch
from .geometry import device_sdf

SLIP_VELOCITY_EPS = 1e-9  # field.py:25 (the kernels hard-code the same value)


@dataclass
class PenaltyParams:
    k_n: float = 1000.0
    k_d: float = 100.0
    k_t: float = 10.0
    mu: float = 2.0

    def __post_init__(self):
        if min(self.k_n, self.k_d, self.k_t, self.mu) < 0:
            raise ValueError("penalty parameters must be non-negative")


@dataclass
class ForceField:
    """Per-point normal and shear forces, sensor frame, (..., R, C, 3) (field.py:40-58)."""

    f_n: object
    f_t: object
    env_index: int | None = None
    frame_index: int | None = None

    @property
    def rows(self) -> int:
        return self.f_n.shape[-3]

    @property
    def cols(self) -> int:
        return self.f_n.shape[-2]

    def net(self):
        return self.f_n.sum(axis=(-3, -2)) + self.f_t.sum(axis=(-3, -2))


@dataclass
class TactilePointGrid:
    """rows x cols taxels on the gel surface, sensor frame (points.py:13-30)."""

    points: np.ndarray
    rest_normals: np.ndarray
    spacing: tuple

    @property
    def rows(self) -> int:
        return self.points.shape[0]

    @property
    def cols(self) -> int:
        return self.points.shape[1]

    def flat(self) -> np.ndarray:
        return self.points.reshape(-1, 3)


def sample_tactile_points(sensor, rows: int, cols: int) -> TactilePointGrid:
    """Taxel [r, c] at x = linspace(-ax/2, ax/2, cols)[c], y = linspace(-ay/2,
    ay/2, rows)[r] (points.py:33-57): at the pad's height on a flat pad; on a
    curved gel dropped onto the surface mesh along -z from z = 1, with the
    nearest face's outward normal (points.py:59-80), after the reference's
    ResolutionTooFine check (points.py:40-45)."""
    from .errors import ResolutionTooFine
    from .sensors import ray_triangles_t

    ax, ay = sensor.active_area
    dx = ax / (cols - 1) if cols > 1 else ax
    dy = ay / (rows - 1) if rows > 1 else ay
    mesh = sensor.surface_mesh
    flat = sensor.is_flat()
    if not flat:
        feature = float(mesh.edge_lengths().min())
        if min(dx, dy) < feature / 4.0:
            raise ResolutionTooFine(f"grid spacing {min(dx, dy):.2e} under mesh feature {feature:.2e}/4")
    xs = np.linspace(-ax / 2, ax / 2, cols)
    ys = np.linspace(-ay / 2, ay / 2, rows)
    gx, gy = np.meshgrid(xs, ys, indexing="xy")
    if flat:
        z0 = float(mesh.vertices[0, 2])
        pts = np.stack([gx, gy, np.full_like(gx, z0)], axis=-1)
        normals = np.zeros_like(pts)
        normals[..., 2] = 1.0
        return TactilePointGrid(points=pts, rest_normals=normals, spacing=(dx, dy))
    origins = np.stack([gx, gy, np.full_like(gx, 1.0)], axis=-1).reshape(-1, 3)
    dirs = np.tile(np.array([0.0, 0.0, -1.0]), (len(origins), 1))
    t = ray_triangles_t(origins, dirs, mesh.triangles)
    if not np.all(np.isfinite(t)):
        raise ValueError("active area extends beyond the surface mesh")
    pts = (origins + dirs * t[:, None]).reshape(rows, cols, 3)
    # nearest-face normal, outward = +z hemisphere (points.py:70-78)
    tri = mesh.triangles
    centroids = tri.mean(axis=1)
    fn = mesh.face_normals()
    flat_pts = pts.reshape(-1, 3)
    d2 = ((flat_pts[:, None] - centroids[None]) ** 2).sum(-1)
    n = fn[np.argmin(d2, axis=1)]
    normals = (n * np.sign(n[:, 2:3])).reshape(rows, cols, 3)
    return TactilePointGrid(points=pts, rest_normals=normals, spacing=(dx, dy))


# ---------------------------------------------------------------------------
# device-side taxel tables (cached per grid object and device)
# ---------------------------------------------------------------------------

_tax_lock = threading.Lock()
_tax_cache: dict = {}


def device_taxels(points, device):
    """(R*C, 3) float64 CUDA tensor of a TactilePointGrid (or (R, C, 3) array)."""
    t = _device.torch()
    arr = points.points if hasattr(points, "points") else points
    if _device.is_cuda_tensor(arr):
        return arr.to(device=device, dtype=t.float64).reshape(-1, 3).contiguous()
    key = (id(points), device.index)
    with _tax_lock:
        hit = _tax_cache.get(key)
        if hit is not None and hit[0]() is points:
            return hit[1]
    tens = _device.to_device(np.asarray(arr, dtype=np.float64).reshape(-1, 3), t.float64, device)
    try:
        ref = weakref.ref(points, lambda _r, k=key: _tax_cache.pop(k, None))
        with _tax_lock:
            _tax_cache[key] = (ref, tens)
    except TypeError:
        pass
    return tens


def force_field_launches(rows: int, cols: int) -> int:
    """Kernels one force-field call launches without kinematics: the taxels'
    fp32 copy and the certified fp32-mask kernel on dense pads (more than
    1024 taxels, rows*cols % 4 == 0; csrc/force_field.cu, quad kernel), else
    the fp64 fast kernel alone.  TACSL_FF_QUAD=0/1 forces the choice."""
    import os
    n = rows * cols
    q = os.environ.get("TACSL_FF_QUAD")
    want = (q == "1") if q is not None else n > 1024
    return 2 if want and n % 4 == 0 else 1


def _state_array(pos, quat, v, w, E, name):
    """Broadcast pos (3), quat (4), linvel (3), angvel (3) to an (E, 13) state."""
    parts = []
    for x, k in ((pos, 3), (quat, 4), (v, 3), (w, 3)):
        x = np.asarray(x, dtype=np.float64)
        x = x if x.ndim == 2 else x[None]
        if x.shape[-1] != k or x.shape[0] not in (1, E):
            raise ValueError(f"{name}: cannot broadcast shape {x.shape} to ({E}, {k})")
        parts.append(np.broadcast_to(x, (E, k)))
    return np.ascontiguousarray(np.concatenate(parts, axis=1))


def force_field_device(sdf, taxels, rows, cols, obj_state, sen_state, params, f_n=None, f_t=None,
                       wrench=None, kin=None, contact=None, n_sensors=1, obj_stride=13, sen_stride=None,
                       stream=None, obs=None, n_envs=None):
    """Device-level K2 on pre-allocated CUDA tensors.

    obj_state (E, 13) float64 (or one state with obj_stride=0); sen_state
    (E, S, 13) float64; f_n, f_t (E, S, R, C, 3) float32 or float64; obs
    (E, S, R, C, 3) float32 packed [f_n.z, f_t.x, f_t.y].  Any output may
    be None (not all).
    """
    t = _device.torch()
    ref = next(x for x in (f_n, f_t, obs, wrench, kin, contact) if x is not None)
    dsdf = device_sdf(sdf, ref.device)
    if n_envs is None:
        n_envs = sen_state.shape[0]
    if sen_stride is None:
        sen_stride = 13 * n_sensors
    out64 = 1 if (f_n is not None and f_n.dtype == t.float64) or (f_t is not None and f_t.dtype == t.float64) else 0
    lib = _lib.load()
    sh = _device.stream_handle(ref.device) if stream is None else stream
    _lib.check(lib.tacsl_force_field(
        dsdf.handle, taxels.data_ptr(), rows, cols, obj_state.data_ptr(), obj_stride, sen_state.data_ptr(),
        sen_stride, int(n_envs), n_sensors, _lib.penalty(params), out64, _device.ptr(f_n), _device.ptr(f_t),
        _device.ptr(wrench), _device.ptr(kin), _device.ptr(contact), _device.ptr(obs), sh))


def compute_force_field(points, object_sdf, object_pos, object_quat, object_linvel, object_angvel,
                        sensor_pos, sensor_quat, sensor_linvel, sensor_angvel, params, frame_index=None,
                        return_kinematics=False):
    """Drop-in for gelsim.tactile.compute_force_field (field.py:79-129).

    Pose / velocity arguments broadcast over a leading env axis exactly as in
    the reference: E = max(len(object_pos), len(sensor_pos)), and the result
    is batched iff ``object_pos`` is 2-D (field.py:90-100).  Returns
    ForceField(f_n, f_t) of float64 (E, R, C, 3) arrays in the sensor frame
    (or (R, C, 3) unbatched); with ``return_kinematics`` also
    {d, d_dot, v_t, n} in the world frame.
    """
    t = _device.torch()
    if min(params.k_n, params.k_d, params.k_t, params.mu) < 0:
        raise ValueError("penalty parameters must be non-negative")
    object_pos = np.asarray(object_pos, dtype=np.float64)
    batched = object_pos.ndim == 2
    o_pos = object_pos if object_pos.ndim == 2 else object_pos[None]
    s_pos = np.asarray(sensor_pos, dtype=np.float64)
    s_pos = s_pos if s_pos.ndim == 2 else s_pos[None]
    E = max(o_pos.shape[0], s_pos.shape[0])
    obj = _state_array(object_pos, object_quat, object_linvel, object_angvel, E, "object state")
    sen = _state_array(sensor_pos, sensor_quat, sensor_linvel, sensor_angvel, E, "sensor state")
    R, C = int(points.rows), int(points.cols)

    dsdf = device_sdf(object_sdf)
    dev = dsdf.device
    tax = device_taxels(points, dev)
    obj_d = _device.to_device(obj, t.float64, dev)
    sen_d = _device.to_device(sen, t.float64, dev)
    f_n = t.empty((E, R, C, 3), dtype=t.float64, device=dev)
    f_t = t.empty_like(f_n)
    kin = t.empty((E, R, C, 8), dtype=t.float64, device=dev) if return_kinematics else None
    force_field_device(dsdf, tax, R, C, obj_d, sen_d, params, f_n, f_t, kin=kin)
    fn, ft = _device.download(f_n), _device.download(f_t)  # straight into page-locked result arrays
    if not batched:
        fn, ft = fn[0], ft[0]
    fld = ForceField(f_n=fn, f_t=ft, frame_index=frame_index)
    if not return_kinematics:
        return fld
    k = _device.download(kin)
    if not batched:
        k = k[0]
    kinematics = {"d": k[..., 0], "d_dot": k[..., 1], "v_t": k[..., 2:5], "n": k[..., 5:8]}
    return fld, kinematics


def penalty_forces(d, d_dot, n, v_t, params):
    """Drop-in for gelsim.tactile.penalty_forces (field.py:61-76); inputs
    broadcast, d >= 0 yields zeros."""
    t = _device.torch()
    if min(params.k_n, params.k_d, params.k_t, params.mu) < 0:
        raise ValueError("penalty parameters must be non-negative")
    d = np.asarray(d, dtype=np.float64)
    d_dot = np.asarray(d_dot, dtype=np.float64)
    n = np.asarray(n, dtype=np.float64)
    v_t = np.asarray(v_t, dtype=np.float64)
    shape = np.broadcast_shapes(d.shape, d_dot.shape, n.shape[:-1], v_t.shape[:-1])
    dev = _device.resolve_device()
    bd = _device.to_device(np.broadcast_to(d, shape), t.float64, dev)
    bdd = _device.to_device(np.broadcast_to(d_dot, shape), t.float64, dev)
    bn = _device.to_device(np.broadcast_to(n, shape + (3,)), t.float64, dev)
    bv = _device.to_device(np.broadcast_to(v_t, shape + (3,)), t.float64, dev)
    count = int(np.prod(shape, dtype=np.int64))
    f_n = t.empty(shape + (3,), dtype=t.float64, device=dev)
    f_t = t.empty_like(f_n)
    _lib.check(_lib.load().tacsl_penalty_forces(bd.data_ptr(), bdd.data_ptr(), bn.data_ptr(), bv.data_ptr(), count,
                                                _lib.penalty(params), f_n.data_ptr(), f_t.data_ptr(),
                                                _device.stream_handle(dev)))
    return f_n.cpu().numpy(), f_t.cpu().numpy()


def net_wrench(fld, points):
    """Drop-in for gelsim.tactile.net_wrench (field.py:132-141): total force
    and torque about the sensor origin, sensor frame; DimensionMismatch when
    the field's (R, C) differs from the grid's."""
    t = _device.torch()
    if tuple(fld.f_n.shape[-3:-1]) != (points.rows, points.cols):
        raise DimensionMismatch(f"field {tuple(fld.f_n.shape[-3:-1])} vs grid {(points.rows, points.cols)}")
    on_device = _device.is_cuda_tensor(fld.f_n)
    dev = _device.resolve_device(fld.f_n.device if on_device else None)
    fn = _device.to_device(fld.f_n, t.float64, dev)
    ft = _device.to_device(fld.f_t, t.float64, dev)
    lead = tuple(fn.shape[:-3])
    frames = int(np.prod(lead, dtype=np.int64)) if lead else 1
    R, C = int(points.rows), int(points.cols)
    tax = device_taxels(points, dev)
    force = t.empty(lead + (3,), dtype=t.float64, device=dev)
    torque = t.empty_like(force)
    _lib.check(_lib.load().tacsl_net_wrench(fn.data_ptr(), ft.data_ptr(), tax.data_ptr(), frames, R, C,
                                            force.data_ptr(), torque.data_ptr(), _device.stream_handle(dev)))
    if on_device:
        return force, torque
    return force.cpu().numpy(), torque.cpu().numpy()
