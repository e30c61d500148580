"""Sensor geometry and camera set-up (one-off, host side).

Mirrors the parts of ``gelsim.sensors`` (sensors.py:26-50) and
``gelsim.render.camera`` (camera.py:13-66) that fix the hot path's shapes:
the active area, the image size, the pinhole intrinsics and the flat-pad
membrane depth (the reference's ray cast against its two-triangle pad mesh,
restated so the background is bit-identical).  Curved gels (ray casts
against an arbitrary surface mesh) are asset preparation and out of scope.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

IDENTITY_QUAT = np.array([1.0, 0.0, 0.0, 0.0])


@dataclass
class TactileSensorSpec:
    """Flat GelSight-style pad (sensors.py:26-50)."""

    name: str = "gelpad"
    active_area: tuple = (0.024, 0.018)   # x, y extent (m)
    gel_thickness: float = 0.004
    cam_distance: float = 0.02            # camera at (0, 0, -cam_distance)
    image_size: tuple = (80, 60)          # W, H
    near: float = 0.002
    far: float = 0.2

    @property
    def focal_px(self) -> float:
        # active area fills the image width at the gel plane (sensors.py:44-46)
        return self.image_size[0] * self.cam_distance / self.active_area[0]

    def is_flat(self) -> bool:
        return True


@dataclass
class TactileCamera:
    """Pinhole camera at a fixed pose in the sensor frame, looking along its
    +z (camera.py:13-43); ``quat`` (w, x, y, z) rotates the rays."""

    pos: np.ndarray = field(default_factory=lambda: np.array([0.0, 0.0, -0.02]))
    quat: np.ndarray = field(default_factory=lambda: IDENTITY_QUAT.copy())
    fx: float = 66.7
    fy: float = 66.7
    cx: float = 40.0
    cy: float = 30.0
    width: int = 80
    height: int = 60
    near: float = 0.002
    far: float = 0.2

    def __post_init__(self):  # camera.py:28-34
        self.pos = np.asarray(self.pos, dtype=np.float64)
        self.quat = np.asarray(self.quat, dtype=np.float64)
        if self.width <= 0 or self.height <= 0:
            raise ValueError("image size must be positive")
        if not (0 < self.near < self.far):
            raise ValueError("need 0 < near < far")

    def rays(self) -> np.ndarray:
        """Unit ray directions (H, W, 3) in the sensor frame; pixel centres at
        +0.5, rotated by ``quat`` (camera.py:36-43)."""
        from .transforms import quat_rotate

        u = (np.arange(self.width) + 0.5 - self.cx) / self.fx
        v = (np.arange(self.height) + 0.5 - self.cy) / self.fy
        gu, gv = np.meshgrid(u, v, indexing="xy")
        d = np.stack([gu, gv, np.ones_like(gu)], axis=-1)
        d = d / np.linalg.norm(d, axis=-1, keepdims=True)
        return quat_rotate(self.quat, d)


def camera_for_sensor(sensor: TactileSensorSpec) -> TactileCamera:
    W, H = sensor.image_size
    f = sensor.focal_px
    return TactileCamera(pos=np.array([0.0, 0.0, -sensor.cam_distance]), fx=f, fy=f, cx=W / 2.0, cy=H / 2.0,
                         width=W, height=H, near=sensor.near, far=sensor.far)


def flat_pad_triangles(active_area, skirt: float = 0.002) -> np.ndarray:
    """The flat pad's gel surface: two triangles at z = 0 covering the active
    area plus a skirt, (2, 3, 3) (sensors.py:17-23 flat_pad_mesh)."""
    hx = active_area[0] / 2.0 + skirt
    hy = active_area[1] / 2.0 + skirt
    v = np.array([[-hx, -hy, 0.0], [hx, -hy, 0.0], [hx, hy, 0.0], [-hx, hy, 0.0]])
    return v[np.array([[0, 1, 2], [0, 2, 3]])]


def _cross(a, b):
    """np.cross component order: each product rounded, then subtracted."""
    return np.stack([a[..., 1] * b[..., 2] - a[..., 2] * b[..., 1],
                     a[..., 2] * b[..., 0] - a[..., 0] * b[..., 2],
                     a[..., 0] * b[..., 1] - a[..., 1] * b[..., 0]], axis=-1)


def _dot(a, b):
    """3-term dot product summed left to right (np.einsum's order)."""
    return (a[..., 0] * b[..., 0] + a[..., 1] * b[..., 1]) + a[..., 2] * b[..., 2]


def ray_triangles_t(origins, directions, triangles) -> np.ndarray:
    """Nearest non-negative hit parameter per ray over a triangle list, +inf on
    a miss: Moller-Trumbore with the reference's tolerances and operation order
    (geometry/mesh.py:166-193), so the membrane depth is bit-identical."""
    o = np.asarray(origins, dtype=np.float64)[:, None]      # (R, 1, 3)
    d = np.asarray(directions, dtype=np.float64)[:, None]
    tri = np.asarray(triangles, dtype=np.float64)
    v0, e1, e2 = tri[:, 0], tri[:, 1] - tri[:, 0], tri[:, 2] - tri[:, 0]
    pvec = _cross(d, e2[None])
    det = _dot(pvec, e1[None])
    ok = np.abs(det) > 1e-14
    inv = np.where(ok, 1.0 / np.where(ok, det, 1.0), 0.0)
    tvec = o - v0[None]
    u = _dot(tvec, pvec) * inv
    qvec = _cross(tvec, e1[None])
    v = _dot(d, qvec) * inv
    t = _dot(e2[None], qvec) * inv
    hit = ok & (u >= -1e-12) & (v >= -1e-12) & (u + v <= 1 + 1e-12) & (t >= 0)
    return np.where(hit, t, np.inf).min(axis=1)


def reference_depth(camera: TactileCamera, sensor: TactileSensorSpec | None = None) -> np.ndarray:
    """Membrane depth per pixel (camera.py:56-66): the rays cast against the
    flat pad's surface triangles, misses at the far plane, clipped to
    [near, far].  Bit-identical to the reference's (which casts against the
    same two-triangle mesh)."""
    sensor = sensor or TactileSensorSpec(image_size=(camera.width, camera.height))
    dirs = camera.rays().reshape(-1, 3)
    origins = np.broadcast_to(camera.pos, dirs.shape)
    t = ray_triangles_t(origins, dirs, flat_pad_triangles(sensor.active_area))
    t = np.where(np.isfinite(t), t, camera.far)
    return np.clip(t, camera.near, camera.far).reshape(camera.height, camera.width)
