"""Sensor geometry and camera set-up (one-off, host side).

Mirrors the parts of ``gelsim.sensors`` (sensors.py:17-50) and
``gelsim.render.camera`` (camera.py:13-66) that fix the hot path's shapes:
the active area, the image size, the pinhole intrinsics (with the camera's
orientation) and the membrane depth -- the reference's Moller-Trumbore ray
cast against the sensor's surface mesh (the flat pad's two triangles, or a
curved gel's mesh), restated in its operation order.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

IDENTITY_QUAT = np.array([1.0, 0.0, 0.0, 0.0])


class SurfaceMesh:
    """The gel surface as a triangle mesh, sensor frame: the parts of the
    reference's TriMesh (geometry/mesh.py:22-70) a sensor uses -- vertices,
    faces with degenerate faces dropped (area2 <= 1e-16, mesh.py:45-53),
    ``triangles``, ``face_normals``, ``edge_lengths``.  The reference's own
    TriMesh objects are accepted wherever a SurfaceMesh is."""

    def __init__(self, vertices, faces):
        self.vertices = np.asarray(vertices, dtype=np.float64).reshape(-1, 3)
        self.faces = np.asarray(faces, dtype=np.int64).reshape(-1, 3)
        if len(self.faces) == 0:
            raise ValueError("mesh has no faces")
        if self.faces.min() < 0 or self.faces.max() >= len(self.vertices):
            raise ValueError("face index out of range")
        tri = self.vertices[self.faces]
        area2 = np.linalg.norm(np.cross(tri[:, 1] - tri[:, 0], tri[:, 2] - tri[:, 0]), axis=1)
        keep = area2 > 1e-16
        if not keep.any():
            raise ValueError("all faces degenerate")
        self.faces = self.faces[keep]

    @property
    def triangles(self) -> np.ndarray:
        return self.vertices[self.faces]

    def face_normals(self) -> np.ndarray:
        tri = self.triangles
        n = np.cross(tri[:, 1] - tri[:, 0], tri[:, 2] - tri[:, 0])
        return n / np.linalg.norm(n, axis=1, keepdims=True)

    def edge_lengths(self) -> np.ndarray:
        tri = self.triangles
        e = np.concatenate([tri[:, 1] - tri[:, 0], tri[:, 2] - tri[:, 1], tri[:, 0] - tri[:, 2]])
        return np.linalg.norm(e, axis=1)


def flat_pad_mesh(active_area, skirt: float = 0.002) -> SurfaceMesh:
    """Two-triangle rectangle at z = 0 covering the active area plus a skirt
    (sensors.py:17-23)."""
    hx = active_area[0] / 2.0 + skirt
    hy = active_area[1] / 2.0 + skirt
    v = np.array([[-hx, -hy, 0.0], [hx, -hy, 0.0], [hx, hy, 0.0], [-hx, hy, 0.0]])
    return SurfaceMesh(v, np.array([[0, 1, 2], [0, 2, 3]]))


@dataclass
class TactileSensorSpec:
    """GelSight-style pad (sensors.py:26-50): a flat rectangle by default, or
    any sensor-frame ``surface_mesh`` for a curved gel."""

    name: str = "gelpad"
    active_area: tuple = (0.024, 0.018)   # x, y extent (m)
    surface_mesh: object = None           # SurfaceMesh / TriMesh; None -> flat pad
    gel_thickness: float = 0.004
    cam_distance: float = 0.02            # camera at (0, 0, -cam_distance)
    image_size: tuple = (80, 60)          # W, H
    near: float = 0.002
    far: float = 0.2

    def __post_init__(self):
        if self.surface_mesh is None:
            self.surface_mesh = flat_pad_mesh(self.active_area)

    @property
    def focal_px(self) -> float:
        # active area fills the image width at the gel plane (sensors.py:44-46)
        return self.image_size[0] * self.cam_distance / self.active_area[0]

    def is_flat(self) -> bool:
        n = self.surface_mesh.face_normals()
        return bool(np.allclose(n, n[0], atol=1e-9))


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


def _cross(a, b):
    """np.cross component order: each product rounded, then subtracted."""
    return np.stack([a[..., 1] * b[..., 2] - a[..., 2] * b[..., 1],
                     a[..., 2] * b[..., 0] - a[..., 0] * b[..., 2],
                     a[..., 0] * b[..., 1] - a[..., 1] * b[..., 0]], axis=-1)


def _dot(a, b):
    """3-term dot product in np.einsum's order for a length-3 axis,
    (x0 + x2) + x1 of the rounded products (numpy 2.3; checked against the
    reference's own einsum calls of ray_mesh_intersect, mesh.py:182-189)."""
    return (a[..., 0] * b[..., 0] + a[..., 2] * b[..., 2]) + a[..., 1] * b[..., 1]


def ray_triangles_t(origins, directions, triangles) -> np.ndarray:
    """Nearest non-negative hit parameter per ray over a triangle list, +inf on
    a miss: Moller-Trumbore with the reference's tolerances and operation order
    (geometry/mesh.py:166-193), in ray blocks of the reference's size, so the
    membrane depth is bit-identical."""
    o_all = np.atleast_2d(np.asarray(origins, dtype=np.float64))
    d_all = np.atleast_2d(np.asarray(directions, dtype=np.float64))
    tri = np.asarray(triangles, dtype=np.float64)
    v0, e1, e2 = tri[:, 0], tri[:, 1] - tri[:, 0], tri[:, 2] - tri[:, 0]
    best = np.full(len(o_all), np.inf)
    block = max(1, 4_000_000 // max(len(tri), 1))
    for s in range(0, len(o_all), block):
        o = o_all[s:s + block, None]      # (R, 1, 3)
        d = d_all[s:s + block, None]
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
        best[s:s + block] = np.where(hit, t, np.inf).min(axis=1)
    return best


def reference_depth(camera: TactileCamera, sensor: TactileSensorSpec | None = None) -> np.ndarray:
    """Membrane depth per pixel (camera.py:56-66): the rays cast against the
    sensor's surface mesh (flat pad or curved gel), misses at the far plane,
    clipped to [near, far]."""
    sensor = sensor or TactileSensorSpec(image_size=(camera.width, camera.height))
    dirs = camera.rays().reshape(-1, 3)
    origins = np.broadcast_to(camera.pos, dirs.shape)
    t = ray_triangles_t(origins, dirs, sensor.surface_mesh.triangles)
    t = np.where(np.isfinite(t), t, camera.far)
    return np.clip(t, camera.near, camera.far).reshape(camera.height, camera.width)
