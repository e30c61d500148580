"""Sensor geometry and camera set-up (one-off, host side).

Mirrors the parts of ``gelsim.sensors`` (sensors.py:26-50) and
``gelsim.render.camera`` (camera.py:13-66) that fix the hot path's shapes:
the active area, the image size, the pinhole intrinsics and the flat-pad
membrane depth.  Curved gels (ray casts against a surface mesh) are asset
preparation and out of scope.
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
    """Pinhole camera in the sensor frame looking along +z (camera.py:13-43)."""

    pos: np.ndarray = field(default_factory=lambda: np.array([0.0, 0.0, -0.02]))
    fx: float = 66.7
    fy: float = 66.7
    cx: float = 40.0
    cy: float = 30.0
    width: int = 80
    height: int = 60
    near: float = 0.002
    far: float = 0.2

    def rays(self) -> np.ndarray:
        """Unit ray directions (H, W, 3); pixel centres at +0.5 (camera.py:36-43)."""
        u = (np.arange(self.width) + 0.5 - self.cx) / self.fx
        v = (np.arange(self.height) + 0.5 - self.cy) / self.fy
        gu, gv = np.meshgrid(u, v, indexing="xy")
        d = np.stack([gu, gv, np.ones_like(gu)], axis=-1)
        return d / np.linalg.norm(d, axis=-1, keepdims=True)


def camera_for_sensor(sensor: TactileSensorSpec) -> TactileCamera:
    W, H = sensor.image_size
    f = sensor.focal_px
    return TactileCamera(pos=np.array([0.0, 0.0, -sensor.cam_distance]), fx=f, fy=f, cx=W / 2.0, cy=H / 2.0,
                         width=W, height=H, near=sensor.near, far=sensor.far)


def reference_depth(camera: TactileCamera, sensor: TactileSensorSpec | None = None) -> np.ndarray:
    """Membrane depth per pixel for the flat pad at z = 0: the ray parameter
    where the ray meets the gel plane, clipped to [near, far] (camera.py:56-66)."""
    d = camera.rays()
    t = -camera.pos[2] / d[..., 2]
    return np.clip(t, camera.near, camera.far)
