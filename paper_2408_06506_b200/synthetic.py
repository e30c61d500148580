"""Synthetic workloads of BASELINE.json's configs.

* analytic spherical-indenter depth maps (float32) on the sensor camera,
* the 32x32x64 (or 128^3) peg SDF,
* peg-across-the-pad poses and velocities for every (env, sensor),
* the gradient-rescaled synthetic LUT.

Everything is seeded from np.random.SeedSequence((20240812, config_id)) so
tests, the oracle and the benchmark see identical inputs.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .geometry import cylinder_grid
from .render import DepthImage, synthetic_lut
from .sensors import TactileSensorSpec, camera_for_sensor, reference_depth
from .tactile import sample_tactile_points

SEED = 20240812
PEG_RADIUS = 0.008
PEG_HEIGHT = 0.05


@dataclass
class Workload:
    config_id: int
    n_envs: int
    n_sensors: int
    image_size: tuple      # (W, H)
    ff_grid: tuple         # (rows, cols)
    sdf_dims: tuple
    lut_degree: int = 2
    rgb: bool = True          # tactile RGB in the step
    ff: bool = True           # force field + wrench in the step
    pyramid_levels: int = 1   # RGB levels per frame (level l at 2^-l resolution)
    smooth_sigma: float = 0.0  # Gaussian smoothing of the depth before shading

    @property
    def frames(self) -> int:
        return self.n_envs * self.n_sensors


CONFIGS = {
    1: Workload(1, 1, 1, (320, 240), (20, 25), (32, 32, 64)),
    2: Workload(2, 1024, 2, (320, 240), (20, 25), (32, 32, 64)),
    3: Workload(3, 4096, 2, (320, 240), (20, 25), (32, 32, 64)),
    4: Workload(4, 16384, 1, (320, 240), (80, 100), (128, 128, 128), rgb=False),
    5: Workload(5, 8192, 1, (640, 480), (20, 25), (32, 32, 64), ff=False, pyramid_levels=3, smooth_sigma=1.0),
}


def lut_scale(image_size) -> float:
    """s = 1333 at 320 px width (|linear shading| ~ 0.1), proportional to W."""
    return 1333.0 * image_size[0] / 320.0


def sensor_setup(image_size=(320, 240), ff_grid=(20, 25), lut_degree=2, lut_seed=0):
    sensor = TactileSensorSpec(image_size=tuple(image_size))
    camera = camera_for_sensor(sensor)
    background = reference_depth(camera, sensor)
    lut = synthetic_lut(sensor.image_size, degree=lut_degree, seed=lut_seed,
                        gradient_scale=lut_scale(sensor.image_size))
    points = sample_tactile_points(sensor, *ff_grid)
    return sensor, camera, background, lut, points


def indenter_depth(camera, background, radius, cx, cy, delta) -> np.ndarray:
    """Depth along each ray of a sphere (centre (cx, cy, radius - delta)) pressed
    delta into the gel: min(first hit, membrane), clipped to [near, far]
    (as render_depth composes it, render/depth.py:114-131)."""
    d = camera.rays()
    o = np.asarray(camera.pos, dtype=np.float64)
    c = np.array([cx, cy, radius - delta])
    oc = o - c
    b = d @ oc
    cc = oc @ oc - radius * radius
    disc = b * b - cc
    hit = disc >= 0
    t = np.where(hit, -b - np.sqrt(np.where(hit, disc, 0.0)), np.inf)
    t = np.where(t > 0, t, np.inf)
    depth = np.minimum(t, background)
    return np.clip(depth, camera.near, camera.far)


def depth_batch(camera, background, n, config_id=3, pool=None) -> np.ndarray:
    """(n, H, W) float32 indenter maps; per image r ~ U[3, 8] mm, centre
    ~ U(+-4 mm, +-3 mm), indentation ~ U[0.2, 1.0] mm.  With ``pool`` only
    that many distinct maps are rendered and then tiled (benchmark inputs)."""
    m = n if pool is None else min(n, pool)
    rng = np.random.default_rng(np.random.SeedSequence((SEED, config_id, 1)))
    out = np.empty((m, camera.height, camera.width), dtype=np.float32)
    for i in range(m):
        r = rng.uniform(0.003, 0.008)
        cx, cy = rng.uniform(-0.004, 0.004), rng.uniform(-0.003, 0.003)
        delta = rng.uniform(0.0002, 0.001)
        out[i] = indenter_depth(camera, background, r, cx, cy, delta)
    if m == n:
        return out
    reps = -(-n // m)
    return np.tile(out, (reps, 1, 1))[:n]


def depth_image(camera, background, n, config_id=3) -> DepthImage:
    return DepthImage(values=depth_batch(camera, background, n, config_id), background=background)


def peg_grid(dims=(32, 32, 64)):
    """The peg of envs/peg_tasks.py:94-95 as a float32-representable grid."""
    return cylinder_grid(PEG_RADIUS, PEG_HEIGHT, dims=tuple(dims), padding=0.004)


def _quat_axis_angle(axis, angle):
    axis = np.asarray(axis, dtype=np.float64)
    axis = axis / np.linalg.norm(axis, axis=-1, keepdims=True)
    half = np.asarray(angle)[..., None] / 2.0
    return np.concatenate([np.cos(half), axis * np.sin(half)], axis=-1)


def _quat_mul(a, b):
    aw, ax, ay, az = np.moveaxis(a, -1, 0)
    bw, bx, by, bz = np.moveaxis(b, -1, 0)
    return np.stack([aw * bw - ax * bx - ay * by - az * bz, aw * bx + ax * bw + ay * bz - az * by,
                     aw * by - ax * bz + ay * bw + az * bx, aw * bz + ax * by - ay * bx + az * bw], axis=-1)


def _rotate(q, v):
    qv, w = q[..., 1:], q[..., :1]
    t = 2.0 * np.cross(qv, v)
    return v + w * t + np.cross(qv, t)


def peg_states(n_envs, n_sensors=1, config_id=3, random_sensor_pose=True):
    """Object (E, 13) and sensor (E, S, 13) states [pos, quat(wxyz), v, w].

    The peg lies across each pad (rotation about y of pi/2 +- U(0.1)), centre
    xy ~ U(+-2 mm), pressed 0..1 mm into the gel, v ~ N(0, 0.01 m/s),
    w ~ N(0, 0.1 rad/s); sensor 0's frame is the world frame for the object
    and every sensor s sees the peg at its own sampled relative pose (its
    world pose is a random rigid transform when ``random_sensor_pose``).
    For S > 1 the object state is shared by the env's sensors, so each
    sensor's pose is derived from the object pose and its relative pose.
    """
    rng = np.random.default_rng(np.random.SeedSequence((SEED, config_id, 2)))
    E, S = n_envs, n_sensors
    # relative peg pose in each sensor's frame
    ang = np.pi / 2 + rng.uniform(-0.1, 0.1, (E, S))
    q_rel = _quat_axis_angle(np.array([0.0, 1.0, 0.0]), ang)
    p_rel = np.stack([rng.uniform(-0.002, 0.002, (E, S)), rng.uniform(-0.002, 0.002, (E, S)),
                      PEG_RADIUS - rng.uniform(0.0, 0.001, (E, S))], axis=-1)
    # object world pose
    if random_sensor_pose:
        axis = rng.normal(size=(E, 3))
        q_obj = _quat_axis_angle(axis, rng.uniform(0, np.pi, E))
        p_obj = rng.uniform(-0.05, 0.05, (E, 3))
    else:
        q_obj = np.tile([1.0, 0.0, 0.0, 0.0], (E, 1))
        p_obj = np.zeros((E, 3))
    if not random_sensor_pose and S == 1:
        q_obj, p_obj = q_rel[:, 0], p_rel[:, 0]
    # sensor world pose so that sensor^-1 * object = relative pose:
    # q_s = q_obj * q_rel^-1 ; p_s = p_obj - R_s p_rel
    q_rel_inv = q_rel * np.array([1.0, -1.0, -1.0, -1.0])
    q_s = _quat_mul(np.broadcast_to(q_obj[:, None], (E, S, 4)), q_rel_inv)
    q_s = q_s / np.linalg.norm(q_s, axis=-1, keepdims=True)
    p_s = p_obj[:, None] - _rotate(q_s, p_rel)
    obj = np.zeros((E, 13))
    obj[:, 0:3], obj[:, 3:7] = p_obj, q_obj
    obj[:, 7:10] = rng.normal(0.0, 0.01, (E, 3))
    obj[:, 10:13] = rng.normal(0.0, 0.1, (E, 3))
    sen = np.zeros((E, S, 13))
    sen[..., 0:3], sen[..., 3:7] = p_s, q_s
    sen[..., 7:10] = rng.normal(0.0, 0.01, (E, S, 3))
    return obj, sen
