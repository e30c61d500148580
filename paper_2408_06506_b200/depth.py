"""In-sensor depth rendering: drop-in for ``gelsim.render.render_depth``.

``render_depth(camera, object_sdf, object_pos, object_quat, background)``
(render/depth.py:88-134) sphere-traces the object's SDF per pixel on the GPU
(K3, csrc/render_depth.cu), bit-identical to the reference's float64 numba
march.  The per-env set-up the reference does in numpy -- the rotation matrix
of the object quaternion and the object's grid-box AABB in the sensor frame
(depth.py:102-112) -- is computed here with the same numpy operations, so
the kernel receives bit-identical inputs.
"""
from __future__ import annotations

import numpy as np

from . import _device, _lib
from .geometry import device_sdf
from .render import DepthImage

HIT_TOLERANCE = 2e-5   # depth.py:18
MAX_STEPS = 64         # depth.py:19


def _quat_rotate(q, v):
    qv, w = q[..., 1:], q[..., :1]
    t = 2.0 * np.cross(qv, v)
    return v + w * t + np.cross(qv, t)


def _quat_to_mat(q):
    """Rotation matrix of the normalised quaternion (transforms.py:78-91)."""
    q = np.asarray(q, dtype=np.float64)
    q = q / np.linalg.norm(q, axis=-1, keepdims=True)
    w, x, y, z = np.moveaxis(q, -1, 0)
    xx, yy, zz = x * x, y * y, z * z
    xy, xz, yz = x * y, x * z, y * z
    wx, wy, wz = w * x, w * y, w * z
    m = np.stack([1 - 2 * (yy + zz), 2 * (xy - wz), 2 * (xz + wy),
                  2 * (xy + wz), 1 - 2 * (xx + zz), 2 * (yz - wx),
                  2 * (xz - wy), 2 * (yz + wx), 1 - 2 * (xx + yy)], axis=-1)
    return m.reshape(m.shape[:-1] + (3, 3))


def env_params(object_sdf, o_pos, o_quat) -> np.ndarray:
    """(E, 18) per-env kernel inputs: pos, R (object->sensor), AABB lo, hi."""
    dims = np.array(object_sdf.dims)
    corners_obj = np.asarray(object_sdf.origin) + object_sdf.spacing * (
        np.stack(np.meshgrid([0, dims[0] - 1], [0, dims[1] - 1], [0, dims[2] - 1], indexing="ij"),
                 axis=-1).reshape(-1, 3))
    cw = _quat_rotate(o_quat[:, None], corners_obj[None]) + o_pos[:, None]
    lo, hi = cw.min(axis=1), cw.max(axis=1)
    rot = _quat_to_mat(o_quat)
    E = o_pos.shape[0]
    out = np.empty((E, 18))
    out[:, 0:3] = o_pos
    out[:, 3:12] = rot.reshape(E, 9)
    out[:, 12:15] = lo
    out[:, 15:18] = hi
    return out


class RayTable:
    """Per-camera device constants: unit rays and membrane depth."""

    def __init__(self, camera, background, device):
        t = _device.torch()
        self.height, self.width = int(camera.height), int(camera.width)
        self.pos = np.ascontiguousarray(np.asarray(camera.pos, dtype=np.float64))
        self.near, self.far = float(camera.near), float(camera.far)
        dirs = np.asarray(camera.rays(), dtype=np.float64).reshape(-1, 3)
        self.dirs = _device.to_device(dirs, t.float64, device)
        self.background = _device.to_device(np.asarray(background, dtype=np.float64).reshape(-1), t.float64, device)


def env_render_params_device(object_sdf, poses, n_sensors: int, out=None, stream=None):
    """env_params on the device for E envs x n_sensors sensors from one
    float64 CUDA tensor of world poses, (E, 7 * n_sensors + 7): each sensor's
    pos[3] + quat[4], then the object's.  Row e * n_sensors + s is the object
    pose in sensor s's frame (envs/peg_tasks.py:440-442) expanded into
    env_params' layout -- bit-identical to env_params(object_sdf,
    *relative poses) on the host."""
    t = _device.torch()
    E = int(poses.shape[0])
    if poses.dtype != t.float64 or not poses.is_cuda or poses.shape[1] != 7 * n_sensors + 7:
        raise ValueError("poses must be a float64 CUDA tensor of shape (E, 7 * n_sensors + 7)")
    poses = poses.contiguous()
    if out is None:
        out = t.empty((E * n_sensors, 18), dtype=t.float64, device=poses.device)
    dsdf = device_sdf(object_sdf, poses.device)
    sh = _device.stream_handle(poses.device) if stream is None else stream
    _lib.check(_lib.load().tacsl_env_render_params(dsdf.handle, poses.data_ptr(), E, int(n_sensors),
                                                   out.data_ptr(), sh))
    return out


def render_depth_device(camera_table: RayTable, sdf, params, out_f64=None, out_f32=None, stream=None):
    """Device-level K3: params (E, 18) float64 CUDA tensor -> (E, H, W) depth."""
    dsdf = device_sdf(sdf, params.device)
    E = params.shape[0]
    lib = _lib.load()
    sh = _device.stream_handle(params.device) if stream is None else stream
    _lib.check(lib.tacsl_render_depth(
        dsdf.handle, camera_table.dirs.data_ptr(), camera_table.background.data_ptr(), camera_table.height,
        camera_table.width, camera_table.pos.ctypes.data, camera_table.near, camera_table.far, HIT_TOLERANCE,
        MAX_STEPS, params.data_ptr(), E, _device.ptr(out_f64), _device.ptr(out_f32), sh))
    return out_f64, out_f32


def render_depth(camera, object_sdf, object_pos, object_quat, background) -> DepthImage:
    """Drop-in for gelsim.render.render_depth (render/depth.py:88-134).

    object_pos / object_quat: object pose in the sensor frame, optionally with
    a leading env axis (then the depth is (E, H, W), else (H, W)).  Returns a
    DepthImage of float64 numpy depth, bit-identical to the reference.
    """
    t = _device.torch()
    object_pos = np.asarray(object_pos, dtype=np.float64)
    batched = object_pos.ndim == 2
    o_pos = np.atleast_2d(object_pos)
    o_quat = np.atleast_2d(np.asarray(object_quat, dtype=np.float64))
    dsdf = device_sdf(object_sdf)
    dev = dsdf.device
    table = RayTable(camera, background, dev)
    params = _device.to_device(env_params(object_sdf, o_pos, o_quat), t.float64, dev)
    out = t.empty((o_pos.shape[0], table.height, table.width), dtype=t.float64, device=dev)
    render_depth_device(table, dsdf, params, out_f64=out)
    depth = out.cpu().numpy()
    if not batched:
        depth = depth[0]
    return DepthImage(values=depth, background=np.asarray(background).copy())
