"""Host quaternion helpers, (w, x, y, z), in the reference's numpy operation
order (transforms.py:17-47) so that poses derived here -- e.g. the object
pose in each sensor frame the env passes to render_depth -- are bit-identical
to the reference's.  Set-up / per-step host math on a handful of values per
env; the per-pixel and per-taxel work is on the device."""
from __future__ import annotations

import numpy as np


def quat_mul(a, b):
    """Hamilton product a * b, each component summed left to right."""
    aw, ax, ay, az = np.moveaxis(np.asarray(a, dtype=np.float64), -1, 0)
    bw, bx, by, bz = np.moveaxis(np.asarray(b, dtype=np.float64), -1, 0)
    return np.stack([aw * bw - ax * bx - ay * by - az * bz,
                     aw * bx + ax * bw + ay * bz - az * by,
                     aw * by - ax * bz + ay * bw + az * bx,
                     aw * bz + ax * by - ay * bx + az * bw], axis=-1)


def quat_conj(q):
    return np.asarray(q, dtype=np.float64) * np.array([1.0, -1.0, -1.0, -1.0])


def _cross(a, b):
    return np.stack([a[..., 1] * b[..., 2] - a[..., 2] * b[..., 1],
                     a[..., 2] * b[..., 0] - a[..., 0] * b[..., 2],
                     a[..., 0] * b[..., 1] - a[..., 1] * b[..., 0]], axis=-1)


def quat_rotate(q, v):
    """v + w t + q_v x t with t = 2 q_v x v."""
    q = np.asarray(q, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    qv, w = q[..., 1:], q[..., :1]
    t = 2.0 * _cross(qv, v)
    return v + w * t + _cross(qv, t)


def quat_rotate_inv(q, v):
    return quat_rotate(quat_conj(q), v)
