"""CPU oracle for the TacSL sensor-simulation hot path -- TEST INFRASTRUCTURE ONLY.

This module is a plain-numpy restatement of the reference package ``gelsim``
(``/root/reference/pkg/src/gelsim``) for the two hot-path stages:

* depth -> tactile RGB  (``render/lut.py:20-76``, ``render/imageio.py:8-11``)
* penalty force field   (``tactile/field.py:61-141``, ``geometry/sdf.py:271-321``,
  ``transforms.py:36-47``)

It is written independently of the reference source (explicit slicing and
loops instead of ``np.gradient`` / ``np.cross`` / design-matrix stacking) and
is **pinned** against golden vectors produced by the reference itself
(``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``, checked by
``tests/test_oracle_golden.py``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import this module, and only as the checker or
the timed CPU baseline.  The product path (``paper_2408_06506_b200``) never
imports it and has no CPU fallback.

All arithmetic is float64, as in the reference.
"""
from __future__ import annotations

import numpy as np

SLIP_VELOCITY_EPS = 1e-9  # tactile/field.py:25


# ---------------------------------------------------------------------------
# depth -> RGB
# ---------------------------------------------------------------------------


def monomial_exponents(degree: int):
    """Term order of the polynomial LUT (render/lut.py:20-22):
    total degree s ascending, and within s the power of g_y ascending."""
    out = []
    for s in range(degree + 1):
        for j in range(s + 1):
            out.append((s - j, j))
    return out


def _axis_gradient(f: np.ndarray, axis: int) -> np.ndarray:
    """np.gradient with unit spacing and edge_order=1 along one axis
    (render/lut.py:27): central (f[i+1]-f[i-1])/2 inside, one-sided
    f[1]-f[0] / f[-1]-f[-2] (not halved) at the two borders."""
    f = np.moveaxis(np.asarray(f, dtype=np.float64), axis, -1)
    n = f.shape[-1]
    if n < 2:
        raise ValueError("gradient needs at least 2 samples along each image axis")
    g = np.empty_like(f)
    g[..., 1:-1] = (f[..., 2:] - f[..., :-2]) / 2.0
    g[..., 0] = f[..., 1] - f[..., 0]
    g[..., -1] = f[..., -1] - f[..., -2]
    return np.moveaxis(g, -1, axis)


def depth_gradients(values: np.ndarray):
    """(g_x, g_y) in m/px (render/lut.py:25-28)."""
    values = np.asarray(values, dtype=np.float64)
    g_y = _axis_gradient(values, values.ndim - 2)
    g_x = _axis_gradient(values, values.ndim - 1)
    return g_x, g_y


def poly_lut_evaluate(coeffs: np.ndarray, degree: int, g_x, g_y) -> np.ndarray:
    """sum_k c[ch,k] g_x^i g_y^j, clipped to [0,1] (render/lut.py:56-65)."""
    coeffs = np.asarray(coeffs, dtype=np.float64).reshape(3, -1)
    g_x = np.asarray(g_x, dtype=np.float64)
    g_y = np.asarray(g_y, dtype=np.float64)
    out = np.zeros(g_x.shape + (3,), dtype=np.float64)
    for k, (i, j) in enumerate(monomial_exponents(degree)):
        term = np.ones_like(g_x) if (i, j) == (0, 0) else (g_x ** i) * (g_y ** j)
        for ch in range(3):
            out[..., ch] += coeffs[ch, k] * term
    return np.clip(out, 0.0, 1.0)


def depth_to_rgb(values: np.ndarray, coeffs: np.ndarray, degree: int) -> np.ndarray:
    """(..., H, W) depth -> (..., H, W, 3) float64 in [0,1] (render/lut.py:68-76)."""
    g_x, g_y = depth_gradients(values)
    return poly_lut_evaluate(coeffs, degree, g_x, g_y)


def to_uint8(img: np.ndarray) -> np.ndarray:
    """clip(rint(x*255), 0, 255) with round-half-even (render/imageio.py:8-11)."""
    img = np.asarray(img)
    if img.dtype == np.uint8:
        return img
    return np.clip(np.rint(img.astype(np.float64) * 255.0), 0, 255).astype(np.uint8)


# ---------------------------------------------------------------------------
# quaternions (w, x, y, z)
# ---------------------------------------------------------------------------


def _cross(a, b):
    a0, a1, a2 = a[..., 0], a[..., 1], a[..., 2]
    b0, b1, b2 = b[..., 0], b[..., 1], b[..., 2]
    return np.stack([a1 * b2 - a2 * b1, a2 * b0 - a0 * b2, a0 * b1 - a1 * b0], axis=-1)


def quat_rotate(q, v):
    """v + w t + q_v x t, t = 2 q_v x v  (transforms.py:36-43)."""
    q = np.asarray(q, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    qv = q[..., 1:4]
    w = q[..., 0:1]
    t = 2.0 * _cross(np.broadcast_to(qv, np.broadcast_shapes(qv.shape, v.shape)), v)
    return v + w * t + _cross(np.broadcast_to(qv, t.shape), t)


def quat_rotate_inv(q, v):
    """Rotation by the conjugate (transforms.py:46-47, conj at 30-32)."""
    q = np.asarray(q, dtype=np.float64)
    qc = np.concatenate([q[..., :1], -q[..., 1:]], axis=-1)
    return quat_rotate(qc, v)


# ---------------------------------------------------------------------------
# SDF query
# ---------------------------------------------------------------------------


def query_sdf(origin, spacing, dims, values, gradients, points):
    """Trilinear distance + renormalised gradient (geometry/sdf.py:271-321).

    Returns (distance (N,), normal (N,3), valid (N,) bool); out-of-grid
    points give distance=+inf, normal=0.
    """
    origin = np.asarray(origin, dtype=np.float64)
    dims_a = np.asarray(dims, dtype=np.int64)
    values = np.asarray(values, dtype=np.float64)
    gradients = np.asarray(gradients, dtype=np.float64)
    pts = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    rel = (pts - origin) / float(spacing)
    valid = np.ones(len(pts), dtype=bool)
    for a in range(3):
        valid &= (rel[:, a] >= 0) & (rel[:, a] <= dims_a[a] - 1)
    upper = (dims_a - 1) - 1e-9
    rel_c = np.minimum(np.maximum(rel, 0.0), upper)
    i0 = np.minimum(np.trunc(rel_c).astype(np.int64), dims_a - 2)
    f = rel_c - i0
    ix, iy, iz = i0[:, 0], i0[:, 1], i0[:, 2]
    wx, wy, wz = f[:, 0], f[:, 1], f[:, 2]

    def lerp3(arr):
        if arr.ndim == 4:
            ex = (slice(None), None)
        else:
            ex = (slice(None),)
        ax, ay, az = wx[ex], wy[ex], wz[ex]
        c = {}
        for dx in (0, 1):
            for dy in (0, 1):
                for dz in (0, 1):
                    c[dx, dy, dz] = arr[ix + dx, iy + dy, iz + dz]
        c00 = c[0, 0, 0] * (1 - ax) + c[1, 0, 0] * ax
        c10 = c[0, 1, 0] * (1 - ax) + c[1, 1, 0] * ax
        c01 = c[0, 0, 1] * (1 - ax) + c[1, 0, 1] * ax
        c11 = c[0, 1, 1] * (1 - ax) + c[1, 1, 1] * ax
        c0 = c00 * (1 - ay) + c10 * ay
        c1 = c01 * (1 - ay) + c11 * ay
        return c0 * (1 - az) + c1 * az

    d = lerp3(values)
    g = lerp3(gradients)
    norm = np.sqrt(g[:, 0] * g[:, 0] + g[:, 1] * g[:, 1] + g[:, 2] * g[:, 2])
    n = g / np.maximum(norm, 1e-12)[:, None]
    d = np.where(valid, d, np.inf)
    n = np.where(valid[:, None], n, 0.0)
    return d, n, valid


# ---------------------------------------------------------------------------
# penalty force field
# ---------------------------------------------------------------------------


def penalty_forces(d, d_dot, n, v_t, k_n, k_d, k_t, mu):
    """f_n = max((-k_n + k_d d_dot) d, 0) n on contact; shear clamped to the
    friction cone (tactile/field.py:61-76)."""
    d = np.asarray(d, dtype=np.float64)
    d_dot = np.asarray(d_dot, dtype=np.float64)
    n = np.asarray(n, dtype=np.float64)
    v_t = np.asarray(v_t, dtype=np.float64)
    contact = d < 0.0
    coeff = np.where(contact, (-k_n + k_d * d_dot) * d, 0.0)
    coeff = np.maximum(coeff, 0.0)
    f_n = coeff[..., None] * n
    speed = np.sqrt(np.sum(v_t * v_t, axis=-1))
    slipping = contact & (speed > SLIP_VELOCITY_EPS)
    mag = np.minimum(k_t * speed, mu * coeff)
    safe = np.where(slipping, speed, 1.0)
    scale = np.where(slipping, mag / safe, 0.0)
    f_t = -scale[..., None] * v_t
    return f_n, f_t


def force_field_scalar(d, d_dot, n, v_t, k_n, k_d, k_t, mu):
    """Per-point scalar formula, as the reference test oracle states it
    (pkg/tests/oracles.py:67-85)."""
    if not (d < 0.0):
        return (0.0, 0.0, 0.0), (0.0, 0.0, 0.0)
    coeff = max((-k_n + k_d * d_dot) * d, 0.0)
    fn = tuple(coeff * c for c in n)
    fn_norm = sum(c * c for c in fn) ** 0.5
    vt_norm = sum(c * c for c in v_t) ** 0.5
    if vt_norm < 1e-9:
        return fn, (0.0, 0.0, 0.0)
    mag = min(k_t * vt_norm, mu * fn_norm)
    return fn, tuple(-c / vt_norm * mag for c in v_t)


def compute_force_field(points, origin, spacing, dims, values, gradients,
                        object_pos, object_quat, object_linvel, object_angvel,
                        sensor_pos, sensor_quat, sensor_linvel, sensor_angvel,
                        k_n=1000.0, k_d=100.0, k_t=10.0, mu=2.0):
    """Batched force field, sensor frame (tactile/field.py:79-129).

    points: (R, C, 3); pose / velocity arrays (E, k) or (k,) broadcasting.
    Returns f_n, f_t (E, R, C, 3) and kinematics dict {d, d_dot, v_t, n}
    (world frame), always with the leading env axis.
    """
    def bat(x):
        x = np.asarray(x, dtype=np.float64)
        return x if x.ndim == 2 else x[None]

    o_pos, o_q, o_v, o_w = (bat(x) for x in (object_pos, object_quat, object_linvel, object_angvel))
    s_pos, s_q, s_v, s_w = (bat(x) for x in (sensor_pos, sensor_quat, sensor_linvel, sensor_angvel))
    E = max(o_pos.shape[0], s_pos.shape[0])
    pts = np.asarray(points, dtype=np.float64)
    R, C = pts.shape[0], pts.shape[1]
    P = R * C
    p = np.broadcast_to(pts.reshape(1, P, 3), (E, P, 3))

    def ex(x):
        return np.broadcast_to(x[:, None, :], (E, P, x.shape[-1]))

    p_world = quat_rotate(ex(s_q), p) + ex(s_pos)
    p_obj = quat_rotate_inv(ex(o_q), p_world - ex(o_pos))
    d, n_obj, valid = query_sdf(origin, spacing, dims, values, gradients, p_obj.reshape(-1, 3))
    d = d.reshape(E, P)
    n_world = quat_rotate(ex(o_q), n_obj.reshape(E, P, 3))
    v_point = ex(s_v) + _cross(ex(s_w), p_world - ex(s_pos))
    v_obj = ex(o_v) + _cross(ex(o_w), p_world - ex(o_pos))
    x_dot = v_point - v_obj
    d_dot = np.sum(n_world * x_dot, axis=-1)
    v_t = x_dot - d_dot[..., None] * n_world
    f_n_w, f_t_w = penalty_forces(d, d_dot, n_world, v_t, k_n, k_d, k_t, mu)
    f_n = quat_rotate_inv(ex(s_q), f_n_w).reshape(E, R, C, 3)
    f_t = quat_rotate_inv(ex(s_q), f_t_w).reshape(E, R, C, 3)
    kin = {
        "d": d.reshape(E, R, C),
        "d_dot": d_dot.reshape(E, R, C),
        "v_t": v_t.reshape(E, R, C, 3),
        "n": n_world.reshape(E, R, C, 3),
        "valid": valid.reshape(E, R, C),
    }
    return f_n, f_t, kin


def net_wrench(f_n, f_t, points):
    """Total force and torque about the sensor origin (tactile/field.py:132-141)."""
    f = np.asarray(f_n, dtype=np.float64) + np.asarray(f_t, dtype=np.float64)
    pts = np.asarray(points, dtype=np.float64)
    force = f.sum(axis=(-3, -2))
    torque = _cross(np.broadcast_to(pts, f.shape), f).sum(axis=(-3, -2))
    return force, torque


# ---------------------------------------------------------------------------
# one sensor-frame pipeline (what bench.py's CPU baseline times)
# ---------------------------------------------------------------------------


def sensor_frames(depth, coeffs, degree, points, sdf, obj_state, sen_state, params):
    """RGB (uint8) + force field + wrench for a batch of sensor frames.

    depth (F, H, W); obj_state / sen_state (F, 13) = pos, quat(w,x,y,z), v, w.
    sdf = (origin, spacing, dims, values, gradients).
    """
    rgb = to_uint8(depth_to_rgb(depth, coeffs, degree))
    o, s = np.asarray(obj_state), np.asarray(sen_state)
    f_n, f_t, _ = compute_force_field(
        points, *sdf, o[:, 0:3], o[:, 3:7], o[:, 7:10], o[:, 10:13],
        s[:, 0:3], s[:, 3:7], s[:, 7:10], s[:, 10:13], *params)
    force, torque = net_wrench(f_n, f_t, points)
    return rgb, f_n, f_t, force, torque


# ---------------------------------------------------------------------------
# SDF sphere-traced depth (render/depth.py:88-134, numba march 174-233)
# ---------------------------------------------------------------------------


def quat_to_mat(q):
    """Rotation matrix of the normalised quaternion (transforms.py:78-91)."""
    q = np.asarray(q, dtype=np.float64)
    q = q / np.linalg.norm(q, axis=-1, keepdims=True)
    w, x, y, z = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    m = np.empty(q.shape[:-1] + (3, 3))
    m[..., 0, 0] = 1 - 2 * (y * y + z * z)
    m[..., 0, 1] = 2 * (x * y - w * z)
    m[..., 0, 2] = 2 * (x * z + w * y)
    m[..., 1, 0] = 2 * (x * y + w * z)
    m[..., 1, 1] = 1 - 2 * (x * x + z * z)
    m[..., 1, 2] = 2 * (y * z - w * x)
    m[..., 2, 0] = 2 * (x * z - w * y)
    m[..., 2, 1] = 2 * (y * z + w * x)
    m[..., 2, 2] = 1 - 2 * (x * x + y * y)
    return m


def render_depth(dirs, background, cam_pos, near, far, origin, spacing, dims, values, o_pos, o_quat,
                 tol=2e-5, max_steps=64):
    """Per-ray sphere trace of the object SDF; depth = min(hit, membrane),
    clipped to [near, far].  dirs (H, W, 3) unit rays, background (H, W);
    o_pos (E, 3), o_quat (E, 4) object pose in the sensor frame.  Follows
    the reference's default (numba) march operation for operation, vectorised
    over the still-marching rays.  Returns (E, H, W) float64."""
    dirs = np.asarray(dirs, dtype=np.float64).reshape(-1, 3)
    bg = np.asarray(background, dtype=np.float64).reshape(-1)
    cam = np.asarray(cam_pos, dtype=np.float64)
    origin = np.asarray(origin, dtype=np.float64)
    values = np.asarray(values, dtype=np.float64)
    nx, ny, nz = (int(v) for v in dims)
    o_pos = np.atleast_2d(np.asarray(o_pos, dtype=np.float64))
    o_quat = np.atleast_2d(np.asarray(o_quat, dtype=np.float64))
    E, R = o_pos.shape[0], dirs.shape[0]
    # object grid box in the sensor frame (depth.py:102-112)
    ext = np.array([[0, 0, 0], [0, 0, nz - 1], [0, ny - 1, 0], [0, ny - 1, nz - 1],
                    [nx - 1, 0, 0], [nx - 1, 0, nz - 1], [nx - 1, ny - 1, 0], [nx - 1, ny - 1, nz - 1]])
    corners = origin + spacing * ext
    cw = quat_rotate(o_quat[:, None], corners[None]) + o_pos[:, None]
    lo, hi = cw.min(axis=1), cw.max(axis=1)
    # slab test (depth.py:77-85)
    inv = 1.0 / np.where(np.abs(dirs) < 1e-300, 1e-300, dirs)
    t0 = (lo[:, None] - cam) * inv[None]
    t1 = (hi[:, None] - cam) * inv[None]
    tmin = np.minimum(t0, t1).max(axis=-1)
    tmax = np.maximum(t0, t1).min(axis=-1)
    hit = tmax >= np.maximum(tmin, 0.0)
    t_in = np.where(hit, np.maximum(tmin, 0.0), np.inf)
    t_out = np.where(hit, tmax, -np.inf)
    t_stop = np.minimum(bg[None], t_out)
    t_start = np.maximum(t_in, near)
    depth = np.broadcast_to(bg, (E, R)).copy()
    rot = quat_to_mat(o_quat)
    hix = origin[0] + spacing * (nx - 1)
    hiy = origin[1] + spacing * (ny - 1)
    hiz = origin[2] + spacing * (nz - 1)
    e_idx, r_idx = np.nonzero(t_start <= t_stop)
    t = t_start[e_idx, r_idx]
    stop = t_stop[e_idx, r_idx]
    for _ in range(max_steps):
        if e_idx.size == 0:
            break
        d_ = dirs[r_idx]
        p = o_pos[e_idx]
        m = rot[e_idx]
        wx = (cam[0] + d_[:, 0] * t) - p[:, 0]
        wy = (cam[1] + d_[:, 1] * t) - p[:, 1]
        wz = (cam[2] + d_[:, 2] * t) - p[:, 2]
        ox = (m[:, 0, 0] * wx + m[:, 1, 0] * wy) + m[:, 2, 0] * wz
        oy = (m[:, 0, 1] * wx + m[:, 1, 1] * wy) + m[:, 2, 1] * wz
        oz = (m[:, 0, 2] * wx + m[:, 1, 2] * wy) + m[:, 2, 2] * wz
        out = (ox < origin[0]) | (oy < origin[1]) | (oz < origin[2]) | (ox > hix) | (oy > hiy) | (oz > hiz)
        bx = np.maximum(origin[0] - ox, 0.0) + np.maximum(ox - hix, 0.0)
        by = np.maximum(origin[1] - oy, 0.0) + np.maximum(oy - hiy, 0.0)
        bz = np.maximum(origin[2] - oz, 0.0) + np.maximum(oz - hiz, 0.0)
        d_out = np.maximum(np.sqrt((bx * bx + by * by) + bz * bz), spacing)
        gx = np.where(out, 0.0, (ox - origin[0]) / spacing)
        gy = np.where(out, 0.0, (oy - origin[1]) / spacing)
        gz = np.where(out, 0.0, (oz - origin[2]) / spacing)
        ix = np.minimum(gx.astype(np.int64), nx - 2)
        iy = np.minimum(gy.astype(np.int64), ny - 2)
        iz = np.minimum(gz.astype(np.int64), nz - 2)
        fx, fy, fz = gx - ix, gy - iy, gz - iz
        v = values
        c00 = v[ix, iy, iz] * (1 - fx) + v[ix + 1, iy, iz] * fx
        c10 = v[ix, iy + 1, iz] * (1 - fx) + v[ix + 1, iy + 1, iz] * fx
        c01 = v[ix, iy, iz + 1] * (1 - fx) + v[ix + 1, iy, iz + 1] * fx
        c11 = v[ix, iy + 1, iz + 1] * (1 - fx) + v[ix + 1, iy + 1, iz + 1] * fx
        c0 = c00 * (1 - fy) + c10 * fy
        c1 = c01 * (1 - fy) + c11 * fy
        d_in = c0 * (1 - fz) + c1 * fz
        dist = np.where(out, d_out, d_in)
        hit_now = dist < tol
        cur = depth[e_idx[hit_now], r_idx[hit_now]]
        depth[e_idx[hit_now], r_idx[hit_now]] = np.minimum(cur, t[hit_now])
        t_next = t + dist
        keep = ~hit_now & ~(t_next > stop)
        e_idx, r_idx, t, stop = e_idx[keep], r_idx[keep], t_next[keep], stop[keep]
    return np.clip(depth, near, far).reshape((E,) + np.asarray(background).shape)
