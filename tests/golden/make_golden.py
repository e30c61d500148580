"""Generate golden vectors by running the REFERENCE implementation.

    python tests/golden/make_golden.py

Imports the reference package ``gelsim`` read-only from
/root/reference/pkg/src (this container only -- /root/reference does not
exist on the GPU box) and records inputs + reference outputs of every
hot-path function into tests/golden/*.npz.  The committed .npz files are
what the tests read; this script is kept so the fixtures can be re-made.

Fixtures:
  rgb.npz        depth_to_rgb (+ to_uint8) at 60x80 (degrees 2-4, scaled and
                 unscaled LUTs), 240x320 (uint8), odd sizes, and the
                 reference tests' flat / tilted / clamp cases
  sdf.npz        query_sdf on a reference-built (build_sdf) peg grid
  ff.npz         compute_force_field (+ kinematics) and net_wrench for a
                 batch of random peg presses with random sensor poses,
                 plus one unbatched call
  penalty.npz    penalty_forces on the seed-11 draws of
                 test_tactile_field.py:153-168
  env.npz        PegEnvBatch tactile image / force-field observations with
                 augmentation and their inputs (``make_golden.py env``)
  scene.npz      shape_sensing_scene end to end (``make_golden.py scene``)
  extras.npz     TactileCamera with a rotated pose (rays, reference_depth) and
                 relative_penetration_rate (+ the InvalidQuery case) on the
                 sdf.npz grid (``make_golden.py extras``)
"""
from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
REF_SRC = Path("/root/reference/pkg/src")

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(ROOT))

from gelsim.geometry import build_sdf, make_cylinder, query_sdf  # noqa: E402
from gelsim.render import camera_for_sensor, reference_depth, render_depth  # noqa: E402
from gelsim.render import DepthImage, PolyLut, depth_to_rgb, synthetic_lut, to_uint8  # noqa: E402
from gelsim.sensors import TactileSensorSpec  # noqa: E402
from gelsim.tactile import PenaltyParams, compute_force_field, net_wrench, penalty_forces  # noqa: E402
from gelsim.tactile import sample_tactile_points  # noqa: E402

from paper_2408_06506_b200 import synthetic  # noqa: E402  (input generators only)
from paper_2408_06506_b200.sensors import camera_for_sensor as my_camera  # noqa: E402
from paper_2408_06506_b200.sensors import reference_depth as my_background  # noqa: E402


def scaled_lut(image_size, degree, seed=0, s=1.0):
    lut = synthetic_lut(image_size, degree=degree, seed=seed)
    coeffs = lut.coeffs.copy()
    k = 0
    for tot in range(degree + 1):
        for j in range(tot + 1):
            coeffs[:, k] *= s ** tot
            k += 1
    return PolyLut(degree=degree, coeffs=coeffs, image_size=tuple(image_size))


def depth_maps(W, H, n, config_id):
    sensor = TactileSensorSpec(image_size=(W, H))
    cam = my_camera(sensor)
    bg = my_background(cam, sensor)
    return synthetic.depth_batch(cam, bg, n, config_id=config_id), bg


def make_rgb():
    out = {}
    # 60x80 (reference default camera), scaled LUTs, degrees 2..4
    d, bg = depth_maps(80, 60, 3, config_id=101)
    out["d60"] = d
    for deg in (2, 3, 4):
        lut = scaled_lut((80, 60), deg, seed=deg, s=synthetic.lut_scale((80, 60)))
        rgb = depth_to_rgb(DepthImage(values=d.astype(np.float64), background=bg), lut)
        out[f"c60_deg{deg}"] = lut.coeffs
        out[f"rgb60_deg{deg}"] = rgb
        out[f"u8_60_deg{deg}"] = to_uint8(rgb)
    # unscaled reference demo LUT (flat-looking images)
    lut = synthetic_lut((80, 60), degree=2, seed=0)
    out["c60_plain"] = lut.coeffs
    out["rgb60_plain"] = depth_to_rgb(DepthImage(values=d.astype(np.float64), background=bg), lut)
    # 240x320, uint8 only (degree 2, the env default)
    d2, bg2 = depth_maps(320, 240, 1, config_id=102)
    lut = scaled_lut((320, 240), 2, seed=0, s=synthetic.lut_scale((320, 240)))
    out["d240"] = d2
    out["c240"] = lut.coeffs
    out["u8_240"] = to_uint8(depth_to_rgb(DepthImage(values=d2.astype(np.float64), background=bg2), lut))
    # odd sizes (misaligned rows: generic kernel path)
    rng = np.random.default_rng(5)
    for (H, W) in ((2, 3), (5, 7), (9, 18), (3, 2)):
        v = (0.02 + rng.uniform(-1e-4, 1e-4, (2, H, W))).astype(np.float32)
        lut = scaled_lut((W, H), 3, seed=1, s=300.0)
        out[f"odd_{H}x{W}_d"] = v
        out[f"odd_{H}x{W}_c"] = lut.coeffs
        out[f"odd_{H}x{W}_rgb"] = depth_to_rgb(DepthImage(values=v.astype(np.float64), background=v[0]), lut)
    # reference tests' analytic cases (test_render.py:108-138)
    tilt = np.zeros((3, 6))
    tilt[:, 0] = 0.5
    tilt[0, 1] = 1.0
    xs = (np.arange(80) * 1e-4).astype(np.float32)
    v = np.broadcast_to(xs, (60, 80)).copy()
    out["tilt_d"] = v
    out["tilt_c"] = tilt
    out["tilt_rgb"] = depth_to_rgb(DepthImage(values=v.astype(np.float64), background=v),
                                   PolyLut(degree=2, coeffs=tilt, image_size=(80, 60)))
    xs = (np.arange(80) * 10.0).astype(np.float32)
    v = np.broadcast_to(xs, (60, 80)).copy()
    out["clamp_d"] = v
    out["clamp_rgb"] = depth_to_rgb(DepthImage(values=v.astype(np.float64), background=v),
                                    PolyLut(degree=2, coeffs=tilt, image_size=(80, 60)))
    np.savez_compressed(HERE / "rgb.npz", **out)


def peg_grid_reference():
    # small dims keep the fixture at ~0.25 MB; float64 values as build_sdf makes them
    return build_sdf(make_cylinder(0.008, 0.05, segments=32), dims=(16, 16, 32), padding=0.004)


def make_sdf(grid):
    rng = np.random.default_rng(7)
    lo, hi = grid.origin, grid.upper
    span = hi - lo
    pts = lo - 0.1 * span + rng.uniform(0, 1.2, (3000, 3)) * span   # ~half outside on some axis
    inside = lo + rng.uniform(0, 1, (2000, 3)) * span
    # exact boundary / corner points (rel == 0 and rel == dims-1)
    corners = np.array([lo, hi, [lo[0], hi[1], lo[2]], [hi[0], lo[1], hi[2]]])
    pts = np.concatenate([pts, inside, corners])
    q = query_sdf(grid, pts)
    np.savez_compressed(HERE / "sdf.npz", origin=grid.origin, spacing=grid.spacing, dims=np.array(grid.dims),
                        values=grid.values, gradients=grid.gradients, points=pts,
                        distance=q.distance, normal=q.normal, valid=q.valid)


def make_ff(grid):
    sensor = TactileSensorSpec(image_size=(320, 240))
    pts = sample_tactile_points(sensor, 20, 25)
    obj, sen = synthetic.peg_states(12, 1, config_id=103, random_sensor_pose=True)
    sen = sen[:, 0]
    params = PenaltyParams()
    fld, kin = compute_force_field(pts, grid, obj[:, 0:3], obj[:, 3:7], obj[:, 7:10], obj[:, 10:13],
                                   sen[:, 0:3], sen[:, 3:7], sen[:, 7:10], sen[:, 10:13], params,
                                   return_kinematics=True)
    force, torque = net_wrench(fld, pts)
    # one unbatched call (sensor at identity, object relative pose of env 0)
    o1, s1 = synthetic.peg_states(1, 1, config_id=104, random_sensor_pose=False)
    p2 = PenaltyParams(k_n=850.0, k_d=40.0, k_t=7.0, mu=1.3)
    fld1 = compute_force_field(pts, grid, o1[0, 0:3], o1[0, 3:7], o1[0, 7:10], o1[0, 10:13],
                               s1[0, 0, 0:3], s1[0, 0, 3:7], s1[0, 0, 7:10], s1[0, 0, 10:13], p2)
    np.savez_compressed(HERE / "ff.npz", points=pts.points, obj=obj, sen=sen,
                        f_n=fld.f_n, f_t=fld.f_t, d=kin["d"], d_dot=kin["d_dot"], v_t=kin["v_t"], n=kin["n"],
                        force=force, torque=torque, obj1=o1[0], sen1=s1[0, 0], params1=np.array(
                            [p2.k_n, p2.k_d, p2.k_t, p2.mu]), f_n1=fld1.f_n, f_t1=fld1.f_t)


def make_penalty():
    rng = np.random.default_rng(11)
    n_pts = 10000
    d = rng.uniform(-2e-3, 1e-3, n_pts)
    d_dot = rng.uniform(-0.5, 0.5, n_pts)
    n = rng.normal(size=(n_pts, 3))
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    v_t = rng.normal(size=(n_pts, 3)) * 0.05
    params = PenaltyParams(k_n=850.0, k_d=40.0, k_t=7.0, mu=1.3)
    f_n, f_t = penalty_forces(d, d_dot, n, v_t, params)
    sel = slice(0, 3000)
    np.savez_compressed(HERE / "penalty.npz", d=d[sel], d_dot=d_dot[sel], n=n[sel], v_t=v_t[sel],
                        params=np.array([params.k_n, params.k_d, params.k_t, params.mu]),
                        f_n=f_n[sel], f_t=f_t[sel])


def make_depth(grid):
    """render_depth (numba march, render/depth.py:88-134) on the reference
    peg grid: peg lying across the pad at several presses, one pose out of
    contact, one arbitrary rotation; 60x80 (E=6) and 240x320 (E=1)."""
    out = {}
    for (W, H), E in (((80, 60), 6), ((320, 240), 1)):
        sensor = TactileSensorSpec(image_size=(W, H))
        cam = camera_for_sensor(sensor)
        bg = reference_depth(cam, sensor)
        obj, sen = synthetic.peg_states(E, 1, config_id=105 + W, random_sensor_pose=False)
        pos, quat = obj[:, 0:3].copy(), obj[:, 3:7].copy()
        if E > 2:
            pos[-1, 2] += 0.01                                   # lifted: no contact
            quat[-2] = np.array([0.9, 0.2, -0.3, 0.25]) / np.linalg.norm([0.9, 0.2, -0.3, 0.25])
            pos[-2, 2] = 0.006
        img = render_depth(cam, grid, pos, quat, bg)
        key = f"{H}x{W}"
        out[f"bg_{key}"] = bg
        out[f"pos_{key}"] = pos
        out[f"quat_{key}"] = quat
        out[f"depth_{key}"] = img.values
    single = render_depth(camera_for_sensor(TactileSensorSpec()), grid, out["pos_60x80"][0], out["quat_60x80"][0],
                          out["bg_60x80"])
    out["depth_single"] = single.values
    np.savez_compressed(HERE / "depth.npz", **out)


def make_formats():
    """Files written by the reference's own writers: LUT text
    (render/lut.py:122-137) and TFF1 frames (tactile/io.py:13-23)."""
    from gelsim.render import write_lut
    from gelsim.tactile import ForceField, write_force_field_frames

    lut = synthetic_lut((320, 240), degree=3, seed=4)
    lut.sensor_id = "gelpad-A"
    lut.calibrated_on = "2026-01-15"
    lut.residual_rms = 0.00123
    write_lut(lut, HERE / "ref.lut")
    z = np.load(HERE / "ff.npz")
    frames = [ForceField(f_n=z["f_n"][e], f_t=z["f_t"][e]) for e in (0, 1)]
    write_force_field_frames(HERE / "ref.tff", frames)


AUG_CFGS = {
    "full": dict(shift_px=2.5, zoom=(1.05, 1.2), brightness=0.1, contrast=(0.8, 1.2), saturation=(0.7, 1.3),
                 hue=0.05, channel_permutation=True, step_brightness=0.02, step_contrast=(0.95, 1.05),
                 step_saturation=(0.9, 1.1), step_hue=0.01, seed=3),
    "color": dict(shift_px=0.0, zoom=(1.0, 1.0), brightness=0.2, contrast=(0.5, 1.5), saturation=(0.2, 1.8),
                  hue=0.5, channel_permutation=False, step_brightness=0.0, step_contrast=(1.0, 1.0),
                  step_saturation=(1.0, 1.0), step_hue=0.0, seed=11),
    "spatial": dict(shift_px=6.0, zoom=(0.7, 1.4), brightness=0.0, contrast=(1.0, 1.0), saturation=(1.0, 1.0),
                    hue=0.0, channel_permutation=True, step_brightness=0.0, step_contrast=(1.0, 1.0),
                    step_saturation=(1.0, 1.0), step_hue=0.0, seed=0),
    "identity": dict(shift_px=0.0, zoom=(1.0, 1.0), brightness=0.0, contrast=(1.0, 1.0), saturation=(1.0, 1.0),
                     hue=0.0, channel_permutation=False, step_brightness=0.0, step_contrast=(1.0, 1.0),
                     step_saturation=(1.0, 1.0), step_hue=0.0, seed=5),
}
AUG_SEEDS = [(0, 0), (17, 3), (2 ** 33 + 12345, 123), (987654321, 7)]


def make_augment():
    """render/augment.py:156-173 on float32 tactile images (the env applies
    it to depth_to_rgb(...).astype(float32), envs/peg_tasks.py:445-452)."""
    from gelsim.render import AugmentConfig, augment

    out = {}
    for size in ((80, 60), (40, 30)):
        d, bg = depth_maps(size[0], size[1], len(AUG_SEEDS), config_id=106)
        lut = scaled_lut(size, 2, seed=0, s=synthetic.lut_scale(size))
        imgs = depth_to_rgb(DepthImage(values=d.astype(np.float64), background=bg), lut).astype(np.float32)
        key = f"{size[1]}x{size[0]}"
        out[f"img_{key}"] = imgs
        for name, kw in AUG_CFGS.items():
            cfg = AugmentConfig(**kw)
            out[f"aug_{name}_{key}"] = np.stack([augment(imgs[i], cfg, ep, st)
                                                 for i, (ep, st) in enumerate(AUG_SEEDS)])
    np.savez_compressed(HERE / "augment.npz", **out)


def make_env():
    """PegEnvBatch tactile observations (envs/peg_tasks.py:434-477) after a
    reset and two zero-action steps, with augmentation and the "diff"
    representation, plus every input needed to recompute them on the device:
    the per-sensor depth maps the env renders (render_depth, as
    _tactile_images does), the peg / sensor states _tactile_ff passes, the
    per-env augmentation seeds and step counts, the LUT and taxel grid."""
    from gelsim.envs.base import EnvConfig
    from gelsim.envs.peg_tasks import PEG, PegEnvBatch
    from gelsim.render.augment import AugmentConfig
    from gelsim.transforms import quat_conj, quat_mul, quat_rotate_inv

    aug = AugmentConfig(shift_px=1.5, zoom=(0.95, 1.08), brightness=0.05, contrast=(0.9, 1.1),
                        saturation=(0.85, 1.15), hue=0.02, channel_permutation=True, step_brightness=0.01,
                        step_contrast=(0.98, 1.02), step_saturation=(0.97, 1.03), step_hue=0.005, seed=7)
    E = 6
    cfg = EnvConfig(num_envs=E, seed=3, tactile_rep="diff", augment=aug,
                    obs_modalities=("tactile_img", "tactile_ff"))
    env = PegEnvBatch(cfg)
    env.reset()
    for _ in range(2):
        env.step(np.zeros((E, 6)))
    images = env._tactile_images()
    ff = env._tactile_ff()
    depth, sen, rel_p, rel_q = [], [], [], []
    for s_idx in range(2):
        pos, quat = env._sensor_world_pose(s_idx)
        rel_pos = quat_rotate_inv(quat, env.bodies.pos[:, PEG] - pos)
        rel_quat = quat_mul(quat_conj(quat), env.bodies.quat[:, PEG])
        rel_p.append(rel_pos)
        rel_q.append(rel_quat)
        depth.append(render_depth(env.camera, env.peg_sdf, rel_pos, rel_quat, env.background).values)
        v, w = env._sensor_world_velocity(pos)
        sen.append(np.concatenate([pos, quat, v, w], axis=1))
    obj = np.concatenate([env.bodies.pos[:, PEG], env.bodies.quat[:, PEG], env.bodies.linvel[:, PEG],
                          env.bodies.angvel[:, PEG]], axis=1)
    g = env.peg_sdf  # the env's own build_sdf peg (32x32x64, float64)
    p = cfg.penalty
    np.savez_compressed(
        HERE / "env.npz", images=images, ff=ff, depth=np.stack(depth, axis=1), obj=obj,
        rel_pos=np.stack(rel_p, axis=1), rel_quat=np.stack(rel_q, axis=1), background=env.background,
        cam_dirs=env.camera.rays(),
        sen=np.stack(sen, axis=1), seeds=(env.env_seeds * 1000003 + env.episode).astype(np.int64),
        steps=env.step_count.astype(np.int64), env_seeds=env.env_seeds.astype(np.int64),
        episode=env.episode.astype(np.int64), lut_coeffs=env.lut.coeffs, lut_degree=env.lut.degree,
        image_size=np.array(cfg.tactile_image_size), ff_points=env.ff_grid.points,
        penalty=np.array([p.k_n, p.k_d, p.k_t, p.mu]),
        sdf_origin=np.asarray(g.origin), sdf_spacing=np.float64(g.spacing), sdf_dims=np.array(g.dims),
        sdf_values=g.values, sdf_gradients=g.gradients,
        aug=np.array([aug.shift_px, aug.zoom[0], aug.zoom[1], aug.brightness, aug.contrast[0], aug.contrast[1],
                      aug.saturation[0], aug.saturation[1], aug.hue, float(aug.channel_permutation),
                      aug.step_brightness, aug.step_contrast[0], aug.step_contrast[1], aug.step_saturation[0],
                      aug.step_saturation[1], aug.step_hue, aug.seed]))


def make_scene(grid):
    """envs/scenes.py:27-57 shape_sensing_scene end to end (render_depth ->
    depth_to_rgb, compute_force_field) for four batched peg presses on the
    reference-built 16x16x32 peg grid of sdf.npz."""
    from gelsim.envs.scenes import shape_sensing_scene
    from gelsim.transforms import quat_from_axis_angle

    rng = np.random.default_rng(np.random.SeedSequence((20240812, 77)))
    E = 4
    pos = np.stack([rng.uniform(-0.002, 0.002, E), rng.uniform(-0.002, 0.002, E),
                    0.008 - rng.uniform(0.0002, 0.0009, E)], axis=1)
    ang = np.pi / 2 + rng.uniform(-0.1, 0.1, E)
    quat = quat_from_axis_angle(np.tile([0.0, 1.0, 0.0], (E, 1)), ang)
    rgb, fld = shape_sensing_scene(grid, pos, quat, num_envs=E)
    np.savez_compressed(HERE / "scene.npz", press_pos=pos, press_quat=quat, rgb=rgb.astype(np.float32),
                        f_n=fld.f_n, f_t=fld.f_t)


def make_extras(grid):
    from gelsim.errors import InvalidQuery
    from gelsim.geometry import relative_penetration_rate
    from gelsim.render.camera import TactileCamera
    from gelsim.transforms import quat_from_axis_angle

    sensor = TactileSensorSpec(image_size=(80, 60))
    base = camera_for_sensor(sensor)
    quat = quat_from_axis_angle(np.array([0.3, -0.5, 0.8]), 0.21)
    cam = TactileCamera(pos=base.pos, quat=quat, fx=base.fx, fy=base.fy, cx=base.cx, cy=base.cy,
                        width=base.width, height=base.height, near=base.near, far=base.far)
    rays = cam.rays()
    bg = reference_depth(cam, sensor)
    rng = np.random.default_rng(9)
    lo, hi = grid.origin, grid.upper
    inside = lo + rng.uniform(0.01, 0.99, (500, 3)) * (hi - lo)
    q = query_sdf(grid, inside)
    x_dot = rng.normal(0.0, 0.05, (500, 3))
    rate = relative_penetration_rate(q, x_dot)
    x1 = np.array([0.01, -0.02, 0.03])
    rate1 = relative_penetration_rate(q, x1)
    mixed = np.concatenate([inside[:10], [hi + 0.01]])
    try:
        relative_penetration_rate(query_sdf(grid, mixed), x_dot[:11])
        raised = False
    except InvalidQuery:
        raised = True
    # curved gel: the reference test's dome mesh (test_tactile_field.py:68-79)
    from gelsim.geometry.mesh import TriMesh
    from gelsim.tactile import sample_tactile_points as ref_points
    n_d, rad, ext = 24, 0.05, 0.016
    gxs = np.linspace(-ext, ext, n_d)
    gx, gy = np.meshgrid(gxs, gxs, indexing="xy")
    gz = np.sqrt(rad ** 2 - gx ** 2 - gy ** 2) - rad
    dverts = np.stack([gx, gy, gz], axis=-1).reshape(-1, 3)
    dfaces = np.array([[r * n_d + c, r * n_d + c + 1, r * n_d + c + n_d] for r in range(n_d - 1)
                       for c in range(n_d - 1)] + [[r * n_d + c + 1, r * n_d + c + n_d + 1, r * n_d + c + n_d]
                                                   for r in range(n_d - 1) for c in range(n_d - 1)])
    dome = TriMesh(dverts, dfaces)
    curved = TactileSensorSpec(active_area=(0.02, 0.02), surface_mesh=dome, image_size=(80, 60))
    cgrid = ref_points(curved, 12, 12)
    curved_bg = reference_depth(camera_for_sensor(curved), curved)
    np.savez_compressed(HERE / "extras.npz", dome_vertices=dverts, dome_faces=dfaces,
                        curved_points=cgrid.points, curved_normals=cgrid.rest_normals, curved_background=curved_bg,
                        cam_quat=quat, cam_pos=cam.pos, cam_f=np.array([cam.fx, cam.fy]),
                        cam_c=np.array([cam.cx, cam.cy]), rays=rays, background=bg, points=inside, x_dot=x_dot,
                        rate=rate, x1=x1, rate1=rate1, mixed=mixed, mixed_raises=np.array(raised))


if __name__ == "__main__" and len(sys.argv) > 1:
    for name in sys.argv[1:]:
        fn = globals()[f"make_{name}"]
        fn(peg_grid_reference()) if name in ("sdf", "ff", "depth", "scene", "extras") else fn()
elif __name__ == "__main__":
    make_augment()
    make_rgb()
    g = peg_grid_reference()
    make_sdf(g)
    make_ff(g)
    make_penalty()
    make_depth(g)
    make_formats()
    make_env()
    make_scene(g)
    make_extras(g)
    for p in sorted(HERE.glob("*.npz")):
        print(p.name, p.stat().st_size)
