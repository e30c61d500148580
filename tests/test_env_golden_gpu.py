"""The whole tactile observation chain of the reference env, against the
env itself: tests/golden/env.npz holds PegEnvBatch._tactile_images /
_tactile_ff outputs (envs/peg_tasks.py:434-477) recorded by running the
REFERENCE env (6 envs x 2 fingers, augmentation on, "diff" representation,
its own build_sdf peg) plus the inputs the env used.  Here:

* K3 render_depth of the env's relative peg poses reproduces the env's depth
  maps bit for bit;
* TactileObservations (K1 float epilogue + K4 augmentation + K2 packed
  force-field observation) reproduces the observations: images within one
  uint8 step (the fp32 shading differs from the reference's fp64 by <= 1e-6
  and the HSV round trip passes that through), force-field observation within
  1e-5 relative with the contact mask exact.
"""
import numpy as np
import pytest
import torch

from conftest import GOLDEN, vec_close
from paper_2408_06506_b200 import AugmentConfig
from paper_2408_06506_b200.depth import render_depth
from paper_2408_06506_b200.geometry import SdfGrid
from paper_2408_06506_b200.pipeline import TactileObservations
from paper_2408_06506_b200.render import PolyLut
from paper_2408_06506_b200.sensors import TactileSensorSpec, camera_for_sensor, reference_depth
from paper_2408_06506_b200.tactile import PenaltyParams, TactilePointGrid

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    z = dict(np.load(GOLDEN / "env.npz"))
    z["sdf"] = SdfGrid(origin=z["sdf_origin"], spacing=float(z["sdf_spacing"]), dims=tuple(int(v) for v in z["sdf_dims"]),
                       values=z["sdf_values"], gradients=z["sdf_gradients"])
    z["lut"] = PolyLut(degree=int(z["lut_degree"]), coeffs=z["lut_coeffs"],
                       image_size=tuple(int(v) for v in z["image_size"]))
    return z


def test_env_depth_bit_exact(env):
    W, H = (int(v) for v in env["image_size"])
    spec = TactileSensorSpec(image_size=(W, H))
    cam = camera_for_sensor(spec)
    bg = reference_depth(cam, spec)
    for s in range(2):
        d = render_depth(cam, env["sdf"], env["rel_pos"][:, s], env["rel_quat"][:, s], bg)
        assert np.array_equal(d.values, env["depth"][:, s]), s


def test_env_tactile_observations(env):
    a = env["aug"]
    cfg = AugmentConfig(shift_px=a[0], zoom=(a[1], a[2]), brightness=a[3], contrast=(a[4], a[5]),
                        saturation=(a[6], a[7]), hue=a[8], channel_permutation=bool(a[9]), step_brightness=a[10],
                        step_contrast=(a[11], a[12]), step_saturation=(a[13], a[14]), step_hue=a[15],
                        seed=int(a[16]))
    pts = env["ff_points"]
    grid = TactilePointGrid(points=pts, rest_normals=np.broadcast_to([0.0, 0.0, 1.0], pts.shape).copy(),
                            spacing=(float(pts[0, 1, 0] - pts[0, 0, 0]), float(pts[1, 0, 1] - pts[0, 0, 1])))
    E = env["obj"].shape[0]
    obs = TactileObservations(env["lut"], env["sdf"], grid, PenaltyParams(*env["penalty"]), E, 2, tactile_rep="diff",
                              augment=cfg)
    depth = torch.from_numpy(env["depth"].astype(np.float32)).cuda()
    images, ff = obs(depth, torch.from_numpy(env["obj"]).cuda(), torch.from_numpy(np.ascontiguousarray(env["sen"])).cuda(),
                     episode_seeds=env["seeds"], step_indices=env["steps"])
    torch.cuda.synchronize()
    got = images.cpu().numpy()
    ref = env["images"]
    diff = np.abs(got - ref)
    assert diff.max() <= 1.0 / 255.0, diff.max()
    assert (diff > 1e-5).mean() < 0.01, (diff > 1e-5).mean()
    f = ff.cpu().numpy()
    assert np.array_equal(np.abs(f).sum(-1) > 0, np.abs(env["ff"]).sum(-1) > 0)
    assert (np.abs(env["ff"]).sum(-1) > 0).mean() > 0.05
    assert vec_close(f, env["ff"], 1e-5, atol=1e-7)[0]


def test_shape_sensing_scene_end_to_end(golden_grid):
    """envs/scenes.py:27-57 shape_sensing_scene recomputed with this package's
    drop-ins (render_depth -> depth_to_rgb, compute_force_field) against the
    reference's own output (tests/golden/scene.npz)."""
    from oracle.gelsim_oracle import to_uint8
    from paper_2408_06506_b200.render import depth_to_rgb, synthetic_lut
    from paper_2408_06506_b200.sensors import IDENTITY_QUAT
    from paper_2408_06506_b200.tactile import compute_force_field, sample_tactile_points
    z = np.load(GOLDEN / "scene.npz")
    spec = TactileSensorSpec()
    cam = camera_for_sensor(spec)
    bg = reference_depth(cam, spec)
    lut = synthetic_lut(spec.image_size)
    depth = render_depth(cam, golden_grid, z["press_pos"], z["press_quat"], bg)
    rgb = depth_to_rgb(depth, lut)
    assert rgb.dtype == np.float64 and rgb.shape == z["rgb"].shape
    assert np.abs(rgb - z["rgb"]).max() < 1e-5
    assert np.abs(to_uint8(rgb).astype(int) - to_uint8(z["rgb"].astype(np.float64)).astype(int)).max() <= 1
    zeros = np.zeros_like(z["press_pos"])
    fld = compute_force_field(sample_tactile_points(spec, 10, 14), golden_grid, z["press_pos"], z["press_quat"],
                              zeros, zeros, np.zeros(3), IDENTITY_QUAT, np.zeros(3), np.zeros(3), PenaltyParams())
    assert np.array_equal(np.linalg.norm(fld.f_n, axis=-1) > 0, np.linalg.norm(z["f_n"], axis=-1) > 0)
    assert vec_close(fld.f_n, z["f_n"], 1e-5)[0]
    assert vec_close(fld.f_t, z["f_t"], 1e-5)[0]


def _standin_env(env, aug_cfg):
    """An object with exactly the attributes PegEnvBatch._tactile_images /
    _tactile_ff read, filled from the recorded reference env."""
    from types import SimpleNamespace

    from paper_2408_06506_b200.envs import PEG
    E = env["obj"].shape[0]
    W, H = (int(v) for v in env["image_size"])
    spec = TactileSensorSpec(image_size=(W, H))
    cam = camera_for_sensor(spec)
    bodies = SimpleNamespace(pos=np.zeros((E, 4, 3)), quat=np.zeros((E, 4, 4)), linvel=np.zeros((E, 4, 3)),
                             angvel=np.zeros((E, 4, 3)))
    bodies.pos[:, PEG], bodies.quat[:, PEG] = env["obj"][:, 0:3], env["obj"][:, 3:7]
    bodies.linvel[:, PEG], bodies.angvel[:, PEG] = env["obj"][:, 7:10], env["obj"][:, 10:13]
    pts = env["ff_points"]
    grid = TactilePointGrid(points=pts, rest_normals=np.broadcast_to([0.0, 0.0, 1.0], pts.shape).copy(),
                            spacing=(1.0, 1.0))
    sen = env["sen"]
    cfg = SimpleNamespace(tactile_image_size=(W, H), tactile_ff_grid=pts.shape[:2], tactile_rep="diff",
                          augment=aug_cfg, penalty=PenaltyParams(*env["penalty"]))
    return SimpleNamespace(
        cfg=cfg, num_envs=E, camera=cam, background=reference_depth(cam, spec), peg_sdf=env["sdf"],
        lut=env["lut"], env_seeds=env["env_seeds"], episode=env["episode"], step_count=env["steps"],
        bodies=bodies, ff_grid=grid,
        _sensor_world_pose=lambda s: (sen[:, s, 0:3], sen[:, s, 3:7]),
        _sensor_world_velocity=lambda p: next((sen[:, s, 7:10], sen[:, s, 10:13]) for s in range(2)
                                              if np.array_equal(p, sen[:, s, 0:3])))


def test_batched_env_methods_reproduce_the_env(env):
    """envs.tactile_images / tactile_ff (what patch() binds as
    PegEnvBatch._tactile_images / _tactile_ff) on an object carrying the
    recorded env's state reproduce the env's own observations."""
    from paper_2408_06506_b200 import envs
    a = env["aug"]
    cfg = AugmentConfig(shift_px=a[0], zoom=(a[1], a[2]), brightness=a[3], contrast=(a[4], a[5]),
                        saturation=(a[6], a[7]), hue=a[8], channel_permutation=bool(a[9]), step_brightness=a[10],
                        step_contrast=(a[11], a[12]), step_saturation=(a[13], a[14]), step_hue=a[15],
                        seed=int(a[16]))
    e = _standin_env(env, cfg)
    images = envs.tactile_images(e)
    assert images.dtype == np.float32 and images.shape == env["images"].shape
    diff = np.abs(images - env["images"])
    assert diff.max() <= 1.0 / 255.0 and (diff > 1e-5).mean() < 0.01
    ff = envs.tactile_ff(e)
    assert ff.dtype == np.float32 and ff.shape == env["ff"].shape
    assert np.array_equal(np.abs(ff).sum(-1) > 0, np.abs(env["ff"]).sum(-1) > 0)
    assert vec_close(ff, env["ff"], 1e-5, atol=1e-7)[0]
    # second step reuses the cached device state
    assert np.array_equal(envs.tactile_images(e), images)


def _world_poses(sen, obj):
    """(E, 7 * S + 7) rows for env_render_params_device: sensor pos + quat,
    then the object's."""
    E, S = sen.shape[:2]
    return np.concatenate([sen[:, :, 0:7].reshape(E, 7 * S), obj[:, 0:7]], axis=1)


def test_env_render_params_on_device_bit_exact(env):
    """The env's per-step host pose math on the device (K3's inputs): the
    object pose in each finger's frame equals the reference env's recorded
    relative pose bit for bit, R / AABB equal the host env_params of it, and
    K3 fed straight from the device rows reproduces the env's depth maps."""
    from paper_2408_06506_b200.depth import RayTable, env_params, env_render_params_device, render_depth_device
    sdf = env["sdf"]
    poses = torch.from_numpy(_world_poses(env["sen"], env["obj"])).cuda()
    got = env_render_params_device(sdf, poses, 2).cpu().numpy()
    assert np.array_equal(got[:, 0:3], env["rel_pos"].reshape(-1, 3))
    host = env_params(sdf, env["rel_pos"].reshape(-1, 3), env["rel_quat"].reshape(-1, 4))
    assert np.array_equal(got, host)
    W, H = (int(v) for v in env["image_size"])
    spec = TactileSensorSpec(image_size=(W, H))
    cam = camera_for_sensor(spec)
    rays = RayTable(cam, reference_depth(cam, spec), "cuda")
    depth = torch.empty((got.shape[0], H, W), dtype=torch.float64, device="cuda")
    render_depth_device(rays, sdf, torch.from_numpy(got).cuda(), out_f64=depth)
    assert np.array_equal(depth.cpu().numpy().reshape(env["depth"].shape), env["depth"])


@pytest.mark.parametrize("scale", [1e-3, 1.0, 30.0])
def test_env_render_params_random_poses(env, scale):
    """Random world poses (unnormalised quaternions, several magnitudes):
    the device rows equal the host restatement (envs._relative_peg_poses +
    depth.env_params, numpy's float64 order) bit for bit."""
    from types import SimpleNamespace

    from paper_2408_06506_b200.depth import env_params, env_render_params_device
    from paper_2408_06506_b200.envs import PEG, _relative_peg_poses
    rng = np.random.default_rng(int(scale * 1000) + 5)
    E, S = 777, 2
    sen = np.concatenate([rng.normal(size=(E, S, 3)) * scale, rng.normal(size=(E, S, 4)) * 0.7], axis=2)
    obj = np.concatenate([rng.normal(size=(E, 3)) * scale, rng.normal(size=(E, 4)) * 1.3], axis=1)
    pos = np.zeros((E, 4, 3))
    quat = np.zeros((E, 4, 4))
    pos[:, PEG], quat[:, PEG] = obj[:, 0:3], obj[:, 3:7]
    fake = SimpleNamespace(bodies=SimpleNamespace(pos=pos, quat=quat),
                           _sensor_world_pose=lambda s: (sen[:, s, 0:3], sen[:, s, 3:7]))
    rp, rq = _relative_peg_poses(fake)
    host = env_params(env["sdf"], rp.reshape(-1, 3), rq.reshape(-1, 4))
    got = env_render_params_device(env["sdf"], torch.from_numpy(_world_poses(sen, obj)).cuda(), S).cpu().numpy()
    assert np.array_equal(got, host)


def test_env_render_params_shapes_and_errors(env):
    """One sensor per env, an empty batch, and malformed pose tables."""
    from paper_2408_06506_b200.depth import env_params, env_render_params_device
    sen, obj = env["sen"][:, :1], env["obj"]
    got = env_render_params_device(env["sdf"], torch.from_numpy(_world_poses(sen, obj)).cuda(), 1).cpu().numpy()
    assert np.array_equal(got, env_params(env["sdf"], env["rel_pos"][:, 0], env["rel_quat"][:, 0]))
    empty = env_render_params_device(env["sdf"], torch.zeros((0, 21), dtype=torch.float64, device="cuda"), 2)
    assert empty.shape == (0, 18)
    with pytest.raises(ValueError):
        env_render_params_device(env["sdf"], torch.zeros((3, 20), dtype=torch.float64, device="cuda"), 2)
    with pytest.raises(ValueError):
        env_render_params_device(env["sdf"], torch.zeros((3, 21), dtype=torch.float32, device="cuda"), 2)


@pytest.mark.parametrize("rep", ["color", "diff", "concat"])
def test_batched_env_images_without_augmentation(env, rep):
    """envs.tactile_images with augmentation off, in each representation
    (envs/peg_tasks.py:445-458): the reference env's recorded depth maps
    shaded by the CPU restatement, cast to float32, then "diff" subtracts
    and "concat" appends the LUT's background colour."""
    from oracle import gelsim_oracle as O
    from paper_2408_06506_b200 import envs
    e = _standin_env(env, None)
    e.cfg.tactile_rep = rep
    got = envs.tactile_images(e)
    rgb = O.depth_to_rgb(env["depth"], env["lut_coeffs"], int(env["lut_degree"])).astype(np.float32)
    nominal = env["lut_coeffs"][:, 0].astype(np.float32)
    if rep == "diff":
        ref = rgb - nominal
    elif rep == "concat":
        ref = np.concatenate([rgb, np.broadcast_to(nominal, rgb.shape)], axis=-1)
    else:
        ref = rgb
    assert got.dtype == np.float32 and got.shape == ref.shape
    np.testing.assert_allclose(got, ref, rtol=0, atol=2e-6)
