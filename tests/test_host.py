"""Host-side logic that needs no GPU: sharding, state broadcasting, patch(),
synthetic inputs, TSDF round trip."""
import sys
import types

import numpy as np
import pytest

from paper_2408_06506_b200 import geometry, patching as patch, pipeline, synthetic, tactile
from paper_2408_06506_b200.render import PolyLut


@pytest.mark.parametrize("n,world", [(4096, 1), (4096, 2), (4096, 8), (10, 3), (3, 8), (0, 2)])
def test_shard_range_partitions(n, world):
    spans = [pipeline.shard_range(n, r, world) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == n
    for (a, b), (c, d) in zip(spans, spans[1:]):
        assert b == c
    sizes = [b - a for a, b in spans]
    assert max(sizes) - min(sizes) <= 1


def test_state_broadcast():
    s = tactile._state_array(np.zeros(3), [1, 0, 0, 0], np.zeros((4, 3)), np.zeros(3), 4, "x")
    assert s.shape == (4, 13) and np.all(s[:, 3] == 1)
    with pytest.raises(ValueError):
        tactile._state_array(np.zeros((3, 3)), [1, 0, 0, 0], np.zeros(3), np.zeros(3), 4, "x")


def test_patch_rebinds_every_import_site(monkeypatch):
    names = {}
    for mod_name, fns in patch._SITES.items():
        m = types.ModuleType(mod_name)
        for f in fns:
            setattr(m, f, lambda *a, **k: "reference")
        names[mod_name] = m
        monkeypatch.setitem(sys.modules, mod_name, m)
    done = patch.patch()
    assert len(done) == sum(len(v) for v in patch._SITES.values())
    from paper_2408_06506_b200 import render
    assert sys.modules["gelsim.envs.peg_tasks"].depth_to_rgb is render.depth_to_rgb
    assert sys.modules["gelsim.tactile.field"].compute_force_field is tactile.compute_force_field
    patch.unpatch()
    assert sys.modules["gelsim.envs.scenes"].compute_force_field() == "reference"


def test_peg_states_relative_pose():
    obj, sen = synthetic.peg_states(5, 2, config_id=9)
    assert obj.shape == (5, 13) and sen.shape == (5, 2, 13)
    np.testing.assert_allclose(np.linalg.norm(obj[:, 3:7], axis=-1), 1.0, atol=1e-12)
    np.testing.assert_allclose(np.linalg.norm(sen[..., 3:7], axis=-1), 1.0, atol=1e-12)
    # the peg axis lies (nearly) in each sensor's xy plane
    from oracle.gelsim_oracle import quat_rotate, quat_rotate_inv
    axis_w = quat_rotate(obj[:, None, 3:7], np.array([0.0, 0.0, 1.0]))
    axis_s = quat_rotate_inv(sen[..., 3:7], axis_w)
    assert np.all(np.abs(axis_s[..., 2]) < np.sin(0.11))


def test_depth_batch_deterministic_and_pooled():
    _, cam, bg, _, _ = synthetic.sensor_setup((80, 60))
    a = synthetic.depth_batch(cam, bg, 6, config_id=3)
    b = synthetic.depth_batch(cam, bg, 6, config_id=3)
    assert a.dtype == np.float32 and np.array_equal(a, b)
    assert np.all(a <= bg.astype(np.float32) + 1e-9)
    assert (a < bg - 1e-6).any()
    c = synthetic.depth_batch(cam, bg, 6, config_id=3, pool=2)
    assert np.array_equal(c[2], c[0])


def test_tsdf_roundtrip(tmp_path):
    g = geometry.box_grid(dims=(12, 12, 10))
    p = tmp_path / "g.tsdf"
    geometry.write_sdf_cache(g, p)
    back = geometry.read_sdf_cache(p)
    assert back.dims == g.dims
    np.testing.assert_array_equal(back.values, g.values)  # grids are float32-representable
    assert p.read_bytes()[:4] == b"TSDF"


def test_analytic_grid_layout_matches_build_sdf_rule():
    g = synthetic.peg_grid((32, 32, 64))
    # build_sdf: spacing = max(extent / (dims - 1)), extent = bounds + 2*padding
    assert g.spacing == pytest.approx(max(0.024 / 31, 0.058 / 63))
    np.testing.assert_allclose(g.origin + g.spacing * (np.array(g.dims) - 1) / 2, 0.0, atol=1e-15)


def test_polylut_validation():
    with pytest.raises(ValueError):
        PolyLut(degree=5, coeffs=np.zeros((3, 21)), image_size=(8, 8))


def test_reference_depth_bit_identical_to_env_background():
    """The membrane depth (ray cast against the pad's two triangles) equals
    the background the reference env computed (tests/golden/env.npz)."""
    from conftest import GOLDEN
    from paper_2408_06506_b200.sensors import TactileSensorSpec, camera_for_sensor, reference_depth
    z = np.load(GOLDEN / "env.npz")
    spec = TactileSensorSpec(image_size=tuple(int(v) for v in z["image_size"]))
    cam = camera_for_sensor(spec)
    assert np.array_equal(cam.rays(), z["cam_dirs"])
    assert np.array_equal(reference_depth(cam, spec), z["background"])


def test_host_quaternion_helpers_match_the_oracle_bit_for_bit():
    """transforms.py (used for the env's relative peg poses) against the
    oracle's restatement of transforms.py:17-47, on random inputs."""
    from oracle import gelsim_oracle as O
    from paper_2408_06506_b200 import transforms as T
    rng = np.random.default_rng(11)
    q = rng.normal(size=(257, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    v = rng.normal(size=(257, 3))
    assert np.array_equal(T.quat_rotate(q, v), O.quat_rotate(q, v))
    assert np.array_equal(T.quat_rotate_inv(q, v), O.quat_rotate_inv(q, v))
    r = rng.normal(size=(257, 4))
    a, b = q, r
    aw, ax, ay, az = a.T
    bw, bx, by, bz = b.T
    ref = np.stack([aw * bw - ax * bx - ay * by - az * bz, aw * bx + ax * bw + ay * bz - az * by,
                    aw * by - ax * bz + ay * bw + az * bx, aw * bz + ax * by - ay * bx + az * bw], axis=-1)
    assert np.array_equal(T.quat_mul(a, b), ref)
    assert np.array_equal(T.quat_conj(q), q * np.array([1.0, -1.0, -1.0, -1.0]))


def test_rotated_camera_rays_and_background_bit_exact(golden):
    """TactileCamera.quat rotates the rays (render/camera.py:17,43); rays and
    the membrane depth of a rotated camera equal the reference's bit for bit."""
    from paper_2408_06506_b200.sensors import TactileCamera, TactileSensorSpec, reference_depth
    z = golden("extras")
    cam = TactileCamera(pos=z["cam_pos"], quat=z["cam_quat"], fx=float(z["cam_f"][0]), fy=float(z["cam_f"][1]),
                        cx=float(z["cam_c"][0]), cy=float(z["cam_c"][1]), width=80, height=60)
    np.testing.assert_array_equal(cam.rays(), z["rays"])
    np.testing.assert_array_equal(reference_depth(cam, TactileSensorSpec(image_size=(80, 60))), z["background"])


def test_camera_validation_and_identity_quat():
    import pytest
    from paper_2408_06506_b200.sensors import TactileCamera
    with pytest.raises(ValueError):
        TactileCamera(width=0)
    with pytest.raises(ValueError):
        TactileCamera(near=0.5, far=0.1)
    cam = TactileCamera()
    u = (np.arange(80) + 0.5 - 40.0) / 66.7
    v = (np.arange(60) + 0.5 - 30.0) / 66.7
    gu, gv = np.meshgrid(u, v, indexing="xy")
    d = np.stack([gu, gv, np.ones_like(gu)], axis=-1)
    np.testing.assert_array_equal(cam.rays(), d / np.linalg.norm(d, axis=-1, keepdims=True))


def _dome(golden):
    from paper_2408_06506_b200.sensors import SurfaceMesh, TactileSensorSpec
    z = golden("extras")
    mesh = SurfaceMesh(z["dome_vertices"], z["dome_faces"])
    return z, TactileSensorSpec(active_area=(0.02, 0.02), surface_mesh=mesh, image_size=(80, 60))


def test_curved_pad_taxels_normals_and_background_bit_exact(golden):
    """Curved gel (sensors.py:32,39-50; points.py:59-80; camera.py:56-66):
    taxels dropped onto the surface mesh, their nearest-face normals and the
    membrane depth equal the reference's bit for bit (the reference test's
    dome mesh, tests/test_tactile_field.py:68-79)."""
    from paper_2408_06506_b200.sensors import camera_for_sensor, reference_depth
    from paper_2408_06506_b200.tactile import sample_tactile_points
    z, sensor = _dome(golden)
    assert not sensor.is_flat()
    g = sample_tactile_points(sensor, 12, 12)
    np.testing.assert_array_equal(g.points, z["curved_points"])
    np.testing.assert_array_equal(g.rest_normals, z["curved_normals"])
    np.testing.assert_array_equal(reference_depth(camera_for_sensor(sensor), sensor), z["curved_background"])


def test_curved_pad_errors(golden):
    import pytest
    from paper_2408_06506_b200.errors import ResolutionTooFine
    from paper_2408_06506_b200.sensors import TactileSensorSpec
    from paper_2408_06506_b200.tactile import sample_tactile_points
    z, sensor = _dome(golden)
    with pytest.raises(ResolutionTooFine):  # points.py:40-45
        sample_tactile_points(sensor, 200, 200)
    wide = TactileSensorSpec(active_area=(0.04, 0.04), surface_mesh=sensor.surface_mesh)
    with pytest.raises(ValueError):  # points.py:63-64
        sample_tactile_points(wide, 8, 8)
    flat = TactileSensorSpec()
    assert flat.is_flat() and sample_tactile_points(flat, 3, 4).points[..., 2].max() == 0.0
