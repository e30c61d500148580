"""K3 (render_depth, SDF sphere tracer) on the GPU: bit-identical to the
reference's float64 numba march (golden vectors), plus the reference's own
render tests (pkg/tests/test_render.py:44-95) re-pinned on the GPU path."""
import numpy as np
import pytest

from oracle import gelsim_oracle as O
from paper_2408_06506_b200 import geometry
from paper_2408_06506_b200.depth import render_depth
from paper_2408_06506_b200.sensors import IDENTITY_QUAT, TactileSensorSpec, camera_for_sensor, reference_depth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("size", [(80, 60), (320, 240)])
def test_render_depth_golden_bit_exact(golden, golden_grid, size):
    z = golden("depth")
    W, H = size
    cam = camera_for_sensor(TactileSensorSpec(image_size=size))
    k = f"{H}x{W}"
    img = render_depth(cam, golden_grid, z["pos_" + k], z["quat_" + k], z["bg_" + k])
    assert img.values.shape == z["depth_" + k].shape and img.values.dtype == np.float64
    assert np.array_equal(img.values, z["depth_" + k])
    assert np.array_equal(img.background, z["bg_" + k])


def test_render_depth_unbatched_golden(golden, golden_grid):
    z = golden("depth")
    cam = camera_for_sensor(TactileSensorSpec())
    img = render_depth(cam, golden_grid, z["pos_60x80"][0], z["quat_60x80"][0], z["bg_60x80"])
    assert img.values.shape == (60, 80)
    assert np.array_equal(img.values, z["depth_single"])


@pytest.fixture(scope="module")
def scene():
    sensor = TactileSensorSpec()
    cam = camera_for_sensor(sensor)
    bg = reference_depth(cam, sensor)
    sphere = geometry.sphere_grid(0.005, dims=(64, 64, 64), padding=0.002)
    return cam, bg, sphere


def test_object_above_membrane_gives_exact_background(scene):
    cam, bg, sphere = scene
    img = render_depth(cam, sphere, np.array([0, 0, 0.0062]), IDENTITY_QUAT, bg)
    assert np.array_equal(img.values, bg)


def test_footprint_area_matches_sphere_cap(scene):
    cam, bg, sphere = scene
    delta = 0.0005
    img = render_depth(cam, sphere, np.array([0, 0, 0.005 - delta]), IDENTITY_QUAT, bg)
    indent = img.indentation() > 1e-6
    r_disk = np.sqrt(max(2 * 0.005 * delta - delta * delta, 0.0))
    expected_px = np.pi * r_disk ** 2 * (cam.fx / 0.02) ** 2
    assert indent.sum() == pytest.approx(expected_px, rel=0.05)


def test_translation_shifts_footprint_by_projection(scene):
    cam, bg, sphere = scene
    delta, dx = 0.0005, 0.001
    i0 = render_depth(cam, sphere, np.array([0, 0, 0.005 - delta]), IDENTITY_QUAT, bg)
    i1 = render_depth(cam, sphere, np.array([dx, 0, 0.005 - delta]), IDENTITY_QUAT, bg)

    def cu(img):
        m = img.indentation()
        return (m * np.arange(img.width)[None, :]).sum() / m.sum()

    assert cu(i1) - cu(i0) == pytest.approx(cam.fx * dx / 0.02, abs=1.0)


def test_batched_render_matches_single_and_oracle(scene):
    cam, bg, sphere = scene
    poses = np.array([[0, 0, 0.0046], [0.002, 0, 0.0044], [0, 0, 0.01]])
    quats = np.tile(IDENTITY_QUAT, (3, 1))
    batch = render_depth(cam, sphere, poses, quats, bg)
    assert batch.values.shape == (3, 60, 80)
    for e in range(3):
        solo = render_depth(cam, sphere, poses[e], IDENTITY_QUAT, bg)
        assert np.array_equal(batch.values[e], solo.values)
    ref = O.render_depth(cam.rays(), bg, cam.pos, cam.near, cam.far, sphere.origin, sphere.spacing, sphere.dims,
                         sphere.values, poses, quats)
    assert np.array_equal(batch.values, ref)
