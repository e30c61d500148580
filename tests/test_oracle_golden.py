"""Pin the CPU oracle (oracle/gelsim_oracle.py) against golden vectors made by
the reference itself (tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

from conftest import sdf_tuple, vec_close
from oracle import gelsim_oracle as O
from paper_2408_06506_b200 import synthetic
from paper_2408_06506_b200.render import monomial_exponents, synthetic_lut
from paper_2408_06506_b200.sensors import TactileSensorSpec
from paper_2408_06506_b200.tactile import PenaltyParams, sample_tactile_points


def test_monomial_order():
    assert O.monomial_exponents(2) == [(0, 0), (1, 0), (0, 1), (2, 0), (1, 1), (0, 2)]
    for deg in (2, 3, 4):
        assert O.monomial_exponents(deg) == monomial_exponents(deg)
        assert len(O.monomial_exponents(deg)) == (deg + 1) * (deg + 2) // 2


@pytest.mark.parametrize("deg", [2, 3, 4])
def test_oracle_rgb_matches_reference(golden, deg):
    z = golden("rgb")
    got = O.depth_to_rgb(z["d60"], z[f"c60_deg{deg}"], deg)
    np.testing.assert_allclose(got, z[f"rgb60_deg{deg}"], rtol=0, atol=1e-13)
    assert np.array_equal(O.to_uint8(got), z[f"u8_60_deg{deg}"])


def test_oracle_rgb_large_and_plain(golden):
    z = golden("rgb")
    got = O.to_uint8(O.depth_to_rgb(z["d240"], z["c240"], 2))
    assert np.array_equal(got, z["u8_240"])
    np.testing.assert_allclose(O.depth_to_rgb(z["d60"], z["c60_plain"], 2), z["rgb60_plain"], atol=1e-13)


@pytest.mark.parametrize("hw", [(2, 3), (5, 7), (9, 18), (3, 2)])
def test_oracle_rgb_odd_sizes(golden, hw):
    z = golden("rgb")
    H, W = hw
    got = O.depth_to_rgb(z[f"odd_{H}x{W}_d"], z[f"odd_{H}x{W}_c"], 3)
    np.testing.assert_allclose(got, z[f"odd_{H}x{W}_rgb"], atol=1e-13)


def test_oracle_rgb_tilt_and_clamp(golden):
    z = golden("rgb")
    np.testing.assert_allclose(O.depth_to_rgb(z["tilt_d"], z["tilt_c"], 2), z["tilt_rgb"], atol=1e-13)
    np.testing.assert_array_equal(O.depth_to_rgb(z["clamp_d"], z["tilt_c"], 2), z["clamp_rgb"])


def test_oracle_gradient_border_semantics():
    f = np.array([[0.0, 1.0, 4.0, 9.0], [1.0, 3.0, 5.0, 10.0]])
    gx, gy = O.depth_gradients(f)
    np.testing.assert_array_equal(gx[0], [1.0, 2.0, 4.0, 5.0])   # one-sided borders NOT halved
    np.testing.assert_array_equal(gy[0], [1.0, 2.0, 1.0, 1.0])
    with pytest.raises(ValueError):
        O.depth_gradients(np.zeros((1, 5)))


def test_synthetic_lut_restatement_matches_reference(golden):
    z = golden("rgb")
    np.testing.assert_array_equal(synthetic_lut((80, 60), degree=2, seed=0).coeffs, z["c60_plain"])
    for deg in (2, 3, 4):
        mine = synthetic_lut((80, 60), degree=deg, seed=deg, gradient_scale=synthetic.lut_scale((80, 60)))
        np.testing.assert_allclose(mine.coeffs, z[f"c60_deg{deg}"], rtol=1e-15)


def test_oracle_query_sdf_matches_reference(golden):
    z = golden("sdf")
    d, n, valid = O.query_sdf(z["origin"], float(z["spacing"]), z["dims"], z["values"], z["gradients"], z["points"])
    assert np.array_equal(valid, z["valid"])
    assert np.array_equal(d, z["distance"])          # bit-exact, inf where invalid
    np.testing.assert_allclose(n, z["normal"], rtol=0, atol=1e-15)


def test_oracle_force_field_matches_reference(golden, golden_grid):
    z = golden("ff")
    obj, sen = z["obj"], z["sen"]
    f_n, f_t, kin = O.compute_force_field(
        z["points"], *sdf_tuple(golden_grid), obj[:, 0:3], obj[:, 3:7], obj[:, 7:10], obj[:, 10:13],
        sen[:, 0:3], sen[:, 3:7], sen[:, 7:10], sen[:, 10:13])
    assert np.array_equal(kin["d"] < 0, z["d"] < 0)
    assert np.array_equal(kin["d"], z["d"])
    assert vec_close(f_n, z["f_n"], rtol=1e-12)[0]
    assert vec_close(f_t, z["f_t"], rtol=1e-12)[0]
    np.testing.assert_allclose(kin["n"], z["n"], atol=1e-15)
    force, torque = O.net_wrench(f_n, f_t, z["points"])
    np.testing.assert_allclose(force, z["force"], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(torque, z["torque"], rtol=1e-10, atol=1e-15)


def test_oracle_unbatched_force_field(golden, golden_grid):
    z = golden("ff")
    o, s, p = z["obj1"], z["sen1"], z["params1"]
    f_n, f_t, _ = O.compute_force_field(z["points"], *sdf_tuple(golden_grid), o[0:3], o[3:7], o[7:10], o[10:13],
                                        s[0:3], s[3:7], s[7:10], s[10:13], *p)
    assert vec_close(f_n[0], z["f_n1"], rtol=1e-12)[0]
    assert vec_close(f_t[0], z["f_t1"], rtol=1e-12)[0]


def test_oracle_penalty_matches_reference_and_scalar(golden):
    z = golden("penalty")
    f_n, f_t = O.penalty_forces(z["d"], z["d_dot"], z["n"], z["v_t"], *z["params"])
    np.testing.assert_allclose(f_n, z["f_n"], atol=1e-15)
    np.testing.assert_allclose(f_t, z["f_t"], atol=1e-15)
    for i in range(0, len(z["d"]), 37):
        rn, rt = O.force_field_scalar(z["d"][i], z["d_dot"][i], tuple(z["n"][i]), tuple(z["v_t"][i]), *z["params"])
        assert np.max(np.abs(f_n[i] - rn)) < 1e-12
        assert np.max(np.abs(f_t[i] - rt)) < 1e-12


def test_taxel_layout_bit_exact(golden):
    z = golden("ff")
    grid = sample_tactile_points(TactileSensorSpec(image_size=(320, 240)), 20, 25)
    assert np.array_equal(grid.points, z["points"])
    assert grid.rows == 20 and grid.cols == 25


def test_penalty_params_validation():
    with pytest.raises(ValueError):
        PenaltyParams(k_n=-1.0)


@pytest.mark.parametrize("size", [(80, 60), (320, 240)])
def test_oracle_render_depth_bit_exact(golden, golden_grid, size):
    from paper_2408_06506_b200.sensors import camera_for_sensor
    z = golden("depth")
    W, H = size
    cam = camera_for_sensor(TactileSensorSpec(image_size=size))
    k = f"{H}x{W}"
    got = O.render_depth(cam.rays(), z["bg_" + k], cam.pos, cam.near, cam.far, golden_grid.origin,
                         golden_grid.spacing, golden_grid.dims, golden_grid.values, z["pos_" + k], z["quat_" + k])
    assert np.array_equal(got, z["depth_" + k])
