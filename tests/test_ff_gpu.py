"""K2 (force field + wrench), query_sdf and penalty_forces parity on the GPU.

Contract (BASELINE.json north_star): force fields within 1e-5 relative;
taxel indexing and contact masks bit-exact.  The kernel's float64 mask chain
reproduces the reference's distance bit for bit, so the tests also assert
d == d_ref exactly."""
import numpy as np
import pytest
import torch

from conftest import sdf_tuple, vec_close
from oracle import gelsim_oracle as O
from paper_2408_06506_b200 import geometry, synthetic, tactile
from paper_2408_06506_b200.errors import DimensionMismatch
from paper_2408_06506_b200.geometry import query_sdf
from paper_2408_06506_b200.sensors import IDENTITY_QUAT, TactileSensorSpec
from paper_2408_06506_b200.tactile import (
    ForceField,
    PenaltyParams,
    TactilePointGrid,
    compute_force_field,
    net_wrench,
    penalty_forces,
    sample_tactile_points,
)

pytestmark = pytest.mark.gpu

FF_RTOL = 1e-5

STILL = dict(object_linvel=np.zeros(3), object_angvel=np.zeros(3), sensor_pos=np.zeros(3),
             sensor_quat=IDENTITY_QUAT, sensor_linvel=np.zeros(3), sensor_angvel=np.zeros(3))


@pytest.fixture(scope="module")
def plate_sdf():
    return geometry.box_grid((0.1, 0.1, 0.02), dims=(48, 48, 24), padding=0.01)


def sensor_grid(rows=10, cols=10):
    return sample_tactile_points(TactileSensorSpec(), rows, cols)


# ------------------------------------------------------------------ golden ---

def test_query_sdf_golden_bit_exact(golden, golden_grid):
    z = golden("sdf")
    q = query_sdf(golden_grid, z["points"])
    assert np.array_equal(q.valid, z["valid"])
    assert np.array_equal(q.distance, z["distance"])
    np.testing.assert_allclose(q.normal, z["normal"], rtol=0, atol=1e-14)
    single = query_sdf(golden_grid, z["points"][3000])
    assert single.distance == z["distance"][3000] and bool(single.valid) == bool(z["valid"][3000])


def test_force_field_golden(golden, golden_grid):
    z = golden("ff")
    obj, sen = z["obj"], z["sen"]
    pts = TactilePointGrid(points=z["points"], rest_normals=np.zeros_like(z["points"]), spacing=(1e-3, 1e-3))
    fld, kin = compute_force_field(pts, golden_grid, obj[:, 0:3], obj[:, 3:7], obj[:, 7:10], obj[:, 10:13],
                                   sen[:, 0:3], sen[:, 3:7], sen[:, 7:10], sen[:, 10:13], PenaltyParams(),
                                   return_kinematics=True)
    assert np.array_equal(kin["d"], z["d"])                    # distance bit-exact (=> mask bit-exact)
    assert np.array_equal(kin["d"] < 0, z["d"] < 0)
    ok, worst = vec_close(fld.f_n, z["f_n"], FF_RTOL)
    assert ok, worst
    ok, worst = vec_close(fld.f_t, z["f_t"], FF_RTOL)
    assert ok, worst
    # achieved precision is far inside the contract
    assert vec_close(fld.f_n, z["f_n"], 1e-11)[0] and vec_close(fld.f_t, z["f_t"], 1e-9)[0]
    np.testing.assert_allclose(kin["n"], z["n"], atol=1e-13)
    np.testing.assert_allclose(kin["d_dot"], z["d_dot"], atol=1e-14)
    force, torque = net_wrench(fld, pts)
    np.testing.assert_allclose(force, z["force"], rtol=1e-10, atol=1e-14)
    np.testing.assert_allclose(torque, z["torque"], rtol=1e-8, atol=1e-15)


def test_force_field_unbatched_golden(golden, golden_grid):
    z = golden("ff")
    o, s, p = z["obj1"], z["sen1"], z["params1"]
    pts = TactilePointGrid(points=z["points"], rest_normals=np.zeros_like(z["points"]), spacing=(1e-3, 1e-3))
    fld = compute_force_field(pts, golden_grid, o[0:3], o[3:7], o[7:10], o[10:13], s[0:3], s[3:7], s[7:10],
                              s[10:13], PenaltyParams(*p))
    assert fld.f_n.shape == (20, 25, 3)
    assert vec_close(fld.f_n, z["f_n1"], FF_RTOL)[0]
    assert vec_close(fld.f_t, z["f_t1"], FF_RTOL)[0]


def test_penalty_forces_golden_and_scalar(golden):
    z = golden("penalty")
    f_n, f_t = penalty_forces(z["d"], z["d_dot"], z["n"], z["v_t"], PenaltyParams(*z["params"]))
    np.testing.assert_allclose(f_n, z["f_n"], atol=1e-12)
    np.testing.assert_allclose(f_t, z["f_t"], atol=1e-12)


# ------------------------------------------------------- oracle, larger ------

@pytest.mark.parametrize("ff_grid", [(20, 25), (80, 100)])
def test_force_field_vs_oracle_random_sensor_poses(ff_grid):
    sdf = synthetic.peg_grid((32, 32, 64))
    pts = sample_tactile_points(TactileSensorSpec(image_size=(320, 240)), *ff_grid)
    E = 64 if ff_grid == (20, 25) else 8
    obj, sen = synthetic.peg_states(E, 1, config_id=21, random_sensor_pose=True)
    sen = sen[:, 0]
    params = PenaltyParams()
    fld, kin = compute_force_field(pts, sdf, obj[:, 0:3], obj[:, 3:7], obj[:, 7:10], obj[:, 10:13],
                                   sen[:, 0:3], sen[:, 3:7], sen[:, 7:10], sen[:, 10:13], params,
                                   return_kinematics=True)
    f_n, f_t, rk = O.compute_force_field(pts.points, *sdf_tuple(sdf), obj[:, 0:3], obj[:, 3:7], obj[:, 7:10],
                                         obj[:, 10:13], sen[:, 0:3], sen[:, 3:7], sen[:, 7:10], sen[:, 10:13])
    contact = rk["d"] < 0
    assert 0.05 < contact.mean() < 0.6                          # non-vacuous
    assert np.array_equal(kin["d"], rk["d"])
    assert vec_close(fld.f_n, f_n, FF_RTOL)[0]
    assert vec_close(fld.f_t, f_t, FF_RTOL)[0]


def test_device_path_fp32_two_sensors_mask_and_wrench():
    t = torch
    sdf = synthetic.peg_grid((32, 32, 64))
    pts = sample_tactile_points(TactileSensorSpec(image_size=(320, 240)), 20, 25)
    E, S = 48, 2
    obj, sen = synthetic.peg_states(E, S, config_id=22)
    dev = t.device("cuda")
    tax = tactile.device_taxels(pts, dev)
    o = t.from_numpy(obj).to(dev)
    s = t.from_numpy(np.ascontiguousarray(sen)).to(dev)
    f_n = t.empty((E, S, 20, 25, 3), dtype=t.float32, device=dev)
    f_t = t.empty_like(f_n)
    wrench = t.empty((E, S, 6), dtype=t.float64, device=dev)
    contact = t.empty((E, S, 20, 25), dtype=t.uint8, device=dev)
    tactile.force_field_device(sdf, tax, 20, 25, o, s, PenaltyParams(), f_n, f_t, wrench=wrench,
                               contact=contact, n_sensors=S)
    t.cuda.synchronize()
    objE = np.repeat(obj, S, axis=0)
    senE = sen.reshape(E * S, 13)
    rn, rt, rk = O.compute_force_field(pts.points, *sdf_tuple(sdf), objE[:, 0:3], objE[:, 3:7], objE[:, 7:10],
                                       objE[:, 10:13], senE[:, 0:3], senE[:, 3:7], senE[:, 7:10], senE[:, 10:13])
    assert np.array_equal(contact.cpu().numpy().reshape(E * S, 20, 25).astype(bool), rk["d"] < 0)
    assert vec_close(f_n.cpu().numpy().reshape(E * S, 20, 25, 3), rn, FF_RTOL, atol=1e-9)[0]
    assert vec_close(f_t.cpu().numpy().reshape(E * S, 20, 25, 3), rt, FF_RTOL, atol=1e-9)[0]
    force, torque = O.net_wrench(rn, rt, pts.points)
    w = wrench.cpu().numpy().reshape(E * S, 6)
    scale = np.abs(rn + rt).sum(axis=(1, 2))       # sum of |f| bounds the cancellation
    assert np.all(np.abs(w[:, 0:3] - force) <= 1e-12 * scale + 1e-15)
    assert np.all(np.abs(w[:, 3:6] - torque) <= 1e-12 * scale * 0.02 + 1e-15)


# ----------------------------------------- reference tests, re-pinned on GPU --
# (pkg/tests/test_tactile_field.py)

def test_no_penetration_zero_field(plate_sdf):
    fld = compute_force_field(sensor_grid(), plate_sdf, object_pos=np.array([0, 0, 0.02]),
                              object_quat=IDENTITY_QUAT, params=PenaltyParams(), **STILL)
    assert np.all(fld.f_n == 0) and np.all(fld.f_t == 0)


def test_static_press_normal_magnitude(plate_sdf):
    params = PenaltyParams(k_n=1000.0, k_d=0.0, k_t=10.0, mu=2.0)
    fld = compute_force_field(sensor_grid(), plate_sdf, object_pos=np.array([0, 0, 0.01 - 0.001]),
                              object_quat=IDENTITY_QUAT, params=params, **STILL)
    mags = np.linalg.norm(fld.f_n, axis=-1)
    np.testing.assert_allclose(mags, 1.0, rtol=1e-6)


def test_sliding_press_hits_cone_boundary(plate_sdf):
    params = PenaltyParams(k_n=1000.0, k_d=0.0, k_t=1e4, mu=1.0)
    kw = dict(STILL)
    kw["sensor_linvel"] = np.array([0.01, 0.0, 0.0])
    fld = compute_force_field(sensor_grid(), plate_sdf, object_pos=np.array([0, 0, 0.01 - 0.001]),
                              object_quat=IDENTITY_QUAT, params=params, **kw)
    expected = np.zeros((10, 10, 3))
    expected[..., 0] = -1.0
    np.testing.assert_allclose(fld.f_t, expected, atol=1e-9)


def test_batched_matches_single_bit_exact(plate_sdf):
    params = PenaltyParams()
    pos = np.array([[0, 0, 0.0095], [0, 0, 0.0090], [0, 0, 0.02]])
    quat = np.tile(IDENTITY_QUAT, (3, 1))
    fld = compute_force_field(sensor_grid(), plate_sdf, pos, quat, np.zeros((3, 3)), np.zeros((3, 3)),
                              np.zeros((3, 3)), quat, np.zeros((3, 3)), np.zeros((3, 3)), params)
    for e in range(3):
        solo = compute_force_field(sensor_grid(), plate_sdf, pos[e], IDENTITY_QUAT, params=params, **STILL)
        assert np.array_equal(fld.f_n[e], solo.f_n)
        assert np.array_equal(fld.f_t[e], solo.f_t)


def test_cone_and_directionality_random_sweep():
    rng = np.random.default_rng(12)
    n_pts = 10000
    d = rng.uniform(-3e-3, 5e-4, n_pts)
    d_dot = rng.uniform(-1, 1, n_pts)
    n = rng.normal(size=(n_pts, 3))
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    v_t = rng.normal(size=(n_pts, 3)) * rng.uniform(0, 0.2, (n_pts, 1))
    params = PenaltyParams(k_n=1200.0, k_d=90.0, k_t=15.0, mu=0.9)
    f_n, f_t = penalty_forces(d, d_dot, n, v_t, params)
    fn_mag = np.linalg.norm(f_n, axis=-1)
    ft_mag = np.linalg.norm(f_t, axis=-1)
    assert np.all(ft_mag <= params.mu * fn_mag + 1e-9)
    assert np.all(np.einsum("ij,ij->i", f_t, v_t) <= 0)
    assert np.all(np.einsum("ij,ij->i", f_n, n) >= 0)


def test_repulsion_clamp_when_separating_fast():
    f_n, f_t = penalty_forces(-1e-3, 50.0, np.array([0, 0, 1.0]), np.zeros(3), PenaltyParams(k_n=100.0, k_d=10.0))
    assert np.all(f_n == 0) and np.all(f_t == 0)


def test_resolution_consistency_after_density_normalization():
    r = 0.02
    big_sphere = geometry.sphere_grid(r, dims=(64, 64, 64), padding=0.004)
    params = PenaltyParams()
    wrenches = {}
    for res in (10, 100):
        grid = sample_tactile_points(TactileSensorSpec(), res, res)
        fld = compute_force_field(grid, big_sphere, object_pos=np.array([0, 0, r - 0.0015]),
                                  object_quat=IDENTITY_QUAT, params=params, **STILL)
        force, _ = net_wrench(fld, grid)
        wrenches[res] = force * grid.spacing[0] * grid.spacing[1]
    assert np.linalg.norm(wrenches[10] - wrenches[100]) / np.linalg.norm(wrenches[100]) < 0.05


def test_symmetric_press_zero_torque(plate_sdf):
    grid = sensor_grid()
    fld = compute_force_field(grid, plate_sdf, object_pos=np.array([0, 0, 0.01 - 0.0005]),
                              object_quat=IDENTITY_QUAT, params=PenaltyParams(), **STILL)
    force, torque = net_wrench(fld, grid)
    assert np.linalg.norm(torque) < 1e-9 * np.linalg.norm(force) * 0.024 + 1e-15


def test_two_point_wrench_hand_sum():
    pts = np.zeros((1, 2, 3))
    pts[0, 0, 0] = 0.01
    pts[0, 1, 0] = -0.01
    grid = TactilePointGrid(points=pts, rest_normals=np.zeros((1, 2, 3)), spacing=(0.02, 0.02))
    f_n = np.zeros((1, 2, 3))
    f_n[..., 2] = 1.0
    force, torque = net_wrench(ForceField(f_n=f_n, f_t=np.zeros((1, 2, 3))), grid)
    np.testing.assert_allclose(force, [0, 0, 2.0])
    np.testing.assert_allclose(torque, [0, 0, 0], atol=1e-15)


def test_wrench_dimension_mismatch():
    with pytest.raises(DimensionMismatch):
        net_wrench(ForceField(f_n=np.zeros((5, 5, 3)), f_t=np.zeros((5, 5, 3))), sensor_grid(10, 10))


def test_query_sdf_sentinel_and_device_tensors():
    g = geometry.sphere_grid(0.005, dims=(32, 32, 32))
    pts = np.array([[0.0, 0.0, 0.0], [1.0, 1.0, 1.0], [0.0, 0.0, 0.004]])
    q = query_sdf(g, pts)
    assert list(q.valid) == [True, False, True]
    assert np.isinf(q.distance[1]) and np.all(q.normal[1] == 0)
    qd = query_sdf(g, torch.from_numpy(pts).cuda())
    assert torch.equal(qd.distance.cpu(), torch.from_numpy(q.distance))


@pytest.mark.parametrize("kernel", ["quad", "fp64"])
@pytest.mark.parametrize("offset", [0.0, 100.0])
def test_fast_mask_chain_equals_exact_chain(monkeypatch, offset, kernel):
    """force_field_fast_kernel (affine cell coordinates + exact fallback near
    every decision boundary) against the all-exact kernel and the oracle:
    identical contact masks, forces within 1e-9 relative -- also with the
    envs placed 100 m from the world origin.  ``quad`` is the certified fp32
    pre-pass (force_field_quad_kernel), ``fp64`` the fp64 fast kernel."""
    t = torch
    monkeypatch.setenv("TACSL_FF_QUAD", "1" if kernel == "quad" else "0")
    sdf = synthetic.peg_grid((32, 32, 64))
    pts = sample_tactile_points(TactileSensorSpec(image_size=(320, 240)), 20, 25)
    E, S = 256, 2
    obj, sen = synthetic.peg_states(E, S, config_id=23, random_sensor_pose=True)
    shift = np.array([offset, -0.5 * offset, 0.2 * offset])
    obj[:, 0:3] += shift
    sen[:, :, 0:3] += shift
    dev = t.device("cuda")
    tax = tactile.device_taxels(pts, dev)
    o = t.from_numpy(obj).to(dev)
    s = t.from_numpy(np.ascontiguousarray(sen)).to(dev)

    def run():
        f_n = t.empty((E, S, 20, 25, 3), dtype=t.float64, device=dev)
        f_t = t.empty_like(f_n)
        w = t.empty((E, S, 6), dtype=t.float64, device=dev)
        c = t.empty((E, S, 20, 25), dtype=t.uint8, device=dev)
        tactile.force_field_device(sdf, tax, 20, 25, o, s, PenaltyParams(), f_n, f_t, wrench=w, contact=c,
                                   n_sensors=S)
        t.cuda.synchronize()
        return [x.cpu().numpy() for x in (f_n, f_t, w, c)]

    fast = run()
    monkeypatch.setenv("TACSL_FF_EXACT", "1")
    exact = run()
    assert np.array_equal(fast[3], exact[3])
    assert 0.05 < fast[3].mean() < 0.6
    # the reference chain itself rounds positions at ulp(|pos|): 100 m away
    # the two chains legitimately differ by ~1e-14 m in d
    rtol = 1e-9 if offset == 0 else 1e-6
    for a, b in zip(fast[:3], exact[:3]):
        assert vec_close(a, b, rtol, atol=1e-12)[0]
    objE = np.repeat(obj, S, axis=0)
    senE = sen.reshape(E * S, 13)
    rn, rt, rk = O.compute_force_field(pts.points, *sdf_tuple(sdf), objE[:, 0:3], objE[:, 3:7], objE[:, 7:10],
                                       objE[:, 10:13], senE[:, 0:3], senE[:, 3:7], senE[:, 7:10], senE[:, 10:13])
    assert np.array_equal(fast[3].reshape(E * S, 20, 25).astype(bool), rk["d"] < 0)
    assert vec_close(fast[0].reshape(rn.shape), rn, FF_RTOL, atol=1e-9)[0]
    assert vec_close(fast[1].reshape(rt.shape), rt, FF_RTOL, atol=1e-9)[0]


@pytest.mark.parametrize("kernel", ["quad", "fp64"])
def test_fast_chain_decides_boundary_taxels_exactly(monkeypatch, kernel):
    """Taxels placed exactly on the contact surface (d = 0 in the grid) and
    on the grid boundary go through the exact fallback: masks still match."""
    t = torch
    monkeypatch.setenv("TACSL_FF_QUAD", "1" if kernel == "quad" else "0")
    sdf = geometry.box_grid((0.1, 0.1, 0.02), dims=(48, 48, 24), padding=0.01)
    pts = sensor_grid(12, 12)
    E = 64
    rng = np.random.default_rng(5)
    obj = np.zeros((E, 13))
    obj[:, 3] = 1.0
    sen = np.zeros((E, 1, 13))
    sen[:, 0, 3] = 1.0
    # the pad plane at z = 0.01 touches the box top (d = 0) for half of the envs
    sen[:, 0, 2] = np.where(np.arange(E) % 2 == 0, 0.01, rng.uniform(0.0095, 0.0105, E)) - float(pts.points[0, 0, 2])
    sen[:, 0, 7:10] = rng.normal(0, 0.01, (E, 3))
    dev = t.device("cuda")
    tax = tactile.device_taxels(pts, dev)
    o = t.from_numpy(obj).to(dev)
    s = t.from_numpy(sen).to(dev)

    def run():
        c = t.empty((E, 1, 12, 12), dtype=t.uint8, device=dev)
        f_n = t.empty((E, 1, 12, 12, 3), dtype=t.float64, device=dev)
        tactile.force_field_device(sdf, tax, 12, 12, o, s, PenaltyParams(), f_n, None, contact=c, n_sensors=1)
        t.cuda.synchronize()
        return c.cpu().numpy(), f_n.cpu().numpy()

    fast_c, fast_f = run()
    monkeypatch.setenv("TACSL_FF_EXACT", "1")
    exact_c, exact_f = run()
    assert np.array_equal(fast_c, exact_c)
    assert vec_close(fast_f, exact_f, 1e-9, atol=1e-15)[0]


def test_relative_penetration_rate_golden_and_invalid_query(golden, golden_grid):
    """geometry/sdf.py:324-328 on the GPU: bit-exact d_dot, broadcast x_dot,
    and InvalidQuery for an out-of-grid query (the C ABI's INVALID_QUERY)."""
    from paper_2408_06506_b200.errors import InvalidQuery
    from paper_2408_06506_b200.geometry import query_sdf, relative_penetration_rate
    z = golden("extras")
    q = query_sdf(golden_grid, z["points"])
    # the normals match the reference to rounding (only the distance is
    # bit-exact), so d_dot does too; on the same normals the dot product is
    # numpy 2.3's einsum order, (n0 x0 + n2 x2) + n1 x1, bit for bit
    got = relative_penetration_rate(q, z["x_dot"])
    np.testing.assert_allclose(got, z["rate"], rtol=1e-12, atol=1e-15)
    n, x = q.normal, z["x_dot"]
    np.testing.assert_array_equal(got, (n[:, 0] * x[:, 0] + n[:, 2] * x[:, 2]) + n[:, 1] * x[:, 1])
    np.testing.assert_allclose(relative_penetration_rate(q, z["x1"]), z["rate1"], rtol=1e-12, atol=1e-15)
    qd = query_sdf(golden_grid, torch.from_numpy(z["points"]).cuda())
    got_d = relative_penetration_rate(qd, torch.from_numpy(z["x_dot"]).cuda())
    assert got_d.is_cuda
    np.testing.assert_array_equal(got_d.cpu().numpy(), got)
    assert bool(z["mixed_raises"])
    with pytest.raises(InvalidQuery):
        relative_penetration_rate(query_sdf(golden_grid, z["mixed"]), z["x_dot"][:11])


def test_force_field_on_curved_pad_taxels_vs_oracle(golden):
    """Taxels of a curved gel (any point set) through K2 vs the oracle."""
    from paper_2408_06506_b200.sensors import SurfaceMesh, TactileSensorSpec
    z = golden("extras")
    sensor = TactileSensorSpec(active_area=(0.02, 0.02), surface_mesh=SurfaceMesh(z["dome_vertices"],
                                                                                   z["dome_faces"]))
    pts = tactile.sample_tactile_points(sensor, 12, 12)
    sdf = synthetic.peg_grid((32, 32, 64))
    E = 64
    obj, sen = synthetic.peg_states(E, 1, config_id=21)
    o, s = obj, sen[:, 0]
    fld = tactile.compute_force_field(pts, sdf, o[:, 0:3], o[:, 3:7], o[:, 7:10], o[:, 10:13], s[:, 0:3],
                                      s[:, 3:7], s[:, 7:10], s[:, 10:13], tactile.PenaltyParams())
    r_fn, r_ft, _ = O.compute_force_field(pts.points, *sdf_tuple(sdf), o[:, 0:3], o[:, 3:7], o[:, 7:10],
                                          o[:, 10:13], s[:, 0:3], s[:, 3:7], s[:, 7:10], s[:, 10:13],
                                          1000.0, 100.0, 10.0, 2.0)
    assert vec_close(fld.f_n, r_fn, 1e-9, atol=1e-12)[0] and vec_close(fld.f_t, r_ft, 1e-9, atol=1e-12)[0]
    assert (np.abs(r_fn).sum(-1) > 0).any()


# ------------------------------------- certified fp32 pre-pass (quad kernel) --

def _ff_run(sdf, pts_dev, rows, cols, obj, sen, S=1, fp64=True):
    t = torch
    E = obj.shape[0]
    dev = t.device("cuda")
    dt = t.float64 if fp64 else t.float32
    f_n = t.empty((E, S, rows, cols, 3), dtype=dt, device=dev)
    f_t = t.empty_like(f_n)
    w = t.empty((E, S, 6), dtype=t.float64, device=dev)
    c = t.empty((E, S, rows, cols), dtype=t.uint8, device=dev)
    tactile.force_field_device(sdf, pts_dev, rows, cols, t.from_numpy(obj).to(dev),
                               t.from_numpy(np.ascontiguousarray(sen)).to(dev), PenaltyParams(), f_n, f_t,
                               wrench=w, contact=c, n_sensors=S)
    t.cuda.synchronize()
    return [x.cpu().numpy() for x in (f_n, f_t, w, c)]


def _ff_vs_exact(monkeypatch, sdf, pts_dev, rows, cols, obj, sen, S=1):
    monkeypatch.setenv("TACSL_FF_QUAD", "1")  # the quad kernel also on these small pads
    quad = _ff_run(sdf, pts_dev, rows, cols, obj, sen, S)
    monkeypatch.setenv("TACSL_FF_EXACT", "1")
    exact = _ff_run(sdf, pts_dev, rows, cols, obj, sen, S)
    monkeypatch.delenv("TACSL_FF_EXACT")
    assert np.array_equal(quad[3], exact[3])
    for a, b in zip(quad[:3], exact[:3]):
        assert vec_close(a, b, 1e-9, atol=1e-12)[0]
    return quad


def test_quad_kernel_taxels_on_grid_faces_and_lines(monkeypatch, plate_sdf):
    """Taxels exactly on the SDF grid's faces, on cell boundaries, just
    inside / outside the one-cell shell and far outside: the fp32
    classification and its explicit shell test decide validity exactly."""
    g = plate_sdf
    h, o, up = g.spacing, g.origin, g.upper
    xs = np.concatenate([o[0] + h * np.array([-3.0, -1.0, -0.5, 0.0, 1e-12, 0.5, 1.0, 2.0, 7.0]),
                         up[0] - h * np.array([2.0, 1.0, 0.5, 0.0, -1e-12, -0.5, -1.0, -3.0])])
    ys = np.concatenate([o[1] + h * np.array([-1.0, 0.0, 0.25, 1.0]), up[1] - h * np.array([1.0, 0.0, -0.25, -1.0]),
                         [0.0, 0.003, -0.004, 0.011]])
    rows, cols = len(ys), len(xs)                         # 12 x 17 = 204 taxels (a multiple of 4)
    zs = [up[2], g.origin[2], 0.01, 0.0099999, 0.0100001]  # grid top, bottom, box top (d = 0) and around it
    E = len(zs) * 4
    pts = np.zeros((rows, cols, 3))
    pts[..., 0] = xs[None, :]
    pts[..., 1] = ys[:, None]
    obj = np.zeros((E, 13))
    obj[:, 3] = 1.0
    sen = np.zeros((E, 1, 13))
    sen[:, 0, 3] = 1.0
    rng = np.random.default_rng(3)
    for e in range(E):
        sen[e, 0, 2] = zs[e // 4]
        sen[e, 0, 7:10] = rng.normal(0, 0.01, 3)
    dev = torch.device("cuda")
    tax = torch.from_numpy(pts.reshape(-1, 3)).to(dev)
    quad = _ff_vs_exact(monkeypatch, g, tax, rows, cols, obj, sen)
    assert 0 < quad[3].mean() < 1
    objE, senE = obj, sen.reshape(E, 13)
    rn, rt, rk = O.compute_force_field(pts, *sdf_tuple(g), objE[:, 0:3], objE[:, 3:7], objE[:, 7:10], objE[:, 10:13],
                                       senE[:, 0:3], senE[:, 3:7], senE[:, 7:10], senE[:, 10:13])
    assert np.array_equal(quad[3].reshape(E, rows, cols).astype(bool), rk["d"] < 0)


def test_quad_kernel_nan_and_non_unit_poses(monkeypatch):
    """A NaN object pose (the reference: every taxel invalid, zero forces)
    and non-unit quaternions (the world-frame contact path)."""
    sdf = synthetic.peg_grid((32, 32, 64))
    pts = sample_tactile_points(TactileSensorSpec(image_size=(320, 240)), 20, 25)
    obj, sen = synthetic.peg_states(16, 1, config_id=31)
    obj[3, 0] = np.nan
    obj[5, 3:7] *= 1.25
    sen[7, 0, 3:7] *= 0.8
    tax = tactile.device_taxels(pts, torch.device("cuda"))
    quad = _ff_vs_exact(monkeypatch, sdf, tax, 20, 25, obj, sen)
    assert not quad[3][3].any() and np.all(quad[0][3] == 0)


def test_quad_kernel_fallbacks_and_taxel_refresh(monkeypatch, plate_sdf):
    """rows*cols % 4 != 0 and an SDF with non-finite values run the fp64
    kernel; a taxel tensor edited in place is never served stale."""
    sdf = synthetic.peg_grid((32, 32, 64))
    obj, sen = synthetic.peg_states(8, 1, config_id=32)
    pts = sample_tactile_points(TactileSensorSpec(image_size=(320, 240)), 5, 5)  # 25 taxels
    _ff_vs_exact(monkeypatch, sdf, tactile.device_taxels(pts, torch.device("cuda")), 5, 5, obj, sen)
    inf_sdf = synthetic.peg_grid((32, 32, 64))
    inf_sdf.values = inf_sdf.values.copy()
    inf_sdf.values[0, 0, 0] = np.inf                     # far corner, never interpolated by the pad
    pts = sample_tactile_points(TactileSensorSpec(image_size=(320, 240)), 20, 25)
    tax = tactile.device_taxels(pts, torch.device("cuda")).clone()
    _ff_vs_exact(monkeypatch, inf_sdf, tax, 20, 25, obj, sen)
    monkeypatch.setenv("TACSL_FF_QUAD", "1")
    first = _ff_run(sdf, tax, 20, 25, obj, sen)
    tax[:, 2] += 0.0005                                   # same pointer, new contents
    moved = _ff_run(sdf, tax, 20, 25, obj, sen)
    fresh = _ff_run(sdf, tax.clone(), 20, 25, obj, sen)
    for a, b in zip(moved, fresh):
        assert np.array_equal(a, b)
    assert not np.array_equal(first[3], moved[3])


def test_quad_kernel_under_graph_capture(monkeypatch):
    """The quad path (fp32 taxel copy in a stream-ordered allocation + the
    quad kernel) captured in a CUDA graph: replays with new states written
    in place equal eager calls on the same states."""
    monkeypatch.setenv("TACSL_FF_QUAD", "1")
    sdf = synthetic.peg_grid((32, 32, 64))
    pts = sample_tactile_points(TactileSensorSpec(image_size=(320, 240)), 20, 25)
    dev = torch.device("cuda")
    tax = tactile.device_taxels(pts, dev)
    E = 64
    o = torch.empty((E, 13), dtype=torch.float64, device=dev)
    s = torch.empty((E, 1, 13), dtype=torch.float64, device=dev)
    f_n = torch.empty((E, 1, 20, 25, 3), dtype=torch.float32, device=dev)
    f_t = torch.empty_like(f_n)
    w = torch.empty((E, 1, 6), dtype=torch.float64, device=dev)

    def call():
        tactile.force_field_device(sdf, tax, 20, 25, o, s, PenaltyParams(), f_n, f_t, wrench=w, n_sensors=1)

    obj, sen = synthetic.peg_states(E, 1, config_id=41)
    o.copy_(torch.from_numpy(obj))
    s.copy_(torch.from_numpy(np.ascontiguousarray(sen)))
    call()  # warm-up outside the capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    stream = torch.cuda.Stream()
    stream.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(stream):
        with torch.cuda.graph(g, stream=stream):
            call()
    torch.cuda.synchronize()
    for seed in (42, 43):
        obj, sen = synthetic.peg_states(E, 1, config_id=seed)
        o.copy_(torch.from_numpy(obj))
        s.copy_(torch.from_numpy(np.ascontiguousarray(sen)))
        g.replay()
        torch.cuda.synchronize()
        got = [x.clone() for x in (f_n, f_t, w)]
        call()
        torch.cuda.synchronize()
        for a, b in zip(got, (f_n, f_t, w)):
            assert torch.equal(a, b)
        assert (got[0].abs().sum() > 0).item()


@pytest.mark.parametrize("field", ["noise", "steep", "fp64_values"])
def test_quad_kernel_certified_mask_on_adversarial_grids(monkeypatch, field):
    """The certified fp32 decisions on grids that are not smooth SDFs: a
    random field with sign changes in many cells, a steep field (large
    Lipschitz bounds), and float64 values that float32 cannot represent --
    with random poses that put pads across the grid faces.  Masks must equal
    the reference chain's; forces the all-exact kernel's."""
    rng = np.random.default_rng({"noise": 1, "steep": 2, "fp64_values": 3}[field])
    dims = (24, 20, 16)
    h = 0.002
    origin = np.array([-0.024, -0.02, -0.016])
    if field == "noise":
        v = rng.normal(0, 0.004, dims)
    elif field == "steep":
        v = np.tanh(rng.normal(0, 3.0, dims)) * 0.05
    else:
        x, y, z = np.meshgrid(*(origin[a] + h * np.arange(dims[a]) for a in range(3)), indexing="ij")
        v = np.sqrt(x * x + y * y + z * z) - 0.011 + rng.normal(0, 1e-9, dims)  # not float32-representable
    g = np.stack(np.gradient(v, h), axis=-1)
    g /= np.maximum(np.linalg.norm(g, axis=-1, keepdims=True), 1e-12)
    sdf = geometry.SdfGrid(origin=origin, spacing=h, dims=dims, values=v, gradients=g)
    pts = sample_tactile_points(TactileSensorSpec(image_size=(320, 240)), 16, 20)  # 320 taxels
    E = 96
    obj = np.zeros((E, 13))
    q = rng.normal(size=(E, 4))
    obj[:, 3:7] = q / np.linalg.norm(q, axis=1, keepdims=True)
    obj[:, 0:3] = rng.uniform(-0.02, 0.02, (E, 3))
    obj[:, 7:13] = rng.normal(0, 0.01, (E, 6))
    sen = np.zeros((E, 1, 13))
    sen[:, 0, 3] = 1.0
    sen[:, 0, 7:13] = rng.normal(0, 0.01, (E, 6))
    dev = torch.device("cuda")
    tax = tactile.device_taxels(pts, dev)
    quad = _ff_vs_exact(monkeypatch, sdf, tax, 16, 20, obj, sen)
    assert 0 < quad[3].mean() < 1
    rn, rt, rk = O.compute_force_field(pts.points, origin, h, dims, v, g, obj[:, 0:3], obj[:, 3:7], obj[:, 7:10],
                                       obj[:, 10:13], sen[:, 0, 0:3], sen[:, 0, 3:7], sen[:, 0, 7:10],
                                       sen[:, 0, 10:13])
    assert np.array_equal(quad[3].reshape(E, 16, 20).astype(bool), rk["d"] < 0)


def test_quad_kernel_fuzz_vs_exact_kernel(monkeypatch):
    """2.6 M taxels: random poses over a sphere SDF and a noise field,
    quad kernel vs the all-exact kernel -- identical masks, forces within
    1e-9."""
    rng = np.random.default_rng(7)
    dims = (40, 36, 32)
    h = 0.001
    origin = -0.5 * h * (np.array(dims) - 1)
    x, y, z = np.meshgrid(*(origin[a] + h * np.arange(dims[a]) for a in range(3)), indexing="ij")
    fields = [np.sqrt(x * x + y * y + z * z) - 0.012, rng.normal(0, 0.002, dims)]
    pts = sample_tactile_points(TactileSensorSpec(image_size=(320, 240)), 16, 20)
    dev = torch.device("cuda")
    tax = tactile.device_taxels(pts, dev)
    E = 4096
    for v in fields:
        g = np.stack(np.gradient(v, h), axis=-1)
        g /= np.maximum(np.linalg.norm(g, axis=-1, keepdims=True), 1e-12)
        sdf = geometry.SdfGrid(origin=origin, spacing=h, dims=dims, values=v, gradients=g)
        obj = np.zeros((E, 13))
        q = rng.normal(size=(E, 4))
        obj[:, 3:7] = q / np.linalg.norm(q, axis=1, keepdims=True)
        obj[:, 0:3] = rng.uniform(-0.025, 0.025, (E, 3))
        obj[:, 7:13] = rng.normal(0, 0.01, (E, 6))
        sen = np.zeros((E, 1, 13))
        sen[:, 0, 3] = 1.0
        sen[:, 0, 7:13] = rng.normal(0, 0.01, (E, 6))
        quad = _ff_vs_exact(monkeypatch, sdf, tax, 16, 20, obj, sen)
        assert 0.01 < quad[3].mean() < 0.99
