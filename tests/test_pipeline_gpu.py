"""The batched sensor step (SensorArray): RGB + force field + wrench for
E envs x S sensors in two overlapped launches, eager and CUDA-graph replay,
against the CPU oracle."""
import numpy as np
import pytest
import torch

from conftest import sdf_tuple, vec_close
from oracle import gelsim_oracle as O
from paper_2408_06506_b200 import SensorArray, synthetic
from paper_2408_06506_b200.tactile import PenaltyParams

pytestmark = pytest.mark.gpu


def setup(E=6, S=2, image=(320, 240)):
    _, cam, bg, lut, pts = synthetic.sensor_setup(image, (20, 25))
    sdf = synthetic.peg_grid((32, 32, 64))
    depth = synthetic.depth_batch(cam, bg, E * S, config_id=31).reshape(E, S, image[1], image[0])
    obj, sen = synthetic.peg_states(E, S, config_id=31)
    return lut, pts, sdf, depth, obj, sen


def oracle_step(lut, pts, sdf, depth, obj, sen):
    E, S = sen.shape[:2]
    objE = np.repeat(obj, S, axis=0)
    senE = sen.reshape(E * S, 13)
    rgb, f_n, f_t, force, torque = O.sensor_frames(depth.reshape((E * S,) + depth.shape[2:]), lut.coeffs,
                                                   lut.degree, pts.points, sdf_tuple(sdf), objE, senE,
                                                   (1000.0, 100.0, 10.0, 2.0))
    return rgb, f_n, f_t, force, torque


@pytest.mark.parametrize("overlap", [True, False])
def test_sensor_array_step_vs_oracle(overlap):
    lut, pts, sdf, depth, obj, sen = setup()
    E, S = sen.shape[:2]
    arr = SensorArray(lut, sdf, pts, PenaltyParams(), E, S, overlap=overlap)
    d = torch.from_numpy(depth).cuda()
    o = torch.from_numpy(obj).cuda()
    s = torch.from_numpy(np.ascontiguousarray(sen)).cuda()
    rgb, f_n, f_t, wrench = arr.step(d, o, s)
    torch.cuda.synchronize()
    r_rgb, r_fn, r_ft, r_force, r_torque = oracle_step(lut, pts, sdf, depth, obj, sen)
    diff = np.abs(rgb.cpu().numpy().reshape(r_rgb.shape).astype(int) - r_rgb.astype(int))
    assert diff.max() <= 1
    assert vec_close(f_n.cpu().numpy().reshape(r_fn.shape), r_fn, 1e-5, atol=1e-9)[0]
    assert vec_close(f_t.cpu().numpy().reshape(r_ft.shape), r_ft, 1e-5, atol=1e-9)[0]
    w = wrench.cpu().numpy().reshape(E * S, 6)
    np.testing.assert_allclose(w[:, :3], r_force, rtol=1e-9, atol=1e-12)


def test_cuda_graph_replay_matches_eager():
    lut, pts, sdf, depth, obj, sen = setup(E=16)
    E, S = sen.shape[:2]
    arr = SensorArray(lut, sdf, pts, PenaltyParams(), E, S)
    d = torch.from_numpy(depth).cuda()
    o = torch.from_numpy(obj).cuda()
    s = torch.from_numpy(np.ascontiguousarray(sen)).cuda()
    arr.launch(d, o, s)
    torch.cuda.synchronize()
    eager = [x.clone() for x in (arr.rgb_u8, arr.f_n, arr.f_t, arr.wrench)]
    arr.capture(d, o, s)
    for x in (arr.rgb_u8, arr.f_n, arr.f_t, arr.wrench):
        x.zero_()
    # new inputs in the captured buffers are picked up by replay
    d2 = torch.from_numpy(np.ascontiguousarray(depth[::-1])).cuda()
    d.copy_(d2)
    arr.replay()
    torch.cuda.synchronize()
    rgb_rev = arr.rgb_u8.clone()
    d.copy_(torch.from_numpy(depth).cuda())
    arr.replay()
    torch.cuda.synchronize()
    for a, b in zip(eager, (arr.rgb_u8, arr.f_n, arr.f_t, arr.wrench)):
        assert torch.equal(a, b)
    assert torch.equal(rgb_rev, eager[0].flip(0))


@pytest.mark.parametrize("chunks", [1, 3, 8])
def test_run_host_pipelined_matches_device_step(chunks):
    lut, pts, sdf, depth, obj, sen = setup(E=10)
    E, S = sen.shape[:2]
    arr = SensorArray(lut, sdf, pts, PenaltyParams(), E, S)
    d = torch.from_numpy(depth).cuda()
    o = torch.from_numpy(obj).cuda()
    s = torch.from_numpy(np.ascontiguousarray(sen)).cuda()
    arr.launch(d, o, s)
    torch.cuda.synchronize()
    ref = [x.cpu() for x in (arr.rgb_u8, arr.f_n, arr.f_t, arr.wrench)]
    host = arr.host_buffers()
    host["depth"].copy_(torch.from_numpy(depth))
    host["obj"].copy_(torch.from_numpy(obj))
    host["sen"].copy_(torch.from_numpy(np.ascontiguousarray(sen)))
    d.zero_()
    arr.run_host(host, d, o, s, chunks=chunks)
    torch.cuda.synchronize()
    for name, r in zip(("rgb", "f_n", "f_t", "wrench"), ref):
        assert torch.equal(host[name], r), name


def test_host_pipeline_graph_matches_device_step():
    lut, pts, sdf, depth, obj, sen = setup(E=12)
    E, S = sen.shape[:2]
    arr = SensorArray(lut, sdf, pts, PenaltyParams(), E, S)
    d = torch.from_numpy(depth).cuda()
    o = torch.from_numpy(obj).cuda()
    s = torch.from_numpy(np.ascontiguousarray(sen)).cuda()
    arr.launch(d, o, s)
    torch.cuda.synchronize()
    ref = [x.cpu() for x in (arr.rgb_u8, arr.f_n, arr.f_t, arr.wrench)]
    host = arr.host_buffers()
    host["depth"].copy_(torch.from_numpy(depth))
    host["obj"].copy_(torch.from_numpy(obj))
    host["sen"].copy_(torch.from_numpy(np.ascontiguousarray(sen)))
    arr.capture_host(host, d, o, s, chunks=4)
    for k in ("rgb", "f_n", "f_t", "wrench"):
        host[k].zero_()
    d.zero_()
    arr.replay_host()
    torch.cuda.synchronize()
    for name, r in zip(("rgb", "f_n", "f_t", "wrench"), ref):
        assert torch.equal(host[name], r), name
    # new host inputs are picked up by the replay
    host["depth"].copy_(torch.from_numpy(np.ascontiguousarray(depth[::-1])))
    arr.replay_host()
    torch.cuda.synchronize()
    assert torch.equal(host["rgb"], ref[0].flip(0))


@pytest.mark.parametrize("deg,size,S", [(4, (84, 61), 1), (3, (320, 240), 2)])
def test_sensor_array_u8_and_f32_fp64_forces(deg, size, S):
    """Both RGB outputs at once (u8 + float), float64 forces, LUT degrees 3-4,
    an odd image height: every output against the oracle."""
    E = 5
    _, cam, bg, _, pts = synthetic.sensor_setup(size, (20, 25))
    lut = synthetic.synthetic_lut(size, degree=deg, gradient_scale=synthetic.lut_scale(size))
    sdf = synthetic.peg_grid((32, 32, 64))
    depth = synthetic.depth_batch(cam, bg, E * S, config_id=33).reshape(E, S, size[1], size[0])
    obj, sen = synthetic.peg_states(E, S, config_id=33)
    arr = SensorArray(lut, sdf, pts, PenaltyParams(), E, S, ff_fp64=True, rgb_u8=True, rgb_f32=True)
    arr.step(torch.from_numpy(depth).cuda(), torch.from_numpy(obj).cuda(),
             torch.from_numpy(np.ascontiguousarray(sen)).cuda())
    torch.cuda.synchronize()
    r_rgb, r_fn, r_ft, r_force, r_torque = oracle_step(lut, pts, sdf, depth, obj, sen)
    F = E * S
    u8 = arr.rgb_u8.cpu().numpy().reshape(r_rgb.shape)
    assert np.abs(u8.astype(int) - r_rgb.astype(int)).max() <= 1
    f32 = arr.rgb_f32.cpu().numpy().reshape((F,) + r_rgb.shape[1:])
    ref_f = O.depth_to_rgb(depth.reshape((F,) + depth.shape[2:]), lut.coeffs, lut.degree)
    assert np.abs(f32 - ref_f).max() < 2e-5
    assert arr.f_n.dtype == torch.float64
    assert vec_close(arr.f_n.cpu().numpy().reshape(r_fn.shape), r_fn, 1e-9, atol=1e-12)[0]
    assert vec_close(arr.f_t.cpu().numpy().reshape(r_ft.shape), r_ft, 1e-9, atol=1e-12)[0]
    w = arr.wrench.cpu().numpy().reshape(F, 6)
    np.testing.assert_allclose(w[:, :3], r_force, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(w[:, 3:], r_torque, rtol=1e-9, atol=1e-12)
