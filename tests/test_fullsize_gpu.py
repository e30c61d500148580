"""Parity at BASELINE.json's full sizes (config 3: 4096 envs x 2 sensors,
240x320 RGB + 20x25 force field; config 5: 8192 frames of 480x640, more than
2^31 pixels per launch).  The oracle cannot run 8192 frames in seconds, so the
whole batch is checked through size-independent properties:

* sampled frames (first, last, scheduler-unit boundaries, random) against the
  oracle (RGB +-1 LSB, force field 1e-5 relative);
* batch independence: every sampled frame computed alone is bit-identical to
  the same frame inside the full batch;
* shift equivariance of the gradient stencil: rolling every depth map by k
  rows / columns rolls the RGB interior by exactly k (bit-exact; catches band,
  halo and column-quad bookkeeping errors anywhere in the batch);
* linearity of the wrench: the fused per-sensor reduction equals the fp64
  sum over the returned per-taxel forces;
* empty batches are a no-op.
"""
import numpy as np
import pytest
import torch

from conftest import sdf_tuple, vec_close
from oracle import gelsim_oracle as O
from paper_2408_06506_b200 import SensorArray, synthetic
from paper_2408_06506_b200.render import depth_to_rgb_device, device_lut
from paper_2408_06506_b200.tactile import PenaltyParams, device_taxels, force_field_device

pytestmark = pytest.mark.gpu

E, S = 4096, 2
F = E * S


def _distinct_batch(cam, bg, n, H, W, seed):
    """n distinct depth maps on the device: 64 rendered indenters tiled, each
    copy perturbed by its own +-0.5 um noise (changes every gradient)."""
    pool = torch.from_numpy(synthetic.depth_batch(cam, bg, 64, config_id=seed)).cuda()
    reps = -(-n // 64)
    d = pool.repeat(reps, 1, 1)[:n].contiguous()
    g = torch.Generator(device="cuda").manual_seed(seed)
    d += (torch.rand(d.shape, generator=g, device="cuda") - 0.5) * 1e-6
    return d


@pytest.fixture(scope="module")
def full():
    _, cam, bg, lut, pts = synthetic.sensor_setup((320, 240), (20, 25))
    sdf = synthetic.peg_grid((32, 32, 64))
    obj, sen = synthetic.peg_states(E, S, config_id=3)
    depth = _distinct_batch(cam, bg, F, 240, 320, seed=3).view(E, S, 240, 320)
    arr = SensorArray(lut, sdf, pts, PenaltyParams(), E, S, ff_fp64=True)
    o = torch.from_numpy(obj).cuda()
    s = torch.from_numpy(np.ascontiguousarray(sen)).cuda()
    arr.step(depth, o, s)
    torch.cuda.synchronize()
    return dict(lut=lut, pts=pts, sdf=sdf, obj=obj, sen=sen, depth=depth, arr=arr, o=o, s=s)


def _ff(full, o, s):
    """K2 on env rows (o (e, 13), s (e, S, 13)) into fresh fp64 outputs."""
    e = s.shape[0]
    f_n = torch.empty((e, S, 20, 25, 3), dtype=torch.float64, device="cuda")
    f_t = torch.empty_like(f_n)
    w = torch.empty((e, S, 6), dtype=torch.float64, device="cuda")
    tax = device_taxels(full["pts"], f_n.device)
    force_field_device(full["sdf"], tax, 20, 25, o.contiguous(), s.contiguous(), PenaltyParams(), f_n, f_t, w,
                       n_sensors=S)
    return f_n, f_t, w


def _sample(n, rng, extra=()):
    idx = {0, 1, n // 2, n - 2, n - 1, *extra}
    idx.update(int(i) for i in rng.integers(0, n, 8))
    return np.array(sorted(i for i in idx if 0 <= i < n))


def test_full_batch_sampled_frames_vs_oracle(full):
    arr = full["arr"]
    idx = _sample(F, np.random.default_rng(0), extra=(147, 148, 295, 296, 4095, 4096))
    depth = full["depth"].view(F, 240, 320)[torch.from_numpy(idx).cuda()].cpu().numpy()
    env, sensor = idx // S, idx % S
    obj = full["obj"][env]
    sen = full["sen"][env, sensor]
    rgb, f_n, f_t, force, torque = O.sensor_frames(depth, full["lut"].coeffs, full["lut"].degree,
                                                   full["pts"].points, sdf_tuple(full["sdf"]), obj, sen,
                                                   (1000.0, 100.0, 10.0, 2.0))
    got = arr.rgb_u8.view(F, 240, 320, 3)[torch.from_numpy(idx).cuda()].cpu().numpy()
    assert np.abs(got.astype(int) - rgb.astype(int)).max() <= 1
    fn = arr.f_n.view(F, 20, 25, 3).cpu().numpy()[idx]
    ft = arr.f_t.view(F, 20, 25, 3).cpu().numpy()[idx]
    assert vec_close(fn, f_n, 1e-5, atol=1e-9)[0]
    assert vec_close(ft, f_t, 1e-5, atol=1e-9)[0]
    w = arr.wrench.view(F, 6).cpu().numpy()[idx]
    np.testing.assert_allclose(w[:, :3], force, rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(w[:, 3:], torque, rtol=1e-9, atol=1e-12)
    assert (np.abs(f_n).sum(axis=(1, 2, 3)) > 0).any(), "sample has no contact"


def test_full_batch_frames_are_independent(full):
    arr = full["arr"]
    idx = torch.from_numpy(_sample(F, np.random.default_rng(1), extra=(7, 8191))).cuda()
    sub = full["depth"].view(F, 240, 320)[idx].contiguous()
    rgb = torch.empty(sub.shape + (3,), dtype=torch.uint8, device="cuda")
    depth_to_rgb_device(sub, device_lut(full["lut"]), out_u8=rgb)
    torch.cuda.synchronize()
    assert torch.equal(rgb, arr.rgb_u8.view(F, 240, 320, 3)[idx])

    env = torch.unique(idx // S)
    f_n, f_t, w = _ff(full, full["o"][env], full["s"][env])
    torch.cuda.synchronize()
    assert torch.equal(f_n, arr.f_n[env])
    assert torch.equal(f_t, arr.f_t[env])
    # a small batch runs wider CTAs per frame, so the per-sensor fp64 sum is
    # reduced in a different order: equal to rounding, not bit for bit
    torch.testing.assert_close(w, arr.wrench[env], rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("axis,k", [(-1, 1), (-1, 4), (-1, 37), (-2, 1), (-2, 8), (-2, 61)])
def test_full_batch_shift_equivariance(full, axis, k):
    arr = full["arr"]
    d = full["depth"].view(F, 240, 320)
    shifted = torch.roll(d, k, dims=axis).contiguous()
    out = torch.empty(shifted.shape + (3,), dtype=torch.uint8, device="cuda")
    depth_to_rgb_device(shifted, device_lut(full["lut"]), out_u8=out)
    torch.cuda.synchronize()
    ref = arr.rgb_u8.view(F, 240, 320, 3)
    dim = 2 if axis == -1 else 1
    n = 320 if axis == -1 else 240
    # interior pixels whose 3-wide stencil does not touch a border or the wrap
    a = ref.narrow(dim, 1, n - k - 2)
    b = out.narrow(dim, 1 + k, n - k - 2)
    assert torch.equal(a, b)
    del out, shifted


def test_full_batch_wrench_is_sum_of_taxel_forces(full):
    arr = full["arr"]
    f = (arr.f_n + arr.f_t).view(F, 500, 3)
    p = torch.from_numpy(np.asarray(full["pts"].points, dtype=np.float64).reshape(500, 3)).cuda()
    force = f.sum(dim=1)
    torque = torch.cross(p.expand_as(f), f, dim=-1).sum(dim=1)
    w = arr.wrench.view(F, 6)
    scale_f = f.abs().sum(dim=1).clamp_min(1e-300)  # (F, 3)
    scale_t = (p.norm(dim=-1) * f.norm(dim=-1)).sum(dim=1).clamp_min(1e-300).unsqueeze(-1)
    assert ((w[:, :3] - force).abs() <= 1e-12 * scale_f + 1e-300).all()
    assert ((w[:, 3:] - torque).abs() <= 1e-12 * scale_t + 1e-300).all()
    assert (force.abs().sum(dim=1) > 0).sum() > F // 10, "too few frames in contact"


def test_empty_batches_are_noops(full):
    lut = device_lut(full["lut"])
    d = torch.empty((0, 240, 320), dtype=torch.float32, device="cuda")
    out = torch.empty((0, 240, 320, 3), dtype=torch.uint8, device="cuda")
    depth_to_rgb_device(d, lut, out_u8=out)
    f_n, f_t, w = _ff(full, full["o"][:0], full["s"][:0])
    torch.cuda.synchronize()
    assert f_n.shape[0] == 0 and w.shape[0] == 0
    # the numpy-level drop-in keeps the reference's shape/dtype for E = 0
    from paper_2408_06506_b200.render import DepthImage, depth_to_rgb
    img = depth_to_rgb(DepthImage(values=np.zeros((0, 240, 320)), background=np.zeros((240, 320))), full["lut"])
    assert img.shape == (0, 240, 320, 3) and img.dtype == np.float64


def test_over_2e31_pixels_single_launch():
    """Config 5 (8192 x 480x640 = 2.5 G pixels): offsets past 2^31 elements."""
    _, cam, bg, lut, _ = synthetic.sensor_setup((640, 480), (20, 25))
    n = 8192
    free, _ = torch.cuda.mem_get_info()
    need = n * 480 * 640 * (4 + 3)
    if free < need * 1.2:
        pytest.skip("not enough device memory")
    d = _distinct_batch(cam, bg, n, 480, 640, seed=5)
    out = torch.empty((n, 480, 640, 3), dtype=torch.uint8, device="cuda")
    depth_to_rgb_device(d, device_lut(lut), out_u8=out)
    torch.cuda.synchronize()
    idx = np.array([0, 4096, 4661, 6990, 8190, 8191])  # 4661 ~ the 2^31 element
    ref = O.to_uint8(O.depth_to_rgb(d[torch.from_numpy(idx).cuda()].cpu().numpy(), lut.coeffs, lut.degree))
    got = out[torch.from_numpy(idx).cuda()].cpu().numpy()
    assert np.abs(got.astype(int) - ref.astype(int)).max() <= 1
    del d, out
    torch.cuda.empty_cache()


def test_config4_shape_fast_kernel_vs_oracle():
    """Config 4's shapes (80x100 taxels, 128^3 SDF) through the fast K2 path
    (no kinematics): masks bit-exact, forces within 1e-5 of the oracle, and
    the full 16384-env batch equals its sampled envs computed alone."""
    from paper_2408_06506_b200.sensors import TactileSensorSpec
    from paper_2408_06506_b200.tactile import sample_tactile_points
    sdf = synthetic.peg_grid((128, 128, 128))
    pts = sample_tactile_points(TactileSensorSpec(image_size=(320, 240)), 80, 100)
    E4 = 16384
    obj, sen = synthetic.peg_states(E4, 1, config_id=4)
    o = torch.from_numpy(obj).cuda()
    s = torch.from_numpy(np.ascontiguousarray(sen)).cuda()
    tax = device_taxels(pts, o.device)
    f_n = torch.empty((E4, 1, 80, 100, 3), dtype=torch.float32, device="cuda")
    f_t = torch.empty_like(f_n)
    c = torch.empty((E4, 1, 80, 100), dtype=torch.uint8, device="cuda")
    force_field_device(sdf, tax, 80, 100, o, s, PenaltyParams(), f_n, f_t, contact=c, n_sensors=1)
    torch.cuda.synchronize()
    idx = np.array([0, 1, 4097, 9000, E4 - 1])
    rn, rt, rk = O.compute_force_field(pts.points, *sdf_tuple(sdf), obj[idx, 0:3], obj[idx, 3:7], obj[idx, 7:10],
                                       obj[idx, 10:13], sen[idx, 0, 0:3], sen[idx, 0, 3:7], sen[idx, 0, 7:10],
                                       sen[idx, 0, 10:13])
    ti = torch.from_numpy(idx).cuda()
    assert np.array_equal(c[ti, 0].cpu().numpy().astype(bool), rk["d"] < 0)
    assert (rk["d"] < 0).mean() > 0.02
    assert vec_close(f_n[ti, 0].cpu().numpy(), rn, 1e-5, atol=1e-9)[0]
    assert vec_close(f_t[ti, 0].cpu().numpy(), rt, 1e-5, atol=1e-9)[0]
    sub_n = torch.empty((len(idx), 1, 80, 100, 3), dtype=torch.float32, device="cuda")
    sub_t = torch.empty_like(sub_n)
    force_field_device(sdf, tax, 80, 100, o[ti].contiguous(), s[ti].contiguous(), PenaltyParams(), sub_n, sub_t,
                       n_sensors=1)
    torch.cuda.synchronize()
    assert torch.equal(sub_n, f_n[ti]) and torch.equal(sub_t, f_t[ti])


def test_config4_quad_kernel_equals_fp64_kernel_full_batch(monkeypatch):
    """The whole config-4 batch (16384 x 8000 taxels, 128^3 SDF): the
    certified fp32 pre-pass (quad kernel, the default on dense pads) and the
    fp64 fast kernel give identical contact masks on all 131 M taxels, and
    forces / wrenches within the fp32 output rounding."""
    from conftest import vec_close as vc
    from paper_2408_06506_b200.sensors import TactileSensorSpec
    from paper_2408_06506_b200.tactile import sample_tactile_points
    sdf = synthetic.peg_grid((128, 128, 128))
    pts = sample_tactile_points(TactileSensorSpec(image_size=(320, 240)), 80, 100)
    E4 = 16384
    obj, sen = synthetic.peg_states(E4, 1, config_id=4)
    o = torch.from_numpy(obj).cuda()
    s = torch.from_numpy(np.ascontiguousarray(sen)).cuda()
    tax = device_taxels(pts, o.device)

    def run():
        f_n = torch.empty((E4, 1, 80, 100, 3), dtype=torch.float32, device="cuda")
        f_t = torch.empty_like(f_n)
        w = torch.empty((E4, 1, 6), dtype=torch.float64, device="cuda")
        c = torch.empty((E4, 1, 80, 100), dtype=torch.uint8, device="cuda")
        force_field_device(sdf, tax, 80, 100, o, s, PenaltyParams(), f_n, f_t, wrench=w, contact=c, n_sensors=1)
        torch.cuda.synchronize()
        return f_n, f_t, w, c

    q = run()
    monkeypatch.setenv("TACSL_FF_QUAD", "0")
    f = run()
    assert torch.equal(q[3], f[3])
    assert 0.2 < q[3].float().mean().item() < 0.35
    for a, b in zip(q[:2], f[:2]):
        d = (a.double() - b.double()).norm(dim=-1)
        assert bool((d <= 2e-7 * b.double().norm(dim=-1) + 1e-12).all())
    scale = (q[0].double() + q[1].double()).abs().sum(dim=(1, 2, 3)).unsqueeze(-1)
    assert bool(((q[2] - f[2])[..., 0:3].abs() <= 1e-6 * scale + 1e-12).all())
