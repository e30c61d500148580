"""K1 (depth -> RGB) parity on the GPU against the reference's golden vectors
and the CPU oracle.  Contract (BASELINE.json north_star): uint8 RGB within
+-1 LSB per channel; float RGB within 2e-6 absolute (fp32 evaluation of a
polynomial whose reference value is float64)."""
import numpy as np
import pytest
import torch

from oracle import gelsim_oracle as O
from paper_2408_06506_b200 import render, synthetic
from paper_2408_06506_b200.errors import LutResolutionMismatch
from paper_2408_06506_b200.render import DepthImage, PolyLut, depth_to_rgb

pytestmark = pytest.mark.gpu

RGB_ATOL = 2e-6
LSB = 1


def lut_of(coeffs, W, H):
    deg = {6: 2, 10: 3, 15: 4}[np.asarray(coeffs).reshape(3, -1).shape[1]]
    return PolyLut(degree=deg, coeffs=coeffs, image_size=(W, H))


def check_u8(got, ref, max_frac=1e-4):
    diff = np.abs(got.astype(np.int16) - ref.astype(np.int16))
    assert diff.max() <= LSB, diff.max()
    assert (diff > 0).mean() <= max_frac, (diff > 0).mean()


@pytest.mark.parametrize("deg", [2, 3, 4])
def test_rgb_matches_reference_golden(golden, deg):
    z = golden("rgb")
    lut = lut_of(z[f"c60_deg{deg}"], 80, 60)
    got = depth_to_rgb(DepthImage(values=z["d60"], background=z["d60"][0]), lut)
    assert got.shape == (3, 60, 80, 3) and got.dtype == np.float64
    np.testing.assert_allclose(got, z[f"rgb60_deg{deg}"], rtol=0, atol=RGB_ATOL)
    u8 = depth_to_rgb(z["d60"], lut, out_dtype=np.uint8)
    check_u8(u8, z[f"u8_60_deg{deg}"])


def test_rgb_240x320_u8_golden(golden):
    z = golden("rgb")
    lut = lut_of(z["c240"], 320, 240)
    u8 = depth_to_rgb(z["d240"], lut, out_dtype=np.uint8)
    check_u8(u8, z["u8_240"])


def test_rgb_plain_lut_golden(golden):
    z = golden("rgb")
    got = depth_to_rgb(z["d60"], lut_of(z["c60_plain"], 80, 60))
    np.testing.assert_allclose(got, z["rgb60_plain"], atol=RGB_ATOL)


@pytest.mark.parametrize("hw", [(2, 3), (5, 7), (9, 18), (3, 2)])
def test_rgb_odd_sizes_golden(golden, hw):
    z = golden("rgb")
    H, W = hw
    got = depth_to_rgb(z[f"odd_{H}x{W}_d"], lut_of(z[f"odd_{H}x{W}_c"], W, H))
    np.testing.assert_allclose(got, z[f"odd_{H}x{W}_rgb"], atol=RGB_ATOL)


def test_rgb_flat_depth_is_background_exactly():
    # test_render.py:108-111
    lut = render.synthetic_lut((80, 60))
    rgb = depth_to_rgb(DepthImage(values=np.full((60, 80), 0.02), background=np.full((60, 80), 0.02)), lut)
    bg32 = lut.coeffs[:, 0].astype(np.float32).astype(np.float64)
    assert np.array_equal(rgb, np.broadcast_to(bg32, rgb.shape))


def test_rgb_tilted_plane_and_clamp(golden):
    # test_render.py:114-138
    z = golden("rgb")
    lut = PolyLut(degree=2, coeffs=z["tilt_c"], image_size=(80, 60))
    np.testing.assert_allclose(depth_to_rgb(z["tilt_d"], lut), z["tilt_rgb"], atol=RGB_ATOL)
    clamp = depth_to_rgb(z["clamp_d"], lut)
    assert clamp.max() <= 1.0 and np.all(clamp[..., 0] == 1.0)
    np.testing.assert_array_equal(clamp, z["clamp_rgb"])


def test_rgb_resolution_mismatch_and_small_images():
    lut = render.synthetic_lut((10, 10))
    with pytest.raises(LutResolutionMismatch):
        depth_to_rgb(np.zeros((60, 80), np.float32), lut)
    with pytest.raises(ValueError):
        depth_to_rgb(np.zeros((1, 10), np.float32), render.synthetic_lut((10, 1)))


@pytest.mark.parametrize("deg", [2, 3, 4])
@pytest.mark.parametrize("size", [(320, 240), (640, 480)])
def test_rgb_vs_oracle_full_resolution(deg, size):
    _, cam, bg, _, _ = synthetic.sensor_setup(size)
    lut = render.synthetic_lut(size, degree=deg, seed=deg, gradient_scale=synthetic.lut_scale(size))
    n = 6 if size[0] == 320 else 3
    d = synthetic.depth_batch(cam, bg, n, config_id=40 + deg)
    ref = O.depth_to_rgb(d, lut.coeffs, deg)
    got_f = depth_to_rgb(d, lut)
    np.testing.assert_allclose(got_f, ref, atol=RGB_ATOL)
    got_u8 = depth_to_rgb(d, lut, out_dtype=np.uint8)
    check_u8(got_u8, O.to_uint8(ref))
    assert len(np.unique(got_u8.reshape(-1, 3), axis=0)) > 1000   # non-vacuous parity


def test_rgb_device_tensors_and_batched_layout():
    size = (320, 240)
    _, cam, bg, lut, _ = synthetic.sensor_setup(size)
    d = synthetic.depth_batch(cam, bg, 6, config_id=7).reshape(3, 2, 240, 320)
    dev = torch.from_numpy(d).cuda()
    u8 = torch.empty((3, 2, 240, 320, 3), dtype=torch.uint8, device="cuda")
    f32 = torch.empty((3, 2, 240, 320, 3), dtype=torch.float32, device="cuda")
    render.depth_to_rgb_device(dev, lut, out_u8=u8, out_f32=f32)
    torch.cuda.synchronize()
    ref = O.depth_to_rgb(d, lut.coeffs, 2)
    np.testing.assert_allclose(f32.cpu().numpy(), ref, atol=RGB_ATOL)
    check_u8(u8.cpu().numpy(), O.to_uint8(ref))
    # fused u8 == to_uint8 of the fused float output, bit for bit
    assert torch.equal(render.to_uint8(f32), u8)


def test_rgb_scalar_path_equals_bulk_path(monkeypatch):
    size = (320, 240)
    _, cam, bg, lut, _ = synthetic.sensor_setup(size)
    d = torch.from_numpy(synthetic.depth_batch(cam, bg, 4, config_id=8)).cuda()
    a = depth_to_rgb(d, lut, out_dtype=np.uint8)
    monkeypatch.setenv("TACSL_RGB_FORCE_SCALAR", "1")
    b = depth_to_rgb(d, lut, out_dtype=np.uint8)
    assert torch.equal(a, b)


@pytest.mark.parametrize("groups,stages", [(1, 2), (2, 3), (4, 4), (6, 1), (5, 2), (13, 2)])
def test_rgb_pipeline_shapes(monkeypatch, groups, stages):
    size = (320, 240)
    _, cam, bg, lut, _ = synthetic.sensor_setup(size)
    d = torch.from_numpy(synthetic.depth_batch(cam, bg, 5, config_id=9)).cuda()
    ref = depth_to_rgb(d, lut, out_dtype=np.uint8)
    monkeypatch.setenv("TACSL_RGB_GROUPS", str(groups))
    monkeypatch.setenv("TACSL_RGB_STAGES", str(stages))
    assert torch.equal(depth_to_rgb(d, lut, out_dtype=np.uint8), ref)


def test_to_uint8_is_bit_exact():
    x = np.concatenate([np.linspace(-0.1, 1.1, 100001), (np.arange(256) + 0.5) / 255.0]).astype(np.float32)
    np.testing.assert_array_equal(render.to_uint8(x), O.to_uint8(x.astype(np.float64)))


def test_to_uint8_f64_is_bit_exact_at_rounding_boundaries():
    # values whose 255*x sits on, or one float64 ulp either side of, k + 1/2:
    # the f32-narrowing path of round 1 rounded some of these the other way
    k = np.arange(-2, 257, dtype=np.float64)
    mid = (k + 0.5) / 255.0
    x = np.concatenate([mid, np.nextafter(mid, np.inf), np.nextafter(mid, -np.inf),
                        np.nextafter(np.nextafter(mid, np.inf), np.inf),
                        k / 255.0, np.linspace(-0.2, 1.2, 200003),
                        np.array([0.0, -0.0, 1.0, np.inf, -np.inf, 1e300, -1e300])])
    ref = np.clip(np.rint(x * 255), 0, 255).astype(np.uint8)  # imageio.py:8-11 verbatim
    got = render.to_uint8(x)
    np.testing.assert_array_equal(got, ref)
    # and the f32-narrowed route really differs somewhere here (the test has teeth)
    with np.errstate(over="ignore"):
        x32 = x.astype(np.float32)
    assert (render.to_uint8(x32) != ref).any()
    # device float64 tensors take the same path
    assert torch.equal(render.to_uint8(torch.from_numpy(x).cuda()).cpu(), torch.from_numpy(ref))


def test_depth_to_rgb_float64_input_narrowed_on_device():
    size = (320, 240)
    _, cam, bg, lut, _ = synthetic.sensor_setup(size)
    d64 = synthetic.depth_batch(cam, bg, 3, config_id=12).astype(np.float64)
    d64 += np.random.default_rng(3).uniform(-1e-9, 1e-9, d64.shape)  # not f32-representable
    a = depth_to_rgb(d64, lut, out_dtype=np.uint8)
    b = depth_to_rgb(d64.astype(np.float32), lut, out_dtype=np.uint8)
    np.testing.assert_array_equal(a, b)  # device narrowing == numpy astype(float32)
    f = depth_to_rgb(render.DepthImage(values=d64, background=bg), lut)
    assert f.dtype == np.float64 and f.shape == d64.shape + (3,)
    ref = O.depth_to_rgb(d64, lut.coeffs, 2)
    # the kernels shade in fp32: sub-ulp depth noise moves values by ~1e-5
    np.testing.assert_allclose(f, ref, atol=3e-5)
    check_u8(O.to_uint8(f), O.to_uint8(ref), max_frac=1e-3)
    t64 = torch.from_numpy(d64).cuda()
    assert torch.equal(depth_to_rgb(t64, lut, out_dtype=np.uint8).cpu(), torch.from_numpy(a))


def test_dtype_conversions_round_like_numpy():
    from paper_2408_06506_b200 import _device
    rng = np.random.default_rng(5)
    for n in (0, 1, 3, 4, 5, 1023, 100001):
        x = rng.standard_normal(n) * 10.0 ** rng.integers(-30, 30, n)
        g = _device.as_f32(x, torch.device("cuda", 0))
        np.testing.assert_array_equal(g.cpu().numpy(), x.astype(np.float32))
        w = _device.widen_f64(g)
        np.testing.assert_array_equal(w.cpu().numpy(), x.astype(np.float32).astype(np.float64))
    # unaligned views take the scalar path
    x = rng.standard_normal(1001)
    t = torch.from_numpy(x).cuda()[1:]
    np.testing.assert_array_equal(_device.as_f32(t, t.device).cpu().numpy(), x[1:].astype(np.float32))
