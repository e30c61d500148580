"""Gaussian smoothing / pyramid (north_star stages with no reference
counterpart: parity against gelsim is unpinned).
The CPU restatement is checked against scipy.ndimage; the kernels against
the restatement."""
import numpy as np
import pytest

from oracle import gelsim_oracle as O
from oracle.pyramid_oracle import separable_filter
from paper_2408_06506_b200 import smoothing, synthetic


def test_gaussian_taps_match_scipy():
    from scipy.ndimage import _filters
    for sigma in (0.5, 1.0, 2.3):
        w = smoothing.gaussian_taps(sigma)
        r = int(4.0 * sigma + 0.5)
        ref = _filters._gaussian_kernel1d(sigma, 0, r)[::-1]
        np.testing.assert_allclose(w, ref, rtol=1e-15)


@pytest.mark.parametrize("sigma", [0.8, 1.5])
def test_restatement_matches_scipy_gaussian_filter(sigma):
    from scipy.ndimage import gaussian_filter
    rng = np.random.default_rng(0)
    img = rng.normal(size=(2, 23, 31))
    got = separable_filter(img, smoothing.gaussian_taps(sigma), 1)
    ref = np.stack([gaussian_filter(im, sigma, mode="nearest", truncate=4.0) for im in img])
    np.testing.assert_allclose(got, ref, atol=1e-12)


def test_restatement_pyr_down_matches_scipy():
    from scipy.ndimage import correlate1d
    rng = np.random.default_rng(1)
    img = rng.normal(size=(17, 24))
    ref = correlate1d(correlate1d(img, smoothing.BINOMIAL5, axis=1, mode="nearest"),
                      smoothing.BINOMIAL5, axis=0, mode="nearest")[::2, ::2]
    np.testing.assert_allclose(separable_filter(img, smoothing.BINOMIAL5, 2), ref, atol=1e-13)


def test_level_lut_scaling():
    lut = synthetic.sensor_setup((640, 480))[3]
    l2 = smoothing.level_lut(lut, 2)
    assert l2.image_size == (160, 120)
    np.testing.assert_allclose(l2.coeffs[:, 1], lut.coeffs[:, 1] / 4)
    np.testing.assert_allclose(l2.coeffs[:, 3], lut.coeffs[:, 3] / 16)


@pytest.mark.gpu
@pytest.mark.parametrize("size", [(320, 240), (37, 29)])
@pytest.mark.parametrize("sigma", [0.0, 1.0, 2.5])
def test_gpu_filters_match_restatement(size, sigma):
    import torch
    _, cam, bg, _, _ = synthetic.sensor_setup(size)
    d = synthetic.depth_batch(cam, bg, 3, config_id=71)
    dev = torch.from_numpy(d).cuda()
    if sigma:
        got = smoothing.gaussian_blur_device(dev, sigma).cpu().numpy()
        ref = separable_filter(d, smoothing.gaussian_taps(sigma), 1)
        np.testing.assert_allclose(got, ref, rtol=0, atol=2e-8)
    got = smoothing.pyr_down_device(dev).cpu().numpy()
    ref = separable_filter(d, smoothing.BINOMIAL5, 2)
    assert got.shape == ref.shape
    np.testing.assert_allclose(got, ref, rtol=0, atol=2e-8)


@pytest.mark.gpu
def test_gpu_rgb_pyramid_vs_restatement():
    import torch
    size = (640, 480)
    _, cam, bg, lut, _ = synthetic.sensor_setup(size)
    d = synthetic.depth_batch(cam, bg, 2, config_id=72)
    levels = smoothing.rgb_pyramid_device(torch.from_numpy(d).cuda(), lut, levels=3, sigma=1.0)
    x = separable_filter(d, smoothing.gaussian_taps(1.0), 1)
    for lvl, u8 in enumerate(levels):
        if lvl:
            x = separable_filter(x, smoothing.BINOMIAL5, 2)
        ll = smoothing.level_lut(lut, lvl)
        ref = O.to_uint8(O.depth_to_rgb(x, ll.coeffs, ll.degree))
        got = u8.cpu().numpy()
        assert got.shape == ref.shape
        diff = np.abs(got.astype(int) - ref.astype(int))
        assert diff.max() <= 1 and (diff > 0).mean() < 2e-2, (lvl, diff.max(), (diff > 0).mean())


@pytest.mark.gpu
@pytest.mark.parametrize("hw", [(240, 320), (480, 640), (29, 40), (31, 72), (6, 16)])
@pytest.mark.parametrize("radius", [1, 2, 4, 7])
@pytest.mark.parametrize("step", [1, 2])
def test_gpu_bulk_filter_equals_generic_bit_exact(monkeypatch, hw, radius, step):
    """The warp-specialised band pipeline and the generic row-ring kernel
    accumulate in the same order: identical bits, every size and radius."""
    import torch
    H, W = hw
    if step == 2 and (-(-W // 2)) % 4:
        pytest.skip("bulk path needs Wo % 4 == 0")
    rng = np.random.default_rng(radius * 10 + step)
    d = torch.from_numpy(rng.uniform(0.02, 0.025, size=(5, H, W)).astype(np.float32)).cuda()
    taps = rng.uniform(0.1, 1.0, size=2 * radius + 1)
    taps /= taps.sum()
    fast = smoothing.separable_filter_device(d, taps, step)
    monkeypatch.setenv("TACSL_FILTER_GENERIC", "1")
    slow = smoothing.separable_filter_device(d, taps, step)
    torch.cuda.synchronize()
    assert torch.equal(fast, slow)
    ref = separable_filter(d.cpu().numpy(), taps.astype(np.float32), step)
    np.testing.assert_allclose(fast.cpu().numpy(), ref, rtol=0, atol=2e-8)


@pytest.mark.gpu
def test_sensor_array_pyramid_step_and_host_path():
    """SensorArray with smoothing + 3 pyramid levels (config 5's step) equals
    rgb_pyramid_device bit for bit, through the graph and the host path."""
    import torch
    from paper_2408_06506_b200 import SensorArray
    from paper_2408_06506_b200.tactile import PenaltyParams
    _, cam, bg, lut, pts = synthetic.sensor_setup((640, 480))
    E = 6
    d = torch.from_numpy(synthetic.depth_batch(cam, bg, E, config_id=73)).cuda().view(E, 1, 480, 640)
    arr = SensorArray(lut, synthetic.peg_grid(), pts, PenaltyParams(), E, 1, with_ff=False, pyramid_levels=3,
                      smooth_sigma=1.0)
    assert arr.fused_pyramid and arr.launches_per_step == 1  # K7: one pass
    ref = smoothing.rgb_pyramid_device(d, lut, levels=3, sigma=1.0)  # the level-by-level chain
    arr.capture(d, None, None)
    arr.replay()
    torch.cuda.synchronize()
    for lvl in range(3):
        assert torch.equal(arr.rgb_levels[lvl], ref[lvl]), lvl
    host = arr.host_buffers()
    host["depth"].copy_(d.cpu())
    d2 = torch.zeros_like(d)
    arr.run_host(host, d2, None, None, chunks=4)
    torch.cuda.synchronize()
    assert torch.equal(host["rgb"], ref[0].cpu())
    assert torch.equal(host["rgb_l1"], ref[1].cpu())
    assert torch.equal(host["rgb_l2"], ref[2].cpu())
