"""K7 (csrc/pyramid_fused.cu): smoothing + every pyramid level's RGB in one
pass.  CPU: the kernel's tick schedule (which rows each phase of a tick
touches) produces every output row exactly once, after all its inputs, for
every height, radius and level count.  GPU: bit-identical to the unfused
chain (K5 smoothing / pyr_down -> K1 per level), which tests/test_pyramid.py
pins to the float64 restatement."""
import numpy as np
import pytest

from paper_2408_06506_b200 import smoothing, synthetic


def _ticks(H, levels):
    # pyramid_fused.cu pyramid_ticks
    k = (H + 1 + 7) // 8 + 1
    if levels >= 2:
        k = max(k, (H + 4 + 7) // 8 + 1, (H // 2 + 3 + 3) // 4 + 1)
    if levels >= 3:
        k = max(k, (H // 4 + 2 + 1) // 2 + 1)
    return k


def _schedule(H, R, levels):
    """Replays the kernel's per-tick row sets; asserts the dependencies."""
    H1, H2 = H // 2, H // 4
    clamp = lambda v, n: min(max(v, 0), n - 1)  # noqa: E731
    s0, l1, l2, shaded = set(), set(), set(), [set(), set(), set()]
    acc1, acc2 = {}, {}
    kG = (H + 7) // 8
    for k in range(_ticks(H, levels)):
        if k <= kG:
            for j in range(8 * k - 4, 8 * k + 4):
                if 0 <= j - R < H:
                    # every tap row clamp(j - 2R .. j) has been loaded by now
                    s0.add(j - R)
        for y in range(8 * k - 9, 8 * k - 1):
            if 0 <= y < H:
                assert {clamp(y - 1, H), y, clamp(y + 1, H)} <= s0, (k, y)
                assert y not in shaded[0]
                shaded[0].add(y)
        if levels >= 2:
            for i in range(8 * k - 10, 8 * k - 2):
                for t in range(4, -1, -1):
                    if (i - t) % 2:
                        continue
                    y1 = (i + 2 - t) // 2
                    if not 0 <= y1 < H1:
                        continue
                    assert clamp(i, H) in s0
                    acc1.setdefault(y1, []).append(t)
                    if t == 4:
                        assert acc1[y1] == [0, 1, 2, 3, 4] and y1 not in l1
                        l1.add(y1)
            for y in range(4 * k - 7, 4 * k - 3):
                if 0 <= y < H1:
                    assert {clamp(y - 1, H1), y, clamp(y + 1, H1)} <= l1, (k, y)
                    assert y not in shaded[1]
                    shaded[1].add(y)
        if levels >= 3:
            for i in range(4 * k - 6, 4 * k - 2):
                for t in range(4, -1, -1):
                    if (i - t) % 2:
                        continue
                    y2 = (i + 2 - t) // 2
                    if not 0 <= y2 < H2:
                        continue
                    assert clamp(i, H1) in l1
                    acc2.setdefault(y2, []).append(t)
                    if t == 4:
                        assert acc2[y2] == [0, 1, 2, 3, 4]
                        l2.add(y2)
            rows = list(range(2 * k - 5, 2 * k - 3)) + ([2 * k - 3] if 2 * k - 3 == H2 - 1 else [])
            for y in rows:
                if 0 <= y < H2:
                    assert {clamp(y - 1, H2), y, clamp(y + 1, H2)} <= l2, (k, y)
                    assert y not in shaded[2]
                    shaded[2].add(y)
    assert shaded[0] == set(range(H))
    if levels >= 2:
        assert shaded[1] == set(range(H1))
    if levels >= 3:
        assert shaded[2] == set(range(H2))


@pytest.mark.parametrize("levels", [1, 2, 3])
@pytest.mark.parametrize("R", [0, 1, 2, 3, 4])
def test_tick_schedule_covers_every_row_once(levels, R):
    for H in range(4, 1000, 4):
        _schedule(H, R, levels)


# ------------------------------------------------------------------ GPU ---

def _chain(d, lut, levels, sigma):
    return smoothing.rgb_pyramid_device(d, lut, levels=levels, sigma=sigma)


@pytest.mark.gpu
@pytest.mark.parametrize("hw", [(480, 640), (240, 320), (60, 80), (36, 44), (36, 48), (8, 8), (100, 768),
                                (484, 644), (484, 648)])
@pytest.mark.parametrize("sigma", [0.0, 1.0])
def test_fused_pyramid_bit_identical_to_chain(hw, sigma):
    import torch
    H, W = hw
    _, cam, bg, lut, _ = synthetic.sensor_setup((W, H))
    d = torch.from_numpy(synthetic.depth_batch(cam, bg, 5, config_id=81)).cuda()
    d += (torch.rand(d.shape, generator=torch.Generator(device="cuda").manual_seed(1), device="cuda") - 0.5) * 1e-6
    for levels in (1, 2, 3):
        if not smoothing.fused_pyramid_supported(H, W, levels, sigma):
            assert levels == 3 and W % 8 != 0  # three levels need W % 8 == 0 (level-2 pixel pairs)
            continue
        got = smoothing.rgb_pyramid_fused_device(d, lut, levels=levels, sigma=sigma)
        ref = _chain(d, lut, levels, sigma)
        torch.cuda.synchronize()
        for lvl in range(levels):
            assert got[lvl].shape == ref[lvl].shape
            assert torch.equal(got[lvl], ref[lvl]), (hw, sigma, levels, lvl,
                                                     (got[lvl] != ref[lvl]).nonzero()[:5].tolist())


@pytest.mark.gpu
@pytest.mark.parametrize("sigma", [0.3, 0.5, 0.75])
@pytest.mark.parametrize("degree", [2, 3, 4])
def test_fused_pyramid_radii_and_degrees(sigma, degree):
    import torch
    H, W = 120, 160
    _, cam, bg, lut, _ = synthetic.sensor_setup((W, H), lut_degree=degree)
    d = torch.from_numpy(synthetic.depth_batch(cam, bg, 3, config_id=82)).cuda()
    got = smoothing.rgb_pyramid_fused_device(d, lut, levels=3, sigma=sigma)
    ref = _chain(d, lut, 3, sigma)
    torch.cuda.synchronize()
    for a, b in zip(got, ref):
        assert torch.equal(a, b)


@pytest.mark.gpu
def test_fused_pyramid_many_images_per_cta_and_batched_shape():
    """More images than resident CTAs (each CTA streams several images
    through its rings) and a (E, S, H, W) batch."""
    import torch
    H, W = 64, 96
    _, cam, bg, lut, _ = synthetic.sensor_setup((W, H))
    d = torch.from_numpy(synthetic.depth_batch(cam, bg, 64, config_id=83)).cuda()
    d = d.repeat(20, 1, 1)
    d += (torch.rand(d.shape, generator=torch.Generator(device="cuda").manual_seed(2), device="cuda") - 0.5) * 1e-6
    d = d.view(640, 2, H, W)
    got = smoothing.rgb_pyramid_fused_device(d, lut, levels=3, sigma=1.0)
    ref = _chain(d, lut, 3, 1.0)
    torch.cuda.synchronize()
    assert got[0].shape == (640, 2, H, W, 3) and got[2].shape == (640, 2, H // 4, W // 4, 3)
    for a, b in zip(got, ref):
        assert torch.equal(a, b)


@pytest.mark.gpu
def test_fused_pyramid_errors():
    import torch
    from paper_2408_06506_b200.errors import LutResolutionMismatch
    _, cam, bg, lut, _ = synthetic.sensor_setup((80, 60))
    assert not smoothing.fused_pyramid_supported(62, 80, 3)   # H % 4
    assert not smoothing.fused_pyramid_supported(60, 82, 3)   # W % 4
    assert not smoothing.fused_pyramid_supported(60, 2048, 3)  # too wide
    assert not smoothing.fused_pyramid_supported(60, 76, 3) and smoothing.fused_pyramid_supported(60, 76, 2)
    assert not smoothing.fused_pyramid_supported(60, 80, 4)   # levels
    d = torch.zeros((2, 62, 80), device="cuda")
    with pytest.raises(ValueError):
        smoothing.rgb_pyramid_fused_device(d, lut, levels=3)
    d = torch.full((2, 64, 80), 0.02, device="cuda")
    with pytest.raises(LutResolutionMismatch):
        smoothing.rgb_pyramid_fused_device(d, lut, levels=3)  # LUT calibrated at 80x60
