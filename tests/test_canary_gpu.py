"""Out-of-bounds writes: every kernel writes into a slice of a larger buffer
whose tail (and head) carry a canary pattern; after the launch the canaries
must be intact.  compute-sanitizer is not available on the GPU pool, so this
guards the bulk-store / band / tail logic at awkward sizes directly."""
import numpy as np
import pytest
import torch

from paper_2408_06506_b200 import smoothing, synthetic
from paper_2408_06506_b200.binned import depth_to_rgb_binned_device, vignetted_lut
from paper_2408_06506_b200.render import depth_to_rgb_device
from paper_2408_06506_b200.tactile import PenaltyParams, device_taxels, force_field_device

pytestmark = pytest.mark.gpu

PAD = 4096  # bytes of canary on each side


def guarded(shape, dtype):
    """(view, full): `view` is a contiguous tensor of `shape` inside `full`,
    16-B aligned, with PAD canary bytes before and after."""
    n = int(np.prod(shape))
    esz = torch.empty((), dtype=dtype).element_size()
    full = torch.full((n + 2 * PAD // esz,), 0, dtype=dtype, device="cuda")
    full.view(torch.uint8).fill_(0xA5)
    view = full[PAD // esz: PAD // esz + n].view(shape)
    return view, full


def intact(full, dtype):
    esz = torch.empty((), dtype=dtype).element_size()
    b = full.view(torch.uint8)
    return bool((b[:PAD] == 0xA5).all()) and bool((b[b.numel() - PAD:] == 0xA5).all())


@pytest.mark.parametrize("hw", [(240, 320), (61, 84), (29, 37), (2, 4), (7, 1284)])
@pytest.mark.parametrize("n", [1, 3, 37])
def test_k1_canaries(hw, n):
    H, W = hw
    _, cam, bg, lut, _ = synthetic.sensor_setup((W, H))
    d = torch.rand((n, H, W), device="cuda") * 1e-3 + 0.02
    u8, fu = guarded((n, H, W, 3), torch.uint8)
    f32, ff = guarded((n, H, W, 3), torch.float32)
    depth_to_rgb_device(d, lut, out_u8=u8, out_f32=f32)
    torch.cuda.synchronize()
    assert intact(fu, torch.uint8) and intact(ff, torch.float32)
    assert int(u8.view(torch.uint8).float().sum()) > 0


@pytest.mark.parametrize("hw,step,radius", [((240, 320), 1, 4), ((480, 640), 2, 2), ((29, 40), 2, 2),
                                            ((31, 72), 1, 7), ((5, 12), 1, 1)])
def test_k5_canaries(hw, step, radius):
    H, W = hw
    d = torch.rand((3, H, W), device="cuda")
    Ho, Wo = -(-H // step), -(-W // step)
    out, full = guarded((3, Ho, Wo), torch.float32)
    taps = np.ones(2 * radius + 1) / (2 * radius + 1)
    smoothing.separable_filter_device(d, taps, step, out=out)
    torch.cuda.synchronize()
    assert intact(full, torch.float32)


@pytest.mark.parametrize("size,bins", [((320, 240), (6, 8)), ((37, 29), (5, 7)), ((84, 61), (61, 3))])
def test_k6_canaries(size, bins):
    W, H = size
    _, cam, bg, lut, _ = synthetic.sensor_setup(size)
    d = torch.rand((5, H, W), device="cuda") * 1e-3 + 0.02
    u8, fu = guarded((5, H, W, 3), torch.uint8)
    depth_to_rgb_binned_device(d, vignetted_lut(lut, bins), out_u8=u8)
    torch.cuda.synchronize()
    assert intact(fu, torch.uint8)


@pytest.mark.parametrize("grid,E,S", [((20, 25), 37, 2), ((10, 14), 1, 2), ((80, 100), 5, 1), ((3, 5), 300, 1)])
def test_k2_canaries(grid, E, S):
    from paper_2408_06506_b200.sensors import TactileSensorSpec
    from paper_2408_06506_b200.tactile import sample_tactile_points
    R, C = grid
    sdf = synthetic.peg_grid((32, 32, 64))
    pts = sample_tactile_points(TactileSensorSpec(), R, C)
    obj, sen = synthetic.peg_states(E, S, config_id=5)
    o = torch.from_numpy(obj).cuda()
    s = torch.from_numpy(np.ascontiguousarray(sen)).cuda()
    f_n, fa = guarded((E, S, R, C, 3), torch.float32)
    f_t, fb = guarded((E, S, R, C, 3), torch.float32)
    w, fc = guarded((E, S, 6), torch.float64)
    obs, fd = guarded((E, S, R, C, 3), torch.float32)
    force_field_device(sdf, device_taxels(pts, o.device), R, C, o, s, PenaltyParams(), f_n, f_t, wrench=w, obs=obs,
                       n_sensors=S)
    torch.cuda.synchronize()
    assert all(intact(f, dt) for f, dt in ((fa, torch.float32), (fb, torch.float32), (fc, torch.float64),
                                           (fd, torch.float32)))


@pytest.mark.parametrize("size,E", [((80, 60), 3), ((37, 29), 5)])
def test_k3_k4_canaries(size, E):
    from paper_2408_06506_b200 import AugmentConfig
    from paper_2408_06506_b200.augment import augment_device
    from paper_2408_06506_b200.depth import RayTable, env_params, render_depth_device
    W, H = size
    _, cam, bg, lut, _ = synthetic.sensor_setup(size)
    sdf = synthetic.peg_grid((32, 32, 64))
    obj, _ = synthetic.peg_states(E, 1, config_id=6, random_sensor_pose=False)
    params = torch.from_numpy(env_params(sdf, obj[:, 0:3], obj[:, 3:7])).cuda()
    d64, f64 = guarded((E, H, W), torch.float64)
    d32, f32 = guarded((E, H, W), torch.float32)
    render_depth_device(RayTable(cam, bg, torch.device("cuda")), sdf, params, out_f64=d64, out_f32=d32)
    rgb = torch.rand((E, H, W, 3), device="cuda")
    cfg = AugmentConfig(shift_px=1.0, zoom=(0.9, 1.1), brightness=0.05, hue=0.02, channel_permutation=True, seed=3)
    seeds = torch.arange(E, dtype=torch.int64, device="cuda")
    out, fo = guarded((E, H, W, 6), torch.float32)
    augment_device(rgb, cfg, seeds, seeds, tactile_rep="concat", nominal=np.float32([0.3, 0.4, 0.5]), out=out)
    torch.cuda.synchronize()
    assert intact(f64, torch.float64) and intact(f32, torch.float32) and intact(fo, torch.float32)


@pytest.mark.parametrize("hw", [(480, 640), (36, 48), (8, 8), (484, 648), (12, 1024)])
@pytest.mark.parametrize("n", [1, 5])
def test_k7_canaries(hw, n):
    """K7 writes every level's RGB (3 outputs per image) and nothing beyond."""
    H, W = hw
    _, cam, bg, lut, _ = synthetic.sensor_setup((W, H))
    d = torch.rand((n, H, W), device="cuda") * 1e-3 + 0.02
    views = [guarded((n, H >> lvl, W >> lvl, 3), torch.uint8) for lvl in range(3)]
    smoothing.rgb_pyramid_fused_device(d, lut, levels=3, sigma=1.0, outs=[v for v, _ in views])
    torch.cuda.synchronize()
    for v, full in views:
        assert intact(full, torch.uint8)
        assert int(v.float().sum()) > 0
