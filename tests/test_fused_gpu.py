"""The fused sensor step (tacsl_sensor_step): K1 shading warps and K2
force-field warps in one persistent launch must produce the outputs of the
two separate launches (RGB bit for bit, forces to float64 rounding)."""
import numpy as np
import pytest
import torch

from paper_2408_06506_b200 import SensorArray, synthetic
from paper_2408_06506_b200.tactile import PenaltyParams

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("E,S,size,grid", [(37, 2, (320, 240), (20, 25)), (5, 1, (80, 60), (80, 100)),
                                           (600, 2, (320, 240), (20, 25)), (3, 2, (42, 30), (10, 14))])
def test_fused_equals_two_launches(E, S, size, grid):
    _, cam, bg, lut, pts = synthetic.sensor_setup(size, grid)
    sdf = synthetic.peg_grid((32, 32, 64))
    depth = synthetic.depth_batch(cam, bg, E * S, config_id=81, pool=16).reshape(E, S, size[1], size[0])
    obj, sen = synthetic.peg_states(E, S, config_id=81)
    d = torch.from_numpy(np.ascontiguousarray(depth)).cuda()
    o = torch.from_numpy(obj).cuda()
    s = torch.from_numpy(np.ascontiguousarray(sen)).cuda()
    fused = SensorArray(lut, sdf, pts, PenaltyParams(), E, S, fused=True)
    split = SensorArray(lut, sdf, pts, PenaltyParams(), E, S, fused=False)
    assert fused.fused and not split.fused
    fused.launch(d, o, s)
    split.launch(d, o, s)
    torch.cuda.synchronize()
    assert torch.equal(fused.rgb_u8, split.rgb_u8)
    # the fused force-field warps run the reference chain for every taxel,
    # the standalone K2 its fast chain (exact only near decisions): same
    # contact mask, forces equal up to float64 rounding before the fp32 cast
    assert torch.equal(fused.f_n.abs().sum(-1) > 0, split.f_n.abs().sum(-1) > 0)
    torch.testing.assert_close(fused.f_n, split.f_n, rtol=1e-6, atol=1e-12)
    torch.testing.assert_close(fused.f_t, split.f_t, rtol=1e-6, atol=1e-12)
    torch.testing.assert_close(fused.wrench, split.wrench, rtol=1e-9, atol=1e-12)


def test_fused_graph_and_host_pipeline():
    E, S = 64, 2
    _, cam, bg, lut, pts = synthetic.sensor_setup((320, 240), (20, 25))
    sdf = synthetic.peg_grid((32, 32, 64))
    depth = synthetic.depth_batch(cam, bg, E * S, config_id=82, pool=16).reshape(E, S, 240, 320)
    obj, sen = synthetic.peg_states(E, S, config_id=82)
    arr = SensorArray(lut, sdf, pts, PenaltyParams(), E, S)
    d = torch.from_numpy(np.ascontiguousarray(depth)).cuda()
    o = torch.from_numpy(obj).cuda()
    s = torch.from_numpy(np.ascontiguousarray(sen)).cuda()
    arr.launch(d, o, s)
    torch.cuda.synchronize()
    ref = [x.clone() for x in (arr.rgb_u8, arr.f_n, arr.f_t, arr.wrench)]
    arr.capture(d, o, s)
    arr.replay()
    torch.cuda.synchronize()
    for a, b in zip(ref, (arr.rgb_u8, arr.f_n, arr.f_t, arr.wrench)):
        assert torch.equal(a, b)
    host = arr.host_buffers()
    host["depth"].copy_(d.cpu())
    host["obj"].copy_(o.cpu())
    host["sen"].copy_(s.cpu())
    arr.run_host(host, d, o, s, chunks=5)
    torch.cuda.synchronize()
    assert torch.equal(host["rgb"], ref[0].cpu())
    assert torch.equal(host["f_n"], ref[1].cpu())
