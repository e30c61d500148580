"""Observation packing of the 2-finger peg env:
envs/peg_tasks.py:434-477 tactile images in the color / diff / concat
representations and the packed [f_n.z, f_t.x, f_t.y] force-field
observation, against the CPU oracle."""
import numpy as np
import pytest
import torch

from conftest import sdf_tuple
from oracle import gelsim_oracle as O
from paper_2408_06506_b200 import synthetic
from paper_2408_06506_b200.pipeline import TactileObservations
from paper_2408_06506_b200.tactile import PenaltyParams

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("rep", ["color", "diff", "concat"])
@pytest.mark.parametrize("size", [(320, 240), (40, 30)])
def test_peg_env_observations(rep, size):
    E, S = 5, 2
    _, cam, bg, lut, pts = synthetic.sensor_setup(size, (14, 10))
    sdf = synthetic.peg_grid((32, 32, 64))
    depth = synthetic.depth_batch(cam, bg, E * S, config_id=61).reshape(E, S, size[1], size[0])
    obj, sen = synthetic.peg_states(E, S, config_id=61)
    obs = TactileObservations(lut, sdf, pts, PenaltyParams(), E, S, tactile_rep=rep)
    imgs, ff = obs(torch.from_numpy(depth).cuda(), torch.from_numpy(obj).cuda(),
                   torch.from_numpy(np.ascontiguousarray(sen)).cuda())
    torch.cuda.synchronize()
    # reference semantics (peg_tasks.py:445, 453-458)
    rgb = O.depth_to_rgb(depth, lut.coeffs, lut.degree).astype(np.float32)
    nominal = np.broadcast_to(lut.coeffs[:, 0].astype(np.float32), rgb.shape[2:])
    if rep == "diff":
        ref = rgb - nominal[None, None]
    elif rep == "concat":
        ref = np.concatenate([rgb, np.broadcast_to(nominal, rgb.shape)], axis=-1)
    else:
        ref = rgb
    got = imgs.cpu().numpy()
    assert got.shape == ref.shape
    np.testing.assert_allclose(got, ref, atol=2e-6)
    # packed force-field observation (peg_tasks.py:474-476)
    objE = np.repeat(obj, S, axis=0)
    senE = sen.reshape(E * S, 13)
    f_n, f_t, _ = O.compute_force_field(pts.points, *sdf_tuple(sdf), objE[:, 0:3], objE[:, 3:7], objE[:, 7:10],
                                        objE[:, 10:13], senE[:, 0:3], senE[:, 3:7], senE[:, 7:10], senE[:, 10:13])
    ref_ff = np.stack([f_n[..., 2], f_t[..., 0], f_t[..., 1]], axis=-1).astype(np.float32).reshape(ff.shape)
    np.testing.assert_allclose(ff.cpu().numpy(), ref_ff, rtol=1e-6, atol=1e-9)
