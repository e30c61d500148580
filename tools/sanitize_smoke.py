"""Small launches of every kernel, for compute-sanitizer memcheck."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2408_06506_b200 import SensorArray, smoothing, synthetic  # noqa: E402
from paper_2408_06506_b200.augment import AugmentConfig, augment_device  # noqa: E402
from paper_2408_06506_b200.depth import render_depth  # noqa: E402
from paper_2408_06506_b200.geometry import query_sdf  # noqa: E402
from paper_2408_06506_b200.pipeline import TactileObservations  # noqa: E402
from paper_2408_06506_b200.render import depth_to_rgb, tactile_image_obs_device, to_uint8  # noqa: E402
from paper_2408_06506_b200.tactile import PenaltyParams, net_wrench, penalty_forces  # noqa: E402

for size in ((320, 240), (80, 60), (37, 29)):
    _, cam, bg, lut, pts = synthetic.sensor_setup(size, (20, 25))
    sdf = synthetic.peg_grid((16, 16, 32))
    d = synthetic.depth_batch(cam, bg, 6, config_id=5).reshape(3, 2, size[1], size[0])
    obj, sen = synthetic.peg_states(3, 2, config_id=5)
    dd = torch.from_numpy(d).cuda()
    for rep in ("color", "diff", "concat"):
        tactile_image_obs_device(dd, lut, rep)
    depth_to_rgb(dd, lut, out_dtype=np.uint8)
    arr = SensorArray(lut, sdf, pts, PenaltyParams(), 3, 2, rgb_f32=True)
    arr.launch(dd, torch.from_numpy(obj).cuda(), torch.from_numpy(np.ascontiguousarray(sen)).cuda())
    obs = TactileObservations(lut, sdf, pts, PenaltyParams(), 3, 2, tactile_rep="concat",
                              augment=AugmentConfig(shift_px=3.0, zoom=(0.8, 1.2), hue=0.1, saturation=(0.5, 1.5),
                                                    channel_permutation=True))
    obs(dd, torch.from_numpy(obj).cuda(), torch.from_numpy(np.ascontiguousarray(sen)).cuda(),
        episode_seeds=np.arange(3), step_indices=np.arange(3))
    render_depth(cam, sdf, obj[:, 0:3], obj[:, 3:7], bg)
    smoothing.rgb_pyramid_device(dd, lut, levels=2, sigma=1.5)
    to_uint8(np.linspace(-1, 2, 1001, dtype=np.float32))
q = query_sdf(sdf, np.random.default_rng(0).uniform(-0.05, 0.05, (999, 3)))
penalty_forces(np.full(7, -1e-3), np.zeros(7), np.tile([0, 0, 1.0], (7, 1)), np.ones((7, 3)), PenaltyParams())
net_wrench(arr and type("F", (), {"f_n": arr.f_n[0], "f_t": arr.f_t[0]})(), pts) if False else None
torch.cuda.synchronize()
print("sanitize smoke ok")
