"""One launch of each secondary kernel at benchmark scale, for ncu:
K3 render_depth, K4 augment, K5 separable filter (240x320 and 480x640),
K1 obs epilogue, K6 binned LUT."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2408_06506_b200 import smoothing, synthetic  # noqa: E402
from paper_2408_06506_b200.augment import AugmentConfig, augment_device  # noqa: E402
from paper_2408_06506_b200.depth import RayTable, env_params, render_depth_device  # noqa: E402
from paper_2408_06506_b200.geometry import device_sdf  # noqa: E402
from paper_2408_06506_b200.render import tactile_image_obs_device  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
_, cam, bg, lut, _ = synthetic.sensor_setup((320, 240))
sdf = synthetic.peg_grid((32, 32, 64))
dev = torch.device("cuda")
obj, _ = synthetic.peg_states(N, 1, config_id=3, random_sensor_pose=False)
params = torch.from_numpy(env_params(sdf, obj[:, 0:3], obj[:, 3:7])).to(dev)
depth = torch.empty((N, 240, 320), dtype=torch.float32, device=dev)
table = RayTable(cam, bg, dev)
render_depth_device(table, device_sdf(sdf, dev), params, out_f32=depth)
rgb = tactile_image_obs_device(depth, lut, "color")
cfg = AugmentConfig(shift_px=2.0, zoom=(0.95, 1.1), brightness=0.05, contrast=(0.9, 1.1), saturation=(0.8, 1.2),
                    hue=0.02, channel_permutation=True, step_brightness=0.01, seed=1)
seeds = torch.arange(N, dtype=torch.int64, device=dev) * 1000003
steps = torch.full((N,), 5, dtype=torch.int64, device=dev)
augment_device(rgb, cfg, seeds, steps, tactile_rep="diff", nominal=np.float32(lut.coeffs[:, 0]))
smoothing.gaussian_blur_device(depth, 1.0)
smoothing.pyr_down_device(depth)
_, cam5, bg5, _, _ = synthetic.sensor_setup((640, 480))
d5 = torch.from_numpy(synthetic.depth_batch(cam5, bg5, 32)).to(dev)[torch.arange(N // 4, device=dev) % 32]
d5 = d5.contiguous()
smoothing.gaussian_blur_device(d5, 1.0)
smoothing.pyr_down_device(d5)
from paper_2408_06506_b200.binned import depth_to_rgb_binned_device, vignetted_lut  # noqa: E402
u8 = torch.empty(depth.shape + (3,), dtype=torch.uint8, device=dev)
depth_to_rgb_binned_device(depth, vignetted_lut(lut, (6, 8)), out_u8=u8)
torch.cuda.synchronize()
print("ok", N)
