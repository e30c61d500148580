"""Quick start on one B200: the reference-compatible drop-ins, then the
batched sensor step.

    python -m paper_2408_06506_b200.build     # once (nvcc, sm_100a)
    python examples/quickstart.py
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2408_06506_b200 as tb  # noqa: E402
from paper_2408_06506_b200 import synthetic  # noqa: E402

# ---- 1. drop-ins with the reference's signatures (numpy in, numpy out)
spec = tb.TactileSensorSpec(image_size=(320, 240))
cam = tb.camera_for_sensor(spec)
background = tb.reference_depth(cam, spec)
lut = tb.synthetic_lut(spec.image_size, gradient_scale=synthetic.lut_scale(spec.image_size))
peg = synthetic.peg_grid((32, 32, 64))
quat = np.array([np.cos(np.pi / 4), 0.0, np.sin(np.pi / 4), 0.0])  # peg lying across the pad
depth = tb.render_depth(cam, peg, np.array([0.0, 0.0, 0.0075]), quat, background)
rgb = tb.depth_to_rgb(depth, lut)                                    # (240, 320, 3) float64
taxels = tb.sample_tactile_points(spec, 20, 25)
fld = tb.compute_force_field(taxels, peg, np.array([0.0, 0.0, 0.0075]), quat, np.zeros(3), np.zeros(3),
                             np.zeros(3), np.array([1.0, 0, 0, 0]), np.zeros(3), np.zeros(3), tb.PenaltyParams())
force, torque = tb.net_wrench(fld, taxels)
print(f"drop-ins: rgb {rgb.shape} {rgb.dtype}, contact taxels {(np.linalg.norm(fld.f_n, axis=-1) > 0).mean():.2f}, "
      f"net force {force.round(4)} N")

# ---- 2. the batched step: all envs x fingers in one CUDA-graph replay
E, S = 4096, 2
depth_pool = torch.from_numpy(synthetic.depth_batch(cam, background, 64)).cuda()
d = depth_pool[torch.arange(E * S, device="cuda") % 64].reshape(E, S, 240, 320).contiguous()
obj, sen = synthetic.peg_states(E, S)
o, s = torch.from_numpy(obj).cuda(), torch.from_numpy(np.ascontiguousarray(sen)).cuda()
arr = tb.SensorArray(lut, peg, taxels, tb.PenaltyParams(), E, S)
arr.capture(d, o, s)
for _ in range(5):
    arr.replay()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(50):
    arr.replay()
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / 50
print(f"batched step: {E} envs x {S} fingers in {dt * 1e3:.3f} ms = {E * S / dt / 1e6:.2f} M sensor-frames/s "
      f"(rgb {tuple(arr.rgb_u8.shape)} uint8, forces {tuple(arr.f_n.shape)}, wrench {tuple(arr.wrench.shape)})")
