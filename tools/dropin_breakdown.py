"""Where the time of the numpy drop-in path goes (N frames of 240x320,
steady state: every call's result dropped before the next)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2408_06506_b200 import _device, render, synthetic, tactile  # noqa: E402
from paper_2408_06506_b200.render import DepthImage  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
_, cam, bg, lut, pts = synthetic.sensor_setup((320, 240))
sdf = synthetic.peg_grid((32, 32, 64))
pool = synthetic.depth_batch(cam, bg, 64, config_id=3)
d64 = pool[np.arange(N) % 64].astype(np.float64)
obj, sen = synthetic.peg_states(N, 1, config_id=3)
senF = sen.reshape(N, 13)


def tm(name, fn, reps=6):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    print(f"{name}: median {np.median(ts) * 1e3:.1f} ms  min {min(ts) * 1e3:.1f} ms")


tm("host copy numpy -> cached page-locked (to_pinned)", lambda: _device.to_pinned(d64, torch.float64))
tm("np.empty + first touch of a 1.9 GB result", lambda: np.empty((N, 240, 320, 3)).fill(0.0))
tm("depth_to_rgb numpy f64 -> f64 numpy", lambda: render.depth_to_rgb(DepthImage(values=d64, background=bg), lut))
tm("depth_to_rgb numpy f64 -> u8 numpy", lambda: render.depth_to_rgb(d64, lut, out_dtype=np.uint8))
tm("compute_force_field numpy", lambda: tactile.compute_force_field(
    pts, sdf, obj[:, 0:3], obj[:, 3:7], obj[:, 7:10], obj[:, 10:13], senF[:, 0:3], senF[:, 3:7], senF[:, 7:10],
    senF[:, 10:13], tactile.PenaltyParams()))
dv = torch.from_numpy(d64).cuda()
tm("depth_to_rgb device f64 -> f32 tensor", lambda: render.depth_to_rgb(dv, lut))
print("torch threads", torch.get_num_threads())
