"""Where the time of the numpy drop-in path goes (1024 frames of 240x320)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2408_06506_b200 import _device, render, synthetic  # noqa: E402
from paper_2408_06506_b200.render import DepthImage  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
_, cam, bg, lut, pts = synthetic.sensor_setup((320, 240))
pool = synthetic.depth_batch(cam, bg, 64, config_id=3)
d64 = pool[np.arange(N) % 64].astype(np.float64)


def tm(name, fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        r = fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    print(f"{name}: {dt * 1e3:.1f} ms")
    return r


tm("to_pinned (host copy into page-locked)", lambda: _device.to_pinned(d64, torch.float64))
tm("pinned_empty out (1.9 GB)", lambda: _device.pinned_empty((N, 240, 320, 3), torch.float64))
x = torch.from_numpy(d64)
tm("torch copy_ numpy->pinned", lambda: _device.pinned_empty(x.shape, torch.float64).copy_(x))
tm("np.copyto into pinned", lambda: np.copyto(_device.pinned_empty(x.shape, torch.float64).numpy(), d64))
tm("depth_to_rgb numpy f64 -> f64", lambda: render.depth_to_rgb(DepthImage(values=d64, background=bg), lut))
tm("depth_to_rgb numpy f64 -> u8", lambda: render.depth_to_rgb(d64, lut, out_dtype=np.uint8))
dv = torch.from_numpy(d64).cuda()
tm("depth_to_rgb device f64 -> f32 (device only)", lambda: render.depth_to_rgb(dv, lut))
print("threads", torch.get_num_threads())
