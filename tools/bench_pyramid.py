"""Time the smoothing / pyramid kernels (K5) on 480x640 depth maps."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2408_06506_b200 import smoothing, synthetic  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
_, cam, bg, lut, _ = synthetic.sensor_setup((640, 480))
d = torch.from_numpy(synthetic.depth_batch(cam, bg, 32)).cuda()
d = d[torch.arange(N, device="cuda") % 32].contiguous()
px = N * 480 * 640
cases = (("gaussian sigma=1", lambda: smoothing.gaussian_blur_device(d, 1.0), 8 * px),
         ("pyr_down", lambda: smoothing.pyr_down_device(d), 5 * px),
         ("rgb pyramid 3 levels + sigma=1", lambda: smoothing.rgb_pyramid_device(d, lut, 3, 1.0), None))
if len(sys.argv) > 2 and sys.argv[2] == "filters":
    cases = cases[:2]
for name, fn, nbytes in cases:
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(5):
        fn()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    extra = f", {nbytes / ms / 1e6:.0f} GB/s" if nbytes else ""
    print(f"{name}: {ms:.3f} ms for {N} frames 480x640{extra}")
