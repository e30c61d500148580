"""Time K7 (the one-pass smoothing + 3-level RGB pyramid) against the
unfused chain on N 480x640 depth maps (config 5: N = 8192).

    python tools/bench_pyramid_fused.py [N]
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2408_06506_b200 import smoothing, synthetic  # noqa: E402
from paper_2408_06506_b200.render import device_lut  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 and not sys.argv[1].startswith("-") else 8192
H, W = 480, 640
_, cam, bg, lut, _ = synthetic.sensor_setup((W, H))
d = torch.from_numpy(synthetic.depth_batch(cam, bg, 64, config_id=5)).cuda()
d = d[torch.arange(N, device="cuda") % 64].contiguous()
px = N * H * W
alg = px * (4 + 3 + 3 / 4 + 3 / 16)  # depth read + every level's RGB written
luts = [device_lut(smoothing.level_lut(lut, lvl)) for lvl in range(3)]
outs = [torch.empty((N, H >> lvl, W >> lvl, 3), dtype=torch.uint8, device="cuda") for lvl in range(3)]


def fused():
    smoothing.rgb_pyramid_fused_device(d, lut, 3, 1.0, outs=outs, luts=luts)


def chain():
    smoothing.rgb_pyramid_device(d, lut, 3, 1.0)


peak = 6555.5
for name, fn in (("K7 fused", fused), ("unfused chain", chain)):
    fn()
    torch.cuda.synchronize()
    per = []
    for _ in range(3):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        for _ in range(5):
            fn()
        b.record()
        torch.cuda.synchronize()
        per.append(a.elapsed_time(b) / 5)
    ms = sorted(per)[1]
    print(f"{name}: {ms:.3f} ms for {N} frames {W}x{H} (3 levels, sigma=1): "
          f"{alg / ms / 1e6:.0f} GB/s algorithmic = {alg / ms / 1e6 / peak:.3f} of {peak} GB/s "
          "")
