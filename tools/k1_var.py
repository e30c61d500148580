"""K1 launch-time variance across allocations (config 3 shapes)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2408_06506_b200 import synthetic  # noqa: E402
from paper_2408_06506_b200.render import depth_to_rgb_device  # noqa: E402

_, cam, bg, lut, _ = synthetic.sensor_setup((320, 240))
pool = torch.from_numpy(synthetic.depth_batch(cam, bg, 64)).cuda()
keep = []
for trial in range(4):
    if trial == 2:
        keep.append(torch.empty(int(1.3e9), dtype=torch.uint8, device="cuda"))  # shift later allocations
    d = pool[torch.arange(8192, device="cuda") % 64].contiguous()
    u8 = torch.empty(d.shape + (3,), dtype=torch.uint8, device="cuda")
    depth_to_rgb_device(d, lut, out_u8=u8)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        depth_to_rgb_device(d, lut, out_u8=u8)
    per = []
    for _ in range(12):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        for _ in range(10):
            g.replay()
        b.record()
        torch.cuda.synchronize()
        per.append(a.elapsed_time(b) / 10)
    print(trial, hex(d.data_ptr()), hex(u8.data_ptr()), " ".join(f"{x:.3f}" for x in per), "median", np.median(per))
    keep += [d, u8]
