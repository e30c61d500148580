"""One K6 launch per bin shape (6x8, 24x32) at 2048 x 240x320, for
`ncu --set full -k regex:rgb_bulk_kernel` (both go through the band pipeline
at degree 2; at degree 3 only 24x32 does).

    python tools/prof_binned.py [frames] [degree]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2408_06506_b200 import synthetic  # noqa: E402
from paper_2408_06506_b200.binned import depth_to_rgb_binned_device, device_binned_lut, vignetted_lut  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
DEG = int(sys.argv[2]) if len(sys.argv) > 2 else 2
_, cam, bg, lut, _ = synthetic.sensor_setup((320, 240), lut_degree=DEG)
pool = torch.from_numpy(synthetic.depth_batch(cam, bg, 64)).cuda()
d = pool[torch.arange(N, device="cuda") % 64].contiguous()
u8 = torch.empty(d.shape + (3,), dtype=torch.uint8, device="cuda")
for bins in ((6, 8), (24, 32)):
    b = device_binned_lut(vignetted_lut(lut, bins), d.device)
    depth_to_rgb_binned_device(d, b, out_u8=u8)
torch.cuda.synchronize()
print("ok")
