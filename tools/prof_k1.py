"""One K1 launch (uint8 RGB) on N frames of 240x320 (for ncu)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402
from paper_2408_06506_b200 import synthetic  # noqa: E402
from paper_2408_06506_b200.render import depth_to_rgb_device  # noqa: E402
N = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
_, cam, bg, lut, _ = synthetic.sensor_setup((320, 240))
d = torch.from_numpy(synthetic.depth_batch(cam, bg, N, pool=64)).cuda()
out = torch.empty((N, 240, 320, 3), dtype=torch.uint8, device="cuda")
for _ in range(2):
    depth_to_rgb_device(d, lut, out_u8=out)
torch.cuda.synchronize()
