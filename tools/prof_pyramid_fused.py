"""One K7 launch on N 480x640 maps (for ncu captures)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2408_06506_b200 import smoothing, synthetic  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
_, cam, bg, lut, _ = synthetic.sensor_setup((640, 480))
d = torch.from_numpy(synthetic.depth_batch(cam, bg, 64, config_id=5)).cuda()
d = d[torch.arange(N, device="cuda") % 64].contiguous()
for _ in range(2):
    smoothing.rgb_pyramid_fused_device(d, lut, 3, 1.0)
torch.cuda.synchronize()
