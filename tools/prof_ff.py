"""One K2 launch at config-4 shape (80x100 taxels, 128^3 peg SDF) on N frames
(for ncu captures); a second argument "lifted" moves every peg 1.5 mm off
its pad (no contact)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2408_06506_b200 import synthetic  # noqa: E402
from paper_2408_06506_b200.geometry import device_sdf  # noqa: E402
from paper_2408_06506_b200.tactile import PenaltyParams, device_taxels, force_field_device  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
_, cam, bg, lut, pts = synthetic.sensor_setup((320, 240), (80, 100))
sdf = device_sdf(synthetic.peg_grid((128, 128, 128)), torch.device("cuda", 0))
obj, sen = synthetic.peg_states(N, 1, config_id=4)
if len(sys.argv) > 2 and sys.argv[2] == "lifted":
    from paper_2408_06506_b200.transforms import quat_rotate
    obj[:, 0:3] += quat_rotate(sen[:, 0, 3:7], np.array([0.0, 0.0, 0.0015]))
o = torch.from_numpy(obj).cuda()
s = torch.from_numpy(np.ascontiguousarray(sen)).cuda()
tax = device_taxels(pts, o.device)
f_n = torch.empty((N, 1, 80, 100, 3), dtype=torch.float32, device="cuda")
f_t = torch.empty_like(f_n)
w = torch.empty((N, 1, 6), dtype=torch.float64, device="cuda")
for _ in range(2):
    force_field_device(sdf, tax, 80, 100, o, s, PenaltyParams(), f_n, f_t, wrench=w, n_sensors=1)
torch.cuda.synchronize()
