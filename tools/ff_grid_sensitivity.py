"""K2 time at config-4 shape (16384 frames x 80x100 taxels) against SDF grids
of different sizes: how much of K2 is the corner gathers' locality."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2408_06506_b200 import synthetic  # noqa: E402
from paper_2408_06506_b200.geometry import device_sdf  # noqa: E402
from paper_2408_06506_b200.tactile import PenaltyParams, device_taxels, force_field_device  # noqa: E402

N = 16384
_, cam, bg, lut, pts = synthetic.sensor_setup((320, 240), (80, 100))
obj, sen = synthetic.peg_states(N, 1, config_id=4)
o = torch.from_numpy(obj).cuda()
s = torch.from_numpy(np.ascontiguousarray(sen)).cuda()
tax = device_taxels(pts, o.device)
f_n = torch.empty((N, 1, 80, 100, 3), dtype=torch.float32, device="cuda")
f_t = torch.empty_like(f_n)
w = torch.empty((N, 1, 6), dtype=torch.float64, device="cuda")
for dims in ((32, 32, 64), (64, 64, 64), (128, 128, 128), (256, 256, 256)):
    sdf = device_sdf(synthetic.peg_grid(dims), o.device)
    for _ in range(2):
        force_field_device(sdf, tax, 80, 100, o, s, PenaltyParams(), f_n, f_t, wrench=w, n_sensors=1)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(5):
        force_field_device(sdf, tax, 80, 100, o, s, PenaltyParams(), f_n, f_t, wrench=w, n_sensors=1)
    b.record()
    torch.cuda.synchronize()
    contact = float((f_n.abs().sum(-1) > 0).float().mean())
    print(f"grid {dims}: {a.elapsed_time(b) / 5:.3f} ms, contact taxels {contact:.1%}")
    del sdf
