"""K2 time at config-4 shape with the standard peg presses (~27 % contact
taxels) and with every peg lifted 1.5 mm off the pad (no contact, same grid
region): the contact path's share of K2."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2408_06506_b200 import synthetic  # noqa: E402
from paper_2408_06506_b200.geometry import device_sdf  # noqa: E402
from paper_2408_06506_b200.tactile import PenaltyParams, device_taxels, force_field_device  # noqa: E402
from paper_2408_06506_b200.transforms import quat_rotate  # noqa: E402

N = 16384
_, cam, bg, lut, pts = synthetic.sensor_setup((320, 240), (80, 100))
obj, sen = synthetic.peg_states(N, 1, config_id=4)
sdf = device_sdf(synthetic.peg_grid((128, 128, 128)), torch.device("cuda", 0))
tax = device_taxels(pts, torch.device("cuda", 0))
f_n = torch.empty((N, 1, 80, 100, 3), dtype=torch.float32, device="cuda")
f_t = torch.empty_like(f_n)
w = torch.empty((N, 1, 6), dtype=torch.float64, device="cuda")
lift = obj.copy()
# move each object 1.5 mm along its sensor's +z (away from the pad)
lift[:, 0:3] += quat_rotate(sen[:, 0, 3:7], np.array([0.0, 0.0, 0.0015]))
for name, o_np in (("presses", obj), ("lifted 1.5 mm", lift)):
    o = torch.from_numpy(o_np).cuda()
    s = torch.from_numpy(np.ascontiguousarray(sen)).cuda()
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
    print(f"{name}: {a.elapsed_time(b) / 5:.3f} ms, contact taxels {contact:.1%}")
