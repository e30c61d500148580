"""Per-call latency of the numpy-level drop-ins (what a patched env calls per
finger per step): compute_force_field for 16 envs x 10x14 taxels,
depth_to_rgb for 16 images of 80x60, render_depth for 16 poses."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

import paper_2408_06506_b200 as tb  # noqa: E402
from paper_2408_06506_b200 import synthetic  # noqa: E402

E = 16
spec = tb.TactileSensorSpec(image_size=(80, 60))
cam = tb.camera_for_sensor(spec)
bg = tb.reference_depth(cam, spec)
lut = tb.synthetic_lut((80, 60))
peg = synthetic.peg_grid((32, 32, 64))
pts = tb.sample_tactile_points(spec, 10, 14)
obj, sen = synthetic.peg_states(E, 1, config_id=2)
sen = sen[:, 0]


def ff():
    return tb.compute_force_field(pts, peg, obj[:, 0:3], obj[:, 3:7], obj[:, 7:10], obj[:, 10:13], sen[:, 0:3],
                                  sen[:, 3:7], sen[:, 7:10], sen[:, 10:13], tb.PenaltyParams())


def rd():
    return tb.render_depth(cam, peg, obj[:, 0:3] * 0 + np.array([0, 0, 0.0075]), obj[:, 3:7], bg)


depth = rd()


def rgb():
    return tb.depth_to_rgb(depth, lut)


for name, fn in (("compute_force_field", ff), ("render_depth", rd), ("depth_to_rgb", rgb)):
    fn()
    t0 = time.perf_counter()
    for _ in range(50):
        fn()
    print(f"{name}: {(time.perf_counter() - t0) / 50 * 1e3:.3f} ms per call ({E} envs, numpy in / numpy out)")
