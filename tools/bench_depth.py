"""Time K3 (render_depth sphere tracer) on the peg workload.

    python tools/bench_depth.py [--envs 4096] [--sensors 2] [--size 320x240]
"""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2408_06506_b200 import synthetic  # noqa: E402
from paper_2408_06506_b200.depth import RayTable, env_params, render_depth_device  # noqa: E402
from paper_2408_06506_b200.geometry import device_sdf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--envs", type=int, default=4096)
    ap.add_argument("--sensors", type=int, default=2)
    ap.add_argument("--size", default="320x240")
    ap.add_argument("--iters", type=int, default=5)
    a = ap.parse_args()
    W, H = (int(v) for v in a.size.split("x"))
    _, cam, bg, _, _ = synthetic.sensor_setup((W, H))
    sdf = synthetic.peg_grid((32, 32, 64))
    dev = torch.device("cuda")
    dsdf = device_sdf(sdf, dev)
    table = RayTable(cam, bg, dev)
    obj, sen = synthetic.peg_states(a.envs * a.sensors, 1, config_id=3, random_sensor_pose=False)
    params = torch.from_numpy(env_params(sdf, obj[:, 0:3], obj[:, 3:7])).to(dev)
    out = torch.empty((a.envs * a.sensors, H, W), dtype=torch.float32, device=dev)
    render_depth_device(table, dsdf, params, out_f32=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(a.iters):
        render_depth_device(table, dsdf, params, out_f32=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.iters
    frames = a.envs * a.sensors
    hit = (out < torch.from_numpy(bg.astype(np.float32)).to(dev) - 1e-6).float().mean().item()
    print(json.dumps({"kernel": "render_depth", "frames": frames, "image": [H, W], "ms": ms,
                      "frames_per_s": frames / ms * 1e3, "rays_per_s": frames * H * W / ms * 1e3,
                      "indented_pixel_frac": hit}))


if __name__ == "__main__":
    main()
