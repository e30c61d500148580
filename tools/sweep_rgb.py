"""Time K1 (depth -> RGB) alone over launch-shape knobs; prints GB/s of
algorithmic traffic (4 B in + 3 B out per pixel) for each setting.

    python tools/sweep_rgb.py [--frames 8192] [--size 320x240] [--deg 2]
"""
import argparse
import itertools
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2408_06506_b200 import render, synthetic  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--frames", type=int, default=8192)
    ap.add_argument("--size", default="320x240")
    ap.add_argument("--deg", type=int, default=2)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--groups", default="")
    ap.add_argument("--stages", default="2,3,4")
    ap.add_argument("--ctas", default="1,2")
    ap.add_argument("--f32", action="store_true")
    ap.add_argument("--rpt", default="4,8")
    a = ap.parse_args()
    W, H = (int(v) for v in a.size.split("x"))
    _, cam, bg, _, _ = synthetic.sensor_setup((W, H))
    lut = render.synthetic_lut((W, H), degree=a.deg, gradient_scale=synthetic.lut_scale((W, H)))
    pool = torch.from_numpy(synthetic.depth_batch(cam, bg, 32)).cuda()
    depth = pool[torch.arange(a.frames, device="cuda") % 32].contiguous()
    u8 = torch.empty((a.frames, H, W, 3), dtype=torch.uint8, device="cuda")
    f32 = torch.empty((a.frames, H, W, 3), dtype=torch.float32, device="cuda") if a.f32 else None
    bytes_ = a.frames * H * W * (4 + 3 + (12 if a.f32 else 0))
    QW = W // 4
    groups = [int(g) for g in a.groups.split(",")] if a.groups else sorted({g for g in (1, 2, 3, 4, 5, 6) if QW * g <= 384})
    results = []
    for rpt, g, st, c in itertools.product([int(v) for v in a.rpt.split(",")], groups,
                                           [int(v) for v in a.stages.split(",")], [int(v) for v in a.ctas.split(",")]):
        os.environ["TACSL_RGB_RPT"] = str(rpt)
        os.environ["TACSL_RGB_GROUPS"] = str(g)
        os.environ["TACSL_RGB_STAGES"] = str(st)
        os.environ["TACSL_RGB_CTAS_PER_SM"] = str(c)
        try:
            for _ in range(3):
                render.depth_to_rgb_device(depth, lut, out_u8=u8, out_f32=f32)
            torch.cuda.synchronize()
        except Exception as e:  # noqa: BLE001
            print(json.dumps({"rpt": rpt, "groups": g, "stages": st, "ctas": c, "error": str(e)}))
            continue
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        for _ in range(a.iters):
            render.depth_to_rgb_device(depth, lut, out_u8=u8, out_f32=f32)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.iters
        r = {"rpt": rpt, "groups": g, "stages": st, "ctas": c, "ms": round(ms, 4), "GBps": round(bytes_ / ms / 1e6, 1)}
        results.append(r)
        print(json.dumps(r), flush=True)
    best = max(results, key=lambda r: r["GBps"])
    print("BEST", json.dumps(best))


if __name__ == "__main__":
    main()
