"""The REFERENCE package's per-call latency for the calls tools/dropin_latency.py
times (this container only: imports gelsim read-only from /root/reference)."""
import os, sys, time
import numpy as np
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__)))); sys.path.insert(0, "/root/reference/pkg/src")
from paper_2408_06506_b200 import synthetic
import gelsim.render as gr, gelsim.tactile as gt, gelsim.geometry as gg
from gelsim.sensors import TactileSensorSpec
E = 16
spec = TactileSensorSpec(image_size=(80, 60)); cam = gr.camera_for_sensor(spec); bg = gr.reference_depth(cam, spec)
lut = gr.synthetic_lut((80, 60))
p = synthetic.peg_grid((32, 32, 64))
peg = gg.SdfGrid(origin=p.origin, spacing=p.spacing, dims=p.dims, values=p.values, gradients=p.gradients)
pts = gt.sample_tactile_points(spec, 10, 14)
obj, sen = synthetic.peg_states(E, 1, config_id=2); sen = sen[:, 0]
ff = lambda: gt.compute_force_field(pts, peg, obj[:, 0:3], obj[:, 3:7], obj[:, 7:10], obj[:, 10:13], sen[:, 0:3], sen[:, 3:7], sen[:, 7:10], sen[:, 10:13], gt.PenaltyParams())
rd = lambda: gr.render_depth(cam, peg, obj[:, 0:3] * 0 + np.array([0, 0, 0.0075]), obj[:, 3:7], bg)
depth = rd()
rgb = lambda: gr.depth_to_rgb(depth, lut)
for name, fn in (("compute_force_field", ff), ("render_depth", rd), ("depth_to_rgb", rgb)):
    fn(); t0 = time.perf_counter()
    for _ in range(3): fn()
    print(f"reference {name}: {(time.perf_counter() - t0) / 3 * 1e3:.1f} ms per call")
