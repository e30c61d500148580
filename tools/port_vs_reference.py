"""Single-core speed of the oracle port (the CPU baseline bench.py times)
against the REFERENCE package itself on the same config-3 frames (this
container only: imports gelsim read-only from /root/reference)."""
import os, sys, time
import numpy as np
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
os.environ["OMP_NUM_THREADS"] = "1"; os.environ["OPENBLAS_NUM_THREADS"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__)))); sys.path.insert(0, "/root/reference/pkg/src")
from oracle import gelsim_oracle as O
from paper_2408_06506_b200 import synthetic
import gelsim.render as gr, gelsim.tactile as gt
wl = synthetic.CONFIGS[3]
_, cam, bg, lut, pts = synthetic.sensor_setup(wl.image_size, wl.ff_grid)
sdf = synthetic.peg_grid(wl.sdf_dims)
depth = synthetic.depth_batch(cam, bg, 8, config_id=3)
obj, sen = synthetic.peg_states(4, 2, config_id=3)
objE = np.repeat(obj, 2, axis=0); senE = sen.reshape(8, 13)
rlut = gr.PolyLut(degree=lut.degree, coeffs=lut.coeffs, image_size=lut.image_size)
from gelsim.geometry import SdfGrid as RG
rsdf = RG(origin=sdf.origin, spacing=sdf.spacing, dims=sdf.dims, values=sdf.values, gradients=sdf.gradients)
rpts = gt.TactilePointGrid(points=pts.points, rest_normals=pts.rest_normals, spacing=pts.spacing) if hasattr(gt, 'TactilePointGrid') else pts
def ref():
    rgb = gr.to_uint8(gr.depth_to_rgb(gr.DepthImage(values=depth.astype(np.float64), background=bg), rlut))
    fld = gt.compute_force_field(rpts, rsdf, objE[:, 0:3], objE[:, 3:7], objE[:, 7:10], objE[:, 10:13], senE[:, 0:3], senE[:, 3:7], senE[:, 7:10], senE[:, 10:13], gt.PenaltyParams())
    return gt.net_wrench(fld, rpts)
def port():
    rgb = O.to_uint8(O.depth_to_rgb(depth, lut.coeffs, lut.degree))
    f_n, f_t, _ = O.compute_force_field(pts.points, sdf.origin, sdf.spacing, sdf.dims, sdf.values, sdf.gradients, objE[:, 0:3], objE[:, 3:7], objE[:, 7:10], objE[:, 10:13], senE[:, 0:3], senE[:, 3:7], senE[:, 7:10], senE[:, 10:13])
    return O.net_wrench(f_n, f_t, pts.points)
for name, fn in (("reference", ref), ("port", port)):
    fn(); t0 = time.perf_counter()
    for _ in range(3): fn()
    dt = (time.perf_counter() - t0) / 3
    print(f"{name}: {8 / dt:.1f} sensor-frames/s on one core (config 3 frames, 8 per call)")
