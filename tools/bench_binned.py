"""Time the binned-LUT kernel (K6) against K1 on config-3-sized batches;
each K6 shape is timed through its dispatch choice and both forced paths
(TACSL_BINNED_BAND = band pipeline, TACSL_BINNED_SIMPLE = per-quad kernel)."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2408_06506_b200 import synthetic  # noqa: E402
from paper_2408_06506_b200.binned import depth_to_rgb_binned_device, device_binned_lut, vignetted_lut  # noqa: E402
from paper_2408_06506_b200.render import depth_to_rgb_device  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
DEG = int(sys.argv[2]) if len(sys.argv) > 2 else 2  # LUT degree
_, cam, bg, lut, _ = synthetic.sensor_setup((320, 240), lut_degree=DEG)
pool = torch.from_numpy(synthetic.depth_batch(cam, bg, 64)).cuda()
d = pool[torch.arange(N, device="cuda") % 64].contiguous()
u8 = torch.empty(d.shape + (3,), dtype=torch.uint8, device="cuda")
nbytes = N * 240 * 320 * 7


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


b1 = device_binned_lut(vignetted_lut(lut, (6, 8)), d.device)
b2 = device_binned_lut(vignetted_lut(lut, (24, 32)), d.device)

def run(name, fn):
    try:
        ms = timeit(fn)
    except ValueError as e:  # e.g. a table too large for the forced per-quad kernel
        print(f"{name} (degree {DEG}): n/a ({e})")
        return
    print(f"{name} (degree {DEG}): {ms:.3f} ms for {N} frames 240x320, {nbytes / ms / 1e6:.0f} GB/s")


run("K1 global LUT", lambda: depth_to_rgb_device(d, lut, out_u8=u8))
for tag, b in (("6x8", b1), ("24x32", b2)):
    for mode in ("", "TACSL_BINNED_BAND", "TACSL_BINNED_SIMPLE") + (("TACSL_BINNED_L1",) if DEG > 2 else ()):
        if mode:
            os.environ[mode] = "1"
        run(f"K6 binned {tag} {mode or 'dispatch'}", lambda: depth_to_rgb_binned_device(d, b, out_u8=u8))
        os.environ.pop(mode, None)
