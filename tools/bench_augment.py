"""Time K4 (augment apply, params precomputed) on 2048 frames of 240x320."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2408_06506_b200.augment import AugmentConfig, augment_device, augment_params_device  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
g = torch.Generator(device="cuda").manual_seed(0)
img = torch.rand((N, 240, 320, 3), generator=g, device="cuda") * 0.5 + 0.25
cfg = AugmentConfig(shift_px=2.0, zoom=(0.95, 1.1), brightness=0.05, contrast=(0.9, 1.1), saturation=(0.8, 1.2),
                    hue=0.02, channel_permutation=True, step_brightness=0.01, seed=1)
seeds = torch.arange(N, dtype=torch.int64, device="cuda") * 1000003
steps = torch.full((N,), 5, dtype=torch.int64, device="cuda")
params = augment_params_device(cfg, seeds, steps)
out = torch.empty_like(img)
nom = np.float32([0.35, 0.38, 0.45])
fn = lambda: augment_device(img, cfg, seeds, steps, tactile_rep="diff", nominal=nom, out=out, params=params)  # noqa: E731
fn()
torch.cuda.synchronize()
a, b = torch.cuda.Event(True), torch.cuda.Event(True)
a.record()
for _ in range(10):
    fn()
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 10
print(f"augment apply: {ms:.3f} ms for {N} frames 240x320, {N * 240 * 320 * 24 / ms / 1e6:.0f} GB/s")
