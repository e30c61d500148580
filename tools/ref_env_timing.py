"""Time the REFERENCE env's tactile observation methods on this machine's CPU
(this container only: imports gelsim read-only from /root/reference).

    python tools/ref_env_timing.py [num_envs]
"""
import os
import sys
import time

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.path.insert(0, "/root/reference/pkg/src")

from gelsim.envs.base import EnvConfig  # noqa: E402
from gelsim.envs.peg_tasks import PegEnvBatch  # noqa: E402
from gelsim.render.augment import AugmentConfig  # noqa: E402

E = int(sys.argv[1]) if len(sys.argv) > 1 else 16
aug = AugmentConfig(shift_px=1.5, zoom=(0.95, 1.08), brightness=0.05, contrast=(0.9, 1.1), saturation=(0.85, 1.15),
                    hue=0.02, channel_permutation=True, step_brightness=0.01, seed=7)
env = PegEnvBatch(EnvConfig(num_envs=E, seed=3, tactile_rep="diff", augment=aug,
                            obs_modalities=("tactile_img", "tactile_ff")))
env.reset()
env.step(np.zeros((E, 6)))
for name, fn in (("_tactile_images", env._tactile_images), ("_tactile_ff", env._tactile_ff)):
    fn()
    t0 = time.perf_counter()
    reps = 3
    for _ in range(reps):
        fn()
    dt = (time.perf_counter() - t0) / reps
    print(f"reference {name}: {dt * 1e3:.1f} ms for {E} envs x 2 fingers = {2 * E / dt:.0f} sensor-frames/s "
          f"(1 core, {tuple(env.cfg.tactile_image_size)} images, {tuple(env.cfg.tactile_ff_grid)} taxels)")
