"""Time the batched env observation methods (envs.tactile_images /
envs.tactile_ff, what patch() binds as PegEnvBatch._tactile_images /
_tactile_ff) for E envs x 2 fingers at the env's default sizes (80x60
images, 10x14 taxels), augmentation on, "diff" representation.  The env
state comes from synthetic peg presses on a stand-in object carrying the
attributes the methods read.

    python tools/bench_env.py [num_envs]
"""
import sys
import time
from pathlib import Path
from types import SimpleNamespace

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2408_06506_b200 import AugmentConfig, envs, synthetic  # noqa: E402
from paper_2408_06506_b200.envs import PEG  # noqa: E402
from paper_2408_06506_b200.render import synthetic_lut  # noqa: E402
from paper_2408_06506_b200.sensors import TactileSensorSpec, camera_for_sensor, reference_depth  # noqa: E402
from paper_2408_06506_b200.tactile import PenaltyParams, sample_tactile_points  # noqa: E402

E = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
W, H = 80, 60
spec = TactileSensorSpec(image_size=(W, H))
cam = camera_for_sensor(spec)
obj, sen = synthetic.peg_states(E, 2, config_id=9)
bodies = SimpleNamespace(pos=np.zeros((E, 4, 3)), quat=np.zeros((E, 4, 4)), linvel=np.zeros((E, 4, 3)),
                         angvel=np.zeros((E, 4, 3)))
bodies.pos[:, PEG], bodies.quat[:, PEG] = obj[:, 0:3], obj[:, 3:7]
bodies.linvel[:, PEG], bodies.angvel[:, PEG] = obj[:, 7:10], obj[:, 10:13]
aug = AugmentConfig(shift_px=1.5, zoom=(0.95, 1.08), brightness=0.05, contrast=(0.9, 1.1), saturation=(0.85, 1.15),
                    hue=0.02, channel_permutation=True, step_brightness=0.01, seed=7)
env = SimpleNamespace(
    cfg=SimpleNamespace(tactile_image_size=(W, H), tactile_ff_grid=(10, 14), tactile_rep="diff", augment=aug,
                        penalty=PenaltyParams()),
    num_envs=E, camera=cam, background=reference_depth(cam, spec), peg_sdf=synthetic.peg_grid((32, 32, 64)),
    lut=synthetic_lut((W, H)), env_seeds=np.arange(E, dtype=np.int64) + 3, episode=np.zeros(E, np.int64),
    step_count=np.full(E, 2, np.int64), bodies=bodies, ff_grid=sample_tactile_points(spec, 10, 14),
    _sensor_world_pose=lambda s: (sen[:, s, 0:3], sen[:, s, 3:7]),
    _sensor_world_velocity=lambda p: next((sen[:, s, 7:10], sen[:, s, 10:13]) for s in range(2)
                                          if np.array_equal(p, sen[:, s, 0:3])))
for name, fn in (("tactile_images", envs.tactile_images), ("tactile_ff", envs.tactile_ff),
                 ("tactile_images_device", lambda e: envs.tactile_images_device(e).sum().item()),
                 ("tactile_ff_device", lambda e: envs.tactile_ff_device(e).sum().item())):
    fn(env)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    reps = 10
    for _ in range(reps):
        fn(env)  # returns a host numpy array: each call ends synchronised
    dt = (time.perf_counter() - t0) / reps
    print(f"batched {name}: {dt * 1e3:.2f} ms for {E} envs x 2 fingers = {2 * E / dt:.0f} sensor-frames/s "
          f"(wall clock incl. host pose math{'' if 'device' in name else ' and the host copy of the result'})")
