"""PegEnvBatch._tactile_images with augmentation (envs/peg_tasks.py:434-458):
rgb.astype(float32) -> augment(env's episode seed, step) -> representation,
for all envs x sensors in two launches, bit-exact vs the oracle chain."""
import numpy as np
import pytest
import torch

from oracle import augment_oracle as A
from oracle import gelsim_oracle as O
from paper_2408_06506_b200 import synthetic
from paper_2408_06506_b200.augment import AugmentConfig
from paper_2408_06506_b200.pipeline import TactileObservations
from paper_2408_06506_b200.render import tactile_image_obs_device
from paper_2408_06506_b200.tactile import PenaltyParams

pytestmark = pytest.mark.gpu

CFG = dict(shift_px=1.5, zoom=(0.95, 1.1), brightness=0.05, contrast=(0.9, 1.1), saturation=(0.8, 1.2), hue=0.02,
           channel_permutation=True, step_brightness=0.01, step_contrast=(0.98, 1.02),
           step_saturation=(0.95, 1.05), step_hue=0.005, seed=42)


@pytest.mark.parametrize("rep", ["color", "diff", "concat"])
def test_augmented_observations(rep):
    E, S, size = 4, 2, (40, 30)
    _, cam, bg, lut, pts = synthetic.sensor_setup(size, (14, 10))
    sdf = synthetic.peg_grid((32, 32, 64))
    depth = synthetic.depth_batch(cam, bg, E * S, config_id=62).reshape(E, S, size[1], size[0])
    obj, sen = synthetic.peg_states(E, S, config_id=62)
    env_seeds = np.array([11, 22, 33, 44])
    episode = np.array([0, 3, 1, 7])
    ep_seeds = (env_seeds * 1000003 + episode).astype(np.int64)
    steps = np.array([0, 5, 17, 2], dtype=np.int64)
    obs = TactileObservations(lut, sdf, pts, PenaltyParams(), E, S, tactile_rep=rep,
                              augment=AugmentConfig(**CFG))
    d = torch.from_numpy(depth).cuda()
    imgs, _ = obs(d, torch.from_numpy(obj).cuda(), torch.from_numpy(np.ascontiguousarray(sen)).cuda(),
                  episode_seeds=ep_seeds, step_indices=steps)
    torch.cuda.synchronize()
    # the reference chain on the GPU's own float32 RGB (K1 is +-1e-7 from float64, checked elsewhere)
    rgb = tactile_image_obs_device(d, lut, "color").cpu().numpy()
    nominal = lut.coeffs[:, 0].astype(np.float32)
    ref = np.empty_like(rgb)
    for e in range(E):
        for s in range(S):
            ref[e, s] = A.augment(rgb[e, s], CFG, int(ep_seeds[e]), int(steps[e]))
    if rep == "diff":
        ref = ref - nominal
    elif rep == "concat":
        ref = np.concatenate([ref, np.broadcast_to(nominal, ref.shape)], axis=-1)
    assert np.array_equal(imgs.cpu().numpy(), ref)
    # and the float64 reference RGB gives the same within the fp32 tolerance
    rgb64 = O.depth_to_rgb(depth, lut.coeffs, lut.degree).astype(np.float32)
    np.testing.assert_allclose(rgb, rgb64, atol=2e-6)
