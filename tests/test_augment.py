"""Augmentation: the numpy Philox restatement and the
augment oracle pinned against numpy / the reference (CPU), and the device
kernels bit-exact against the reference's golden vectors (GPU)."""
import numpy as np
import pytest

from oracle import augment_oracle as A
from oracle.philox import Stream

GOLDEN = __import__("pathlib").Path(__file__).resolve().parent / "golden"

CFGS = {
    "full": dict(shift_px=2.5, zoom=(1.05, 1.2), brightness=0.1, contrast=(0.8, 1.2), saturation=(0.7, 1.3),
                 hue=0.05, channel_permutation=True, step_brightness=0.02, step_contrast=(0.95, 1.05),
                 step_saturation=(0.9, 1.1), step_hue=0.01, seed=3),
    "color": dict(shift_px=0.0, zoom=(1.0, 1.0), brightness=0.2, contrast=(0.5, 1.5), saturation=(0.2, 1.8),
                  hue=0.5, channel_permutation=False, step_brightness=0.0, step_contrast=(1.0, 1.0),
                  step_saturation=(1.0, 1.0), step_hue=0.0, seed=11),
    "spatial": dict(shift_px=6.0, zoom=(0.7, 1.4), brightness=0.0, contrast=(1.0, 1.0), saturation=(1.0, 1.0),
                    hue=0.0, channel_permutation=True, step_brightness=0.0, step_contrast=(1.0, 1.0),
                    step_saturation=(1.0, 1.0), step_hue=0.0, seed=0),
    "identity": dict(shift_px=0.0, zoom=(1.0, 1.0), brightness=0.0, contrast=(1.0, 1.0), saturation=(1.0, 1.0),
                     hue=0.0, channel_permutation=False, step_brightness=0.0, step_contrast=(1.0, 1.0),
                     step_saturation=(1.0, 1.0), step_hue=0.0, seed=5),
}
SEEDS = [(0, 0), (17, 3), (2 ** 33 + 12345, 123), (987654321, 7)]


@pytest.mark.parametrize("key", [(0, 5, 0), (7, 123456789012, 1, 55), (2 ** 40 + 3,), (0, 0, 0), (1, 2, 3, 4, 5, 6)])
def test_philox_restatement_matches_numpy(key):
    g = np.random.Generator(np.random.Philox(np.random.SeedSequence(key)))
    s = Stream(key)
    assert [g.uniform(-0.3, 0.3) for _ in range(7)] == [s.uniform(-0.3, 0.3) for _ in range(7)]
    assert [int(v) for v in g.permutation(3)] == s.permutation(3)
    assert [g.uniform(0.9, 1.1) for _ in range(5)] == [s.uniform(0.9, 1.1) for _ in range(5)]


@pytest.mark.parametrize("name", sorted(CFGS))
@pytest.mark.parametrize("key", ["60x80", "30x40"])
def test_augment_oracle_matches_reference(name, key):
    z = np.load(GOLDEN / "augment.npz")
    imgs = z["img_" + key]
    got = np.stack([A.augment(imgs[i], CFGS[name], ep, st) for i, (ep, st) in enumerate(SEEDS)])
    assert np.array_equal(got, z[f"aug_{name}_{key}"])


def test_augment_config_validation():
    from paper_2408_06506_b200.augment import AugmentConfig
    with pytest.raises(ValueError):
        AugmentConfig(zoom=(0.0, 1.0))
    with pytest.raises(ValueError):
        AugmentConfig(brightness=0.1, step_brightness=0.2)


def test_host_episode_transform_matches_oracle():
    from paper_2408_06506_b200.augment import AugmentConfig, sample_episode_transform
    cfg = AugmentConfig(**CFGS["full"])
    for ep, _ in SEEDS:
        tr = sample_episode_transform(cfg, ep)
        o = A.episode_params(3, 2.5, (1.05, 1.2), 0.1, (0.8, 1.2), (0.7, 1.3), 0.05, True, ep)
        assert (tr.shift, tr.zoom, tr.brightness, tr.contrast, tr.saturation, tr.hue, tr.permutation) == o


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CFGS))
@pytest.mark.parametrize("key", ["60x80", "30x40"])
def test_augment_device_bit_exact(name, key):
    import torch
    from paper_2408_06506_b200.augment import AugmentConfig, augment_device, augment_params_device
    z = np.load(GOLDEN / "augment.npz")
    cfg = AugmentConfig(**CFGS[name])
    imgs = torch.from_numpy(z["img_" + key]).cuda()
    seeds = torch.tensor([s for s, _ in SEEDS], dtype=torch.int64, device="cuda")
    steps = torch.tensor([t for _, t in SEEDS], dtype=torch.int64, device="cuda")
    out = augment_device(imgs, cfg, seeds, steps)
    assert np.array_equal(out.cpu().numpy(), z[f"aug_{name}_{key}"])
    # device parameters == the reference's Philox draws
    p = augment_params_device(cfg, seeds, steps).cpu().numpy()
    for i, (ep, st) in enumerate(SEEDS):
        shift, zm, b, c, s, h, perm = A.episode_params(cfg.seed, cfg.shift_px, cfg.zoom, cfg.brightness,
                                                       cfg.contrast, cfg.saturation, cfg.hue,
                                                       cfg.channel_permutation, ep)
        jit = A.step_params(cfg.seed, cfg.step_brightness, cfg.step_contrast, cfg.step_saturation,
                            cfg.step_hue, ep, st)
        assert tuple(p[i, :14]) == (shift[0], shift[1], zm, b, c, s, h, *map(float, perm), *jit)


@pytest.mark.gpu
@pytest.mark.parametrize("rep", ["diff", "concat"])
def test_augment_device_representation(rep):
    import torch
    from paper_2408_06506_b200.augment import AugmentConfig, augment_device
    z = np.load(GOLDEN / "augment.npz")
    cfg = AugmentConfig(**CFGS["full"])
    imgs = torch.from_numpy(z["img_60x80"]).cuda()
    seeds = torch.tensor([s for s, _ in SEEDS], dtype=torch.int64, device="cuda")
    steps = torch.tensor([t for _, t in SEEDS], dtype=torch.int64, device="cuda")
    nominal = np.array([0.35, 0.38, 0.45], dtype=np.float32)
    out = augment_device(imgs, cfg, seeds, steps, tactile_rep=rep, nominal=nominal).cpu().numpy()
    ref = z["aug_full_60x80"]
    if rep == "diff":
        assert np.array_equal(out, ref - nominal)
    else:
        assert np.array_equal(out, np.concatenate([ref, np.broadcast_to(nominal, ref.shape)], axis=-1))


@pytest.mark.gpu
def test_augment_single_image_dropin():
    from paper_2408_06506_b200.augment import AugmentConfig, augment
    z = np.load(GOLDEN / "augment.npz")
    cfg = AugmentConfig(**CFGS["full"])
    out = augment(z["img_60x80"][2], cfg, SEEDS[2][0], SEEDS[2][1])
    assert out.dtype == np.float32 and np.array_equal(out, z["aug_full_60x80"][2])
