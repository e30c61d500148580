"""Tactile-image augmentation: drop-in for ``gelsim.render.augment``.

``augment(image, cfg, episode_seed, step_index)`` (render/augment.py:156-173)
and the batched ``augment_device`` run K4 (csrc/augment.cu): the per-image
parameters come from the reference's tuple-keyed Philox streams restated on
the device, the image ops are float32 in numpy's order -- results are
bit-identical to the reference.  ``AugmentConfig`` and
``sample_episode_transform`` mirror the reference's set-up API
(augment.py:15-75).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _device, _lib


@dataclass
class AugmentConfig:
    """Per-episode ranges with optional reduced per-step colour ranges
    (render/augment.py:15-48)."""

    shift_px: float = 0.0
    zoom: tuple = (1.0, 1.0)
    brightness: float = 0.0
    contrast: tuple = (1.0, 1.0)
    saturation: tuple = (1.0, 1.0)
    hue: float = 0.0
    channel_permutation: bool = False
    step_brightness: float = 0.0
    step_contrast: tuple = (1.0, 1.0)
    step_saturation: tuple = (1.0, 1.0)
    step_hue: float = 0.0
    seed: int = 0

    def __post_init__(self):
        if self.zoom[0] <= 0 or self.zoom[1] <= 0:
            raise ValueError("zoom must be positive")

        def width(rng):
            return max(abs(rng[0] - 1.0), abs(rng[1] - 1.0))

        if self.step_brightness > self.brightness + 1e-12:
            raise ValueError("per-step brightness exceeds episode range")
        if width(self.step_contrast) > width(self.contrast) + 1e-12:
            raise ValueError("per-step contrast exceeds episode range")
        if width(self.step_saturation) > width(self.saturation) + 1e-12:
            raise ValueError("per-step saturation exceeds episode range")
        if self.step_hue > self.hue + 1e-12:
            raise ValueError("per-step hue exceeds episode range")


@dataclass
class EpisodeTransform:
    shift: tuple
    zoom: float
    brightness: float
    contrast: float
    saturation: float
    hue: float
    permutation: tuple


def _stream(*key):
    return np.random.Generator(np.random.Philox(np.random.SeedSequence(key)))


def sample_episode_transform(cfg, episode_seed: int) -> EpisodeTransform:
    """Host-side episode transform (augment.py:65-75), for inspection; the
    kernels derive the same numbers on the device."""
    rng = _stream(cfg.seed, int(episode_seed), 0)
    shift = tuple(rng.uniform(-cfg.shift_px, cfg.shift_px, size=2))
    zoom = float(rng.uniform(cfg.zoom[0], cfg.zoom[1]))
    brightness = float(rng.uniform(-cfg.brightness, cfg.brightness))
    contrast = float(rng.uniform(cfg.contrast[0], cfg.contrast[1]))
    saturation = float(rng.uniform(cfg.saturation[0], cfg.saturation[1]))
    hue = float(rng.uniform(-cfg.hue, cfg.hue))
    perm = tuple(int(p) for p in rng.permutation(3)) if cfg.channel_permutation else (0, 1, 2)
    return EpisodeTransform(shift, zoom, brightness, contrast, saturation, hue, perm)


def c_config(cfg) -> _lib.AugmentCfg:
    return _lib.AugmentCfg(
        float(cfg.shift_px), float(cfg.zoom[0]), float(cfg.zoom[1]), float(cfg.brightness),
        float(cfg.contrast[0]), float(cfg.contrast[1]), float(cfg.saturation[0]), float(cfg.saturation[1]),
        float(cfg.hue), int(bool(cfg.channel_permutation)), float(cfg.step_brightness),
        float(cfg.step_contrast[0]), float(cfg.step_contrast[1]), float(cfg.step_saturation[0]),
        float(cfg.step_saturation[1]), float(cfg.step_hue), int(cfg.seed))


_REPS = {"color": 0, "diff": 1, "concat": 2}


def augment_params_device(cfg, episode_seeds, step_indices, out=None):
    """(N, 16) float64 CUDA tensor of per-image parameters (see tacsl_b200.h)."""
    t = _device.torch()
    seeds = episode_seeds
    n = seeds.numel()
    if out is None:
        out = t.empty((n, 16), dtype=t.float64, device=seeds.device)
    c = c_config(cfg)
    _lib.check(_lib.load().tacsl_augment_params(ctypes.byref(c), seeds.data_ptr(), step_indices.data_ptr(), n,
                                                out.data_ptr(), _device.stream_handle(seeds.device)))
    return out


def augment_device(images, cfg, episode_seeds, step_indices, tactile_rep="color", nominal=None, out=None,
                   params=None):
    """Batched K4: images (..., H, W, 3) float32 CUDA tensor; episode_seeds /
    step_indices int64 CUDA tensors with one entry per image.  Returns the
    augmented images in the observation representation ("color" / "diff"
    / "concat" against ``nominal``, envs/peg_tasks.py:453-458)."""
    t = _device.torch()
    if tactile_rep not in _REPS:
        raise ValueError(f"tactile_rep must be one of {sorted(_REPS)}")
    if not (_device.is_cuda_tensor(images) and images.dtype == t.float32 and images.shape[-1] == 3):
        raise TypeError("augment_device wants a float32 (..., H, W, 3) CUDA tensor")
    images = images.contiguous()
    H, W = images.shape[-3], images.shape[-2]
    n = images.numel() // (H * W * 3)
    seeds = _device.to_device(episode_seeds, t.int64, images.device).reshape(-1)
    steps = _device.to_device(step_indices, t.int64, images.device).reshape(-1)
    if seeds.numel() != n or steps.numel() != n:
        raise ValueError("one episode seed and one step index per image")
    if params is None:
        params = augment_params_device(cfg, seeds, steps)
    ch = 6 if tactile_rep == "concat" else 3
    if out is None:
        out = t.empty(tuple(images.shape[:-1]) + (ch,), dtype=t.float32, device=images.device)
    nom = np.ascontiguousarray(np.asarray(nominal if nominal is not None else (0, 0, 0), dtype=np.float32))
    _lib.check(_lib.load().tacsl_augment(images.data_ptr(), n, H, W, params.data_ptr(), _REPS[tactile_rep],
                                         nom.ctypes.data, out.data_ptr(), _device.stream_handle(images.device)))
    return out


def augment(image, cfg, episode_seed: int, step_index: int):
    """Drop-in for gelsim.render.augment (augment.py:156-173): float32
    (H, W, 3) in [0, 1], a pure function of (image, cfg, episode_seed,
    step_index).  numpy in -> numpy out; CUDA tensor in -> CUDA tensor out."""
    t = _device.torch()
    on_device = _device.is_cuda_tensor(image)
    dev = _device.resolve_device(image.device if on_device else None)
    img = _device.to_device(image, t.float32, dev)
    seeds = t.tensor([int(episode_seed)], dtype=t.int64, device=dev)
    steps = t.tensor([int(step_index)], dtype=t.int64, device=dev)
    out = augment_device(img[None], cfg, seeds, steps)[0]
    return out if on_device else out.cpu().numpy()
