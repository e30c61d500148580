"""numpy restatement of the reference's tactile-image augmentation
(render/augment.py:51-173) -- TEST INFRASTRUCTURE ONLY.

Same fixed op order (bilinear zoom about the centre then shift, edge-padded
-> channel permutation -> contrast / brightness -> HSV saturation / hue ->
per-step jitter -> clamp), all colour math in float32, parameters from the
tuple-keyed Philox streams (oracle/philox.py).  Pinned against the reference
by tests/test_augment.py (golden vectors from render/augment.py itself).
"""
from __future__ import annotations

import numpy as np

from .philox import Stream


def episode_params(seed, shift_px, zoom, brightness, contrast, saturation, hue, channel_permutation, episode_seed):
    """sample_episode_transform (augment.py:65-75)."""
    s = Stream((seed, int(episode_seed), 0))
    shift = (s.uniform(-shift_px, shift_px), s.uniform(-shift_px, shift_px))
    z = s.uniform(zoom[0], zoom[1])
    b = s.uniform(-brightness, brightness)
    c = s.uniform(contrast[0], contrast[1])
    sat = s.uniform(saturation[0], saturation[1])
    h = s.uniform(-hue, hue)
    perm = tuple(s.permutation(3)) if channel_permutation else (0, 1, 2)
    return shift, z, b, c, sat, h, perm


def step_params(seed, step_brightness, step_contrast, step_saturation, step_hue, episode_seed, step_index):
    """_sample_step_jitter (augment.py:78-85)."""
    s = Stream((seed, int(episode_seed), 1, int(step_index)))
    return (s.uniform(-step_brightness, step_brightness), s.uniform(step_contrast[0], step_contrast[1]),
            s.uniform(step_saturation[0], step_saturation[1]), s.uniform(-step_hue, step_hue))


def _remainder1(x):
    """np.remainder(x, float32(1)) for float32 x: fmod, +1 when negative."""
    m = np.fmod(x, np.float32(1.0))
    m = np.where(m < 0, m + np.float32(1.0), m)
    return np.where(m == 0, np.float32(0.0), m).astype(np.float32)


def rgb_to_hsv(img):
    img = img.astype(np.float32)
    r, g, b = img[..., 0], img[..., 1], img[..., 2]
    mx = np.maximum(np.maximum(r, g), b)
    mn = np.minimum(np.minimum(r, g), b)
    span = mx - mn
    s = np.where(mx > 0, span / np.maximum(mx, np.float32(1e-12)), np.float32(0.0))
    safe = np.where(span > 0, span, np.float32(1.0))
    rc, gc, bc = (mx - r) / safe, (mx - g) / safe, (mx - b) / safe
    h = np.where(r == mx, bc - gc, np.where(g == mx, (np.float32(2.0) + rc) - bc, (np.float32(4.0) + gc) - rc))
    h = np.where(span > 0, _remainder1(h / np.float32(6.0)), np.float32(0.0))
    return np.stack([h, s, mx], axis=-1).astype(np.float32)


def hsv_to_rgb(img):
    h, s, v = img[..., 0], img[..., 1], img[..., 2]
    h6 = h * np.float32(6.0)
    i = np.floor(h6)
    f = h6 - i
    p = v * (np.float32(1.0) - s)
    q = v * (np.float32(1.0) - s * f)
    t = v * (np.float32(1.0) - s * (np.float32(1.0) - f))
    i = i.astype(np.int64) % 6
    r = np.choose(i, [v, q, p, p, t, v])
    g = np.choose(i, [t, v, v, q, p, p])
    b = np.choose(i, [p, p, t, v, v, q])
    return np.stack([r, g, b], axis=-1).astype(np.float32)


def resample(img, zoom, shift):
    H, W = img.shape[:2]
    zf = np.float32(zoom)
    ys = (np.arange(H, dtype=np.float32) - np.float32((H - 1) / 2)) / zf + np.float32((H - 1) / 2) \
        - np.float32(shift[1])
    xs = (np.arange(W, dtype=np.float32) - np.float32((W - 1) / 2)) / zf + np.float32((W - 1) / 2) \
        - np.float32(shift[0])
    ys = np.clip(ys, np.float32(0), np.float32(H - 1))
    xs = np.clip(xs, np.float32(0), np.float32(W - 1))
    y0 = np.clip(ys.astype(np.int64), 0, H - 2)
    x0 = np.clip(xs.astype(np.int64), 0, W - 2)
    fy = (ys - y0.astype(np.float32))[:, None, None]
    fx = (xs - x0.astype(np.float32))[None, :, None]
    a = img[y0][:, x0]
    b = img[y0][:, x0 + 1]
    c = img[y0 + 1][:, x0]
    d = img[y0 + 1][:, x0 + 1]
    one = np.float32(1.0)
    top = a * (one - fx) + b * fx
    bot = c * (one - fx) + d * fx
    return (top * (one - fy) + bot * fy).astype(np.float32)


def color(img, brightness, contrast, saturation, hue):
    if contrast != 1.0:
        img = (img - np.float32(0.5)) * np.float32(contrast) + np.float32(0.5)
    if brightness != 0.0:
        img = img + np.float32(brightness)
    if saturation != 1.0 or hue != 0.0:
        hsv = rgb_to_hsv(np.clip(img, np.float32(0.0), np.float32(1.0)))
        hsv[..., 0] = _remainder1(hsv[..., 0] + np.float32(hue))
        hsv[..., 1] = np.clip(hsv[..., 1] * np.float32(saturation), np.float32(0.0), np.float32(1.0))
        img = hsv_to_rgb(hsv)
    return img.astype(np.float32)


def augment(image, cfg: dict, episode_seed, step_index):
    """cfg: AugmentConfig fields as a dict (augment.py:15-48)."""
    shift, z, b, c, s, h, perm = episode_params(
        cfg["seed"], cfg["shift_px"], cfg["zoom"], cfg["brightness"], cfg["contrast"], cfg["saturation"],
        cfg["hue"], cfg["channel_permutation"], episode_seed)
    img = np.asarray(image, dtype=np.float32)
    if z != 1.0 or shift != (0.0, 0.0):
        img = resample(img, z, shift)
    if perm != (0, 1, 2):
        img = img[..., list(perm)]
    img = color(img, b, c, s, h)
    jit = step_params(cfg["seed"], cfg["step_brightness"], cfg["step_contrast"], cfg["step_saturation"],
                      cfg["step_hue"], episode_seed, step_index)
    if jit != (0.0, 1.0, 1.0, 0.0):
        img = color(img, *jit)
    return np.clip(img, np.float32(0.0), np.float32(1.0)).astype(np.float32)
