"""Separable Gaussian smoothing and multi-scale Gaussian pyramid of depth maps
(north_star stages; BASELINE.json config 5).

These stages are NOT in the reference package, so
the semantics are defined here, scipy.ndimage-style:

* ``gaussian_taps(sigma, truncate=4.0)``: radius = int(truncate * sigma + 0.5),
  w[k] = exp(-k^2 / (2 sigma^2)) normalised (scipy.ndimage.gaussian_filter1d);
* borders replicate the edge sample (mode='nearest', the np.gradient edge
  spirit);
* a pyramid level is the 5-tap binomial [1, 4, 6, 4, 1] / 16 blur followed by
  keeping every second row and column (even indices);
* level l of a tactile pyramid is shaded with the LUT rescaled for pixels 2^l
  times larger: gradients in m/px grow by 2^l, so c_ij -> c_ij 2^(-l(i+j))
  keeps the same shading for the same surface slope.

parity is "unpinned" against the reference (it has no such stage); the CPU
restatement in oracle/pyramid_oracle.py pins the kernels and is itself
checked against scipy.ndimage.
"""
from __future__ import annotations

import numpy as np

from . import _device, _lib
from .render import PolyLut, depth_to_rgb_device, monomial_exponents

BINOMIAL5 = np.array([1.0, 4.0, 6.0, 4.0, 1.0]) / 16.0


def gaussian_taps(sigma: float, truncate: float = 4.0) -> np.ndarray:
    if sigma <= 0:
        return np.array([1.0])
    radius = int(truncate * float(sigma) + 0.5)
    x = np.arange(-radius, radius + 1)
    w = np.exp(-0.5 / (sigma * sigma) * x * x)
    return w / w.sum()


def separable_filter_device(depth, taps, step=1, out=None):
    """(..., H, W) float32 CUDA depth -> filtered (and for step 2 decimated)."""
    t = _device.torch()
    v = depth.contiguous()
    H, W = v.shape[-2], v.shape[-1]
    Ho, Wo = -(-H // step), -(-W // step)
    n = int(np.prod(v.shape[:-2], dtype=np.int64)) if v.ndim > 2 else 1
    taps32 = np.ascontiguousarray(np.asarray(taps, dtype=np.float64).astype(np.float32))
    if out is None:
        out = t.empty(tuple(v.shape[:-2]) + (Ho, Wo), dtype=t.float32, device=v.device)
    _lib.check(_lib.load().tacsl_separable_filter(v.data_ptr(), n, H, W, taps32.ctypes.data,
                                                  (len(taps32) - 1) // 2, step, out.data_ptr(),
                                                  _device.stream_handle(v.device)))
    return out


def gaussian_blur_device(depth, sigma, truncate=4.0, out=None):
    return separable_filter_device(depth, gaussian_taps(sigma, truncate), 1, out)


def pyr_down_device(depth, out=None):
    return separable_filter_device(depth, BINOMIAL5, 2, out)


def level_lut(lut, level: int) -> PolyLut:
    """The LUT for pyramid level `level` (pixels 2^level larger)."""
    W, H = lut.image_size
    for _ in range(level):
        W, H = -(-W // 2), -(-H // 2)
    coeffs = np.asarray(lut.coeffs, dtype=np.float64).copy()
    for k, (i, j) in enumerate(monomial_exponents(lut.degree)):
        coeffs[:, k] *= 2.0 ** (-level * (i + j))
    return PolyLut(degree=lut.degree, coeffs=coeffs, image_size=(W, H))


def fused_pyramid_supported(H, W, levels, sigma=0.0, truncate=4.0) -> bool:
    """Whether K7 (tacsl_rgb_pyramid, one pass) serves this shape."""
    radius = (len(gaussian_taps(sigma, truncate)) - 1) // 2 if sigma > 0 else 0
    return bool(_lib.load().tacsl_rgb_pyramid_supported(int(H), int(W), radius, int(levels)))


def rgb_pyramid_fused_device(depth, lut, levels=3, sigma=0.0, truncate=4.0, outs=None, luts=None):
    """K7: smoothing + every pyramid level's uint8 RGB in ONE kernel pass
    (bit-identical to rgb_pyramid_device's level-by-level chain).  depth
    (..., H, W) float32 CUDA; returns the list of (..., H >> l, W >> l, 3)
    uint8 tensors (``outs`` to reuse buffers; ``luts`` the level DeviceLuts)."""
    import ctypes

    from .render import device_lut

    t = _device.torch()
    d = depth
    if not (_device.is_cuda_tensor(d) and d.dtype == t.float32 and d.is_contiguous()):
        raise TypeError("rgb_pyramid_fused_device wants a contiguous float32 CUDA tensor")
    H, W = int(d.shape[-2]), int(d.shape[-1])
    n = int(np.prod(d.shape[:-2], dtype=np.int64)) if d.ndim > 2 else 1
    taps = gaussian_taps(sigma, truncate) if sigma > 0 else np.array([1.0])
    radius = (len(taps) - 1) // 2
    taps32 = np.ascontiguousarray(taps.astype(np.float32))
    if luts is None:
        luts = [device_lut(level_lut(lut, lvl)) for lvl in range(levels)]
    if outs is None:
        outs = [t.empty(tuple(d.shape[:-2]) + (H >> lvl, W >> lvl, 3), dtype=t.uint8, device=d.device)
                for lvl in range(levels)]
    handles = (ctypes.c_void_p * levels)(*[lu.handle.value for lu in luts])
    ptrs = (ctypes.c_void_p * levels)(*[o.data_ptr() for o in outs])
    _lib.check(_lib.load().tacsl_rgb_pyramid(ctypes.addressof(handles), levels, d.data_ptr(), n, H, W,
                                             taps32.ctypes.data, radius, ctypes.addressof(ptrs),
                                             _device.stream_handle(d.device)))
    return outs


def rgb_pyramid_device(depth, lut, levels=3, sigma=0.0, truncate=4.0):
    """Multi-scale tactile RGB: optional Gaussian smoothing of the full-res
    depth, then `levels` uint8 RGB images, level l at 2^-l resolution.
    Returns the list of (..., H_l, W_l, 3) uint8 CUDA tensors."""
    t = _device.torch()
    d = depth.contiguous()
    if sigma > 0:
        d = gaussian_blur_device(d, sigma, truncate)
    outs = []
    for lvl in range(levels):
        if lvl:
            d = pyr_down_device(d)
        u8 = t.empty(tuple(d.shape) + (3,), dtype=t.uint8, device=d.device)
        depth_to_rgb_device(d, level_lut(lut, lvl), out_u8=u8)
        outs.append(u8)
    return outs
