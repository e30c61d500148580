"""Per-pixel binned polynomial LUT (north_star "per-pixel binned polynomial
calibration lookup").

NOT in the reference: gelsim's ``PolyLut`` (render/lut.py:31-59) is one
global per-channel polynomial.  The binned table generalises it the way
per-region GelSight calibrations do -- the image is cut into
``bins_y x bins_x`` rectangles, each with its own (3, T) coefficient table:

    bin(y, x) = (y * bins_y // H, x * bins_x // W)
    rgb[y, x, c] = clip(sum_k C[bin(y, x), c, k] g_x^i g_y^j, 0, 1)

with the gradients of ``depth_to_rgb`` (render/lut.py:25-28).  A one-bin
table is exactly ``PolyLut`` and the kernel (csrc/binned.cu) then reproduces
K1 bit for bit; the CPU restatement is oracle/binned_oracle.py (parity
against the reference: unpinned -- there is nothing to pin to).
"""
from __future__ import annotations

import threading
import weakref
from dataclasses import dataclass

import numpy as np

from . import _device, _lib
from .errors import LutResolutionMismatch
from .render import PolyLut, _values, monomial_exponents


@dataclass
class BinnedPolyLut:
    degree: int
    coeffs: np.ndarray      # (bins_y, bins_x, 3, T) float64, monomial_exponents order
    image_size: tuple       # (W, H), as PolyLut

    def __post_init__(self):
        if not (2 <= self.degree <= 4):
            raise ValueError("LUT degree must be in [2, 4]")
        T = len(monomial_exponents(self.degree))
        c = np.asarray(self.coeffs, dtype=np.float64)
        if c.ndim != 4 or c.shape[2:] != (3, T):
            raise ValueError(f"binned coefficients must be (bins_y, bins_x, 3, {T})")
        W, H = (int(v) for v in self.image_size)
        if not (1 <= c.shape[0] <= H and 1 <= c.shape[1] <= W):
            raise ValueError("bins must be in [1, image size]")
        self.coeffs = c
        self.image_size = (W, H)

    @property
    def bins(self) -> tuple:
        return self.coeffs.shape[0], self.coeffs.shape[1]

    @classmethod
    def from_poly_lut(cls, lut: PolyLut, bins=(1, 1)) -> "BinnedPolyLut":
        """The global LUT replicated into every bin (same shading everywhere)."""
        c = np.broadcast_to(np.asarray(lut.coeffs, dtype=np.float64), tuple(bins) + np.shape(lut.coeffs))
        return cls(degree=lut.degree, coeffs=np.ascontiguousarray(c), image_size=tuple(lut.image_size))


def vignetted_lut(lut: PolyLut, bins=(6, 8), falloff: float = 0.25) -> BinnedPolyLut:
    """A binned table from a global one with radial illumination fall-off:
    every coefficient of bin b scaled by 1 - falloff * r_b^2 (r_b = the bin
    centre's normalised distance from the image centre) -- the kind of
    non-uniformity per-region calibrations capture."""
    by, bx = bins
    yc = (np.arange(by) + 0.5) / by * 2 - 1
    xc = (np.arange(bx) + 0.5) / bx * 2 - 1
    r2 = (yc[:, None] ** 2 + xc[None, :] ** 2) / 2
    scale = 1.0 - falloff * r2
    c = np.asarray(lut.coeffs, dtype=np.float64)[None, None] * scale[:, :, None, None]
    return BinnedPolyLut(degree=lut.degree, coeffs=c, image_size=tuple(lut.image_size))


class DeviceBinnedLut:
    """A binned-LUT handle of libtacsl_b200 (table uploaded to one device)."""

    def __init__(self, lut: BinnedPolyLut, device):
        lib = _lib.load()
        coeffs = np.ascontiguousarray(lut.coeffs)
        W, H = lut.image_size
        by, bx = lut.bins
        handle = _lib.c_void_p()
        _lib.check(lib.tacsl_binned_lut_create(int(device.index or 0), coeffs.ctypes.data, int(lut.degree), by,
                                               bx, W, H, _lib.ctypes.byref(handle)))
        self.handle = handle
        self.image_size = (W, H)
        self.device = device
        self._finalizer = weakref.finalize(self, lib.tacsl_binned_lut_destroy, handle)


_lock = threading.Lock()
_cache: dict = {}


def device_binned_lut(lut, device=None) -> DeviceBinnedLut:
    if isinstance(lut, DeviceBinnedLut):
        return lut
    dev = _device.resolve_device(device)
    key = (int(lut.degree), lut.image_size, lut.coeffs.shape, lut.coeffs.tobytes(), str(dev))
    with _lock:
        h = _cache.get(key)
        if h is None:
            h = DeviceBinnedLut(lut, dev)
            if len(_cache) > 32:
                _cache.clear()
            _cache[key] = h
    return h


def depth_to_rgb_binned_device(depth_values, lut, out_u8=None, out_f32=None, stream=None):
    """(..., H, W) float32 CUDA depth -> (..., H, W, 3) uint8 and/or float32."""
    t = _device.torch()
    v = depth_values
    if not (_device.is_cuda_tensor(v) and v.dtype == t.float32 and v.is_contiguous()):
        raise TypeError("depth_to_rgb_binned_device wants a contiguous float32 CUDA tensor")
    dl = device_binned_lut(lut, v.device)
    H, W = v.shape[-2], v.shape[-1]
    n = int(np.prod(v.shape[:-2], dtype=np.int64)) if v.ndim > 2 else 1
    sh = _device.stream_handle(v.device) if stream is None else stream
    _lib.check(_lib.load().tacsl_depth_to_rgb_binned(dl.handle, v.data_ptr(), n, H, W, _device.ptr(out_u8),
                                                     _device.ptr(out_f32), sh))
    return out_u8, out_f32


def depth_to_rgb_binned(depth, lut: BinnedPolyLut, out_dtype=None):
    """``depth_to_rgb`` with a binned table: numpy float64 out for numpy in,
    CUDA float32 (or uint8 with ``out_dtype=np.uint8``) for CUDA in."""
    t = _device.torch()
    values = _values(depth)
    W, H = values.shape[-1], values.shape[-2]
    if (W, H) != tuple(lut.image_size):
        raise LutResolutionMismatch(f"LUT calibrated at {tuple(lut.image_size)}, image is {(W, H)}")
    on_device = _device.is_cuda_tensor(values)
    dev = _device.resolve_device(values.device if on_device else None)
    v = _device.to_device(values, t.float32, dev)
    want_u8 = out_dtype in (np.uint8, t.uint8, "uint8")
    out = t.empty(tuple(v.shape) + (3,), dtype=t.uint8 if want_u8 else t.float32, device=dev)
    if want_u8:
        depth_to_rgb_binned_device(v, lut, out_u8=out)
    else:
        depth_to_rgb_binned_device(v, lut, out_f32=out)
    if on_device:
        return out
    host = out.cpu().numpy()
    return host if want_u8 else host.astype(np.float64)
