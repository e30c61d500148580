"""On-disk formats of the hot path's inputs and outputs.

* LUT text file ``GELSIM-LUT v1`` (render/lut.py:117-162): ``write_lut`` /
  ``read_lut``, byte-compatible with the reference;
* TFF1 force-field frames (tactile/io.py:13-39): ``write_force_field_frames``
  / ``read_force_field_frames``, plus ``export_force_field_frames`` which
  packs [f_n, f_t] per taxel on the device and moves one contiguous float32
  block to the host per call;
* ``shear_map_image`` (tactile/io.py:42-58);
* the TSDF grid cache lives in ``geometry`` (sdf.py:331-361).
"""
from __future__ import annotations

import struct

import numpy as np

from . import _device
from .render import PolyLut, monomial_exponents
from .tactile import ForceField

LUT_FORMAT_VERSION = 1
TFF_MAGIC = b"TFF1"


# ---------------------------------------------------------------- LUT text ---

def write_lut(lut, path) -> None:
    """Versioned text header + coefficient table (render/lut.py:122-137)."""
    exps = monomial_exponents(lut.degree)
    coeffs = np.asarray(lut.coeffs, dtype=np.float64).reshape(3, -1)
    bg = coeffs[:, 0]
    lines = [
        f"GELSIM-LUT v{LUT_FORMAT_VERSION}",
        f"degree: {lut.degree}",
        "channels: 3",
        f"background: {bg[0]:.9g} {bg[1]:.9g} {bg[2]:.9g}",
        f"image_size: {lut.image_size[0]} {lut.image_size[1]}",
        f"sensor_id: {getattr(lut, 'sensor_id', '')}",
        f"calibrated_on: {getattr(lut, 'calibrated_on', '')}",
        f"residual_rms: {getattr(lut, 'residual_rms', 0.0):.9g}",
        f"terms: {len(exps)}",
    ]
    for k, (i, j) in enumerate(exps):
        c = coeffs[:, k]
        lines.append(f"{i} {j} {c[0]:.17g} {c[1]:.17g} {c[2]:.17g}")
    with open(path, "w") as fh:
        fh.write("\n".join(lines) + "\n")


def read_lut(path) -> PolyLut:
    """Parse a ``GELSIM-LUT v1`` file (render/lut.py:140-162)."""
    with open(path, "r") as fh:
        header = fh.readline().strip()
        if not header.startswith("GELSIM-LUT v"):
            raise ValueError(f"{path}: not a LUT file")
        if int(header.split("v")[-1]) != LUT_FORMAT_VERSION:
            raise ValueError(f"{path}: unsupported LUT version")
        meta = {}
        for _ in range(8):
            key, val = fh.readline().split(":", 1)
            meta[key.strip()] = val.strip()
        degree = int(meta["degree"])
        exps = monomial_exponents(degree)
        n_terms = int(meta["terms"])
        if n_terms != len(exps):
            raise ValueError(f"{path}: {n_terms} terms for degree {degree}")
        coeffs = np.zeros((3, n_terms))
        for k in range(n_terms):
            parts = fh.readline().split()
            if (int(parts[0]), int(parts[1])) != exps[k]:
                raise ValueError(f"{path}: term {k} is {parts[:2]}, expected {exps[k]}")
            coeffs[:, k] = [float(p) for p in parts[2:5]]
    W, H = (int(x) for x in meta["image_size"].split())
    return PolyLut(degree=degree, coeffs=coeffs, image_size=(W, H), sensor_id=meta["sensor_id"],
                   calibrated_on=meta["calibrated_on"], residual_rms=float(meta["residual_rms"]))


# ------------------------------------------------------------------- TFF1 ---

def _frames_bytes(per_point: np.ndarray) -> bytes:
    """(F, R, C, 6) float32 -> back-to-back TFF1 frames."""
    F, R, C = per_point.shape[:3]
    head = TFF_MAGIC + struct.pack("<2I", R, C)
    data = np.ascontiguousarray(per_point, dtype="<f4")
    chunks = []
    for f in range(F):
        chunks.append(head)
        chunks.append(data[f].tobytes(order="C"))
    return b"".join(chunks)


def write_force_field_frames(path, fields) -> None:
    """One (rows, cols, 3) ForceField per frame: magic, rows, cols, then
    6 float32 per taxel [f_n, f_t] (tactile/io.py:13-23)."""
    per = []
    for fld in fields:
        if fld.f_n.ndim != 3:
            raise ValueError("write one env per frame (rows, cols, 3)")
        f_n = fld.f_n.cpu().numpy() if _device.is_cuda_tensor(fld.f_n) else np.asarray(fld.f_n)
        f_t = fld.f_t.cpu().numpy() if _device.is_cuda_tensor(fld.f_t) else np.asarray(fld.f_t)
        per.append(np.concatenate([f_n, f_t], axis=-1).astype("<f4")[None])
    with open(path, "wb") as fh:
        for p in per:
            fh.write(_frames_bytes(p))


def export_force_field_frames(path, f_n, f_t, append=False) -> int:
    """Dataset export straight from device tensors: f_n, f_t (..., R, C, 3)
    CUDA tensors (any float dtype) -> TFF1 frames, one per leading index.
    The [f_n, f_t] interleave and the float32 cast run on the device; one
    device->host copy moves the payload.  Returns the number of frames."""
    t = _device.torch()
    R, C = f_n.shape[-3], f_n.shape[-2]
    packed = t.cat([f_n.reshape(-1, R, C, 3), f_t.reshape(-1, R, C, 3)], dim=-1).to(t.float32)
    host = packed.cpu().numpy()
    with open(path, "ab" if append else "wb") as fh:
        fh.write(_frames_bytes(host))
    return host.shape[0]


def read_force_field_frames(path) -> list:
    """TFF1 frames -> list of float64 ForceField (tactile/io.py:26-39)."""
    out = []
    with open(path, "rb") as fh:
        while True:
            head = fh.read(4)
            if not head:
                break
            if head != TFF_MAGIC:
                raise ValueError(f"{path}: bad frame magic {head!r}")
            rows, cols = struct.unpack("<2I", fh.read(8))
            data = np.frombuffer(fh.read(rows * cols * 6 * 4), dtype="<f4").reshape(rows, cols, 6)
            data = data.astype(np.float64)
            out.append(ForceField(f_n=data[..., :3], f_t=data[..., 3:]))
    return out


def shear_map_image(fld, upscale: int = 16) -> np.ndarray:
    """RG-encoded uint8 shear map normalised by the frame's peak shear, B
    neutral (tactile/io.py:42-58)."""
    f_t = fld.f_t.cpu().numpy() if _device.is_cuda_tensor(fld.f_t) else np.asarray(fld.f_t)
    fx, fy = f_t[..., 0], f_t[..., 1]
    peak = max(float(np.abs(fx).max(initial=0.0)), float(np.abs(fy).max(initial=0.0)), 1e-12)
    r = 0.5 + 0.5 * fx / peak
    g = 0.5 + 0.5 * fy / peak
    img = np.stack([r, g, np.full_like(r, 0.5)], axis=-1)
    img = np.clip(np.rint(img * 255), 0, 255).astype(np.uint8)
    if upscale > 1:
        img = np.repeat(np.repeat(img, upscale, axis=0), upscale, axis=1)
    return img
