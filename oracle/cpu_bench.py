"""CPU baseline runner -- TEST INFRASTRUCTURE ONLY (bench.py's cpu_baseline
leg and --impl reference arm).

Times the numpy restatement of the reference path (gelsim_oracle, which
follows gelsim's depth_to_rgb + to_uint8 + compute_force_field + net_wrench
operation for operation) on a bounded sample of the benchmark workload, one
single-threaded worker process per host core (OMP/OPENBLAS/MKL threads = 1
per process: threaded BLAS slows the LUT matmul).
"""
from __future__ import annotations

import os
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

_W = {}


def _init(image_size, ff_grid, sdf_dims, degree, n_sensors, config_id, pool_maps, with_rgb=True, with_ff=True,
          levels=1, sigma=0.0):
    for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[k] = "1"
    from paper_2408_06506_b200 import synthetic

    _, cam, bg, lut, pts = synthetic.sensor_setup(image_size, ff_grid, lut_degree=degree)
    sdf = synthetic.peg_grid(sdf_dims)
    _W.update(
        depth=synthetic.depth_batch(cam, bg, pool_maps, config_id=config_id),
        lut=lut, pts=pts.points,
        sdf=(sdf.origin, sdf.spacing, sdf.dims, sdf.values, sdf.gradients),
        states=synthetic.peg_states(64, n_sensors, config_id=config_id),
        with_rgb=with_rgb, with_ff=with_ff, levels=levels, sigma=sigma,
    )
    if levels > 1 or sigma > 0:
        from paper_2408_06506_b200 import smoothing
        _W["taps"] = smoothing.gaussian_taps(sigma) if sigma > 0 else None
        _W["binomial"] = smoothing.BINOMIAL5
        _W["level_luts"] = [smoothing.level_lut(lut, lvl) for lvl in range(levels)]


def _run(args):
    lo, hi = args
    from oracle import gelsim_oracle as O

    depth, lut = _W["depth"], _W["lut"]
    obj, sen = _W["states"]
    E, S = sen.shape[:2]
    t0 = time.perf_counter()
    acc = 0.0
    for c0 in range(lo, hi, 8):  # 8 frames per call bounds the temporaries (~100 MB)
        idx = np.arange(c0, min(c0 + 8, hi))
        d = depth[idx % len(depth)]
        objF = obj[(idx // S) % E]
        senF = sen.reshape(E * S, 13)[idx % (E * S)]
        if _W["with_rgb"] and "level_luts" in _W:
            from oracle.pyramid_oracle import separable_filter
            x = separable_filter(d, _W["taps"], 1) if _W["taps"] is not None else d
            for lvl, ll in enumerate(_W["level_luts"]):
                if lvl:
                    x = separable_filter(x, _W["binomial"], 2)
                rgb = O.to_uint8(O.depth_to_rgb(x, ll.coeffs, ll.degree))
                acc += float(rgb[0, 0, 0, 0])
        elif _W["with_rgb"]:
            rgb = O.to_uint8(O.depth_to_rgb(d, lut.coeffs, lut.degree))
            acc += float(rgb[0, 0, 0, 0])
        if _W["with_ff"]:
            f_n, f_t, _ = O.compute_force_field(_W["pts"], *_W["sdf"], objF[:, 0:3], objF[:, 3:7], objF[:, 7:10],
                                                objF[:, 10:13], senF[:, 0:3], senF[:, 3:7], senF[:, 7:10],
                                                senF[:, 10:13])
            force, _ = O.net_wrench(f_n, f_t, _W["pts"])
            acc += float(force.sum())
    return hi - lo, time.perf_counter() - t0, acc


class CpuBaseline:
    """A warm pool of `cores` single-threaded oracle workers."""

    def __init__(self, workload, cores=None, pool_maps=8):
        self.cores = int(cores or os.cpu_count() or 1)
        self.workload = workload
        init = (tuple(workload.image_size), tuple(workload.ff_grid), tuple(workload.sdf_dims),
                workload.lut_degree, workload.n_sensors, workload.config_id, pool_maps,
                getattr(workload, "rgb", True), getattr(workload, "ff", True),
                getattr(workload, "pyramid_levels", 1), getattr(workload, "smooth_sigma", 0.0))
        self.pool = ProcessPoolExecutor(max_workers=self.cores, initializer=_init, initargs=init)
        # warm every worker (imports + asset set-up) outside any timing
        list(self.pool.map(_run, [(i, i + 1) for i in range(self.cores)]))

    def run(self, frames_per_core: int) -> tuple:
        """One bounded sample: `frames_per_core` sensor frames on every worker.
        Returns (frames, wall seconds)."""
        chunks = [(c * frames_per_core, (c + 1) * frames_per_core) for c in range(self.cores)]
        t0 = time.perf_counter()
        done = sum(r[0] for r in self.pool.map(_run, chunks))
        return done, time.perf_counter() - t0

    def close(self):
        self.pool.shutdown(wait=True, cancel_futures=True)


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"
