"""Benchmark: sensor frames/s (tactile RGB + force field + wrench) at 4096 envs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 3] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

One step = one pass of the hot path over the whole workload: for every
(env, sensor) frame, 240x320 depth -> uint8 RGB (K1) and the 20x25-taxel
force field + net wrench against the 32x32x64 peg SDF (K2).  Config 3 =
4096 envs x 2 fingertip sensors = 8192 sensor frames per step, sharded over
ranks by env (strong scaling; no collective on the data path).

Printed on rank 0 as ONE JSON line.  ``value`` is device-timed throughput
with inputs resident in HBM; ``e2e`` is the same metric through the host
buffer API (pinned host -> device copies of every step's inputs and
device -> host copies of every step's outputs inside the timed region);
``roofline`` reports the dominant kernel (K1) against the measured HBM
copy bandwidth; ``cpu_baseline`` is the CPU oracle (a numpy restatement of
the reference) on a bounded sample on this host's cores.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "sensor frames/sec (RGB+force field) at 4096 envs, 1-8 GPUs; % of HBM roofline"
UNIT = "sensor-frames/s"
FALLBACK_HBM_GBS = 6650.0


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--settle", type=float, default=2.0,
                   help="idle seconds between two warm-up phases before the timed region (0: none)")
    p.add_argument("--config", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--no-graph", action="store_true")
    p.add_argument("--no-overlap", action="store_true")
    p.add_argument("--fused", action="store_true", help="one launch (force-field warps inside K1) per step")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=8)
    p.add_argument("--no-e2e", action="store_true", help="skip the host-buffer e2e leg (profiling runs)")
    p.add_argument("--e2e-chunks", type=int, default=64, help="env chunks pipelined over H2D / compute / D2H")
    p.add_argument("--cpu-seconds", type=float, default=10.0, help="target CPU-baseline sample length")
    p.add_argument("--dropin-frames", type=int, default=1024,
                   help="sensor frames per call of the numpy drop-in e2e leg (0: skip)")
    p.add_argument("--also", default="4,5",
                   help="comma-separated other configs timed briefly after the main one (N=1 only; '' to skip)")
    p.add_argument("--also-steps", type=int, default=10)
    p.add_argument("--sustain-s", type=float, default=1.5,
                   help="seconds of back-to-back steps for value_sustained (0: skip)")
    p.add_argument("--envs", type=int, default=None,
                   help="override the config's env count (experiments, e.g. one GPU's share at N GPUs)")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def hbm_peak():
    f = ROOT / "MEASURED_PEAKS.json"
    try:
        v = float(json.loads(f.read_text())["hbm_gbs"])
        return v, "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:  # noqa: BLE001
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """NVML SM-clock / throttle-reason sampling while the timed region runs."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
    }

    def __init__(self, index, period=0.005):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self.nvml = None

    def _loop(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nvml.nvmlDeviceGetClockInfo(self.h, self.nvml.NVML_CLOCK_SM))
                r = self.nvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nvml is not None:
            self._t = threading.Thread(target=self._loop, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join()

    def summary(self):
        med = float(np.median(self.samples)) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def traffic_from_profiles(kernel_key):
    """dram bytes per launch from the committed ncu --set full summary."""
    f = ROOT / "profiles" / "traffic.json"
    try:
        return json.loads(f.read_text()).get(kernel_key)
    except Exception:  # noqa: BLE001
        return None


def workload_text(wl):
    parts = []
    if wl.rgb:
        img = f"{wl.image_size[1]}x{wl.image_size[0]} RGB (uint8)"
        if wl.smooth_sigma > 0:
            img = f"Gaussian-smoothed (sigma={wl.smooth_sigma:g} px) {img}"
        if wl.pyramid_levels > 1:
            img += f" as a {wl.pyramid_levels}-level pyramid"
        parts.append(img)
    if wl.ff:
        parts.append(f"{wl.ff_grid[0]}x{wl.ff_grid[1]} force field + wrench, peg SDF "
                     f"{'x'.join(map(str, wl.sdf_dims))}")
    return f"config {wl.config_id}: {wl.n_envs} envs x {wl.n_sensors} sensors, " + " + ".join(parts)


def workload_config(wl, world):
    return {
        "workload": workload_text(wl),
        "envs": wl.n_envs, "sensors_per_env": wl.n_sensors, "sensor_frames_per_step": wl.frames,
        "image": [wl.image_size[1], wl.image_size[0]], "taxels": list(wl.ff_grid),
        "sdf_dims": list(wl.sdf_dims), "lut_degree": wl.lut_degree,
        "pyramid_levels": wl.pyramid_levels, "smooth_sigma": wl.smooth_sigma,
        "parallelism": f"env-sharded x{world} (no data-path collective)",
        "l2": "inputs (2.5 GB depth at config 3) exceed the 126 MB L2; no flush needed",
    }


# ----------------------------------------------------------------- reference ---

def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    from oracle.cpu_bench import CpuBaseline, cpu_model
    from paper_2408_06506_b200.synthetic import CONFIGS

    wl = CONFIGS[args.config]
    base = CpuBaseline(wl)
    # size one step so the whole K+W run stays within a few minutes
    n, dt = base.run(1)
    per_frame = dt / max(n, 1) * base.cores  # core-seconds per frame
    budget = 120.0 / max(args.steps + args.warmup, 1)
    fpc = max(1, min(int(budget / max(per_frame, 1e-4)), wl.frames // base.cores))
    for _ in range(args.warmup):
        base.run(fpc)
    frames, secs = 0, 0.0
    for _ in range(args.steps):
        n, dt = base.run(fpc)
        frames += n
        secs += dt
    base.close()
    value = frames / secs
    sample = (f"{fpc} sensor frames per core per step x {base.cores} cores ({fpc * base.cores} of the "
              f"{wl.frames} frames of a config-{wl.config_id} step); {cpu_model()}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {**workload_config(wl, 1),
                   "parallelism": f"host CPU: {base.cores} single-threaded worker processes on rank 0 "
                                  "(oracle port of gelsim's numpy path)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": base.cores, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------- ours ---

class Ctx:
    """One rank's share of a benchmark workload, resident on its GPU."""


def setup_workload(wl, rank, world, dev, fused=False, overlap=True):
    """Build this rank's env shard of config `wl` exactly as the timed step
    runs it: device-resident inputs (global frame g uses indenter map g % 64
    and the states of env g // S, whatever the rank count) and the
    SensorArray (fp32 force outputs, uint8 RGB)."""
    import torch

    from paper_2408_06506_b200 import SensorArray, synthetic
    from paper_2408_06506_b200.pipeline import shard_range
    from paper_2408_06506_b200.tactile import PenaltyParams

    c = Ctx()
    c.wl = wl
    c.lo, c.hi = shard_range(wl.n_envs, rank, world)
    E, S = c.hi - c.lo, wl.n_sensors
    W, H = wl.image_size
    c.E, c.S, c.H, c.W = E, S, H, W
    _, c.cam, c.bg, c.lut, c.pts = synthetic.sensor_setup(wl.image_size, wl.ff_grid, lut_degree=wl.lut_degree)
    c.sdf = synthetic.peg_grid(wl.sdf_dims)
    c.params = PenaltyParams()
    c.pool = synthetic.depth_batch(c.cam, c.bg, 64, config_id=wl.config_id)
    pool = torch.from_numpy(c.pool).to(dev)
    idx = (torch.arange(E * S, device=dev) + c.lo * S) % pool.shape[0]  # this shard's slice of the global job
    c.depth = pool[idx].reshape(E, S, H, W).contiguous()
    del pool, idx
    c.obj_all, c.sen_all = synthetic.peg_states(wl.n_envs, S, config_id=wl.config_id)
    c.obj = torch.from_numpy(c.obj_all[c.lo:c.hi]).to(dev)
    c.sen = torch.from_numpy(np.ascontiguousarray(c.sen_all[c.lo:c.hi])).to(dev)
    c.arr = SensorArray(c.lut, c.sdf, c.pts, c.params, E, S, device=dev, overlap=overlap, rgb_u8=wl.rgb,
                        with_ff=wl.ff, fused=fused, pyramid_levels=wl.pyramid_levels,
                        smooth_sigma=wl.smooth_sigma)
    return c


def sample_indices(frames, n=16):
    """Deterministic global frame indices checked against the oracle: both
    ends, the middle, the first/last frame of every eighth of the job (rank
    boundaries at N = 1, 2, 4, 8) and seeded random picks."""
    idx = {0, frames - 1, frames // 2}
    for k in range(1, 8):
        b = k * frames // 8
        idx.update((b - 1, b))
    rng = np.random.default_rng(20240812)
    extra = [int(i) for i in rng.integers(0, frames, 4 * n)]
    for i in extra:
        if len(idx) >= n:
            break
        idx.add(i)
    return np.array(sorted(i for i in idx if 0 <= i < frames), dtype=np.int64)


def gather_rows(outputs, owned, n_rows, world, coll_dev):
    """All-gather sampled per-frame rows to every rank (rank 0 uses them).

    outputs: list of (name, (n_local_frames, ...) device tensor); owned: list
    of (row in the sample, local frame index) this rank holds.  Each rank
    sends an (n_rows, frame bytes) uint8 block with its own rows filled
    (zeros elsewhere) over the process group (NCCL on the GPU box, gloo in
    the CPU tests); the result maps name -> (n_rows, frame bytes) uint8 numpy
    with every row taken from the rank that owns it."""
    import torch
    import torch.distributed as dist

    out = {}
    for name, x in outputs:
        flat = x.reshape(x.shape[0], -1)
        nb = flat.shape[1] * flat.element_size()
        block = torch.zeros((n_rows, nb), dtype=torch.uint8, device=x.device)
        have = torch.zeros(n_rows, dtype=torch.uint8, device=x.device)
        if owned:
            rows = torch.tensor([r for r, _ in owned], device=x.device)
            loc = torch.tensor([f for _, f in owned], device=x.device)
            block[rows] = flat[loc].contiguous().view(torch.uint8).reshape(len(owned), nb)
            have[rows] = 1
        block, have = block.to(coll_dev), have.to(coll_dev)
        if world > 1:
            parts = [torch.empty_like(block) for _ in range(world)]
            hv = [torch.empty_like(have) for _ in range(world)]
            dist.all_gather(parts, block)
            dist.all_gather(hv, have)
            owner = torch.stack(hv).to(torch.int64).argmax(dim=0)  # the rank that holds each row
            block = torch.stack(parts)[owner, torch.arange(n_rows, device=block.device)]
        out[name] = (block.cpu().numpy(), np.dtype(str(x.dtype).replace("torch.", "")), tuple(x.shape[1:]))
    return {k: b.view(dt).reshape((n_rows,) + shp) for k, (b, dt, shp) in out.items()}


def gather_digests(digests, n_local, world, coll_dev):
    """Concatenate every rank's (n_local, k) int64 frame digests in rank
    (= global env) order; returns the (frames, k) numpy array on every rank."""
    import torch
    import torch.distributed as dist

    d = digests.to(coll_dev)
    if world == 1:
        return d.cpu().numpy()
    n = torch.tensor([n_local], dtype=torch.int64, device=coll_dev)
    ns = [torch.empty_like(n) for _ in range(world)]
    dist.all_gather(ns, n)
    counts = [int(v.item()) for v in ns]
    pad = torch.zeros((max(counts), d.shape[1]), dtype=d.dtype, device=coll_dev)
    pad[:n_local] = d
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    return np.concatenate([p[:c].cpu().numpy() for p, c in zip(parts, counts)])


def digest_summary(names, table):
    """sha256 over the per-frame digest table (frame order, little endian),
    whole and per output -- independent of the rank count."""
    import hashlib

    tab = np.ascontiguousarray(table.astype("<i8"))
    return {"sha256": hashlib.sha256(tab.tobytes()).hexdigest(),
            "per_output": {n: hashlib.sha256(np.ascontiguousarray(tab[:, j]).tobytes()).hexdigest()[:16]
                           for j, n in enumerate(names)},
            "frames": int(tab.shape[0]),
            "rule": "per-frame tacsl_frame_digest of every output, concatenated over ranks in env order"}


def check_parity(c, idx, got):
    """Rank 0: the oracle (numpy restatement of gelsim, pinned to the
    reference's golden vectors) on the sampled frames' inputs, regenerated
    from the same seeds, against the gathered device outputs."""
    from oracle import gelsim_oracle as O

    wl = c.wl
    S = wl.n_sensors
    res = {"frames_checked": [int(i) for i in idx]}
    env, sensor = idx // S, idx % S
    ok = True
    if wl.rgb:
        depth = c.pool[idx % len(c.pool)].astype(np.float64)
        if wl.pyramid_levels > 1 or wl.smooth_sigma > 0:
            from oracle.pyramid_oracle import separable_filter
            from paper_2408_06506_b200 import smoothing
            x = separable_filter(depth, smoothing.gaussian_taps(wl.smooth_sigma), 1) if wl.smooth_sigma else depth
            refs = []
            for lvl in range(wl.pyramid_levels):
                if lvl:
                    x = separable_filter(x, smoothing.BINOMIAL5, 2)
                ll = smoothing.level_lut(c.lut, lvl)
                refs.append(("rgb" if lvl == 0 else f"rgb_l{lvl}", O.to_uint8(O.depth_to_rgb(x, ll.coeffs, ll.degree))))
            frac_tol = 2e-2  # fp32 chain vs the float64 restatement (tests/test_pyramid.py)
        else:
            refs = [("rgb", O.to_uint8(O.depth_to_rgb(depth, c.lut.coeffs, c.lut.degree)))]
            frac_tol = 1e-4  # fp32 polynomial vs the float64 reference
        lsb, off, n = 0, 0, 0
        for name, ref in refs:
            d = np.abs(got[name].astype(np.int64) - ref.astype(np.int64))
            lsb = max(lsb, int(d.max()))
            off += int((d > 0).sum())
            n += d.size
        res.update(rgb_max_lsb=lsb, rgb_frac_off=off / n, rgb_values_checked=n, rgb_frac_tol=frac_tol)
        ok &= lsb <= 1 and off / n <= frac_tol
    if wl.ff:
        o = c.obj_all[env]
        s = c.sen_all[env, sensor]
        sdf = (c.sdf.origin, c.sdf.spacing, c.sdf.dims, c.sdf.values, c.sdf.gradients)
        f_n, f_t, _ = O.compute_force_field(c.pts.points, *sdf, o[:, 0:3], o[:, 3:7], o[:, 7:10], o[:, 10:13],
                                            s[:, 0:3], s[:, 3:7], s[:, 7:10], s[:, 10:13],
                                            c.params.k_n, c.params.k_d, c.params.k_t, c.params.mu)
        force, torque = O.net_wrench(f_n, f_t, c.pts.points)
        worst, zero_abs, mism = 0.0, 0.0, 0
        for g, r in ((got["f_n"], f_n), (got["f_t"], f_t)):
            g = g.astype(np.float64)
            err = np.linalg.norm(g - r, axis=-1)
            nr = np.linalg.norm(r, axis=-1)
            nz = nr > 0
            if nz.any():
                worst = max(worst, float((err[nz] / nr[nz]).max()))
            if (~nz).any():
                zero_abs = max(zero_abs, float(err[~nz].max()))
        gm = (np.abs(got["f_n"]).sum(-1) + np.abs(got["f_t"]).sum(-1)) > 0
        rm = (np.abs(f_n).sum(-1) + np.abs(f_t).sum(-1)) > 0
        mism = int((gm != rm).sum())
        w = got["wrench"]
        ref_w = np.concatenate([force, torque], axis=-1)
        scale = np.abs(f_n).sum(axis=(-3, -2, -1)) + np.abs(f_t).sum(axis=(-3, -2, -1)) + 1e-30
        w_rel = float((np.abs(w - ref_w).max(axis=-1) / scale).max())
        res.update(ff_max_rel=worst, ff_max_abs_where_ref_zero=zero_abs, mask_mismatches=mism,
                   contact_taxels=int(rm.sum()), taxels_checked=int(rm.size), wrench_max_rel_of_sum_abs_f=w_rel)
        ok &= worst <= 1e-5 and zero_abs <= 1e-9 and mism == 0 and w_rel <= 1e-6
    res["ok"] = bool(ok)
    res["rule"] = ("sampled frames of the last timed step vs the oracle on the same inputs: RGB <= 1 LSB "
                   "(fraction of values off by one <= rgb_frac_tol), forces <= 1e-5 relative per taxel, "
                   "identical nonzero-force (contact) masks, wrench <= 1e-6 of sum |f|")
    return res


def validate(c, world, rank, coll_dev, n_samples=16):
    """Outside every timed region: sampled-frame oracle parity of the last
    step (gathered to rank 0 over the process group) and the whole-job
    per-frame digest table (gathered the same way)."""
    import torch

    arr = c.arr
    S = c.wl.n_sensors
    names, dig = arr.frame_digests()
    table = gather_digests(dig, c.E * S, world, coll_dev)
    idx = sample_indices(c.wl.frames, n_samples)
    owned = [(r, int(g) - c.lo * S) for r, g in enumerate(idx) if c.lo * S <= g < c.hi * S]
    outs = []
    for name, x in arr.outputs():
        if name == "rgb_f32":
            continue
        outs.append((name, x.reshape((c.E * S,) + tuple(x.shape[2:]))))
    got = gather_rows(outs, owned, len(idx), world, coll_dev)
    torch.cuda.synchronize()
    if rank != 0:
        return None
    return {"parity": check_parity(c, idx, got), "digest": digest_summary(names, table)}


def run_other_config(cid, dev, args, peak):
    """One extra config on this GPU: graph-captured step, K steps timed with
    CUDA events, the dominant kernel timed alone, the parity block."""
    import torch

    from paper_2408_06506_b200 import synthetic

    wl = synthetic.CONFIGS[cid]
    c = setup_workload(wl, 0, 1, dev)
    arr = c.arr
    arr.capture(c.depth, c.obj, c.sen)
    for _ in range(3):
        arr.replay()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream(dev)

    def timed(fn, n):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record(stream)
        for _ in range(n):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n

    ms = timed(arr.replay, args.also_steps)
    bytes_ = arr.algorithmic_bytes()
    if wl.rgb:
        name, kbytes = arr.image_kernel_name() if (arr.levels > 1 or arr.sigma > 0) else "rgb_bulk_kernel", \
            bytes_["rgb"]
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            arr._launch_rgb(c.depth)
    else:
        name, kbytes = arr.ff_kernel_name(), bytes_["ff"]
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            arr._launch_ff(c.obj, c.sen)
    g.replay()
    torch.cuda.synchronize()
    kms = timed(g.replay, args.also_steps)
    v = validate(c, 1, 0, dev)
    out = {"workload": workload_text(wl), "value": wl.frames / (ms / 1e3), "unit": UNIT, "ms_per_step": ms,
           "steps": args.also_steps, "kernel": name, "kernel_ms": kms,
           "kernel_frac_of_hbm_peak": kbytes / (kms / 1e3) / 1e9 / peak,
           "traffic": traffic_from_profiles(f"{name}/config{cid}/world1"),
           "algorithmic_bytes_per_launch": kbytes, "parity": v["parity"], "validation_sha256": v["digest"]["sha256"]}
    del c, arr, g
    torch.cuda.empty_cache()
    return out


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    from paper_2408_06506_b200 import synthetic

    rank, world, local = dist_env()
    # one process per GPU; TACSL_DIST_BACKEND=gloo lets a multi-rank run share
    # one GPU as a functional check of the sharding (never a measurement)
    backend = os.environ.get("TACSL_DIST_BACKEND", "nccl")
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    coll_dev = dev if backend == "nccl" else torch.device("cpu")
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    wl = synthetic.CONFIGS[args.config]
    if args.envs:
        import dataclasses
        wl = dataclasses.replace(wl, n_envs=args.envs)
    c = setup_workload(wl, rank, world, dev, fused=args.fused, overlap=not args.no_overlap)
    arr, depth, obj, sen = c.arr, c.depth, c.obj, c.sen

    use_graph = not args.no_graph
    if use_graph:
        arr.capture(depth, obj, sen)
    step = arr.replay if use_graph else (lambda: arr.launch(depth, obj, sen))

    def graph_of(fn):
        """fn's launches as a replayable CUDA graph (per-kernel timing without
        Python launch overhead between back-to-back launches)."""
        if not use_graph:
            return fn
        side = torch.cuda.Stream(device=dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):
            fn()
        torch.cuda.current_stream(dev).wait_stream(side)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        return g.replay

    k1_fn = graph_of(lambda: arr._launch_rgb(depth)) if wl.rgb else None
    k2_fn = graph_of(lambda: arr._launch_ff(obj, sen)) if wl.ff else None
    kf_fn = graph_of(lambda: arr._launch_fused(depth, obj, sen)) if arr.fused else None

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if args.settle > 0:
        # Start the timed region from the same board state every run: after a
        # preceding workload (the driver runs the test suite first) the power
        # limiter holds SM clocks low for a while; idle, then warm up again.
        time.sleep(args.settle)
        for _ in range(max(args.warmup, 3)):
            step()
        torch.cuda.synchronize()

    stream = torch.cuda.current_stream(dev)

    def timed_steps(n):
        barrier()
        torch.cuda.synchronize()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(n):
            step()
        t1.record(stream)
        torch.cuda.synchronize()
        barrier()
        return t0.elapsed_time(t1)

    clocks = ClockSampler(local)
    with clocks:
        ms_local = timed_steps(args.steps)
    ms = max_over_ranks(ms_local)
    ms_per_step = ms / args.steps
    frames_total = wl.frames  # all ranks together
    value = frames_total / (ms_per_step / 1e3)

    # ---- validation of the last timed step (outside every timed region)
    validation = validate(c, world, rank, coll_dev)

    # ---- sustained: back-to-back steps for >= --sustain-s seconds (RL
    # training steps continuously; the board power limiter then lowers the
    # SM clock), with its own clock record
    sustained = None
    if args.sustain_s > 0:
        n_sus = max(args.steps, int(np.ceil(args.sustain_s / max(ms_per_step / 1e3, 1e-6))))
        sclk = ClockSampler(local)
        with sclk:
            ms_sus = max_over_ranks(timed_steps(n_sus))
        sustained = {"value": frames_total / (ms_sus / n_sus / 1e3), "ms_per_step": ms_sus / n_sus,
                     "steps": n_sus, "seconds": ms_sus / 1e3, "clocks": sclk.summary()}

    # ---- per-kernel durations (each kernel's own graph, replayed on the
    # current stream -- the stream its launches were captured from)
    def time_kernel(fn, n, segments=5):
        # median over `segments` back-to-back event-timed segments of n launches
        s = torch.cuda.current_stream(dev)
        per = []
        for _ in range(segments):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(s)
            for _ in range(n):
                fn()
            b.record(s)
            torch.cuda.synchronize()
            per.append(a.elapsed_time(b) / n)
        return float(np.median(per))

    nk = max(4, args.steps // 5)
    # Burst: each kernel timed alone from an idle GPU, the condition the
    # MEASURED_PEAKS copy bandwidth (best of 10 short copies) is taken in.
    # Under sustained full-HBM load the board's power limiter (sw_power_cap)
    # lowers the SM clock within ~0.1 s and these issue-heavy kernels slow
    # down; that regime is reported beside it (tools/k1_drift.py).
    time.sleep(1.0)
    kclocks = ClockSampler(local)
    with kclocks:
        k1_ms = time_kernel(k1_fn, nk, 3) if wl.rgb else None
        k2_ms = time_kernel(k2_fn, nk, 3) if wl.ff else None
        kf_ms = time_kernel(kf_fn, nk, 3) if arr.fused else None
    sclocks = ClockSampler(local)
    with sclocks:
        for _ in range(max(args.steps, 400)):
            step()
        k1_sus = time_kernel(k1_fn, nk, 3) if wl.rgb else None
        k2_sus = time_kernel(k2_fn, nk, 3) if wl.ff else None

    # ---- end to end through the host-buffer API
    def measure_e2e():
        host = arr.host_buffers(pinned=True)
        for k, v in (("depth", depth), ("obj", obj), ("sen", sen)):
            if host[k] is not None:
                host[k].copy_(v)

        if use_graph:  # the whole pipelined host-to-host step as one graph (SensorArray.capture_host)
            arr.capture_host(host, depth, obj, sen, chunks=args.e2e_chunks)
            e2e_step = arr.replay_host
        else:
            def e2e_step():
                arr.run_host(host, depth, obj, sen, chunks=args.e2e_chunks)

        for _ in range(2):  # warm: first-touch of the pinned pages, stream / event pools
            e2e_step()
        torch.cuda.synchronize()
        barrier()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.e2e_steps + 1)]
        ev[0].record(stream)
        for i in range(args.e2e_steps):
            e2e_step()
            ev[i + 1].record(stream)
        torch.cuda.synchronize()
        barrier()
        per_step = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.e2e_steps)]
        ms = max_over_ranks(ev[0].elapsed_time(ev[-1])) / args.e2e_steps
        h2d = sum(host[k].numel() * host[k].element_size() for k in ("depth", "obj", "sen")
                  if host[k] is not None) * world
        d2h = sum(v.numel() * v.element_size() for k, v in host.items()
                  if v is not None and k not in ("depth", "obj", "sen")) * world
        return {"value": frames_total / (ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "ms_per_step": ms,
                "step_ms_min_median_max": [min(per_step), float(np.median(per_step)), max(per_step)],
                "api": ("SensorArray.capture_host/replay_host" if use_graph else "SensorArray.run_host")
                       + ": pinned host depth+states in, pinned host RGB+forces+wrench out, "
                       f"{args.e2e_chunks} env chunks pipelined over H2D / kernels / D2H streams"
                       + (", one CUDA graph per step" if use_graph else "")}

    e2e = None if args.no_e2e else measure_e2e()

    # ---- end to end through the reference-signature numpy drop-ins (what a
    # gelsim user gets after patch(): float64 numpy in, float64 numpy out)
    def measure_dropin():
        from paper_2408_06506_b200 import render, tactile
        from paper_2408_06506_b200.render import DepthImage

        S, H, W = c.S, c.H, c.W
        envs = max(1, min(c.E, args.dropin_frames // S))
        F = envs * S
        g = np.arange(F) + c.lo * S
        depth64 = c.pool[g % len(c.pool)].astype(np.float64).reshape(envs, S, H, W) if wl.rgb else None
        objF = np.repeat(c.obj_all[c.lo:c.lo + envs], S, axis=0)
        senF = c.sen_all[c.lo:c.lo + envs].reshape(F, 13)

        def call():
            out = {}
            if wl.rgb:
                out["rgb"] = render.depth_to_rgb(DepthImage(values=depth64, background=c.bg), c.lut)
            if wl.ff:
                out["ff"] = tactile.compute_force_field(
                    c.pts, c.sdf, objF[:, 0:3], objF[:, 3:7], objF[:, 7:10], objF[:, 10:13],
                    senF[:, 0:3], senF[:, 3:7], senF[:, 7:10], senF[:, 10:13], c.params)
            return out

        out = None
        for _ in range(3):  # warm with the timed loop's pattern (the previous result alive during a call)
            out = call()
        reps = max(2, args.e2e_steps // 2)
        barrier()
        t0 = time.perf_counter()
        for _ in range(reps):
            out = call()
        secs = max_over_ranks(time.perf_counter() - t0) / reps
        h2d = (depth64.nbytes if wl.rgb else 0) + objF.nbytes + senF.nbytes
        d2h = (out["rgb"].nbytes if wl.rgb else 0) + (out["ff"].f_n.nbytes * 2 if wl.ff else 0)
        # the link's measured speed on this box (pinned, each direction alone)
        a = torch.empty(256 << 20, dtype=torch.uint8, pin_memory=True)
        dv = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        bw = {}
        for name, (dst, src) in (("h2d", (dv, a)), ("d2h", (a, dv))):
            dst.copy_(src, non_blocking=True)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(4):
                dst.copy_(src, non_blocking=True)
            e1.record()
            torch.cuda.synchronize()
            bw[name] = 4 * a.numel() / (e0.elapsed_time(e1) / 1e3)
        floor_s = max(h2d / bw["h2d"], d2h / bw["d2h"])  # copies in both directions overlapped
        return {"value": F * world / secs, "unit": UNIT, "frames_per_call": F * world, "s_per_call": secs,
                "h2d_bytes_per_step": int(h2d * world), "d2h_bytes_per_step": int(d2h * world),
                "link_gbs": {k: v / 1e9 for k, v in bw.items()},
                "pcie_floor_value": F * world / floor_s, "frac_of_pcie_floor": floor_s / secs,
                "api": "render.depth_to_rgb(DepthImage float64 numpy) + tactile.compute_force_field(numpy poses) "
                       "-> float64 numpy (the functions patch() binds into gelsim), wall clock per call pair"}

    e2e_dropin = None if (args.no_e2e or args.dropin_frames <= 0) else measure_dropin()

    # ---- roofline of the dominant kernel (K1, or K2 when the step has no RGB) and of the whole step
    peak, peak_src = hbm_peak()
    bytes_ = arr.algorithmic_bytes()
    step_gbs = bytes_["total"] / (ms_local / args.steps / 1e3) / 1e9
    if arr.fused:
        kname, kms, kbytes = "rgb_bulk_kernel_ff", kf_ms, bytes_["total"]
        desc = ("rgb_bulk_kernel<..., FF> (fused step: K1 depth->RGB shading warps + K2 force-field warps "
                "in one persistent launch)")
        rule = ("7 B/px (4 B fp32 depth read + 3 B uint8 RGB written) + 24 B/taxel fp32 f_n,f_t + "
                "208 B fp64 states + 48 B wrench per frame")
    elif wl.rgb and arr.levels == 1 and arr.sigma == 0:
        kname, kms, kbytes = "rgb_bulk_kernel", k1_ms, bytes_["rgb"]
        desc, rule = "rgb_bulk_kernel (K1 depth->RGB)", "7 B/px: 4 B fp32 depth read + 3 B uint8 RGB written"
    elif wl.rgb:
        kname, kms, kbytes = arr.image_kernel_name(), k1_ms, bytes_["rgb"]
        desc = arr.image_kernel_desc()
        rule = ("SURVEY.md 8d: 4 B fp32 depth read per level-0 pixel + 3 B uint8 RGB written per pixel of "
                "every pyramid level (intermediates are not algorithmic bytes)")
    else:
        kname, kms, kbytes = arr.ff_kernel_name(), k2_ms, bytes_["ff"]
        if kname == "force_field_quad_kernel":
            desc = ("force_field_quad_kernel (K2 force field + wrench: certified fp32 contact-mask pass, fp64 "
                    "contact path on a warp queue; timed with its taxel fp32-copy launch; issue-bound, HBM "
                    "fraction shown)")
        else:
            desc = ("force_field_fast_kernel (K2 force field + wrench; float64 / L2-gather-latency bound, "
                    "HBM fraction shown)")
        rule = "24 B/taxel fp32 f_n,f_t written + 208 B fp64 states read + 48 B wrench per frame"
    k_gbs = kbytes / (kms / 1e3) / 1e9
    traffic = traffic_from_profiles(f"{kname}/config{wl.config_id}/world{world}")

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32 (RGB) / f64 (force field)",
        "data": "synthetic (analytic spherical-indenter depth maps, analytic peg SDF, random peg poses)",
        "config": workload_config(wl, world),
        "e2e": e2e,
        "e2e_dropin": e2e_dropin,
        "value_sustained": sustained["value"] if sustained else None,
        "sustained": sustained,
        "roofline": {"bound": "hbm", "kernel": desc, "achieved": k_gbs,
                     "peak": peak, "unit": "GB/s", "frac": k_gbs / peak, "traffic": traffic,
                     "peak_source": peak_src, "kernel_ms": kms,
                     "algorithmic_bytes_per_launch": kbytes, "bytes_rule": rule,
                     "step_achieved_gbs": step_gbs, "step_frac": step_gbs / peak,
                     "k1_rgb_ms": k1_ms, "k1_rgb_frac": (bytes_["rgb"] / (k1_ms / 1e3) / 1e9 / peak
                                                         if k1_ms else None),
                     "k2_force_field_ms": k2_ms, "k2_bytes_per_launch": bytes_["ff"], "fused_ms": kf_ms,
                     "kernel_timing": "burst: each kernel alone after 1 s idle, median of 3 x "
                                      f"{nk} graph replays (clocks: kernel_clocks)",
                     "kernel_clocks": kclocks.summary(),
                     "sustained": {"k1_rgb_ms": k1_sus, "k2_force_field_ms": k2_sus,
                                   "k1_rgb_frac_of_burst_peak": (bytes_["rgb"] / (k1_sus / 1e3) / 1e9 / peak
                                                                 if k1_sus else None),
                                   "after_steps": max(args.steps, 400), "clocks": sclocks.summary()}},
        "gpu_launches": arr.launches_per_step * args.steps,
        "clocks": clocks.summary(),
        "graph": use_graph, "fused": arr.fused, "overlap": arr.overlap,
        "settle_s": args.settle,
    }
    if validation is not None:
        line["parity"] = validation["parity"]
        line["validation"] = validation["digest"]

    # ---- the other BASELINE configs on the same box, briefly (device-timed
    # value, dominant kernel vs the HBM peak, sampled-frame parity), so the
    # default run leaves evidence for every configuration
    if rank == 0 and world == 1 and args.also:
        other = {}
        for cid in [int(x) for x in args.also.split(",") if x.strip()]:
            if cid == wl.config_id:
                continue
            other[str(cid)] = run_other_config(cid, dev, args, peak)
        line["other_configs"] = other

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle.cpu_bench import CpuBaseline, cpu_model
        base = CpuBaseline(wl)
        n, dt = base.run(1)
        per_core_frame = dt  # one frame per core, in parallel
        fpc = max(1, min(int(args.cpu_seconds / max(per_core_frame, 1e-3)), wl.frames // base.cores))
        n, dt = base.run(fpc)
        base.close()
        # the 1-process figure beside it: one single-threaded worker
        one = CpuBaseline(wl, cores=1)
        n1, t1 = one.run(1)
        k1 = max(1, min(int(3.0 / max(t1, 1e-3)), 64))
        n1, t1 = one.run(k1)
        one.close()
        line["cpu_baseline"] = {
            "value": n / dt, "unit": UNIT, "cores": base.cores, "kind": "port",
            "sample": f"{n} sensor frames of config {wl.config_id} ({fpc} per core), numpy oracle "
                      f"restating gelsim depth_to_rgb+to_uint8+compute_force_field+net_wrench; {cpu_model()}",
            "single_process": {"value": n1 / t1, "unit": UNIT, "cores": 1,
                               "sample": f"{n1} sensor frames on one single-threaded worker"},
        }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
