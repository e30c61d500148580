"""Batched sensor step on one GPU: every (env, sensor) frame's tactile RGB,
force field and net wrench from device-resident inputs.

This is the multi-sensor caller of the two hot-path kernels -- the role of
``PegEnvBatch._tactile_images`` / ``_tactile_ff`` (envs/peg_tasks.py:434-477)
without their per-sensor Python loops: K1 runs once over all E*S depth maps
and K2 once over all E*S force fields.  The two launches go to two streams so
K2 fills the SMs K1's tail leaves idle; ``capture()`` records the pair in a
CUDA graph so a step costs one graph launch, and ``capture_host()`` records
a whole pipelined host-to-host step the same way.
"""
from __future__ import annotations

import numpy as np

from . import _device, smoothing, tactile
from .geometry import device_sdf
from .render import depth_to_rgb_device, device_lut
from .tactile import device_taxels, force_field_device


class SensorArray:
    def __init__(self, lut, sdf, points, params, n_envs, n_sensors=1, device=None, ff_fp64=False,
                 rgb_u8=True, rgb_f32=False, overlap=True, with_ff=True, fused=False, pyramid_levels=1,
                 smooth_sigma=0.0):
        t = _device.torch()
        self.device = _device.resolve_device(device)
        self.lut = device_lut(lut)
        self.sdf = device_sdf(sdf, self.device)
        self.taxels = device_taxels(points, self.device)
        self.rows, self.cols = int(points.rows), int(points.cols)
        self.params = params
        self.E, self.S = int(n_envs), int(n_sensors)
        W, H = self.lut.image_size
        self.H, self.W = H, W
        dev = self.device
        F = self.E * self.S
        self.rgb_u8 = t.empty((self.E, self.S, H, W, 3), dtype=t.uint8, device=dev) if rgb_u8 else None
        self.rgb_f32 = t.empty((self.E, self.S, H, W, 3), dtype=t.float32, device=dev) if rgb_f32 else None
        ff_dtype = t.float64 if ff_fp64 else t.float32
        self.with_rgb = rgb_u8 or rgb_f32
        self.with_ff = with_ff
        if with_ff:
            self.f_n = t.empty((self.E, self.S, self.rows, self.cols, 3), dtype=ff_dtype, device=dev)
            self.f_t = t.empty_like(self.f_n)
            self.wrench = t.empty((self.E, self.S, 6), dtype=t.float64, device=dev)
        else:
            self.f_n = self.f_t = self.wrench = None
        # optional image pipeline around K1 (north_star stages without a
        # reference counterpart, smoothing.py): Gaussian smoothing of the
        # depth (K5), then pyramid levels l >= 1 = K5 pyr_down + K1 with the
        # level's LUT, each into its own uint8 RGB buffer
        self.levels = max(1, int(pyramid_levels)) if self.with_rgb else 1
        self.sigma = float(smooth_sigma) if self.with_rgb else 0.0
        # K7: smoothing + every pyramid level's RGB in one pass over the
        # depth (no intermediate in HBM) whenever the shape allows it;
        # otherwise the level-by-level chain (K5 + K1 per level)
        self.fused_pyramid = bool(self.with_rgb and rgb_u8 and not rgb_f32 and (self.levels > 1 or self.sigma > 0)
                                  and smoothing.fused_pyramid_supported(H, W, self.levels, self.sigma))
        chain = not self.fused_pyramid  # the intermediates exist only for the level-by-level chain
        self._smooth = (t.empty((self.E, self.S, H, W), dtype=t.float32, device=dev)
                        if self.sigma > 0 and chain else None)
        self._taps = smoothing.gaussian_taps(self.sigma) if self.sigma > 0 else None
        self.rgb_levels = [self.rgb_u8]
        self._lvl_depth = [None]
        self._lvl_luts = [self.lut]
        h, w = H, W
        for lvl in range(1, self.levels):
            h, w = -(-h // 2), -(-w // 2)
            self._lvl_depth.append(t.empty((self.E, self.S, h, w), dtype=t.float32, device=dev) if chain else None)
            self.rgb_levels.append(t.empty((self.E, self.S, h, w, 3), dtype=t.uint8, device=dev))
            self._lvl_luts.append(device_lut(smoothing.level_lut(lut, lvl)))
        # one fused launch (force-field warps beside the shading warps) when
        # the step is uint8 RGB + float32 force field
        self.fused = bool(fused and rgb_u8 and not rgb_f32 and with_ff and not ff_fp64 and self.levels == 1
                          and self.sigma == 0)
        self.overlap = overlap and self.with_rgb and with_ff and not self.fused
        rgb_launches = (1 + int(self.sigma > 0) + 2 * (self.levels - 1)) if self.with_rgb else 0
        if self.fused_pyramid:
            rgb_launches = 1
        ff_launches = tactile.force_field_launches(self.rows, self.cols) if with_ff else 0
        self.launches_per_step = 1 if self.fused else rgb_launches + ff_launches
        self._workspace = t.zeros(1, dtype=t.int64, device=dev) if self.fused else None
        self._ff_stream = t.cuda.Stream(device=dev) if overlap else None
        self._graph = None
        self._graph_inputs = None
        assert F > 0

    # bytes the step must move through HBM (our exact layout):
    # the fp32 depth read once, every output byte written once; smoothed and
    # decimated intermediates are not algorithmic bytes (a fused pipeline
    # never writes them)
    def algorithmic_bytes(self) -> dict:
        px = self.H * self.W
        rgb_out = (3 if self.rgb_u8 is not None else 0) + (12 if self.rgb_f32 is not None else 0)
        F = self.E * self.S
        rgb = F * px * (4 + rgb_out) if self.with_rgb else 0
        for lvl in range(1, self.levels):
            h, w = self.rgb_levels[lvl].shape[2:4]
            rgb += F * h * w * 3  # level l's uint8 RGB
        ff = 0
        if self.with_ff:
            taxel_out = self.rows * self.cols * 3 * self.f_n.element_size() * 2
            ff = F * (taxel_out + 13 * 8 + 6 * 8) + self.E * 13 * 8
        return {"rgb": rgb, "ff": ff, "total": rgb + ff}

    def ff_kernel_name(self) -> str:
        """The K2 variant a step launches (csrc/force_field.cu)."""
        return ("force_field_quad_kernel" if tactile.force_field_launches(self.rows, self.cols) == 2
                else "force_field_fast_kernel")

    def image_kernel_name(self) -> str:
        return "pyramid_fused_kernel" if self.fused_pyramid else "image_pipeline"

    def image_kernel_desc(self) -> str:
        if self.fused_pyramid:
            return ("pyramid_fused_kernel (K7: Gaussian smoothing + RGB of every pyramid level in one pass; "
                    "only the depth is read and the uint8 RGB written)")
        return ("image pipeline: sep_bulk_kernel smoothing + rgb_bulk_kernel, then per pyramid level "
                "sep_bulk_kernel pyr_down + rgb_bulk_kernel (all launches of the RGB side)")

    def launch(self, depth, obj_state, sen_state):
        """Enqueue one step on the current stream (K2 on a forked stream that
        joins back before returning)."""
        t = _device.torch()
        main = t.cuda.current_stream(self.device)
        if self.fused:
            self._launch_fused(depth, obj_state, sen_state)
        elif self.overlap:
            self._ff_stream.wait_stream(main)
            with t.cuda.stream(self._ff_stream):
                self._launch_ff(obj_state, sen_state)
            self._launch_rgb(depth)
            main.wait_stream(self._ff_stream)
        else:
            if self.with_rgb:
                self._launch_rgb(depth)
            if self.with_ff:
                self._launch_ff(obj_state, sen_state)

    def _launch_fused(self, depth, obj_state, sen_state, lo=0, hi=None):
        from . import _lib
        hi = self.E if hi is None else hi
        E = hi - lo
        d = depth[lo:hi]
        lib = _lib.load()
        _lib.check(lib.tacsl_sensor_step(
            self.lut.handle, d.data_ptr(), E * self.S, self.H, self.W, self.rgb_u8[lo:hi].data_ptr(),
            self.sdf.handle, self.taxels.data_ptr(), self.rows, self.cols, obj_state[lo:hi].data_ptr(), 13,
            sen_state[lo:hi].data_ptr(), 13 * self.S, E, self.S, _lib.penalty(self.params),
            self.f_n[lo:hi].data_ptr(), self.f_t[lo:hi].data_ptr(), self.wrench[lo:hi].data_ptr(),
            self._workspace.data_ptr(), _device.stream_handle(self.device)))

    def _launch_rgb(self, depth, lo=0, hi=None):
        hi = self.E if hi is None else hi
        sl = slice(lo, hi)
        d = depth[sl]
        if self.fused_pyramid:
            smoothing.rgb_pyramid_fused_device(d, self.lut, self.levels, self.sigma,
                                               outs=[self.rgb_levels[lvl][sl] for lvl in range(self.levels)],
                                               luts=self._lvl_luts)
            return
        if self._smooth is not None:
            d = smoothing.separable_filter_device(d, self._taps, 1, out=self._smooth[sl])
        if self.levels == 1:
            depth_to_rgb_device(d, self.lut, out_u8=None if self.rgb_u8 is None else self.rgb_u8[sl],
                                out_f32=None if self.rgb_f32 is None else self.rgb_f32[sl])
            return
        # pyramid: level l's shading (current stream) overlaps the next
        # level's decimation (side stream); both only read level l's depth
        t = _device.torch()
        main = t.cuda.current_stream(self.device)
        if getattr(self, "_pyr_stream", None) is None:
            self._pyr_stream = t.cuda.Stream(device=self.device)
        side = self._pyr_stream
        luts = self._lvl_luts
        for lvl in range(self.levels):
            nxt = None
            if lvl + 1 < self.levels:
                side.wait_stream(main)  # level lvl's depth is ready
                with t.cuda.stream(side):
                    nxt = smoothing.pyr_down_device(d, out=self._lvl_depth[lvl + 1][sl])
            if lvl == 0:
                depth_to_rgb_device(d, luts[0], out_u8=None if self.rgb_u8 is None else self.rgb_u8[sl],
                                    out_f32=None if self.rgb_f32 is None else self.rgb_f32[sl])
            else:
                depth_to_rgb_device(d, luts[lvl], out_u8=self.rgb_levels[lvl][sl])
            if nxt is not None:
                main.wait_stream(side)
                d = nxt

    def _launch_ff(self, obj_state, sen_state):
        force_field_device(self.sdf, self.taxels, self.rows, self.cols, obj_state, sen_state, self.params,
                           self.f_n, self.f_t, wrench=self.wrench, n_sensors=self.S,
                           obj_stride=13, sen_stride=13 * self.S)

    def capture(self, depth, obj_state, sen_state):
        """Record launch(depth, obj_state, sen_state) in a CUDA graph bound to
        these input tensors; replay() then re-runs it with their current
        contents."""
        t = _device.torch()
        s = t.cuda.Stream(device=self.device)
        s.wait_stream(t.cuda.current_stream(self.device))
        with t.cuda.stream(s):
            self.launch(depth, obj_state, sen_state)  # warm-up outside capture (kernel attrs, lazy init)
        t.cuda.current_stream(self.device).wait_stream(s)
        t.cuda.synchronize(self.device)
        g = t.cuda.CUDAGraph()
        with t.cuda.graph(g):
            self.launch(depth, obj_state, sen_state)
        self._graph = g
        self._graph_inputs = (depth, obj_state, sen_state)
        return g

    def replay(self):
        self._graph.replay()

    def step(self, depth, obj_state, sen_state):
        if self._graph is not None and all(a is b for a, b in zip(self._graph_inputs,
                                                                   (depth, obj_state, sen_state))):
            self.replay()  # the graph reads the captured tensors: replay only for those very inputs
        else:
            self.launch(depth, obj_state, sen_state)
        return self.rgb_u8 if self.rgb_u8 is not None else self.rgb_f32, self.f_n, self.f_t, self.wrench

    def outputs(self):
        """(name, device tensor) of every output of a step, in a fixed order."""
        outs = [("rgb", self.rgb_u8), ("rgb_f32", self.rgb_f32)]
        outs += [(f"rgb_l{lvl}", self.rgb_levels[lvl]) for lvl in range(1, self.levels)]
        outs += [("f_n", self.f_n), ("f_t", self.f_t), ("wrench", self.wrench)]
        return [(k, v) for k, v in outs if v is not None]

    def frame_digests(self):
        return frame_digests(self.outputs())

    def host_buffers(self, pinned=True):
        """Pinned host mirrors of the step's inputs and outputs."""
        t = _device.torch()

        def like(shape, dtype):
            return t.empty(shape, dtype=dtype, pin_memory=pinned)

        W, H = self.W, self.H
        ff = self.with_ff
        return {
            "depth": like((self.E, self.S, H, W), t.float32) if self.with_rgb else None,
            "obj": like((self.E, 13), t.float64) if ff else None,
            "sen": like((self.E, self.S, 13), t.float64) if ff else None,
            "rgb": like(tuple(self.rgb_u8.shape), t.uint8) if self.rgb_u8 is not None else None,
            "f_n": like(tuple(self.f_n.shape), self.f_n.dtype) if ff else None,
            "f_t": like(tuple(self.f_t.shape), self.f_t.dtype) if ff else None,
            "wrench": like(tuple(self.wrench.shape), t.float64) if ff else None,
            **{f"rgb_l{lvl}": like(tuple(self.rgb_levels[lvl].shape), t.uint8) for lvl in range(1, self.levels)},
        }

    def run_host(self, host, depth, obj_state, sen_state, chunks=8):
        """One step from pinned HOST inputs to pinned HOST outputs.

        The env axis is cut into `chunks`; chunk i's host->device copy, chunk
        i-1's kernels and chunk i-2's device->host copy run concurrently on
        three streams (two copy engines + the SMs), so a step costs about the
        larger of the two PCIe directions rather than their sum.  `depth`,
        `obj_state`, `sen_state` are the device staging tensors.
        """
        t = _device.torch()
        dev = self.device
        if not hasattr(self, "_h2d"):
            self._h2d = t.cuda.Stream(device=dev)
            self._d2h = t.cuda.Stream(device=dev)
        main = t.cuda.current_stream(dev)
        self._h2d.wait_stream(main)
        bounds = [shard_range(self.E, i, chunks) for i in range(chunks)]
        bounds = [(lo, hi) for lo, hi in bounds if hi > lo]
        outs = [("rgb", self.rgb_u8), ("f_n", self.f_n), ("f_t", self.f_t), ("wrench", self.wrench)]
        outs += [(f"rgb_l{lvl}", self.rgb_levels[lvl]) for lvl in range(1, self.levels)]
        for lo, hi in bounds:
            with t.cuda.stream(self._h2d):
                if self.with_rgb:
                    depth[lo:hi].copy_(host["depth"][lo:hi], non_blocking=True)
                if self.with_ff:
                    obj_state[lo:hi].copy_(host["obj"][lo:hi], non_blocking=True)
                    sen_state[lo:hi].copy_(host["sen"][lo:hi], non_blocking=True)
            main.wait_stream(self._h2d)
            if self.fused:
                self._launch_fused(depth, obj_state, sen_state, lo, hi)
            elif self.with_rgb:
                self._launch_rgb(depth, lo, hi)
            if self.with_ff and not self.fused:
                force_field_device(self.sdf, self.taxels, self.rows, self.cols, obj_state[lo:hi],
                                   sen_state[lo:hi], self.params, self.f_n[lo:hi], self.f_t[lo:hi],
                                   wrench=self.wrench[lo:hi], n_sensors=self.S, obj_stride=13,
                                   sen_stride=13 * self.S)
            self._d2h.wait_stream(main)
            with t.cuda.stream(self._d2h):
                for name, dev_t in outs:
                    if dev_t is not None and host.get(name) is not None:
                        host[name][lo:hi].copy_(dev_t[lo:hi], non_blocking=True)
        main.wait_stream(self._d2h)
        return host

    def capture_host(self, host, depth, obj_state, sen_state, chunks=8):
        """Record run_host(...) -- every chunk's copies and kernels on the
        three streams -- as one CUDA graph bound to these host and device
        buffers; replay_host() then runs a whole host-to-host step with one
        launch and no per-chunk host work."""
        t = _device.torch()
        s = t.cuda.Stream(device=self.device)
        s.wait_stream(t.cuda.current_stream(self.device))
        with t.cuda.stream(s):
            self.run_host(host, depth, obj_state, sen_state, chunks)  # warm-up outside capture
        t.cuda.current_stream(self.device).wait_stream(s)
        t.cuda.synchronize(self.device)
        g = t.cuda.CUDAGraph()
        with t.cuda.graph(g):
            self.run_host(host, depth, obj_state, sen_state, chunks)
        self._host_graph = g
        return g

    def replay_host(self):
        self._host_graph.replay()


class TactileObservations:
    """Batched tactile observations of the 2-finger peg env from given depth
    maps and states: the outputs of ``PegEnvBatch._tactile_images``
    (envs/peg_tasks.py:434-459, with the optional per-(env, episode, step)
    augmentation) and ``_tactile_ff`` (peg_tasks.py:461-477) for all E envs x
    S sensors, with no per-sensor Python loop.  (``envs.tactile_images``
    also renders the depth maps from the env's poses.)

    images: (E, S, H, W, 3) float32 ("color" / "diff") or (E, S, H, W, 6)
    ("concat"); ff: (E, S, R, C, 3) float32 = [f_n.z, f_t.x, f_t.y] in each
    sensor's frame.
    """

    def __init__(self, lut, sdf, points, params, n_envs, n_sensors=2, tactile_rep="color", device=None,
                 augment=None):
        t = _device.torch()
        self.augment_cfg = augment
        self.device = _device.resolve_device(device)
        self.lut = lut
        self.sdf = device_sdf(sdf, self.device)
        self.taxels = device_taxels(points, self.device)
        self.rows, self.cols = int(points.rows), int(points.cols)
        self.params = params
        self.E, self.S = int(n_envs), int(n_sensors)
        self.rep = tactile_rep
        W, H = (int(v) for v in lut.image_size)
        ch = 6 if tactile_rep == "concat" else 3
        self.images = t.empty((self.E, self.S, H, W, ch), dtype=t.float32, device=self.device)
        self.ff = t.empty((self.E, self.S, self.rows, self.cols, 3), dtype=t.float32, device=self.device)

        if augment is not None:
            self._rgb = t.empty((self.E, self.S, H, W, 3), dtype=t.float32, device=self.device)
            self._nominal = np.asarray(lut.coeffs, dtype=np.float64)[:, 0].astype(np.float32)

    def __call__(self, depth, obj_state, sen_state, episode_seeds=None, step_indices=None):
        """episode_seeds / step_indices: per-env int64 (the env's
        int(env_seed * 1000003 + episode) and step_count, peg_tasks.py:449-450),
        required when an AugmentConfig was given."""
        from .render import tactile_image_obs_device

        if self.augment_cfg is None:
            tactile_image_obs_device(depth, self.lut, self.rep, out=self.images)
        else:
            from .augment import augment_device

            t = _device.torch()
            if episode_seeds is None or step_indices is None:
                raise ValueError("augmentation needs per-env episode seeds and step indices")
            tactile_image_obs_device(depth, self.lut, "color", out=self._rgb)
            seeds = _device.to_device(episode_seeds, t.int64, self.device).reshape(self.E, 1)
            steps = _device.to_device(step_indices, t.int64, self.device).reshape(self.E, 1)
            augment_device(self._rgb, self.augment_cfg, seeds.expand(self.E, self.S).contiguous(),
                           steps.expand(self.E, self.S).contiguous(), tactile_rep=self.rep,
                           nominal=self._nominal, out=self.images)
        force_field_device(self.sdf, self.taxels, self.rows, self.cols, obj_state, sen_state, self.params,
                           obs=self.ff, n_sensors=self.S, obj_stride=13, sen_stride=13 * self.S, n_envs=self.E)
        return self.images, self.ff


def shard_range(n_envs: int, rank: int, world: int):
    """Contiguous env shard [lo, hi) of `rank`."""
    base, rem = divmod(n_envs, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def frame_digests(outputs):
    """Per-frame 64-bit digests (tacsl_frame_digest) of a step's outputs.

    outputs: list of (name, tensor) with tensors of shape (E, S, ...) on the
    device (None entries are skipped).  Returns (names, (E*S, k) int64 CUDA
    tensor): column j is the digest of frame f of output j -- position
    dependent, and the same for a frame whichever rank or batch computed it,
    so the concatenation over ranks in env order is the N=1 list."""
    from . import _lib

    t = _device.torch()
    names, cols = [], []
    for name, x in outputs:
        if x is None:
            continue
        n = int(x.shape[0]) * int(x.shape[1])
        if not x.is_contiguous():
            x = x.contiguous()
        fb = x.numel() // max(n, 1) * x.element_size()
        out = t.empty(n, dtype=t.int64, device=x.device)
        _lib.check(_lib.load().tacsl_frame_digest(x.data_ptr(), n, fb, out.data_ptr(),
                                                  _device.stream_handle(x.device)))
        names.append(name)
        cols.append(out)
    return names, t.stack(cols, dim=1) if cols else None
