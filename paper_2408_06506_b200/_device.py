"""Device plumbing: torch owns device memory and streams; kernels come from
libtacsl_b200.so.  No CPU fallback -- every entry point requires a B200."""
from __future__ import annotations

import numpy as np

from . import _lib


def torch():
    import torch as _t  # local import keeps `import paper_2408_06506_b200` light

    return _t


_checked: dict = {}  # device index -> supported; availability checked once per process


def resolve_device(device=None):
    t = torch()
    if "available" not in _checked:  # torch.cuda.is_available() can cost tens of ms per call
        _checked["available"] = t.cuda.is_available()
    if not _checked["available"]:
        raise RuntimeError(
            "paper_2408_06506_b200 runs on a CUDA B200 (sm_100a) device only; "
            "torch.cuda.is_available() is False and there is no CPU fallback")
    if device is None:
        dev = t.device("cuda", t.cuda.current_device())
    else:
        dev = t.device(device)
        if dev.type != "cuda":
            raise RuntimeError(f"device {dev} is not a CUDA device; there is no CPU fallback")
        if dev.index is None:
            dev = t.device("cuda", t.cuda.current_device())
    ok = _checked.get(dev.index)
    if ok is None:
        ok = _checked[dev.index] = bool(_lib.load().tacsl_device_supported(dev.index))
    if not ok:
        raise RuntimeError(f"cuda:{dev.index} is not an sm_100 (B200) GPU; libtacsl_b200 has sm_100a code only")
    return dev


def is_cuda_tensor(x) -> bool:
    t = torch()
    return isinstance(x, t.Tensor) and x.is_cuda


def to_device(x, dtype, device):
    """numpy / python / torch -> contiguous torch tensor of `dtype` on `device`."""
    t = torch()
    if isinstance(x, t.Tensor):
        return x.to(device=device, dtype=dtype).contiguous()
    np_dtype = {t.float32: np.float32, t.float64: np.float64, t.uint8: np.uint8, t.int64: np.int64,
                t.int32: np.int32}[dtype]
    arr = np.ascontiguousarray(np.asarray(x, dtype=np_dtype))
    if not arr.flags.writeable:
        arr = arr.copy()
    return t.from_numpy(arr).to(device)


def stream_handle(device) -> int:
    return torch().cuda.current_stream(device).cuda_stream


def ptr(x) -> int | None:
    return None if x is None else x.data_ptr()


def as_f32(x, device):
    """numpy / torch float data -> contiguous float32 CUDA tensor on `device`.
    float64 input is uploaded as it is and narrowed ON THE DEVICE
    (tacsl_f64_to_f32, numpy's astype rounding), so the host never touches
    the values; other dtypes take the plain path."""
    t = torch()
    if isinstance(x, t.Tensor):
        if x.dtype == t.float32:
            return x.to(device=device).contiguous()
        if x.dtype != t.float64:
            return x.to(device=device, dtype=t.float32).contiguous()
        src = x.to(device=device).contiguous()
    else:
        arr = np.asarray(x)
        if arr.dtype != np.float64:
            return to_device(arr, t.float32, device)
        src = to_device(arr, t.float64, device)
    out = t.empty(src.shape, dtype=t.float32, device=device)
    _lib.check(_lib.load().tacsl_f64_to_f32(src.data_ptr(), src.numel(), out.data_ptr(), stream_handle(device)))
    return out


def widen_f64(x):
    """float32 CUDA tensor -> float64 CUDA tensor (tacsl_f32_to_f64)."""
    t = torch()
    out = t.empty(x.shape, dtype=t.float64, device=x.device)
    _lib.check(_lib.load().tacsl_f32_to_f64(x.data_ptr(), x.numel(), out.data_ptr(), stream_handle(x.device)))
    return out


# ---- host <-> device for the numpy drop-ins (pinned staging, pipelined)

def pinned_empty(shape, dtype):
    """A page-locked host tensor from torch's caching host allocator (blocks
    are reused across calls once the tensors that held them are freed)."""
    return torch().empty(tuple(shape), dtype=dtype, pin_memory=True)


def to_pinned(arr, dtype):
    """numpy -> page-locked host tensor of `dtype` (one host copy, which
    torch spreads over the host's threads), for full-speed DMA uploads."""
    t = torch()
    src = t.from_numpy(np.ascontiguousarray(arr))
    out = pinned_empty(src.shape, dtype)
    out.copy_(src)
    return out


def download(x):
    """CUDA tensor -> numpy array backed by page-locked memory (one DMA at
    the link's speed into the array the caller receives; no extra host copy)."""
    if x.numel() * x.element_size() < (1 << 20):  # small: a plain copy has the lower latency
        return x.cpu().numpy()
    out = pinned_empty(x.shape, x.dtype)
    out.copy_(x, non_blocking=True)
    torch().cuda.current_stream(x.device).synchronize()
    return out.numpy()


def pipelined(host_in, host_out, fn, device, chunk):
    """Run fn over the leading axis in chunks, overlapping the host copy of
    chunk i+1 (numpy -> page-locked staging, on the calling thread), chunk
    i's upload, chunk i-1's kernels and chunk i-2's download (three streams:
    the two copy engines + the SMs).  host_in: numpy arrays or page-locked
    tensors; host_out: page-locked tensors.  fn(dev_ins, dev_outs) enqueues
    its kernels on the current stream; device and staging buffers are double
    buffered."""
    t = torch()
    n = host_in[0].shape[0]
    main = t.cuda.current_stream(device)
    up, down = t.cuda.Stream(device=device), t.cuda.Stream(device=device)
    srcs = [h if isinstance(h, t.Tensor) else t.from_numpy(np.ascontiguousarray(h)) for h in host_in]
    staged = [not (isinstance(h, t.Tensor) and h.is_pinned()) for h in host_in]
    stage = [[pinned_empty((chunk,) + tuple(x.shape[1:]), x.dtype) if st else None for x, st in zip(srcs, staged)]
             for _ in range(2)]
    bufs = [([t.empty((chunk,) + tuple(x.shape[1:]), dtype=x.dtype, device=device) for x in srcs],
             [t.empty((chunk,) + tuple(h.shape[1:]), dtype=h.dtype, device=device) for h in host_out])
            for _ in range(2)]
    free = [None, None]      # event: buffer set b may be overwritten (its download finished)
    uploaded = [None, None]  # event: staging set b has been read by its upload
    up.wait_stream(main)
    for i, lo in enumerate(range(0, n, chunk)):
        hi = min(lo + chunk, n)
        b = i & 1
        ins, outs = bufs[b]
        if uploaded[b] is not None:
            uploaded[b].synchronize()  # the host may now refill staging set b
        for k, x in enumerate(srcs):
            if staged[k]:
                stage[b][k][:hi - lo].copy_(x[lo:hi])  # host copy, torch's threads
        with t.cuda.stream(up):
            if free[b] is not None:
                up.wait_event(free[b])
            for k, (d, x) in enumerate(zip(ins, srcs)):
                d[:hi - lo].copy_(stage[b][k][:hi - lo] if staged[k] else x[lo:hi], non_blocking=True)
            ev = t.cuda.Event()
            ev.record(up)
            uploaded[b] = ev
        main.wait_stream(up)
        fn([d[:hi - lo] for d in ins], [d[:hi - lo] for d in outs])
        down.wait_stream(main)
        with t.cuda.stream(down):
            for d, h in zip(outs, host_out):
                h[lo:hi].copy_(d[:hi - lo], non_blocking=True)
            ev = t.cuda.Event()
            ev.record(down)
            free[b] = ev
    main.wait_stream(down)
    main.synchronize()
