"""K1 launch time vs GPU power / clocks / temperature over a long run."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import pynvml  # noqa: E402
import torch  # noqa: E402

from paper_2408_06506_b200 import synthetic  # noqa: E402
from paper_2408_06506_b200.render import depth_to_rgb_device  # noqa: E402

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
_, cam, bg, lut, _ = synthetic.sensor_setup((320, 240))
pool = torch.from_numpy(synthetic.depth_batch(cam, bg, 64)).cuda()
d = pool[torch.arange(8192, device="cuda") % 64].contiguous()
u8 = torch.empty(d.shape + (3,), dtype=torch.uint8, device="cuda")
depth_to_rgb_device(d, lut, out_u8=u8)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    depth_to_rgb_device(d, lut, out_u8=u8)
for seg in range(int(sys.argv[1]) if len(sys.argv) > 1 else 30):
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(20):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 20
    pw = pynvml.nvmlDeviceGetPowerUsage(h) / 1000
    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    mem = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_MEM)
    t = pynvml.nvmlDeviceGetTemperature(h, pynvml.NVML_TEMPERATURE_GPU)
    try:
        tm = pynvml.nvmlDeviceGetFieldValues(h, [pynvml.NVML_FI_DEV_MEMORY_TEMP])[0].value.uiVal
    except Exception:  # noqa: BLE001
        tm = -1
    rs = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
    print(f"{seg:3d} {ms:.3f} ms  {pw:6.0f} W  sm {sm} MHz  mem {mem} MHz  gpu {t} C  hbm {tm} C  reasons 0x{rs:x}")
