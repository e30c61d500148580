import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import bench
from paper_2408_06506_b200 import synthetic
dev = torch.device("cuda", 0)
c = bench.setup_workload(synthetic.CONFIGS[4], 0, 1, dev)
arr = c.arr
def eager(n):
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(n): arr._launch_ff(c.obj, c.sen)
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b) / n
for _ in range(3): arr._launch_ff(c.obj, c.sen)
torch.cuda.synchronize()
print("eager", eager(5), eager(5))
g = torch.cuda.CUDAGraph()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    with torch.cuda.graph(g, stream=s):
        for _ in range(5): arr._launch_ff(c.obj, c.sen)
torch.cuda.synchronize()
g.replay(); torch.cuda.synchronize()
a, b = torch.cuda.Event(True), torch.cuda.Event(True)
a.record(); g.replay(); b.record(); torch.cuda.synchronize()
print("graph", a.elapsed_time(b) / 5)
print("contact frac", float((arr.f_n.abs().sum(-1) > 0).float().mean()))
