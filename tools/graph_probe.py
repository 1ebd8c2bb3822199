"""CUDA-graph replay of small single-view renders (C1): per-frame device time
for eager calls and for graphs of 16 .. 2000 captured renders."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2204_11762_b200 import Model, workloads as WL

c = int(sys.argv[1]) if len(sys.argv) > 1 else 1
w = WL.make_config(c)
m = Model.from_workload(w)
tf = torch.from_numpy(w.tf).cuda()
V, H, W = len(w.cameras), w.cameras[0].height, w.cameras[0].width
img = torch.empty((V, H, W, 4), device="cuda")
cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
s = torch.cuda.Stream()


def render():
    m.render(w.cameras, tf, w.v_lo, w.v_hi, w.params, out=img, samples=cnt, stream=s)


with torch.cuda.stream(s):
    for _ in range(3):
        render()
torch.cuda.synchronize()
total = 4000
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(s)
with torch.cuda.stream(s):
    for _ in range(total):
        render()
e1.record(s)
torch.cuda.synchronize()
print(f"C{c} eager        : {e0.elapsed_time(e1) * 1e3 / total:7.2f} us per frame")
for n in (16, 64, 256, 2000):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(n):
            render()
    torch.cuda.synchronize()
    with torch.cuda.stream(s):
        g.replay()
    torch.cuda.synchronize()
    reps = max(1, total // n)
    e0.record(s)
    with torch.cuda.stream(s):
        for _ in range(reps):
            g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    print(f"C{c} graph x{n:5d}: {e0.elapsed_time(e1) * 1e3 / (reps * n):7.2f} us per frame")
    del g
