"""mfa_eval_batch throughput on C3 (2^24 random points) per control-point layout."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2204_11762_b200 import Model, workloads as WL

w = WL.make_config(3, width=16, height=16)
u, v, ww = (torch.from_numpy(x).cuda() for x in WL.query_points(3, 1 << 24))
for layout in ("quads", "bezier"):
    m = Model.from_workload(w, layout=layout)
    out = m.eval(u, v, ww)
    for grad in (True, False):
        o = out if grad else out[:1]
        m.eval(u, v, ww, out=o, grad=grad)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            m.eval(u, v, ww, out=o, grad=grad)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"{layout:7s} grad={grad}: {ms:.3f} ms  {(1 << 24) / ms / 1e6:.2f} G pts/s")
    del m
