"""mfa_eval_hessian throughput (2^24 random points, value + gradient + Hessian,
binned) on the given workloads, default C3 and C5."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2204_11762_b200 import Model, workloads as WL

for c in [int(a) for a in sys.argv[1:]] or [3, 5]:
    w = WL.make_config(c, width=16, height=16)
    m = Model.from_workload(w)
    u, v, ww = (torch.from_numpy(x).cuda() for x in WL.query_points(c, 1 << 24))
    for _ in range(2):
        m.eval_hessian(u, v, ww)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        m.eval_hessian(u, v, ww)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"C{c} {m.info()['layout']:7s}: {ms:.3f} ms  {(1 << 24) / ms / 1e6:.2f} G pts/s (Hessian)")
    del m
