"""mfa_eval_batch on C3 (2^24 random points): layouts x (direct, binned)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2204_11762_b200 import Model, workloads as WL

c = int(sys.argv[1]) if len(sys.argv) > 1 else 3
w = WL.make_config(c, width=16, height=16)
u, v, ww = (torch.from_numpy(x).cuda() for x in WL.query_points(c, 1 << 24))
for layout in ("quads", "bricks", "bezier"):
    try:
        m = Model.from_workload(w, layout=layout)
    except Exception as ex:
        print(layout, "n/a", ex)
        continue
    for binned in (False, "auto"):
        out = m.eval(u, v, ww, binned=binned)
        for _ in range(2):
            m.eval(u, v, ww, out=out, binned=binned)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            m.eval(u, v, ww, out=out, binned=binned)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(f"C{c} {layout:7s} binned={binned!s:5s}: {ms:.3f} ms  {(1 << 24) / ms / 1e6:.2f} G pts/s  "
              f"device {m.info()['device_bytes'] / 2**20:.0f} MiB", flush=True)
    del m
    torch.cuda.empty_cache()
