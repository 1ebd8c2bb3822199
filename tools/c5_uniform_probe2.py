"""C5's grid and views with uniform knots (same Bezier layout): the cost of
the non-uniform span tracking, as an upper bound on what cheaper tracking
could gain (round 2)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2204_11762_b200 import Model, workloads as WL

w = WL.make_config(5)
res = {}
for kind in ("nonuniform", "uniform"):
    if kind == "uniform":
        w.knots = [WL.clamped_uniform_knots(n, w.degree) for n in w.nctrl]
        w.uniform = True
    m = Model.from_workload(w)
    tf = torch.from_numpy(w.tf).cuda()
    img = torch.empty((len(w.cameras), w.cameras[0].height, w.cameras[0].width, 4), device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    for _ in range(2):
        m.render(w.cameras, tf, w.v_lo, w.v_hi, w.params, out=img, samples=cnt)
    torch.cuda.synchronize()
    cnt.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        m.render(w.cameras, tf, w.v_lo, w.v_hi, w.params, out=img, samples=cnt)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"C5 {kind:10s} ({m.info()['layout']}): {int(cnt.item()) / 3 / (ms / 1e3) / 1e9:.2f} G samples/s, {ms:.1f} ms", flush=True)
    del m, img
    torch.cuda.empty_cache()
