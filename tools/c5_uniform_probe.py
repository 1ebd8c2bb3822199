"""Diagnostic: render C5's grid and views with (a) its non-uniform knots and
(b) uniform knots, to isolate the cost of the non-uniform span path.
Round 2, 64 views: non-uniform Bezier 52.3 G, uniform Bezier 61.0 G, uniform
quads 63.5 G samples/s."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2204_11762_b200 import Model, workloads as WL

views = int(sys.argv[1]) if len(sys.argv) > 1 else 8
w = WL.make_config(5, n_views=views)
tf = torch.from_numpy(w.tf).cuda()
uknots = [WL.clamped_uniform_knots(n, w.degree) for n in w.nctrl]
for label, knots, layout in (("nonuniform", w.knots, "auto"), ("uniform", uknots, "auto"),
                             ("uniform", uknots, "bezier")):
    m = Model(w.degree, knots, w.ctrl, layout=layout)
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    for _ in range(2):
        m.render(w.cameras, tf, w.v_lo, w.v_hi, w.params, samples=cnt)
    torch.cuda.synchronize()
    cnt.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        m.render(w.cameras, tf, w.v_lo, w.v_hi, w.params, samples=cnt)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(f"{label:10s} ({m.info()['layout']}) {views} views: {ms:8.2f} ms  {cnt.item() / 3 / ms / 1e6:7.2f} G samples/s")
    del m
