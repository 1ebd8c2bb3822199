"""Render a config a few times (for ncu).  python tools/profile_render.py c3 [--views N] [--reps R]"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2204_11762_b200 import Model, workloads as WL

ap = argparse.ArgumentParser()
ap.add_argument("workload")
ap.add_argument("--views", type=int, default=None)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--eval", action="store_true", help="profile mfa_eval_batch on 2^24 points instead")
ap.add_argument("--uniform-knots", action="store_true", help="diagnostic: replace the knots by uniform ones")
ap.add_argument("--layout", default="auto")
a = ap.parse_args()
c = int(a.workload[1:])
w = WL.make_config(c, **({"n_views": a.views} if a.views else {}))
if a.uniform_knots:
    w.knots = [WL.clamped_uniform_knots(n, w.degree) for n in w.nctrl]
m = Model.from_workload(w, layout=a.layout)
if a.eval:
    u, v, ww = (torch.from_numpy(x).cuda() for x in WL.query_points(c, 1 << 24))
    for _ in range(a.reps):
        m.eval(u, v, ww)
else:
    tf = torch.from_numpy(w.tf).cuda()
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    for _ in range(a.reps):
        img = m.render(w.cameras, tf, w.v_lo, w.v_hi, w.params, samples=cnt)
torch.cuda.synchronize()
print("ok", int(cnt.item()) if not a.eval else "")
