"""mfa_eval_hessian on C3 at 2^24 random points (for ncu)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2204_11762_b200 import Model, workloads as WL

w = WL.make_config(3, width=16, height=16)
m = Model.from_workload(w)
u, v, ww = (torch.from_numpy(x).cuda() for x in WL.query_points(3, 1 << 24))
m.eval_hessian(u, v, ww)
torch.cuda.synchronize()
print("ok")
