"""Diagnostic (build with MFA_EXTRA_NVCC_FLAGS=-DMFA_DIAG_MULTICOUNT=1): how often
a ray step crosses more than one knot span on C5 (lane-samples and
warp-iterations of the flat sample loop)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2204_11762_b200 import Model, workloads as WL

w = WL.make_config(5, n_views=4)
m = Model.from_workload(w)
cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
m.render(w.cameras, torch.from_numpy(w.tf).cuda(), w.v_lo, w.v_hi, w.params, samples=cnt)
torch.cuda.synchronize()
s, ml, mw, it = (int(x) for x in cnt.cpu())
print(f"C5 4 views: samples {s}, multi-span lane-samples {ml} ({ml / max(s, 1):.4f}), "
      f"warp-iterations {it}, with any multi-span lane {mw} ({mw / max(it, 1):.4f})")
