"""Diagnostic (build with MFA_EXTRA_NVCC_FLAGS=-DMFA_LANE_STATS=1): fraction of
lane-iterations of the sample loop whose ray is still live (ERT / chord-length
divergence inside warps)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2204_11762_b200 import Model, workloads as WL

for c, kw in ((5, dict(n_views=4)), (3, {}), (4, {})):
    w = WL.make_config(c, **kw)
    m = Model.from_workload(w)
    cnt = torch.zeros(3, dtype=torch.int64, device="cuda")
    m.render(w.cameras, torch.from_numpy(w.tf).cuda(), w.v_lo, w.v_hi, w.params, samples=cnt)
    torch.cuda.synchronize()
    s, slots, live = (int(x) for x in cnt.cpu())
    print(f"C{c}: samples {s}, lane slots {slots}, live {live}, live fraction {live / max(slots, 1):.3f}")
