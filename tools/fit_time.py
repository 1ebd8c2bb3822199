"""Wall time of mfa_fit_grid at a few sizes (host + device), for the encoder's
fixed-overhead analysis.  python tools/fit_time.py [big]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2204_11762_b200 import fit_grid, workloads as WL

cases = (((256, 256, 256), 128), ((64, 64, 64), 32), ((16, 16, 16), 8))
if sys.argv[1:] == ["big"]:
    cases = cases[:1]
for dims, n in cases:
    q = torch.from_numpy(WL.analytic_grid("gb", dims).astype(np.float32)).cuda()
    kn = [WL.clamped_uniform_knots(n, 3)] * 3
    fit_grid(q, 3, kn)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        fit_grid(q, 3, kn)
    torch.cuda.synchronize()
    print(dims, n, f"{(time.perf_counter() - t0) / 10 * 1e3:.3f} ms wall")
