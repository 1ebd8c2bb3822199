"""Time mfa_fit_grid (256^3 Gaussian beam -> 128^3, p = 3) for ncu / timing."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2204_11762_b200 import fit_grid, workloads as WL

q = torch.from_numpy(WL.analytic_grid("gb", (256, 256, 256)).astype(np.float32)).cuda()
kn = [WL.clamped_uniform_knots(128, 3)] * 3
for i in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fit_grid(q, 3, kn)
    torch.cuda.synchronize()
    print(f"fit {i}: {1e3 * (time.perf_counter() - t0):.2f} ms")
