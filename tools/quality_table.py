"""The paper's quality protocol end to end on the GPU (§4.2.1, Tables
1-2, MFA-DVR column only): a discrete Marschner-Lobb dataset
is ENCODED into an MFA (mfa_fit_grid, least squares, NEXT-3), rendered
(mfa_render_ex) and scored against the analytic ground truth along the same
rays (mfa_render_field) with MSE / PSNR / SSIM (mfa_image_quality, NEXT-2),
for the gradient-only test and the overall test.

    python tools/quality_table.py [--size 512] [--data 64 128] [--degrees 2 3]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2204_11762_b200 import Model, fit_grid, image_quality, workloads as WL

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=512)
ap.add_argument("--data", type=int, nargs="+", default=[64, 128])
ap.add_argument("--degrees", type=int, nargs="+", default=[2, 3])
ap.add_argument("--ratio", type=float, nargs="+", default=[0.25, 0.5, 0.9], help="control points per data point per axis")
a = ap.parse_args()

print("data  p  nctrl  test      MSE       PSNR(dB)  SSIM     render G samples/s (MFA image, device time)")
for m in a.data:
    q = torch.from_numpy(WL.analytic_grid("ml", (m, m, m)).astype(np.float32)).cuda()
    for p in a.degrees:
        for r in a.ratio:
            n = max(p + 1, int(round(r * m)))
            knots = [WL.clamped_uniform_knots(n, p)] * 3
            try:
                ctrl = fit_grid(q, p, knots)
            except Exception as ex:   # e.g. an ill-posed square system (the fit reports it)
                print(f"{m:4d}^3 {p}  {n:4d}^3 fit failed: {ex}")
                continue
            for test in ("gradient", "overall"):
                # geometry, TF and camera of the quality workload (step opacity, white, shading on)
                w, f_mfa, f_true = WL.make_quality("ml", 8, 3, test, a.size, a.size)
                spans = n - p
                L, bmin, bmax = WL._box((spans,) * 3)
                w.params.box_min, w.params.box_max = bmin, bmax
                w.params.step = 0.5 / spans
                w.v_lo, w.v_hi = 0.0, 1.0
                model = Model(p, knots, ctrl)
                tf = torch.from_numpy(w.tf).cuda()
                img = model.render(w.cameras, tf, w.v_lo, w.v_hi, w.params, field=f_mfa)
                tru = model.render(w.cameras, tf, w.v_lo, w.v_hi, w.params, field=f_true)
                res = image_quality(img[0], tru[0])
                # per-sample query cost (Fig. 12 methodology): the plain MFA render
                cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                model.render(w.cameras, tf, w.v_lo, w.v_hi, w.params, out=img)
                e0.record()
                for _ in range(5):
                    model.render(w.cameras, tf, w.v_lo, w.v_hi, w.params, out=img, samples=cnt)
                e1.record()
                torch.cuda.synchronize()
                rate = int(cnt.item()) / (e0.elapsed_time(e1) / 1e3) / 1e9
                print(f"{m:4d}^3 {p}  {n:4d}^3 {test:9s} {res['mse']:9.2f} {res['psnr']:9.2f} {res['ssim']:7.4f}  {rate:6.2f}")
                del model
