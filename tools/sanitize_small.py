"""Small end-to-end workload for compute-sanitizer: eval + render on C1/C2 in
both layouts, C5 (non-uniform, Bezier) at a reduced image, tiled render."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import dataclasses

import numpy as np
import torch

from paper_2204_11762_b200 import Model, unpack_tiles, workloads as WL

for c, kw in ((1, {}), (2, dict(width=96, height=64)), (5, dict(width=64, height=48, n_views=2))):
    w = WL.make_config(c, **kw)
    for layout in ("quads", "bezier", "bricks") + (("bezier_grouped",) if w.degree == 3 else ()):
        m = Model.from_workload(w, layout=layout)
        u, v, ww = (torch.from_numpy(x).cuda() for x in WL.query_points(c, 4096))
        m.eval(u, v, ww)
        m.eval(u, v, ww, grad=False)
        tf = torch.from_numpy(w.tf).cuda()
        img = m.render(w.cameras, tf, w.v_lo, w.v_hi, w.params)
        tiles = torch.tensor([[0, 0, 0], [len(w.cameras) - 1, 1, 1], [-1, -1, -1]], dtype=torch.int32).cuda()
        packed = m.render(w.cameras, tf, w.v_lo, w.v_hi, w.params, tiles=tiles, out_fp16=True)
        unpack_tiles(packed, tiles, len(w.cameras), w.cameras[0].width, w.cameras[0].height)
        torch.cuda.synchronize()
        for shading in (0, 2, 3):   # value only, gradient skip, transparent-block skip
            m.render(w.cameras, tf, w.v_lo, w.v_hi, dataclasses.replace(w.params, shading=shading))
        torch.cuda.synchronize()
        print(c, layout, "ok", float(img.sum()))

# the other entry points: binned eval (>= 2^16 points) and Hessian, the
# extended render (lights, curvature table, analytic field), image metrics,
# least-squares fit and the adaptive encoder
from paper_2204_11762_b200 import encode_grid, fit_grid, image_quality  # noqa: E402

w = WL.make_config(2, width=96, height=64)
for layout in ("quads", "bezier", "bezier_grouped"):
    m = Model.from_workload(w, layout=layout)
    u, v, ww = (torch.from_numpy(x).cuda() for x in WL.query_points(2, 1 << 16))
    m.eval(u, v, ww, binned=True)
    m.eval_hessian(u, v, ww, binned=True)
    m.eval_hessian(u[:999], v[:999], ww[:999], binned=False)
    tf = torch.from_numpy(w.tf).cuda()
    a = m.render(w.cameras, tf, w.v_lo, w.v_hi, w.params, lights=[((1.0, 0.5, 0.2), 0.7), ((0.0, -1.0, 0.3), 0.4)])
    tab = torch.rand((9, 9, 4), device="cuda")
    b = m.render(w.cameras, tf, w.v_lo, w.v_hi, w.params, curvature=(tab, 30.0))
    c = m.render(w.cameras, tf, w.v_lo, w.v_hi, w.params, field=WL.AnalyticField.gaussian_beam(1, 1))
    q = image_quality(a[0], c[0], err_map=True)
    torch.cuda.synchronize()
    print("next", layout, "ok", q["psnr"], float(b.sum()))
g = torch.from_numpy(WL.analytic_grid("gb", (40, 36, 32)).astype(np.float32)).cuda()
fit_grid(g, 3, [WL.clamped_uniform_knots(n, 3) for n in (12, 11, 10)])
encode_grid(g, 2, (4, 4, 4), 1e-3, 3, (20, 20, 20))
torch.cuda.synchronize()
print("fit/encode ok")

# host-buffer renders (model-owned staging) and the IPC image buffer
from paper_2204_11762_b200._lib import IpcBuffer  # noqa: E402

w = WL.make_config(2, width=80, height=48, n_views=3)
m = Model.from_workload(w)
H, W = w.cameras[0].height, w.cameras[0].width
host = torch.empty((3, H, W, 4), dtype=torch.float32).pin_memory()
m.render_host(w.cameras, w.tf, w.v_lo, w.v_hi, w.params, host)
m.render_host_views(w.cameras, w.tf, w.v_lo, w.v_hi, w.params, [host[i].data_ptr() for i in range(3)])
buf = IpcBuffer(3 * H * W * 16)
m.render(w.cameras, torch.from_numpy(w.tf).cuda(), w.v_lo, w.v_hi, w.params, out=buf.tensor((3, H, W, 4), torch.float32))
torch.cuda.synchronize()
del buf
print("host/ipc ok")
