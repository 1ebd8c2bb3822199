"""Small end-to-end workload for compute-sanitizer: eval + render on C1/C2 in
both layouts, C5 (non-uniform, Bezier) at a reduced image, tiled render."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2204_11762_b200 import Model, unpack_tiles, workloads as WL

for c, kw in ((1, {}), (2, dict(width=96, height=64)), (5, dict(width=64, height=48, n_views=2))):
    w = WL.make_config(c, **kw)
    for layout in ("quads", "bezier"):
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
        print(c, layout, "ok", float(img.sum()))
