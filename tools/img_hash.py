"""Hash of rendered images, to check that a build variant (a scheduling or
load-order change) leaves every pixel bit-identical.

    python tools/img_hash.py [config ...]     (default: 2 5)

C5 renders its first 2 views at full resolution; other configs their full
workload. Prints one line per config: sha256 of the fp32 RGBA bytes and the
composited sample count.
"""
import hashlib
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_11762_b200 import Model, workloads  # noqa: E402


def main():
    cfgs = [int(c) for c in sys.argv[1:]] or [2, 5]
    for c in cfgs:
        w = workloads.make_config(c, n_views=2 if c == 5 else None)
        m = Model.from_workload(w)
        samples = torch.zeros(1, dtype=torch.int64, device="cuda")
        img = m.render(w.cameras, torch.from_numpy(w.tf).cuda(), w.v_lo, w.v_hi, w.params, samples=samples)
        torch.cuda.synchronize()
        h = hashlib.sha256(img.cpu().numpy().tobytes()).hexdigest()[:16]
        print(f"C{c}: sha256 {h} samples {int(samples.item())}")


if __name__ == "__main__":
    main()
