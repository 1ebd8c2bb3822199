"""Run the K5 roofline probes on the current GPU and print JSON."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_11762_b200 import _lib as L

out = {}
for m in ("ffma", "ffma2", "ffma_imm"):
    out[f"fp32_{m}_tflops"] = max(L.probe_fp32(m) for _ in range(3))
for mb in (16, 32, 64, 96):
    out[f"read_{mb}MiB_gbps"] = max(L.probe_read_bw(mb << 20, 50) for _ in range(3))
out["read_4GiB_gbps"] = max(L.probe_read_bw(4 << 30, 3) for _ in range(2))
print(json.dumps(out))
