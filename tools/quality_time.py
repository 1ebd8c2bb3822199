"""mfa_image_quality time on a 3840x2160 pair (device-timed)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2204_11762_b200 import image_quality

g = torch.Generator(device="cuda").manual_seed(0)
a = torch.rand((2160, 3840, 4), device="cuda", generator=g)
b = (a + 0.02 * torch.rand((2160, 3840, 4), device="cuda", generator=g)).clamp(0, 1)
ws = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
q = image_quality(a, b, workspace=ws)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    image_quality(a, b, workspace=ws)
e1.record()
torch.cuda.synchronize()
print(f"image_quality 4K pair: {e0.elapsed_time(e1) / 10:.3f} ms  ssim {q['ssim']:.12f}  psnr {q['psnr']:.6f}")
