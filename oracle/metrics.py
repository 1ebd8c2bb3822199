"""TEST INFRASTRUCTURE ONLY: fp64 numpy oracle of the image-quality metrics
(NEXT-2).  Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may
import it; it shares nothing with the CUDA path (csrc/quality.cu).

The paper scores volume-rendered images against the ground-truth rendering
with "mean squared error (MSE), peak signal-to-noise ratio (PSNR), and
structural similarity index (SSIM) ... at the pixel level" (PAPER.md P:191,
Tables 1-2).  It does not define them further; the readings used
(R-22) follow SPEC S:469-516:

  * an image is the displayed colour: premultiplied RGB composited over a
    black background (alpha excluded), quantised to 8 bits as
    q = floor(255 * clamp(x, 0, 1) + 1/2) ("squared 8-bit differences");
  * MSE = mean over pixels and the 3 channels of (q_a - q_b)^2;
    PSNR = 10 log10(255^2 / MSE), +inf for identical images;
  * SSIM (Wang et al. 2004) on the luma Y = 0.299 R + 0.587 G + 0.114 B of the
    8-bit values, 11x11 Gaussian window sigma = 1.5 normalised
    to sum 1, C1 = (0.01 * 255)^2, C2 = (0.03 * 255)^2, averaged over every
    window position fully inside the image ("valid" windows).

Each step is written out directly: the windowed sums are a plain double loop
over the 121 window offsets (no separable filtering).
"""
from __future__ import annotations

import math

import numpy as np

WIN = 11
SIGMA = 1.5
C1 = (0.01 * 255.0) ** 2
C2 = (0.03 * 255.0) ** 2
LUMA = (0.299, 0.587, 0.114)


def quantize8(img) -> np.ndarray:
    """(H, W, >=3) premultiplied float RGB(A) -> (H, W, 3) 8-bit levels as fp64."""
    x = np.asarray(img, dtype=np.float64)[..., :3]
    return np.floor(255.0 * np.clip(x, 0.0, 1.0) + 0.5)


def gaussian_window() -> np.ndarray:
    k = np.arange(WIN) - WIN // 2
    g = np.exp(-(k[:, None] ** 2 + k[None, :] ** 2) / (2.0 * SIGMA * SIGMA))
    return g / g.sum()


def mse(a, b) -> float:
    qa, qb = quantize8(a), quantize8(b)
    return float(np.mean((qa - qb) ** 2))


def psnr_from_mse(m: float) -> float:
    return math.inf if m == 0.0 else 10.0 * math.log10(255.0 * 255.0 / m)


def luma(q) -> np.ndarray:
    return LUMA[0] * q[..., 0] + LUMA[1] * q[..., 1] + LUMA[2] * q[..., 2]


def ssim_map(ya, yb) -> np.ndarray:
    """SSIM at every valid window position of two luma images (fp64)."""
    H, W = ya.shape
    if H < WIN or W < WIN:
        raise ValueError("image smaller than the 11x11 SSIM window")
    g = gaussian_window()
    oh, ow = H - WIN + 1, W - WIN + 1
    mu_a = np.zeros((oh, ow))
    mu_b = np.zeros((oh, ow))
    saa = np.zeros((oh, ow))
    sbb = np.zeros((oh, ow))
    sab = np.zeros((oh, ow))
    for di in range(WIN):
        for dj in range(WIN):
            A = ya[di:di + oh, dj:dj + ow]
            B = yb[di:di + oh, dj:dj + ow]
            w = g[di, dj]
            mu_a += w * A
            mu_b += w * B
            saa += w * A * A
            sbb += w * B * B
            sab += w * A * B
    var_a = saa - mu_a * mu_a
    var_b = sbb - mu_b * mu_b
    cov = sab - mu_a * mu_b
    return ((2.0 * mu_a * mu_b + C1) * (2.0 * cov + C2)) / ((mu_a ** 2 + mu_b ** 2 + C1) * (var_a + var_b + C2))


def ssim(a, b) -> float:
    return float(ssim_map(luma(quantize8(a)), luma(quantize8(b))).mean())


def error_map(a, b) -> np.ndarray:
    """Per-pixel Euclidean RGB error in 8-bit levels (Fig. 6 "pixel level
    rendering error distribution")."""
    d = quantize8(a) - quantize8(b)
    return np.sqrt((d * d).sum(axis=-1))


def quality(a, b) -> dict:
    m = mse(a, b)
    return {"mse": m, "psnr": psnr_from_mse(m), "ssim": ssim(a, b)}
