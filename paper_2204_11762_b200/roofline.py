"""Counted work per unit and the roofline denominators (SURVEY §8(d),
DESIGN.md §6).

Per composited ray-sample of degree p (q = p + 1), FMA = 2 FLOPs, other
add / mul / div / rsqrt / exp2 / log2 = 1 FLOP:
  a7 contraction   2 (2 q^3 + 3 q^2 + 4 q)
  a5 basis + N'    3 (5 p (p+1)/2 + 2 p + 4 q)
  a3 position 14, a4 local coordinate 12, a8 TF 16, a9 Phong 36, a10 composite 9
  -> F(p) = 366 / 627 / 1011 for p = 2 / 3 / 4.
Counted control-point bytes per sample B(p) = 4 q^3 (108 / 256 / 500).
Per eval point: contraction + basis + 12.  Per Hessian point (NEXT-4):
2 (3 q^3 + 6 q^2 + 10 q) + 3 q (6 p + 1) + 21.

FP32 peak (CUDA cores): SMs x 128 lanes x 2 FLOP x SM clock.  B200 has 148
SMs and clocks.max.sm = 1965 MHz (B200_PROFILING.md) -> 74.4 TFLOP/s.
"""
from __future__ import annotations

import json
import os

N_SM = 148
FP32_LANES_PER_SM = 128
SM_MAX_MHZ_FALLBACK = 1965.0
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def flops_contraction(p: int) -> int:
    q = p + 1
    return 2 * (2 * q ** 3 + 3 * q ** 2 + 4 * q)


def flops_basis(p: int) -> int:
    q = p + 1
    return 3 * (5 * p * (p + 1) // 2 + 2 * p + 4 * q)


def flops_per_sample(p: int, shading: bool = True) -> int:
    if not shading:
        q = p + 1
        # value-only: q^3 + q^2 + q FMAs; basis values only ~ 3*(5p(p+1)/2 + 2p)
        return 2 * (q ** 3 + q ** 2 + q) + 3 * (5 * p * (p + 1) // 2 + 2 * p) + 14 + 12 + 16 + 9
    return flops_contraction(p) + flops_basis(p) + 14 + 12 + 16 + 36 + 9


def flops_per_eval_point(p: int) -> int:
    return flops_contraction(p) + flops_basis(p) + 12


def flops_per_hessian_point(p: int) -> int:
    """NEXT-4 per point: x-stage 3 q^3, y-stage 6 q^2, z-stage 10 q FMAs; per
    axis q three-output Horner evaluations (3p FMA + 1 mul each); locate 12;
    t -> u scaling 9."""
    q = p + 1
    return 2 * (3 * q ** 3 + 6 * q ** 2 + 10 * q) + 3 * q * (6 * p + 1) + 12 + 9


def bytes_per_sample(p: int) -> int:
    return 4 * (p + 1) ** 3


def measured_peaks() -> dict:
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return {}


def fp32_peak_tflops(sm_mhz: float | None = None) -> tuple[float, str]:
    """FP32 CUDA-core peak in TFLOP/s at the given (default: max) SM clock."""
    src = "derived: 148 SMs x 128 FP32 lanes x 2 FLOP x clocks.max.sm"
    if sm_mhz is None:
        pk = measured_peaks()
        sm_mhz = float(pk.get("sm_max_mhz", SM_MAX_MHZ_FALLBACK))
        src += " (%s)" % ("MEASURED_PEAKS.json" if "sm_max_mhz" in pk else "B200_PROFILING.md fallback")
    return N_SM * FP32_LANES_PER_SM * 2 * sm_mhz * 1e6 / 1e12, src


def hbm_peak_gbs() -> tuple[float, str]:
    pk = measured_peaks()
    if "hbm_gbs" in pk:
        return float(pk["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    return 6650.0, "B200_PROFILING.md fallback"
