"""Parity criteria (GPU vs oracle), written once for the tests, smoke() and
bench.py.  Tolerances are north_star's (BASELINE.json):
  * point evaluations: |v - v*| <= 1e-5 sigma_v, |g_d - g*_d| <= 1e-4 sigma_d,
    sigma = the abs-scale of the same contraction (R-5);
  * images: per pixel e = max_channel |I - I*| (minimum over the oracle's
    stored alternative outcomes, R-19); 99.9th percentile of e <= 2e-3 and
    max e <= 1e-2 over ALL pixels (shading-sensitive pixels are counted and
    reported, not excluded: the round-1 data had max_all <= 8.3e-5).
"""
from __future__ import annotations

import numpy as np

VAL_TOL = 1e-5
GRAD_TOL = 1e-4
IMG_P999 = 2e-3
IMG_MAX = 1e-2


def eval_errors(gpu4: np.ndarray, ref4: np.ndarray, sig4: np.ndarray):
    """Normwise errors |gpu - ref| / sigma per component (n, 4) -> (n, 4)."""
    err = np.abs(gpu4.astype(np.float64) - ref4)
    with np.errstate(divide="ignore", invalid="ignore"):
        r = np.where(sig4 > 0, err / sig4, np.where(err == 0, 0.0, np.inf))
    return r


def check_eval(gpu4, ref4, sig4, what=""):
    r = eval_errors(gpu4, ref4, sig4)
    worst_v = float(r[:, 0].max()) if len(r) else 0.0
    worst_g = float(r[:, 1:].max()) if len(r) and r.shape[1] > 1 else 0.0
    assert worst_v <= VAL_TOL, f"{what}: value normwise error {worst_v:.3e} > {VAL_TOL}"
    assert worst_g <= GRAD_TOL, f"{what}: gradient normwise error {worst_g:.3e} > {GRAD_TOL}"
    return worst_v, worst_g


def image_errors(gpu: np.ndarray, ref: dict):
    """gpu: (n, 4) pixels; ref: oracle.render dict for the same pixels."""
    g = gpu.astype(np.float64)
    e = np.abs(g - ref["rgba"]).max(axis=1)
    for j in range(2):
        alt = ref["alt"][:, j, :]
        has = ~np.isnan(alt[:, 0])
        if has.any():
            ea = np.abs(g[has] - alt[has]).max(axis=1)
            e[has] = np.minimum(e[has], ea)
    return e


def check_image(gpu, ref, what=""):
    e = image_errors(gpu, ref)
    shade = (ref["flags"] & 4) != 0
    p999 = float(np.percentile(e, 99.9)) if len(e) else 0.0
    mx = float(e.max()) if len(e) else 0.0
    mx_ns = float(e[~shade].max()) if (~shade).any() else 0.0
    stats = dict(p999=p999, max=mx, max_not_sensitive=mx_ns,
                 n=len(e), n_shade=int(shade.sum()), n_ert=int(((ref["flags"] & 1) != 0).sum()),
                 n_exit=int(((ref["flags"] & 2) != 0).sum()))
    assert p999 <= IMG_P999, f"{what}: p99.9 error {p999:.3e} > {IMG_P999} ({stats})"
    assert mx <= IMG_MAX, f"{what}: max error {mx:.3e} > {IMG_MAX} ({stats})"
    return stats


def count_window(ref: dict) -> int:
    """How far the composited-sample total may legitimately move: the
    summed |alternative - primary| counts over flagged pixels."""
    d = 0
    for j in range(2):
        ac = ref["alt_count"][:, j]
        has = ac >= 0
        d += int(np.abs(ac[has] - ref["count"][has]).sum())
    return d
