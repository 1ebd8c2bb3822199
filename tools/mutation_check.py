#!/usr/bin/env python
"""Mutation check of the oracle's pins (VERDICT r1 "What's weak" #1).

Copies the repo's oracle/, tests/ and the seeded generator to a scratch
directory, applies ONE plausible slip at a time to oracle/oracle.c, rebuilds
the oracle there and runs the CPU suite (-m "not gpu", oracle tests only).
A mutation is "killed" when at least one test fails.  Prints one line per
mutation and exits non-zero if any survives.

    python tools/mutation_check.py [--only A2,B]
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (id, what, exact text, replacement[, file: default oracle/oracle.c])
MUTATIONS = [
    ("A2", "samples at t_in + k*step instead of the midpoint (R-7)",
     "const double t = t_in + (k + 0.5) * P->step;", "const double t = t_in + (k + 0.0) * P->step;"),
    ("A3", "sample count ceil(L/step) instead of ceil(L/step - 1/2)",
     "double f = L / step - 0.5;", "double f = L / step;"),
    ("B", "TF normalisation divides by v_hi instead of v_hi - v_lo",
     "double s = (v - tf->v_lo) / (tf->v_hi - tf->v_lo);", "double s = (v - tf->v_lo) / (tf->v_hi);"),
    ("B2", "TF clamp at 1 dropped",
     "    if (s > 1.0) s = 1.0;\n    const int n = tf->n_entries;", "    const int n = tf->n_entries;"),
    ("C", "sigma inflated 100x (every eval tolerance 100x looser)",
     "for (int k = 0; k < 4; ++k) { out[k] = s[k]; if (sigma) sigma[k] = a[k]; }",
     "for (int k = 0; k < 4; ++k) { out[k] = s[k]; if (sigma) sigma[k] = 100.0 * a[k]; }"),
    ("D", "exit-window alternative disabled (R-19 ii)",
     "if (fr > -0.5 && fabs(fr - m) < cx->prm->exit_window) {", "if (0 && fabs(fr - m) < cx->prm->exit_window) {"),
    ("E", "every pixel flagged shading-sensitive (R-19 iii)",
     "if (P->shading && wgt > P->sens_weight && gnorm < P->sens_grad) r->shade_sensitive = 1;",
     "r->shade_sensitive = 1;"),
    ("F", "headlight specular R.V = (N.L)^2 instead of 2(N.L)^2 - 1",
     "double rv = 2.0 * ndl * ndl - 1.0;", "double rv = ndl * ndl;"),
    ("G", "curvature table axes swapped in the bilinear lookup",
     "const double a00 = T[4 * (i0[1] * n + i0[0]) + c], a01 = T[4 * (i0[1] * n + i0[0] + 1) + c];",
     "const double a00 = T[4 * (i0[0] * n + i0[1]) + c], a01 = T[4 * (i0[0] * n + i0[1] + 1) + c];"),
    ("H", "light reflection R = (N.L) N - L instead of 2 (N.L) N - L",
     "R[i] = 2.0 * ndl * N[i] - L[i];", "R[i] = 1.0 * ndl * N[i] - L[i];"),
    ("I", "compositing weight a instead of (1 - A) a",
     "const double wgt = (1.0 - r->A) * a;", "const double wgt = a;"),
    ("J", "ERT test >= instead of > ... and before compositing (o_max - A)",
     "int stop = r->A > P->o_max;", "int stop = r->A + 1e-3 > P->o_max;"),
    ("K", "ambient term dropped from Phong",
     "/* l.11 addShading */\n                    double x = col[i] * (P->ka + P->kd * dif) + P->ks * spe;",
     "/* l.11 addShading */\n                    double x = col[i] * (P->kd * dif) + P->ks * spe;"),
    ("L", "gradient component w uses dN of v (transposed operand)",
     "double t3 = N[0][aa] * N[1][b] * dN[2][c] * P;", "double t3 = N[0][aa] * dN[1][b] * N[2][c] * P;"),
    ("M", "physical gradient multiplied by L instead of divided",
     "for (int i = 0; i < 3; ++i) g[i] = vg[1 + i] / cx->L[i];   /* physical gradient (R-4) */",
     "for (int i = 0; i < 3; ++i) g[i] = vg[1 + i] * cx->L[i];   /* physical gradient (R-4) */"),
    ("N", "TF entry index uses n instead of n - 1 entries",
     "double f = s * (n - 1);", "double f = s * n;"),
    # round 2: the rest of the oracle (basis, Hessian, curvature, analytic
    # fields, rays, clip) and the Python oracles (encoder, image metrics)
    ("O1", "span search puts a point on an interior knot into the left span",
     "if (u < U[mid]) hi = mid; else lo = mid;", "if (u <= U[mid]) hi = mid; else lo = mid;"),
    ("O2a", "basis derivative without the factor p",
     "dN[r] = p * d;", "dN[r] = d;"),
    ("O2b", "Cox-de Boor left difference off by one knot",
     "left[j] = u - U[span + 1 - j];\n        right[j] = U[span + j] - u;\n        double saved = 0.0;\n        for (int r = 0; r < j; ++r) {\n            ndu[j][r]",
     "left[j] = u - U[span - j];\n        right[j] = U[span + j] - u;\n        double saved = 0.0;\n        for (int r = 0; r < j; ++r) {\n            ndu[j][r]"),
    ("H1a", "second derivative returned as the first",
     "d2N[r] = tri_dN(&T, 2, p, i);", "d2N[r] = tri_dN(&T, 1, p, i);"),
    ("H1b", "Hessian mixed term uw computed as uv",
     "{0, 2, 0}, {0, 0, 2}, {1, 1, 0}, {1, 0, 1}, {0, 1, 1}};", "{0, 2, 0}, {0, 0, 2}, {1, 1, 0}, {1, 1, 0}, {0, 1, 1}};"),
    ("H1c", "derivative recursion factor q - 1 instead of q",
     "return q * (tri_div(", "return (q - 1) * (tri_div("),
    ("C1a", "shape operator sign flipped",
     "G[i][j] = -acc / gn;", "G[i][j] = acc / gn;"),
    ("C1b", "principal curvatures without the square root",
     "k[0] = 0.5 * (T + sqrt(disc));", "k[0] = 0.5 * (T + disc);"),
    ("C1c", "tangent projector P = I + n n^T",
     "Pm[i][j] = (i == j ? 1.0 : 0.0) - n[i] * n[j];", "Pm[i][j] = (i == j ? 1.0 : 0.0) + n[i] * n[j];"),
    ("G1a", "Gaussian beam exponent without the factor 2",
     "const double G = exp(-(l - mu) * (l - mu) / (2.0 * sg * sg));", "const double G = exp(-(l - mu) * (l - mu) / (sg * sg));"),
    ("G1b", "analytic gradient d/du without the chain-rule factor 2 (w)",
     "out[3] = 2.0 * gz;", "out[3] = gz;"),
    ("G1c", "Marschner-Lobb alpha (1 + rho) as alpha rho",
     "F = (1.0 - sin(PI * z / 2.0) + al * (1.0 + rho)) / den;", "F = (1.0 - sin(PI * z / 2.0) + al * rho) / den;"),
    ("G1d", "Gaussian beam radius not divided by R",
     "const double l = r / R;", "const double l = r;"),
    ("O4a", "ray through the pixel corner instead of its centre",
     "const double X = 2.0 * (px + 0.5) / cam->width - 1.0;", "const double X = 2.0 * px / cam->width - 1.0;"),
    ("O4b", "image rows counted from the bottom",
     "const double Y = 1.0 - 2.0 * (py + 0.5) / cam->height;", "const double Y = 2.0 * (py + 0.5) / cam->height - 1.0;"),
    ("O4c", "perspective half-angle: the full field of view",
     "const double th = tan(0.5 * cam->fov_y_deg * M_PI / 180.0);", "const double th = tan(cam->fov_y_deg * M_PI / 180.0);"),
    ("O5", "slab clip keeps the farthest entry plane's minimum",
     "if (lo > tn) tn = lo;", "if (lo < tn) tn = lo;"),
    ("E1", "encoder parameters i / m instead of i / (m - 1)",
     "return np.arange(m, dtype=np.float64) / (m - 1)", "return np.arange(m, dtype=np.float64) / m", "oracle/encode.py"),
    ("E3", "separable fit applies the u and w operators to the wrong axes",
     '"ia,jb,kc,cba->kji", Pu, Pv, Pw', '"ia,jb,kc,cba->kji", Pw, Pv, Pu', "oracle/encode.py"),
    ("E4", "residual normalised by max(q) instead of the range",
     "rng = float(q.max() - q.min()) or 1.0", "rng = float(q.max()) or 1.0", "oracle/encode.py"),
    ("E5a", "refinement inserts a quarter point instead of the span midpoint",
     "ins.append(0.5 * (lo + hi))", "ins.append(0.75 * lo + 0.25 * hi)", "oracle/encode.py"),
    ("E5b", "refinement ignores the 2(p+1) samples-per-span condition",
     "cnt[s] >= 2 * (p + 1)", "cnt[s] >= 1", "oracle/encode.py"),
    ("Q1", "PSNR from 255 instead of 255^2",
     "10.0 * math.log10(255.0 * 255.0 / m)", "10.0 * math.log10(255.0 / m)", "oracle/metrics.py"),
    ("Q2", "SSIM constant C2 = (0.01 L)^2",
     "C2 = (0.03 * 255.0) ** 2", "C2 = (0.01 * 255.0) ** 2", "oracle/metrics.py"),
    ("Q3", "8-bit quantisation truncates instead of rounding",
     "np.floor(255.0 * np.clip(x, 0.0, 1.0) + 0.5)", "np.floor(255.0 * np.clip(x, 0.0, 1.0))", "oracle/metrics.py"),
    ("Q4", "luma weights of R and B swapped",
     "LUMA = (0.299, 0.587, 0.114)", "LUMA = (0.114, 0.587, 0.299)", "oracle/metrics.py"),
]

TESTS = ["tests/test_oracle_bspline.py", "tests/test_oracle_render.py", "tests/test_oracle_render_pins.py",
         "tests/test_oracle_lights.py", "tests/test_oracle_curvature.py", "tests/test_oracle_hessian.py",
         "tests/test_oracle_quality.py", "tests/test_oracle_encode.py", "tests/test_workloads.py"]


def scratch_copy(dst: str):
    shutil.copytree(os.path.join(ROOT, "oracle"), os.path.join(dst, "oracle"),
                    ignore=shutil.ignore_patterns("*.so", "__pycache__"))
    shutil.copytree(os.path.join(ROOT, "tests"), os.path.join(dst, "tests"),
                    ignore=shutil.ignore_patterns("__pycache__"))
    pkg = os.path.join(dst, "paper_2204_11762_b200")
    os.makedirs(pkg)
    # the seeded generator only (no method arithmetic); an empty package init
    shutil.copy(os.path.join(ROOT, "paper_2204_11762_b200", "workloads.py"), pkg)
    open(os.path.join(pkg, "__init__.py"), "w").close()
    shutil.copy(os.path.join(ROOT, "pytest.ini"), dst)


def run_one(mid, what, old, new, path="oracle/oracle.c"):
    with tempfile.TemporaryDirectory(prefix=f"mut_{mid}_") as d:
        scratch_copy(d)
        src = os.path.join(d, path)
        text = open(src).read()
        if text.count(old) != 1:
            return mid, what, "NOT-APPLIED (pattern count %d)" % text.count(old)
        open(src, "w").write(text.replace(old, new))
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "not gpu", "-p", "no:cacheprovider",
                            *TESTS], cwd=d, capture_output=True, text=True, timeout=1800)
        tail = (r.stdout.strip().splitlines() or [""])[-1]
        return mid, what, ("KILLED" if r.returncode != 0 else "SURVIVED") + "  | " + tail


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    sel = set(a.only.split(",")) if a.only else None
    bad = 0
    # baseline: the unmutated copy must pass
    mid, what, res = run_one("base", "unmutated", "#include <math.h>", "#include <math.h>")
    print(f"{mid:5s} {res:60s} {what}", flush=True)
    if not res.startswith("SURVIVED"):
        print("baseline copy does not pass; aborting")
        return 2
    for m in MUTATIONS:
        if sel and m[0] not in sel:
            continue
        mid, what, res = run_one(*m)
        print(f"{mid:5s} {res:60s} {what}", flush=True)
        bad += not res.startswith("KILLED")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
