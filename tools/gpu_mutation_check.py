#!/usr/bin/env python
"""GPU-side mutation check: the -m gpu parity tests must bite.

Applies ONE plausible slip at a time to the CUDA sources (in place, with a
pristine copy restored after each), rebuilds libmfa.so and runs the GPU
parity tests that exercise the slipped step; a mutation is "killed" when a
test fails.  Run on a GPU box (gpurun), never in the dev tree:

    python tools/gpu_mutation_check.py [--only K1,K2]
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_2204_11762_b200", "csrc")
RK, KC, EV = "render_kernel.cuh", "kernels.cuh", "eval.cu"

# (id, what, file, exact text (every occurrence replaced), replacement, pytest -k selection)
MUTATIONS = [
    ("K1", "samples at t_in + k*step instead of the midpoint (R-7)", RK,
     "const double t0 = t_in + 0.5 * args.step;", "const double t0 = t_in;", "render or subset or image"),
    ("K2", "TF position ignores v_lo", RK,
     "float f = (v - args.v_lo) * args.s_scale;", "float f = v * args.s_scale;", "render or subset or image"),
    ("K3", "compositing weight a instead of (1 - A) a", RK,
     "const float wgt = comp_on ? (1.f - A) * a : 0.f;", "const float wgt = comp_on ? a : 0.f;", "render or subset or image"),
    ("K4", "ambient term dropped from Phong", RK,
     "const float lit = zero ? args.ka : fmaf(args.kd, dif, args.ka);", "const float lit = zero ? args.ka : args.kd * dif;",
     "render or subset or image"),
    ("K5", "ERT threshold raised by 0.05", RK,
     "live = live && !(A > args.o_max) && k < K;", "live = live && !(A > args.o_max + 0.05f) && k < K;",
     "render or subset or image"),
    ("K6", "backward span crossings step forward (non-uniform tracker)", KC,
     "st.s = max(st.s + ((d >> 31) | 1), 0);", "st.s = max(st.s + 1, 0);", "render or subset or image"),
    ("K7", "eval gradient not scaled to parameter space", EV,
     "        gu *= sc[0];", "        gu *= 1.f;", "eval"),
    ("K8", "eval v-derivative basis at u's local coordinate (Bezier)", EV,
     "bernstein<P, true>(t[1], Bv);", "bernstein<P, true>(t[0], Bv);", "eval"),
    ("K9", "cubic Bernstein derivative of B_1 with the wrong sign", KC,
     "fmaf(ts3, -2.f, -d0)", "fmaf(ts3, 2.f, -d0)", "eval or render"),
    ("K10", "quad-lane warp unit: the x bit of a 2 x 2 quad taken from lane bit 1 (rows and columns of a quad swapped)", RK,
     "lx = (sub & 1) * 8 + ((lane >> 2) & 3) * 2 + (lane & 1);", "lx = (sub & 1) * 8 + ((lane >> 2) & 3) * 2 + ((lane >> 1) & 1);",
     "render or subset or image"),
]


def build() -> bool:
    r = subprocess.run([sys.executable, "-m", "paper_2204_11762_b200.build"], cwd=ROOT, capture_output=True, text=True)
    return r.returncode == 0


def run_one(mid, what, fname, old, new, sel, pristine):
    src = os.path.join(CSRC, fname)
    text = open(os.path.join(pristine, fname)).read()
    if old not in text:
        return f"NOT-APPLIED (pattern absent in {fname})"
    open(src, "w").write(text.replace(old, new))
    try:
        if not build():
            return "BUILD-FAILED"
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                            "tests/test_gpu_parity.py", "-k", sel], cwd=ROOT, capture_output=True, text=True,
                           timeout=1800)
        tail = (r.stdout.strip().splitlines() or [""])[-1]
        return ("KILLED" if r.returncode == 1 else ("SURVIVED" if r.returncode == 0 else f"ERROR rc={r.returncode}")) + \
            "  | " + tail
    finally:
        shutil.copy(os.path.join(pristine, fname), src)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    a = ap.parse_args()
    sel = set(a.only.split(",")) if a.only else None
    pristine = os.path.join(ROOT, "gpurun_out", "_csrc_pristine")
    shutil.rmtree(pristine, ignore_errors=True)
    shutil.copytree(CSRC, pristine)
    bad = 0
    try:
        for m in MUTATIONS:
            if sel and m[0] not in sel:
                continue
            res = run_one(*m, pristine)
            print(f"{m[0]:4s} {res:62s} {m[1]}", flush=True)
            bad += not res.startswith("KILLED")
    finally:
        for f in os.listdir(pristine):
            shutil.copy(os.path.join(pristine, f), os.path.join(CSRC, f))
        shutil.rmtree(pristine, ignore_errors=True)
        build()
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
