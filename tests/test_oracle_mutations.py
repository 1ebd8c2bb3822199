"""The oracle's pins must bite: the five slips the round-1 review found
undetected (samples at t_in + k*step, TF normalised by v_hi, sigma inflated
100x, the exit-window alternative disabled, every pixel shading-sensitive)
are applied one at a time to a scratch copy of oracle/oracle.c, and the CPU
oracle suite must FAIL on each; so must one slip each in the basis
derivatives, the Hessian, the curvature operator, the encoder's refinement
and the SSIM luma (tools/mutation_check.py runs all 42 slips).  No GPU."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import mutation_check as MC   # noqa: E402

REVIEW_SLIPS = ("A2", "B", "C", "D", "E", "O2a", "H1b", "C1a", "E5a", "Q4")


def test_unmutated_copy_passes():
    mid, what, res = MC.run_one("base", "unmutated", "#include <math.h>", "#include <math.h>")
    assert res.startswith("SURVIVED"), res


@pytest.mark.parametrize("mid", REVIEW_SLIPS)
def test_review_slip_is_killed(mid):
    m = next(x for x in MC.MUTATIONS if x[0] == mid)
    _, what, res = MC.run_one(*m)
    assert res.startswith("KILLED"), f"{mid} ({what}) survived the oracle pins: {res}"
