"""Pins for the NEXT-4 oracle lights (several directional lights, PAPER.md
P:307 "multiple light sources can be added in the future"; R-30): a closed-
form render of the linear field under side lights, the headlight special
case, linearity in the intensities and lights from behind.  No GPU."""
import numpy as np
import pytest

import oracle as O
from test_oracle_render import _closed_form_linear, box_model, ortho_down, params_for

KA, KD = 0.1, 0.7


def linear_setup():
    m, L = box_model(p=2, n=(8, 6, 5), field="u")
    n = 256
    i = np.arange(n) / (n - 1)
    tf = np.stack([i, 1 - i, np.full(n, 0.5), 0.02 + 0.08 * i], axis=1).astype(np.float32)
    return m, L, tf


@pytest.mark.parametrize("inten", [0.3, 1.0, 2.5])
def test_side_light_linear_field_closed_form(inten):
    """f = u under an orthographic view along -z: N = -x (unit), V = +z.  A
    light towards -x (L = N) gives N.L = 1 and R = N, so R.V = 0: diffuse
    I, no specular: pixel = min(1, (k_a + k_d I) rgb(u)) (1 - (1-a)^K).  A
    light towards +x (behind the surface) adds nothing."""
    m, L, tf = linear_setup()
    W = H = 24
    step = 0.021
    prm = params_for(L, step=step, o_max=0.99)
    r = O.render(m, ortho_down(W, H, 0.6), tf, 0.0, 1.0, prm, lights=[((-1.0, 0.0, 0.0), inten), ((1.0, 0, 0), 5.0)])
    lit = KA + KD * inten
    ref, cnt = _closed_form_linear(
        L, W, H, 0.6, step, 0.99,
        a_of_s=lambda s: 0.02 + 0.08 * s,
        c_of_s=lambda s: np.minimum(1.0, lit * np.array([s, 1 - s, 0.5])))
    np.testing.assert_array_equal(r["count"], cnt)
    np.testing.assert_allclose(r["rgba"], ref, rtol=0, atol=2e-7)


def test_single_headlight_equals_default_ortho():
    """For an orthographic camera every ray has the same direction d, so one
    light towards -d with intensity 1 is the headlight (R-11)."""
    from paper_2204_11762_b200 import workloads as WL
    w = WL.make_config(1)
    om = O.Model.from_workload(w)
    cam = w.cameras[0]
    o, d = O.ray(cam, 3, 5)
    a = O.render(om, cam, w.tf, w.v_lo, w.v_hi, w.params)
    b = O.render(om, cam, w.tf, w.v_lo, w.v_hi, w.params, lights=[(-d, 1.0)])
    np.testing.assert_array_equal(a["count"], b["count"])
    np.testing.assert_allclose(a["rgba"], b["rgba"], rtol=0, atol=1e-12)


def test_lights_linear_in_intensity():
    """Two equal lights of intensity 1/2 = one light of intensity 1 (the sum
    is taken before the clamp); the order of the lights does not matter."""
    from paper_2204_11762_b200 import workloads as WL
    w = WL.make_config(2, width=40, height=32)
    om = O.Model.from_workload(w)
    cam = w.cameras[0]
    L1, L2 = (0.3, -0.5, 0.8), (-0.7, 0.2, 0.1)
    a = O.render(om, cam, w.tf, w.v_lo, w.v_hi, w.params, lights=[(L1, 1.0), (L2, 0.4)])
    b = O.render(om, cam, w.tf, w.v_lo, w.v_hi, w.params, lights=[(L2, 0.4), (L1, 0.5), (L1, 0.5)])
    np.testing.assert_array_equal(a["count"], b["count"])
    np.testing.assert_allclose(a["rgba"], b["rgba"], rtol=0, atol=1e-12)
    c = O.render(om, cam, w.tf, w.v_lo, w.v_hi, w.params, lights=[(L1, 0.0)])   # no light: ambient only
    d = O.render(om, cam, w.tf, w.v_lo, w.v_hi, w.params, lights=[((1, 1, 1), 0.0), ((0, 0, 1), 0.0)])
    np.testing.assert_allclose(c["rgba"], d["rgba"], rtol=0, atol=1e-15)
