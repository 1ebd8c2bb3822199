"""Pins for the NEXT-2 oracle: the analytic ground-truth fields (PAPER.md
Eq. 1-2), the ground-truth renderer that takes sample values
and/or gradients from them, and the image-quality metrics
(MSE / PSNR / SSIM; readings from SPEC S:469-516).  No GPU."""
import math

import numpy as np
import pytest

import oracle as O
from oracle import metrics as QM
from paper_2204_11762_b200 import workloads as WL
from test_oracle_render import box_model, const_tf, ortho_down, params_for

ML = WL.AnalyticField.marschner_lobb
GB = WL.AnalyticField.gaussian_beam


# --------------------------------------------------------------------------
# G1: analytic fields
# --------------------------------------------------------------------------
def test_field_values_closed_form():
    """SPEC S:257-258 (ML(0,0,-1) = 1, ML(0,0,1) = 0.2) and S:239-240
    (GB(0,0,0) = 255, GB(1,1,1) = 255 e^-4.5), at x = 2u - 1."""
    assert O.field_eval(ML(), 0.5, 0.5, 0.0)[0] == pytest.approx(1.0, abs=1e-15)
    assert O.field_eval(ML(), 0.5, 0.5, 1.0)[0] == pytest.approx(0.2, abs=1e-15)
    assert O.field_eval(GB(), 0.5, 0.5, 0.5)[0] == 255.0
    assert O.field_eval(GB(), 1.0, 1.0, 1.0)[0] == pytest.approx(255.0 * math.exp(-4.5), rel=1e-14)
    r = np.random.default_rng(1)
    for u, v, w in r.uniform(0, 1, (200, 3)):
        f = O.field_eval(ML(), u, v, w)[0]
        assert 0.0 <= f <= 1.0
        g = O.field_eval(GB(), u, v, w)[0]
        assert 255.0 * math.exp(-4.5) - 1e-12 <= g <= 255.0


@pytest.mark.parametrize("fld", [ML(), GB()])
def test_field_gradient_matches_central_differences(fld):
    """Parameter-space gradient = central differences of the value (h = 1e-5;
    truncation O(h^2 f''') is ~1e-8 relative here)."""
    r = np.random.default_rng(2)
    h = 1e-5
    for u, v, w in r.uniform(0.02, 0.98, (300, 3)):
        g = O.field_eval(fld, u, v, w)[1:]
        fd = []
        for d in range(3):
            p = [u, v, w]
            m = [u, v, w]
            p[d] += h
            m[d] -= h
            fd.append((O.field_eval(fld, *p)[0] - O.field_eval(fld, *m)[0]) / (2 * h))
        scale = 1.0 + np.abs(g).max()
        assert np.abs(np.array(fd) - g).max() <= 2e-6 * scale, (u, v, w, g, fd)


def test_field_gradient_special_points():
    """GB: zero gradient at the centre, radial direction elsewhere; ML: on the
    z axis the radial part vanishes and dF/dw = 2 * (-(pi/2) cos(pi z/2)) / (2(1+alpha))."""
    np.testing.assert_array_equal(O.field_eval(GB(), 0.5, 0.5, 0.5)[1:], 0.0)
    g = O.field_eval(GB(), 0.8, 0.6, 0.3)[1:]
    x = np.array([0.6, 0.2, -0.4])
    np.testing.assert_allclose(np.cross(g, x), 0.0, atol=1e-12)
    assert np.dot(g, x) < 0                                       # decreasing outwards (mu = 0)
    for w in (0.0, 0.3, 0.5, 0.9):
        out = O.field_eval(ML(), 0.5, 0.5, w)
        z = 2 * w - 1
        assert out[1] == 0.0 and out[2] == 0.0
        assert out[3] == pytest.approx(2 * (-(math.pi / 2) * math.cos(math.pi * z / 2)) / 2.5, rel=1e-14)


# --------------------------------------------------------------------------
# G2: ground-truth render
# --------------------------------------------------------------------------
def test_constant_analytic_field_ert_closed_form():
    """A Gaussian beam with V_min = V_max = c is the constant c with zero
    gradient whatever the MFA holds: the constant-field closed form
    (A_44 = 1 - 0.9^44, ambient colour) must come out of the analytic path."""
    m, L = box_model(p=2, n=(8, 8, 8), field="u")       # the MFA is NOT constant
    fld = WL.AnalyticField(WL.FIELD_GAUSSIAN_BEAM, 1, 1, (0.5, 0.5, 0.0, 1.0 / 3.0, math.sqrt(3.0)))
    cam = ortho_down(16, 16, 0.3)
    rgb = np.array([0.8, 0.4, 0.2])
    prm = params_for(L, step=1.0 / 200, shading=1)
    r = O.render(m, cam, const_tf(rgb, 0.1), 0.0, 1.0, prm, field=fld)
    assert (r["count"] == 44).all()
    a32 = float(np.float32(0.1))
    rgb32 = rgb.astype(np.float32).astype(np.float64)
    A44 = 1 - (1 - a32) ** 44
    np.testing.assert_allclose(r["rgba"][:, 3], A44, rtol=0, atol=1e-14)
    np.testing.assert_allclose(r["rgba"][:, :3], np.outer(np.ones(256), 0.1 * rgb32 * A44), atol=1e-14)


def _small_ml(n, w=40, h=32):
    wl = WL.make_config(2, width=w, height=h)
    knots = [WL.clamped_uniform_knots(n, 3)] * 3
    xi = [WL.greville(k, 3) for k in knots]
    X = 2 * xi[0][None, None, :] - 1
    Y = 2 * xi[1][None, :, None] - 1
    Z = 2 * xi[2][:, None, None] - 1
    ctrl = WL.marschner_lobb(X, Y, Z).astype(np.float32)
    return wl, O.Model(3, knots, ctrl)


def test_source_routing_invariants():
    """value/gradient routing: (MFA, MFA) == plain render; with shading off the
    gradient source is irrelevant."""
    import dataclasses
    wl, om = _small_ml(16)
    cam = wl.cameras[0]
    plain = O.render(om, cam, wl.tf, 0.0, 1.0, wl.params)
    both_mfa = O.render(om, cam, wl.tf, 0.0, 1.0, wl.params, field=ML(0, 0))
    np.testing.assert_array_equal(plain["rgba"], both_mfa["rgba"])
    off = dataclasses.replace(wl.params, shading=0)
    a = O.render(om, cam, wl.tf, 0.0, 1.0, off, field=ML(1, 0))
    b = O.render(om, cam, wl.tf, 0.0, 1.0, off, field=ML(1, 1))
    np.testing.assert_array_equal(a["rgba"], b["rgba"])
    c = O.render(om, cam, wl.tf, 0.0, 1.0, off, field=ML(0, 1))
    np.testing.assert_array_equal(c["rgba"], O.render(om, cam, wl.tf, 0.0, 1.0, off)["rgba"])


def test_mfa_image_converges_to_ground_truth():
    """"higher 3D resolution increases fidelity".  As the MFA of the
    Marschner-Lobb function is refined (16^3 -> 32^3 -> 64^3 control points,
    p = 3) its rendering approaches the analytic ground truth in the value-only
    test (shading off), the gradient-only test (analytic value, MFA
    gradient) and overall.  A wrong sign or factor in the
    analytic gradient would leave the gradient-only error at O(1)."""
    import dataclasses
    errs = {k: [] for k in ("value", "gradient", "overall")}
    for n in (16, 32, 64):
        wl, om = _small_ml(n)
        cam = wl.cameras[0]
        off = dataclasses.replace(wl.params, shading=0)
        img = lambda prm, fld: O.render(om, cam, wl.tf, 0.0, 1.0, prm, field=fld)["rgba"].reshape(32, 40, 4)
        errs["value"].append(QM.mse(img(off, None), img(off, ML(1, 1))))
        errs["gradient"].append(QM.mse(img(wl.params, ML(1, 0)), img(wl.params, ML(1, 1))))
        errs["overall"].append(QM.mse(img(wl.params, None), img(wl.params, ML(1, 1))))
    for k, e in errs.items():
        assert e[0] > e[1] > e[2], (k, e)
        assert e[2] < 0.25 * e[0], (k, e)
    assert errs["gradient"][2] < 5.0, errs


# --------------------------------------------------------------------------
# metrics
# --------------------------------------------------------------------------
def rgba(h, w, seed):
    r = np.random.default_rng(seed)
    return r.uniform(0, 1, (h, w, 4))


def test_mse_psnr_spec_examples():
    """identical -> 0 / +inf; black vs white -> 65025 / 0 dB;
    one channel of one pixel off by 255 in 10x10 -> 65025/300 = 216.75."""
    a = rgba(10, 10, 0)
    assert QM.mse(a, a) == 0.0 and QM.psnr_from_mse(0.0) == math.inf
    blk, wht = np.zeros((10, 10, 4)), np.ones((10, 10, 4))
    assert QM.mse(blk, wht) == 65025.0 and QM.psnr_from_mse(65025.0) == 0.0
    b = blk.copy()
    b[3, 4, 1] = 1.0
    assert QM.mse(blk, b) == 216.75
    m = [QM.mse(blk, blk + k / 255.0) for k in (1, 2, 5, 9)]
    p = [QM.psnr_from_mse(x) for x in m]
    assert all(x < y for x, y in zip(m, m[1:])) and all(x > y for x, y in zip(p, p[1:]))


def test_quantize_and_alpha_excluded():
    a = np.zeros((12, 12, 4))
    b = a.copy()
    b[..., 3] = 1.0                                   # alpha only: no difference
    assert QM.mse(a, b) == 0.0 and QM.ssim(a, b) == 1.0
    q = QM.quantize8(np.array([[[0.5 / 255, 1.5 / 255 - 1e-9, -0.2]]]))
    np.testing.assert_array_equal(q, [[[1.0, 1.0, 0.0]]])


def test_ssim_identity_symmetry_and_constant_closed_form():
    a, b = rgba(20, 17, 1), rgba(20, 17, 2)
    assert QM.ssim(a, a) == pytest.approx(1.0, abs=1e-15)
    assert QM.ssim(a, b) == pytest.approx(QM.ssim(b, a), abs=1e-12)
    g = np.full((16, 16, 4), 100 / 255.0)
    h = np.full((16, 16, 4), 110 / 255.0)
    ya, yb = QM.luma(QM.quantize8(g))[0, 0], QM.luma(QM.quantize8(h))[0, 0]
    # constant windows: variances and covariance vanish -> SSIM = luminance term
    want = (2 * ya * yb + QM.C1) / (ya * ya + yb * yb + QM.C1)
    assert QM.ssim(g, h) == pytest.approx(want, rel=1e-12)
    with pytest.raises(ValueError):
        QM.ssim(np.zeros((10, 30, 4)), np.zeros((10, 30, 4)))


def test_ssim_brute_force_central_moments():
    """Per-window brute force with central moments sum w (A - mu)^2 (the
    definition, not the raw-moment form the oracle uses) on a 13x14 image."""
    a, b = rgba(13, 14, 3), rgba(13, 14, 4)
    ya, yb = QM.luma(QM.quantize8(a)), QM.luma(QM.quantize8(b))
    k = np.arange(11) - 5
    g = np.exp(-(k[:, None] ** 2 + k[None, :] ** 2) / 4.5)
    g /= g.sum()
    vals = []
    for i in range(13 - 10):
        for j in range(14 - 10):
            A = ya[i:i + 11, j:j + 11]
            B = yb[i:i + 11, j:j + 11]
            ma, mb = (g * A).sum(), (g * B).sum()
            va, vb = (g * (A - ma) ** 2).sum(), (g * (B - mb) ** 2).sum()
            cab = (g * (A - ma) * (B - mb)).sum()
            vals.append((2 * ma * mb + QM.C1) * (2 * cab + QM.C2) / ((ma * ma + mb * mb + QM.C1) * (va + vb + QM.C2)))
    assert QM.ssim(a, b) == pytest.approx(np.mean(vals), abs=1e-12)
    assert -1.0 <= QM.ssim(a, b) <= 1.0


def test_error_map():
    a, b = rgba(8, 9, 5), rgba(8, 9, 6)
    e = QM.error_map(a, b)
    np.testing.assert_array_equal(e, QM.error_map(b, a))
    assert (QM.error_map(a, a) == 0).all()
    d = QM.quantize8(a) - QM.quantize8(b)
    assert e[2, 3] == pytest.approx(math.sqrt((d[2, 3] ** 2).sum()), rel=1e-15)


def test_ssim_luma_weights_and_c1_closed_form():
    """S:492 / S:514: SSIM on BT.601 luma 0.299 R + 0.587 G + 0.114 B with
    C1 = (0.01 * 255)^2.  Constant images: SSIM = (2 ya yb + C1) / (ya^2 +
    yb^2 + C1); against black, a pure red / green / blue level 200 image gives
    C1 / ((w * 200)^2 + C1) with w its luma weight."""
    c1 = (0.01 * 255.0) ** 2
    blk = np.zeros((12, 12, 4))
    for ch, wgt in enumerate((0.299, 0.587, 0.114)):
        a = np.zeros((12, 12, 4))
        a[..., ch] = 200 / 255.0
        y = wgt * 200.0
        assert QM.ssim(a, blk) == pytest.approx(c1 / (y * y + c1), rel=1e-12)


def test_ssim_c2_single_window_closed_form():
    """C2 = (0.03 * 255)^2, 11 x 11 Gaussian window, sigma = 1.5.  On
    an 11 x 11 image (one window) whose only non-zero luma is the centre pixel
    y, against black: mu_a = g0 y, var_a = g0 (1 - g0) y^2 (g0 = the
    normalised centre weight), mu_b = var_b = cov = 0, so
    SSIM = C1 / (mu_a^2 + C1) * C2 / (var_a + C2)."""
    c1, c2 = (0.01 * 255.0) ** 2, (0.03 * 255.0) ** 2
    k = np.arange(11) - 5
    g0 = 1.0 / np.exp(-(k[:, None] ** 2 + k[None, :] ** 2) / (2 * 1.5 ** 2)).sum()
    a = np.zeros((11, 11, 4))
    a[5, 5, :3] = 1.0                          # white centre: luma 255
    y = 255.0
    mu, var = g0 * y, g0 * (1 - g0) * y * y
    want = c1 / (mu * mu + c1) * c2 / (var + c2)
    assert QM.ssim(a, np.zeros((11, 11, 4))) == pytest.approx(want, rel=1e-12)
