"""Pins for the parts of the oracle's ray caster that the constant-along-the-ray
closed forms of test_oracle_render.py cannot see (Algorithm 1,
P:102-131):

* sample placement t_k = t_in + (k + 1/2) * step and the sample count K
  (R-7; Alg. 1 l.3-4; "constant sample distance" P:100; first and
  last sample inside the volume) -- a field LINEAR along the ray, so
  every composited sample's colour depends on its own position;
* the TF domain normalisation s = (v - v_lo) / (v_hi - v_lo) and its clamp
  (Alg. 1 l.7; R-9) -- v_lo != 0 and values outside [v_lo, v_hi];
* Phong at an oblique N.L with hand values (Alg. 1 l.10-11; R-11,
  R-30);
* the R-19 flags (exit window, shading sensitivity) -- cases that must and
  must not set them;
* the curvature-table bilinear lookup (R-31) with a non-constant table.

Every expected value is written out here from the definitions (the sample
positions enumerated one by one, K counted by enumerating midpoints), not by
calling the oracle's formula again.  No GPU."""
import math

import numpy as np
import pytest

import oracle as O
from test_oracle_bspline import blossom_coeffs, uniform_knots
from test_oracle_render import box_model, const_tf, ortho_down, params_for

KA, KD, KS = 0.1, 0.7, 0.2


def midpoints(chord, step):
    """Positions (distance from the entry point) of the samples: the
    midpoints (k + 1/2) * step that lie inside the chord, enumerated."""
    out = []
    k = 0
    while (k + 0.5) * step < chord:
        out.append((k + 0.5) * step)
        k += 1
    return np.array(out)


def composite(colours, alphas, o_max):
    """Front-to-back over operator with strict ERT after the sample (Alg. 1
    l.13-15), written out: returns (C, A, samples composited)."""
    C = np.zeros(3)
    A = 0.0
    n = 0
    for c, a in zip(colours, alphas):
        w = (1.0 - A) * a
        C = C + w * np.asarray(c)
        A += w
        n += 1
        if A > o_max:
            break
    return C, A, n


def linear_tf(n=256):
    """Entry i: rgb = (x, 1 - x, 1/2), alpha = 0.02 + 0.08 x, x = i/(n-1):
    linear in x, so linear interpolation reproduces it (fp32 entries)."""
    x = np.arange(n) / (n - 1)
    return np.stack([x, 1 - x, np.full(n, 0.5), 0.02 + 0.08 * x], axis=1).astype(np.float32)


def tf_closed(s):
    return np.array([s, 1 - s, 0.5]), 0.02 + 0.08 * s


# --------------------------------------------------------------------------
# sample placement + TF normalisation / clamp (mutations: samples at t_in + k
# step; s = (v - v_lo) / v_hi)
# --------------------------------------------------------------------------
@pytest.mark.parametrize("v_lo,v_hi", [(0.0, 1.0), (0.2, 0.7), (-0.5, 0.8), (0.35, 1.6)])
@pytest.mark.parametrize("o_max", [1.0, 0.5])
def test_midpoint_samples_on_a_field_linear_along_the_ray(v_lo, v_hi, o_max):
    """f = w (Greville control values reproduce it), orthographic view along
    -z: the ray enters at the top face (w = 1) and sample k sits at
    w_k = 1 - (k + 1/2) step / L_z, so its value, TF colour and opacity all
    change along the ray.  Shading off."""
    m, L = box_model(p=2, n=(8, 6, 5), field="w")
    W = H = 24
    step = 0.021
    prm = params_for(L, step=step, shading=0, o_max=o_max)
    r = O.render(m, ortho_down(W, H, 0.6), linear_tf(), v_lo, v_hi, prm)
    t = midpoints(L[2], step)
    w_k = 1.0 - t / L[2]
    s_k = np.clip((w_k - v_lo) / (v_hi - v_lo), 0.0, 1.0)
    if (v_lo, v_hi) != (0.0, 1.0):
        assert (s_k == 0).any() or (s_k == 1).any()      # the clamp is exercised
    cols, alps = zip(*[tf_closed(s) for s in s_k])
    C, A, n = composite(cols, alps, o_max)
    hit = r["count"] > 0
    assert hit.sum() > 100
    assert np.all(r["count"][hit] == n)
    if o_max >= 1.0:
        assert n == len(t) == 24                          # ceil(0.5 / 0.021 - 1/2) by enumeration
    ref = np.concatenate([C, [A]])
    np.testing.assert_allclose(r["rgba"][hit], np.tile(ref, (hit.sum(), 1)), rtol=0, atol=2e-7)
    assert not (r["flags"] & (O.FLAG_EXIT | O.FLAG_SHADE)).any()


def test_midpoint_samples_perspective_single_ray():
    """The same on an oblique perspective ray: the one pixel whose ray is the
    camera axis hits the look-at point; along it f = u + v + w is linear in
    t, sampled at the midpoints of the clipped chord (centre ray, odd image,
    SPEC S:400)."""
    p, n = 2, (7, 7, 7)
    U = uniform_knots(p, 7)
    one, lin = blossom_coeffs(U, p, 0), blossom_coeffs(U, p, 1)
    ctrl = (lin[None, None, :] * one[None, :, None] * one[:, None, None]
            + one[None, None, :] * lin[None, :, None] * one[:, None, None]
            + one[None, None, :] * one[None, :, None] * lin[:, None, None])
    m = O.Model(p, [U, U, U], ctrl)
    from paper_2204_11762_b200.workloads import Camera
    eye = np.array([1.3, -0.9, 0.7])
    cam = Camera(eye=tuple(eye), look_at=(0.05, 0.02, -0.03), up=(0, 0, 1), fov_y_deg=40.0,
                 ortho_half_height=0.0, width=9, height=7)
    step = 0.0173
    prm = params_for(np.ones(3), step=step, shading=0, o_max=1.0)
    pix = [3 * 9 + 4]
    r = O.render(m, cam, linear_tf(), 0.0, 3.0, prm, pixels=pix)
    d = np.array(cam.look_at) - eye
    d /= np.linalg.norm(d)
    # slab clip of the unit box [-1/2, 1/2]^3 written out
    t0 = (-0.5 - eye) / d
    t1 = (0.5 - eye) / d
    t_in, t_out = max(np.minimum(t0, t1).max(), 0.0), np.maximum(t0, t1).min()
    t = t_in + midpoints(t_out - t_in, step)
    x = eye[None, :] + t[:, None] * d[None, :]
    f = (x + 0.5).sum(axis=1)          # u + v + w
    cols, alps = zip(*[tf_closed(s) for s in np.clip(f / 3.0, 0, 1)])
    C, A, k = composite(cols, alps, 1.0)
    assert r["count"][0] == k == len(t)
    np.testing.assert_allclose(r["rgba"][0], np.concatenate([C, [A]]), rtol=0, atol=2e-7)


def test_shaded_midpoints_facing_light():
    """f = 1 - w: N = -g/|g| = +z faces the headlight (N.L = 1, R.V = 1), so
    every sample has c = clamp(rgb(s_k) (k_a + k_d) + k_s) with s_k = f at the
    sample's own position (SPEC S:427 with a varying colour)."""
    m, L = box_model(p=2, n=(8, 6, 5), field="1-w")
    step = 0.021
    v_lo, v_hi = 0.1, 0.9
    prm = params_for(L, step=step, o_max=0.9)
    r = O.render(m, ortho_down(16, 16, 0.6), linear_tf(), v_lo, v_hi, prm)
    f_k = midpoints(L[2], step) / L[2]
    s_k = np.clip((f_k - v_lo) / (v_hi - v_lo), 0.0, 1.0)
    cols, alps = [], []
    for s in s_k:
        rgb, a = tf_closed(s)
        cols.append(np.clip(rgb * (KA + KD) + KS, 0, 1))
        alps.append(a)
    C, A, n = composite(cols, alps, 0.9)
    hit = r["count"] > 0
    assert np.all(r["count"][hit] == n)
    np.testing.assert_allclose(r["rgba"][hit], np.tile(np.concatenate([C, [A]]), (hit.sum(), 1)), rtol=0,
                               atol=2e-7)
    assert not (r["flags"] & O.FLAG_SHADE).any()         # |g| = 1/L_z, far above sens_grad


# --------------------------------------------------------------------------
# Phong at an oblique N.L (hand values)
# --------------------------------------------------------------------------
def u_minus_w_model():
    """f = u - w, p = 2, spans (6, 6, 4): L = (1, 1, 2/3).  g_phys =
    (1, 0, -3/2), N = -g/|g| = (-2, 0, 3)/sqrt(13)."""
    p = 2
    n = (8, 8, 6)
    knots = [uniform_knots(p, n[d]) for d in range(3)]
    gu = np.array([knots[0][i + 1:i + p + 1].sum() / p for i in range(n[0])])
    gw = np.array([knots[2][i + 1:i + p + 1].sum() / p for i in range(n[2])])
    ctrl = np.broadcast_to(gu[None, None, :] - gw[:, None, None], (n[2], n[1], n[0])).copy()
    return O.Model(p, knots, ctrl), np.array([1.0, 1.0, 2.0 / 3.0])


@pytest.mark.parametrize("shin", [2.0, 10.0])
def test_oblique_headlight_specular_by_hand(shin):
    """Headlight l = V = +z: N.l = 3/sqrt(13); R.V = 2 (N.l)^2 - 1 = 5/13.
    Constant TF -> every sample has c = clamp(rgb (k_a + k_d 3/sqrt13) +
    k_s (5/13)^n) and the pixel is c (1 - (1 - a)^K)."""
    m, L = u_minus_w_model()
    rgb = np.array([0.3, 0.5, 0.7]).astype(np.float32).astype(np.float64)
    a = float(np.float32(0.05))
    step = 0.019
    prm = params_for(L, step=step, o_max=1.0, shininess=shin)
    r = O.render(m, ortho_down(16, 16, 0.3), const_tf(rgb, a), -1.0, 1.0, prm)
    K = len(midpoints(L[2], step))
    c = np.clip(rgb * (KA + KD * 3 / math.sqrt(13)) + KS * (5 / 13) ** shin, 0, 1)
    A = 1 - (1 - a) ** K
    assert (r["count"] == K).all()
    np.testing.assert_allclose(r["rgba"], np.tile(np.concatenate([c * A, [A]]), (256, 1)), rtol=0, atol=1e-13)


def test_oblique_side_light_by_hand():
    """One directional light towards -x (L = (-1,0,0)), V = +z: N.L =
    2/sqrt(13), R = 2 (N.L) N - L, R.V = 2 (2/sqrt13)(3/sqrt13) = 12/13.
    A second light from behind the surface (N.L < 0) adds nothing (R-30)."""
    m, L = u_minus_w_model()
    rgb = np.array([0.6, 0.2, 0.4]).astype(np.float32).astype(np.float64)
    a = float(np.float32(0.07))
    step = 0.023
    for inten in (0.5, 1.5):
        prm = params_for(L, step=step, o_max=1.0, shininess=3.0)
        r = O.render(m, ortho_down(12, 12, 0.3), const_tf(rgb, a), -1.0, 1.0, prm,
                     lights=[((-1.0, 0.0, 0.0), inten), ((1.0, 0.0, 0.0), 4.0)])
        K = len(midpoints(L[2], step))
        c = np.clip(rgb * (KA + KD * inten * 2 / math.sqrt(13)) + KS * inten * (12 / 13) ** 3, 0, 1)
        A = 1 - (1 - a) ** K
        assert (r["count"] == K).all()
        np.testing.assert_allclose(r["rgba"], np.tile(np.concatenate([c * A, [A]]), (144, 1)), rtol=0,
                                   atol=1e-13)


# --------------------------------------------------------------------------
# R-19 flags
# --------------------------------------------------------------------------
def test_exit_window_flag_and_alternative():
    """L_z / step = 10.5 (to rounding): the midpoint count is 10 or 11
    depending on the last bit, so the oracle must flag the exit window and
    store the other count as the alternative (R-19 (ii))."""
    m, L = box_model(p=2, n=(8, 6, 5), field="const")
    step = L[2] / 10.5
    prm = params_for(L, step=step, shading=0, o_max=1.0)
    r = O.render(m, ortho_down(12, 12, 0.6), const_tf([1, 1, 1], 0.1), 0.0, 1.0, prm)
    hit = r["count"] > 0
    assert hit.sum() > 10
    assert (r["flags"][hit] & O.FLAG_EXIT).all()
    assert not (r["flags"][~hit] & O.FLAG_EXIT).any()
    pair = np.sort(np.stack([r["count"][hit], r["alt_count"][hit, 1]], axis=1), axis=1)
    assert (pair == [10, 11]).all()
    # the alternative image is the other count's closed form
    a = float(np.float32(0.1))
    for j in np.nonzero(hit)[0][:5]:
        Ka = r["alt_count"][j, 1]
        np.testing.assert_allclose(r["alt"][j, 1, 3], 1 - (1 - a) ** Ka, atol=1e-14)
    # away from the window: no flag, no alternative
    prm2 = params_for(L, step=L[2] / 10.2, shading=0, o_max=1.0)
    r2 = O.render(m, ortho_down(12, 12, 0.6), const_tf([1, 1, 1], 0.1), 0.0, 1.0, prm2)
    assert not (r2["flags"] & O.FLAG_EXIT).any()
    assert (r2["alt_count"][:, 1] == -1).all()
    assert (r2["count"][r2["count"] > 0] == len(midpoints(L[2], L[2] / 10.2))).all()


def test_shading_sensitive_flag_set_and_not_set():
    """R-19 (iii): a composited sample with weight > sens_weight and
    |g_phys| < sens_grad flags the pixel.  A constant field (g = 0) with
    shading on must be flagged; with shading off it must not; a linear field
    (|g_phys| = 1/L_x) must not; a tiny opacity (weights below sens_weight)
    must not."""
    m, L = box_model(p=2, n=(8, 8, 8))
    cam = ortho_down(8, 8, 0.3)
    r = O.render(m, cam, const_tf([1, 1, 1], 0.1), 0.0, 1.0, params_for(L, step=0.05, shading=1))
    assert (r["flags"] & O.FLAG_SHADE).all()
    r = O.render(m, cam, const_tf([1, 1, 1], 0.1), 0.0, 1.0, params_for(L, step=0.05, shading=0))
    assert not (r["flags"] & O.FLAG_SHADE).any()
    r = O.render(m, cam, const_tf([1, 1, 1], 5e-4), 0.0, 1.0, params_for(L, step=0.05, shading=1))
    assert not (r["flags"] & O.FLAG_SHADE).any()
    mu, Lu = box_model(p=2, n=(8, 6, 5), field="u")
    r = O.render(mu, ortho_down(16, 16, 0.6), linear_tf(), 0.0, 1.0, params_for(Lu, step=0.021, shading=1))
    assert (r["count"] > 0).any()
    assert not (r["flags"] & O.FLAG_SHADE).any()


# --------------------------------------------------------------------------
# curvature table lookup with a non-constant table (R-31)
# --------------------------------------------------------------------------
def test_curvature_bilinear_lookup_non_constant_table():
    """f = (u - c_u)^2 + (w - c_w)^2 (blossom control values, exact for
    p = 2) has cylindrical level sets around an axis parallel to v: principal
    curvatures (kappa_1, kappa_2) = (0, -1/r), r = the distance to the axis
    in the (u, w) plane (unit box, L = 1).  The table is a BILINEAR function
    of x_d = (kappa_d + R)/(2R), so bilinear interpolation reproduces it and
    each sample's opacity factor is known in closed form; the table is not
    symmetric, so swapped axes or a wrong cell would show.  Shading off,
    constant TF."""
    p, nn = 2, 7
    U = uniform_knots(p, nn)
    cu, cw = 0.43, 1.35
    one, lin, sq = (blossom_coeffs(U, p, k) for k in range(3))
    qu = sq - 2 * cu * lin + cu ** 2 * one
    qw = sq - 2 * cw * lin + cw ** 2 * one
    ctrl = (qu[None, None, :] * one[None, :, None] * one[:, None, None]
            + one[None, None, :] * one[None, :, None] * qw[:, None, None])
    m = O.Model(p, [U, U, U], ctrl)
    R = 6.0
    n = 17
    x = np.arange(n) / (n - 1)
    X1, X2 = np.meshgrid(x, x)            # [kappa_2 index][kappa_1 index]

    def tab_fn(x1, x2):                   # bilinear, not symmetric in (x1, x2)
        return np.stack([0.2 + 0.5 * x1 + 0.1 * x2, 0.9 - 0.3 * x2, 0.4 + 0.2 * x1 * x2,
                         0.1 + 0.6 * x1 + 0.25 * x2 - 0.3 * x1 * x2], axis=-1)

    tab = tab_fn(X1, X2).astype(np.float32)
    rgb = np.array([0.9, 0.6, 0.3])
    a = 0.08
    step = 0.031
    prm = params_for(np.ones(3), step=step, shading=0, o_max=0.95)
    W = H = 10
    cam = ortho_down(W, H, 0.45)
    r = O.render(m, cam, const_tf(rgb, a), 0.0, 4.0, prm, curvature=(tab, R))
    t = midpoints(1.0, step)
    w_k = 1.0 - t
    n_checked = 0
    for py in range(H):
        for px in range(W):
            X = (2 * (px + 0.5) / W - 1) * 0.45
            u = X + 0.5
            rad = np.hypot(u - cu, w_k - cw)
            k1, k2 = np.zeros_like(rad), -1.0 / rad
            f = tab_fn((k1 + R) / (2 * R), (k2 + R) / (2 * R))
            cols = [rgb * fi[:3] for fi in f]
            alps = [a * fi[3] for fi in f]
            C, A, cnt = composite(cols, alps, 0.95)
            j = py * W + px
            assert r["count"][j] == cnt
            np.testing.assert_allclose(r["rgba"][j], np.concatenate([C, [A]]), rtol=0, atol=5e-7)
            n_checked += 1
    assert n_checked == W * H
