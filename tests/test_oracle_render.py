"""Pins for the oracle's ray caster (Algorithm 1):
camera/ray/clip geometry, compositing and ERT closed forms
(S:417-419), shading special cases, an end-to-end
closed-form render of a linear field, and the row-thread bit-identity
invariant.  No GPU."""
import math

import numpy as np
import pytest

import oracle as O
from paper_2204_11762_b200.workloads import Camera, RenderParams, make_config


def uniform_knots(p, n):
    S = n - p
    return np.concatenate([np.zeros(p + 1), np.arange(1, S) / S, np.ones(p + 1)])


def greville(U, p):
    n = len(U) - p - 1
    return np.array([U[i + 1:i + p + 1].sum() / p for i in range(n)])


def box_model(p=2, n=(8, 6, 5), field="const", value=0.5):
    knots = [uniform_knots(p, n[d]) for d in range(3)]
    spans = [n[d] - p for d in range(3)]
    L = np.array(spans, float) / max(spans)
    shape = (n[2], n[1], n[0])
    if field == "const":
        ctrl = np.full(shape, value)
    elif field == "u":
        ctrl = np.broadcast_to(greville(knots[0], p)[None, None, :], shape).copy()
    elif field == "w":
        ctrl = np.broadcast_to(greville(knots[2], p)[:, None, None], shape).copy()
    elif field == "1-w":
        ctrl = np.broadcast_to(1.0 - greville(knots[2], p)[:, None, None], shape).copy()
    else:
        raise ValueError(field)
    return O.Model(p, knots, ctrl), L


def ortho_down(W=32, H=32, h=0.6):
    # looking along -z, up = +y: right = +x
    return Camera(eye=(0.0, 0.0, 2.0), look_at=(0.0, 0.0, 0.0), up=(0.0, 1.0, 0.0), fov_y_deg=0.0,
                  ortho_half_height=h, width=W, height=H)


def params_for(L, step, **kw):
    kw.setdefault("grad_eps", 1e-9)   # |g| of a constant field is rounding noise (~1e-16)
    return RenderParams(box_min=tuple(-L / 2), box_max=tuple(L / 2), step=step, **kw)


def const_tf(rgb, a, n=256):
    t = np.empty((n, 4), np.float32)
    t[:, :3] = rgb
    t[:, 3] = a
    return t


# --------------------------------------------------------------------------
# geometry
# --------------------------------------------------------------------------
def test_ortho_rays_share_direction():
    cam = Camera(eye=(1.0, 2.0, 3.0), look_at=(0.1, -0.2, 0.3), up=(0, 0, 1), fov_y_deg=0.0,
                 ortho_half_height=0.7, width=7, height=5)
    d0 = O.ray(cam, 0, 0)[1]
    for px, py in [(6, 4), (3, 2), (0, 4)]:
        np.testing.assert_allclose(O.ray(cam, px, py)[1], d0, atol=1e-15)
    f = np.array(cam.look_at) - np.array(cam.eye)
    np.testing.assert_allclose(d0, f / np.linalg.norm(f), atol=1e-15)


def test_perspective_center_ray_hits_look_at():
    cam = Camera(eye=(1.0, -2.0, 0.5), look_at=(0.2, 0.1, -0.3), up=(0, 0, 1), fov_y_deg=40.0,
                 ortho_half_height=0, width=9, height=7)
    o, d = O.ray(cam, 4, 3)
    f = np.array(cam.look_at) - np.array(cam.eye)
    np.testing.assert_allclose(o, cam.eye, atol=0)
    np.testing.assert_allclose(d, f / np.linalg.norm(f), atol=1e-12)


def test_perspective_fov90_corner_by_hand():
    """eye 0, looking along -z, up +y, fov_y 90 deg, 2x2 image:
    pixel (0,0) centre at X=-1/2, Y=+1/2 -> d = (-1/2, 1/2, -1)/sqrt(3/2)."""
    cam = Camera(eye=(0, 0, 0), look_at=(0, 0, -1), up=(0, 1, 0), fov_y_deg=90.0,
                 ortho_half_height=0, width=2, height=2)
    _, d = O.ray(cam, 0, 0)
    np.testing.assert_allclose(d, np.array([-0.5, 0.5, -1.0]) / math.sqrt(1.5), atol=1e-12)
    _, d = O.ray(cam, 1, 1)
    np.testing.assert_allclose(d, np.array([0.5, -0.5, -1.0]) / math.sqrt(1.5), atol=1e-12)


def test_clip_cases():
    bmin, bmax = (-0.5, -0.5, -0.5), (0.5, 0.5, 0.5)
    hit, ti, to = O.clip(bmin, bmax, (-3.0, 0.0, 0.0), (1.0, 0.0, 0.0))
    assert hit and ti == pytest.approx(2.5) and to - ti == pytest.approx(1.0, abs=1e-12)
    hit, _, _ = O.clip(bmin, bmax, (-3.0, 0.7, 0.0), (1.0, 0.0, 0.0))     # S:409 parallel outside
    assert not hit
    hit, ti, to = O.clip(bmin, bmax, (0.1, 0.2, 0.3), (0.0, 0.0, 1.0))    # origin inside
    assert hit and ti == 0.0 and to == pytest.approx(0.2)
    hit, _, _ = O.clip(bmin, bmax, (-3.0, 0.0, 0.0), (-1.0, 0.0, 0.0))    # box behind
    assert not hit
    d = np.array([1.0, 1.0, 1.0]) / math.sqrt(3)
    hit, ti, to = O.clip(bmin, bmax, -2 * d, d)                            # diagonal chord = sqrt(3)
    assert hit and to - ti == pytest.approx(math.sqrt(3), abs=1e-12)


# --------------------------------------------------------------------------
# compositing / ERT closed forms
# --------------------------------------------------------------------------
def test_constant_field_ert_at_sample_44():
    """Constant field, TF alpha 0.1: A_k = 1 - 0.9^k; with o_max = 0.99 the
    first k with A_k > o_max is 44 (A = 0.990302..., 43 gives 0.989225...).
    Shading on with zero gradient -> ambient k_a*rgb."""
    m, L = box_model(p=2, n=(8, 8, 8))
    assert 1 - 0.9 ** 44 > 0.99 > 1 - 0.9 ** 43
    cam = ortho_down(16, 16, 0.3)
    rgb = np.array([0.8, 0.4, 0.2])
    prm = params_for(L, step=1.0 / 200, shading=1)       # chord 1 -> K = 200 samples
    r = O.render(m, cam, const_tf(rgb, 0.1), 0.0, 1.0, prm)
    hitp = r["count"] > 0
    assert hitp.all()
    assert (r["count"] == 44).all()
    a32 = float(np.float32(0.1))                     # the table is fp32
    rgb32 = rgb.astype(np.float32).astype(np.float64)
    A44 = 1 - (1 - a32) ** 44
    np.testing.assert_allclose(r["rgba"][:, 3], A44, rtol=0, atol=1e-14)
    np.testing.assert_allclose(r["rgba"][:, :3], np.outer(np.ones(256), 0.1 * rgb32 * A44), atol=1e-14)


def test_two_half_alpha_samples():
    """two a = 0.5 samples -> A = 0.75 (chord 1, step 1/2 -> K = 2)."""
    m, L = box_model(p=2, n=(8, 8, 8))
    prm = params_for(L, step=0.5, shading=0)
    r = O.render(m, ortho_down(8, 8, 0.3), const_tf([1.0, 0.5, 0.25], 0.5), 0.0, 1.0, prm)
    assert (r["count"] == 2).all()
    np.testing.assert_allclose(r["rgba"], np.tile([0.75, 0.375, 0.1875, 0.75], (64, 1)), atol=1e-15)


def test_zero_opacity_is_background_and_counts_all_samples():
    """SPEC S:435 (zero-opacity TF -> background) and K = ceil(L/step - 1/2) (R-7)."""
    m, L = box_model(p=2, n=(8, 6, 5), field="u")
    step = 0.013
    prm = params_for(L, step=step)
    cam = ortho_down(32, 32, 0.6)
    r = O.render(m, cam, const_tf([1, 1, 1], 0.0), 0.0, 1.0, prm)
    assert np.all(r["rgba"] == 0.0)
    K = math.ceil(L[2] / step - 0.5)
    hit = r["count"] > 0
    assert hit.sum() > 0 and np.all(r["count"][hit] == K)


def test_opaque_silhouette():
    """fully opaque constant-colour TF, shading off -> the box
    silhouette in that colour, one sample per hit ray."""
    m, L = box_model(p=2, n=(8, 6, 5), field="u")
    cam = ortho_down(32, 32, 0.6)
    prm = params_for(L, step=0.01, shading=0)
    r = O.render(m, cam, const_tf([0.2, 0.6, 0.9], 1.0), 0.0, 1.0, prm)
    hit = r["count"] > 0
    assert np.all(r["count"][hit] == 1)
    np.testing.assert_allclose(r["rgba"][hit], np.tile([0.2, 0.6, 0.9, 1.0], (hit.sum(), 1)), atol=1e-15)
    assert np.all(r["rgba"][~hit] == 0.0)
    # silhouette = pixels whose ortho ray passes inside |x| < Lx/2, |y| < Ly/2
    W = H = 32
    px, py = np.meshgrid(np.arange(W), np.arange(H))
    X = (2 * (px + 0.5) / W - 1) * 0.6
    Y = (1 - 2 * (py + 0.5) / H) * 0.6
    inside = (np.abs(X) < L[0] / 2) & (np.abs(Y) < L[1] / 2)
    np.testing.assert_array_equal(hit, inside.ravel())


def _closed_form_linear(L, W, H, h, step, o_max, a_of_s, c_of_s):
    px, py = np.meshgrid(np.arange(W), np.arange(H))
    X = (2 * (px + 0.5) / W - 1) * h
    Y = (1 - 2 * (py + 0.5) / H) * h
    inside = ((np.abs(X) < L[0] / 2) & (np.abs(Y) < L[1] / 2)).ravel()
    u = ((X + L[0] / 2) / L[0]).ravel()
    K = math.ceil(L[2] / step - 0.5)
    out = np.zeros((W * H, 4))
    cnt = np.zeros(W * H, np.int64)
    for i in np.nonzero(inside)[0]:
        a = a_of_s(u[i])
        ks = np.arange(1, K + 1)
        Ak = 1 - (1 - a) ** ks
        over = np.nonzero(Ak > o_max)[0]
        Keff = int(over[0]) + 1 if len(over) else K
        A = 1 - (1 - a) ** Keff
        out[i, :3] = c_of_s(u[i]) * A
        out[i, 3] = A
        cnt[i] = Keff
    return out, cnt


@pytest.mark.parametrize("o_max", [0.99, 0.5, 1.0])
def test_linear_field_end_to_end_closed_form(o_max):
    """End to end: f = u (Greville control values reproduce it exactly),
    orthographic view along -z.  Along each ray u is constant, so every
    sample has the same s = u, TF(s) (a TF linear in the entry index is
    exact under linear interpolation), and physical gradient (1/L_x,0,0)
    perpendicular to the headlight -> diffuse = specular = 0:
    pixel = k_a*rgb(u)*(1-(1-a(u))^K_eff)."""
    m, L = box_model(p=2, n=(8, 6, 5), field="u")
    n = 256
    i = np.arange(n) / (n - 1)
    tf = np.stack([i, 1 - i, np.full(n, 0.5), 0.02 + 0.08 * i], axis=1).astype(np.float32)
    W = H = 32
    step = 0.021
    prm = params_for(L, step=step, o_max=o_max)
    r = O.render(m, ortho_down(W, H, 0.6), tf, 0.0, 1.0, prm)
    ref, cnt = _closed_form_linear(
        L, W, H, 0.6, step, o_max,
        a_of_s=lambda s: 0.02 + 0.08 * s,
        c_of_s=lambda s: 0.1 * np.array([s, 1 - s, 0.5]))
    np.testing.assert_array_equal(r["count"], cnt)
    np.testing.assert_allclose(r["rgba"], ref, rtol=0, atol=2e-7)  # fp32 TF table entries


def test_shading_special_cases():
    """normal facing the light, k_s = 0 -> (k_a + k_d)*rgb;
    with k_s > 0 the full specular adds k_s (R.V = 1).  Light from behind
    (f = w, N.L = -1) -> ambient only."""
    W = H = 16
    rgb = np.array([0.3, 0.5, 0.7]).astype(np.float32).astype(np.float64)
    a = float(np.float32(0.05))
    for field, ks, expect in [("1-w", 0.0, (0.1 + 0.7) * rgb), ("1-w", 0.2, np.minimum((0.1 + 0.7) * rgb + 0.2, 1)),
                              ("w", 0.2, 0.1 * rgb)]:
        m, L = box_model(p=3, n=(8, 8, 8), field=field)
        prm = params_for(L, step=0.02, ks=ks)
        r = O.render(m, ortho_down(W, H, 0.3), const_tf(rgb, a), 0.0, 1.0, prm)
        K = math.ceil(1.0 / 0.02 - 0.5)
        A = 1 - (1 - a) ** K
        assert (r["count"] == K).all()
        np.testing.assert_allclose(r["rgba"][:, :3], np.outer(np.ones(W * H), expect * A), atol=1e-12)


def test_ert_bound():
    """enabling ERT changes any channel by at most 1 - o_max."""
    w = make_config(2, width=48, height=48)
    m = O.Model.from_workload(w)
    import dataclasses
    p1 = dataclasses.replace(w.params, o_max=0.9)
    p2 = dataclasses.replace(w.params, o_max=1.0)
    r1 = O.render(m, w.cameras[0], w.tf, w.v_lo, w.v_hi, p1)
    r2 = O.render(m, w.cameras[0], w.tf, w.v_lo, w.v_hi, p2)
    assert np.abs(r1["rgba"] - r2["rgba"]).max() <= 0.1 + 1e-12
    assert (r1["count"] <= r2["count"]).all()
    # opacity never decreases when more samples are composited
    assert (r1["rgba"][:, 3] <= r2["rgba"][:, 3] + 1e-15).all()


def test_thread_count_bit_identity():
    """1 vs N row-block threads give bit-identical images."""
    w = make_config(1)
    m = O.Model.from_workload(w)
    a = O.render(m, w.cameras[0], w.tf, w.v_lo, w.v_hi, w.params, nthreads=1)
    b = O.render(m, w.cameras[0], w.tf, w.v_lo, w.v_hi, w.params, nthreads=5)
    for k in a:
        np.testing.assert_array_equal(a[k], b[k])
    pix = np.arange(0, 64 * 64, 7)
    c = O.render(m, w.cameras[0], w.tf, w.v_lo, w.v_hi, w.params, pixels=pix, nthreads=3)
    np.testing.assert_array_equal(c["rgba"], a["rgba"][pix])
    np.testing.assert_array_equal(c["count"], a["count"][pix])


def test_ert_alternative_recorded():
    """R-19 (i): a pixel whose opacity passes within the window of o_max
    carries the alternative outcome (one more / one fewer sample)."""
    m, L = box_model(p=2, n=(8, 8, 8))
    a = float(np.float32(0.1))
    A44 = 1 - (1 - a) ** 44
    prm = params_for(L, step=1.0 / 200, shading=0, o_max=A44 - 5e-5)
    r = O.render(m, ortho_down(4, 4, 0.3), const_tf([1, 1, 1], a), 0.0, 1.0, prm)
    assert (r["flags"] & O.FLAG_ERT).all()
    assert (r["count"] == 44).all() and (r["alt_count"][:, 0] == 45).all()
