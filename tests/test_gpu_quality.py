"""GPU parity for NEXT-2: the ground-truth renderer
(mfa_render_field: samples take their value and/or gradient from the
analytic Gaussian beam / Marschner-Lobb functions, Eq. 1-2)
and the image-quality metrics (mfa_image_quality: MSE / PSNR / SSIM), both
against the fp64 oracle (oracle.c orc_render_ex, oracle/metrics.py)."""
import functools

import numpy as np
import pytest

import oracle as O
import parity
from oracle import metrics as QM
from paper_2204_11762_b200 import workloads as WL

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@functools.lru_cache(maxsize=None)
def quality_case(kind, n, p, test, W, H):
    from paper_2204_11762_b200 import Model
    w, f_mfa, f_true = WL.make_quality(kind, n, p, test, W, H)
    return w, f_mfa, f_true, Model.from_workload(w), O.Model.from_workload(w)


def gpu_img(m, w, field):
    img = m.render(w.cameras, cuda(w.tf), w.v_lo, w.v_hi, w.params, field=field)
    torch.cuda.synchronize()
    return img[0]


@pytest.mark.parametrize("kind,n,p", [("ml", 32, 3), ("gb", 24, 2), ("ml", 20, 4)])
@pytest.mark.parametrize("test", WL.QUALITY_TESTS)
def test_field_render_parity(kind, n, p, test):
    """Both images of each of the paper's three tests -- the MFA image and the
    ground truth -- on the GPU vs the oracle (full frames, the image parity
    bar of north_star)."""
    w, f_mfa, f_true, m, om = quality_case(kind, n, p, test, 160, 120)
    for fld in (f_mfa, f_true):
        img = gpu_img(m, w, fld)
        ref = O.render(om, w.cameras[0], w.tf, w.v_lo, w.v_hi, w.params, field=fld)
        st = parity.check_image(img.cpu().numpy().reshape(-1, 4), ref, f"{kind}{n} p{p} {test} {fld}")
        print(kind, n, p, test, None if fld is None else (fld.value_src, fld.grad_src), st)


def test_field_render_nonuniform_and_tiles():
    """The analytic path on a non-uniform (Bezier-layout) model and through a
    tile list equals the full-frame render (bit-identical)."""
    from paper_2204_11762_b200 import Model
    w = WL.make_config(5, width=96, height=64, n_views=1, nctrl=(48, 24, 24))
    fld = WL.AnalyticField.gaussian_beam(1, 1)
    w.v_lo, w.v_hi = 0.0, 255.0
    m = Model.from_workload(w)
    om = O.Model.from_workload(w)
    img = gpu_img(m, w, fld)
    ref = O.render(om, w.cameras[0], w.tf, w.v_lo, w.v_hi, w.params, field=fld)
    parity.check_image(img.cpu().numpy().reshape(-1, 4), ref, "C5-small GB truth")
    tiles = np.array([(0, x, y) for y in range(4) for x in range(6)], np.int32)
    packed = m.render(w.cameras, cuda(w.tf), w.v_lo, w.v_hi, w.params, tiles=cuda(tiles), field=fld)
    from paper_2204_11762_b200 import unpack_tiles
    full = unpack_tiles(packed, cuda(tiles), 1, 96, 64)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(full[0].cpu().numpy(), img.cpu().numpy())


def test_field_render_bad_kind_raises():
    from paper_2204_11762_b200 import MfaError
    w, _, _, m, _ = quality_case("ml", 32, 3, "overall", 160, 120)
    bad = WL.AnalyticField(7, 1, 1, ())
    with pytest.raises(MfaError, match="INVALID_ARG"):
        m.render(w.cameras, cuda(w.tf), w.v_lo, w.v_hi, w.params, field=bad)


@pytest.mark.parametrize("shape", [(120, 160), (11, 11), (13, 300), (257, 31)])
def test_quality_metrics_parity(shape):
    """mfa_image_quality vs oracle/metrics.py on rendered-like images (random
    premultiplied RGBA with structure), including the smallest valid image and
    ragged tiles; fp64 on both sides."""
    from paper_2204_11762_b200 import image_quality
    H, W = shape
    r = np.random.default_rng(H * 1000 + W)
    base = r.uniform(0, 1, (H, W, 4)).astype(np.float32)
    other = np.clip(base + r.normal(0, 0.05, base.shape), -0.1, 1.1).astype(np.float32)
    got = image_quality(cuda(base), cuda(other), err_map=True)
    want = QM.quality(base, other)
    assert got["mse"] == pytest.approx(want["mse"], rel=1e-12)
    assert got["psnr"] == pytest.approx(want["psnr"], rel=1e-12)
    assert got["ssim"] == pytest.approx(want["ssim"], abs=1e-10)
    np.testing.assert_allclose(got["err_map"].cpu().numpy(), QM.error_map(base, other), rtol=1e-6, atol=1e-5)
    same = image_quality(cuda(base), cuda(base))
    assert same["mse"] == 0.0 and same["psnr"] == float("inf") and same["ssim"] == pytest.approx(1.0, abs=1e-12)


def test_quality_metrics_invalid():
    from paper_2204_11762_b200 import MfaError, image_quality
    a = torch.zeros((10, 40, 4), device="cuda")
    with pytest.raises(MfaError, match="INVALID_ARG"):
        image_quality(a, a)


def test_quality_table_on_gpu_images():
    """The paper's protocol end to end on the GPU (Tables 1-2 methodology for
    MFA-DVR alone): MFA image vs ground truth for the gradient-only and overall
    tests on Marschner-Lobb; GPU metrics equal the oracle metrics of the same
    GPU images, and refining the MFA improves every score."""
    from paper_2204_11762_b200 import image_quality
    rows = []
    for n in (16, 32, 64):
        for test in ("gradient", "overall"):
            w, f_mfa, f_true, m, _ = quality_case("ml", n, 3, test, 256, 256)
            a, b = gpu_img(m, w, f_mfa), gpu_img(m, w, f_true)
            q = image_quality(a, b)
            ref = QM.quality(a.cpu().numpy(), b.cpu().numpy())
            assert q["mse"] == pytest.approx(ref["mse"], rel=1e-12)
            assert q["ssim"] == pytest.approx(ref["ssim"], abs=1e-10)
            rows.append((n, test, q["mse"], q["psnr"], q["ssim"]))
    print("n test MSE PSNR SSIM")
    for r in rows:
        print(*r)
    for test in ("gradient", "overall"):
        seq = [r for r in rows if r[1] == test]
        assert seq[0][2] > seq[1][2] > seq[2][2], seq
        assert seq[0][4] < seq[2][4], seq


@pytest.mark.parametrize("c", [2, 5])
def test_lights_parity(c):
    """NEXT-4 lights (mfa_render_ex, R-30) against the oracle: three lights
    on C2 (uniform) and a reduced C5 (non-uniform Bezier), also combined with
    the analytic field; one light towards -d on an orthographic view equals
    the default headlight render."""
    from paper_2204_11762_b200 import Model
    w = WL.make_config(c, width=128, height=96, n_views=1) if c == 5 else WL.make_config(c, width=160, height=128)
    m = Model.from_workload(w)
    om = O.Model.from_workload(w)
    lights = [((0.3, -0.5, 0.8), 0.8), ((-0.7, 0.2, 0.1), 0.5), ((0.0, 0.0, -1.0), 0.3)]
    for fld in (None, WL.AnalyticField.marschner_lobb(0, 1)):
        img = m.render(w.cameras[:1], cuda(w.tf), w.v_lo, w.v_hi, w.params, lights=lights, field=fld)
        torch.cuda.synchronize()
        ref = O.render(om, w.cameras[0], w.tf, w.v_lo, w.v_hi, w.params, lights=lights, field=fld)
        st = parity.check_image(img[0].cpu().numpy().reshape(-1, 4), ref, f"C{c} lights field={fld}")
        print(c, fld is not None, st)


def test_single_headlight_light_equals_default():
    from paper_2204_11762_b200 import Model
    w = WL.make_config(1)
    m = Model.from_workload(w)
    o, d = O.ray(w.cameras[0], 0, 0)
    a = m.render(w.cameras, cuda(w.tf), w.v_lo, w.v_hi, w.params)
    b = m.render(w.cameras, cuda(w.tf), w.v_lo, w.v_hi, w.params, lights=[(-d, 1.0)])
    torch.cuda.synchronize()
    assert np.abs(a.cpu().numpy() - b.cpu().numpy()).max() <= 1e-6


def curvature_table(n=16, seed=3):
    r = np.random.default_rng(seed)
    k = np.linspace(0, 1, n)
    t = np.empty((n, n, 4), np.float32)
    for c in range(4):   # smooth: low-order polynomial in (kappa_1, kappa_2) plus a tiny seeded term
        a, b, d = r.uniform(-0.3, 0.3, 3)
        t[:, :, c] = np.clip(0.6 + a * k[None, :] + b * k[:, None] + d * np.outer(k, k), 0.05, 1.0)
    return t


@pytest.mark.parametrize("c,layout", [(2, "auto"), (5, "auto"), (4, "auto"), (5, "quads")])
def test_curvature_tf_parity(c, layout):
    """Curvature transfer function (mfa_render_ex, R-31; oracle C1): the
    GPU's fp32 gradient / Hessian / principal curvatures / bilinear table
    against the fp64 oracle, on uniform quads (C2), the Bezier layout (C5),
    streamed p = 4 slabs (C4) and non-uniform quads (C5)."""
    from paper_2204_11762_b200 import Model
    kw = dict(width=96, height=72, n_views=1)
    if c == 4:
        kw["nctrl"] = (40, 40, 40)
    if c == 5:
        kw["nctrl"] = (96, 32, 32)
    w = WL.make_config(c, **kw)
    m = Model.from_workload(w, layout=layout)
    om = O.Model.from_workload(w)
    tab = curvature_table()
    rng = {2: 60.0, 4: 80.0, 5: 120.0}[c]
    img = m.render(w.cameras[:1], cuda(w.tf), w.v_lo, w.v_hi, w.params, curvature=(cuda(tab), rng))
    torch.cuda.synchronize()
    ref = O.render(om, w.cameras[0], w.tf, w.v_lo, w.v_hi, w.params, curvature=(tab, rng))
    st = parity.check_image(img[0].cpu().numpy().reshape(-1, 4), ref, f"C{c} {layout} curvature TF")
    plain = O.render(om, w.cameras[0], w.tf, w.v_lo, w.v_hi, w.params)
    assert np.abs(plain["rgba"] - ref["rgba"]).max() > 1e-2      # the table really modulates the image
    print(c, layout, st)
