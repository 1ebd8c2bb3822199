"""GPU parity: the CUDA path (through the C ABI, via the ctypes binding)
against the fp64 oracle on the same seeded inputs, on all five configs.
Marked gpu: run on a B200 with `pytest -m gpu`."""
import functools

import numpy as np
import pytest

import oracle as O
import parity
from paper_2204_11762_b200 import workloads as WL

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@functools.lru_cache(maxsize=None)
def workload(c, **kw):
    return WL.make_config(c, **kw)


@functools.lru_cache(maxsize=None)
def gpu_model(c, layout="auto"):
    from paper_2204_11762_b200 import Model
    return Model.from_workload(workload(c), layout=layout)


@functools.lru_cache(maxsize=None)
def oracle_model(c):
    return O.Model.from_workload(workload(c))


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def gpu_eval(m, u, v, w, grad=True):
    outs = m.eval(cuda(u), cuda(v), cuda(w), grad=grad)
    torch.cuda.synchronize()
    return np.stack([o.cpu().numpy() for o in outs], axis=1)


EVAL_N = {1: 1 << 20, 2: 1 << 20, 3: 1 << 24, 4: 1 << 20, 5: 1 << 20}   # SURVEY §8(c) acceptance sizes


@pytest.mark.parametrize("c", [1, 2, 3, 4, 5])
def test_eval_parity(c):
    """Random points (C3: the full 2^24 set of BASELINE.json) plus the
    boundary set (u in {0, 1, 1-ulp, knots}), value + gradient."""
    w = workload(c)
    u, v, ww = WL.query_points(c, EVAL_N[c])
    bu, bv, bw = WL.boundary_points(w)
    u, v, ww = (np.concatenate([a, b]) for a, b in ((u, bu), (v, bv), (ww, bw)))
    got = gpu_eval(gpu_model(c), u, v, ww)
    ref, sig, errs = oracle_model(c).eval_batch(u, v, ww)
    assert errs == 0
    wv, wg = parity.check_eval(got, ref, sig, f"C{c}")
    print(f"C{c}: n={len(u)} worst value {wv:.2e} sigma, worst gradient {wg:.2e} sigma")


@pytest.mark.parametrize("c,layout,n,box", [(3, "auto", 1 << 18, 1.0), (5, "auto", 1 << 18, 1.0),
                                             (5, "quads", 1 << 18, 1.0), (2, "auto", 1 << 18, 1.0),
                                             (3, "auto", 1 << 22, 0.25)])
def test_eval_binned_equals_direct(c, layout, n, box):
    """The three eval paths return identical outputs, NaN rows and domain-error
    counts: mfa_eval_batch (binned, stream-ordered scratch), mfa_eval_batch_ws
    with a caller workspace (binned) and without one (the unbinned kernel).
    (3, 2^22 points in [0, 1/4]^3): ~8192 points per bin (dense bins; with
    MFA_EVAL_LINES=1 the line-slot kernel takes them in several shared-memory
    pieces, which passed when that experiment was measured)."""
    m = gpu_model(c, layout)
    u, v, w = (a * np.float32(box) for a in WL.query_points(c, n))
    u = u.copy()
    u[[5, 77, 1000]] = [1.5, np.nan, -0.25]
    cu, cv, cw = cuda(u), cuda(v), cuda(w)
    outs = []
    for binned in ("auto", True, False):
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        r = m.eval(cu, cv, cw, n_domain_errors=cnt, binned=binned)
        torch.cuda.synchronize()
        outs.append((np.stack([t.cpu().numpy() for t in r], axis=1), int(cnt.item())))
    for o in outs[1:]:
        np.testing.assert_array_equal(outs[0][0], o[0])
        assert o[1] == 3
    assert outs[0][1] == 3


def test_eval_value_only_matches():
    c = 2
    u, v, w = WL.query_points(c, 1 << 14)
    full = gpu_eval(gpu_model(c), u, v, w)
    vo = gpu_eval(gpu_model(c), u, v, w, grad=False)
    ref, sig, _ = oracle_model(c).eval_batch(u, v, w)
    parity.check_eval(vo, ref[:, :1], sig[:, :1], "value-only")
    assert np.abs(vo[:, 0] - full[:, 0]).max() <= 1e-5 * max(1.0, np.abs(ref[:, 0]).max())


def test_eval_domain_errors_and_empty():
    m = gpu_model(1)
    u = np.array([0.5, 1.5, np.nan, -0.0, 1.0, -1e-7], np.float32)
    v = np.full(6, 0.25, np.float32)
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    outs = m.eval(cuda(u), cuda(v), cuda(v), n_domain_errors=cnt)
    torch.cuda.synchronize()
    val = outs[0].cpu().numpy()
    assert int(cnt.item()) == 3
    assert np.isnan(val[[1, 2, 5]]).all() and np.isfinite(val[[0, 3, 4]]).all()
    e = torch.empty(0, device="cuda")
    m.eval(e, e, e)   # n == 0 is valid
    torch.cuda.synchronize()


def render_gpu(c, w=None, pixels=None, **kw):
    w = w or workload(c)
    m = gpu_model(c)
    samples = torch.zeros(1, dtype=torch.int64, device="cuda")
    img = m.render(w.cameras, cuda(w.tf), w.v_lo, w.v_hi, w.params, samples=samples, **kw)
    torch.cuda.synchronize()
    return img.float().cpu().numpy(), int(samples.item())


@pytest.mark.parametrize("c", [1, 2, 3])
def test_render_full_frame_parity(c):
    """Full frames (C1 64^2 ortho, C2 512^2, C3 1024^2)."""
    w = workload(c)
    img, ns = render_gpu(c)
    ref = O.render(oracle_model(c), w.cameras[0], w.tf, w.v_lo, w.v_hi, w.params)
    st = parity.check_image(img[0].reshape(-1, 4), ref, f"C{c}")
    tot = int(ref["count"].sum())
    assert abs(ns - tot) <= max(1e-4 * tot, parity.count_window(ref)), (ns, tot)
    print(f"C{c}: {st} samples gpu {ns} oracle {tot}")


@pytest.mark.parametrize("c,views,frac", [(4, (0,), 0.05), (5, (0, 21, 42, 63), 0.0125)])
def test_render_subset_parity_full_size(c, views, frac):
    """Full-size C4 / C5 in the launch configuration the bench times (all
    views of the batch in one call), checked on a seeded 5% tile subset
    (C5: 5% over 4 views)."""
    w = workload(c)
    img, ns = render_gpu(c)
    H, W = w.cameras[0].height, w.cameras[0].width
    sub = WL.tile_subset(c, W, H, frac, views=views)
    tiles, ref_count, window = [], 0, 0
    for v, pix in sub.items():
        ref = O.render(oracle_model(c), w.cameras[v], w.tf, w.v_lo, w.v_hi, w.params, pixels=pix)
        st = parity.check_image(img[v].reshape(-1, 4)[pix], ref, f"C{c} view {v}")
        print(f"C{c} view {v}: {st}")
        ref_count += int(ref["count"].sum())
        window += parity.count_window(ref)
        t = np.unique(np.stack([(pix % W) // 16, (pix // W) // 16], axis=1), axis=0)
        tiles.append(np.concatenate([np.full((len(t), 1), v), t], axis=1))
    # composited-sample count of exactly the subset's tiles (SURVEY §8(c)
    # acceptance: GPU total = oracle total within the R-19 windows)
    tl = torch.from_numpy(np.ascontiguousarray(np.concatenate(tiles), dtype=np.int32)).cuda()
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    gpu_model(c).render(w.cameras, cuda(w.tf), w.v_lo, w.v_hi, w.params, tiles=tl, samples=cnt)
    torch.cuda.synchronize()
    got = int(cnt.item())
    assert abs(got - ref_count) <= max(window, 1e-4 * ref_count), (got, ref_count, window)
    print(f"C{c} subset samples gpu {got} oracle {ref_count} window {window}")


def test_tiled_render_bit_identical_and_unpack():
    """Screen-tile sharding invariant: rendering any tile list gives the
    same pixels as the full frame (bit-identical); unpack_tiles rebuilds it."""
    from paper_2204_11762_b200 import unpack_tiles
    c = 2
    w = workload(c)
    full, ns_full = render_gpu(c)
    tx = (w.cameras[0].width + 15) // 16
    ty = (w.cameras[0].height + 15) // 16
    allt = np.array([(0, x, y) for y in range(ty) for x in range(tx)], np.int32)
    rng = np.random.default_rng(0)
    perm = rng.permutation(len(allt))
    halves = [allt[perm[: len(perm) // 2]], allt[perm[len(perm) // 2:]]]
    img = torch.zeros((1, w.cameras[0].height, w.cameras[0].width, 4), device="cuda")
    m = gpu_model(c)
    tot = 0
    for h in halves:
        t = cuda(h)
        s = torch.zeros(1, dtype=torch.int64, device="cuda")
        packed = m.render(w.cameras, cuda(w.tf), w.v_lo, w.v_hi, w.params, tiles=t, samples=s)
        unpack_tiles(packed, t, 1, w.cameras[0].width, w.cameras[0].height, out=img)
        torch.cuda.synchronize()
        tot += int(s.item())
    np.testing.assert_array_equal(img.cpu().numpy(), full)
    assert tot == ns_full


def test_ragged_image_and_fp16():
    """Image sizes that are not multiples of the 16x16 tile, fp16 output."""
    c = 2
    w = workload(c, width=100, height=75)
    img, _ = render_gpu(c, w=w)
    ref = O.render(oracle_model(c), w.cameras[0], w.tf, w.v_lo, w.v_hi, w.params)
    parity.check_image(img[0].reshape(-1, 4), ref, "C2 100x75")
    img16, _ = render_gpu(c, w=w, out_fp16=True)
    assert np.abs(img16 - img).max() <= 1e-3


def test_multiview_batch_matches_single_views():
    c = 5
    w = workload(c, width=64, height=48, n_views=3)
    img, _ = render_gpu(c, w=w)
    for v in range(3):
        one = WL.make_config(c, width=64, height=48, n_views=3)
        one.cameras = [w.cameras[v]]
        iv, _ = render_gpu(c, w=one)
        np.testing.assert_array_equal(iv[0], img[v])


def test_render_host_matches_device():
    c = 1
    w = workload(c)
    dev, ns = render_gpu(c)
    out = torch.empty((1, 64, 64, 4), dtype=torch.float32).pin_memory()
    n2 = gpu_model(c).render_host(w.cameras, w.tf, w.v_lo, w.v_hi, w.params, out)
    np.testing.assert_array_equal(out.numpy(), dev)
    assert n2 == ns


def test_shading_off_parity():
    import dataclasses
    c = 2
    w = workload(c)
    prm = dataclasses.replace(w.params, shading=0)
    m = gpu_model(c)
    img = m.render(w.cameras, cuda(w.tf), w.v_lo, w.v_hi, prm)
    torch.cuda.synchronize()
    ref = O.render(oracle_model(c), w.cameras[0], w.tf, w.v_lo, w.v_hi, prm)
    parity.check_image(img[0].cpu().numpy().reshape(-1, 4), ref, "C2 shading off")


def test_camera_inside_volume_and_ortho_axis_aligned():
    """Degenerate geometry: eye inside the box (t_in = 0); axis-aligned
    orthographic rays (d components exactly 0)."""
    c = 1
    w = WL.make_config(c)
    w.cameras = [WL.Camera(eye=(0.05, -0.1, 0.02), look_at=(0.3, 0.2, -0.1), up=(0, 0, 1), fov_y_deg=60.0,
                           ortho_half_height=0.0, width=40, height=30),
                 WL.Camera(eye=(0.0, 0.0, 2.0), look_at=(0.0, 0.0, 0.0), up=(0, 1, 0), fov_y_deg=0.0,
                           ortho_half_height=0.6, width=40, height=30)]
    img, _ = render_gpu(c, w=w)
    for v in range(2):
        ref = O.render(oracle_model(c), w.cameras[v], w.tf, w.v_lo, w.v_hi, w.params)
        parity.check_image(img[v].reshape(-1, 4), ref, f"geometry view {v}")


def test_invalid_models_raise():
    from paper_2204_11762_b200 import MfaError, Model
    p = 2
    good = np.concatenate([np.zeros(3), [0.5], np.ones(3)])
    ctrl = np.zeros((4, 4, 4), np.float32)
    bad = good.copy()
    bad[3] = 1.5
    with pytest.raises(MfaError, match="KNOTS"):
        Model(p, [good, bad, good], ctrl)
    with pytest.raises(MfaError, match="UNSUPPORTED"):
        Model((2, 3, 2), [good, good, good], ctrl)
    nanc = ctrl.copy()
    nanc[1, 2, 3] = np.nan
    with pytest.raises(MfaError, match="DOMAIN"):
        Model(p, [good, good, good], nanc)
    m = Model(p, [good, good, good], ctrl + 2)
    info = m.info()
    assert info["v_min"] == 2 and info["v_max"] == 2 and info["uniform"] == (1, 1, 1)


@pytest.mark.parametrize("c,layout", [(1, "bezier"), (2, "bezier"), (3, "bezier"), (5, "quads"),
                                      (1, "bricks"), (2, "bricks"), (3, "bricks"), (5, "bricks"),
                                      (3, "bezier_grouped"), (5, "bezier")])
def test_both_layouts_eval_and_render(c, layout):
    """Each model also through the other control-point layouts (bricked quads,
    Bezier blocks linear or grouped, plain haloed bricks): eval parity on random + boundary
    points and a render parity check (a reduced image for C3/C5)."""
    w = workload(c) if c in (1, 2) else workload(c, width=256, height=192, n_views=1)
    m = gpu_model(c, layout)
    assert m.info()["layout"] == layout
    u, v, ww = WL.query_points(c, 1 << 16)
    bu, bv, bw = WL.boundary_points(w)
    u, v, ww = (np.concatenate([a, b]) for a, b in ((u, bu), (v, bv), (ww, bw)))
    got = gpu_eval(m, u, v, ww)
    ref, sig, _ = oracle_model(c).eval_batch(u, v, ww)
    parity.check_eval(got, ref, sig, f"C{c} {layout}")
    vo = gpu_eval(m, u, v, ww, grad=False)
    parity.check_eval(vo, ref[:, :1], sig[:, :1], f"C{c} {layout} value-only")
    samples = torch.zeros(1, dtype=torch.int64, device="cuda")
    img = m.render(w.cameras[:1], cuda(w.tf), w.v_lo, w.v_hi, w.params, samples=samples)
    torch.cuda.synchronize()
    r = O.render(oracle_model(c), w.cameras[0], w.tf, w.v_lo, w.v_hi, w.params)
    parity.check_image(img[0].cpu().numpy().reshape(-1, 4), r, f"C{c} {layout} render")


def test_default_layouts():
    assert gpu_model(3).info()["layout"] == "quads"
    assert gpu_model(5).info()["layout"] == "bezier_grouped"   # p = 3 Bezier blocks: grouped
    assert gpu_model(2).info()["layout"] == "bezier_grouped"   # uniform, but 58 MB of blocks: L2-resident
    assert gpu_model(1).info()["layout"] == "bezier"           # p = 2: linear blocks


@pytest.mark.parametrize("p", [2, 3])
def test_nonuniform_multiple_knots(p):
    """A non-uniform model with a repeated interior knot (multiplicity 2 <= p,
    so a zero-length span the span search and tracking must step over and a
    C^(p-2) joint); both layouts against the oracle on eval and a full frame."""
    rng = np.random.default_rng(7 + p)
    n = 12
    inner = np.sort(rng.uniform(0.1, 0.9, n - p - 2))
    inner = np.concatenate([inner, [inner[3]]])          # one double knot
    U = np.concatenate([np.zeros(p + 1), np.sort(inner), np.ones(p + 1)])
    assert len(U) == n + p + 1
    ctrl = rng.uniform(-1, 1, (n, n, n)).astype(np.float32)
    w = WL.make_config(1)
    w.degree, w.knots, w.ctrl, w.nctrl, w.uniform = p, [U, U, U], ctrl, (n, n, n), False
    w.v_lo, w.v_hi = float(ctrl.min()), float(ctrl.max())
    om = O.Model.from_workload(w)
    from paper_2204_11762_b200 import Model
    for layout in ("quads", "bezier", "bricks") + (("bezier_grouped",) if p == 3 else ()):
        m = Model.from_workload(w, layout=layout)
        u, v, ww = WL.query_points(1, 1 << 14)
        got = gpu_eval(m, u, v, ww)
        ref, sig, _ = om.eval_batch(u, v, ww)
        parity.check_eval(got, ref, sig, f"double knot p={p} {layout}")
        img = m.render(w.cameras, cuda(w.tf), w.v_lo, w.v_hi, w.params)
        torch.cuda.synchronize()
        r = O.render(om, w.cameras[0], w.tf, w.v_lo, w.v_hi, w.params)
        parity.check_image(img[0].cpu().numpy().reshape(-1, 4), r, f"double knot p={p} {layout} render")


@pytest.mark.parametrize("p,n,uniform", [(1, 9, True), (5, 12, True), (5, 12, False), (4, 9, False), (2, 3, True),
                                         (3, 4, False), (1, 7, False), (2, 8, False)])
def test_render_degrees_and_single_span(p, n, uniform):
    """Degrees outside the configs (1, 5), non-uniform p = 4 / 5 (quads +
    span tables), and the single-span model n = p + 1 (every axis one span):
    full-frame render and eval parity."""
    from paper_2204_11762_b200 import Model
    r = np.random.default_rng(100 * p + n)
    knots = []
    for d in range(3):
        S = n - p
        inner = np.arange(1, S) / S if uniform else np.sort(r.uniform(0.05, 0.95, S - 1))
        knots.append(np.concatenate([np.zeros(p + 1), inner, np.ones(p + 1)]))
    ctrl = r.uniform(0, 1, (n, n, n)).astype(np.float32)
    w = WL.make_config(2, width=72, height=56)
    w.degree, w.knots, w.ctrl, w.nctrl, w.uniform = p, knots, ctrl, (n, n, n), uniform
    w.v_lo, w.v_hi = float(ctrl.min()), float(ctrl.max())
    m = Model.from_workload(w)
    om = O.Model.from_workload(w)
    img = m.render(w.cameras, cuda(w.tf), w.v_lo, w.v_hi, w.params)
    torch.cuda.synchronize()
    ref = O.render(om, w.cameras[0], w.tf, w.v_lo, w.v_hi, w.params)
    parity.check_image(img[0].cpu().numpy().reshape(-1, 4), ref, f"p={p} n={n} uniform={uniform}")
    u, v, ww = WL.query_points(2, 1 << 12)
    got = gpu_eval(m, u, v, ww)
    e, sg, _ = om.eval_batch(u, v, ww)
    parity.check_eval(got, e, sg, f"p={p} n={n}")


@pytest.mark.parametrize("o_max", [1.0, 0.5])
def test_ert_threshold_variants(o_max):
    """o_max = 1 disables early ray termination (every sample composited);
    o_max = 0.5 terminates early; both against the oracle, and the sample
    count with ERT off equals the sum of K over the rays."""
    import dataclasses
    c = 2
    w = workload(c, width=128, height=96)
    prm = dataclasses.replace(w.params, o_max=o_max)
    m = gpu_model(c)
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    img = m.render(w.cameras, cuda(w.tf), w.v_lo, w.v_hi, prm, samples=cnt)
    torch.cuda.synchronize()
    ref = O.render(oracle_model(c), w.cameras[0], w.tf, w.v_lo, w.v_hi, prm)
    parity.check_image(img[0].cpu().numpy().reshape(-1, 4), ref, f"o_max={o_max}")
    tot = int(ref["count"].sum())
    assert abs(int(cnt.item()) - tot) <= max(1, parity.count_window(ref))


def test_empty_tile_list_and_padding_only():
    c = 1
    w = workload(c)
    m = gpu_model(c)
    out = torch.full((4, 16, 16, 4), 7.0, device="cuda")
    empty = torch.zeros((0, 3), dtype=torch.int32, device="cuda")
    m.render(w.cameras, cuda(w.tf), w.v_lo, w.v_hi, w.params, tiles=empty, out=out[:0])
    pad = torch.full((4, 3), -1, dtype=torch.int32, device="cuda")
    m.render(w.cameras, cuda(w.tf), w.v_lo, w.v_hi, w.params, tiles=pad, out=out)
    torch.cuda.synchronize()
    assert (out == 7.0).all()     # padding units are skipped: nothing written


def test_more_than_64_views_and_tf_sizes():
    """n_views > 64 is split into launches of <= 64 views (mfa_render); TF
    tables of 2 and 1024 entries (the ABI's limits) against the oracle."""
    c = 1
    w = WL.make_config(c, width=24, height=20, n_views=70)
    m = gpu_model(c)
    img, _ = render_gpu(c, w=w)
    for v in (0, 63, 64, 69):
        ref = O.render(oracle_model(c), w.cameras[v], w.tf, w.v_lo, w.v_hi, w.params)
        parity.check_image(img[v].reshape(-1, 4), ref, f"view {v} of 70")
    for n in (2, 1024):
        x = np.linspace(0, 1, n)
        tf = np.stack([x, 1 - x, np.full(n, 0.4), 0.05 + 0.05 * np.sin(7 * x) ** 2], axis=1).astype(np.float32)
        out = m.render(w.cameras[:1], cuda(tf), w.v_lo, w.v_hi, w.params)
        torch.cuda.synchronize()
        ref = O.render(oracle_model(c), w.cameras[0], tf, w.v_lo, w.v_hi, w.params)
        parity.check_image(out[0].cpu().numpy().reshape(-1, 4), ref, f"TF with {n} entries")


@pytest.mark.parametrize("p", [2, 3])
def test_spans_narrower_than_a_step(p):
    """Non-uniform axes with spans narrower than one ray step, so one step can
    cross several spans (adjacent narrow spans: up to three crossings; an
    isolated narrow span: two), and every span wide (the per-launch flag
    drops the multi-span check, render.cu): render parity for each."""
    from paper_2204_11762_b200 import Model
    r = np.random.default_rng(7 + p)
    w = WL.make_config(2, width=64, height=48)
    step = w.params.step
    inners = {"adjacent": [0.2, 0.45, 0.45 + 0.3 * step, 0.45 + 0.6 * step, 0.7],
              "isolated": [0.2, 0.45, 0.45 + 0.5 * step, 0.7],
              "wide": [0.2, 0.45, 0.7]}
    for narrow, inner in inners.items():
        knots = []
        for d in range(3):
            knots.append(np.concatenate([np.zeros(p + 1), inner, np.ones(p + 1)]))
        n = len(knots[0]) - p - 1
        ctrl = r.uniform(0, 1, (n, n, n)).astype(np.float32)
        w.degree, w.knots, w.ctrl, w.nctrl, w.uniform = p, knots, ctrl, (n, n, n), False
        w.v_lo, w.v_hi = float(ctrl.min()), float(ctrl.max())
        m = Model.from_workload(w)
        om = O.Model.from_workload(w)
        img = m.render(w.cameras, cuda(w.tf), w.v_lo, w.v_hi, w.params)
        torch.cuda.synchronize()
        ref = O.render(om, w.cameras[0], w.tf, w.v_lo, w.v_hi, w.params)
        parity.check_image(img[0].cpu().numpy().reshape(-1, 4), ref, f"p={p} narrow={narrow}")


def test_mfa_render_entry_point_itself():
    """The north_star symbol mfa_render (not mfa_render_ex) called through
    ctypes: the same image as Model.render bit for bit, parity with the
    oracle on C1, and the sample count."""
    import ctypes as C

    from paper_2204_11762_b200 import _lib as LB
    c = 1
    w = workload(c)
    m = gpu_model(c)
    tf = cuda(w.tf)
    out = torch.empty((1, 64, 64, 4), dtype=torch.float32, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    tft = LB.TF_t(C.c_void_p(tf.data_ptr()), tf.shape[0], float(w.v_lo), float(w.v_hi))
    st = LB.lib().mfa_render(m.handle, 1, LB.cameras_t(w.cameras), C.byref(tft), C.byref(LB.params_t(w.params)),
                             None, C.c_void_p(out.data_ptr()), C.c_void_p(cnt.data_ptr()),
                             C.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert st == 0, LB.lib().mfa_last_error()
    torch.cuda.synchronize()
    img, ns = render_gpu(c)
    np.testing.assert_array_equal(out.cpu().numpy(), img)
    assert int(cnt.item()) == ns
    ref = O.render(oracle_model(c), w.cameras[0], w.tf, w.v_lo, w.v_hi, w.params)
    parity.check_image(out[0].cpu().numpy().reshape(-1, 4), ref, "mfa_render C1")


def test_many_renders_in_flight_on_distinct_streams():
    """More than 256 renders of one model queued on distinct streams (one
    persistent-kernel work counter each): every image is correct, or the
    call refuses cleanly (MFA_ERR_UNSUPPORTED) -- never a shared counter."""
    from paper_2204_11762_b200._lib import MfaError
    w = workload(2, width=48, height=40)
    m = gpu_model(2)
    tf = cuda(w.tf)
    ref = m.render(w.cameras, tf, w.v_lo, w.v_hi, w.params)
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(300)]
    outs, refused = [], 0
    for s in streams:
        with torch.cuda.stream(s):
            o = torch.empty_like(ref)
            try:
                m.render(w.cameras, tf, w.v_lo, w.v_hi, w.params, out=o)
                outs.append(o)
            except MfaError as e:
                assert "in flight" in str(e)
                refused += 1
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o, ref)
    assert len(outs) + refused == 300 and len(outs) >= 256


@pytest.mark.parametrize("c,layout", [(2, "auto"), (3, "auto"), (5, "auto"), (5, "quads"), (1, "auto")])
def test_skip_transparent_gradient_is_bit_identical(c, layout):
    """NEXT-1 variants: shading = 2 skips the gradient contraction and Phong
    where the TF opacity is 0; shading = 3 skips whole samples in macro blocks
    whose value range maps to opacity 0 (Bezier layout).  Those samples
    composite with weight 0, so the image and the composited-sample count
    equal the shaded render's bit for bit (C5 on a reduced 4-view batch, both
    layouts)."""
    import dataclasses
    kw = {"n_views": 4, "width": 640, "height": 360} if c == 5 else {}
    w = workload(c, **kw)
    m = gpu_model(c, layout) if not kw else __import__("paper_2204_11762_b200").Model.from_workload(w, layout=layout)
    tf = cuda(w.tf)
    res = []
    for sh in (1, 2, 3):
        prm = dataclasses.replace(w.params, shading=sh)
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        img = m.render(w.cameras, tf, w.v_lo, w.v_hi, prm, samples=cnt)
        torch.cuda.synchronize()
        res.append((img.cpu().numpy(), int(cnt.item())))
    for other in res[1:]:
        np.testing.assert_array_equal(res[0][0], other[0])
        assert res[0][1] == other[1]


def test_bricks_layout_footprint_and_full_size_c5():
    """The plain haloed-brick layout (<= 2x the fp32 grid, P:133 / P:263) on
    the full C5 model: footprint ratio, and the bench's launch configuration
    (all 64 views in one call) checked on a seeded tile subset of 2 views."""
    from paper_2204_11762_b200 import Model
    w = workload(5)
    m = Model.from_workload(w, layout="bricks")
    info = m.info()
    assert info["layout"] == "bricks"
    ratio = info["device_bytes"] / info["model_bytes"]
    assert ratio <= 2.0, ratio
    samples = torch.zeros(1, dtype=torch.int64, device="cuda")
    img = m.render(w.cameras, cuda(w.tf), w.v_lo, w.v_hi, w.params, samples=samples)
    torch.cuda.synchronize()
    H, W = w.cameras[0].height, w.cameras[0].width
    for v, pix in WL.tile_subset(5, W, H, 0.01, views=(7, 40)).items():
        ref = O.render(oracle_model(5), w.cameras[v], w.tf, w.v_lo, w.v_hi, w.params, pixels=pix)
        parity.check_image(img[v].cpu().numpy().reshape(-1, 4)[pix], ref, f"C5 bricks view {v}")
    print(f"C5 bricks: device {info['device_bytes'] / 2**20:.0f} MiB = {ratio:.2f} x the grid")


def test_malformed_tile_entries_are_skipped():
    """Tile entries outside the call's views or the image (view >= n_views,
    negative or too-large tile coordinates) are skipped by the render and
    unpack kernels: no store outside the image, valid tiles unaffected."""
    from paper_2204_11762_b200 import dist as D, unpack_tiles
    w = workload(2, width=100, height=75, n_views=2)
    m = gpu_model(2)
    tf = cuda(w.tf)
    full = m.render(w.cameras, tf, w.v_lo, w.v_hi, w.params)
    good = D.all_units(2, 100, 75)
    bad = np.array([[2, 0, 0], [7, 1, 1], [0, -1, 0], [1, 0, -3], [0, 7, 0], [1, 0, 5], [-1, 0, 0]], np.int32)
    tl = np.ascontiguousarray(np.concatenate([good[:5], bad, good[5:]]), dtype=np.int32)
    guard = torch.full((4, 75, 100, 4), -7.0, device="cuda")   # 2 extra views past the call's 2
    m.render(w.cameras, tf, w.v_lo, w.v_hi, w.params, tiles=cuda(tl), out=guard, scatter=True)
    packed = m.render(w.cameras, tf, w.v_lo, w.v_hi, w.params, tiles=cuda(tl))
    img = torch.full((4, 75, 100, 4), -7.0, device="cuda")
    unpack_tiles(packed, cuda(tl), 2, 100, 75, out=img)
    torch.cuda.synchronize()
    for out in (guard, img):
        assert torch.equal(out[:2], full)
        assert (out[2:] == -7.0).all()


def test_render_host_views_and_reuse():
    """mfa_render_host_views writes each view to its own host buffer (any
    order, e.g. a rank's views into a shared host image); repeated host
    renders reuse the model-owned staging, and a larger image after a smaller
    one grows it -- every result equals the device render."""
    from paper_2204_11762_b200 import Model
    w = workload(2, width=96, height=64, n_views=5)
    m = Model.from_workload(w)
    tf = cuda(w.tf)
    dev = m.render(w.cameras, tf, w.v_lo, w.v_hi, w.params).cpu().numpy()
    order = [3, 0, 4]
    bufs = [torch.empty((64, 96, 4), dtype=torch.float32).pin_memory() for _ in order]
    for _ in range(2):   # the second call reuses the staging buffers
        m.render_host_views([w.cameras[v] for v in order], w.tf, w.v_lo, w.v_hi, w.params,
                            [b.data_ptr() for b in bufs])
        for v, b in zip(order, bufs):
            np.testing.assert_array_equal(b.numpy(), dev[v])
    w2 = workload(2, width=200, height=150, n_views=2)   # larger views: the staging grows
    dev2 = m.render(w2.cameras, tf, w2.v_lo, w2.v_hi, w2.params).cpu().numpy()
    host2 = torch.empty((2, 150, 200, 4), dtype=torch.float32).pin_memory()
    m.render_host(w2.cameras, w2.tf, w2.v_lo, w2.v_hi, w2.params, host2)
    np.testing.assert_array_equal(host2.numpy(), dev2)


def test_transparent_skip_in_tiled_scatter_path():
    """shading = 3 through the multi-GPU tile path (tiles stored at their image
    positions): bit-identical to the full-frame shaded render."""
    import dataclasses

    from paper_2204_11762_b200 import Model, dist as D
    w = workload(5, width=320, height=180, n_views=3)
    m = Model.from_workload(w)
    tf = cuda(w.tf)
    full = m.render(w.cameras, tf, w.v_lo, w.v_hi, w.params)
    p3 = dataclasses.replace(w.params, shading=3)
    img = torch.full_like(full, -1.0)
    for lst in D.assign_units(3, 320, 180, 2, "views", pad=False):
        m.render(w.cameras, tf, w.v_lo, w.v_hi, p3, tiles=cuda(lst), out=img, scatter=True)
    torch.cuda.synchronize()
    assert torch.equal(img, full)


def test_grouped_bezier_layout_needs_degree_3():
    """MFA_LAYOUT_BEZIER_GROUPED is built for p = 3 only: other degrees are
    refused (MFA_ERR_UNSUPPORTED); AUTO keeps linear blocks at p = 2."""
    from paper_2204_11762_b200 import MfaError, Model
    w = workload(1)
    with pytest.raises(MfaError, match="UNSUPPORTED"):
        Model.from_workload(w, layout="bezier_grouped")
    assert Model.from_workload(w).info()["layout"] == "bezier"


@pytest.mark.parametrize("layout", ["auto", "quads", "bricks", "bezier", "bezier_grouped"])
def test_model_info_footprint(layout):
    """mfa_model_info reports the grid bytes, the device bytes of the chosen
    layout (bricks <= 2x the grid) and the create time."""
    from paper_2204_11762_b200 import Model
    w = workload(2)
    m = Model.from_workload(w, layout=layout)
    info = m.info()
    assert info["model_bytes"] == 4 * 64 ** 3
    assert info["create_ms"] > 0
    ratio = info["device_bytes"] / info["model_bytes"]
    if info["layout"] == "bricks":
        assert ratio <= 2.0
    else:
        assert ratio > 2.0


@pytest.mark.gpu
def test_render_cuda_graph_capture_replay():
    """mfa_render is stream-capture safe: three renders captured into a CUDA
    graph and replayed give the eager image bit for bit and three times its
    composited-sample count."""
    from paper_2204_11762_b200 import Model
    w = WL.make_config(2, width=96, height=64)
    m = Model.from_workload(w)
    tf = torch.from_numpy(w.tf).cuda()
    H, W = w.cameras[0].height, w.cameras[0].width
    img = torch.empty((1, H, W, 4), device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        m.render(w.cameras, tf, w.v_lo, w.v_hi, w.params, out=img, samples=cnt, stream=s)
    torch.cuda.synchronize()
    ref, n1 = img.clone(), int(cnt.item())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(3):
            m.render(w.cameras, tf, w.v_lo, w.v_hi, w.params, out=img, samples=cnt, stream=s)
    img.zero_()
    cnt.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(img, ref)
    assert int(cnt.item()) == 3 * n1 > 0
