"""GPU parity for NEXT-3 (mfa_fit_grid / mfa_encode_grid) against the fp64
numpy oracle (oracle/encode.py): least-squares control values to 1e-9
relative (fp64 on both sides; R-29), the adaptive loop's knot vectors exactly,
and the fitted model rendering through the hot path."""
import numpy as np
import pytest

import oracle as O
from oracle import encode as E
from paper_2204_11762_b200 import workloads as WL

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

FIT_TOL = 1e-9


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("p,dims,n", [(1, (17, 13, 11), (6, 5, 4)), (2, (33, 29, 31), (12, 9, 10)),
                                      (3, (40, 24, 32), (20, 8, 14)), (4, (23, 21, 25), (10, 9, 11)),
                                      (5, (19, 18, 20), (12, 11, 12))])
def test_fit_parity(p, dims, n):
    """Random noisy grid, non-uniform knots with samples in every span."""
    from paper_2204_11762_b200 import fit_grid
    r = np.random.default_rng(90 + p)
    q = (WL.analytic_grid("ml", dims) + r.normal(0, 0.05, (dims[2], dims[1], dims[0]))).astype(np.float32)
    knots = []
    for d in range(3):
        S = n[d] - p
        k = np.arange(1, S) / S + r.uniform(-0.2, 0.2, S - 1) / S
        knots.append(np.concatenate([np.zeros(p + 1), k, np.ones(p + 1)]))
    c32, c64 = fit_grid(cuda(q), p, knots, want64=True)
    torch.cuda.synchronize()
    ref = E.fit(q.astype(np.float64), knots, p)
    got = c64.cpu().numpy()
    scale = np.abs(ref).max()
    assert np.abs(got - ref).max() <= FIT_TOL * scale, np.abs(got - ref).max() / scale
    np.testing.assert_array_equal(c32.cpu().numpy(), got.astype(np.float32))


def test_fit_square_interpolates_and_errors():
    from paper_2204_11762_b200 import MfaError, fit_grid
    p = 3
    dims = (9, 8, 10)
    q = np.random.default_rng(5).normal(size=(dims[2], dims[1], dims[0])).astype(np.float32)
    knots = [E.uniform_knots(m, p) for m in dims]
    _, c64 = fit_grid(cuda(q), p, knots, want64=True)
    v = E.evaluate_grid(c64.cpu().numpy(), knots, p, dims)
    np.testing.assert_allclose(v, q, atol=1e-9)
    with pytest.raises(MfaError, match="INVALID_ARG"):        # more control points than samples
        fit_grid(cuda(q), p, [E.uniform_knots(12, p)] + knots[1:])
    bad = knots[0].copy()
    bad[5] = 2.0
    with pytest.raises(MfaError, match="KNOTS"):
        fit_grid(cuda(q), p, [bad] + knots[1:])
    # a knot layout leaving a basis function without samples: the device
    # Cholesky reports the singular pivot (axis and control point)
    sparse = np.concatenate([np.zeros(p + 1), [0.05, 0.06, 0.07], np.ones(p + 1)])   # 7 ctrl, 9 samples
    with pytest.raises(MfaError, match="singular on axis u"):
        fit_grid(cuda(q), p, [sparse] + knots[1:])
    # non-finite input values: MFA_ERR_DOMAIN before any fit (fit and encoder)
    from paper_2204_11762_b200 import encode_grid
    qn = q.copy()
    qn[3, 2, 1] = np.nan
    with pytest.raises(MfaError, match="DOMAIN"):
        fit_grid(cuda(qn), p, knots)
    with pytest.raises(MfaError, match="DOMAIN"):
        encode_grid(cuda(qn), p, (4, 4, 4), 1e-3, 2, dims)


@pytest.mark.parametrize("kind,p,e_max", [("gb", 2, 0.01), ("gb", 3, 0.003), ("ml", 2, 0.05)])
def test_adaptive_matches_oracle(kind, p, e_max):
    """The adaptive loop on a 33^3 grid from 4^3 control points:
    same per-round control counts, same final knots (exact: both sides take
    the split decisions on fp64 errors far from e_max), control values and
    errors within the fit tolerance."""
    from paper_2204_11762_b200 import encode_grid
    q = WL.analytic_grid(kind, (33, 33, 33)).astype(np.float32)
    caps = (33, 33, 33)
    knots, ctrl, res, log = encode_grid(cuda(q), p, (4, 4, 4), e_max, 8, caps)
    ok, oc, orep = E.adaptive(q.astype(np.float64), p, (4, 4, 4), e_max, 8, caps)
    assert res["converged"] == orep["converged"]
    assert [tuple(int(x) for x in row[:3]) for row in log] == [r[0] for r in orep["rounds"]]
    for d in range(3):
        np.testing.assert_array_equal(knots[d], ok[d])
    np.testing.assert_allclose(log[:, 3], [r[1] for r in orep["rounds"]], rtol=1e-7, atol=1e-12)
    np.testing.assert_allclose(log[:, 4], [r[2] for r in orep["rounds"]], rtol=1e-7)
    np.testing.assert_allclose(ctrl.cpu().numpy(), oc.astype(np.float32), rtol=0,
                               atol=1e-6 * np.abs(oc).max())
    print(kind, p, res, [r[:2] for r in orep["rounds"]])


def test_encoded_model_renders():
    """The encoder's output is an MFA the hot path renders (encode -> model ->
    render parity against the oracle on the same control values)."""
    import parity
    from paper_2204_11762_b200 import Model, encode_grid
    q = WL.analytic_grid("ml", (41, 41, 41)).astype(np.float32)
    knots, ctrl, res, _ = encode_grid(cuda(q), 3, (8, 8, 8), 0.02, 6, (41, 41, 41))
    c = ctrl.cpu().numpy()
    m = Model(3, knots, ctrl)
    om = O.Model(3, knots, c)
    w = WL.make_config(1, width=96, height=80)
    w.v_lo, w.v_hi = float(c.min()), float(c.max())
    img = m.render(w.cameras, cuda(w.tf), w.v_lo, w.v_hi, w.params)
    torch.cuda.synchronize()
    ref = O.render(om, w.cameras[0], w.tf, w.v_lo, w.v_hi, w.params)
    parity.check_image(img[0].cpu().numpy().reshape(-1, 4), ref, "encoded ML")
