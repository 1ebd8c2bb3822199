"""GPU parity for NEXT-4 (mfa_eval_hessian): value, gradient and the six
second partials against the fp64 oracle's plain triple sums (oracle.c H2),
normwise to the abs-scale of the same sum (R-5): value 1e-5,
gradient 1e-4 (north_star), Hessian 1e-4 (R-25)."""
import functools

import numpy as np
import pytest

import oracle as O
import parity
from paper_2204_11762_b200 import workloads as WL

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

HESS_TOL = 1e-4


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def knot_window_errors(om, got, u, v, w, r, knots, p):
    """R-26: at a knot the p-th derivative of a degree-p spline jumps (simple
    knots), so for p = 2 the Hessian of a point within rounding of a knot has
    two correct values, the one-sided limits.  For such points the error is
    the smaller of the errors against the oracle evaluated just below and just
    above the knot on that axis (the only rows re-evaluated)."""
    import itertools
    bad = np.where(r[:, 4:].max(axis=1) > HESS_TOL)[0]
    q = np.stack([u, v, w], axis=1).astype(np.float64)
    for i in bad:
        near = []
        for d in range(3):
            kn = knots[d][p:-p]
            j = int(np.argmin(np.abs(kn - q[i, d])))
            if abs(kn[j] - q[i, d]) <= 1e-6:
                near.append((d, kn[j]))
        best = r[i, 4:].max()
        for sides in itertools.product((-1e-9, 1e-9), repeat=len(near)):   # every one-sided limit
            qq = q[i].copy()
            for (d, k), sd in zip(near, sides):
                qq[d] = min(max(k + sd, 0.0), 1.0)
            o, sg, _ = om.eval_hessian(*qq)
            e = parity.eval_errors(got[i:i + 1], o[None], sg[None])[0]
            best = min(best, e[4:].max())
        r[i, 4:] = best
    return r


def check(m, om, u, v, w, what, knots=None, p=None):
    val, grad, hess = m.eval_hessian(cuda(u), cuda(v), cuda(w))
    torch.cuda.synchronize()
    got = np.concatenate([val.cpu().numpy()[:, None], grad.cpu().numpy().T, hess.cpu().numpy().T], axis=1)
    ref, sig, errs = om.eval_hessian_batch(u, v, w)
    assert errs == 0
    r = parity.eval_errors(got, ref, sig)
    if knots is not None and p == 2:
        r = knot_window_errors(om, got, u, v, w, r, knots, p)
    wv, wg, wh = float(r[:, 0].max()), float(r[:, 1:4].max()), float(r[:, 4:].max())
    assert wv <= parity.VAL_TOL and wg <= parity.GRAD_TOL and wh <= HESS_TOL, (what, wv, wg, wh)
    print(f"{what}: n={len(u)} worst value {wv:.2e} grad {wg:.2e} hessian {wh:.2e} sigma")
    return got


@functools.lru_cache(maxsize=None)
def models(c, layout):
    from paper_2204_11762_b200 import Model
    w = WL.make_config(c)
    return w, Model.from_workload(w, layout=layout), O.Model.from_workload(w)


@pytest.mark.parametrize("c,layout", [(1, "quads"), (2, "quads"), (2, "bezier"), (3, "quads"), (4, "quads"),
                                      (5, "bezier"), (5, "quads"), (2, "bricks"), (5, "bricks"),
                                      (5, "bezier_grouped"), (2, "bezier_grouped")])
def test_hessian_parity_configs(c, layout):
    w, m, om = models(c, layout)
    u, v, ww = WL.query_points(c, 1 << 15)
    bu, bv, bw = WL.boundary_points(w)
    u, v, ww = (np.concatenate([a, b]) for a, b in ((u, bu), (v, bv), (ww, bw)))
    got = check(m, om, u, v, ww, f"C{c} {layout}", knots=w.knots, p=w.degree)
    # value and gradient agree with mfa_eval_batch on the same points
    e = m.eval(cuda(u), cuda(v), cuda(ww))
    torch.cuda.synchronize()
    ev = np.stack([t.cpu().numpy() for t in e], axis=1)
    assert np.abs(ev - got[:, :4]).max() <= 1e-4 * max(1.0, np.abs(ev).max())


@pytest.mark.parametrize("p", [1, 2, 5])
def test_hessian_degrees_nonuniform(p):
    """Degrees outside the configs (1 and 5) and random non-uniform knots."""
    from paper_2204_11762_b200 import Model
    r = np.random.default_rng(70 + p)
    n = (p + 9, p + 7, p + 8)
    knots = []
    for d in range(3):
        S = n[d] - p
        knots.append(np.concatenate([np.zeros(p + 1), np.sort(r.uniform(0, 1, S - 1)), np.ones(p + 1)]))
    ctrl = r.uniform(-1, 1, (n[2], n[1], n[0])).astype(np.float32)
    m = Model(p, knots, ctrl)
    om = O.Model(p, knots, ctrl)
    u, v, w = (r.random(1 << 14, dtype=np.float32) for _ in range(3))
    check(m, om, u, v, w, f"p={p} non-uniform", knots=knots, p=p)


def test_hessian_domain_errors_and_empty():
    w, m, _ = models(1, "quads")
    u = np.array([0.5, 1.5, np.nan, 0.0, 1.0], np.float32)
    v = np.full(5, 0.25, np.float32)
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    val, grad, hess = m.eval_hessian(cuda(u), cuda(v), cuda(v), n_domain_errors=cnt)
    torch.cuda.synchronize()
    assert int(cnt.item()) == 2
    h = hess.cpu().numpy()
    assert np.isnan(h[:, [1, 2]]).all() and np.isfinite(h[:, [0, 3, 4]]).all()
    e = torch.empty(0, device="cuda")
    m.eval_hessian(e, e, e)
    torch.cuda.synchronize()


@pytest.mark.parametrize("c,layout", [(3, "quads"), (5, "bezier"), (5, "bezier_grouped")])
def test_hessian_binned_equals_direct(c, layout):
    w, m, _ = models(c, layout)
    u, v, ww = WL.query_points(c, 1 << 17)
    u = u.copy()
    u[[3, 999]] = [np.nan, 2.0]
    res = []
    for binned in ("auto", True, False):
        cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
        r = m.eval_hessian(cuda(u), cuda(v), cuda(ww), n_domain_errors=cnt, binned=binned)
        torch.cuda.synchronize()
        res.append(([t.cpu().numpy() for t in r], int(cnt.item())))
    for other in res[1:]:
        for a, b in zip(res[0][0], other[0]):
            np.testing.assert_array_equal(a, b)
        assert other[1] == 2
    assert res[0][1] == 2
