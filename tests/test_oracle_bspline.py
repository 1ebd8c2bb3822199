"""Pins for the oracle's B-spline part (O1 find_span, O2 basis+derivatives,
O3 eval): SPEC worked examples, hand-derived closed forms, the recursive
definition (tests/bruteforce.py), partition of unity, blossom polynomial
reproduction, endpoint interpolation, local support, central differences.
No GPU.  Each check is chosen so a plausible slip in the oracle (dropped
term, wrong sign/index, transposed operand) fails at least one of them."""
import json
import math
import os
from itertools import combinations

import numpy as np
import pytest

import bruteforce as BF
import oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "bspline_examples.json")


def rand_knots(r, p, n, multiplicity=True):
    """Clamped knot vector with random interior knots (optionally repeated <= p)."""
    S = n - p
    interior = np.sort(r.uniform(0.0, 1.0, S - 1))
    if multiplicity and S - 1 >= 2 and r.random() < 0.5:
        j = r.integers(0, S - 2)
        m = min(p, S - 1 - j)
        interior[j:j + m] = interior[j]
    return np.concatenate([np.zeros(p + 1), interior, np.ones(p + 1)])


def uniform_knots(p, n):
    S = n - p
    return np.concatenate([np.zeros(p + 1), np.arange(1, S) / S, np.ones(p + 1)])


# --------------------------------------------------------------------------
def test_golden_find_span():
    g = json.load(open(GOLDEN))
    for c in g["find_span"]:
        assert O.find_span(c["p"], c["knots"], c["u"]) == c["span"], c["source"]


def test_golden_basis():
    g = json.load(open(GOLDEN))
    for c in g["basis"]:
        s = O.find_span(c["p"], c["knots"], c["u"])
        N, dN = O.basis_derivs(c["p"], c["knots"], s, c["u"])
        np.testing.assert_allclose(N, c["N"], rtol=0, atol=1e-14, err_msg=c["source"])
        np.testing.assert_allclose(dN, c["dN"], rtol=0, atol=1e-13, err_msg=c["source"])


def test_find_span_linear_scan_and_domain():
    r = np.random.default_rng(1)
    for _ in range(300):
        p = int(r.integers(1, 6))
        n = int(r.integers(p + 1, p + 12))
        U = rand_knots(r, p, n)
        for u in list(r.uniform(0, 1, 5)) + [0.0, 1.0] + list(U[p:n + 1]):
            s = O.find_span(p, U, u)
            if u == 1.0:
                assert U[s] < U[s + 1] and U[s + 1] == 1.0
            else:  # linear scan: the unique i in [p, n-1] with U[i] <= u < U[i+1]
                cand = [i for i in range(p, n) if U[i] <= u < U[i + 1]]
                assert cand == [s]
    assert O.find_span(2, [0, 0, 0, 1, 1, 1], 1.0000001) == -1
    assert O.find_span(2, [0, 0, 0, 1, 1, 1], -1e-300) == -1
    assert O.find_span(2, [0, 0, 0, 1, 1, 1], float("nan")) == -1


def test_basis_vs_recursive_definition():
    """O2 (triangle) vs the recursive definition for every active function."""
    r = np.random.default_rng(2)
    worst_n = worst_d = 0.0
    for _ in range(400):
        p = int(r.integers(1, 6))
        n = int(r.integers(p + 1, p + 9))
        U = list(rand_knots(r, p, n))
        for u in list(r.uniform(0, 1, 3)) + [0.0, 1.0]:
            s = O.find_span(p, U, u)
            N, dN = O.basis_derivs(p, U, s, u)
            allN, alldN = BF.all_basis(U, p, u)
            for a in range(p + 1):
                worst_n = max(worst_n, abs(N[a] - allN[s - p + a]))
                worst_d = max(worst_d, abs(dN[a] - alldN[s - p + a]) / max(1.0, abs(alldN[s - p + a])))
            # all other functions vanish (local support)
            others = [abs(allN[i]) for i in range(n) if not (s - p <= i <= s)]
            assert max(others, default=0.0) == 0.0
    assert worst_n < 1e-12 and worst_d < 1e-11


def test_partition_of_unity_and_derivative_sum():
    """SPEC S:98 (sum N = 1, N in [0,1]) and S:67 (sum N' = 0)."""
    r = np.random.default_rng(3)
    for _ in range(1000):
        p = int(r.integers(1, 6))
        n = int(r.integers(p + 1, p + 20))
        U = rand_knots(r, p, n)
        u = float(r.uniform(0, 1))
        s = O.find_span(p, U, u)
        N, dN = O.basis_derivs(p, U, s, u)
        assert abs(N.sum() - 1.0) < 1e-12
        assert N.min() >= -1e-15 and N.max() <= 1 + 1e-15
        assert abs(dN.sum()) < 1e-9 * max(1.0, np.abs(dN).max())


def _esym(xs, m):
    return sum(math.prod(c) for c in combinations(xs, m)) if m > 0 else 1.0


def blossom_coeffs(U, p, m):
    """Control values that reproduce u^m exactly: c_i = e_m(U[i+1..i+p]) / C(p,m)
    (polar form / blossom of u^m at the knots), i = 0..n-1."""
    n = len(U) - p - 1
    return np.array([_esym(U[i + 1:i + p + 1], m) / math.comb(p, m) for i in range(n)])


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
def test_polynomial_reproduction_blossom(p):
    """B-splines of degree p reproduce every tensor polynomial of degree <= p
    per axis exactly (north_star); values and gradients."""
    r = np.random.default_rng(10 + p)
    ns = [p + 1 + int(r.integers(0, 6)) for _ in range(3)]
    knots = [rand_knots(r, p, ns[d], multiplicity=False) for d in range(3)]
    for _ in range(6):
        ma, mb, mc = (int(r.integers(0, p + 1)) for _ in range(3))
        cu, cv, cw = (blossom_coeffs(knots[0], p, ma), blossom_coeffs(knots[1], p, mb),
                      blossom_coeffs(knots[2], p, mc))
        ctrl = np.einsum("k,j,i->kji", cw, cv, cu)  # fp64 grid: exact pin
        m = O.Model(p, knots, ctrl)
        for _ in range(20):
            u, v, w = r.uniform(0, 1, 3)
            out, sig, rc = m.eval(u, v, w)
            assert rc == 0
            f = u ** ma * v ** mb * w ** mc
            gu = ma * u ** (ma - 1) * v ** mb * w ** mc if ma else 0.0
            gv = mb * u ** ma * v ** (mb - 1) * w ** mc if mb else 0.0
            gw = mc * u ** ma * v ** mb * w ** (mc - 1) if mc else 0.0
            np.testing.assert_allclose(out, [f, gu, gv, gw], rtol=0, atol=1e-12 * max(1.0, sig.max()))


def test_constant_and_ramp_models():
    """SPEC S:75/S:84 (constant -> c, zero gradient); S:76/S:85 (f = u from
    Greville control values -> u, gradient (1,0,0))."""
    p = 3
    knots = [uniform_knots(p, 9), uniform_knots(p, 7), uniform_knots(p, 8)]
    shape = (8, 7, 9)
    m = O.Model(p, knots, np.full(shape, 0.375, dtype=np.float32))
    r = np.random.default_rng(4)
    for u, v, w in r.uniform(0, 1, (50, 3)):
        out, _, _ = m.eval(u, v, w)
        np.testing.assert_allclose(out, [0.375, 0, 0, 0], atol=1e-14)
    gre = np.array([knots[0][i + 1:i + p + 1].sum() / p for i in range(9)])
    ramp = np.broadcast_to(gre[None, None, :], shape).copy()
    m = O.Model(p, knots, ramp)  # fp64 grid
    for u, v, w in r.uniform(0, 1, (50, 3)):
        out, _, _ = m.eval(u, v, w)
        np.testing.assert_allclose(out, [u, 1, 0, 0], atol=1e-12)


def test_endpoint_interpolation_and_local_support():
    """SPEC S:100 (corners equal corner control values) and S:99 (values
    outside the active block do not matter)."""
    r = np.random.default_rng(5)
    p = 3
    knots = [rand_knots(r, p, 10), rand_knots(r, p, 8), rand_knots(r, p, 9)]
    ctrl = r.normal(size=(9, 8, 10)).astype(np.float32)
    m = O.Model(p, knots, ctrl)
    for cw in (0, 1):
        for cv in (0, 1):
            for cu in (0, 1):
                out, _, _ = m.eval(float(cu), float(cv), float(cw))
                assert out[0] == pytest.approx(float(ctrl[-cw if cw else 0, -cv if cv else 0, -cu if cu else 0]), abs=1e-12)
    u, v, w = 0.43, 0.61, 0.27
    base, _, _ = m.eval(u, v, w)
    su, sv, sw = (O.find_span(p, knots[d], x) for d, x in enumerate((u, v, w)))
    ctrl2 = ctrl.copy()
    mask = np.ones_like(ctrl2, dtype=bool)
    mask[sw - p:sw + 1, sv - p:sv + 1, su - p:su + 1] = False
    ctrl2[mask] = 1e6
    out, _, _ = O.Model(p, knots, ctrl2).eval(u, v, w)
    np.testing.assert_array_equal(out, base)


def test_eval_vs_full_sum_bruteforce():
    """O3 vs the sum over ALL basis functions (bruteforce.eval_full) on tiny
    models with random non-uniform knots: agreement to 1e-12."""
    r = np.random.default_rng(6)
    for p in (1, 2, 3, 4):
        ns = [p + 1 + int(r.integers(0, 4)) for _ in range(3)]
        knots = [rand_knots(r, p, ns[d]) for d in range(3)]
        ctrl = r.normal(size=(ns[2], ns[1], ns[0])).astype(np.float32)
        m = O.Model(p, knots, ctrl)
        pts = list(r.uniform(0, 1, (8, 3))) + [np.array([1.0, 0.0, 1.0]), np.array([0.0, 1.0, 0.5])]
        for u, v, w in pts:
            out, _, _ = m.eval(u, v, w)
            ref = BF.eval_full([list(k) for k in knots], p, ctrl, u, v, w)
            scale = max(1.0, np.abs(ref).max())
            np.testing.assert_allclose(out, ref, rtol=0, atol=1e-12 * scale)


@pytest.mark.parametrize("p", [2, 3, 4])
def test_gradient_vs_central_differences(p):
    """gradient vs central differences; h = 1e-4 span widths,
    normwise to the abs-scale sigma (R-5)."""
    r = np.random.default_rng(20 + p)
    n = (p + 12, p + 9, p + 10)
    knots = [uniform_knots(p, n[d]) for d in range(3)]
    ctrl = r.uniform(-1, 1, (n[2], n[1], n[0])).astype(np.float32)
    m = O.Model(p, knots, ctrl)
    for _ in range(40):
        q = r.uniform(0.05, 0.95, 3)
        out, sig, _ = m.eval(*q)
        for d in range(3):
            h = 1e-4 / (n[d] - p)
            qp = q.copy(); qp[d] += h
            qm = q.copy(); qm[d] -= h
            fd = (m.eval(*qp)[0][0] - m.eval(*qm)[0][0]) / (2 * h)
            assert abs(fd - out[1 + d]) <= 1e-6 * max(sig[1 + d], 1e-30) + 1e-9


def test_domain_errors_give_nan():
    p = 2
    knots = [uniform_knots(p, 5)] * 3
    m = O.Model(p, knots, np.ones((5, 5, 5), np.float32))
    out, _, rc = m.eval(1.5, 0.5, 0.5)
    assert rc == -1 and np.isnan(out).all()
    o, s, e = m.eval_batch(np.array([0.5, np.nan, -0.1], np.float32), np.full(3, 0.5, np.float32),
                           np.full(3, 0.5, np.float32))
    assert e == 2 and not np.isnan(o[0]).any() and np.isnan(o[1]).all() and np.isnan(o[2]).all()


def test_eval_batch_matches_single_and_thread_count():
    r = np.random.default_rng(7)
    p = 3
    knots = [uniform_knots(p, 12)] * 3
    ctrl = r.normal(size=(12, 12, 12)).astype(np.float32)
    m = O.Model(p, knots, ctrl)
    u, v, w = (r.random(500, dtype=np.float32) for _ in range(3))
    o1, s1, _ = m.eval_batch(u, v, w, nthreads=1)
    o7, s7, _ = m.eval_batch(u, v, w, nthreads=7)
    np.testing.assert_array_equal(o1, o7)
    np.testing.assert_array_equal(s1, s7)
    for i in range(0, 500, 97):
        out, sig, _ = m.eval(u[i], v[i], w[i])
        np.testing.assert_array_equal(out, o1[i])


def test_sigma_abs_scales_closed_forms():
    """The abs-scales sigma that set every eval tolerance (R-5): sigma_k =
    sum |term| of the same triple sum.  Closed forms:
      * constant model c: N >= 0 and sum N = 1 per axis, so sigma_val = |c|,
        and sigma_u = |c| * sum_a |N'_a|;
      * on an interior span of a uniform cubic at local t = 1/2,
        N' = S [-1, -5, 5, 1] / 8 (A.1), so sum |N'| = 3 S / 2 and
        sigma_u = 1.5 S |c|;
      * a model with non-negative control values: every value term is >= 0,
        so sigma_val equals the value itself."""
    p = 3
    n = (13, 9, 11)
    S = [n[d] - p for d in range(3)]
    knots = [uniform_knots(p, n[d]) for d in range(3)]
    c = -0.625
    m = O.Model(p, knots, np.full((n[2], n[1], n[0]), c, dtype=np.float32))
    # interior spans (A.1: spans 2p-1 .. n-p, i.e. knot index; here the span
    # starting at knot value j/S with j in [p-1, S-p]) at t = 1/2 on every axis
    j = (S[0] // 2, S[1] // 2, S[2] // 2)
    q = [(j[d] + 0.5) / S[d] for d in range(3)]
    out, sig, rc = m.eval(*q)
    assert rc == 0
    np.testing.assert_allclose(sig, [abs(c), 1.5 * S[0] * abs(c), 1.5 * S[1] * abs(c), 1.5 * S[2] * abs(c)],
                               rtol=1e-14)
    np.testing.assert_allclose(out, [c, 0, 0, 0], atol=1e-12)
    # a generic point: sigma_val = |c|, sigma_d = |c| sum |N'_d| with the O2
    # derivatives (pinned separately against the recursion / closed forms)
    r = np.random.default_rng(31)
    for u, v, w in r.uniform(0, 1, (20, 3)):
        out, sig, _ = m.eval(u, v, w)
        assert sig[0] == pytest.approx(abs(c), rel=1e-14)
        for d, x in enumerate((u, v, w)):
            sp = O.find_span(p, knots[d], x)
            _, dN = O.basis_derivs(p, knots[d], sp, x)
            assert sig[1 + d] == pytest.approx(abs(c) * np.abs(dN).sum(), rel=1e-13)
    # non-negative control values: sigma_val == value (and sigma_val < 1.01 * value)
    ctrl = r.uniform(0.1, 2.0, (n[2], n[1], n[0])).astype(np.float32)
    m2 = O.Model(p, knots, ctrl)
    for u, v, w in r.uniform(0, 1, (20, 3)):
        out, sig, _ = m2.eval(u, v, w)
        assert sig[0] == pytest.approx(out[0], rel=1e-13)
