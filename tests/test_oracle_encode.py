"""Pins for the NEXT-3 oracle (oracle/encode.py): parameterisation,
least-squares fit (constant, polynomial reproduction, square interpolation,
separable == global Kronecker least squares), residuals, and the adaptive
span-splitting loop of Fig. 1.  No GPU."""
import numpy as np
import pytest

from oracle import encode as E
from paper_2204_11762_b200 import workloads as WL
from test_oracle_bspline import blossom_coeffs


def jittered_knots(r, p, n):
    """Non-uniform clamped knots with every span holding samples (interior
    knots k/S moved by up to 0.2/S): the collocation matrix has full column
    rank (Schoenberg-Whitney), so the least-squares solution is unique."""
    S = n - p
    k = np.arange(1, S) / S + r.uniform(-0.2, 0.2, S - 1) / S
    return np.concatenate([np.zeros(p + 1), k, np.ones(p + 1)])


def test_params_spec_examples():
    np.testing.assert_array_equal(E.params(2), [0.0, 1.0])
    np.testing.assert_array_equal(E.params(5), [0.0, 0.25, 0.5, 0.75, 1.0])


def test_fit_constant():
    q = np.full((7, 6, 9), 3.25)
    knots = [E.uniform_knots(n, 2) for n in (5, 4, 6)]
    c = E.fit(q, knots, 2)
    np.testing.assert_allclose(c, 3.25, atol=1e-12)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_fit_reproduces_polynomials(p):
    """A tensor polynomial of degree <= p per axis lies in the spline space,
    so the least-squares fit is exact: the control values are its blossom
    coefficients and the residual vanishes."""
    r = np.random.default_rng(80 + p)
    dims = (11, 9, 10)
    n = (p + 4, p + 3, p + 5)
    knots = [jittered_knots(r, p, n[d]) for d in range(3)]
    e = [int(r.integers(0, p + 1)) for _ in range(3)]
    t = [E.params(m) for m in dims]
    q = np.einsum("k,j,i->kji", t[2] ** e[2], t[1] ** e[1], t[0] ** e[0])
    c = E.fit(q, knots, p)
    want = np.einsum("k,j,i->kji", *(blossom_coeffs(knots[d], p, e[d]) for d in (2, 1, 0)))
    np.testing.assert_allclose(c, want, atol=1e-10)
    err, _ = E.residual(q, c, knots, p)
    assert err.max() <= 1e-10


def test_square_system_interpolates():
    """m = n samples per axis: the collocation matrix is square and invertible,
    the fit interpolates."""
    r = np.random.default_rng(3)
    p = 2
    dims = (6, 5, 7)
    knots = [E.uniform_knots(m, p) for m in dims]
    q = r.normal(size=(dims[2], dims[1], dims[0]))
    c = E.fit(q, knots, p)
    np.testing.assert_allclose(E.evaluate_grid(c, knots, p, dims), q, atol=1e-10)


def test_separable_equals_global_kronecker_lstsq():
    """the separable solution equals the global least-squares solution
    of the full tensor-product design matrix (built explicitly, solved by
    lstsq) on a small grid."""
    r = np.random.default_rng(4)
    p = 2
    dims = (7, 6, 5)
    n = (5, 4, 4)
    knots = [jittered_knots(r, p, n[d]) for d in range(3)]
    q = r.normal(size=(dims[2], dims[1], dims[0]))
    Nu, Nv, Nw = (E.collocation(knots[d], p, E.params(dims[d])) for d in range(3))
    A = np.kron(Nw, np.kron(Nv, Nu))                       # rows (c,b,a) -> columns (k,j,i)
    sol = np.linalg.lstsq(A, q.reshape(-1), rcond=None)[0].reshape(n[2], n[1], n[0])
    np.testing.assert_allclose(E.fit(q, knots, p), sol, atol=1e-10)


def test_adaptive_trivial_cases():
    q = np.full((9, 9, 9), 2.0)
    knots, c, rep = E.adaptive(q, 2, (4, 4, 4), 1e-3, 5, (9, 9, 9))
    assert rep["converged"] and len(rep["rounds"]) == 1
    g = WL.analytic_grid("gb", (12, 12, 12))
    knots, c, rep = E.adaptive(g, 2, (4, 4, 4), 1.0, 5, (12, 12, 12))
    assert rep["converged"] and len(rep["rounds"]) == 1                 # e_max = 1


def test_adaptive_refines_until_tolerance():
    """Gaussian beam on 33^3 samples, p = 2, from 4^3 control points with
    e_max = 0.01: spans are split until every sample is within tolerance; the
    L2 residual never increases (nested least-squares spaces) and the knot
    vectors only gain knots (each at a span midpoint)."""
    q = WL.analytic_grid("gb", (33, 33, 33))
    knots, c, rep = E.adaptive(q, 2, (4, 4, 4), 0.01, 8, (33, 33, 33))
    rounds = rep["rounds"]
    assert rep["converged"] and rounds[-1][1] <= 0.01 and len(rounds) > 1
    assert all(a[0][d] <= b[0][d] for a, b in zip(rounds, rounds[1:]) for d in range(3))
    assert all(b[2] <= a[2] * (1 + 1e-12) for a, b in zip(rounds, rounds[1:]))       # nested LSQ spaces
    for d in range(3):                                  # every added knot halves a span of the round before
        assert set(np.round(E.uniform_knots(4, 2), 15)) <= set(np.round(knots[d], 15))
    err, _ = E.residual(q, c, knots, 2)
    assert err.max() == pytest.approx(rounds[-1][1], rel=1e-12)


def test_gb_regression_pin():
    """Gaussian beam 64^3, degree 2, 32^3 control points -> max relative
    error below 0.05."""
    q = WL.analytic_grid("gb", (64, 64, 64))
    knots = [E.uniform_knots(32, 2)] * 3
    c = E.fit(q, knots, 2)
    err, _ = E.residual(q, c, knots, 2)
    assert err.max() < 0.05


def test_residual_affine_invariance():
    """S:208 (R-28): the relative error is |f - q| / (max q - min q), so it is
    unchanged when data and control values are both scaled by a and shifted by
    b (the B-spline basis sums to one, so the spline of a c + b is a f + b)."""
    r = np.random.default_rng(11)
    q = r.uniform(-1.0, 2.0, (9, 8, 10))
    knots = [E.uniform_knots(n, 2) for n in (6, 5, 5)]
    c = E.fit(q, knots, 2)
    err, per = E.residual(q, c, knots, 2)
    for a, b in ((1.0, 100.0), (3.5, -7.0), (0.01, 5.0)):
        err2, per2 = E.residual(a * q + b, a * c + b, knots, 2)
        np.testing.assert_allclose(err2, err, rtol=1e-9, atol=1e-12)
        for (p1, c1), (p2, c2) in zip(per, per2):
            np.testing.assert_allclose(p2, p1, rtol=1e-9, atol=1e-12)
            np.testing.assert_array_equal(c2, c1)


def test_adaptive_midpoint_split_is_exact():
    """S:191 / S:209: an offending span is split at its parameter midpoint.
    q = (u - 1/2)_+^3 is a cubic spline with one simple knot at 1/2: from one
    span per axis (4 control points, p = 3), the first refinement inserts 1/2
    on every axis (each axis sees the u error through its max over the other
    axes) and the refit reproduces q to rounding, so round 2 converges."""
    mu, mv, mw = 17, 9, 9
    u = E.params(mu)
    line = np.where(u > 0.5, (u - 0.5) ** 3, 0.0)
    q = np.broadcast_to(line[None, None, :], (mw, mv, mu)).copy()
    knots, c, rep = E.adaptive(q, 3, (4, 4, 4), 1e-9, 6, (20, 20, 20))
    rounds = rep["rounds"]
    assert rep["converged"] and len(rounds) == 2 and rounds[-1][1] <= 1e-10
    for d in range(3):
        np.testing.assert_array_equal(knots[d], [0, 0, 0, 0, 0.5, 1, 1, 1, 1])


def test_adaptive_sample_count_guard():
    """R-28: only spans holding >= 2(p+1) samples are split (each half keeps
    >= p+1 samples).  |u - 0.37| is not a spline, so the error stays above
    e_max; with 12 x 9 x 9 samples and p = 3 the first round splits every
    axis at 1/2, after which no span holds 8 samples: the loop stops
    unconverged with exactly one inserted knot per axis."""
    mu, mv, mw = 12, 9, 9
    line = np.abs(E.params(mu) - 0.37)
    q = np.broadcast_to(line[None, None, :], (mw, mv, mu)).copy()
    knots, c, rep = E.adaptive(q, 3, (4, 4, 4), 1e-6, 6, (40, 40, 40))
    assert not rep["converged"] and len(rep["rounds"]) == 2
    for d in range(3):
        np.testing.assert_array_equal(knots[d], [0, 0, 0, 0, 0.5, 1, 1, 1, 1])
