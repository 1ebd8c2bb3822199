"""Pins for the NEXT-4 oracle (second derivatives; "Higher-order
derivatives, up to the polynomial degree, are also analytically
available"): H1 basis second derivatives, H2 the 6-component Hessian as a
plain triple sum.  No GPU."""
import math

import numpy as np
import pytest

import oracle as O
from test_oracle_bspline import blossom_coeffs, rand_knots, uniform_knots


def test_worked_example_p2():
    """p = 2, U = [0,0,0,1/2,1,1,1], u = 1/4 (span 2): N_0 = (1-2u)^2,
    N_2 = 2u^2, N_1 = 1 - N_0 - N_2, so N'' = [8, -12, 4] (by hand)."""
    U = np.array([0, 0, 0, 0.5, 1, 1, 1.0])
    N, dN, d2N = O.basis_ders2(2, U, 2, 0.25)
    np.testing.assert_allclose(N, [0.25, 0.625, 0.125], atol=1e-15)
    np.testing.assert_allclose(dN, [-2, 1, 1], atol=1e-14)
    np.testing.assert_allclose(d2N, [8, -12, 4], atol=1e-13)


def test_uniform_cubic_interior_closed_form():
    """Uniform cubic pieces b0 = (1-t)^3/6, b1 = (3t^3-6t^2+4)/6,
    b2 = (-3t^3+3t^2+3t+1)/6, b3 = t^3/6: b'' = [1-t, 3t-2, 1-3t, t];
    at t = 1/2 and span width 1/S: N'' = S^2 [1/2, -1/2, -1/2, 1/2]."""
    p, n = 3, 12
    S = n - p
    U = uniform_knots(p, n)
    for sp in range(2 * p - 1, S - p + 1):        # interior spans (local index)
        span = sp + p
        u = (sp + 0.5) / S
        N, dN, d2N = O.basis_ders2(p, U, span, u)
        np.testing.assert_allclose(N, np.array([1, 23, 23, 1]) / 48, atol=1e-14)
        np.testing.assert_allclose(d2N, S * S * np.array([0.5, -0.5, -0.5, 0.5]), atol=1e-10)


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
def test_second_derivative_sum_zero_and_fd(p):
    """sum N'' = 0 (partition of unity); N'' = central differences of N'
    (O2, an independent routine) away from knots; degree 1 -> N'' = 0."""
    r = np.random.default_rng(30 + p)
    for _ in range(60):
        n = p + 1 + int(r.integers(1, 8))
        U = rand_knots(r, p, n)
        u = float(r.uniform(0.02, 0.98))
        s = O.find_span(p, U, u)
        h = 1e-6 * (U[s + 1] - U[s])
        if not (U[s] < u - 2 * h and u + 2 * h < U[s + 1]):
            continue
        N, dN, d2N = O.basis_ders2(p, U, s, u)
        N0, dN0 = O.basis_derivs(p, U, s, u)
        np.testing.assert_allclose(N, N0, atol=1e-14)
        np.testing.assert_allclose(dN, dN0, atol=1e-9 * max(1.0, np.abs(dN0).max()))
        scale = max(1.0, np.abs(d2N).max())
        assert abs(d2N.sum()) <= 1e-9 * scale
        fd = (O.basis_derivs(p, U, s, u + h)[1] - O.basis_derivs(p, U, s, u - h)[1]) / (2 * h)
        np.testing.assert_allclose(d2N, fd, atol=2e-4 * scale)
        if p == 1:
            assert (d2N == 0).all()


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5])
def test_hessian_polynomial_reproduction(p):
    """Blossom control values reproduce u^a v^b w^c exactly, so the Hessian
    must equal the polynomial's second partials (to fp64 rounding)."""
    r = np.random.default_rng(40 + p)
    ns = [p + 1 + int(r.integers(0, 6)) for _ in range(3)]
    knots = [rand_knots(r, p, ns[d], multiplicity=False) for d in range(3)]
    for _ in range(6):
        e = [int(r.integers(0, p + 1)) for _ in range(3)]
        c = [blossom_coeffs(knots[d], p, e[d]) for d in range(3)]
        m = O.Model(p, knots, np.einsum("k,j,i->kji", c[2], c[1], c[0]))
        for _ in range(15):
            q = r.uniform(0, 1, 3)

            def mono(d, k):  # k-th derivative of q_d^e_d
                if k > e[d]:
                    return 0.0
                return math.perm(e[d], k) * q[d] ** (e[d] - k)

            ords = [(0, 0, 0), (1, 0, 0), (0, 1, 0), (0, 0, 1), (2, 0, 0), (0, 2, 0), (0, 0, 2),
                    (1, 1, 0), (1, 0, 1), (0, 1, 1)]
            want = [mono(0, a) * mono(1, b) * mono(2, cc) for a, b, cc in ords]
            out, sig, rc = m.eval_hessian(*q)
            assert rc == 0
            np.testing.assert_allclose(out, want, rtol=0, atol=1e-10 * max(1.0, sig.max()))


@pytest.mark.parametrize("p", [2, 3, 4])
def test_hessian_vs_gradient_differences_and_eval(p):
    """H2 agrees with O3 on value and gradient, is symmetric by construction,
    and equals central differences of O3's gradient (h = 1e-5 span widths)."""
    r = np.random.default_rng(50 + p)
    n = (p + 10, p + 8, p + 9)
    knots = [rand_knots(r, p, n[d], multiplicity=False) for d in range(3)]
    ctrl = r.uniform(-1, 1, (n[2], n[1], n[0])).astype(np.float32)
    m = O.Model(p, knots, ctrl)
    pairs = {(0, 0): 4, (1, 1): 5, (2, 2): 6, (0, 1): 7, (0, 2): 8, (1, 2): 9}
    for _ in range(30):
        q = r.uniform(0.05, 0.95, 3)
        out, sig, _ = m.eval_hessian(*q)
        g, gs, _ = m.eval(*q)
        np.testing.assert_allclose(out[:4], g, atol=1e-13 * max(1.0, gs.max()))
        spans = [O.find_span(p, knots[d], q[d]) for d in range(3)]
        for (i, j), k in pairs.items():
            s = spans[j]
            h = 1e-5 * (knots[j][s + 1] - knots[j][s])
            if not (knots[j][s] < q[j] - h and q[j] + h < knots[j][s + 1]):
                continue
            qp, qm = q.copy(), q.copy()
            qp[j] += h
            qm[j] -= h
            fd = (m.eval(*qp)[0][1 + i] - m.eval(*qm)[0][1 + i]) / (2 * h)
            assert abs(fd - out[k]) <= 1e-5 * sig[k] + 1e-9, (p, i, j, fd, out[k], sig[k])


def test_hessian_batch_matches_single():
    r = np.random.default_rng(60)
    p, n = 3, (9, 8, 7)
    knots = [rand_knots(r, p, n[d]) for d in range(3)]
    m = O.Model(p, knots, r.uniform(-1, 1, (n[2], n[1], n[0])).astype(np.float32))
    u, v, w = (r.random(50, dtype=np.float32) for _ in range(3))
    u[3] = 1.5
    out, sig, errs = m.eval_hessian_batch(u, v, w, nthreads=3)
    assert errs == 1 and np.isnan(out[3]).all()
    for i in (0, 7, 49):
        o, s_, _ = m.eval_hessian(u[i], v[i], w[i])
        np.testing.assert_array_equal(out[i], o)
