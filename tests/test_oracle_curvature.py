"""Pins for the oracle's curvature transfer function (C1; "curvature-based
transfer function (Kindlmann et al. 2003)", an application of
the second derivatives of P:78; R-31): principal curvatures of closed-form
isosurfaces, and the routing of the curvature table into the render.  No GPU."""
import dataclasses

import numpy as np
import pytest

import oracle as O
from paper_2204_11762_b200 import workloads as WL
from test_oracle_bspline import blossom_coeffs, uniform_knots


def test_sphere_cylinder_plane_saddle():
    r = np.random.default_rng(11)
    for _ in range(20):
        x = r.uniform(-1, 1, 3)
        rad = np.linalg.norm(x)
        # f = |x|^2: spheres, both curvatures -1/r (outward normal n = -g/|g| ... points inward here)
        # umbilic: 2F^2 - T^2 = 0 exactly, so rounding in it is amplified by the sqrt (~1e-8)
        np.testing.assert_allclose(O.curvatures(2 * x, [2, 2, 2, 0, 0, 0]), [-1 / rad, -1 / rad], rtol=1e-7)
        # f = x^2 + y^2: cylinders, curvatures (0, -1/r_xy)
        rxy = np.hypot(x[0], x[1])
        np.testing.assert_allclose(O.curvatures([2 * x[0], 2 * x[1], 0], [2, 2, 0, 0, 0, 0]), [0, -1 / rxy],
                                   rtol=1e-12, atol=1e-12)
        # a plane (constant gradient, zero Hessian)
        np.testing.assert_allclose(O.curvatures(x, [0] * 6), [0, 0], atol=1e-15)
    # F = x^2 - y^2 - z at the origin: g = (0,0,-1), H = diag(2,-2,0) -> kappa = +-2
    np.testing.assert_allclose(O.curvatures([0, 0, -1], [2, -2, 0, 0, 0, 0]), [2, -2], rtol=1e-14)
    np.testing.assert_array_equal(O.curvatures([0, 0, 0], [1, 2, 3, 4, 5, 6]), [0, 0])    # R-31


def test_curvature_of_an_exact_quadratic_model():
    """A p = 2 model reproducing f = |xi - c|^2 exactly (blossom control
    values) has spherical level sets in parameter space; on a unit cube box
    (L = 1) the curvature at any point is -1/|xi - c| on both axes (the
    oracle's Hessian -> curvature chain end to end)."""
    p, n = 2, 7
    U = uniform_knots(p, n)
    c = np.array([0.45, 0.52, 0.38])
    # f = sum_d (xi_d^2 - 2 c_d xi_d + c_d^2): tensor sum of 1-D quadratics
    one = blossom_coeffs(U, p, 0)
    lin = blossom_coeffs(U, p, 1)
    sq = blossom_coeffs(U, p, 2)
    axis = [sq - 2 * c[d] * lin + c[d] ** 2 * one for d in range(3)]
    ctrl = (axis[0][None, None, :] * one[None, :, None] * one[:, None, None]
            + one[None, None, :] * axis[1][None, :, None] * one[:, None, None]
            + one[None, None, :] * one[None, :, None] * axis[2][:, None, None])
    m = O.Model(p, [U, U, U], ctrl)
    r = np.random.default_rng(12)
    for q in r.uniform(0.05, 0.95, (20, 3)):
        out, _, _ = m.eval_hessian(*q)
        k = O.curvatures(out[1:4], out[4:10])
        rad = np.linalg.norm(q - c)
        np.testing.assert_allclose(k, [-1 / rad, -1 / rad], rtol=1e-7)   # umbilic (see above)


def test_constant_curvature_table_scales_colour_and_opacity():
    """A constant table (k, k, k, k) multiplies every sample's TF colour and
    opacity by k: the same image as the plain render with the TF scaled by k."""
    w = WL.make_config(2, width=48, height=40)
    om = O.Model.from_workload(w)
    cam = w.cameras[0]
    k = 0.6
    tab = np.full((9, 9, 4), k, np.float32)
    a = O.render(om, cam, w.tf, w.v_lo, w.v_hi, w.params, curvature=(tab, 30.0))
    b = O.render(om, cam, (w.tf.astype(np.float64) * k).astype(np.float32), w.v_lo, w.v_hi, w.params)
    np.testing.assert_array_equal(a["count"], b["count"])
    np.testing.assert_allclose(a["rgba"], b["rgba"], rtol=0, atol=1e-7)    # fp32 products of the scaled table


def test_curvature_table_is_used():
    """A table that is opaque white only for kappa_1 < 0 (convex from the
    normal's side) and transparent elsewhere changes the image, and with
    shading off, every composited sample passed kappa_1 < 0 on its way."""
    w = WL.make_config(2, width=48, height=40)
    om = O.Model.from_workload(w)
    cam = w.cameras[0]
    tab = np.zeros((5, 5, 4), np.float32)
    tab[:, :2, :] = 1.0      # kappa_1 index 0, 1 -> [-R, -R/2]
    prm = dataclasses.replace(w.params, shading=0)
    a = O.render(om, cam, w.tf, w.v_lo, w.v_hi, prm, curvature=(tab, 20.0))
    b = O.render(om, cam, w.tf, w.v_lo, w.v_hi, prm)
    assert np.abs(a["rgba"] - b["rgba"]).max() > 1e-3
    assert (a["rgba"][:, 3] <= b["rgba"][:, 3] + 1e-12).all()
