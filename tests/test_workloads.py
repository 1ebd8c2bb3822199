"""Input generator checks: seeded determinism, valid clamped knots (SPEC
S:24-27), C5 knots fp32-representable (R-3), and the Marschner-Lobb /
Gaussian-beam pins (Eq. 1-2)."""
import math

import numpy as np

from paper_2204_11762_b200 import workloads as W


def test_marschner_lobb_pins():
    assert W.marschner_lobb(0.0, 0.0, -1.0) == 1.0
    assert abs(W.marschner_lobb(0.0, 0.0, 1.0) - 0.2) < 1e-15
    r = np.random.default_rng(0)
    x, y, z = r.uniform(-1, 1, (3, 100000))
    f = W.marschner_lobb(x, y, z)
    assert f.min() >= 0.0 and f.max() <= 1.0


def test_gaussian_beam_pins():
    assert W.gaussian_beam(0.0, 0.0, 0.0) == 255.0
    assert abs(W.gaussian_beam(1.0, 1.0, 1.0) - 255.0 * math.exp(-4.5)) < 1e-12


def _valid_knots(U, p, n):
    assert len(U) == n + p + 1
    assert np.all(np.diff(U) >= 0)
    assert np.all(U[:p + 1] == 0) and np.all(U[-p - 1:] == 1)
    vals, counts = np.unique(U[p + 1:-p - 1], return_counts=True)
    assert counts.max(initial=0) <= p


def test_configs_small_are_deterministic_and_valid():
    for c in (1, 2):
        a = W.make_config(c)
        b = W.make_config(c)
        np.testing.assert_array_equal(a.ctrl, b.ctrl)
        np.testing.assert_array_equal(a.tf, b.tf)
        assert a.cameras == b.cameras
        for d in range(3):
            _valid_knots(a.knots[d], a.degree, a.nctrl[d])
        assert a.ctrl.shape == (a.nctrl[2], a.nctrl[1], a.nctrl[0]) and a.ctrl.dtype == np.float32
        assert a.v_lo == float(a.ctrl.min()) and a.v_hi == float(a.ctrl.max())
        assert a.tf.shape == (256, 4) and a.tf.dtype == np.float32
        assert 0 <= a.tf.min() and a.tf.max() <= 1


def test_c5_knots_nonuniform_fp32_representable():
    p = 3
    r = W.rng(5, W.S_KNOTS)
    q = r.uniform(0.2, 0.8, 3)
    for n, qq in zip((1024, 256, 256), q):
        U = W.clustered_knots(n, p, float(qq))
        _valid_knots(U, p, n)
        assert np.all(U.astype(np.float32).astype(np.float64) == U)
        h = np.diff(U[p:n + 1])
        assert h.min() > 0 and h.max() / h.min() > 3      # clustered


def test_query_points_and_tiles():
    u, v, w = W.query_points(3, 1000)
    assert u.dtype == np.float32 and (0 <= u).all() and (u < 1).all()
    u2, _, _ = W.query_points(3, 1000)
    np.testing.assert_array_equal(u, u2)
    t = W.tile_subset(4, 100, 60, 0.2)
    pix = t[0]
    assert len(np.unique(pix)) == len(pix) and pix.max() < 6000
