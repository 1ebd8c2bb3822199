"""TEST INFRASTRUCTURE ONLY: ctypes binding of the fp64 CPU oracle (oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline/reference
leg may import this package.  The product path (paper_2204_11762_b200) never
imports it, and it never imports the product path: the only shared module is
paper_2204_11762_b200.workloads (seeded inputs, no method arithmetic).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle.so")
SRC_PATH = os.path.join(_HERE, "oracle.c")

FLAG_ERT, FLAG_EXIT, FLAG_SHADE = 1, 2, 4


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (portable flags; no FMA contraction)."""
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(SRC_PATH):
        cmd = ["gcc", "-O2", "-std=c11", "-D_GNU_SOURCE", "-fPIC", "-shared", "-ffp-contract=off",
               "-pthread", "-o", LIB_PATH, SRC_PATH, "-lm"]
        subprocess.check_call(cmd)
    return LIB_PATH


class OrcModel(C.Structure):
    _fields_ = [("degree", C.c_int32 * 3), ("nctrl", C.c_int64 * 3),
                ("knots", C.POINTER(C.c_double) * 3), ("ctrl", C.POINTER(C.c_float)),
                ("ctrl64", C.POINTER(C.c_double))]


class OrcCamera(C.Structure):
    _fields_ = [("eye", C.c_double * 3), ("look_at", C.c_double * 3), ("up", C.c_double * 3),
                ("fov_y_deg", C.c_double), ("ortho_half_height", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32)]


class OrcTF(C.Structure):
    _fields_ = [("rgba", C.POINTER(C.c_float)), ("n_entries", C.c_int32),
                ("v_lo", C.c_double), ("v_hi", C.c_double)]


class OrcField(C.Structure):
    _fields_ = [("kind", C.c_int32), ("value_src", C.c_int32), ("grad_src", C.c_int32),
                ("prm", C.c_double * 6)]


class OrcParams(C.Structure):
    _fields_ = [("box_min", C.c_double * 3), ("box_max", C.c_double * 3), ("step", C.c_double),
                ("o_max", C.c_double), ("shading", C.c_int32), ("ka", C.c_double),
                ("kd", C.c_double), ("ks", C.c_double), ("shininess", C.c_double),
                ("grad_eps", C.c_double), ("ert_window", C.c_double), ("exit_window", C.c_double),
                ("sens_weight", C.c_double), ("sens_grad", C.c_double), ("n_lights", C.c_int32),
                ("light_dir", C.POINTER(C.c_double)), ("light_intensity", C.POINTER(C.c_double)),
                ("curv_n", C.c_int32), ("curv_rgba", C.POINTER(C.c_float)), ("curv_range", C.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        dp = C.POINTER(C.c_double)
        _lib.orc_find_span.restype = C.c_int64
        _lib.orc_find_span.argtypes = [C.c_int32, C.c_int64, dp, C.c_double]
        _lib.orc_basis_derivs.restype = None
        _lib.orc_basis_derivs.argtypes = [C.c_int32, dp, C.c_int64, C.c_double, dp, dp]
        _lib.orc_eval.restype = C.c_int
        _lib.orc_eval.argtypes = [C.POINTER(OrcModel), C.c_double, C.c_double, C.c_double, dp, dp]
        _lib.orc_eval_batch.restype = C.c_int64
        fp = C.POINTER(C.c_float)
        _lib.orc_eval_batch.argtypes = [C.POINTER(OrcModel), C.c_int64, fp, fp, fp, dp, dp, C.c_int32]
        _lib.orc_ray.restype = None
        _lib.orc_ray.argtypes = [C.POINTER(OrcCamera), C.c_int32, C.c_int32, dp, dp]
        _lib.orc_clip.restype = C.c_int
        _lib.orc_clip.argtypes = [dp, dp, dp, dp, dp, dp]
        _lib.orc_basis_ders2.restype = None
        _lib.orc_basis_ders2.argtypes = [C.c_int32, dp, C.c_int64, C.c_double, dp, dp, dp]
        _lib.orc_eval_hessian.restype = C.c_int
        _lib.orc_eval_hessian.argtypes = [C.POINTER(OrcModel), C.c_double, C.c_double, C.c_double, dp, dp]
        _lib.orc_eval_hessian_batch.restype = C.c_int64
        _lib.orc_eval_hessian_batch.argtypes = [C.POINTER(OrcModel), C.c_int64, fp, fp, fp, dp, dp, C.c_int32]
        _lib.orc_curvatures.restype = None
        _lib.orc_curvatures.argtypes = [dp, dp, dp]
        _lib.orc_field_eval.restype = C.c_int
        _lib.orc_field_eval.argtypes = [C.POINTER(OrcField), C.c_double, C.c_double, C.c_double, dp]
        _lib.orc_render_ex.restype = C.c_int
        _lib.orc_render_ex.argtypes = [C.POINTER(OrcModel), C.POINTER(OrcCamera), C.POINTER(OrcTF),
                                       C.POINTER(OrcParams), C.POINTER(OrcField), C.c_int64,
                                       C.POINTER(C.c_int64), dp, C.POINTER(C.c_int64), C.POINTER(C.c_uint8),
                                       dp, C.POINTER(C.c_int64), C.c_int32]
        _lib.orc_render.restype = C.c_int
        _lib.orc_render.argtypes = [C.POINTER(OrcModel), C.POINTER(OrcCamera), C.POINTER(OrcTF),
                                    C.POINTER(OrcParams), C.c_int64, C.POINTER(C.c_int64), dp,
                                    C.POINTER(C.c_int64), C.POINTER(C.c_uint8), dp,
                                    C.POINTER(C.c_int64), C.c_int32]
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def ncores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:  # pragma: no cover
        return os.cpu_count() or 1


# ----------------------------------------------------------------------------
# thin wrappers
# ----------------------------------------------------------------------------
def find_span(p: int, knots, u: float) -> int:
    U = np.ascontiguousarray(knots, dtype=np.float64)
    n = len(U) - p - 1
    return int(lib().orc_find_span(p, n, _dp(U), float(u)))


def basis_derivs(p: int, knots, span: int, u: float):
    U = np.ascontiguousarray(knots, dtype=np.float64)
    N = np.zeros(p + 1)
    dN = np.zeros(p + 1)
    lib().orc_basis_derivs(p, _dp(U), span, float(u), _dp(N), _dp(dN))
    return N, dN


def basis_ders2(p: int, knots, span: int, u: float):
    """H1: (N, N', N'') of the p+1 non-zero basis functions on span."""
    U = np.ascontiguousarray(knots, dtype=np.float64)
    N, dN, d2N = np.zeros(p + 1), np.zeros(p + 1), np.zeros(p + 1)
    lib().orc_basis_ders2(p, _dp(U), span, float(u), _dp(N), _dp(dN), _dp(d2N))
    return N, dN, d2N


class Model:
    """Oracle view of a model: degrees, fp64 knots, fp32 grid [n_w][n_v][n_u]."""

    def __init__(self, degree, knots, ctrl):
        if np.isscalar(degree):
            degree = (int(degree),) * 3
        self.knots = [np.ascontiguousarray(k, dtype=np.float64) for k in knots]
        ctrl = np.asarray(ctrl)
        self.ctrl64 = np.ascontiguousarray(ctrl, dtype=np.float64) if ctrl.dtype == np.float64 else None
        self.ctrl = np.ascontiguousarray(ctrl, dtype=np.float32)
        nw, nv, nu = self.ctrl.shape
        self.s = OrcModel()
        for d in range(3):
            self.s.degree[d] = int(degree[d])
            self.s.knots[d] = _dp(self.knots[d])
        self.s.nctrl[0], self.s.nctrl[1], self.s.nctrl[2] = nu, nv, nw
        for d in range(3):
            assert len(self.knots[d]) == self.s.nctrl[d] + self.s.degree[d] + 1
        self.s.ctrl = self.ctrl.ctypes.data_as(C.POINTER(C.c_float))
        if self.ctrl64 is not None:  # fp64 control values (exact pins only)
            self.s.ctrl64 = _dp(self.ctrl64)

    @classmethod
    def from_workload(cls, w):
        return cls(w.degree, w.knots, w.ctrl)

    def eval(self, u, v, w):
        out = np.zeros(4)
        sig = np.zeros(4)
        rc = lib().orc_eval(C.byref(self.s), float(u), float(v), float(w), _dp(out), _dp(sig))
        return out, sig, rc

    def eval_hessian(self, u, v, w):
        """H2: (out[10], sigma[10], rc): v, v_u, v_v, v_w, v_uu, v_vv, v_ww, v_uv, v_uw, v_vw."""
        out = np.zeros(10)
        sig = np.zeros(10)
        rc = lib().orc_eval_hessian(C.byref(self.s), float(u), float(v), float(w), _dp(out), _dp(sig))
        return out, sig, rc

    def eval_hessian_batch(self, u, v, w, nthreads=None):
        """H2 over fp32 point arrays: (out (n,10), sigma (n,10), n_domain_errors)."""
        u = np.ascontiguousarray(u, dtype=np.float32)
        v = np.ascontiguousarray(v, dtype=np.float32)
        w = np.ascontiguousarray(w, dtype=np.float32)
        n = len(u)
        out, sig = np.zeros((n, 10)), np.zeros((n, 10))
        fp = C.POINTER(C.c_float)
        errs = lib().orc_eval_hessian_batch(C.byref(self.s), n, u.ctypes.data_as(fp), v.ctypes.data_as(fp),
                                            w.ctypes.data_as(fp), _dp(out), _dp(sig), nthreads or ncores())
        return out, sig, int(errs)

    def eval_batch(self, u, v, w, nthreads=None):
        u = np.ascontiguousarray(u, dtype=np.float32)
        v = np.ascontiguousarray(v, dtype=np.float32)
        w = np.ascontiguousarray(w, dtype=np.float32)
        n = len(u)
        out = np.zeros((n, 4))
        sig = np.zeros((n, 4))
        fp = C.POINTER(C.c_float)
        errs = lib().orc_eval_batch(C.byref(self.s), n, u.ctypes.data_as(fp), v.ctypes.data_as(fp),
                                    w.ctypes.data_as(fp), _dp(out), _dp(sig), nthreads or ncores())
        return out, sig, int(errs)


def make_camera(cam) -> OrcCamera:
    c = OrcCamera()
    for i in range(3):
        c.eye[i] = cam.eye[i]
        c.look_at[i] = cam.look_at[i]
        c.up[i] = cam.up[i]
    c.fov_y_deg = cam.fov_y_deg
    c.ortho_half_height = cam.ortho_half_height
    c.width = cam.width
    c.height = cam.height
    return c


def ray(cam, px, py):
    o = np.zeros(3)
    d = np.zeros(3)
    c = make_camera(cam)
    lib().orc_ray(C.byref(c), px, py, _dp(o), _dp(d))
    return o, d


def clip(bmin, bmax, o, d):
    bmin = np.ascontiguousarray(bmin, dtype=np.float64)
    bmax = np.ascontiguousarray(bmax, dtype=np.float64)
    o = np.ascontiguousarray(o, dtype=np.float64)
    d = np.ascontiguousarray(d, dtype=np.float64)
    ti = np.zeros(1)
    to = np.zeros(1)
    hit = lib().orc_clip(_dp(bmin), _dp(bmax), _dp(o), _dp(d), _dp(ti), _dp(to))
    return bool(hit), float(ti[0]), float(to[0])


def make_field(field) -> OrcField:
    """field: workloads.AnalyticField (kind, value_src, grad_src, prm)."""
    f = OrcField()
    f.kind = int(field.kind)
    f.value_src = int(field.value_src)
    f.grad_src = int(field.grad_src)
    for i, x in enumerate(field.prm):
        f.prm[i] = float(x)
    return f


def curvatures(g, h6):
    """C1: principal curvatures (k1 >= k2) from a gradient (3,) and Hessian
    {xx, yy, zz, xy, xz, yz}."""
    g = np.ascontiguousarray(g, dtype=np.float64)
    h = np.ascontiguousarray(h6, dtype=np.float64)
    k = np.zeros(2)
    lib().orc_curvatures(_dp(g), _dp(h), _dp(k))
    return k


def field_eval(field, u, v, w):
    """G1: analytic value and parameter-space gradient at (u, v, w)."""
    out = np.zeros(4)
    f = make_field(field)
    rc = lib().orc_field_eval(C.byref(f), float(u), float(v), float(w), _dp(out))
    assert rc == 0
    return out


def render(model: Model, cam, tf, v_lo, v_hi, params, pixels=None, nthreads=None,
           ert_window=1e-4, exit_window=1e-6, sens_weight=1e-3, sens_grad=None, field=None, lights=None,
           curvature=None):
    """Render one view (all pixels, or a flat pixel-index list).  field (a
    workloads.AnalyticField) takes the value and/or gradient of each sample
    from the analytic function instead of the MFA (ground truth).

    Returns dict(rgba (n,4) fp64, count (n,), flags (n,), alt (n,2,4), alt_count (n,2))."""
    tf = np.ascontiguousarray(tf, dtype=np.float32)
    t = OrcTF(tf.ctypes.data_as(C.POINTER(C.c_float)), tf.shape[0], float(v_lo), float(v_hi))
    p = OrcParams()
    for i in range(3):
        p.box_min[i] = params.box_min[i]
        p.box_max[i] = params.box_max[i]
    p.step = params.step
    p.o_max = params.o_max
    p.shading = int(params.shading)
    p.ka, p.kd, p.ks, p.shininess = params.ka, params.kd, params.ks, params.shininess
    p.grad_eps = params.grad_eps
    p.ert_window = ert_window
    p.exit_window = exit_window
    p.sens_weight = sens_weight
    p.sens_grad = (100.0 * params.grad_eps) if sens_grad is None else sens_grad
    if curvature is not None:   # (table float32 (n, n, 4) [kappa_2][kappa_1], range)
        ctab = np.ascontiguousarray(curvature[0], dtype=np.float32)
        p.curv_n = ctab.shape[0]
        p.curv_rgba = ctab.ctypes.data_as(C.POINTER(C.c_float))
        p.curv_range = float(curvature[1])
    if lights is not None:   # [(direction towards the light (3,), intensity), ...]
        ld = np.ascontiguousarray([l[0] for l in lights], dtype=np.float64).reshape(-1, 3)
        li = np.ascontiguousarray([l[1] for l in lights], dtype=np.float64)
        p.n_lights = len(lights)
        p.light_dir = _dp(ld)
        p.light_intensity = _dp(li)
    c = make_camera(cam)
    if pixels is None:
        n = cam.width * cam.height
        pix_ptr = None
    else:
        pixels = np.ascontiguousarray(pixels, dtype=np.int64)
        n = len(pixels)
        pix_ptr = pixels.ctypes.data_as(C.POINTER(C.c_int64))
    rgba = np.zeros((n, 4))
    count = np.zeros(n, dtype=np.int64)
    flags = np.zeros(n, dtype=np.uint8)
    alt = np.zeros((n, 2, 4))
    alt_count = np.zeros((n, 2), dtype=np.int64)
    fptr = C.byref(make_field(field)) if field is not None else None
    lib().orc_render_ex(C.byref(model.s), C.byref(c), C.byref(t), C.byref(p), fptr, n, pix_ptr, _dp(rgba),
                     count.ctypes.data_as(C.POINTER(C.c_int64)),
                     flags.ctypes.data_as(C.POINTER(C.c_uint8)), _dp(alt),
                     alt_count.ctypes.data_as(C.POINTER(C.c_int64)), nthreads or ncores())
    return dict(rgba=rgba, count=count, flags=flags, alt=alt, alt_count=alt_count)
