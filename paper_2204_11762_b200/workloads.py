"""Seeded synthetic inputs for the five BASELINE.json configs (C1..C5).

This module is the ONE piece shared by the oracle side (tests, bench's
cpu_baseline leg) and the CUDA side.  It holds no arithmetic of the method:
no span search, no basis, no contraction, no ray casting, no transfer-function
lookup, no shading, no compositing.  It only draws the arrays the method
consumes — knot vectors, an fp32 control grid, a 256-entry RGBA table,
cameras, render parameters, query points — exactly once, from
``np.random.SeedSequence([220411762, config, stream])``.

Recipe (DESIGN.md §3 restates it with citations):

* knots: clamped, p+1 zeros and ones; uniform interior knots k/S (C1-C4);
  C5 non-uniform: interior knots are the inverse CDF of a density with one
  seeded Gaussian "cluster plane" per axis, snapped to fp32-representable
  values so both sides use identical knots.
* control values: a field F sampled at the Greville abscissae
  xi_i = (U[i+1]+...+U[i+p])/p (BASELINE.json configs: "sampled at Greville
  abscissae"), computed in fp64, rounded to fp32.
  C1/C2 Marschner-Lobb (Eq. 2, f_M=6, alpha=0.25, on
  [-1,1]^3), C2 + N(0, sigma=0.01) noise; C3 64 isotropic Gaussians; C4
  8-octave value noise; C5 256 anisotropic Gaussians.
* transfer function: 4 seeded tent ramps (piecewise linear, 256 entries).
* cameras: perspective fov 40 deg on a seeded orbit (C2-C5), orthographic C1.
* Phong constants k_a=0.1, k_d=0.7, k_s=0.2, n=10, headlight; o_max=0.99.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SEED = 220411762
# RNG streams
S_CTRL, S_KNOTS, S_TF, S_CAMERA, S_POINTS, S_PIXELS = 0, 1, 2, 3, 4, 5

KA, KD, KS, SHININESS = 0.1, 0.7, 0.2, 10.0
O_MAX = 0.99
TF_ENTRIES = 256


def rng(config: int, stream: int) -> np.random.Generator:
    return np.random.default_rng(np.random.SeedSequence([SEED, config, stream]))


@dataclass
class Camera:
    eye: tuple
    look_at: tuple
    up: tuple
    fov_y_deg: float          # 0 -> orthographic
    ortho_half_height: float  # used when fov_y_deg == 0
    width: int
    height: int


@dataclass
class RenderParams:
    box_min: tuple
    box_max: tuple
    step: float               # world units
    o_max: float = O_MAX      # early-termination alpha (Alg. 1 line 14)
    shading: int = 1
    ka: float = KA
    kd: float = KD
    ks: float = KS
    shininess: float = SHININESS
    grad_eps: float = 0.0     # |g_phys| <= grad_eps -> ambient only


# Analytic ground-truth fields (NEXT-2; Eq. 1-2) as
# render inputs: which function, its parameters, and which of value /
# gradient each sample takes from it (0 = MFA query, 1 = analytic).
FIELD_GAUSSIAN_BEAM = 1
FIELD_MARSCHNER_LOBB = 2
GB_PARAMS = (0.0, 255.0, 0.0, 1.0 / 3.0, math.sqrt(3.0))   # V_min, V_max, mu, sigma, R
ML_PARAMS = (6.0, 0.25)                                      # f_M, alpha


@dataclass
class AnalyticField:
    kind: int
    value_src: int = 1
    grad_src: int = 1
    prm: tuple = ()

    @staticmethod
    def marschner_lobb(value_src=1, grad_src=1):
        return AnalyticField(FIELD_MARSCHNER_LOBB, value_src, grad_src, ML_PARAMS)

    @staticmethod
    def gaussian_beam(value_src=1, grad_src=1):
        return AnalyticField(FIELD_GAUSSIAN_BEAM, value_src, grad_src, GB_PARAMS)


@dataclass
class Workload:
    name: str
    config: int
    degree: int
    nctrl: tuple              # (n_u, n_v, n_w)
    knots: list               # 3 x float64 arrays, length n+p+1
    ctrl: np.ndarray          # float32, shape (n_w, n_v, n_u), u fastest
    uniform: bool
    tf: np.ndarray            # float32 (256, 4) non-premultiplied RGBA
    v_lo: float
    v_hi: float
    cameras: list
    params: RenderParams
    step_spans: float
    extra: dict = field(default_factory=dict)

    @property
    def spans(self):
        return tuple(n - self.degree for n in self.nctrl)


# ----------------------------------------------------------------------------
# knots and Greville abscissae (input construction only)
# ----------------------------------------------------------------------------
def clamped_uniform_knots(n: int, p: int) -> np.ndarray:
    S = n - p
    interior = np.arange(1, S, dtype=np.float64) / S
    return np.concatenate([np.zeros(p + 1), interior, np.ones(p + 1)])


def clustered_knots(n: int, p: int, q: float, width: float = 0.03,
                    peak: float = 8.0) -> np.ndarray:
    """Clamped non-uniform knots clustered near the plane u=q.

    Interior knots are CDF^{-1}(j/S) of rho(u) = 1 + peak*exp(-(u-q)^2/(2 w^2)),
    rounded to fp32-representable doubles, strictly increasing."""
    S = n - p
    g = np.linspace(0.0, 1.0, 1 << 20, dtype=np.float64)
    rho = 1.0 + peak * np.exp(-((g - q) ** 2) / (2.0 * width * width))
    cdf = np.concatenate([[0.0], np.cumsum(0.5 * (rho[1:] + rho[:-1]) * np.diff(g))])
    cdf /= cdf[-1]
    targets = np.arange(1, S, dtype=np.float64) / S
    interior = np.interp(targets, cdf, g)
    interior = interior.astype(np.float32)
    for j in range(1, len(interior)):  # strictly increasing after snapping
        if interior[j] <= interior[j - 1]:
            interior[j] = np.nextafter(interior[j - 1], np.float32(2.0))
    assert interior[0] > 0.0 and interior[-1] < 1.0
    return np.concatenate([np.zeros(p + 1), interior.astype(np.float64), np.ones(p + 1)])


def greville(knots: np.ndarray, p: int) -> np.ndarray:
    n = len(knots) - p - 1
    return np.array([knots[i + 1:i + p + 1].sum() / p for i in range(n)], dtype=np.float64)


# ----------------------------------------------------------------------------
# fields (inputs sampled at Greville points)
# ----------------------------------------------------------------------------
def marschner_lobb(x, y, z, f_m=6.0, alpha=0.25):
    """PAPER.md Eq. 2, domain [-1,1]^3."""
    r = np.sqrt(x * x + y * y)
    rho = np.cos(2.0 * np.pi * f_m * np.cos(np.pi * r / 2.0))
    return (1.0 - np.sin(np.pi * z / 2.0) + alpha * (1.0 + rho)) / (2.0 * (1.0 + alpha))


def gaussian_beam(x, y, z, vmin=0.0, vmax=255.0, mu=0.0, sigma=1.0 / 3.0, R=math.sqrt(3.0)):
    """PAPER.md Eq. 1."""
    l = np.sqrt(x * x + y * y + z * z) / R
    return vmin + (vmax - vmin) * np.exp(-((l - mu) ** 2) / (2.0 * sigma * sigma))


def _ml_grid(xu, xv, xw):
    x = 2.0 * xu - 1.0
    y = 2.0 * xv - 1.0
    z = 2.0 * xw - 1.0
    return marschner_lobb(x[None, None, :], y[None, :, None], z[:, None, None])


def _gauss_sum_grid(xu, xv, xw, a, c, s):
    """sum_k a_k prod_d exp(-(xi_d - c_kd)^2 / (2 s_kd^2)); separable einsum."""
    gu = np.exp(-((xu[None, :] - c[:, 0:1]) ** 2) / (2.0 * s[:, 0:1] ** 2))  # (K, nu)
    gv = np.exp(-((xv[None, :] - c[:, 1:2]) ** 2) / (2.0 * s[:, 1:2] ** 2))
    gw = np.exp(-((xw[None, :] - c[:, 2:3]) ** 2) / (2.0 * s[:, 2:3] ** 2))
    out = np.empty((len(xw), len(xv), len(xu)), dtype=np.float32)
    K = len(a)
    avu = (a[:, None] * gu)  # (K, nu)
    chunk = max(1, (1 << 24) // (len(xv) * len(xu)))
    for k0 in range(0, len(xw), chunk):
        k1 = min(len(xw), k0 + chunk)
        wv = (gw[:, k0:k1, None] * gv[:, None, :]).reshape(K, -1)  # (K, cw*nv)
        blk = wv.T @ avu                                           # (cw*nv, nu)
        out[k0:k1] = blk.reshape(k1 - k0, len(xv), len(xu)).astype(np.float32)
    return out


def _fade(t):
    return t * t * t * (t * (t * 6.0 - 15.0) + 10.0)


def _value_noise_grid(xu, xv, xw, r: np.random.Generator, octaves=8):
    """sum_o 0.5^o VN_o: lattice U[-1,1] on (f+1)^3, f = 2*2^o, trilinear with
    quintic fade; evaluated separably (one axis at a time)."""
    out = np.zeros((len(xw), len(xv), len(xu)), dtype=np.float64)

    def interp_axis(arr, x, f, axis):
        c = np.minimum(np.floor(x * f).astype(np.int64), f - 1)
        w = _fade(x * f - c)
        a0 = np.take(arr, c, axis=axis)
        a1 = np.take(arr, c + 1, axis=axis)
        shape = [1] * arr.ndim
        shape[axis] = len(x)
        w = w.reshape(shape)
        return a0 * (1.0 - w) + a1 * w

    for o in range(octaves):
        f = 2 * (2 ** o)
        lat = r.uniform(-1.0, 1.0, size=(f + 1, f + 1, f + 1))  # [w][v][u]
        t = interp_axis(lat, xu, f, 2)       # (f+1, f+1, nu)
        t = interp_axis(t, xv, f, 1)         # (f+1, nv, nu)
        cw = np.minimum(np.floor(xw * f).astype(np.int64), f - 1)
        ww = _fade(xw * f - cw)
        chunk = 64
        for k0 in range(0, len(xw), chunk):
            k1 = min(len(xw), k0 + chunk)
            w_ = ww[k0:k1, None, None]
            out[k0:k1] += (0.5 ** o) * (t[cw[k0:k1]] * (1.0 - w_) + t[cw[k0:k1] + 1] * w_)
    return out.astype(np.float32)


# ----------------------------------------------------------------------------
# transfer function, cameras
# ----------------------------------------------------------------------------
def tent_tf(r: np.random.Generator, n_ramps=4, n_entries=TF_ENTRIES) -> np.ndarray:
    c = r.uniform(0.15, 0.85, n_ramps)
    w = r.uniform(0.03, 0.12, n_ramps)
    a = r.uniform(0.02, 0.10, n_ramps)
    col = r.uniform(0.2, 1.0, (n_ramps, 3))
    x = np.arange(n_entries, dtype=np.float64) / (n_entries - 1)
    h = a[:, None] * np.maximum(0.0, 1.0 - np.abs(x[None, :] - c[:, None]) / w[:, None])
    hs = h.sum(axis=0)
    rgb = np.where(hs[:, None] > 0, (h.T @ col) / np.where(hs > 0, hs, 1.0)[:, None], 0.5)
    tf = np.empty((n_entries, 4), dtype=np.float32)
    tf[:, :3] = rgb
    tf[:, 3] = h.max(axis=0)
    return tf


def orbit_camera(theta, phi, L, width, height, fov_y_deg=40.0, center=(0.0, 0.0, 0.0)):
    R = 1.5 * float(np.linalg.norm(L))
    eye = (center[0] + R * math.cos(phi) * math.cos(theta),
           center[1] + R * math.cos(phi) * math.sin(theta),
           center[2] + R * math.sin(phi))
    return Camera(eye=eye, look_at=tuple(center), up=(0.0, 0.0, 1.0), fov_y_deg=fov_y_deg,
                  ortho_half_height=0.5 * float(np.linalg.norm(L)), width=width, height=height)


# ----------------------------------------------------------------------------
# configs
# ----------------------------------------------------------------------------
CONFIGS = {
    1: dict(p=2, n=(16, 16, 16), image=(64, 64), views=1, step=0.5, ortho=True),
    2: dict(p=3, n=(64, 64, 64), image=(512, 512), views=1, step=0.5),
    3: dict(p=3, n=(256, 256, 256), image=(1024, 1024), views=1, step=0.25),
    4: dict(p=4, n=(512, 512, 512), image=(2048, 2048), views=1, step=0.25),
    5: dict(p=3, n=(1024, 256, 256), image=(3840, 2160), views=64, step=0.25, nonuniform=True),
}
NAMES = {
    1: "C1-ml16-p2-64ortho",
    2: "C2-ml64noise-p3-512persp",
    3: "C3-gauss256-p3-1024persp",
    4: "C4-fractal512-p4-2048persp",
    5: "C5-aniso1024x256x256-p3-nonuniform-64x3840x2160",
}


def _box(spans):
    m = max(spans)
    L = np.array([s / m for s in spans], dtype=np.float64)
    return L, tuple(-L / 2), tuple(L / 2)


def grad_eps_for(ctrl: np.ndarray, knots, p: int, L) -> float:
    """Threshold below which the physical gradient counts as zero (ambient
    only): 1e-5 * max|P| * max_d p/(L_d * h_min_d)."""
    g = 0.0
    for d in range(3):
        h = np.diff(knots[d])
        hmin = h[h > 0].min()
        g = max(g, p / (L[d] * hmin))
    return float(1e-5 * float(np.abs(ctrl).max()) * g)


def make_config(c: int, *, width: int | None = None, height: int | None = None,
                n_views: int | None = None, nctrl: tuple | None = None) -> Workload:
    """Build config c (1..5). Overrides shrink images / views / grids for
    quick tests while keeping the recipe (the seeds do not change)."""
    cfg = CONFIGS[c]
    p = cfg["p"]
    n = tuple(nctrl) if nctrl is not None else cfg["n"]
    if cfg.get("nonuniform"):
        rk = rng(c, S_KNOTS)
        q = rk.uniform(0.2, 0.8, 3)
        knots = [clustered_knots(n[d], p, float(q[d])) for d in range(3)]
    else:
        knots = [clamped_uniform_knots(n[d], p) for d in range(3)]
    xi = [greville(knots[d], p) for d in range(3)]
    r = rng(c, S_CTRL)
    if c == 1:
        ctrl = _ml_grid(*xi).astype(np.float32)
    elif c == 2:
        g = _ml_grid(*xi)
        g = g + r.normal(0.0, 0.01, size=g.shape)
        ctrl = g.astype(np.float32)
    elif c == 3:
        K = 64
        cc = r.uniform(0.0, 1.0, (K, 3))
        s = r.uniform(0.01, 0.1, K)
        a = r.uniform(-1.0, 1.0, K)
        ctrl = _gauss_sum_grid(*xi, a, cc, np.repeat(s[:, None], 3, axis=1))
    elif c == 4:
        ctrl = _value_noise_grid(*xi, r)
    elif c == 5:
        K = 256
        cc = r.uniform(0.0, 1.0, (K, 3))
        s = r.uniform(0.01, 0.1, (K, 3))
        a = r.uniform(-1.0, 1.0, K)
        ctrl = _gauss_sum_grid(*xi, a, cc, s)
    else:
        raise ValueError(c)
    ctrl = np.ascontiguousarray(ctrl, dtype=np.float32)
    spans = tuple(n[d] - p for d in range(3))
    L, bmin, bmax = _box(spans)
    step = cfg["step"] / max(spans)
    tf = tent_tf(rng(c, S_TF))
    v_lo = float(ctrl.min())
    v_hi = float(ctrl.max())
    W, H = cfg["image"]
    W = width or W
    H = height or H
    V = n_views or cfg["views"]
    rc = rng(c, S_CAMERA)
    cams = []
    if cfg.get("ortho"):
        cam = orbit_camera(math.radians(30.0), math.radians(25.0), L, W, H, fov_y_deg=0.0)
        cams = [cam] * V
    elif c == 5:
        th0 = rc.uniform(0.0, 2.0 * math.pi)
        full_views = cfg["views"]
        cams = [orbit_camera(th0 + 2.0 * math.pi * v / full_views, math.radians(20.0), L, W, H)
                for v in range(V)]
    else:
        for _ in range(V):
            th = rc.uniform(0.0, 2.0 * math.pi)
            ph = math.radians(rc.uniform(15.0, 35.0))
            cams.append(orbit_camera(th, ph, L, W, H))
    params = RenderParams(box_min=bmin, box_max=bmax, step=step,
                          grad_eps=grad_eps_for(ctrl, knots, p, L))
    return Workload(name=NAMES[c], config=c, degree=p, nctrl=n, knots=knots, ctrl=ctrl,
                    uniform=not cfg.get("nonuniform", False), tf=tf, v_lo=v_lo, v_hi=v_hi,
                    cameras=cams, params=params, step_spans=cfg["step"])


# ----------------------------------------------------------------------------
# query points and pixel subsets
# ----------------------------------------------------------------------------
def query_points(c: int, n: int):
    """n iid U[0,1) fp32 points (SoA) for mfa_eval_batch (config C3: n=2^24)."""
    r = rng(c, S_POINTS)
    return (r.random(n, dtype=np.float32), r.random(n, dtype=np.float32),
            r.random(n, dtype=np.float32))


def boundary_points(w: Workload):
    """Boundary set (SURVEY §8(c) acceptance): u in {0, 1, 1-ulp, fp32(k/S)}
    combined over axes with the corners."""
    vals = []
    for d in range(3):
        S = w.spans[d]
        kk = np.unique(np.clip(np.array([0, 1, 2, S // 2, S - 2, S - 1, S]), 0, S))
        interior = np.array([w.knots[d][w.degree + k] for k in kk], dtype=np.float32)
        v = np.concatenate([[0.0, 1.0, np.nextafter(np.float32(1), np.float32(0))], interior])
        vals.append(np.unique(v.astype(np.float32)))
    U, V, W = np.meshgrid(vals[0], vals[1], vals[2], indexing="ij")
    return (U.ravel().astype(np.float32), V.ravel().astype(np.float32),
            W.ravel().astype(np.float32))


def tile_subset(c: int, width: int, height: int, frac: float, tile=16, views=(0,)):
    """Seeded subset of 16x16 tiles -> flat pixel indices per view."""
    r = rng(c, S_PIXELS)
    tx = (width + tile - 1) // tile
    ty = (height + tile - 1) // tile
    out = {}
    for v in views:
        nt = tx * ty
        k = max(1, int(round(frac * nt)))
        sel = np.sort(r.choice(nt, size=k, replace=False))
        pix = []
        for t in sel:
            x0 = (t % tx) * tile
            y0 = (t // tx) * tile
            ys, xs = np.meshgrid(np.arange(y0, min(y0 + tile, height)),
                                 np.arange(x0, min(x0 + tile, width)), indexing="ij")
            pix.append((ys * width + xs).ravel())
        out[v] = np.concatenate(pix).astype(np.int64)
    return out


# ----------------------------------------------------------------------------
# NEXT-2 quality workloads: the paper's ground-truth protocol
# ----------------------------------------------------------------------------
QUALITY_TESTS = ("value", "gradient", "overall")


def ramp_red_tf(n_entries=TF_ENTRIES, a_max=0.08) -> np.ndarray:
    """Value test: "the ramp function is used as the opacity transfer
    function ... The color transfer function is constant red"."""
    t = np.zeros((n_entries, 4), np.float32)
    t[:, 0] = 1.0
    t[:, 3] = np.linspace(0.0, a_max, n_entries)
    return t


def step_white_tf(n_entries=TF_ENTRIES, s0=0.5) -> np.ndarray:
    """Gradient / overall tests: "A step function is used as the
    opacity transfer function in order to construct a surface ... The color
    transfer function is constant white"."""
    t = np.ones((n_entries, 4), np.float32)
    t[:, 3] = (np.arange(n_entries) / (n_entries - 1) >= s0).astype(np.float32)
    return t


def make_quality(kind: str = "ml", n: int = 64, p: int = 3, test: str = "overall", width: int = 512,
                 height: int = 512, theta: float = 0.6, phi: float = 0.45, step_spans: float = 0.5):
    """An MFA of the analytic function (control values = F at the Greville
    abscissae, uniform knots, degree p, n^3 control points) and the pair of
    renderings the paper compares: returns (workload, field of the MFA image,
    field of the ground-truth image, shading).  kind: "ml" (Eq. 2) or "gb"
    (Eq. 1); test: "value" (shading off, both images' values differ), "gradient"
    (both take the analytic value, the MFA image the MFA gradient), "overall"."""
    assert test in QUALITY_TESTS
    knots = [clamped_uniform_knots(n, p) for _ in range(3)]
    xi = [2.0 * greville(k, p) - 1.0 for k in knots]
    f = marschner_lobb if kind == "ml" else gaussian_beam
    ctrl = f(xi[0][None, None, :], xi[1][None, :, None], xi[2][:, None, None]).astype(np.float32)
    spans = (n - p,) * 3
    L, bmin, bmax = _box(spans)
    make_field = AnalyticField.marschner_lobb if kind == "ml" else AnalyticField.gaussian_beam
    shading = 0 if test == "value" else 1
    tf = ramp_red_tf() if test == "value" else step_white_tf()
    cam = orbit_camera(theta, phi, L, width, height)
    params = RenderParams(box_min=bmin, box_max=bmax, step=step_spans / max(spans), shading=shading,
                          grad_eps=grad_eps_for(ctrl, knots, p, L))
    w = Workload(name=f"Q-{kind}{n}-p{p}-{test}-{width}x{height}", config=0, degree=p, nctrl=(n, n, n),
                 knots=knots, ctrl=np.ascontiguousarray(ctrl), uniform=True, tf=tf, v_lo=float(ctrl.min()),
                 v_hi=float(ctrl.max()), cameras=[cam], params=params, step_spans=step_spans)
    mfa_field = {"value": None, "gradient": make_field(1, 0), "overall": None}[test]
    return w, mfa_field, make_field(1, 1)


# ----------------------------------------------------------------------------
# NEXT-3 encoder inputs: structured grids of the analytic functions
# ----------------------------------------------------------------------------
def analytic_grid(kind: str, dims, noise: float = 0.0, seed: int = 0) -> np.ndarray:
    """Grid (m_w, m_v, m_u) of Eq. 1 ("gb") or Eq. 2 ("ml") sampled at the
    uniform parameters j/(m-1) mapped to [-1,1], fp64; optional iid
    N(0, noise) (the discrete datasets of P:155 'generated from those
    functions')."""
    mu, mv, mw = dims
    x = [2.0 * np.arange(m) / (m - 1) - 1.0 for m in (mu, mv, mw)]
    f = marschner_lobb if kind == "ml" else gaussian_beam
    g = f(x[0][None, None, :], x[1][None, :, None], x[2][:, None, None])
    if noise:
        g = g + np.random.default_rng(seed).normal(0.0, noise, g.shape)
    return np.ascontiguousarray(g)
