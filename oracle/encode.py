"""TEST INFRASTRUCTURE ONLY: fp64 numpy oracle of the MFA encoder (NEXT-3).
Only tests/ and bench.py's CPU legs may import it; it shares nothing with
the CUDA path (csrc/encode.cu).

What it computes (Fig. 1 caption P:88; readings R-27..R-29
in DESIGN.md, after SPEC S:124-200):

  E1 parameterize   structured grid of m_d samples per axis -> t_j = j/(m_d - 1)
  E2 collocation    N_d[j, i] = N_{i,p}(t_j) (Cox-de Boor via oracle.basis_derivs)
  E3 fit            least squares min ||(N_w (x) N_v (x) N_u) c - q||_2, solved
                    separably: c = q x_u pinv(N_u) x_v pinv(N_v) x_w pinv(N_w)
                    (pinv(A (x) B) = pinv(A) (x) pinv(B), so this IS the global
                    tensor-product least-squares solution); numpy's lstsq/pinv is
                    the library primitive
  E4 residual       error at every input sample: |(N_w (x) N_v (x) N_u) c - q| / (max q - min q)
  E5 adapt          "New control points and knots are added adaptively until all
                    evaluated points in each span of knots are within the allowable
                    maximum relative error ... knot spans that fall beyond the
                    tolerance are subdivided, and MFA is recomputed":
                    per axis, a span's error = max error over the samples whose
                    coordinate on that axis lies in the span; every span above
                    e_max holding >= 2(p+1) samples is split at its midpoint (so every
                    span keeps >= p+1 samples and the normal equations stay
                    regular, Schoenberg-Whitney), within
                    the per-axis control-count cap; stop when the max error <= e_max,
                    after max_rounds, or when nothing can be split.
"""
from __future__ import annotations

import numpy as np

import oracle as O


def params(m: int) -> np.ndarray:
    """E1: uniform parameters of m >= 2 grid samples."""
    return np.arange(m, dtype=np.float64) / (m - 1)


def uniform_knots(n: int, p: int) -> np.ndarray:
    S = n - p
    return np.concatenate([np.zeros(p + 1), np.arange(1, S) / S, np.ones(p + 1)])


def collocation(knots, p: int, t) -> np.ndarray:
    """E2: dense N[j, i] = N_{i,p}(t_j)."""
    n = len(knots) - p - 1
    N = np.zeros((len(t), n))
    for j, tj in enumerate(t):
        s = O.find_span(p, knots, float(tj))
        vals, _ = O.basis_derivs(p, knots, s, float(tj))
        N[j, s - p:s + 1] = vals
    return N


def fit(q, knots, p: int) -> np.ndarray:
    """E3: control values (n_w, n_v, n_u) fitting grid values q (m_w, m_v, m_u)."""
    q = np.asarray(q, dtype=np.float64)
    mw, mv, mu = q.shape
    Nu, Nv, Nw = (collocation(knots[d], p, params(m)) for d, m in enumerate((mu, mv, mw)))
    Pu, Pv, Pw = np.linalg.pinv(Nu), np.linalg.pinv(Nv), np.linalg.pinv(Nw)
    return np.einsum("ia,jb,kc,cba->kji", Pu, Pv, Pw, q, optimize=True)


def evaluate_grid(c, knots, p: int, dims) -> np.ndarray:
    """The spline at every grid sample: (N_w (x) N_v (x) N_u) c."""
    mu, mv, mw = dims
    Nu, Nv, Nw = (collocation(knots[d], p, params(m)) for d, m in enumerate((mu, mv, mw)))
    return np.einsum("ai,bj,ck,kji->cba", Nu, Nv, Nw, c, optimize=True)


def residual(q, c, knots, p: int):
    """E4: relative errors at the samples and, per axis, the max over each span."""
    q = np.asarray(q, dtype=np.float64)
    mw, mv, mu = q.shape
    rng = float(q.max() - q.min()) or 1.0
    err = np.abs(evaluate_grid(c, knots, p, (mu, mv, mw)) - q) / rng
    per_axis = []
    for d, m in enumerate((mu, mv, mw)):
        t = params(m)
        U = knots[d]
        spans = np.array([O.find_span(p, U, float(x)) for x in t]) - p
        e_line = err.max(axis=tuple(a for a in range(3) if a != 2 - d))   # max over the other axes
        nsp = len(U) - 2 * p - 1
        per = np.zeros(nsp)
        cnt = np.zeros(nsp, dtype=np.int64)
        for j in range(m):
            per[spans[j]] = max(per[spans[j]], e_line[j])
            cnt[spans[j]] += 1
        per_axis.append((per, cnt))
    return err, per_axis


def adaptive(q, p: int, nctrl, e_max: float, max_rounds: int, max_ctrl):
    """E5: returns (knots, c, report); report["rounds"] = list of (nctrl, max
    relative error, rms relative error) per round."""
    knots = [uniform_knots(nctrl[d], p) for d in range(3)]
    report = []
    converged = False
    while True:
        c = fit(q, knots, p)
        err, per_axis = residual(q, c, knots, p)
        report.append((tuple(len(k) - p - 1 for k in knots), float(err.max()), float(np.sqrt(np.mean(err ** 2)))))
        if err.max() <= e_max:
            converged = True
            break
        if len(report) > max_rounds:
            break
        split_any = False
        new = []
        for d in range(3):
            U = knots[d]
            per, cnt = per_axis[d]
            n = len(U) - p - 1
            ins = []
            for s in range(len(per)):
                if per[s] > e_max and cnt[s] >= 2 * (p + 1) and n + len(ins) < max_ctrl[d]:
                    lo, hi = U[p + s], U[p + s + 1]
                    ins.append(0.5 * (lo + hi))
            if ins:
                split_any = True
                U = np.sort(np.concatenate([U, ins]))
            new.append(U)
        knots = new
        if not split_any:
            break
    return knots, c, {"rounds": report, "converged": converged}
