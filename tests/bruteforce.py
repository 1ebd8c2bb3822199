"""Tier-1 brute force (pure Python, tiny inputs only): the recursive Cox-de Boor
DEFINITION of every B-spline basis function, independent of the oracle's
triangle algorithm.  Used only to pin oracle/ (never the CUDA path).

N_{i,0}(u) = 1 if U[i] <= u < U[i+1] else 0   (with the right end u = U[n]
            assigned to the last non-degenerate span)
N_{i,p}(u) = (u-U[i])/(U[i+p]-U[i]) N_{i,p-1}(u)
           + (U[i+p+1]-u)/(U[i+p+1]-U[i+1]) N_{i+1,p-1}(u),   0/0 := 0
N'_{i,p}   = p/(U[i+p]-U[i]) N_{i,p-1} - p/(U[i+p+1]-U[i+1]) N_{i+1,p-1}
"""
from __future__ import annotations


def _n0(U, i, u, n):
    if U[i] <= u < U[i + 1]:
        return 1.0
    # right end: u == U[n] belongs to the last non-degenerate span
    if u == U[n]:
        last = n - 1
        while U[last] == U[n]:
            last -= 1
        return 1.0 if i == last else 0.0
    return 0.0


def N(U, i, p, u):
    return _N(U, i, p, u, len(U))


def _N(U, i, p, u, nk):
    # nk = len(U).  The right-end rule only needs the start of the trailing run
    # of knots equal to U[-1].
    if p == 0:
        # index of the last knot that equals U[-1] defines the end
        nend = nk - 1
        while nend > 0 and U[nend - 1] == U[nend]:
            nend -= 1
        return _n0(U, i, u, nend)
    a = 0.0
    d1 = U[i + p] - U[i]
    if d1 != 0.0:
        a += (u - U[i]) / d1 * _N(U, i, p - 1, u, nk)
    d2 = U[i + p + 1] - U[i + 1]
    if d2 != 0.0:
        a += (U[i + p + 1] - u) / d2 * _N(U, i + 1, p - 1, u, nk)
    return a


def dN(U, i, p, u):
    nk = len(U)
    if p == 0:
        return 0.0
    a = 0.0
    d1 = U[i + p] - U[i]
    if d1 != 0.0:
        a += p / d1 * _N(U, i, p - 1, u, nk)
    d2 = U[i + p + 1] - U[i + 1]
    if d2 != 0.0:
        a -= p / d2 * _N(U, i + 1, p - 1, u, nk)
    return a


def all_basis(U, p, u):
    """Values and derivatives of all n = len(U)-p-1 basis functions at u."""
    n = len(U) - p - 1
    return [_N(U, i, p, u, len(U)) for i in range(n)], [dN(U, i, p, u) for i in range(n)]


def eval_full(knots, p, ctrl, u, v, w):
    """Value and parameter-space gradient by summing over ALL n_u*n_v*n_w
    control points (no span search, no locality).  ctrl[k][j][i]."""
    Nu, dNu = all_basis(knots[0], p, u)
    Nv, dNv = all_basis(knots[1], p, v)
    Nw, dNw = all_basis(knots[2], p, w)
    val = gu = gv = gw = 0.0
    for k in range(len(Nw)):
        for j in range(len(Nv)):
            for i in range(len(Nu)):
                P = float(ctrl[k][j][i])
                val += Nu[i] * Nv[j] * Nw[k] * P
                gu += dNu[i] * Nv[j] * Nw[k] * P
                gv += Nu[i] * dNv[j] * Nw[k] * P
                gw += Nu[i] * Nv[j] * dNw[k] * P
    return val, gu, gv, gw
