/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct fp64 CPU implementation of what the
 * MFA-DVR hot path computes (Sun, Lenz, Yu, Peterka, "MFA-DVR: direct volume
 * rendering of MFA models", arXiv 2204.11762; /root/reference/PAPER.md = "P:n").
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * leg may load this library.  It shares no code, header, table or constant
 * with the CUDA path (paper_2204_11762_b200/csrc); the only shared inputs are
 * the arrays drawn by paper_2204_11762_b200/workloads.py.
 *
 * Structure (each function cites what it follows):
 *   O1 orc_find_span     knot-span search
 *   O2 orc_basis_derivs  Cox-de Boor triangle + N'
 *   O3 orc_eval          plain UNFACTORED triple sum P:100, Alg.1 l.6,9
 *   O4 orc_ray           ray through pixel centre    P:100, Alg.1 l.4
 *   O5 orc_clip          slab clip to the volume     Alg.1 l.2-3
 *   O6-O13 march         Algorithm 1 lines 3-18
 *   O14 orc_render       rows/pixels split over threads (Alg.1 l.1)
 *   O15 ambiguity flags  DESIGN.md "readings" R-19
 *   H1 orc_basis_ders2   second derivatives of the basis (Piegl-Tiller eq. 2.9
 *                        applied twice)              P:78 "Higher-order derivatives,
 *                        up to the polynomial degree, are also analytically available"
 *   H2 orc_eval_hessian  value, gradient and the 6 second partials as plain
 *                        triple sums                 P:78; SURVEY §8(f) NEXT-4
 *   L1 (in march)        several directional lights, Phong summed per light
 *                        P:307 "multiple light sources can be added"; R-30
 *   C1 orc_curvatures    principal curvatures from gradient and Hessian, and
 *                        a curvature transfer function in march (P:100
 *                        "curvature-based transfer function"; R-31)
 *   G1 orc_field_eval    analytic ground truth (Eq. 1 Gaussian beam, Eq. 2
 *                        Marschner-Lobb) with analytic gradient
 *   G2 orc_render_ex     Algorithm 1 with value and/or gradient taken from the
 *                        analytic field ("ground truth volume rendering image by
 *                        computing the value and gradient analytically ... for the
 *                        samples on rays"; gradient-only test P:209)
 *
 * Readings where the paper is silent are listed in DESIGN.md §2 (R-1..R-21);
 * the ones used here are cited inline as "R-n".
 *
 * Parity status: every function is pinned by tests/test_oracle_*.py against
 * closed forms, brute-force recursion, polynomial reproduction, finite
 * differences and SPEC worked examples; see DESIGN.md §4.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_MAXP 8

typedef struct {
    int32_t degree[3];
    int64_t nctrl[3];
    const double* knots[3]; /* length nctrl[d] + degree[d] + 1 */
    const float* ctrl;      /* [n_w][n_v][n_u], u fastest (fp32 values, used exactly in fp64) */
    const double* ctrl64;   /* optional fp64 grid (same layout); used instead of ctrl when non-NULL */
} orc_model;

typedef struct {
    double eye[3], look_at[3], up[3];
    double fov_y_deg;          /* 0 -> orthographic */
    double ortho_half_height;
    int32_t width, height;
} orc_camera;

typedef struct {
    const float* rgba;         /* n_entries x 4, non-premultiplied */
    int32_t n_entries;
    double v_lo, v_hi;
} orc_tf;

typedef struct {
    double box_min[3], box_max[3];
    double step;               /* world units ("constant sample distance") */
    double o_max;              /* Alg.1 l.14 O_Max */
    int32_t shading;           /* Alg.1 l.8 ShadingOn */
    double ka, kd, ks, shininess;
    double grad_eps;           /* |g_phys| <= grad_eps -> ambient only (R-11) */
    double ert_window;         /* R-19 (i): |A - o_max| below this at a decision -> alternative */
    double exit_window;        /* R-19 (ii): L/step - 1/2 this close to an integer -> alternative */
    double sens_weight;        /* R-19 (iii): composited weight above ... */
    double sens_grad;          /*   ... with |g_phys| below this -> shading-sensitive flag */
    int32_t n_lights;          /* L1: 0 -> the headlight (R-11); else directional lights (R-30) */
    const double* light_dir;   /*   [n_lights][3] world directions towards each light */
    const double* light_intensity; /* [n_lights] */
    int32_t curv_n;            /* C1: 0 -> no curvature TF; else a curv_n x curv_n RGBA table */
    const float* curv_rgba;    /*   [curv_n (kappa_2)][curv_n (kappa_1)][4], over [-curv_range, curv_range]^2 */
    double curv_range;
} orc_params;

/* G1: analytic field (NEXT-2).  kind 1 = Gaussian beam (Eq. 1),  */
/* prm = {V_min, V_max, mu, sigma, R}; kind 2 = Marschner-Lobb (Eq. 2,        */
/* P:169-175), prm = {f_M, alpha}.  value_src / grad_src: 0 = MFA query,      */
/* 1 = analytic (the paper's value-only, gradient-only and overall tests,     */
/* P:193).                                                      */
typedef struct {
    int32_t kind;
    int32_t value_src, grad_src;
    double prm[6];
} orc_field;

#define ORC_FIELD_GB 1
#define ORC_FIELD_ML 2

/* ------------------------------------------------------------------------ */
/* O1: knot span.  i with U[i] <= u < U[i+1]; u == U[n] -> n-1 (SPEC S:45,   */
/* S:107; R-2).  Domain error (u outside [U[p],U[n]] or NaN) -> -1.          */
/* ------------------------------------------------------------------------ */
int64_t orc_find_span(int32_t p, int64_t n, const double* U, double u)
{
    if (!(u >= U[p] && u <= U[n])) return -1;   /* also catches NaN */
    if (u == U[n]) {
        int64_t i = n - 1;
        while (i > p && U[i] == U[n]) --i;         /* last non-degenerate span */
        return i;
    }
    int64_t lo = p, hi = n;                         /* invariant U[lo] <= u < U[hi] */
    while (hi - lo > 1) {
        int64_t mid = lo + (hi - lo) / 2;
        if (u < U[mid]) hi = mid; else lo = mid;
    }
    return lo;
}

/* ------------------------------------------------------------------------ */
/* O2: the p+1 non-zero basis functions N_{span-p+r,p}(u), r = 0..p, and     */
/* their first derivatives, by the Cox-de Boor triangle (P:74 tensor-product */
/* B-spline; "analytical ... derivatives").         */
/*   ndu[j][r] (j > r) = U[span+r+1] - U[span+1-j+r]   (knot differences)    */
/*   ndu[r][j] (r <= j) = N_{span-j+r, j}(u)                                  */
/*   N'_{i,p} = p N_{i,p-1}/(U_{i+p}-U_i) - p N_{i+1,p-1}/(U_{i+p+1}-U_{i+1}) */
/* ------------------------------------------------------------------------ */
void orc_basis_derivs(int32_t p, const double* U, int64_t span, double u, double* N, double* dN)
{
    double ndu[ORC_MAXP + 1][ORC_MAXP + 1];
    double left[ORC_MAXP + 1], right[ORC_MAXP + 1];
    ndu[0][0] = 1.0;
    for (int j = 1; j <= p; ++j) {
        left[j] = u - U[span + 1 - j];
        right[j] = U[span + j] - u;
        double saved = 0.0;
        for (int r = 0; r < j; ++r) {
            ndu[j][r] = right[r + 1] + left[j - r];
            double temp = ndu[r][j - 1] / ndu[j][r];
            ndu[r][j] = saved + right[r + 1] * temp;
            saved = left[j - r] * temp;
        }
        ndu[j][j] = saved;
    }
    for (int r = 0; r <= p; ++r) N[r] = ndu[r][p];
    if (!dN) return;
    for (int r = 0; r <= p; ++r) {
        double d = 0.0;
        if (p == 0) { dN[r] = 0.0; continue; }
        if (r >= 1) d += ndu[r - 1][p - 1] / ndu[p][r - 1];
        if (r <= p - 1) d -= ndu[r][p - 1] / ndu[p][r];
        dN[r] = p * d;
    }
}

/* ------------------------------------------------------------------------ */
/* H1: N, N' and N'' of the p+1 non-zero basis functions on span `span`.     */
/* The degree-q functions N_{i,q}(u), q <= p, come from the Cox-de Boor      */
/* triangle (as in O2); the derivatives from the textbook recursion          */
/*   N^(k)_{i,q} = q ( N^(k-1)_{i,q-1} / (U_{i+q} - U_i)                     */
/*                    - N^(k-1)_{i+1,q-1} / (U_{i+q+1} - U_{i+1}) )          */
/* (Piegl & Tiller eq. 2.9) for k = 1, 2, with 0/0 := 0 at repeated knots.   */
/* ------------------------------------------------------------------------ */
typedef struct {
    double ndu[ORC_MAXP + 1][ORC_MAXP + 1];   /* ndu[r][q] = N_{span-q+r, q}(u), r <= q */
    const double* U;
    int64_t span;
} orc_tri;

static double tri_N(const orc_tri* T, int q, int64_t i)
{
    if (q < 0) return 0.0;
    const int64_t r = i - T->span + q;
    return (r >= 0 && r <= q) ? T->ndu[r][q] : 0.0;
}

static double tri_div(double a, double den) { return den != 0.0 ? a / den : 0.0; }

static double tri_dN(const orc_tri* T, int k, int q, int64_t i)   /* k-th derivative of N_{i,q} */
{
    if (k == 0) return tri_N(T, q, i);
    if (q == 0) return 0.0;
    const double* U = T->U;
    return q * (tri_div(tri_dN(T, k - 1, q - 1, i), U[i + q] - U[i]) -
                tri_div(tri_dN(T, k - 1, q - 1, i + 1), U[i + q + 1] - U[i + 1]));
}

void orc_basis_ders2(int32_t p, const double* U, int64_t span, double u, double* N, double* dN, double* d2N)
{
    orc_tri T;
    T.U = U;
    T.span = span;
    double left[ORC_MAXP + 1], right[ORC_MAXP + 1], kd[ORC_MAXP + 1][ORC_MAXP + 1];
    T.ndu[0][0] = 1.0;
    for (int j = 1; j <= p; ++j) {            /* the triangle of O2, values only */
        left[j] = u - U[span + 1 - j];
        right[j] = U[span + j] - u;
        double saved = 0.0;
        for (int r = 0; r < j; ++r) {
            kd[j][r] = right[r + 1] + left[j - r];
            double temp = T.ndu[r][j - 1] / kd[j][r];
            T.ndu[r][j] = saved + right[r + 1] * temp;
            saved = left[j - r] * temp;
        }
        T.ndu[j][j] = saved;
    }
    for (int r = 0; r <= p; ++r) {
        const int64_t i = span - p + r;
        N[r] = tri_N(&T, p, i);
        dN[r] = tri_dN(&T, 1, p, i);
        d2N[r] = tri_dN(&T, 2, p, i);
    }
}

/* ------------------------------------------------------------------------ */
/* O3: value and parameter-space gradient as the plain triple sum over the   */
/* active (p+1)^3 block (SPEC S:72 value, S:81 gradient "substituting        */
/* basis_derivs along one axis at a time"; P:100 all three derivatives).     */
/* Also returns the abs-scales sigma = sum |term| (R-5 tolerance scale).     */
/* out[0]=v, out[1..3]=dv/du,dv/dv,dv/dw.  Returns 0, or -1 on domain error. */
/* ------------------------------------------------------------------------ */
int orc_eval(const orc_model* m, double u, double v, double w, double out[4], double sigma[4])
{
    const double q[3] = {u, v, w};
    double N[3][ORC_MAXP + 1], dN[3][ORC_MAXP + 1];
    int64_t span[3];
    for (int d = 0; d < 3; ++d) {
        span[d] = orc_find_span(m->degree[d], m->nctrl[d], m->knots[d], q[d]);
        if (span[d] < 0) {
            for (int k = 0; k < 4; ++k) { out[k] = NAN; if (sigma) sigma[k] = NAN; }
            return -1;
        }
        orc_basis_derivs(m->degree[d], m->knots[d], span[d], q[d], N[d], dN[d]);
    }
    const int64_t nu = m->nctrl[0], nv = m->nctrl[1];
    const int pu = m->degree[0], pv = m->degree[1], pw = m->degree[2];
    double s[4] = {0, 0, 0, 0}, a[4] = {0, 0, 0, 0};
    for (int c = 0; c <= pw; ++c) {
        for (int b = 0; b <= pv; ++b) {
            for (int aa = 0; aa <= pu; ++aa) {
                int64_t i = span[0] - pu + aa, j = span[1] - pv + b, k = span[2] - pw + c;
                const int64_t idx = (k * nv + j) * nu + i;
                double P = m->ctrl64 ? m->ctrl64[idx] : (double)m->ctrl[idx];
                double t0 = N[0][aa] * N[1][b] * N[2][c] * P;
                double t1 = dN[0][aa] * N[1][b] * N[2][c] * P;
                double t2 = N[0][aa] * dN[1][b] * N[2][c] * P;
                double t3 = N[0][aa] * N[1][b] * dN[2][c] * P;
                s[0] += t0; s[1] += t1; s[2] += t2; s[3] += t3;
                a[0] += fabs(t0); a[1] += fabs(t1); a[2] += fabs(t2); a[3] += fabs(t3);
            }
        }
    }
    for (int k = 0; k < 4; ++k) { out[k] = s[k]; if (sigma) sigma[k] = a[k]; }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* H2: value, gradient and Hessian (parameter space) as plain triple sums:   */
/* out = {v, v_u, v_v, v_w, v_uu, v_vv, v_ww, v_uv, v_uw, v_vw}; each term   */
/* is the product of one basis factor per axis with the derivative orders    */
/* of that component.  sigma[k] = sum |term| (tolerance scale, R-5).         */
/* ------------------------------------------------------------------------ */
int orc_eval_hessian(const orc_model* m, double u, double v, double w, double out[10], double sigma[10])
{
    static const int ord[10][3] = {{0, 0, 0}, {1, 0, 0}, {0, 1, 0}, {0, 0, 1}, {2, 0, 0},
                                   {0, 2, 0}, {0, 0, 2}, {1, 1, 0}, {1, 0, 1}, {0, 1, 1}};
    const double q[3] = {u, v, w};
    double B[3][3][ORC_MAXP + 1];   /* B[axis][order][r] */
    int64_t span[3];
    for (int d = 0; d < 3; ++d) {
        span[d] = orc_find_span(m->degree[d], m->nctrl[d], m->knots[d], q[d]);
        if (span[d] < 0) {
            for (int k = 0; k < 10; ++k) { out[k] = NAN; if (sigma) sigma[k] = NAN; }
            return -1;
        }
        orc_basis_ders2(m->degree[d], m->knots[d], span[d], q[d], B[d][0], B[d][1], B[d][2]);
    }
    const int64_t nu = m->nctrl[0], nv = m->nctrl[1];
    const int pu = m->degree[0], pv = m->degree[1], pw = m->degree[2];
    double s[10] = {0}, a[10] = {0};
    for (int c = 0; c <= pw; ++c)
        for (int b = 0; b <= pv; ++b)
            for (int aa = 0; aa <= pu; ++aa) {
                const int64_t i = span[0] - pu + aa, j = span[1] - pv + b, k = span[2] - pw + c;
                const int64_t idx = (k * nv + j) * nu + i;
                const double P = m->ctrl64 ? m->ctrl64[idx] : (double)m->ctrl[idx];
                for (int o = 0; o < 10; ++o) {
                    const double t = B[0][ord[o][0]][aa] * B[1][ord[o][1]][b] * B[2][ord[o][2]][c] * P;
                    s[o] += t;
                    a[o] += fabs(t);
                }
            }
    for (int k = 0; k < 10; ++k) { out[k] = s[k]; if (sigma) sigma[k] = a[k]; }
    return 0;
}

/* ------------------------------------------------------------------------ */
/* C1: principal curvatures of the isosurface through a point from the      */
/* physical gradient g and Hessian H (Kindlmann et al. 2003, the curvature-  */
/* based transfer functions P:100 names): n = -g/|g|, P = I - n n^T,         */
/* G = -P H P / |g|, T = trace G, F = |G|_F,                                 */
/* kappa_1,2 = (T +- sqrt(2 F^2 - T^2)) / 2.  |g| = 0 -> (0, 0) (R-31).       */
/* H is given as {h_xx, h_yy, h_zz, h_xy, h_xz, h_yz}.                        */
/* ------------------------------------------------------------------------ */
void orc_curvatures(const double g[3], const double h6[6], double k[2])
{
    const double gn = sqrt(g[0] * g[0] + g[1] * g[1] + g[2] * g[2]);
    if (!(gn > 0.0)) { k[0] = k[1] = 0.0; return; }
    const double H[3][3] = {{h6[0], h6[3], h6[4]}, {h6[3], h6[1], h6[5]}, {h6[4], h6[5], h6[2]}};
    double n[3], Pm[3][3], PH[3][3], G[3][3];
    for (int i = 0; i < 3; ++i) n[i] = -g[i] / gn;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) Pm[i][j] = (i == j ? 1.0 : 0.0) - n[i] * n[j];
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double acc = 0.0;
            for (int l = 0; l < 3; ++l) acc += Pm[i][l] * H[l][j];
            PH[i][j] = acc;
        }
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
            double acc = 0.0;
            for (int l = 0; l < 3; ++l) acc += PH[i][l] * Pm[l][j];
            G[i][j] = -acc / gn;
        }
    double T = G[0][0] + G[1][1] + G[2][2], F2 = 0.0;
    for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) F2 += G[i][j] * G[i][j];
    double disc = 2.0 * F2 - T * T;
    if (disc < 0.0) disc = 0.0;
    k[0] = 0.5 * (T + sqrt(disc));
    k[1] = 0.5 * (T - sqrt(disc));
}

/* C1: bilinear lookup of the curvature table at (kappa_1, kappa_2), clamped */
static void curv_lookup(const orc_params* P, const double k[2], double out[4])
{
    const int n = P->curv_n;
    double f[2];
    int i0[2];
    for (int d = 0; d < 2; ++d) {
        double x = (k[d] + P->curv_range) / (2.0 * P->curv_range) * (n - 1);
        if (x < 0.0) x = 0.0;
        if (x > n - 1) x = n - 1;
        i0[d] = (int)floor(x);
        if (i0[d] > n - 2) i0[d] = n - 2;
        f[d] = x - i0[d];
    }
    for (int c = 0; c < 4; ++c) {
        const float* T = P->curv_rgba;
        const double a00 = T[4 * (i0[1] * n + i0[0]) + c], a01 = T[4 * (i0[1] * n + i0[0] + 1) + c];
        const double a10 = T[4 * ((i0[1] + 1) * n + i0[0]) + c], a11 = T[4 * ((i0[1] + 1) * n + i0[0] + 1) + c];
        out[c] = (1.0 - f[1]) * ((1.0 - f[0]) * a00 + f[0] * a01) + f[1] * ((1.0 - f[0]) * a10 + f[0] * a11);
    }
}

/* ------------------------------------------------------------------------ */
/* G1: value and parameter-space gradient of the analytic field at the       */
/* parameter point (u,v,w) in [0,1]^3.  The functions are defined on         */
/* x, y, z in [-1, 1] ("The volume range of x, y, and z is [-1, 1]"),  */
/* so x = 2u - 1 and d/du = 2 d/dx (R-15, R-4).                               */
/* ------------------------------------------------------------------------ */
int orc_field_eval(const orc_field* f, double u, double v, double w, double out[4])
{
    const double x = 2.0 * u - 1.0, y = 2.0 * v - 1.0, z = 2.0 * w - 1.0;
    double F, gx, gy, gz;
    if (f->kind == ORC_FIELD_GB) {
        /* Eq. 1: F = V_min + (V_max - V_min) G(r / R), G(l) = exp(-(l - mu)^2 / (2 sigma^2)) */
        const double vmin = f->prm[0], vmax = f->prm[1], mu = f->prm[2], sg = f->prm[3], R = f->prm[4];
        const double r = sqrt(x * x + y * y + z * z);
        const double l = r / R;
        const double G = exp(-(l - mu) * (l - mu) / (2.0 * sg * sg));
        F = vmin + (vmax - vmin) * G;
        /* dF/dx_i = (V_max - V_min) G'(l) (1/R) x_i / r, G'(l) = -(l - mu)/sigma^2 G(l); 0 at r = 0 */
        const double c = r > 0.0 ? (vmax - vmin) * (-(l - mu) / (sg * sg)) * G / (R * r) : 0.0;
        gx = c * x;
        gy = c * y;
        gz = c * z;
    } else if (f->kind == ORC_FIELD_ML) {
        /* Eq. 2: F = (1 - sin(pi z / 2) + alpha (1 + rho(r))) / (2 (1 + alpha)),
           rho(r) = cos(2 pi f_M cos(pi r / 2)), r = sqrt(x^2 + y^2) */
        const double fm = f->prm[0], al = f->prm[1];
        const double PI = 3.14159265358979323846;
        const double r = sqrt(x * x + y * y);
        const double rho = cos(2.0 * PI * fm * cos(PI * r / 2.0));
        const double den = 2.0 * (1.0 + al);
        F = (1.0 - sin(PI * z / 2.0) + al * (1.0 + rho)) / den;
        /* rho'(r) = sin(2 pi f_M cos(pi r/2)) * 2 pi f_M * sin(pi r/2) * pi/2 */
        const double drho = sin(2.0 * PI * fm * cos(PI * r / 2.0)) * 2.0 * PI * fm * sin(PI * r / 2.0) * (PI / 2.0);
        const double c = r > 0.0 ? al * drho / (r * den) : 0.0;
        gx = c * x;
        gy = c * y;
        gz = -(PI / 2.0) * cos(PI * z / 2.0) / den;
    } else {
        return -1;
    }
    out[0] = F;
    out[1] = 2.0 * gx;
    out[2] = 2.0 * gy;
    out[3] = 2.0 * gz;
    return 0;
}

static void v_sub(const double* a, const double* b, double* r) { for (int i = 0; i < 3; ++i) r[i] = a[i] - b[i]; }
static void v_cross(const double* a, const double* b, double* r)
{
    r[0] = a[1] * b[2] - a[2] * b[1];
    r[1] = a[2] * b[0] - a[0] * b[2];
    r[2] = a[0] * b[1] - a[1] * b[0];
}
static double v_dot(const double* a, const double* b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
static void v_norm(double* a) { double l = sqrt(v_dot(a, a)); for (int i = 0; i < 3; ++i) a[i] /= l; }

/* ------------------------------------------------------------------------ */
/* O4: ray through the centre of pixel (px, py), row 0 at the top (P:100     */
/* "ray cast for each pixel of the viewport according to the relative        */
/* location of the camera and the viewport"; camera reading R-14).           */
/* ------------------------------------------------------------------------ */
void orc_ray(const orc_camera* cam, int32_t px, int32_t py, double o[3], double d[3])
{
    double f[3], r[3], up[3];
    v_sub(cam->look_at, cam->eye, f);
    v_norm(f);
    v_cross(f, cam->up, r);
    v_norm(r);
    v_cross(r, f, up);
    const double X = 2.0 * (px + 0.5) / cam->width - 1.0;
    const double Y = 1.0 - 2.0 * (py + 0.5) / cam->height;
    const double aspect = (double)cam->width / (double)cam->height;
    if (cam->fov_y_deg > 0.0) {
        const double th = tan(0.5 * cam->fov_y_deg * M_PI / 180.0);
        for (int i = 0; i < 3; ++i) {
            o[i] = cam->eye[i];
            d[i] = f[i] + X * aspect * th * r[i] + Y * th * up[i];
        }
        v_norm(d);
    } else {
        const double h = cam->ortho_half_height;
        for (int i = 0; i < 3; ++i) {
            o[i] = cam->eye[i] + X * aspect * h * r[i] + Y * h * up[i];
            d[i] = f[i];
        }
    }
}

/* ------------------------------------------------------------------------ */
/* O5: slab clip (Alg.1 l.3 Sample_First..Sample_Last "inside the volume",  */
/* P:131).  Returns 0 on a miss.  d_i == 0 handled           */
/* explicitly (inside the slab -> unbounded, outside -> miss).               */
/* ------------------------------------------------------------------------ */
int orc_clip(const double* bmin, const double* bmax, const double o[3], const double d[3],
             double* t_in, double* t_out)
{
    double tn = -INFINITY, tf = INFINITY;
    for (int i = 0; i < 3; ++i) {
        if (d[i] == 0.0) {
            if (o[i] < bmin[i] || o[i] > bmax[i]) return 0;
            continue;
        }
        double t0 = (bmin[i] - o[i]) / d[i], t1 = (bmax[i] - o[i]) / d[i];
        double lo = t0 < t1 ? t0 : t1, hi = t0 < t1 ? t1 : t0;
        if (lo > tn) tn = lo;
        if (hi < tf) tf = hi;
    }
    double a = tn > 0.0 ? tn : 0.0;
    if (!(tf > a)) return 0;
    *t_in = a;
    *t_out = tf;
    return 1;
}

/* O6 (R-7): K = #{k >= 0 : (k + 1/2) * step < t_out - t_in} = ceil(L/step - 1/2). */
static int64_t n_samples(double L, double step)
{
    double f = L / step - 0.5;
    return f > 0.0 ? (int64_t)ceil(f) : 0;
}

/* O9 applyTFs (Alg.1 l.7): linear interpolation in the table over  */
/* [v_lo, v_hi], clamped (R-9).                                              */
static void apply_tf(const orc_tf* tf, double v, double rgba[4])
{
    double s = (v - tf->v_lo) / (tf->v_hi - tf->v_lo);
    if (s < 0.0) s = 0.0;
    if (s > 1.0) s = 1.0;
    const int n = tf->n_entries;
    double f = s * (n - 1);
    int i0 = (int)floor(f);
    if (i0 > n - 2) i0 = n - 2;
    double w = f - i0;
    for (int c = 0; c < 4; ++c)
        rgba[c] = (1.0 - w) * (double)tf->rgba[4 * i0 + c] + w * (double)tf->rgba[4 * (i0 + 1) + c];
}

typedef struct {
    const orc_model* m;
    const orc_tf* tf;
    const orc_params* prm;
    double L[3];
    const orc_field* fld;   /* NULL: every value and gradient from the MFA query */
} orc_ctx;

/* Result of marching one ray. */
typedef struct {
    double C[3], A;
    int64_t count;
    int near_k;          /* first step whose ERT decision fell in the window, or -1 */
    int shade_sensitive;
} march_out;

/* O6-O13: Algorithm 1 lines 3-17 for one ray, samples k = 0..K-1.          */
/* flip_k >= 0 inverts the ERT decision at that step (R-19 alternative).     */
static void march(const orc_ctx* cx, const double o[3], const double d[3], double t_in, int64_t K,
                  int64_t flip_k, march_out* r)
{
    const orc_params* P = cx->prm;
    r->C[0] = r->C[1] = r->C[2] = 0.0;
    r->A = 0.0;
    r->count = 0;
    r->near_k = -1;
    r->shade_sensitive = 0;
    for (int64_t k = 0; k < K; ++k) {                       /* l.3 */
        const double t = t_in + (k + 0.5) * P->step;        /* l.4 getSampleLocation (R-7) */
        double q[3];
        for (int i = 0; i < 3; ++i) {                       /* l.5 normalizeSampleLocation (R-8) */
            double x = o[i] + t * d[i];
            double u = (x - P->box_min[i]) / cx->L[i];
            q[i] = u < 0.0 ? 0.0 : (u > 1.0 ? 1.0 : u);
        }
        double vg[4];
        const orc_field* fl = cx->fld;
        if (!(fl && fl->value_src && fl->grad_src))
            orc_eval(cx->m, q[0], q[1], q[2], vg, NULL);   /* l.6 queryValueMFA (+ l.9 gradient) */
        if (fl && (fl->value_src || fl->grad_src)) {        /* G2: analytic ground truth */
            double a[4];
            orc_field_eval(fl, q[0], q[1], q[2], a);
            if (fl->value_src) vg[0] = a[0];
            if (fl->grad_src) { vg[1] = a[1]; vg[2] = a[2]; vg[3] = a[3]; }
        }
        double col[4];
        apply_tf(cx->tf, vg[0], col);                        /* l.7 applyTFs */
        if (P->curv_n > 0) {                                 /* C1: curvature TF modulates colour and opacity */
            double hv[10], g[3], h[6], k[2], ct[4];
            orc_eval_hessian(cx->m, q[0], q[1], q[2], hv, NULL);
            for (int i = 0; i < 3; ++i) g[i] = hv[1 + i] / cx->L[i];
            h[0] = hv[4] / (cx->L[0] * cx->L[0]);
            h[1] = hv[5] / (cx->L[1] * cx->L[1]);
            h[2] = hv[6] / (cx->L[2] * cx->L[2]);
            h[3] = hv[7] / (cx->L[0] * cx->L[1]);
            h[4] = hv[8] / (cx->L[0] * cx->L[2]);
            h[5] = hv[9] / (cx->L[1] * cx->L[2]);
            const double gn = sqrt(v_dot(g, g));
            if (gn <= P->grad_eps) g[0] = g[1] = g[2] = 0.0;   /* zero gradient: no isosurface (R-31) */
            orc_curvatures(g, h, k);
            curv_lookup(P, k, ct);
            for (int i = 0; i < 4; ++i) col[i] *= ct[i];
        }
        double c[3] = {col[0], col[1], col[2]};
        const double a = col[3];
        double gnorm = 0.0;
        if (P->shading) {                                    /* l.8-11 */
            double g[3];
            for (int i = 0; i < 3; ++i) g[i] = vg[1 + i] / cx->L[i];   /* physical gradient (R-4) */
            gnorm = sqrt(v_dot(g, g));
            if (gnorm <= P->grad_eps) {                      /* zero gradient -> ambient (R-11) */
                for (int i = 0; i < 3; ++i) c[i] = P->ka * col[i];
            } else if (P->n_lights > 0) {                   /* L1: directional lights (R-30) */
                double N[3], V[3], dif = 0.0, spe = 0.0;
                for (int i = 0; i < 3; ++i) { N[i] = -g[i] / gnorm; V[i] = -d[i]; }
                for (int l = 0; l < P->n_lights; ++l) {
                    double L[3];
                    const double* Ld = P->light_dir + 3 * l;
                    const double len = sqrt(v_dot(Ld, Ld));
                    for (int i = 0; i < 3; ++i) L[i] = Ld[i] / len;
                    const double ndl = v_dot(N, L);
                    double R[3];                             /* reflection of L about N */
                    for (int i = 0; i < 3; ++i) R[i] = 2.0 * ndl * N[i] - L[i];
                    const double rv = v_dot(R, V);
                    dif += P->light_intensity[l] * (ndl > 0.0 ? ndl : 0.0);
                    if (ndl > 0.0) spe += P->light_intensity[l] * pow(rv > 0.0 ? rv : 0.0, P->shininess);
                }
                for (int i = 0; i < 3; ++i) {
                    double x = col[i] * (P->ka + P->kd * dif) + P->ks * spe;
                    c[i] = x < 0.0 ? 0.0 : (x > 1.0 ? 1.0 : x);
                }
            } else {
                /* headlight: light = view = -d; N = -g/|g|  (R-11) */
                const double ndl = v_dot(g, d) / gnorm;      /* N . (-d) */
                const double dif = ndl > 0.0 ? ndl : 0.0;    /* l.10 getLightingCoefficient */
                double spe = 0.0;
                if (ndl > 0.0) {
                    double rv = 2.0 * ndl * ndl - 1.0;       /* R . V with L = V */
                    spe = pow(rv > 0.0 ? rv : 0.0, P->shininess);
                }
                for (int i = 0; i < 3; ++i) {                /* l.11 addShading */
                    double x = col[i] * (P->ka + P->kd * dif) + P->ks * spe;
                    c[i] = x < 0.0 ? 0.0 : (x > 1.0 ? 1.0 : x);
                }
            }
        }
        const double wgt = (1.0 - r->A) * a;                 /* l.13 doColorCompositing */
        for (int i = 0; i < 3; ++i) r->C[i] += wgt * c[i];
        r->A += wgt;
        r->count += 1;
        if (P->shading && wgt > P->sens_weight && gnorm < P->sens_grad) r->shade_sensitive = 1;
        int stop = r->A > P->o_max;                          /* l.14 (R-13: strict, after compositing) */
        if (r->near_k < 0 && fabs(r->A - P->o_max) < P->ert_window) r->near_k = (int)k;
        if (k == flip_k) stop = !stop;
        if (stop) break;                                     /* l.15 */
    }
}

/* Per-pixel outputs: rgba (premultiplied, fp64), composited count, flags    */
/* (bit0 ERT window, bit1 exit window, bit2 shading-sensitive), and up to    */
/* two alternative outcomes (NaN when absent).                               */
#define ORC_FLAG_ERT 1
#define ORC_FLAG_EXIT 2
#define ORC_FLAG_SHADE 4

static void render_pixel(const orc_ctx* cx, const orc_camera* cam, int64_t pix, double* rgba,
                         int64_t* count, uint8_t* flags, double* alt, int64_t* alt_count)
{
    const int32_t px = (int32_t)(pix % cam->width), py = (int32_t)(pix / cam->width);
    double o[3], d[3], t_in, t_out;
    for (int j = 0; j < 8; ++j) alt[j] = NAN;
    alt_count[0] = alt_count[1] = -1;
    *flags = 0;
    orc_ray(cam, px, py, o, d);                              /* l.4 ray definition */
    if (!orc_clip(cx->prm->box_min, cx->prm->box_max, o, d, &t_in, &t_out)) {
        rgba[0] = rgba[1] = rgba[2] = rgba[3] = 0.0;         /* background (R-12) */
        *count = 0;
        return;
    }
    const double Ls = t_out - t_in;
    const int64_t K = n_samples(Ls, cx->prm->step);
    march_out r;
    march(cx, o, d, t_in, K, -1, &r);
    rgba[0] = r.C[0]; rgba[1] = r.C[1]; rgba[2] = r.C[2]; rgba[3] = r.A;   /* l.18 setPixelColor */
    *count = r.count;
    if (r.shade_sensitive) *flags |= ORC_FLAG_SHADE;
    if (r.near_k >= 0) {                                     /* R-19 (i) */
        march_out a;
        march(cx, o, d, t_in, K, r.near_k, &a);
        *flags |= ORC_FLAG_ERT;
        alt[0] = a.C[0]; alt[1] = a.C[1]; alt[2] = a.C[2]; alt[3] = a.A;
        alt_count[0] = a.count;
    }
    const double fr = Ls / cx->prm->step - 0.5;              /* R-19 (ii) */
    const double m = floor(fr + 0.5);
    if (fr > -0.5 && fabs(fr - m) < cx->prm->exit_window) {
        int64_t K2 = (K == (int64_t)m) ? K + 1 : K - 1;
        if (K2 < 0) K2 = 0;
        march_out a;
        march(cx, o, d, t_in, K2, -1, &a);
        *flags |= ORC_FLAG_EXIT;
        alt[4] = a.C[0]; alt[5] = a.C[1]; alt[6] = a.C[2]; alt[7] = a.A;
        alt_count[1] = a.count;
    }
}

/* ------------------------------------------------------------------------ */
/* O14: pixels split into contiguous blocks over threads (Alg.1 l.1 "rows    */
/* per thread").  Output is independent of the thread count.  */
/* pix == NULL renders every pixel in raster order (then blocks = rows).     */
/* ------------------------------------------------------------------------ */
typedef struct {
    const orc_ctx* cx;
    const orc_camera* cam;
    const int64_t* pix;
    int64_t begin, end;
    double* rgba;
    int64_t* count;
    uint8_t* flags;
    double* alt;
    int64_t* alt_count;
} render_job;

static void* render_worker(void* arg)
{
    render_job* j = (render_job*)arg;
    for (int64_t i = j->begin; i < j->end; ++i) {
        int64_t p = j->pix ? j->pix[i] : i;
        render_pixel(j->cx, j->cam, p, j->rgba + 4 * i, j->count + i, j->flags + i, j->alt + 8 * i,
                     j->alt_count + 2 * i);
    }
    return NULL;
}

int orc_render_ex(const orc_model* m, const orc_camera* cam, const orc_tf* tf, const orc_params* prm,
                  const orc_field* fld, int64_t npix, const int64_t* pix, double* rgba, int64_t* count,
                  uint8_t* flags, double* alt, int64_t* alt_count, int32_t nthreads)
{
    orc_ctx cx = {m, tf, prm, {0, 0, 0}, fld};
    for (int i = 0; i < 3; ++i) cx.L[i] = prm->box_max[i] - prm->box_min[i];
    if (nthreads < 1) nthreads = 1;
    if (npix < nthreads) nthreads = npix > 0 ? (int32_t)npix : 1;
    render_job* jobs = (render_job*)calloc((size_t)nthreads, sizeof(render_job));
    pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
    const int64_t W = cam->width;
    for (int t = 0; t < nthreads; ++t) {
        int64_t b, e;
        if (!pix) { /* whole rows per thread */
            int64_t rows = npix / W;
            b = (rows * t / nthreads) * W;
            e = (rows * (t + 1) / nthreads) * W;
            if (t == nthreads - 1) e = npix;
        } else {
            b = npix * t / nthreads;
            e = npix * (t + 1) / nthreads;
        }
        jobs[t] = (render_job){&cx, cam, pix, b, e, rgba, count, flags, alt, alt_count};
        pthread_create(&th[t], NULL, render_worker, &jobs[t]);
    }
    for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
    free(jobs);
    free(th);
    return 0;
}

int orc_render(const orc_model* m, const orc_camera* cam, const orc_tf* tf, const orc_params* prm,
               int64_t npix, const int64_t* pix, double* rgba, int64_t* count, uint8_t* flags,
               double* alt, int64_t* alt_count, int32_t nthreads)
{
    return orc_render_ex(m, cam, tf, prm, NULL, npix, pix, rgba, count, flags, alt, alt_count, nthreads);
}

/* Batched point evaluation (fp32 inputs used exactly).  Domain errors give  */
/* NaN rows; returns the number of domain errors.                             */
typedef struct {
    const orc_model* m;
    const float *u, *v, *w;
    double *out, *sig;
    int64_t begin, end, errors;
} eval_job;

static void* eval_worker(void* arg)
{
    eval_job* j = (eval_job*)arg;
    for (int64_t i = j->begin; i < j->end; ++i)
        if (orc_eval(j->m, j->u[i], j->v[i], j->w[i], j->out + 4 * i, j->sig ? j->sig + 4 * i : NULL) < 0)
            j->errors++;
    return NULL;
}

int64_t orc_eval_batch(const orc_model* m, int64_t n, const float* u, const float* v, const float* w,
                       double* out4, double* sigma4, int32_t nthreads)
{
    if (nthreads < 1) nthreads = 1;
    if (n < nthreads) nthreads = n > 0 ? (int32_t)n : 1;
    eval_job* jobs = (eval_job*)calloc((size_t)nthreads, sizeof(eval_job));
    pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = (eval_job){m, u, v, w, out4, sigma4, n * t / nthreads, n * (t + 1) / nthreads, 0};
        pthread_create(&th[t], NULL, eval_worker, &jobs[t]);
    }
    int64_t errs = 0;
    for (int t = 0; t < nthreads; ++t) { pthread_join(th[t], NULL); errs += jobs[t].errors; }
    free(jobs);
    free(th);
    return errs;
}

/* Batched H2 over threads (fp32 inputs used exactly); domain errors -> NaN rows. */
typedef struct {
    const orc_model* m;
    const float *u, *v, *w;
    double *out, *sig;
    int64_t begin, end, errors;
} hess_job;

static void* hess_worker(void* arg)
{
    hess_job* j = (hess_job*)arg;
    for (int64_t i = j->begin; i < j->end; ++i)
        if (orc_eval_hessian(j->m, j->u[i], j->v[i], j->w[i], j->out + 10 * i, j->sig ? j->sig + 10 * i : NULL) < 0)
            j->errors++;
    return NULL;
}

int64_t orc_eval_hessian_batch(const orc_model* m, int64_t n, const float* u, const float* v, const float* w,
                               double* out10, double* sigma10, int32_t nthreads)
{
    if (nthreads < 1) nthreads = 1;
    if (n < nthreads) nthreads = n > 0 ? (int32_t)n : 1;
    hess_job* jobs = (hess_job*)calloc((size_t)nthreads, sizeof(hess_job));
    pthread_t* th = (pthread_t*)calloc((size_t)nthreads, sizeof(pthread_t));
    for (int t = 0; t < nthreads; ++t) {
        jobs[t] = (hess_job){m, u, v, w, out10, sigma10, n * t / nthreads, n * (t + 1) / nthreads, 0};
        pthread_create(&th[t], NULL, hess_worker, &jobs[t]);
    }
    int64_t errs = 0;
    for (int t = 0; t < nthreads; ++t) { pthread_join(th[t], NULL); errs += jobs[t].errors; }
    free(jobs);
    free(th);
    return errs;
}
