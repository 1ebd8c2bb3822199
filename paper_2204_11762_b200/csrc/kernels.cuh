// Device building blocks of the hot path:
//   a4 span + local coordinate       (uniform: span units; non-uniform: knot tables)
//   a5 basis + first derivatives     (power basis per span; uniform interior spans
//                                     use FFMA2 pair-Horner on (c_m, c'_m) constants)
//   a6 neighbourhood gather          (bricked row quads: one aligned 16-byte load
//                                     per u-row, all rows at compile-time offsets)
//   a7 sum-factorised contraction    (x, then y, then z; paired FP32 FMAs, FFMA2)
//
// Bricked row-quad layout.  Entry (i, j, k) of the quad array
// holds (P[k][j][i], P[k][j][i+1], P[k][j][i+2], P[k][j][i+3]).  Entries are
// grouped in bricks covering 16x16x16 spans; a brick stores EU x EV x EW
// entries (EV = EW = 16 + p halo rows, EU = 16 (+1 for p = 4, +4 for p = 5))
// so every (p+1)^3 neighbourhood of a span triple lies in one brick and its
// (p+1)^2 rows sit at offsets c*EV*EU + b*EU known at compile time.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "mfa_internal.cuh"

namespace mfa {

// Per-axis arguments as seen by the kernels (passed by value in the launch).
struct AxisArgs {
    const float* coef;
    const float* invh;
    const float* kh;
    const float* kl;
    const long long* kfx;
    const int* bucket;
    const longlong4* srec;
    int nsp;
    int M;
    int mshift;      // 62 - log2(M): bucket of a 2^62 fixed-point coordinate
    int ic_lo, ic_hi;
    float S;
    int dshift;      // non-uniform render: (F - U_s) >> dshift fits 23 bits on every span
    float dscale;    // 2^(dshift - 62)
    unsigned dmagic; // bits of 2^(23 + dshift - 62): (d & 0x7fffff) | dmagic - dbias = d * 2^(dshift - 62) exactly
    float dbias;     // 2^(23 + dshift - 62)
    int multi;       // non-uniform render: 1 if one ray step can cross more than one span (set per launch)
    float gsc;       // non-uniform render: parameter -> physical gradient scale 1/L (set per launch)
};

__host__ inline AxisArgs make_axis_args(const AxisTables& A) {
    AxisArgs a;
    a.coef = A.coef;
    a.invh = A.invh;
    a.kh = A.kh;
    a.kl = A.kl;
    a.kfx = A.kfx;
    a.bucket = A.bucket;
    a.srec = A.srec;
    a.multi = 1;
    a.gsc = 1.f;
    a.nsp = A.nsp;
    a.M = A.M;
    int lg = 0;
    while ((1 << lg) < A.M) ++lg;
    a.mshift = kNonUniFracBits - lg;
    a.ic_lo = A.ic_lo;
    a.ic_hi = A.ic_hi;
    a.S = A.S;
    a.dshift = A.dshift;
    a.dscale = ldexpf(1.0f, A.dshift - kNonUniFracBits);
    a.dmagic = (unsigned)(0x4b000000 + ((A.dshift - kNonUniFracBits) << 23));
    a.dbias = ldexpf(1.0f, 23 + A.dshift - kNonUniFracBits);
    return a;
}

// ---------------------------------------------------------------------------
// brick geometry
// ---------------------------------------------------------------------------
template <int P>
struct Brick {
    static constexpr int B = kBrick;
    static constexpr int EU = B + (P == 4 ? 1 : (P == 5 ? 4 : 0));
    static constexpr int EV = B + P;
    static constexpr int EW = B + P;
    static constexpr int SIZE = EU * EV * EW;   // entries per brick
    static constexpr int F4 = quad_f4(P);       // float4 per entry (row pairs for p <= 3)
    static constexpr int ROW = EU * F4;         // float4 between rows b and b+1 of a slab
    static constexpr int SLAB = EV * EU * F4;   // float4 between slabs c and c+1
};

struct BrickGrid {
    int nbx, nby;          // bricks along u, v
    int64_t q_f4;          // size of the quad array in float4 (debug bounds checks)
};

// float4 offset of the neighbourhood origin (the entry of spans (su, sv, sw)).
template <int P>
__device__ __forceinline__ int64_t brick_entry(const BrickGrid& g, int su, int sv, int sw) {
    const int bx = su >> kBrickLog, by = sv >> kBrickLog, bz = sw >> kBrickLog;
    const int lu = su & (kBrick - 1), lv = sv & (kBrick - 1), lw = sw & (kBrick - 1);
    const int brick = (bz * g.nby + by) * g.nbx + bx;
    const int64_t e = (int64_t)brick * Brick<P>::SIZE + (lw * Brick<P>::EV + lv) * Brick<P>::EU + lu;
    MFA_DCHECK(su >= 0 && sv >= 0 && sw >= 0 && e >= 0 &&
               (e + P * Brick<P>::EV * Brick<P>::EU + P * Brick<P>::EU) * Brick<P>::F4 +
                       (P == 5 ? 5 : (P == 4 ? 2 : Brick<P>::F4)) <= g.q_f4);
    return e * Brick<P>::F4;
}

// ---------------------------------------------------------------------------
// Plain haloed bricks (kBricks, p <= 3; mfa_internal.cuh pbrick_*): the
// neighbourhood of span triple (su, sv, sw) starts at local (lu, lv, lw) =
// s & 15 of its brick; a row of p+1 values sits at float offset lu of a
// 16-byte-aligned row, so it is read as the two aligned float4 around it and
// shifted by o = lu & 3 with two levels of selects.
// ---------------------------------------------------------------------------
template <int P>
struct PBrick {
    static constexpr int EU = pbrick_eu(P);
    static constexpr int EV = pbrick_ev(P);
    static constexpr int SIZE = EU * EV * EV;   // floats per brick
};

struct PlainRef {
    int64_t base;   // float offset of the 16-byte-aligned start of row (0, 0)
    int o;          // shift of the first value inside it (0..3)
};

template <int P>
__device__ __forceinline__ PlainRef plain_entry(const BrickGrid& g, int su, int sv, int sw) {
    const int bx = su >> kBrickLog, by = sv >> kBrickLog, bz = sw >> kBrickLog;
    const int lu = su & (kBrick - 1), lv = sv & (kBrick - 1), lw = sw & (kBrick - 1);
    const int64_t brick = ((int64_t)bz * g.nby + by) * g.nbx + bx;
    const int64_t b = brick * PBrick<P>::SIZE + (lw * PBrick<P>::EV + lv) * PBrick<P>::EU + (lu & ~3);
    MFA_DCHECK(su >= 0 && sv >= 0 && sw >= 0 &&
               4 * (b + (P * PBrick<P>::EV + P) * PBrick<P>::EU + 8) <= 16 * g.q_f4);
    return PlainRef{b, lu & 3};
}

template <int P>
__device__ __forceinline__ void load_prow(const float* __restrict__ Qf, int64_t off, int o, float (&r)[P + 1]) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(Qf + off));
    const float4 c = __ldg(reinterpret_cast<const float4*>(Qf + off) + 1);
    const float x[8] = {a.x, a.y, a.z, a.w, c.x, c.y, c.z, c.w};
    float y[P + 2];
#pragma unroll
    for (int i = 0; i < P + 2; ++i) y[i] = (o & 2) ? x[i + 2] : x[i];
#pragma unroll
    for (int i = 0; i <= P; ++i) r[i] = (o & 1) ? y[i + 1] : y[i];
}

template <int P>
__device__ __forceinline__ void load_pslab(const float4* __restrict__ Q, const PlainRef& e, int c,
                                           float (&r)[P + 1][P + 1]) {
    const float* Qf = reinterpret_cast<const float*>(Q);
#pragma unroll
    for (int b = 0; b <= P; ++b) load_prow<P>(Qf, e.base + (c * PBrick<P>::EV + b) * PBrick<P>::EU, e.o, r[b]);
}

template <int P>
__device__ __forceinline__ void load_pblock(const float4* __restrict__ Q, const PlainRef& e,
                                            float (&nb)[P + 1][P + 1][P + 1]) {
#pragma unroll
    for (int c = 0; c <= P; ++c) load_pslab<P>(Q, e, c, nb[c]);
}

// ---------------------------------------------------------------------------
// a5: basis values and t-derivatives.
//
// Interior spans of a clamped uniform knot vector (spans p-1 .. S-p) all
// carry the same polynomials in the local coordinate t: the uniform B-spline
// basis of degree p, which depends on nothing but p.  UniformBasis<P> derives
// it at compile time from the Cox-de Boor recursion on the integer knots
// 0, 1, ..., 2p+1 (span [p, p+1]), so the Horner FMAs take their
// coefficients as immediates.  Other spans (the p-1 boundary spans at each end
// of a uniform axis, every span of a non-uniform axis) read their
// coefficients from the span table built by span_tables_kernel.
// Derivatives are with respect to t; the caller scales the contracted
// gradient by dt/du once per axis.
// ---------------------------------------------------------------------------
template <int P>
struct UniformBasis {
    double c[P + 1][P + 1];   // N_a(t) = sum_m c[a][m] t^m
};

template <int P>
constexpr UniformBasis<P> make_uniform_basis() {
    UniformBasis<P> ub{};
    double cur[P + 1][P + 1] = {};   // functions of the current level, coefficients of t^m
    cur[0][0] = 1.0;                 // N_{P,0} = 1 on [P, P+1)
    const int i = P;                 // span index; knots U_j = j, u = P + t
    for (int k = 1; k <= P; ++k) {
        double nxt[P + 1][P + 1] = {};
        for (int r = 0; r <= k; ++r) {
            const int j = i - k + r;
            if (r >= 1) {  // (u - U_j)/(U_{j+k} - U_j) N_{j,k-1}, old function r-1
                const double c0 = (double)(i - j) / k, c1 = 1.0 / k;
                for (int m = 0; m < k; ++m) {
                    nxt[r][m] += c0 * cur[r - 1][m];
                    nxt[r][m + 1] += c1 * cur[r - 1][m];
                }
            }
            if (r <= k - 1) {  // (U_{j+k+1} - u)/(U_{j+k+1} - U_{j+1}) N_{j+1,k-1}, old function r
                const double c0 = (double)(j + k + 1 - i) / k, c1 = -1.0 / k;
                for (int m = 0; m < k; ++m) {
                    nxt[r][m] += c0 * cur[r][m];
                    nxt[r][m + 1] += c1 * cur[r][m];
                }
            }
        }
        for (int r = 0; r <= P; ++r)
            for (int m = 0; m <= P; ++m) cur[r][m] = nxt[r][m];
    }
    for (int r = 0; r <= P; ++r)
        for (int m = 0; m <= P; ++m) ub.c[r][m] = cur[r][m];
    return ub;
}

// Interior uniform span: simultaneous value / t-derivative Horner with
// immediate coefficients (2P-1 FFMA per function).
template <int P, bool SWAP>
__device__ __forceinline__ void uniform_horner(float t, float2 (&B)[P + 1]) {
    constexpr UniformBasis<P> UB = make_uniform_basis<P>();
#pragma unroll
    for (int a = 0; a <= P; ++a) {
        float v = fmaf((float)UB.c[a][P], t, (float)UB.c[a][P - 1]);
        float d = fmaf((float)(P * UB.c[a][P]), t, (float)((P - 1) * UB.c[a][P - 1]));
        if (P == 1) d = (float)UB.c[a][1];
#pragma unroll
        for (int m = P - 2; m >= 0; --m) {
            v = fmaf(v, t, (float)UB.c[a][m]);
            if (m >= 1) d = fmaf(d, t, (float)(m * UB.c[a][m]));
        }
        B[a] = SWAP ? make_float2(d, v) : make_float2(v, d);
    }
}

template <int P>
__device__ __forceinline__ void uniform_horner_value(float t, float (&N)[P + 1]) {
    constexpr UniformBasis<P> UB = make_uniform_basis<P>();
#pragma unroll
    for (int a = 0; a <= P; ++a) {
        float v = fmaf((float)UB.c[a][P], t, (float)UB.c[a][P - 1]);
#pragma unroll
        for (int m = P - 2; m >= 0; --m) v = fmaf(v, t, (float)UB.c[a][m]);
        N[a] = v;
    }
}

__device__ __forceinline__ void ldg256(const float* p, float (&r)[8]);

template <int P, bool SWAP>
__device__ __forceinline__ void table_horner(const float* __restrict__ coef, int s, float t, float2 (&B)[P + 1]) {
    MFA_DCHECK(s >= 0);
    float c[rec_floats(P)];
    if constexpr (rec_floats(P) % 8 == 0) {   // p = 3: the 64-byte record as two sector loads
#pragma unroll
        for (int q = 0; q < rec_floats(P) / 8; ++q) {
            float x[8];
            ldg256(coef + (int64_t)s * rec_floats(P) + 8 * q, x);
#pragma unroll
            for (int e = 0; e < 8; ++e) c[8 * q + e] = x[e];
        }
    } else {
        const float4* r = reinterpret_cast<const float4*>(coef + (int64_t)s * rec_floats(P));
#pragma unroll
        for (int q = 0; q < rec_floats(P) / 4; ++q) {
            const float4 x = __ldg(r + q);
            c[4 * q + 0] = x.x;
            c[4 * q + 1] = x.y;
            c[4 * q + 2] = x.z;
            c[4 * q + 3] = x.w;
        }
    }
#pragma unroll
    for (int a = 0; a <= P; ++a) {
        float d = c[a * (P + 1) + P];
        float v = fmaf(d, t, c[a * (P + 1) + P - 1]);
#pragma unroll
        for (int m = P - 2; m >= 0; --m) {
            d = fmaf(d, t, v);
            v = fmaf(v, t, c[a * (P + 1) + m]);
        }
        B[a] = SWAP ? make_float2(d, v) : make_float2(v, d);
    }
}

template <int P, bool SWAP>
__device__ __forceinline__ void axis_basis(const AxisArgs& A, bool uniform, int s, float t, float2 (&B)[P + 1]) {
    if (uniform && s >= A.ic_lo && s <= A.ic_hi)
        uniform_horner<P, SWAP>(t, B);
    else
        table_horner<P, SWAP>(A.coef, s, t, B);
}

// Values only (ShadingOn == false, Alg.1 l.8).
template <int P>
__device__ __forceinline__ void axis_basis_value(const AxisArgs& A, bool uniform, int s, float t, float (&N)[P + 1]) {
    if (uniform && s >= A.ic_lo && s <= A.ic_hi) {
        uniform_horner_value<P>(t, N);
    } else {
        float c[rec_floats(P)];
        const float4* r = reinterpret_cast<const float4*>(A.coef + (int64_t)s * rec_floats(P));
#pragma unroll
        for (int q = 0; q < rec_floats(P) / 4; ++q) {
            const float4 x = __ldg(r + q);
            c[4 * q + 0] = x.x;
            c[4 * q + 1] = x.y;
            c[4 * q + 2] = x.z;
            c[4 * q + 3] = x.w;
        }
#pragma unroll
        for (int a = 0; a <= P; ++a) {
            float v = fmaf(c[a * (P + 1) + P], t, c[a * (P + 1) + P - 1]);
#pragma unroll
            for (int m = P - 2; m >= 0; --m) v = fmaf(v, t, c[a * (P + 1) + m]);
            N[a] = v;
        }
    }
}

// ---------------------------------------------------------------------------
// a4 (uniform axis, render): span-unit fixed point F = X * 2^40.
// s = floor(X), t = frac(X) with 23 exact fraction bits; clamped to [0, S].
// ---------------------------------------------------------------------------
__device__ __forceinline__ void uni_span_fx(long long F, int S, int& s, float& t) {
    const int hi = (int)(F >> 32);
    const unsigned lo = (unsigned)(F & 0xffffffffLL);
    s = hi >> (kUniFracBits - 32);
    const unsigned fb = __funnelshift_r(lo, (unsigned)hi, kUniFracBits - 23) & 0x7fffffu;
    t = __uint_as_float(0x3f800000u | fb) - 1.0f;
    if (s < 0) { s = 0; t = 0.f; }
    if (s >= S) { s = S - 1; t = 1.f; }
}

// a4 (uniform axis, eval): x = u*S as an exact hi + lo pair (FMA residual).
__device__ __forceinline__ void uni_span_f32(float u, float Sf, int S, int& s, float& t) {
    const float hi = u * Sf;
    const float lo = fmaf(u, Sf, -hi);
    const float fl = floorf(hi);
    s = (int)fl;
    t = (hi - fl) + lo;
    if (s >= S) { s = S - 1; t += 1.f; }   // u == 1
    if (s < 0) { s = 0; }
}

// a4 (non-uniform axis, eval): bucket + forward scan, t = ((u - kh) - kl) / h.
__device__ __forceinline__ void nonuni_span_f32(const AxisArgs& A, float u, int& s, float& t, float& invh) {
    int b = (int)(u * (float)A.M);
    b = min(max(b, 0), A.M - 1);
    s = __ldg(A.bucket + b);
    while (s + 1 < A.nsp && u >= __ldg(A.kh + s + 1)) ++s;
    invh = __ldg(A.invh + s);
    t = ((u - __ldg(A.kh + s)) - __ldg(A.kl + s)) * invh;
}

// a4 (non-uniform axis, render): u in 2^62 fixed point.  The current span's
// bounds [lo, hi) and scales stay in registers; only when the sample leaves
// them (spans are monotone along a ray) is the knot table read.  The offset
// F - lo (< h * 2^62) is shifted to < 2^23 and converted exactly with the
// 2^23 magic number, so t costs no int64 -> float conversion.
#ifndef MFA_GSV   // 1: the gradient scale (1/h) * gsc folded into the span state at each crossing
#define MFA_GSV 0
#endif

#ifndef MFA_NU_TMAGIC   // 1: the t scale folded into the magic-number exponent (no per-span tsc)
#define MFA_NU_TMAGIC (MFA_SPAN_REC16 && !MFA_GSV)
#endif
static_assert(!MFA_NU_TMAGIC || (MFA_NU_SHIFTCMP && MFA_SPAN_REC16 && !MFA_GSV), "MFA_NU_TMAGIC: shifted offsets, 16-byte records");
struct NUAxis {
    long long lo;       // left knot of span s (2^62 fixed point)
#if MFA_NU_SHIFTCMP
    int wsh;            // ceil(width / 2^dshift): forward crossing iff (F - lo) >> dshift >= wsh
#else
    long long hi;       // right knot of span s
#endif
#if !MFA_NU_TMAGIC
    float tsc;          // 2^(dshift-62) / h_s
#endif
#if MFA_GSV
    float gsv;          // (1 / h_s) * gsc: the span's t -> physical gradient scale (set at each crossing)
#else
    float invh;         // 1 / h_s
#endif
    int s;
};

#ifndef MFA_SPAN_REC
#define MFA_SPAN_REC 1
#endif

#ifndef MFA_NU_SPLIT
#define MFA_NU_SPLIT 1
#endif

__device__ __forceinline__ void nu_load(const AxisArgs& A, NUAxis& st) {
    MFA_DCHECK(st.s >= 0 && st.s < A.nsp);
#if MFA_SPAN_REC && MFA_SPAN_REC16
    // one 16-byte record {lo, wsh | bits(1/h) << 32} (model.cu span_rec_kernel);
    // tsc = (1/h) * 2^(dshift-62) is an exact power-of-two scaling of 1/h
    long long r0, r1;
    asm("ld.global.nc.v2.s64 {%0,%1}, [%2];" : "=l"(r0), "=l"(r1)
        : "l"(reinterpret_cast<const longlong2*>(A.srec) + st.s));
    st.lo = r0;
    st.wsh = (int)(unsigned)r1;
    const float ih = __int_as_float((int)(r1 >> 32));
#if MFA_GSV
    st.gsv = ih * A.gsc;
#else
    st.invh = ih;
#endif
#if !MFA_NU_TMAGIC
    st.tsc = ih * A.dscale;
#endif
#elif MFA_SPAN_REC
    // one 32-byte record: {lo, hi, bits(1/h), bits(tsc)} (model.cu span_rec_kernel)
    long long r0, r1, r2, r3;
    asm("ld.global.nc.v4.s64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(r0), "=l"(r1), "=l"(r2), "=l"(r3)
                 : "l"(A.srec + st.s));
    st.lo = r0;
#if MFA_NU_SHIFTCMP
    st.wsh = (int)r1;
#else
    st.hi = r1;
#endif
#if MFA_GSV
    st.gsv = __int_as_float((int)r2) * A.gsc;
#else
    st.invh = __int_as_float((int)r2);
#endif
    st.tsc = __int_as_float((int)r3);
#else
    static_assert(!MFA_NU_SHIFTCMP, "MFA_NU_SHIFTCMP needs the span records");
    st.lo = __ldg(A.kfx + st.s);
    st.hi = (st.s + 1 < A.nsp) ? __ldg(A.kfx + st.s + 1) : 0x7fffffffffffffffLL;
    const float ih = __ldg(A.invh + st.s);
#if MFA_GSV
    st.gsv = ih * A.gsc;
#else
    st.invh = ih;
#endif
    st.tsc = ih * A.dscale;
#endif
}

__device__ __forceinline__ void nu_init(const AxisArgs& A, long long F, NUAxis& st) {
    F = max(F, 0LL);
    F = min(F, (1LL << kNonUniFracBits) - 1);
    int b = (int)(F >> A.mshift);
    b = min(max(b, 0), A.M - 1);
    int s = __ldg(A.bucket + b);
    while (s + 1 < A.nsp && F >= __ldg(A.kfx + s + 1)) ++s;
    st.s = s;
    nu_load(A, st);
}

#if !MFA_NU_SHIFTCMP
__device__ __forceinline__ float nu_span(const AxisArgs& A, long long F, NUAxis& st) {
    // F may leave [0, 2^62] by rounding at the entry/exit faces only; the span
    // index is kept in range and the local offset is clamped below instead of
    // clamping the 64-bit coordinate.
    const bool fwd = F >= st.hi;                 // hi of the last span is INT64_MAX
    const bool bwd = F < st.lo && st.s > 0;
    if (fwd || bwd) {
        // common case: the sample moved into the neighbouring span; the new
        // bounds and scale are three independent loads (one round trip)
        st.s += fwd ? 1 : -1;
        nu_load(A, st);
        if (F >= st.hi || (F < st.lo && st.s > 0)) {   // rare: crossed more than one span this step
            int s = st.s;
            while (s + 1 < A.nsp && F >= __ldg(A.kfx + s + 1)) ++s;
            while (s > 0 && F < __ldg(A.kfx + s)) --s;
            st.s = s;
            nu_load(A, st);
        }
    }
    int d = (int)((F - st.lo) >> A.dshift);     // < 2^23 inside the span
    d = min(max(d, 0), 8388607);
    const float fd = __int_as_float(0x4b000000 | d) - 8388608.0f;
    return fd * st.tsc;
}
#endif

// nu_span in two phases (MFA_NU_SPLIT, the render default): first every axis
// moves into its neighbouring span and issues the record load (predicated, no
// branch), then every axis consumes its record, so the crossings of the three
// axes wait for one load round trip instead of three (C5 +6 %).
__device__ __forceinline__ float nu_gscale(const AxisArgs& A, const NUAxis& st) {
#if MFA_GSV
    return st.gsv;
#else
    return st.invh * A.gsc;
#endif
}

#ifndef MFA_NU_UCMP   // 1: crossings in both directions by one unsigned compare (with MFA_NU_SHIFTCMP): C5 +1.6 %
#define MFA_NU_UCMP 1
#endif

// the span-local offset in units of 2^dshift (negative before the span)
__device__ __forceinline__ int nu_offset(const AxisArgs& A, long long F, const NUAxis& st) {
    return (int)((F - st.lo) >> A.dshift);
}

__device__ __forceinline__ void nu_cross(const AxisArgs& A, long long F, NUAxis& st) {
#if MFA_NU_SHIFTCMP && MFA_NU_UCMP
    // one unsigned compare catches both directions: d < 0 wraps above every
    // wsh (a backward crossing), d >= wsh is a forward one; the direction is
    // the sign of d; span 0 never steps below 0 (a negative d there is exit-face
    // rounding: the same record is reloaded and t clamps to 0)
    const int d = nu_offset(A, F, st);
    if ((unsigned)d >= (unsigned)st.wsh) {
        st.s = max(st.s + ((d >> 31) | 1), 0);
        nu_load(A, st);
    }
    return;
#elif MFA_NU_SHIFTCMP
    const int d = nu_offset(A, F, st);
    const bool fwd = d >= st.wsh;
    const bool bwd = d < 0 && st.s > 0;
#else
    const bool fwd = F >= st.hi;
    const bool bwd = F < st.lo && st.s > 0;
#endif
#if !(MFA_NU_SHIFTCMP && MFA_NU_UCMP)
    if (fwd || bwd) {
        st.s += fwd ? 1 : -1;
        nu_load(A, st);
    }
#endif
}

#if MFA_NU_SHIFTCMP && MFA_NU_UCMP
// nu_cross with the offset d = nu_offset(A, F, st) already computed (the
// render's early block load computes it one iteration ahead)
__device__ __forceinline__ void nu_cross_d(const AxisArgs& A, int d, NUAxis& st) {
    if ((unsigned)d >= (unsigned)st.wsh) {
        st.s = max(st.s + ((d >> 31) | 1), 0);
        nu_load(A, st);
    }
}
#endif

#if MFA_NU_SHIFTCMP && MFA_NU_UCMP && MFA_NU_TMAGIC
// The multi-span step in two pieces for the render's deferred fixup
// (MFA_MULTI_DEFER): nu_search moves st to the span that contains F by a
// search over the knots (needed only when a step crossed more than one span,
// i.e. (unsigned)nu_offset(F) >= wsh after nu_cross); nu_t converts the span
// offset d = nu_offset(A, F, st) to the local coordinate, exactly as nu_finish.
__device__ __forceinline__ void nu_search(const AxisArgs& A, long long F, NUAxis& st) {
    int s = st.s;
    while (s + 1 < A.nsp && F >= __ldg(A.kfx + s + 1)) ++s;
    while (s > 0 && F < __ldg(A.kfx + s)) --s;
    st.s = s;
    nu_load(A, st);
}

__device__ __forceinline__ float nu_t(const AxisArgs& A, int d, const NUAxis& st) {
    unsigned bits;
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(bits) : "r"(max(d, 0)), "r"(0x7fffff), "r"(A.dmagic));
    return (__uint_as_float(bits) - A.dbias) * st.invh;
}
#endif

template <bool MULTI = true>
__device__ __forceinline__ float nu_finish(const AxisArgs& A, long long F, NUAxis& st) {
    // rare: crossed more than one span this step; impossible when every span is
    // wider than the largest step (A.multi = 0; the render compiles a loop
    // without the check, MULTI = false, for launches where no axis needs it)
#if MFA_NU_SHIFTCMP
    int d = nu_offset(A, F, st);
#if MFA_NU_UCMP
    // (no A.multi test: on an axis whose spans are all wider than a step the
    // compare is simply never true)
    if (MULTI && (unsigned)d >= (unsigned)st.wsh) {
#else
    if (MULTI && A.multi && (d >= st.wsh || (d < 0 && st.s > 0))) {
#endif
        int s = st.s;
        while (s + 1 < A.nsp && F >= __ldg(A.kfx + s + 1)) ++s;
        while (s > 0 && F < __ldg(A.kfx + s)) --s;
        st.s = s;
        nu_load(A, st);
        d = nu_offset(A, F, st);
    }
#else
    if (MULTI && A.multi && (F >= st.hi || (F < st.lo && st.s > 0))) {
        int s = st.s;
        while (s + 1 < A.nsp && F >= __ldg(A.kfx + s + 1)) ++s;
        while (s > 0 && F < __ldg(A.kfx + s)) --s;
        st.s = s;
        nu_load(A, st);
    }
    int d = (int)((F - st.lo) >> A.dshift);
#endif
#if MFA_NU_SHIFTCMP
    // d < wsh <= 2^23 - 1 inside the span; negative only for exit-face rounding
    // on span 0; the mask keeps the exponent intact whatever happens
    unsigned bits;   // (max(d, 0) & 0x7fffff) | 0x4b000000 in one LOP3
#if MFA_NU_TMAGIC
    // the exponent of the magic number carries 2^(dshift - 62): fd = d * 2^(dshift - 62)
    // exactly, so t = fd * (1/h) rounds the same exact product as d * tsc did
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(bits) : "r"(max(d, 0)), "r"(0x7fffff), "r"(A.dmagic));
    const float fd = __uint_as_float(bits) - A.dbias;
    return fd * st.invh;
#else
    asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(bits) : "r"(max(d, 0)), "r"(0x7fffff), "r"(0x4b000000));
    const float fd = __uint_as_float(bits) - 8388608.0f;
#endif
#else
    d = min(max(d, 0), 8388607);
    const float fd = __int_as_float(0x4b000000 | d) - 8388608.0f;
#endif
#if !MFA_NU_TMAGIC
    return fd * st.tsc;
#endif
}

// ---------------------------------------------------------------------------
// Second derivatives (mfa_eval_hessian, and the curvature transfer function of
// the extended render): per axis (N, N', N'') by a three-output Horner scheme
// on power-basis coefficients, and the value / gradient / Hessian contraction
// of one slab.
// ---------------------------------------------------------------------------
// Bernstein polynomials in power form: B_j(t) = sum_m c[j][m] t^m,
// c[j][m] = C(P,j) C(P-j, m-j) (-1)^(m-j) for m >= j.
template <int P>
struct BernPower {
    double c[P + 1][P + 1];
};

template <int P>
constexpr BernPower<P> make_bern_power() {
    BernPower<P> b{};
    for (int j = 0; j <= P; ++j)
        for (int m = j; m <= P; ++m) {
            double cb = 1.0, cc = 1.0;
            for (int i = 1; i <= j; ++i) cb = cb * (P - j + i) / i;            // C(P, j)
            for (int i = 1; i <= m - j; ++i) cc = cc * (P - m + i) / i;        // C(P-j, m-j)
            b.c[j][m] = (((m - j) & 1) ? -1.0 : 1.0) * cb * cc;
        }
    return b;
}

// f, f', f'' of sum_m c[m] t^m (synthetic division: f''/2 accumulates in d2)
template <int P>
__device__ __forceinline__ void horner3(const float (&c)[P + 1], float t, float& f, float& d1, float& d2) {
    f = c[P];
    d1 = 0.f;
    d2 = 0.f;
#pragma unroll
    for (int m = P - 1; m >= 0; --m) {
        d2 = fmaf(d2, t, d1);
        d1 = fmaf(d1, t, f);
        f = fmaf(f, t, c[m]);
    }
    d2 *= 2.f;
}

template <int P, int LAYOUT, bool UNI>
__device__ __forceinline__ void basis3(const AxisArgs& A, int s, float t, float (&N)[P + 1], float (&D1)[P + 1],
                                       float (&D2)[P + 1]) {
    if constexpr (is_bez(LAYOUT)) {
        constexpr BernPower<P> BP = make_bern_power<P>();
#pragma unroll
        for (int a = 0; a <= P; ++a) {
            float c[P + 1];
#pragma unroll
            for (int m = 0; m <= P; ++m) c[m] = (float)BP.c[a][m];
            horner3<P>(c, t, N[a], D1[a], D2[a]);
        }
    } else {
        if (UNI && s >= A.ic_lo && s <= A.ic_hi) {
            constexpr UniformBasis<P> UB = make_uniform_basis<P>();
#pragma unroll
            for (int a = 0; a <= P; ++a) {
                float c[P + 1];
#pragma unroll
                for (int m = 0; m <= P; ++m) c[m] = (float)UB.c[a][m];
                horner3<P>(c, t, N[a], D1[a], D2[a]);
            }
        } else {
            const float* rec = A.coef + (int64_t)s * rec_floats(P);
#pragma unroll
            for (int a = 0; a <= P; ++a) {
                float c[P + 1];
#pragma unroll
                for (int m = 0; m <= P; ++m) c[m] = __ldg(rec + a * (P + 1) + m);
                horner3<P>(c, t, N[a], D1[a], D2[a]);
            }
        }
    }
}

// One slab c of the (value, gradient, Hessian) contraction (hessian.cu
// documents the 3 / 6 / 10 sum structure); out = {v, v_u, v_v, v_w, v_uu,
// v_vv, v_ww, v_uv, v_uw, v_vw} in t-space, accumulated.
template <int P>
__device__ __forceinline__ void contract_vgh_slab(const float (&r)[P + 1][P + 1], const float (&Nu)[P + 1],
                                                  const float (&Du)[P + 1], const float (&Eu)[P + 1],
                                                  const float (&Nv)[P + 1], const float (&Dv)[P + 1],
                                                  const float (&Ev)[P + 1], float nw, float dw, float ew,
                                                  float (&out)[10]) {
    float B[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int b = 0; b <= P; ++b) {
        float a0 = 0.f, a1 = 0.f, a2 = 0.f;
#pragma unroll
        for (int a = 0; a <= P; ++a) {
            a0 = fmaf(Nu[a], r[b][a], a0);
            a1 = fmaf(Du[a], r[b][a], a1);
            a2 = fmaf(Eu[a], r[b][a], a2);
        }
        B[0] = fmaf(Nv[b], a0, B[0]);
        B[1] = fmaf(Nv[b], a1, B[1]);
        B[2] = fmaf(Dv[b], a0, B[2]);
        B[3] = fmaf(Nv[b], a2, B[3]);
        B[4] = fmaf(Dv[b], a1, B[4]);
        B[5] = fmaf(Ev[b], a0, B[5]);
    }
    out[0] = fmaf(nw, B[0], out[0]);
    out[1] = fmaf(nw, B[1], out[1]);
    out[2] = fmaf(nw, B[2], out[2]);
    out[3] = fmaf(dw, B[0], out[3]);
    out[4] = fmaf(nw, B[3], out[4]);
    out[5] = fmaf(nw, B[5], out[5]);
    out[6] = fmaf(ew, B[0], out[6]);
    out[7] = fmaf(nw, B[4], out[7]);
    out[8] = fmaf(dw, B[1], out[8]);
    out[9] = fmaf(dw, B[2], out[9]);
}

// principal curvatures from a physical gradient g and Hessian h = {xx, yy, zz,
// xy, xz, yz} (Kindlmann et al. 2003; R-31): n = -g/|g|, P = I - n n^T,
// G = -P H P / |g|, kappa = (T +- sqrt(2|G|_F^2 - T^2)) / 2
__device__ __forceinline__ void curvatures(const float (&g)[3], const float (&h)[6], float& k1, float& k2) {
    const float g2 = fmaf(g[0], g[0], fmaf(g[1], g[1], g[2] * g[2]));
    const float inv = rsqrtf(fmaxf(g2, 1e-37f));
    const float n[3] = {-g[0] * inv, -g[1] * inv, -g[2] * inv};
    const float H[3][3] = {{h[0], h[3], h[4]}, {h[3], h[1], h[5]}, {h[4], h[5], h[2]}};
    float Pm[3][3], PH[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) Pm[i][j] = (i == j ? 1.f : 0.f) - n[i] * n[j];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) PH[i][j] = fmaf(Pm[i][0], H[0][j], fmaf(Pm[i][1], H[1][j], Pm[i][2] * H[2][j]));
    float T = 0.f, F2 = 0.f;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            const float Gij = -fmaf(PH[i][0], Pm[0][j], fmaf(PH[i][1], Pm[1][j], PH[i][2] * Pm[2][j])) * inv;
            if (i == j) T += Gij;
            F2 = fmaf(Gij, Gij, F2);
        }
    const float sd = sqrtf(fmaxf(fmaf(2.f, F2, -T * T), 0.f));
    k1 = 0.5f * (T + sd);
    k2 = 0.5f * (T - sd);
}

// ---------------------------------------------------------------------------
// a6: one slab c of the neighbourhood: rows b = 0..P, each P+1 u-values.
// ---------------------------------------------------------------------------
#ifndef MFA_LDG256
#define MFA_LDG256 1
#endif

// 32-byte vector load (sm_100: LDG.E.256): one full sector per lane
__device__ __forceinline__ void ldg256(const float* p, float (&r)[8]) {
    asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7])
                 : "l"(p));
}

template <int P>
__device__ __forceinline__ void load_slab(const float4* __restrict__ q, float (&r)[P + 1][P + 1]) {
    if constexpr (P <= 3) {   // row pairs: rows (0,1) and (2,3) are one 32-byte load each
#pragma unroll
        for (int b = 0; b <= P; b += 2) {
            float x[8];
            ldg256(reinterpret_cast<const float*>(q + b * Brick<P>::ROW), x);
#pragma unroll
            for (int a = 0; a <= P; ++a) {
                r[b][a] = x[a];
                if (b + 1 <= P) r[b + 1][a] = x[4 + a];
            }
        }
        return;
    }
    constexpr int EU = Brick<P>::EU;
#pragma unroll
    for (int b = 0; b <= P; ++b) {
        const float4* e = q + b * EU;
        if constexpr (P == 1) {
            const float2 x = __ldg(reinterpret_cast<const float2*>(e));
            r[b][0] = x.x; r[b][1] = x.y;
        } else if constexpr (P == 2) {
            const float4 x = __ldg(e);
            r[b][0] = x.x; r[b][1] = x.y; r[b][2] = x.z;
        } else if constexpr (P == 3) {
            const float4 x = __ldg(e);
            r[b][0] = x.x; r[b][1] = x.y; r[b][2] = x.z; r[b][3] = x.w;
        } else if constexpr (P == 4) {
            const float4 x = __ldg(e);
            r[b][0] = x.x; r[b][1] = x.y; r[b][2] = x.z; r[b][3] = x.w;
            r[b][4] = __ldg(reinterpret_cast<const float*>(e + 1) + 3);
        } else {
            const float4 x = __ldg(e);
            const float2 y = __ldg(reinterpret_cast<const float2*>(e + 4));
            r[b][0] = x.x; r[b][1] = x.y; r[b][2] = x.z; r[b][3] = x.w; r[b][4] = y.x; r[b][5] = y.y;
        }
    }
}

// ---------------------------------------------------------------------------
// a7: value + t-space gradient, sum-factorised ("all derivatives along
// the three dimensions at once"; "sum operations on each of the three
// dimensions").  Per row (c,b):
//   (a0, a1) = sum_a (Nu_a, Nu'_a) * P            [FFMA2, P broadcast]
//   B  += Nv_b a0 ; (Bv, Bu) += (Nv'_b, Nv_b) * (a0, a1)
// per slab c:  (v, g_w) += (Nw_c, Nw'_c) * B ;  (g_v, g_u) += Nw_c * (Bv, Bu)
// Bu: (N, N'), Bvs: (N', N) (swapped), Bw: (N, N').
// Slab c+1 is loaded while slab c is contracted; the caller has already
// issued slab 0 (so its latency overlaps the basis evaluation).
// ---------------------------------------------------------------------------
template <int P>
__device__ __forceinline__ void contract_slab(const float (&r)[P + 1][P + 1], const float2 (&Bu)[P + 1],
                                              const float2 (&Bvs)[P + 1], float2 wc, float2& vw, float2& gvu) {
    float B = 0.f;
    float2 Bvu = make_float2(0.f, 0.f);
#pragma unroll
    for (int b = 0; b <= P; ++b) {
        float2 a01 = __fmul2_rn(Bu[0], make_float2(r[b][0], r[b][0]));
#pragma unroll
        for (int a = 1; a <= P; ++a) a01 = __ffma2_rn(Bu[a], make_float2(r[b][a], r[b][a]), a01);
        B = fmaf(Bvs[b].y, a01.x, B);
        Bvu = __ffma2_rn(Bvs[b], a01, Bvu);
    }
    vw = __ffma2_rn(wc, make_float2(B, B), vw);
    gvu = __ffma2_rn(make_float2(wc.x, wc.x), Bvu, gvu);
}

template <int P>
__device__ __forceinline__ void contract_vg(const float4* __restrict__ q, float (&r0)[P + 1][P + 1],
                                            const float2 (&Bu)[P + 1], const float2 (&Bvs)[P + 1],
                                            const float2 (&Bw)[P + 1], float& val, float& gu, float& gv,
                                            float& gw) {
    constexpr int SW = Brick<P>::SLAB;
    float2 vw = make_float2(0.f, 0.f), gvu = make_float2(0.f, 0.f);
    float r1[P + 1][P + 1];
#pragma unroll
    for (int c = 0; c <= P; ++c) {
        if (c & 1) {
            if (c < P) load_slab<P>(q + (c + 1) * SW, r0);
            contract_slab<P>(r1, Bu, Bvs, Bw[c], vw, gvu);
        } else {
            if (c < P) load_slab<P>(q + (c + 1) * SW, r1);
            contract_slab<P>(r0, Bu, Bvs, Bw[c], vw, gvu);
        }
    }
    val = vw.x;
    gw = vw.y;
    gv = gvu.x;
    gu = gvu.y;
}

template <int P>
__device__ __forceinline__ float contract_v(const float4* __restrict__ q, float (&r0)[P + 1][P + 1],
                                            const float (&Nu)[P + 1], const float (&Nv)[P + 1],
                                            const float (&Nw)[P + 1]) {
    constexpr int SW = Brick<P>::SLAB;
    float val = 0.f;
    float r1[P + 1][P + 1];
#pragma unroll
    for (int c = 0; c <= P; ++c) {
        float (&r)[P + 1][P + 1] = (c & 1) ? r1 : r0;
        if (c < P) {
            if (c & 1) load_slab<P>(q + (c + 1) * SW, r0);
            else load_slab<P>(q + (c + 1) * SW, r1);
        }
        float B = 0.f;
#pragma unroll
        for (int b = 0; b <= P; ++b) {
            float a0 = Nu[0] * r[b][0];
#pragma unroll
            for (int a = 1; a <= P; ++a) a0 = fmaf(Nu[a], r[b][a], a0);
            B = fmaf(Nv[b], a0, B);
        }
        val = fmaf(Nw[c], B, val);
    }
    return val;
}

// ---------------------------------------------------------------------------
// a6/a7 with a per-lane neighbourhood cache (p <= 3): the (p+1)^3 control
// values stay in registers while consecutive samples of a ray share a span
// triple (about 57% of steps at 0.25 span per step); only lanes whose triple
// changed reload, which cuts L1 wavefronts.
// ---------------------------------------------------------------------------
template <int P>
__device__ __forceinline__ void load_block(const float4* __restrict__ q, float (&nb)[P + 1][P + 1][P + 1]) {
    constexpr int SW = Brick<P>::SLAB;
#pragma unroll
    for (int c = 0; c <= P; ++c) load_slab<P>(q + c * SW, nb[c]);
}

template <int P>
__device__ __forceinline__ void contract_vg_cached(const float (&nb)[P + 1][P + 1][P + 1], const float2 (&Bu)[P + 1],
                                                   const float2 (&Bvs)[P + 1], const float2 (&Bw)[P + 1],
                                                   float& val, float& gu, float& gv, float& gw) {
    float2 vw = make_float2(0.f, 0.f), gvu = make_float2(0.f, 0.f);
#pragma unroll
    for (int c = 0; c <= P; ++c) contract_slab<P>(nb[c], Bu, Bvs, Bw[c], vw, gvu);
    val = vw.x;
    gw = vw.y;
    gv = gvu.x;
    gu = gvu.y;
}

// value only, from the (value, derivative) basis pairs of the shaded path,
// with exactly contract_vg_cached's operation order for the value component
// (so the value -- and the TF opacity decided from it -- is bit-identical)
template <int P>
__device__ __forceinline__ float contract_v_pairs(const float (&nb)[P + 1][P + 1][P + 1], const float2 (&Bu)[P + 1],
                                                  const float2 (&Bvs)[P + 1], const float2 (&Bw)[P + 1]) {
    float val = 0.f;
#pragma unroll
    for (int c = 0; c <= P; ++c) {
        float B = 0.f;
#pragma unroll
        for (int b = 0; b <= P; ++b) {
            float a0 = __fmul_rn(Bu[0].x, nb[c][b][0]);
#pragma unroll
            for (int a = 1; a <= P; ++a) a0 = fmaf(Bu[a].x, nb[c][b][a], a0);
            B = fmaf(Bvs[b].y, a0, B);
        }
        val = fmaf(Bw[c].x, B, val);
    }
    return val;
}

template <int P>
__device__ __forceinline__ float contract_v_cached(const float (&nb)[P + 1][P + 1][P + 1], const float (&Nu)[P + 1],
                                                   const float (&Nv)[P + 1], const float (&Nw)[P + 1]) {
    float val = 0.f;
#pragma unroll
    for (int c = 0; c <= P; ++c) {
        float B = 0.f;
#pragma unroll
        for (int b = 0; b <= P; ++b) {
            float a0 = Nu[0] * nb[c][b][0];
#pragma unroll
            for (int a = 1; a <= P; ++a) a0 = fmaf(Nu[a], nb[c][b][a], a0);
            B = fmaf(Nv[b], a0, B);
        }
        val = fmaf(Nw[c], B, val);
    }
    return val;
}

// ---------------------------------------------------------------------------
// Bezier-block layout (non-uniform models, p <= 3): the spline on span triple
// (su, sv, sw) is sum_{jkl} B_j(t_u) B_k(t_v) B_l(t_w) Z[l][k][j] with the
// Bernstein polynomials B_j(t) = C(p,j) t^j (1-t)^(p-j), the same on every
// span, evaluated here in product form (all terms non-negative).
// ---------------------------------------------------------------------------
#ifndef MFA_BERN3
#define MFA_BERN3 1
#endif

__host__ __device__ constexpr float binomf(int n, int k) {
    float r = 1.f;
    for (int i = 1; i <= k; ++i) r = r * (float)(n - k + i) / (float)i;
    return r;
}

template <int P, bool SWAP>
__device__ __forceinline__ void bernstein(float t, float2 (&B)[P + 1]) {
#if MFA_BERN3
    if constexpr (P == 3) {   // cubic written out: 10 FP32 ops for values and derivatives
        const float s = 1.f - t;
        const float s2 = s * s, t2 = t * t, ts3 = 3.f * (t * s);
        const float d0 = -3.f * s2, d3 = 3.f * t2;
        const float v[4] = {s2 * s, ts3 * s, ts3 * t, t2 * t};
        const float d[4] = {d0, fmaf(ts3, -2.f, -d0), fmaf(ts3, 2.f, -d3), d3};
#pragma unroll
        for (int j = 0; j < 4; ++j) B[j] = SWAP ? make_float2(d[j], v[j]) : make_float2(v[j], d[j]);
        return;
    }
#endif
    const float s = 1.f - t;
    float tp[P + 1], sp[P + 1];
    tp[0] = 1.f;
    sp[0] = 1.f;
#pragma unroll
    for (int m = 1; m <= P; ++m) {
        tp[m] = tp[m - 1] * t;
        sp[m] = sp[m - 1] * s;
    }
    float lo[P + 1];   // degree P-1 Bernstein, b_j = C(P-1, j) t^j s^(P-1-j), j = 0..P-1
#pragma unroll
    for (int j = 0; j < P; ++j) lo[j] = binomf(P - 1, j) * (tp[j] * sp[P - 1 - j]);
#pragma unroll
    for (int j = 0; j <= P; ++j) {
        const float v = binomf(P, j) * (tp[j] * sp[P - j]);
        float d;                                  // B_j' = P (b_{j-1} - b_j)
        if (j == 0) d = -(float)P * lo[0];
        else if (j == P) d = (float)P * lo[P - 1];
        else d = (float)P * (lo[j - 1] - lo[j]);
        B[j] = SWAP ? make_float2(d, v) : make_float2(v, d);
    }
}

template <int P>
__device__ __forceinline__ void bernstein_value(float t, float (&N)[P + 1]) {
    const float s = 1.f - t;
    float tp[P + 1], sp[P + 1];
    tp[0] = 1.f;
    sp[0] = 1.f;
#pragma unroll
    for (int m = 1; m <= P; ++m) {
        tp[m] = tp[m - 1] * t;
        sp[m] = sp[m - 1] * s;
    }
#pragma unroll
    for (int j = 0; j <= P; ++j) N[j] = binomf(P, j) * (tp[j] * sp[P - j]);
}

struct BezGrid {
    int S0, S1;            // spans along u, v
    int S0g, S1g;          // grouped layout: groups along u, v (bez_groups)
    int64_t q_f4;          // size of the block array in float4 (debug bounds checks)
};

template <int P>
struct BezBlock {
    static constexpr int ROW = bez_row(P);                 // floats per stored row
    static constexpr int F4 = (P + 1) * (P + 1) * ROW / 4;  // float4 per block (p >= 2)
    static constexpr int FLOATS = (P + 1) * (P + 1) * ROW;
};

// SEC: floats between a block's 32-byte sectors (bez_sec: 8 for kBezier, 32
// for the grouped kBezierG, p = 3)
template <int P, int SEC = 8>
__device__ __forceinline__ const float4* bez_block(const float4* Q, const BezGrid& g, int su, int sv, int sw) {
    static_assert(SEC == 8 || (SEC == 32 && P == 3), "grouped Bezier blocks are p = 3");
    MFA_DCHECK(su >= 0 && su < g.S0 && sv >= 0 && sv < g.S1 && sw >= 0);
    const int64_t o = SEC == 32 ? bez_group_key(g.S0g, g.S1g, su, sv, sw) << 3
                                : bez_block_offset(P, false, g.S0, g.S1, su, sv, sw);
    MFA_DCHECK((o + (SEC == 32 ? 7 * SEC + 8 : BezBlock<P>::FLOATS)) / 4 <= g.q_f4);
    return reinterpret_cast<const float4*>(reinterpret_cast<const float*>(Q) + o);
}

// block b = (sw * S1 + sv) * S0 + su (< 2^31: mfa_model_create), linear layout only
template <int P>
__device__ __forceinline__ const float4* bez_block_at(const float4* Q, const BezGrid& g, int b) {
    MFA_DCHECK(b >= 0 && (int64_t)(b + 1) * (BezBlock<P>::FLOATS / 4) <= g.q_f4);
    return reinterpret_cast<const float4*>(reinterpret_cast<const float*>(Q) + (int64_t)b * BezBlock<P>::FLOATS);
}

// slab c of a Bezier block: rows b = 0..P at consecutive compile-time offsets

template <int P, int SEC = 8>
__device__ __forceinline__ void load_bslab(const float4* __restrict__ q, float (&r)[P + 1][P + 1]) {
    static_assert(MFA_LDG256 || SEC == 8, "the grouped Bezier layout is read by sector loads");
#if MFA_LDG256
    if constexpr (P == 3) {   // 64 bytes = two sector loads
        const float* f = reinterpret_cast<const float*>(q);
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            float x[8];
            ldg256(f + SEC * k, x);
#pragma unroll
            for (int e = 0; e < 8; ++e) r[2 * k + (e >> 2)][e & 3] = x[e];
        }
        return;
    }
#endif
#pragma unroll
    for (int b = 0; b <= P; ++b) {
        if constexpr (P == 1) {
            const float2 x = __ldg(reinterpret_cast<const float2*>(q) + b);
            r[b][0] = x.x; r[b][1] = x.y;
        } else {
            const float4 x = __ldg(q + b);
            r[b][0] = x.x; r[b][1] = x.y; r[b][2] = x.z;
            if constexpr (P == 3) r[b][3] = x.w;
        }
    }
}

template <int P, int SEC = 8>
__device__ __forceinline__ const float4* bslab_ptr(const float4* q, int c) {
    if constexpr (SEC != 8) return reinterpret_cast<const float4*>(reinterpret_cast<const float*>(q) + c * 2 * SEC);
    return reinterpret_cast<const float4*>(reinterpret_cast<const float*>(q) + c * (P + 1) * BezBlock<P>::ROW);
}

template <int P, int SEC = 8>
__device__ __forceinline__ void load_bblock(const float4* __restrict__ q, float (&nb)[P + 1][P + 1][P + 1]) {
    static_assert(MFA_LDG256 || SEC == 8, "the grouped Bezier layout is read by sector loads");
#if MFA_LDG256
    if constexpr (P == 3) {   // the 256-byte block as 8 sector loads (two rows each)
        const float* f = reinterpret_cast<const float*>(q);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            float r[8];
            ldg256(f + SEC * k, r);
#pragma unroll
            for (int e = 0; e < 8; ++e) nb[k >> 1][2 * (k & 1) + (e >> 2)][e & 3] = r[e];
        }
        return;
    }
#endif
#pragma unroll
    for (int c = 0; c <= P; ++c) load_bslab<P, SEC>(bslab_ptr<P, SEC>(q, c), nb[c]);
}

template <int P, int SEC = 8>
__device__ __forceinline__ void contract_vg_bez(const float4* __restrict__ q, float (&r0)[P + 1][P + 1],
                                                const float2 (&Bu)[P + 1], const float2 (&Bvs)[P + 1],
                                                const float2 (&Bw)[P + 1], float& val, float& gu, float& gv,
                                                float& gw) {
    float2 vw = make_float2(0.f, 0.f), gvu = make_float2(0.f, 0.f);
    float r1[P + 1][P + 1];
#pragma unroll
    for (int c = 0; c <= P; ++c) {
        if (c & 1) {
            if (c < P) load_bslab<P, SEC>(bslab_ptr<P, SEC>(q, c + 1), r0);
            contract_slab<P>(r1, Bu, Bvs, Bw[c], vw, gvu);
        } else {
            if (c < P) load_bslab<P, SEC>(bslab_ptr<P, SEC>(q, c + 1), r1);
            contract_slab<P>(r0, Bu, Bvs, Bw[c], vw, gvu);
        }
    }
    val = vw.x;
    gw = vw.y;
    gv = gvu.x;
    gu = gvu.y;
}

}  // namespace mfa
