// Device building blocks of the hot path:
//   a4 span + local coordinate       (uniform: span units; non-uniform: knot tables)
//   a5 basis + first derivatives     (power-basis Horner per span, simultaneous value/derivative)
//   a6 neighbourhood gather          (row quads: one aligned 16-byte load per u-row)
//   a7 sum-factorised contraction    (x, then y, then z; paired FP32 FMAs, FFMA2)
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
    int nsp;
    int M;
    int mshift;      // 62 - log2(M): bucket of a 2^62 fixed-point coordinate
    int ic_lo, ic_hi;
    float S;
    float interior[(kMaxP + 1) * (kMaxP + 1)];
};

__host__ inline AxisArgs make_axis_args(const AxisTables& A) {
    AxisArgs a;
    a.coef = A.coef;
    a.invh = A.invh;
    a.kh = A.kh;
    a.kl = A.kl;
    a.kfx = A.kfx;
    a.bucket = A.bucket;
    a.nsp = A.nsp;
    a.M = A.M;
    int lg = 0;
    while ((1 << lg) < A.M) ++lg;
    a.mshift = kNonUniFracBits - lg;
    a.ic_lo = A.ic_lo;
    a.ic_hi = A.ic_hi;
    a.S = A.S;
    for (int i = 0; i < (kMaxP + 1) * (kMaxP + 1); ++i) a.interior[i] = A.interior[i];
    return a;
}

// ---------------------------------------------------------------------------
// a5: p+1 basis values and derivatives by Horner on the span's power basis.
// c[a*(P+1)+m] is the coefficient of t^m of function a; scale = dt/du.
// Simultaneous Horner:  b <- b t + c_m,  d <- d t + b  gives P(t), P'(t).
// Output pairs: X-order (N, N') or swapped (N', N) when SWAP.
// ---------------------------------------------------------------------------
template <int P, bool SWAP>
__device__ __forceinline__ void horner_basis(const float* c, float t, float scale, float2 (&B)[P + 1]) {
#pragma unroll
    for (int a = 0; a <= P; ++a) {
        float v = c[a * (P + 1) + P];
        float d = 0.f;
#pragma unroll
        for (int m = P - 1; m >= 0; --m) {
            d = fmaf(d, t, v);
            v = fmaf(v, t, c[a * (P + 1) + m]);
        }
        d *= scale;
        B[a] = SWAP ? make_float2(d, v) : make_float2(v, d);
    }
}

template <int P>
__device__ __forceinline__ void horner_value(const float* c, float t, float (&B)[P + 1]) {
#pragma unroll
    for (int a = 0; a <= P; ++a) {
        float v = c[a * (P + 1) + P];
#pragma unroll
        for (int m = P - 1; m >= 0; --m) v = fmaf(v, t, c[a * (P + 1) + m]);
        B[a] = v;
    }
}

// Load one span record (coefficients) from the table into registers.
template <int P>
__device__ __forceinline__ void load_rec(const float* __restrict__ coef, int s, float (&c)[rec_floats(P)]) {
    const float4* r = reinterpret_cast<const float4*>(coef + (int64_t)s * rec_floats(P));
#pragma unroll
    for (int q = 0; q < rec_floats(P) / 4; ++q) {
        float4 x = __ldg(r + q);
        c[4 * q + 0] = x.x;
        c[4 * q + 1] = x.y;
        c[4 * q + 2] = x.z;
        c[4 * q + 3] = x.w;
    }
}

// Basis of one axis: uniform axes take the constant interior polynomials
// (kernel-parameter constant bank) unless the span is one of the p-1
// boundary-affected spans at either end; non-uniform axes always load.
template <int P, bool SWAP>
__device__ __forceinline__ void axis_basis(const AxisArgs& A, bool uniform, int s, float t, float scale,
                                           float2 (&B)[P + 1]) {
    if (uniform && s >= A.ic_lo && s <= A.ic_hi) {
        horner_basis<P, SWAP>(A.interior, t, scale, B);
    } else {
        float c[rec_floats(P)];
        load_rec<P>(A.coef, s, c);
        horner_basis<P, SWAP>(c, t, scale, B);
    }
}

template <int P>
__device__ __forceinline__ void axis_basis_value(const AxisArgs& A, bool uniform, int s, float t, float (&B)[P + 1]) {
    if (uniform && s >= A.ic_lo && s <= A.ic_hi) {
        horner_value<P>(A.interior, t, B);
    } else {
        float c[rec_floats(P)];
        load_rec<P>(A.coef, s, c);
        horner_value<P>(c, t, B);
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
    float fl = floorf(hi);
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

// a4 (non-uniform axis, render): 2^62 fixed point, incremental search from
// the previous sample's span (spans are monotone along a ray).
__device__ __forceinline__ void nonuni_span_fx(const AxisArgs& A, long long F, int& s, float& t, float& invh) {
    F = max(F, 0LL);
    F = min(F, 1LL << kNonUniFracBits);
    while (s + 1 < A.nsp && F >= __ldg(A.kfx + s + 1)) ++s;
    while (s > 0 && F < __ldg(A.kfx + s)) --s;
    invh = __ldg(A.invh + s);
    const long long d = F - __ldg(A.kfx + s);
    t = __ll2float_rn(d) * (invh * 0x1p-62f);
}

__device__ __forceinline__ int nonuni_first_span_fx(const AxisArgs& A, long long F) {
    F = max(F, 0LL);
    F = min(F, (1LL << kNonUniFracBits) - 1);
    int b = (int)(F >> A.mshift);
    b = min(max(b, 0), A.M - 1);
    return __ldg(A.bucket + b);
}

// ---------------------------------------------------------------------------
// a6: row of p+1 consecutive u-values starting at the quad q.
// ---------------------------------------------------------------------------
template <int P>
__device__ __forceinline__ void load_row(const float4* __restrict__ q, float (&r)[P + 1]) {
    if constexpr (P == 1) {
        float2 x = __ldg(reinterpret_cast<const float2*>(q));
        r[0] = x.x; r[1] = x.y;
    } else if constexpr (P == 2) {
        float4 x = __ldg(q);
        r[0] = x.x; r[1] = x.y; r[2] = x.z;
    } else if constexpr (P == 3) {
        float4 x = __ldg(q);
        r[0] = x.x; r[1] = x.y; r[2] = x.z; r[3] = x.w;
    } else if constexpr (P == 4) {
        float4 x = __ldg(q);
        r[0] = x.x; r[1] = x.y; r[2] = x.z; r[3] = x.w;
        r[4] = __ldg(reinterpret_cast<const float*>(q + 1) + 3);
    } else {
        float4 x = __ldg(q);
        float2 y = __ldg(reinterpret_cast<const float2*>(q + 4));
        r[0] = x.x; r[1] = x.y; r[2] = x.z; r[3] = x.w; r[4] = y.x; r[5] = y.y;
    }
}

// ---------------------------------------------------------------------------
// a7: value + parameter-space gradient, sum-factorised ("all
// derivatives along the three dimensions at once"; "sum operations on
// each of the three dimensions").  Per row (c,b):
//   (a0, a1) = sum_a (Nu_a, Nu'_a) * P            [FFMA2, P broadcast]
//   B  += Nv_b a0 ; (Bv, Bu) += (Nv'_b, Nv_b) * (a0, a1)
// per slab c:  (v, g_w) += (Nw_c, Nw'_c) * B ;  (g_v, g_u) += Nw_c * (Bv, Bu)
// Bu: (N, N'), Bvs: (N', N) (swapped), Bw: (N, N').
// ---------------------------------------------------------------------------
template <int P>
__device__ __forceinline__ void contract_vg(const float4* __restrict__ base, int row_v, int row_w,
                                            const float2 (&Bu)[P + 1], const float2 (&Bvs)[P + 1],
                                            const float2 (&Bw)[P + 1], float& val, float& gu, float& gv,
                                            float& gw) {
    float2 vw = make_float2(0.f, 0.f), gvu = make_float2(0.f, 0.f);
#pragma unroll
    for (int c = 0; c <= P; ++c) {
        float B = 0.f;
        float2 Bvu = make_float2(0.f, 0.f);
#pragma unroll
        for (int b = 0; b <= P; ++b) {
            float r[P + 1];
            load_row<P>(base + c * row_w + b * row_v, r);
            float2 a01 = __fmul2_rn(Bu[0], make_float2(r[0], r[0]));
#pragma unroll
            for (int a = 1; a <= P; ++a) a01 = __ffma2_rn(Bu[a], make_float2(r[a], r[a]), a01);
            B = fmaf(Bvs[b].y, a01.x, B);
            Bvu = __ffma2_rn(Bvs[b], a01, Bvu);
        }
        vw = __ffma2_rn(Bw[c], make_float2(B, B), vw);
        gvu = __ffma2_rn(make_float2(Bw[c].x, Bw[c].x), Bvu, gvu);
    }
    val = vw.x;
    gw = vw.y;
    gv = gvu.x;
    gu = gvu.y;
}

template <int P>
__device__ __forceinline__ float contract_v(const float4* __restrict__ base, int row_v, int row_w,
                                            const float (&Nu)[P + 1], const float (&Nv)[P + 1],
                                            const float (&Nw)[P + 1]) {
    float val = 0.f;
#pragma unroll
    for (int c = 0; c <= P; ++c) {
        float B = 0.f;
#pragma unroll
        for (int b = 0; b <= P; ++b) {
            float r[P + 1];
            load_row<P>(base + c * row_w + b * row_v, r);
            float a0 = Nu[0] * r[0];
#pragma unroll
            for (int a = 1; a <= P; ++a) a0 = fmaf(Nu[a], r[a], a0);
            B = fmaf(Nv[b], a0, B);
        }
        val = fmaf(Nw[c], B, val);
    }
    return val;
}

}  // namespace mfa
