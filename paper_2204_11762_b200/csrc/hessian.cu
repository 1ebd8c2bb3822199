// mfa_eval_hessian: value, gradient and the six second
// partials of the MFA at n points ("Higher-order derivatives, up to the
// polynomial degree, are also analytically available"; the
// curvature-based transfer functions and shading they enable are named as
// applications).
//
// Per point (one thread, grid-stride): a4 span + local coordinate (as
// mfa_eval_batch), a5 basis with first and second t-derivatives per axis by a
// three-output Horner scheme on the span's power-basis coefficients (the
// compile-time uniform set on interior uniform spans, the span table
// elsewhere, the Bernstein set for Bezier blocks), a6 slab gather, a7 a
// sum-factorised contraction with 3 x-sums per row, 6 y-sums per slab and 10
// outputs:
//   x: a0 = sum N_u P, a1 = sum N'_u P, a2 = sum N''_u P
//   y: B0 = N_v a0, B1 = N_v a1, B2 = N'_v a0, B3 = N_v a2, B4 = N'_v a1, B5 = N''_v a0
//   z: v = N_w B0, v_u = N_w B1, v_v = N_w B2, v_w = N'_w B0, v_uu = N_w B3,
//      v_uv = N_w B4, v_vv = N_w B5, v_uw = N'_w B1, v_vw = N'_w B2, v_ww = N''_w B0
// then t -> u scaling per axis (sc = S or 1/h; squared / mixed for 2nd order).
// With a workspace (mfa_eval_hessian_ws) large batches are spatially binned
// first, as in mfa_eval_batch_ws (eval.cu), and gathered back.
#include "kernels.cuh"

namespace mfa {

struct HessArgs {
    const float4* Q;
    BrickGrid g;
    BezGrid bg;
    AxisArgs ax[3];
    const float* u;
    const float* v;
    const float* w;
    float* value;   // optional [n]
    float* grad;    // optional [3][n]
    float* hess;    // [6][n]: uu, vv, ww, uv, uw, vw
    unsigned long long* n_err;
    int64_t n;
    const float4* rec;   // SORTED: (u, v, w, index bits) in bin order
    float4* out;         // SORTED: 3 float4 per sorted position (10 outputs + pad)
};

template <int P, int LAYOUT, bool UNI, bool SORTED>
__global__ void __launch_bounds__(256) hessian_kernel(const __grid_constant__ HessArgs args) {
    constexpr bool BEZ = is_bez(LAYOUT);
    constexpr int SEC = bez_sec(LAYOUT == kBezierG);
    const int64_t n = args.n;
    unsigned errs = 0;
    for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < n; it += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = it;
        float q[3];
        if constexpr (SORTED) {
            const float4 r = __ldg(args.rec + it);
            q[0] = r.x;
            q[1] = r.y;
            q[2] = r.z;
        } else {
            q[0] = __ldg(args.u + i);
            q[1] = __ldg(args.v + i);
            q[2] = __ldg(args.w + i);
        }
        float out[10];
        if (!(q[0] >= 0.f && q[0] <= 1.f && q[1] >= 0.f && q[1] <= 1.f && q[2] >= 0.f && q[2] <= 1.f)) {
            ++errs;
#pragma unroll
            for (int k = 0; k < 10; ++k) out[k] = __int_as_float(0x7fc00000);
        } else {
            int s[3];
            float t[3], sc[3];
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                if (UNI) {
                    uni_span_f32(q[d], args.ax[d].S, args.ax[d].nsp, s[d], t[d]);
                    sc[d] = args.ax[d].S;
                } else {
                    nonuni_span_f32(args.ax[d], q[d], s[d], t[d], sc[d]);
                }
            }
            const float4* base = BEZ ? bez_block<P, SEC>(args.Q, args.bg, s[0], s[1], s[2])
                                     : (LAYOUT == kBricks ? args.Q : args.Q + brick_entry<P>(args.g, s[0], s[1], s[2]));
            PlainRef pe{0, 0};
            if constexpr (LAYOUT == kBricks) pe = plain_entry<P>(args.g, s[0], s[1], s[2]);
            float Nu[P + 1], Du[P + 1], Eu[P + 1], Nv[P + 1], Dv[P + 1], Ev[P + 1], Nw[P + 1], Dw[P + 1], Ew[P + 1];
            basis3<P, LAYOUT, UNI>(args.ax[0], s[0], t[0], Nu, Du, Eu);
            basis3<P, LAYOUT, UNI>(args.ax[1], s[1], t[1], Nv, Dv, Ev);
            basis3<P, LAYOUT, UNI>(args.ax[2], s[2], t[2], Nw, Dw, Ew);
#pragma unroll
            for (int k = 0; k < 10; ++k) out[k] = 0.f;
#pragma unroll
            for (int c = 0; c <= P; ++c) {
                float r[P + 1][P + 1];
                if constexpr (BEZ)
                    load_bslab<P, SEC>(bslab_ptr<P, SEC>(base, c), r);
                else if constexpr (LAYOUT == kBricks)
                    load_pslab<P>(base, pe, c, r);
                else
                    load_slab<P>(base + c * Brick<P>::SLAB, r);
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
                out[0] = fmaf(Nw[c], B[0], out[0]);   // v
                out[1] = fmaf(Nw[c], B[1], out[1]);   // v_u
                out[2] = fmaf(Nw[c], B[2], out[2]);   // v_v
                out[3] = fmaf(Dw[c], B[0], out[3]);   // v_w
                out[4] = fmaf(Nw[c], B[3], out[4]);   // v_uu
                out[5] = fmaf(Nw[c], B[5], out[5]);   // v_vv
                out[6] = fmaf(Ew[c], B[0], out[6]);   // v_ww
                out[7] = fmaf(Nw[c], B[4], out[7]);   // v_uv
                out[8] = fmaf(Dw[c], B[1], out[8]);   // v_uw
                out[9] = fmaf(Dw[c], B[2], out[9]);   // v_vw
            }
            out[1] *= sc[0];
            out[2] *= sc[1];
            out[3] *= sc[2];
            out[4] *= sc[0] * sc[0];
            out[5] *= sc[1] * sc[1];
            out[6] *= sc[2] * sc[2];
            out[7] *= sc[0] * sc[1];
            out[8] *= sc[0] * sc[2];
            out[9] *= sc[1] * sc[2];
        }
        if constexpr (SORTED) {   // coalesced at the sorted position; gathered back afterwards
            args.out[3 * it + 0] = make_float4(out[0], out[1], out[2], out[3]);
            args.out[3 * it + 1] = make_float4(out[4], out[5], out[6], out[7]);
            args.out[3 * it + 2] = make_float4(out[8], out[9], 0.f, 0.f);
        } else {
            if (args.value) args.value[i] = out[0];
            if (args.grad) {
#pragma unroll
                for (int k = 0; k < 3; ++k) args.grad[k * n + i] = out[1 + k];
            }
#pragma unroll
            for (int k = 0; k < 6; ++k) args.hess[k * n + i] = out[4 + k];
        }
    }
    if (args.n_err) {
        for (int o = 16; o > 0; o >>= 1) errs += __shfl_xor_sync(0xffffffffu, errs, o);
        if ((threadIdx.x & 31) == 0 && errs) atomicAdd(args.n_err, (unsigned long long)errs);
    }
}

template <int P, int LAYOUT, bool UNI>
static cudaError_t launch_hess_t(const HessArgs& a, cudaStream_t st) {
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t grid = std::min<int64_t>((a.n + 255) / 256, (int64_t)sms * 16);
    if (a.rec)
        hessian_kernel<P, LAYOUT, UNI, true><<<(unsigned)grid, 256, 0, st>>>(a);
    else
        hessian_kernel<P, LAYOUT, UNI, false><<<(unsigned)grid, 256, 0, st>>>(a);
    return cudaGetLastError();
}

// results of the sorted evaluation back to the caller's SoA arrays
#ifndef MFA_HESS_ILP
#define MFA_HESS_ILP 4
#endif
__global__ void __launch_bounds__(256) hess_gather_kernel(const float4* __restrict__ out, const int* __restrict__ pos,
                                                          int64_t n, float* __restrict__ value,
                                                          float* __restrict__ grad, float* __restrict__ hess) {
    // MFA_HESS_ILP points per thread per iteration: their random 48-byte reads
    // are independent, so more of them are in flight
    constexpr int U = MFA_HESS_ILP;
    const int64_t S = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n; i0 += U * S) {
        int64_t p[U];
        float4 a[U], b[U], c[U];
#pragma unroll
        for (int k = 0; k < U; ++k) p[k] = i0 + k * S < n ? __ldg(pos + i0 + k * S) : 0;
#pragma unroll
        for (int k = 0; k < U; ++k)
            if (i0 + k * S < n) {
                a[k] = __ldg(out + 3 * p[k]);
                b[k] = __ldg(out + 3 * p[k] + 1);
                c[k] = __ldg(out + 3 * p[k] + 2);
            }
#pragma unroll
        for (int k = 0; k < U; ++k) {
            const int64_t i = i0 + k * S;
            if (i >= n) continue;
            if (value) value[i] = a[k].x;
            if (grad) {
                grad[i] = a[k].y;
                grad[n + i] = a[k].z;
                grad[2 * n + i] = a[k].w;
            }
            hess[i] = b[k].x;
            hess[n + i] = b[k].y;
            hess[2 * n + i] = b[k].z;
            hess[3 * n + i] = b[k].w;
            hess[4 * n + i] = c[k].x;
            hess[5 * n + i] = c[k].y;
        }
    }
}

size_t hessian_workspace_bytes(const Model* m, int64_t n) {
    return bin_workspace_bytes(m, n) + ((sizeof(float4) * 3 * (size_t)n + 255) & ~(size_t)255);
}

template <int P>
static cudaError_t dispatch_hess(const HessArgs& a, int layout, bool uni, cudaStream_t st) {
    if constexpr (P <= 3) {
        if (layout == kBezier)
            return uni ? launch_hess_t<P, kBezier, true>(a, st) : launch_hess_t<P, kBezier, false>(a, st);
        if constexpr (P == 3)
            if (layout == kBezierG)
                return uni ? launch_hess_t<P, kBezierG, true>(a, st) : launch_hess_t<P, kBezierG, false>(a, st);
        if (layout == kBricks)
            return uni ? launch_hess_t<P, kBricks, true>(a, st) : launch_hess_t<P, kBricks, false>(a, st);
    }
    return uni ? launch_hess_t<P, kQuads, true>(a, st) : launch_hess_t<P, kQuads, false>(a, st);
}

}  // namespace mfa

using namespace mfa;

extern "C" size_t mfa_hessian_workspace_bytes(mfa_model h, int64_t n) {
    if (!h || n < 0) return 0;
    return hessian_workspace_bytes(reinterpret_cast<const Model*>(h), n);
}

extern "C" mfa_status mfa_eval_hessian(mfa_model h, int64_t n, const float* u, const float* v, const float* w,
                                       float* value, float* grad, float* hess, unsigned long long* n_domain_errors,
                                       mfa_stream stream) {
    if (h && check_device(reinterpret_cast<const Model*>(h)) == MFA_OK && bin_worthwhile(reinterpret_cast<const Model*>(h), n)) {
        // the binned path with stream-ordered scratch (no caller workspace)
        const size_t bytes = hessian_workspace_bytes(reinterpret_cast<const Model*>(h), n);
        void* ws = scratch_alloc(bytes, (cudaStream_t)stream);
        if (ws) {
            const mfa_status s = mfa_eval_hessian_ws(h, n, u, v, w, value, grad, hess, n_domain_errors, ws, bytes,
                                                     stream);
            cudaFreeAsync(ws, (cudaStream_t)stream);
            return s;
        }
    }
    return mfa_eval_hessian_ws(h, n, u, v, w, value, grad, hess, n_domain_errors, nullptr, 0, stream);
}

extern "C" mfa_status mfa_eval_hessian_ws(mfa_model h, int64_t n, const float* u, const float* v, const float* w,
                                          float* value, float* grad, float* hess,
                                          unsigned long long* n_domain_errors, void* workspace,
                                          size_t workspace_bytes, mfa_stream stream) {
    if (!h) return fail(MFA_ERR_INVALID_ARG, "model is NULL");
    if (n < 0) return fail(MFA_ERR_INVALID_ARG, "n < 0");
    if (n == 0) return MFA_OK;
    if (!u || !v || !w || !hess) return fail(MFA_ERR_INVALID_ARG, "u, v, w and hess are required");
    const Model* m = reinterpret_cast<const Model*>(h);
    mfa_status s = check_device(m);
    if (s != MFA_OK) return s;
    HessArgs a;
    a.Q = m->Q;
    a.g.nbx = m->nb[0];
    a.g.nby = m->nb[1];
    a.g.q_f4 = m->q_f4;
    a.bg.q_f4 = m->q_f4;
    a.bg.S0 = (int)(m->n[0] - m->p);
    a.bg.S1 = (int)(m->n[1] - m->p);
    a.bg.S0g = bez_groups(a.bg.S0, kGLu);
    a.bg.S1g = bez_groups(a.bg.S1, kGLv);
    for (int d = 0; d < 3; ++d) a.ax[d] = make_axis_args(m->ax[d]);
    a.u = u;
    a.v = v;
    a.w = w;
    a.value = value;
    a.grad = grad;
    a.hess = hess;
    a.n_err = n_domain_errors;
    a.n = n;
    a.rec = nullptr;
    a.out = nullptr;
    const bool uni = m->uniform[0] && m->uniform[1] && m->uniform[2];
    cudaStream_t st = (cudaStream_t)stream;
    if (workspace && workspace_bytes < hessian_workspace_bytes(m, n))
        return fail(MFA_ERR_INVALID_ARG, "workspace smaller than mfa_hessian_workspace_bytes()");
    const int* pos = nullptr;
    if (workspace && bin_worthwhile(m, n)) {
        const BinnedPoints bp = bin_points(m, n, u, v, w, workspace, st);
        a.rec = bp.rec;
        pos = bp.pos;
        a.out = reinterpret_cast<float4*>((char*)workspace + bin_workspace_bytes(m, n));
    }
    cudaError_t e;
    switch (m->p) {
        case 1: e = dispatch_hess<1>(a, m->layout, uni, st); break;
        case 2: e = dispatch_hess<2>(a, m->layout, uni, st); break;
        case 3: e = dispatch_hess<3>(a, m->layout, uni, st); break;
        case 4: e = dispatch_hess<4>(a, m->layout, uni, st); break;
        default: e = dispatch_hess<5>(a, m->layout, uni, st); break;
    }
    if (e == cudaSuccess && a.rec) {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)sms * 8);
        hess_gather_kernel<<<grid, 256, 0, st>>>(a.out, pos, n, value, grad, hess);
        e = cudaGetLastError();
    }
    return e == cudaSuccess ? MFA_OK : cuda_fail(e, "hessian launch");
}
