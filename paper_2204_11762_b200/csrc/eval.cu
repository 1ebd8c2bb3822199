// mfa_eval_batch kernel: per point a4 span -> a5 basis +
// derivatives -> a6 gather -> a7 contraction; value and parameter-space
// gradient (Algorithm 1 lines 6 and 9; "all derivatives
// along the three dimensions at once").  One point per thread, grid-stride,
// grid = a multiple of the SM count.
#include "kernels.cuh"

namespace mfa {

struct EvalArgs {
    const float4* Q;
    BrickGrid g;
    BezGrid bg;
    AxisArgs ax[3];
    const float* u;
    const float* v;
    const float* w;
    float* value;
    float* du;
    float* dv;
    float* dw;
    unsigned long long* n_err;
    int64_t n;
};

template <int P, int LAYOUT, bool UNI, bool GRAD>
__global__ void __launch_bounds__(256) eval_kernel(const __grid_constant__ EvalArgs args) {
    constexpr bool BEZ = LAYOUT == kBezier;
    unsigned errs = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < args.n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float q[3] = {__ldg(args.u + i), __ldg(args.v + i), __ldg(args.w + i)};
        if (!(q[0] >= 0.f && q[0] <= 1.f && q[1] >= 0.f && q[1] <= 1.f && q[2] >= 0.f && q[2] <= 1.f)) {
            ++errs;
            args.value[i] = __int_as_float(0x7fc00000);
            if (GRAD) {
                args.du[i] = __int_as_float(0x7fc00000);
                args.dv[i] = __int_as_float(0x7fc00000);
                args.dw[i] = __int_as_float(0x7fc00000);
            }
            continue;
        }
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
        if constexpr (BEZ) {
            const float4* base = bez_block<P>(args.Q, args.bg, s[0], s[1], s[2]);
            if (GRAD) {
                float r0[P + 1][P + 1];
                load_bslab<P>(base, r0);
                float2 Bu[P + 1], Bv[P + 1], Bw[P + 1];
                bernstein<P, false>(t[0], Bu);
                bernstein<P, true>(t[1], Bv);
                bernstein<P, false>(t[2], Bw);
                float val, gu, gv, gw;
                contract_vg_bez<P>(base, r0, Bu, Bv, Bw, val, gu, gv, gw);
                args.value[i] = val;
                args.du[i] = gu * sc[0];
                args.dv[i] = gv * sc[1];
                args.dw[i] = gw * sc[2];
            } else {
                float nb[P + 1][P + 1][P + 1];
                load_bblock<P>(base, nb);
                float Nu[P + 1], Nv[P + 1], Nw[P + 1];
                bernstein_value<P>(t[0], Nu);
                bernstein_value<P>(t[1], Nv);
                bernstein_value<P>(t[2], Nw);
                args.value[i] = contract_v_cached<P>(nb, Nu, Nv, Nw);
            }
            continue;
        }
        const float4* base = args.Q + brick_entry<P>(args.g, s[0], s[1], s[2]);
        float r0[P + 1][P + 1];
        load_slab<P>(base, r0);   // issued before the basis so its latency overlaps it
        if (GRAD) {
            float2 Bu[P + 1], Bv[P + 1], Bw[P + 1];
            axis_basis<P, false>(args.ax[0], UNI, s[0], t[0], Bu);
            axis_basis<P, true>(args.ax[1], UNI, s[1], t[1], Bv);
            axis_basis<P, false>(args.ax[2], UNI, s[2], t[2], Bw);
            float val, gu, gv, gw;
            contract_vg<P>(base, r0, Bu, Bv, Bw, val, gu, gv, gw);
            args.value[i] = val;
            args.du[i] = gu * sc[0];
            args.dv[i] = gv * sc[1];
            args.dw[i] = gw * sc[2];
        } else {
            float Nu[P + 1], Nv[P + 1], Nw[P + 1];
            axis_basis_value<P>(args.ax[0], UNI, s[0], t[0], Nu);
            axis_basis_value<P>(args.ax[1], UNI, s[1], t[1], Nv);
            axis_basis_value<P>(args.ax[2], UNI, s[2], t[2], Nw);
            args.value[i] = contract_v<P>(base, r0, Nu, Nv, Nw);
        }
    }
    if (args.n_err) {
        for (int o = 16; o > 0; o >>= 1) errs += __shfl_xor_sync(0xffffffffu, errs, o);
        if ((threadIdx.x & 31) == 0 && errs) atomicAdd(args.n_err, (unsigned long long)errs);
    }
}

template <int P, int LAYOUT, bool UNI, bool GRAD>
static cudaError_t launch_eval_t(const EvalArgs& a, cudaStream_t st) {
    int sms = 148, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (a.n + 255) / 256;
    const int64_t grid = std::min<int64_t>(want, (int64_t)sms * 16);
    eval_kernel<P, LAYOUT, UNI, GRAD><<<(unsigned)grid, 256, 0, st>>>(a);
    return cudaGetLastError();
}

template <int P, int LAYOUT>
static cudaError_t dispatch_eval_l(const EvalArgs& a, bool uni, bool grad, cudaStream_t st) {
    if (uni)
        return grad ? launch_eval_t<P, LAYOUT, true, true>(a, st) : launch_eval_t<P, LAYOUT, true, false>(a, st);
    return grad ? launch_eval_t<P, LAYOUT, false, true>(a, st) : launch_eval_t<P, LAYOUT, false, false>(a, st);
}

template <int P>
static cudaError_t dispatch_eval(const EvalArgs& a, int layout, bool uni, bool grad, cudaStream_t st) {
    if constexpr (P <= 3) {
        if (layout == kBezier) return dispatch_eval_l<P, kBezier>(a, uni, grad, st);
    }
    return dispatch_eval_l<P, kQuads>(a, uni, grad, st);
}

mfa_status launch_eval(const Model* m, int64_t n, const float* u, const float* v, const float* w, float* value,
                       float* du, float* dv, float* dw, unsigned long long* n_err, cudaStream_t st) {
    EvalArgs a;
    a.Q = m->Q;
    a.g.nbx = m->nb[0];
    a.g.nby = m->nb[1];
    a.g.q_f4 = m->q_f4;
    a.bg.q_f4 = m->q_f4;
    a.bg.S0 = (int)(m->n[0] - m->p);
    a.bg.S1 = (int)(m->n[1] - m->p);
    for (int d = 0; d < 3; ++d) a.ax[d] = make_axis_args(m->ax[d]);
    a.u = u;
    a.v = v;
    a.w = w;
    a.value = value;
    a.du = du;
    a.dv = dv;
    a.dw = dw;
    a.n_err = n_err;
    a.n = n;
    const bool uni = m->uniform[0] && m->uniform[1] && m->uniform[2];
    const bool grad = du != nullptr;
    cudaError_t e;
    switch (m->p) {
        case 1: e = dispatch_eval<1>(a, m->layout, uni, grad, st); break;
        case 2: e = dispatch_eval<2>(a, m->layout, uni, grad, st); break;
        case 3: e = dispatch_eval<3>(a, m->layout, uni, grad, st); break;
        case 4: e = dispatch_eval<4>(a, m->layout, uni, grad, st); break;
        default: e = dispatch_eval<5>(a, m->layout, uni, grad, st); break;
    }
    return e == cudaSuccess ? MFA_OK : cuda_fail(e, "eval launch");
}

}  // namespace mfa
