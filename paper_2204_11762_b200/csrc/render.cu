// mfa_render host side: argument marshalling into RenderArgs and the launch
// (the kernel is in render_kernel.cuh; this TU instantiates it for the MFA
// query path, truth.cu for the analytic ground-truth field).
#include <math.h>

#include <algorithm>

#include "render_kernel.cuh"

namespace mfa {

int acquire_queue_slot(const Model* m, cudaStream_t st) {
    std::lock_guard<std::mutex> lk(m->slot_mu);
    int pick = -1, fresh = -1, done = -1;
    for (int i = 0; i < kQueueSlots && pick < 0; ++i) {
        const Model::QueueSlot& q = m->slots[i];
        if (q.pending) continue;                            // being launched by another thread
        if (q.used && q.stream == st) pick = i;             // stream-ordered after its last user
        else if (!q.used) { if (fresh < 0) fresh = i; }
        else if (done < 0 && cudaEventQuery(q.done) == cudaSuccess) done = i;
    }
    if (pick < 0) pick = fresh >= 0 ? fresh : done;
    if (pick < 0) {
        cudaGetLastError();   // clear cudaErrorNotReady left by the queries
        return -1;
    }
    m->slots[pick].pending = true;
    return pick;
}

void release_queue_slot(const Model* m, int slot, cudaStream_t st) {
    std::lock_guard<std::mutex> lk(m->slot_mu);
    Model::QueueSlot& q = m->slots[slot];
    if (!q.done) cudaEventCreateWithFlags(&q.done, cudaEventDisableTiming);
    cudaEventRecord(q.done, st);
    q.stream = st;
    q.used = true;
    q.pending = false;
}

void free_model_resources(Model* m) {
    for (int i = 0; i < kQueueSlots; ++i)
        if (m->slots[i].done) cudaEventDestroy(m->slots[i].done);
    Model::HostRes& h = m->host;
    if (h.copy) cudaStreamSynchronize(h.copy);
    for (int i = 0; i < 2; ++i) {
        if (h.stage[i]) cudaFree(h.stage[i]);
        if (h.rendered[i]) cudaEventDestroy(h.rendered[i]);
        if (h.copied[i]) cudaEventDestroy(h.copied[i]);
    }
    if (h.tf) cudaFree(h.tf);
    if (h.cnt) cudaFree(h.cnt);
    if (h.copy) cudaStreamDestroy(h.copy);
    h = Model::HostRes{};
}

// NEXT-1 transparent-block skip (shading = 3): one bit per macro block of
// kMacro^3 span triples, set when the transfer function's opacity is 0 over
// the block's whole value range [min, max] of its Bernstein coefficients (the
// spline lies in their convex hull).  The test covers every table entry a
// value in the range can touch in the kernel's lookup (f = (v - v_lo) s,
// entries floor(f) .. floor(f) + 1) with two entries of margin for fp32
// rounding of the sample value; a prefix count of the non-zero-opacity
// entries makes it O(1) per block.
__global__ void macro_transparent_kernel(const unsigned* __restrict__ mmx, int64_t nmac, const float4* __restrict__ tf,
                                         int tf_n, float v_lo, float s_scale, unsigned* __restrict__ bits) {
    __shared__ int pre[1025];
    if (threadIdx.x == 0) {
        int c = 0;
        for (int i = 0; i < tf_n; ++i) {
            pre[i] = c;
            c += tf[i].w != 0.f;
        }
        pre[tf_n] = c;
    }
    __syncthreads();
    const int64_t nw = (nmac + 31) / 32;
    for (int64_t wi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; wi < nw; wi += (int64_t)gridDim.x * blockDim.x) {
        unsigned word = 0;
        for (int bit = 0; bit < 32; ++bit) {
            const int64_t mi = wi * 32 + bit;
            if (mi >= nmac) break;
            const unsigned klo = mmx[2 * mi], khi = mmx[2 * mi + 1];
            if (klo == 0xffffffffu) {   // no span triple in this macro block (past the grid): never sampled
                word |= 1u << bit;
                continue;
            }
            const float lo = __uint_as_float((klo & 0x80000000u) ? (klo & 0x7fffffffu) : ~klo);
            const float hi = __uint_as_float((khi & 0x80000000u) ? (khi & 0x7fffffffu) : ~khi);
            const float flo = fminf(fmaxf((lo - v_lo) * s_scale, 0.f), (float)(tf_n - 1));
            const float fhi = fminf(fmaxf((hi - v_lo) * s_scale, 0.f), (float)(tf_n - 1));
            const int i0 = max(0, (int)floorf(flo) - 2), i1 = min(tf_n - 1, (int)floorf(fhi) + 3);
            if (pre[i1 + 1] - pre[i0] == 0) word |= 1u << bit;
        }
        bits[wi] = word;
    }
}

cudaError_t dispatch_render_main(const RenderArgs& a, int p, int layout, bool uni, int shade, cudaStream_t st) {
    switch (p) {
        case 1: return dispatch_render<1, false>(a, layout, uni, shade, st);
        case 2: return dispatch_render<2, false>(a, layout, uni, shade, st);
        case 3: return dispatch_render<3, false>(a, layout, uni, shade, st);
        case 4: return dispatch_render<4, false>(a, layout, uni, shade, st);
        default: return dispatch_render<5, false>(a, layout, uni, shade, st);
    }
}

mfa_status launch_render(const Model* m, int32_t n_views, const mfa_camera* cams, const mfa_tf* tf,
                         const mfa_render_params* prm, const mfa_tiles* tiles, void* out,
                         unsigned long long* samples, cudaStream_t st, const mfa_render_ext* ext) {
    RenderArgs* a = new RenderArgs();  // ~7 KB: keep it off the caller's stack
    // the extended instantiations run only when a sample takes something from
    // the analytic field or there are explicit lights
    const mfa_field* fld = ext ? ext->field : nullptr;
    const bool field = fld && (fld->value_src || fld->grad_src);
    const bool lights = ext && ext->n_lights > 0;
    const bool curv = ext && ext->curv_n > 0;
    a->fld.vsrc = a->fld.gsrc = 0;
    a->lights.n = 0;
    a->curv.n = 0;
    if (curv) {
        a->curv.tab = reinterpret_cast<const float4*>(ext->curv_rgba);
        a->curv.n = ext->curv_n;
        a->curv.range = (float)ext->curv_range;
        a->curv.scale = (float)((ext->curv_n - 1) / (2.0 * ext->curv_range));
    }
    if (lights) {
        a->lights.n = ext->n_lights;
        for (int l = 0; l < ext->n_lights; ++l) {
            const double* L = ext->light_dir + 3 * l;
            const double len = sqrt(L[0] * L[0] + L[1] * L[1] + L[2] * L[2]);
            for (int k = 0; k < 3; ++k) a->lights.dir[l][k] = (float)(L[k] / len);
            a->lights.intensity[l] = (float)ext->light_intensity[l];
        }
    }
    if (field) {
        a->fld.kind = fld->kind;
        a->fld.vsrc = fld->value_src != 0;
        a->fld.gsrc = fld->grad_src != 0;
        for (int k = 0; k < 6; ++k) a->fld.prm[k] = fld->prm[k];
        for (int d = 0; d < 3; ++d) {
            const bool u = m->uniform[0] && m->uniform[1] && m->uniform[2];
            a->fld.fx_scale[d] = u ? ldexp(1.0 / (double)m->ax[d].nsp, -kUniFracBits) : ldexp(1.0, -kNonUniFracBits);
            a->fld.invL[d] = (float)(1.0 / (prm->box_max[d] - prm->box_min[d]));
        }
    }
    a->Q = m->Q;
    a->g.nbx = m->nb[0];
    a->g.nby = m->nb[1];
    a->g.q_f4 = m->q_f4;
    a->bg.q_f4 = m->q_f4;
    a->bg.S0 = (int)(m->n[0] - m->p);
    a->bg.S1 = (int)(m->n[1] - m->p);
    a->bg.S0g = bez_groups(a->bg.S0, kGLu);
    a->bg.S1g = bez_groups(a->bg.S1, kGLv);
    for (int d = 0; d < 3; ++d) a->ax[d] = make_axis_args(m->ax[d]);
    a->tf = reinterpret_cast<const float4*>(tf->rgba);
    a->tf_n = tf->n_entries;
    a->v_lo = tf->v_lo;
    a->s_scale = (float)((double)(tf->n_entries - 1) / ((double)tf->v_hi - (double)tf->v_lo));
    const bool uni = m->uniform[0] && m->uniform[1] && m->uniform[2];
    for (int d = 0; d < 3; ++d) {
        a->bmin[d] = prm->box_min[d];
        a->L[d] = prm->box_max[d] - prm->box_min[d];
        a->gsc[d] = (float)((uni ? (double)m->ax[d].nsp : 1.0) / a->L[d]);
        a->ax[d].gsc = a->gsc[d];   // non-uniform axes: folded into the span state at each crossing
    }
    a->step = prm->step;
    a->inv_step = 1.0 / prm->step;
    a->inv_w2 = 2.0 / (double)cams[0].width;
    a->inv_h2 = 2.0 / (double)cams[0].height;
    for (int d = 0; d < 3; ++d)   // world offset -> fixed-point sample coordinate
        a->fxs[d] = uni ? ldexp((double)m->ax[d].nsp, kUniFracBits) / a->L[d] : ldexp(1.0, kNonUniFracBits) / a->L[d];
    for (int d = 0; d < 3; ++d) {
        // |DF_d| <= step / L_d * 2^62 (unit ray directions) plus rounding; a
        // crossing lands in the next span whenever that is below every span width
        const double maxdf = ldexp(prm->step / a->L[d], kNonUniFracBits) * (1.0 + 1e-9) + 64.0;
        a->ax[d].multi = !(maxdf < (double)m->ax[d].hmin_fx * (1.0 - 1e-9));
    }
    a->o_max = (float)prm->o_max;
    a->ka = (float)prm->ka;
    a->kd = (float)prm->kd;
    a->ks = (float)prm->ks;
    a->shin = (float)prm->shininess;
    a->eps2 = (float)(prm->grad_eps * prm->grad_eps);
    a->W = cams[0].width;
    a->H = cams[0].height;
    a->tiles_x = (a->W + MFA_TILE - 1) / MFA_TILE;
    a->tiles_y = (a->H + MFA_TILE - 1) / MFA_TILE;
    a->st_x = (a->tiles_x + MFA_SUPERTILE - 1) / MFA_SUPERTILE;
    a->st_y = (a->tiles_y + MFA_SUPERTILE - 1) / MFA_SUPERTILE;
    a->out = out;
    a->out_fp16 = prm->out_fp16;
    a->samples = samples;
    // 2 / 3: NEXT-1 variants (gradient skip / transparent-block skip)
    const int shade = (prm->shading == 2 || prm->shading == 3) ? prm->shading : (prm->shading != 0);
    a->tbits = nullptr;
    a->mm0 = m->mm[0];
    a->mm1 = m->mm[1];
    a->mm_n = m->mm[0] * m->mm[1] * m->mm[2];
    void* tscratch = nullptr;
    if (shade == 3 && is_bez(m->layout) && m->mmx && !(field || lights || curv)) {
        const int64_t nmac = (int64_t)m->mm[0] * m->mm[1] * m->mm[2];
        tscratch = scratch_alloc(sizeof(unsigned) * ((nmac + 31) / 32), st);
        if (tscratch) {
            const int64_t nw = (nmac + 31) / 32;
            macro_transparent_kernel<<<(unsigned)std::min<int64_t>((nw + 255) / 256, 2048), 256, 0, st>>>(
                m->mmx, nmac, a->tf, a->tf_n, a->v_lo, a->s_scale, (unsigned*)tscratch);
            a->tbits = (const unsigned*)tscratch;
        }
    }
    cudaError_t e = cudaSuccess;
    bool exhausted = false;
    auto run = [&]() -> cudaError_t {
        if (a->n_units == 0) return cudaSuccess;
        if (a->n_units >= (int64_t)0xffffffffu) return cudaErrorInvalidValue;
        const int slot = acquire_queue_slot(m, st);
        if (slot < 0) {   // every work counter is held by an unfinished launch on another stream
            exhausted = true;
            return cudaErrorNotReady;
        }
        a->queue = m->queue + slot;
        cudaError_t r = cudaMemsetAsync(a->queue, 0, sizeof(unsigned int), st);
        if (r == cudaSuccess)
            r = (field || lights || curv) ? dispatch_render_ext(*a, m->p, m->layout, uni, shade, st)
                                          : dispatch_render_main(*a, m->p, m->layout, uni, shade, st);
        release_queue_slot(m, slot, st);   // also on failure: the slot must not stay pending
        return r;
    };
    if (tiles) {
        if (n_views > kMaxViewsPerLaunch) {
            delete a;
            if (tscratch) cudaFreeAsync(tscratch, st);
            return fail(MFA_ERR_UNSUPPORTED, "tiled render supports at most 64 views per call");
        }
        for (int v = 0; v < n_views; ++v) compute_frame(cams[v], a->frames[v]);
        a->n_views = n_views;
        a->tiles = tiles->tiles;
        a->tile_scatter = tiles->scatter != 0;
        a->n_tiles = tiles->n_tiles;
        a->n_units = tiles->n_tiles * 8;
        a->view_base = 0;
        e = run();
    } else {
        a->tiles = nullptr;
        a->tile_scatter = 0;
        a->n_tiles = 0;
        for (int v0 = 0; v0 < n_views && e == cudaSuccess; v0 += kMaxViewsPerLaunch) {
            const int nv = std::min(kMaxViewsPerLaunch, n_views - v0);
            for (int v = 0; v < nv; ++v) compute_frame(cams[v0 + v], a->frames[v]);
            a->n_views = nv;
            a->view_base = v0;
            a->n_units = (int64_t)nv * a->st_x * a->st_y * (MFA_SUPERTILE * MFA_SUPERTILE) * 8;
            e = run();
        }
    }
    delete a;
    if (tscratch) cudaFreeAsync(tscratch, st);
    if (exhausted)
        return fail(MFA_ERR_UNSUPPORTED, "render: more than 256 renders in flight on distinct streams for one model");
    return e == cudaSuccess ? MFA_OK : cuda_fail(e, "render launch");
}

}  // namespace mfa
