// render_kernel instantiated with the extensions (EXT = true): the NEXT-2
// ground truth -- every sample can take its value and/or gradient from the
// analytic function (Eq. 1-2) along exactly the rays, sample
// positions, TF, shading and compositing of mfa_render ("we generate the
// ground truth volume rendering image by computing the value and gradient
// analytically from the synthetic functions for the samples on rays", P:191;
// value-only, gradient-only and overall tests P:193) -- and
// NEXT-4's several directional lights.  The hot path (render.cu,
// EXT = false) carries neither.
#include "render_kernel.cuh"

namespace mfa {

cudaError_t dispatch_render_ext(const RenderArgs& a, int p, int layout, bool uni, int shade, cudaStream_t st) {
    switch (p) {
        case 1: return dispatch_render<1, true>(a, layout, uni, shade, st);
        case 2: return dispatch_render<2, true>(a, layout, uni, shade, st);
        case 3: return dispatch_render<3, true>(a, layout, uni, shade, st);
        case 4: return dispatch_render<4, true>(a, layout, uni, shade, st);
        default: return dispatch_render<5, true>(a, layout, uni, shade, st);
    }
}

}  // namespace mfa
